// sfmp_internal.h -- device model layout and kernel launchers (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sfmp_cuda.h"

namespace sfmpk {

// Kernels launched by this host thread (cumulative): every launcher calls
// note_launch() once per kernel it enqueues (sfmp_launch_count()).
inline thread_local uint64_t t_launches = 0;
inline void note_launch() { ++t_launches; }

// Error message of the last failing call on this host thread (abi.cu).
sfmp_status api_fail(sfmp_status s, const std::string& msg);

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Device layout.  The SFMPPKD1 block payload
// is stored UNIT-MAJOR: a unit is TR consecutive reordered rows x one block
// column (n_b columns), TR = 128 when m_b % 128 == 0, else TR = m_b.  A unit
// is one contiguous span
//     scales[TR] (fp16) | zeros[TR] (fp16) | plane_0 .. plane_{bits-1}
// with each plane TR*n_b/8 bytes (row-major, weight k of a row = bit k%8 of
// byte k/8, as in layout.cpp:58-61).  Units are ordered row-tile-major
// (rt, bc).  The bytes are exactly the SFMPPKD1 bytes; only their order
// changes (when TR == m_b the layout is byte-identical to SFMPPKD1's).
// unit_desc[u] = byte offset of unit u (bits 0-47) | bit-width (bits 48-51).
struct UnitGeom {
    const uint8_t* payload;
    const uint64_t* unit_desc;
    uint32_t TR, n_b, BC;
    bool repacked;  // <= 4-bit units in the decode layout of repack.cuh
};

struct DevModel {
    int device = 0;
    int num_sms = 148;
    uint64_t rows = 0, cols = 0;  // rows = rows held by this (shard) model
    uint32_t m_b = 0, n_b = 0;
    int floor_bits = 0, ceil_bits = 0, mode = 0;
    uint64_t K = 0;  // blocks held
    uint64_t blocks_high = 0;
    double avg_bits = 0;
    uint64_t payload_bytes = 0;
    uint64_t device_bytes = 0;

    uint32_t TR = 0;          // unit rows
    uint32_t RT = 0, BC = 0;  // row tiles, block columns
    std::vector<uint64_t> h_unit_desc;

    uint8_t* d_payload = nullptr;
    uint64_t* d_unit_desc = nullptr;
    uint32_t* d_col_perm = nullptr;  // always present (identity when mode lacks col)
    uint32_t* d_out_map = nullptr;   // local reordered row -> column index of y row
    uint64_t out_rows = 0;           // stride of a y row

    // sharding
    uint32_t shard = 0, num_shards = 1;
    uint64_t global_rows = 0;
    uint64_t shard_rows = 0;
    uint32_t* d_gather_map = nullptr;  // [num_shards*shard_rows] -> original row (or ~0 pad)
    uint32_t* d_gather_inv = nullptr;  // [global_rows] original row -> shard << 24 | local position

    // K2 row-tile layout (gemm_tcgen05.cu): units of 128 output rows x 128
    // reordered columns, per-row bit-widths, gl_row_tiles (even) x cols/128.
    uint8_t* d_gl = nullptr;
    uint64_t* d_gl_off = nullptr;
    uint64_t gl_row_tiles = 0;
    uint64_t gl_bytes = 0;
    uint32_t* d_xslot = nullptr;  // [cols] col_perm in the K order of the GEMM B operand

    // K6 LUT comparison kernel (lut.cu): the SFMPPKD1 block payloads as stored,
    // each block 16-byte aligned; built only with SFMP_MODEL_LUT_LAYOUT
    uint8_t* d_lut = nullptr;
    uint64_t* d_lut_off = nullptr;
    uint8_t* d_lut_bits = nullptr;

    bool gemv_ok = false;
    bool gemm_ok = false;

    float* d_ws = nullptr;  // default workspace
    size_t ws_bytes = 0;
    // staging for the host-buffer entry point (sfmp_gemm_host)
    std::mutex host_mu;
    uint8_t* d_host_stage = nullptr;
    size_t host_stage_bytes = 0;
    std::vector<void*> allocs;

    UnitGeom geom() const { return UnitGeom{d_payload, d_unit_desc, TR, n_b, BC, gemv_ok}; }
};

// RMSNorm fused into the activation pre-pass (prenorm.cuh); on = 0: identity.
struct PreNorm {
    const void* gamma = nullptr;  // [cols] norm weight (nullptr: 1)
    int gdt = 0;                  // its sfmp_dtype
    float eps = 0.f;
    int on = 0;
};

// Launchers (return cudaError_t of the launch).
cudaError_t launch_gemv(const DevModel& m, const void* x, sfmp_dtype dt, int M, float* y,
                        float* ws, cudaStream_t st, const PreNorm* norm = nullptr);
size_t gemv_workspace_bytes(const DevModel& m, int M);
// Several independent linears in one xprep + one GEMV launch (same n_b, floor bits, device).
bool gemv_groupable(const DevModel& a, const DevModel& b);
cudaError_t launch_gemv_group(const DevModel* const* ms, const void* const* xs, float* const* ys, uint8_t* const* wss,
                              const int* Ms, int n, sfmp_dtype dt, cudaStream_t st, bool overlap_prev,
                              const PreNorm* norms = nullptr);
int gemv_ctas_per_sm(int NT);
// Two pipeline stages of the widest unit + activation record fit in shared memory.
bool gemv_feasible(const DevModel& m);

cudaError_t launch_generic(const DevModel& m, const void* x, sfmp_dtype dt, int64_t M, float* y,
                           cudaStream_t st);
cudaError_t launch_dequant(const DevModel& m, float* w, cudaStream_t st);
bool lut_supported(const DevModel& m);
cudaError_t launch_lut(const DevModel& m, const float* x, int64_t M, float* y, cudaStream_t st);
cudaError_t launch_gemv_block(const DevModel& m, uint64_t block, const float* xr, float* out, cudaStream_t st);
cudaError_t launch_unpack(const DevModel& m, uint8_t* codes, cudaStream_t st);
cudaError_t launch_unpermute_gathered(const DevModel& m, const float* gathered, int64_t M,
                                      float* y, cudaStream_t st);

// Device-side ingest (ingest.cu): the unit-major lane-major layout and the
// row-tile layout built from the blocks as stored.
cudaError_t device_unit_layout(const uint8_t* raw, const uint64_t* raw_off, const uint8_t* bits, uint32_t m_b,
                               uint32_t n_b, uint32_t BC, uint32_t units, const uint64_t* unit_desc, uint8_t* dst,
                               cudaStream_t st);
cudaError_t device_tile_layout(const uint8_t* raw, const uint64_t* raw_off, const uint8_t* bits, uint32_t m_b,
                               uint32_t n_b, uint32_t BC, const uint32_t* inv, const uint64_t* woff, uint64_t tiles,
                               uint32_t KC, int F, uint8_t* dst, cudaStream_t st);

// K2 prefill GEMM (tcgen05)
bool gemm_supported(const DevModel& m);
std::vector<uint32_t> gemm_slot_table(const std::vector<uint32_t>& col_perm);
bool build_gemm_layout(DevModel& d, const std::vector<uint8_t>& payload, const std::vector<uint32_t>& out_map,
                       std::vector<uint8_t>& wl, std::vector<uint64_t>& woff);
size_t gemm_workspace_bytes(const DevModel& m, int64_t M);
cudaError_t launch_gemm(const DevModel& m, const void* x, sfmp_dtype dt, int64_t M, float* y,
                        void* ws, cudaStream_t st, const PreNorm* norm = nullptr);

}  // namespace sfmpk
