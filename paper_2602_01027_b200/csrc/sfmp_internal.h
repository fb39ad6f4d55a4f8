// sfmp_internal.h -- device model layout and kernel launchers (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/sfmp_cuda.h"

namespace sfmpk {

// Work schedule of the decode GEMV (K1): units are (row tile, block column)
// pairs in row-tile-major order; CTA c owns units [cta_begin[c], cta_begin[c+1]).
// A row tile touched by several CTAs is reduced by the last arriving CTA in
// fixed segment order (deterministic split-K).
struct GemvSchedule {
    int tile_rows = 128;  // TR
    int row_tiles = 0;    // RT
    int block_cols = 0;   // BC
    int grid = 0;         // G
    int total_slots = 0;  // partial-sum slots (segments of multi-CTA row tiles)
    int* d_cta_begin = nullptr;  // G+1
    int* d_rt_nseg = nullptr;    // RT
    int* d_rt_slot = nullptr;    // RT: first slot of the tile
    int* d_rt_first = nullptr;   // RT: first CTA touching the tile
    unsigned* d_counters = nullptr;  // RT arrival counters (self-resetting)
};

// Device-resident model.  The block payload region of the SFMPPKD1 stream is
// uploaded verbatim (scales | zeros | planes per block, block-row-major).
struct DevModel {
    int device = 0;
    int num_sms = 148;
    uint64_t rows = 0, cols = 0;  // rows = rows held by this (shard) model
    uint32_t m_b = 0, n_b = 0;
    int floor_bits = 0, ceil_bits = 0, mode = 0;
    uint64_t K = 0;
    uint64_t blocks_high = 0;
    double avg_bits = 0;
    uint64_t payload_bytes = 0;
    uint64_t device_bytes = 0;
    std::vector<uint8_t> h_bits;
    std::vector<uint64_t> h_off;  // relative to payload start

    uint8_t* d_payload = nullptr;
    uint64_t* d_off = nullptr;
    uint8_t* d_bits = nullptr;
    uint32_t* d_col_perm = nullptr;  // always present (identity when mode lacks col)
    uint32_t* d_out_map = nullptr;   // local reordered row -> column index of y row
    uint64_t out_rows = 0;           // stride of a y row

    // sharding
    uint32_t shard = 0, num_shards = 1;
    uint64_t global_rows = 0;
    uint64_t shard_rows = 0;
    uint32_t* d_gather_map = nullptr;  // [num_shards*shard_rows] -> original row (or ~0 pad)

    GemvSchedule gemv;
    bool gemv_ok = false;
    bool gemm_ok = false;

    float* d_ws = nullptr;  // default workspace
    size_t ws_bytes = 0;
    std::vector<void*> allocs;
};

// Launchers (return cudaError_t of the launch).
cudaError_t launch_gemv(const DevModel& m, const void* x, sfmp_dtype dt, int M, float* y,
                        float* ws, cudaStream_t st);
size_t gemv_workspace_bytes(const DevModel& m, int M);
int gemv_ctas_per_sm();

cudaError_t launch_generic(const DevModel& m, const void* x, sfmp_dtype dt, int64_t M, float* y,
                           cudaStream_t st);
cudaError_t launch_dequant(const DevModel& m, const uint32_t* d_row_orig, float* w,
                           cudaStream_t st);
cudaError_t launch_unpack(const DevModel& m, uint8_t* codes, cudaStream_t st);
cudaError_t launch_unpermute_gathered(const DevModel& m, const float* gathered, int64_t M,
                                      float* y, cudaStream_t st);

// K2 prefill GEMM (tcgen05)
bool gemm_supported(const DevModel& m);
size_t gemm_workspace_bytes(const DevModel& m, int64_t M);
cudaError_t launch_gemm(const DevModel& m, const void* x, sfmp_dtype dt, int64_t M, float* y,
                        void* ws, cudaStream_t st);

}  // namespace sfmpk
