// generic.cu -- geometry-agnostic kernels: the generic GEMM (any m_b, n_b, M),
// K3 dequant/unpack (bit-exact parity entry points) and the sharded-output
// un-permutation.  All read the unit-major device layout (sfmp_internal.h).
// Paths relative to /root/reference/proj.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstring>

#include "repack.cuh"
#include "sfmp_internal.h"

namespace sfmpk {

namespace {

template <sfmp_dtype DT>
__device__ __forceinline__ float ldx(const void* x, size_t i) {
    if constexpr (DT == SFMP_F32) return __ldg(static_cast<const float*>(x) + i);
    else if constexpr (DT == SFMP_F16)
        return __half2float(__ldg(static_cast<const __half*>(x) + i));
    else
        return __bfloat162float(__ldg(static_cast<const __nv_bfloat16*>(x) + i));
}

// One row segment of one unit: scale/zero widened exactly from fp16
// (fp16.hpp:58-83) and a code reader restating unpack_block (layout.cpp:77-83).
// Two unit layouts (sfmp_internal.h): the SFMPPKD1 order (scales | zeros |
// planes row-major), and the decode GEMV's lane-major order (TR = 128, n_b in
// {128, 256}; repack.cuh) with <= 4-bit groups repacked.
struct RowRef {
    const uint8_t* planes;  // plane region of the unit
    uint32_t bits;
    bool lane_major;
    uint32_t rr;            // row within the unit
    uint64_t plane_bytes;   // (SFMPPKD1 order) TR * n_b / 8
    uint32_t row_off;       // (SFMPPKD1 order) rr * n_b / 8
    float s, z;
    __device__ __forceinline__ uint32_t code(uint32_t jj) const {
        if (lane_major) {
            uint32_t w[8];
            const uint8_t* p = planes + lm_word_off(bits, jj >> 7, rr, (jj >> 5) & 3, 0);
            for (uint32_t i = 0; i < bits; ++i) w[i] = *reinterpret_cast<const uint32_t*>(p + i * 512);
            if (bits <= 4) return rp_code(w, static_cast<int>(bits), static_cast<int>(jj & 31));
            uint32_t c = 0;
            for (uint32_t i = 0; i < bits; ++i) c |= ((w[i] >> (jj & 31)) & 1u) << i;
            return c;
        }
        uint32_t c = 0;
        for (uint32_t i = 0; i < bits; ++i)
            c |= ((planes[i * plane_bytes + row_off + (jj >> 3)] >> (jj & 7)) & 1u) << i;
        return c;
    }
};

__device__ __forceinline__ RowRef row_ref(const UnitGeom& g, uint64_t r, uint32_t bc) {
    const uint64_t u = (r / g.TR) * g.BC + bc;
    const uint64_t d = g.unit_desc[u];
    const uint8_t* base = g.payload + (d & 0xFFFFFFFFFFFFull);
    const uint32_t rr = static_cast<uint32_t>(r % g.TR);
    RowRef ref;
    ref.bits = static_cast<uint32_t>((d >> 48) & 0xF);
    ref.lane_major = g.repacked;
    ref.rr = rr;
    if (g.repacked) {
        const uint32_t so = lm_sz_off(rr);
        ref.s = __half2float(*reinterpret_cast<const __half*>(base + so));
        ref.z = __half2float(*reinterpret_cast<const __half*>(base + so + 2));
        ref.planes = base + 512;
    } else {
        ref.s = __half2float(*reinterpret_cast<const __half*>(base + 2 * rr));
        ref.z = __half2float(*reinterpret_cast<const __half*>(base + 2ull * g.TR + 2 * rr));
        ref.planes = base + 4ull * g.TR;
    }
    ref.plane_bytes = static_cast<uint64_t>(g.TR) * (g.n_b >> 3);
    ref.row_off = rr * (g.n_b >> 3);
    return ref;
}

struct GenParams {
    UnitGeom g;
    const uint32_t* col_perm;
    const uint32_t* out_map;
    const void* x;
    float* y;
    int64_t M;
    uint64_t rows, cols, out_rows;
};

// One warp per reordered row, 8 tokens per pass; dequantised weight
// s*c+z (quantizer.cpp:53) times the gathered activation, f32 accumulate.
template <sfmp_dtype DT>
__global__ void __launch_bounds__(256) generic_kernel(const GenParams p) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= p.rows) return;
    for (int64_t t0 = 0; t0 < p.M; t0 += 8) {
        float acc[8];
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) acc[tt] = 0.f;
        for (uint32_t bc = 0; bc < p.g.BC; ++bc) {
            const RowRef ref = row_ref(p.g, r, bc);
            for (uint32_t j = lane; j < p.g.n_b; j += 32) {
                const float w = __fadd_rn(__fmul_rn(ref.s, static_cast<float>(ref.code(j))), ref.z);
                const uint32_t col = p.col_perm[static_cast<uint64_t>(bc) * p.g.n_b + j];
#pragma unroll
                for (int tt = 0; tt < 8; ++tt)
                    if (t0 + tt < p.M) acc[tt] += w * ldx<DT>(p.x, (t0 + tt) * p.cols + col);
            }
        }
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
            float v = acc[tt];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && t0 + tt < p.M) p.y[(t0 + tt) * p.out_rows + p.out_map[r]] = v;
        }
    }
}

// K3: dequantize_model (layout.cpp:316-332): w[orig_row][orig_col] = s*c + z
// with the reference's two f32 roundings (no FMA contraction).
__global__ void dequant_kernel(GenParams p, float* w) {
    const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= p.rows * p.cols) return;
    const uint64_t r = idx / p.cols, j = idx % p.cols;
    const uint32_t bc = static_cast<uint32_t>(j / p.g.n_b), jj = static_cast<uint32_t>(j % p.g.n_b);
    const RowRef ref = row_ref(p.g, r, bc);
    w[static_cast<uint64_t>(p.out_map[r]) * p.cols + p.col_perm[j]] =
        __fadd_rn(__fmul_rn(ref.s, static_cast<float>(ref.code(jj))), ref.z);
}

__global__ void unpack_kernel(GenParams p, uint8_t* codes) {
    const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= p.rows * p.cols) return;
    const uint64_t r = idx / p.cols, j = idx % p.cols;
    const uint32_t bc = static_cast<uint32_t>(j / p.g.n_b), jj = static_cast<uint32_t>(j % p.g.n_b);
    codes[idx] = static_cast<uint8_t>(row_ref(p.g, r, bc).code(jj));
}

// y[t][r] = gathered[g][t][i] with g << 24 | i = inv[r] (inverse gather map):
// CTA (row chunk, token); 4 rows per thread with one 16-byte write.  Writes
// are coalesced and, since every shard's rows are in ascending original
// order, the reads follow G sequential streams.
__global__ void __launch_bounds__(256) unpermute_kernel(const float* __restrict__ gathered, const uint32_t* __restrict__ inv,
                                                        float* __restrict__ y, int64_t M, uint64_t SR, uint64_t rows) {
    const uint64_t t = blockIdx.y;
    const uint64_t r0 = (static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x) * 4;
    if (r0 >= rows) return;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        v[j] = 0.f;
        if (r0 + j < rows) {
            const uint32_t k = __ldg(inv + r0 + j);
            v[j] = __ldg(gathered + ((k >> 24) * M + t) * SR + (k & 0xFFFFFFu));
        }
    }
    float* yr = y + t * rows + r0;
    if (r0 + 4 <= rows && (reinterpret_cast<uintptr_t>(yr) & 15) == 0) {
        *reinterpret_cast<float4*>(yr) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
        for (int j = 0; j < 4 && r0 + j < rows; ++j) yr[j] = v[j];
    }
}

// gemv_block (lutgemm.cpp:87-93): the contribution of block (br, bc) to its
// m_b rows in stored order, from the REORDERED activation; one warp per row.
__global__ void __launch_bounds__(256) gemv_block_kernel(const GenParams p, uint64_t br, uint32_t bc, uint32_t m_b,
                                                         const float* __restrict__ xr, float* __restrict__ out) {
    const uint32_t i = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= m_b) return;
    const RowRef ref = row_ref(p.g, br * m_b + i, bc);
    float acc = 0.f;
    for (uint32_t j = lane; j < p.g.n_b; j += 32)
        acc += __fadd_rn(__fmul_rn(ref.s, static_cast<float>(ref.code(j))), ref.z) * xr[static_cast<uint64_t>(bc) * p.g.n_b + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[i] = acc;
}

GenParams make_params(const DevModel& m) {
    GenParams p{};
    p.g = m.geom();
    p.col_perm = m.d_col_perm;
    p.out_map = m.d_out_map;
    p.rows = m.rows;
    p.cols = m.cols;
    p.out_rows = m.out_rows;
    return p;
}

}  // namespace

cudaError_t launch_generic(const DevModel& m, const void* x, sfmp_dtype dt, int64_t M, float* y,
                           cudaStream_t st) {
    GenParams p = make_params(m);
    p.x = x;
    p.y = y;
    p.M = M;
    const unsigned grid = static_cast<unsigned>((m.rows + 7) / 8);
    note_launch();
    switch (dt) {
        case SFMP_F32: generic_kernel<SFMP_F32><<<grid, 256, 0, st>>>(p); break;
        case SFMP_F16: generic_kernel<SFMP_F16><<<grid, 256, 0, st>>>(p); break;
        default: generic_kernel<SFMP_BF16><<<grid, 256, 0, st>>>(p); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_gemv_block(const DevModel& m, uint64_t block, const float* xr, float* out, cudaStream_t st) {
    GenParams p = make_params(m);
    const uint64_t br = block / m.BC;
    const uint32_t bc = static_cast<uint32_t>(block % m.BC);
    note_launch();
    gemv_block_kernel<<<(m.m_b + 7) / 8, 256, 0, st>>>(p, br, bc, m.m_b, xr, out);
    return cudaGetLastError();
}

cudaError_t launch_dequant(const DevModel& m, float* w, cudaStream_t st) {
    GenParams p = make_params(m);
    const uint64_t n = m.rows * m.cols;
    note_launch();
    dequant_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(p, w);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const DevModel& m, uint8_t* codes, cudaStream_t st) {
    GenParams p = make_params(m);
    const uint64_t n = m.rows * m.cols;
    note_launch();
    unpack_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(p, codes);
    return cudaGetLastError();
}

cudaError_t launch_unpermute_gathered(const DevModel& m, const float* gathered, int64_t M, float* y,
                                      cudaStream_t st) {
    if (M == 0 || m.global_rows == 0) return cudaSuccess;
    if (M > 65535) return cudaErrorInvalidValue;
    note_launch();
    unpermute_kernel<<<dim3(static_cast<unsigned>((m.global_rows + 1023) / 1024), static_cast<unsigned>(M)), 256, 0, st>>>(
        gathered, m.d_gather_inv, y, M, m.shard_rows, m.global_rows);
    return cudaGetLastError();
}

}  // namespace sfmpk
