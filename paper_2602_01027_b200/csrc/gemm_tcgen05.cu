// gemm_tcgen05.cu -- K2: prefill GEMM (M > 16) for SFMP block-wise
// mixed-precision weights on the 5th-generation tensor cores (tcgen05/TMEM).
//
// Replaces sfmp::gemv looped per token (lutgemm.cpp:95-135) for
// large token counts.  Result semantics: y[t] = dequantize_model(W) . x[t]
// with x in the ORIGINAL column order (col_perm gather, reorder.cpp:103-111)
// and y in the ORIGINAL row order (row_perm scatter, reorder.cpp:113-121).
// Paths relative to /root/reference/proj.
//
// Design:
//  * Weights use a second device layout built at upload ("row-tile layout",
//    build_gemm_layout below): tiles of 128 consecutive OUTPUT rows x 128
//    reordered columns.  Rows keep their own block's bit-width: planes
//    0..floor-1 are stored for all rows, the ceil plane only for the rows
//    whose block is at ceil bits (compact, located by a 128-bit row mask).
//    Because a tile's rows are consecutive output rows, the epilogue writes
//    y with coalesced stores -- the row un-permutation costs nothing.
//  * The pre-pass (xprep_gemm_*) gathers x[t][col_perm[.]], scales each
//    token by a power of two 2^-e_t (max|x_t| -> [2^14, 2^15): no finite
//    input overflows f16), converts to f16 and lays every (token tile,
//    128-column chunk) out as the exact 128-byte-swizzled K-major
//    shared-memory image of the MMA B operand, so the GEMM fetches it with one
//    1-D bulk copy (no tensor map).  The epilogue multiplies back by 2^e_t.
//  * Persistent warp-specialised kernel, one CTA per SM, tile = 128 output
//    rows (MMA M) x N <= 256 tokens (MMA N):
//      warp 0       weight producer (lane 0, cp.async.bulk)
//      warp 1       TMEM allocator + tcgen05.mma issuer (one elected lane)
//      warp 2       X producer (lane 0) -- its own warp: as lane 1 of warp 0 it
//                   stalled behind the weight producer's ring waits (8192x28672
//                   M=32/64: 73.6/74.7 -> 65.7/67.6 us)
//      warps 3-18   epilogue: tcgen05.ld accumulators -> coalesced y stores
//      warps 19-26  dequant (two per TMEM lane quarter, whole chunks in turn):
//                   bit-planes -> codes -> f16(s*c+z) (one exact
//                   HSUB2 + one HFMA2 per weight pair, fp16 s/z as stored)
//                   written straight into TMEM as the MMA A operand
//                   (tcgen05.st), so weights never take a shared-memory trip.
//    TMEM (512 columns): accumulator 256 columns, 4 A buffers x 64 columns.
//  * Schedule: work items (tile, K split), round-robin over the CTAs, tiles
//    in a grouped raster order (tile_coords) for L2 reuse of X and W.  The
//    number of K splits depends on the UNSHARDED matrix shape and M only
//    (k_splits, a cost model over a virtual 148-SM grid), so results are
//    bit-identical on any device and for any shard count; split partials are
//    summed in split order (gemm_reduce_kernel).
//  * Precision: weights are rounded once to f16 (SURVEY §7 hard part 1:
//    f16 dequant stays ~5x inside the 1e-3 bar, bf16 would not); the scaled
//    activations are rounded to f16 (exact for bf16 input); accumulation is
//    f32 in TMEM.  The f16 weight rounding (~2^-12 relative per weight)
//    dominates the error, so f32 input gets no hi/lo split here (unlike K1).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "prenorm.cuh"
#include "ptx.cuh"
#include "sfmp_internal.h"
#include "tc.cuh"
#include "unpack.cuh"

namespace sfmpk {

namespace {

constexpr int kUnitHdr = 528;             // scales[128] | zeros[128] | highmask[4]
constexpr int kPlaneBytes = 128 * 16;     // one plane of a unit
// Tile = 128 output rows (MMA M) x N <= 256 tokens (MMA N).
#ifndef SFMP_DEQ_WARPS
#define SFMP_DEQ_WARPS 8
#endif
#ifndef SFMP_EPI_WARPS
#define SFMP_EPI_WARPS 16
#endif
constexpr int kDeqWarps = SFMP_DEQ_WARPS;  // dequant warps: 4 TMEM lane quarters x kKS K-splits
constexpr int kKS = kDeqWarps / 4;        // K splits of a 128-column unit among dequant warps
// SFMP_DEQ_IL: the kKS dequant warps of a TMEM lane quarter take whole chunks in turn
// (chunk i -> group i % kKS) instead of splitting every chunk's K among them
#ifndef SFMP_DEQ_IL
#define SFMP_DEQ_IL 1
#endif
constexpr int kWords = SFMP_DEQ_IL ? 4 : 4 / kKS;  // 32-weight words per dequant thread per unit
constexpr int kDeqPerChunk = SFMP_DEQ_IL ? 4 : kDeqWarps;  // dequant warps that handle one chunk
constexpr int kEpiWarps = SFMP_EPI_WARPS;  // epilogue warps: 4 lane quarters x column groups
// SFMP_XPROD_WARP: the X producer runs in its own warp (warp 2) instead of
// lane 1 of the weight producer's warp
#ifndef SFMP_XPROD_WARP
#define SFMP_XPROD_WARP 1
#endif
constexpr int kXW = SFMP_XPROD_WARP;
// SFMP_DEQ_PIPE (experiment, off): a dequant warp waits for its previous chunk's tcgen05.st after
// this chunk's math (measured: M=32 -1.5 us, q_proj M=2048 +1.7 us -- STTM latency is not the limiter)
#ifndef SFMP_DEQ_PIPE
#define SFMP_DEQ_PIPE 0
#endif
// SFMP_EPI_NAMEDBAR: one epilogue warp polls the accumulator barrier, the rest wait on a named barrier
#ifndef SFMP_EPI_NAMEDBAR
#define SFMP_EPI_NAMEDBAR 1
#endif
// SFMP_PROD_SPIN: the producers and dequant warps poll without a suspend hint
#ifndef SFMP_PROD_SPIN
#define SFMP_PROD_SPIN 1
#endif
__device__ __forceinline__ void role_wait(uint64_t* bar, uint32_t parity, uint32_t ns) {
    if (SFMP_PROD_SPIN) mbar_wait(bar, parity);
    else mbar_wait_sleep(bar, parity, ns);
}
constexpr int kEpi0 = 2 + kXW;             // first epilogue warp
constexpr int kThreads = (kEpi0 + kEpiWarps + kDeqWarps) * 32;
constexpr int kMaxN = 256;                // tokens per tile
constexpr int kTmemCols = 512;
constexpr int kAccCol = 0;                // accumulator: columns [0, N)
constexpr int kACol = 256;                // A buffer ab at kACol + ab*64 (128 f16 of K per row)
constexpr int kNA = 4;                    // A buffers
#ifndef SFMP_SX_MAX
#define SFMP_SX_MAX 8                     // X ring stages (64-column atoms), at most
#endif
#ifndef SFMP_SW_MAX
#define SFMP_SW_MAX 8                     // weight ring stages (units), at most
#endif
constexpr int kSmemLimit = 227 * 1024;
#ifndef SFMP_XPREP_WARP
#define SFMP_XPREP_WARP 1  // warp-per-token prefill pre-pass (0: CTA-per-token, experiment builds)
#endif

struct GemmParams {
    const uint8_t* wl;       // row-tile layout payload
    const uint64_t* woff;    // [RT2*KC + 1] unit byte offsets
    const uint8_t* xs;       // [TT][KC][2][N][128 B] swizzled f16 X
    const float* ysc;        // [TT*N] per-token output scale 2^e_t (pre-pass)
    float* y;
    int M, N, TT, KC, RT;    // tokens, tokens/tile, token tiles, 128-col chunks, row tiles
    uint64_t out_rows;
    int floor_bits, has_extra;
    int SX, SW;              // X / W ring stages
    int ks;                  // K splits per tile (a function of the matrix shape and M alone)
    int GT;                  // token tiles per raster group (tile order, L2 reuse of X)
    int items;               // tiles * ks
    float* part;             // [items][N][128] f32 split-K partial tiles (ks > 1)
    uint32_t stage_w;        // W stage bytes (one unit)
    uint32_t idesc;
};

// x[t][col_perm[...]] -> f16, in the K order of the unpacked A operand:
// slot s of a 128-column chunk holds reordered column 32w + 4h + a + 16e
// with w = s/32, p = s%32, j = p/2 = 4a + h, e = p%2 (unpack_word register
// order: H[4a+h] = weights (4h+a, 4h+a+16) of the word, low half first).
__host__ __device__ __forceinline__ int slot_col(int s) {
    const int w = s >> 5, p = s & 31, j = p >> 1, e = p & 1;
    return 32 * w + 4 * (j & 3) + (j >> 2) + 16 * e;
}

template <sfmp_dtype DT>
__device__ __forceinline__ float x_as_float(std::conditional_t<DT == SFMP_F32, float, uint16_t> v) {
    if constexpr (DT == SFMP_F32) return v;
    else if constexpr (DT == SFMP_F16) return __half2float(__ushort_as_half(v));
    else return __bfloat162float(__ushort_as_bfloat16(v));
}

// Per-token power-of-two scale (as the decode pre-pass, gemv_tc.cu): e such
// that max|x_t| * 2^-e lies in [2^14, 2^15), so no finite input overflows
// f16; 0 for a zero or non-finite row.  f16 input is not scaled.
__device__ __forceinline__ int token_exp(float amax) {
    if (!(amax > 0.f) || !isfinite(amax)) return 0;
    const int e = ilogbf(amax) - 14;
    return e < -110 ? -110 : (e > 110 ? 110 : e);
}
__device__ __forceinline__ float block_max(float m, float* red) {
    const int NW = static_cast<int>(blockDim.x >> 5);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __syncthreads();  // red[] free (previous use finished)
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = 0.f;
    for (int w = 0; w < NW; ++w) m = fmaxf(m, red[w]);
    return m;
}

// Persistent pre-pass (cols < 65536): each CTA keeps the slot table as u16 in
// shared memory (loaded once, instead of once per token) and streams its
// tokens' x rows through two shared buffers with 1-D bulk copies, so the next
// row lands while the current one is gathered into the swizzled B image.
// Tokens M..TT*N-1 of the last tile are written as zeros.
template <sfmp_dtype DT>
__global__ void __launch_bounds__(512) xprep_gemm_rows_kernel(const void* __restrict__ x,
                                                              const uint32_t* __restrict__ xslot,
                                                              uint8_t* __restrict__ xs, float* __restrict__ ysc, int M,
                                                              int N, int KC, int cols, int Mpad, const PreNorm norm) {
    using T = std::conditional_t<DT == SFMP_F32, float, uint16_t>;
    extern __shared__ __align__(16) uint8_t xsm[];
    __shared__ float red[16];
    pdl_launch_dependents();
    uint64_t* bar = reinterpret_cast<uint64_t*>(xsm);            // [2] row buffer full
    uint16_t* idx = reinterpret_cast<uint16_t*>(xsm + 16);        // [cols] slot table
    const uint32_t row_bytes = static_cast<uint32_t>(cols) * sizeof(T);
    uint8_t* rowbuf = xsm + 16 + ((static_cast<size_t>(cols) * 2 + 15) / 16) * 16;  // [2][row_bytes]
    const int G = gridDim.x;
    auto row_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * G; };  // k-th token of this CTA
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        const uint64_t pol = policy_evict_first();
        for (int k = 0; k < 2; ++k) {
            const int t = row_of(k);
            if (t < M) {
                mbar_arrive_expect_tx(&bar[k], row_bytes);
                bulk_g2s(rowbuf + k * static_cast<size_t>(row_bytes),
                         static_cast<const uint8_t*>(x) + static_cast<size_t>(t) * row_bytes, row_bytes, &bar[k], pol);
            }
        }
    }
    for (int i = threadIdx.x; i < cols / 4; i += blockDim.x) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(xslot) + i);
        reinterpret_cast<uint2*>(idx)[i] = make_uint2(v.x | (v.y << 16), v.z | (v.w << 16));
    }
    __syncthreads();
    for (int k = 0;; ++k) {
        const int t = row_of(k);
        if (t >= Mpad) break;
        const int buf = k & 1;
        const int tt = t / N, r = t - tt * N;
        uint8_t* dst = xs + static_cast<size_t>(tt) * KC * 2 * N * 128 + r * 128;
        const T* xr = reinterpret_cast<const T*>(rowbuf + buf * static_cast<size_t>(row_bytes));
        if (t < M) mbar_wait(&bar[buf], static_cast<uint32_t>(k >> 1) & 1u);
        float sc = 1.f, inv = 1.f;  // inv: fused RMSNorm (prenorm.cuh)
        if (DT != SFMP_F16 || norm.on) {
            float m = 0.f;
            if (norm.on) {
                inv = row_inv_rms([&](int i) { return t < M ? x_as_float<DT>(xr[i]) : 0.f; }, cols, norm.eps, red);
                if (t < M)
                    for (int i = threadIdx.x; i < cols; i += blockDim.x)
                        m = fmaxf(m, fabsf(x_as_float<DT>(xr[i]) * gamma_at(norm, i)));
                m = block_max(m, red) * inv;
            } else {
                if (t < M)
                    for (int i = threadIdx.x; i < cols; i += blockDim.x) m = fmaxf(m, fabsf(x_as_float<DT>(xr[i])));
                m = block_max(m, red);
            }
            const int e = token_exp(m);
            sc = ldexpf(1.f, -e);
            if (threadIdx.x == 0) ysc[t] = t < M ? ldexpf(1.f, e) : 0.f;
        } else {
            if (threadIdx.x == 0) ysc[t] = t < M ? 1.f : 0.f;
        }
        for (int c = threadIdx.x; c < KC * 16; c += blockDim.x) {
            const int kc = c >> 4, a = (c >> 3) & 1, j = c & 7;
            uint4 out = make_uint4(0u, 0u, 0u, 0u);
            if (t < M) {
                const uint4 ii = *reinterpret_cast<const uint4*>(idx + kc * 128 + 64 * a + 8 * j);
                const uint32_t iv[4] = {ii.x, ii.y, ii.z, ii.w};
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t clo = iv[e] & 0xFFFFu, chi = iv[e] >> 16;
                    const T lo = xr[clo], hi = xr[chi];
                    if (DT == SFMP_F16 && !norm.on) {
                        o[e] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
                    } else if (norm.on) {
                        o[e] = h2_as_u32(__floats2half2_rn((x_as_float<DT>(lo) * inv) * gamma_at(norm, clo) * sc,
                                                           (x_as_float<DT>(hi) * inv) * gamma_at(norm, chi) * sc));
                    } else {
                        o[e] = h2_as_u32(__floats2half2_rn(x_as_float<DT>(lo) * sc, x_as_float<DT>(hi) * sc));
                    }
                }
                out = make_uint4(o[0], o[1], o[2], o[3]);
            }
            *reinterpret_cast<uint4*>(dst + (static_cast<size_t>(kc) * 2 + a) * N * 128 + ((j ^ (r & 7)) << 4)) = out;
        }
        __syncthreads();  // buffer `buf` is free again
        if (threadIdx.x == 0) {
            const int t2 = row_of(k + 2);
            if (t2 < M) {
                mbar_arrive_expect_tx(&bar[buf], row_bytes);
                bulk_g2s(rowbuf + buf * static_cast<size_t>(row_bytes),
                         static_cast<const uint8_t*>(x) + static_cast<size_t>(t2) * row_bytes, row_bytes, &bar[buf],
                         policy_evict_first());
            }
        }
    }
}

// Warp-per-token pre-pass (rows up to ~12K columns): NW warps per CTA share the
// u16 slot table in shared memory; each warp owns one row buffer, bulk-copies
// its token's x row into it and does the absmax (and fused norm), scaling,
// conversion and swizzled gather alone -- no CTA barrier per token, so up to
// 148 x NW tokens are in flight at once (the CTA-per-token pre-pass above
// serialises a few tokens per CTA behind two row buffers: 17 us for 2048 x
// 4096 bf16, ~3x its HBM time).  Tokens M..Mpad-1 are written as zeros.
template <sfmp_dtype DT>
__global__ void __launch_bounds__(512) xprep_gemm_warp_kernel(const void* __restrict__ x,
                                                              const uint32_t* __restrict__ xslot,
                                                              uint8_t* __restrict__ xs, float* __restrict__ ysc, int M,
                                                              int N, int KC, int cols, int Mpad, const PreNorm norm) {
    using T = std::conditional_t<DT == SFMP_F32, float, uint16_t>;
    constexpr int kPerVec = 16 / sizeof(T);  // x elements per 16-byte shared load
    extern __shared__ __align__(16) uint8_t xsm[];
    pdl_launch_dependents();
    const int NW = static_cast<int>(blockDim.x >> 5), w = static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(xsm);                      // [NW]
    uint16_t* idx = reinterpret_cast<uint16_t*>(xsm + 8 * 16);             // [cols] slot table (<= 16 warps)
    const uint32_t row_bytes = static_cast<uint32_t>(cols) * sizeof(T);
    uint8_t* rowbuf = xsm + 8 * 16 + ((static_cast<size_t>(cols) * 2 + 15) / 16) * 16 + static_cast<size_t>(w) * row_bytes;
    const T* xr = reinterpret_cast<const T*>(rowbuf);
    const int stride = static_cast<int>(gridDim.x) * NW;
    int t = static_cast<int>(blockIdx.x) * NW + w;
    const uint32_t bar_a = smem_u32(&bar[w]);
    if (lane == 0) {
        mbar_init(&bar[w], 1);
        fence_mbar_init();
        if (t < M) {
            mbar_arrive_expect_tx(&bar[w], row_bytes);
            bulk_g2s(rowbuf, static_cast<const uint8_t*>(x) + static_cast<size_t>(t) * row_bytes, row_bytes, &bar[w],
                     policy_evict_first());
        }
    }
    for (int i = threadIdx.x; i < cols / 4; i += blockDim.x) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(xslot) + i);
        reinterpret_cast<uint2*>(idx)[i] = make_uint2(v.x | (v.y << 16), v.z | (v.w << 16));
    }
    __syncthreads();  // slot table and barrier init visible
    (void)bar_a;
    for (int k = 0; t < Mpad; ++k, t += stride) {
        const int tt = t / N, r = t - tt * N;
        uint8_t* dst = xs + static_cast<size_t>(tt) * KC * 2 * N * 128 + r * 128;
        const bool live = t < M;
        if (live) mbar_wait(&bar[w], static_cast<uint32_t>(k) & 1u);
        float sc = 1.f, inv = 1.f;
        if (live && (DT != SFMP_F16 || norm.on)) {
            float m = 0.f, ss = 0.f;
            for (int v = lane; v < cols / kPerVec; v += 32) {
                const uint4 q = *reinterpret_cast<const uint4*>(rowbuf + 16 * v);
                const T* e = reinterpret_cast<const T*>(&q);
#pragma unroll
                for (int i = 0; i < kPerVec; ++i) {
                    const float f = x_as_float<DT>(e[i]);
                    if (norm.on) {
                        ss = fmaf(f, f, ss);
                        m = fmaxf(m, fabsf(f * gamma_at(norm, kPerVec * v + i)));
                    } else {
                        m = fmaxf(m, fabsf(f));
                    }
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                ss += __shfl_xor_sync(0xffffffffu, ss, o);
            }
            if (norm.on) {
                inv = 1.f / sqrtf(ss / static_cast<float>(cols) + norm.eps);
                m *= inv;
            }
            const int e = token_exp(m);
            sc = ldexpf(1.f, -e);
            if (lane == 0) ysc[t] = ldexpf(1.f, e);
        } else if (lane == 0) {
            ysc[t] = live ? 1.f : 0.f;
        }
        for (int c = lane; c < KC * 16; c += 32) {
            const int kc = c >> 4, a = (c >> 3) & 1, j = c & 7;
            uint4 out = make_uint4(0u, 0u, 0u, 0u);
            if (live) {
                const uint4 ii = *reinterpret_cast<const uint4*>(idx + kc * 128 + 64 * a + 8 * j);
                const uint32_t iv[4] = {ii.x, ii.y, ii.z, ii.w};
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t clo = iv[e] & 0xFFFFu, chi = iv[e] >> 16;
                    const T lo = xr[clo], hi = xr[chi];
                    if (DT == SFMP_F16 && !norm.on) {
                        o[e] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
                    } else if (norm.on) {
                        o[e] = h2_as_u32(__floats2half2_rn((x_as_float<DT>(lo) * inv) * gamma_at(norm, clo) * sc,
                                                           (x_as_float<DT>(hi) * inv) * gamma_at(norm, chi) * sc));
                    } else {
                        o[e] = h2_as_u32(__floats2half2_rn(x_as_float<DT>(lo) * sc, x_as_float<DT>(hi) * sc));
                    }
                }
                out = make_uint4(o[0], o[1], o[2], o[3]);
            }
            *reinterpret_cast<uint4*>(dst + (static_cast<size_t>(kc) * 2 + a) * N * 128 + ((j ^ (r & 7)) << 4)) = out;
        }
        __syncwarp();  // the warp's reads of its row buffer are done
        if (lane == 0 && t + stride < M) {
            fence_proxy_async();  // generic-proxy reads before the async-proxy overwrite
            mbar_arrive_expect_tx(&bar[w], row_bytes);
            bulk_g2s(rowbuf, static_cast<const uint8_t*>(x) + static_cast<size_t>(t + stride) * row_bytes, row_bytes,
                     &bar[w], policy_evict_first());
        }
    }
}

// One CTA per token (grid-stride), for wide rows or misaligned x: the x row
// is staged in shared memory as f16 (scaled), then every 16-byte chunk of the
// swizzled B image is gathered from shared memory through the slot table
// xslot (xslot[kc*128 + s] = col_perm[kc*128 + slot_col(s)], built at upload).
// Tokens M..TT*N-1 of the last tile are written as zeros.
template <sfmp_dtype DT>
__global__ void __launch_bounds__(1024) xprep_gemm_kernel(const void* __restrict__ x, const uint32_t* __restrict__ xslot,
                                                         uint8_t* __restrict__ xs, float* __restrict__ ysc, int M, int N,
                                                         int KC, int cols, int Mpad, const PreNorm norm) {
    using T = std::conditional_t<DT == SFMP_F32, float, uint16_t>;
    extern __shared__ __align__(16) __half xrow[];
    __shared__ float red[32];
    pdl_launch_dependents();
    for (int t = blockIdx.x; t < Mpad; t += gridDim.x) {
        const int tt = t / N, r = t - tt * N;
        uint8_t* dst = xs + static_cast<size_t>(tt) * KC * 2 * N * 128 + r * 128;
        if (t < M) {
            const T* src = static_cast<const T*>(x) + static_cast<size_t>(t) * cols;
            float sc = 1.f, inv = 1.f;  // inv: fused RMSNorm (prenorm.cuh)
            if (DT != SFMP_F16 || norm.on) {
                float m = 0.f;
                if (norm.on) {
                    inv = row_inv_rms([&](int i) { return x_as_float<DT>(src[i]); }, cols, norm.eps, red);
                    for (int i = threadIdx.x; i < cols; i += blockDim.x)
                        m = fmaxf(m, fabsf(x_as_float<DT>(src[i]) * gamma_at(norm, i)));
                    m = block_max(m, red) * inv;
                } else {
                    for (int i = threadIdx.x; i < cols; i += blockDim.x) m = fmaxf(m, fabsf(x_as_float<DT>(src[i])));
                    m = block_max(m, red);
                }
                const int e = token_exp(m);
                sc = ldexpf(1.f, -e);
                if (threadIdx.x == 0) ysc[t] = ldexpf(1.f, e);
            } else if (threadIdx.x == 0) {
                ysc[t] = 1.f;
            }
            for (int i = threadIdx.x; i < cols; i += blockDim.x) {
                if (DT == SFMP_F16 && !norm.on) xrow[i] = __ushort_as_half(src[i]);
                else if (norm.on) xrow[i] = __float2half_rn((x_as_float<DT>(src[i]) * inv) * gamma_at(norm, i) * sc);
                else xrow[i] = __float2half_rn(x_as_float<DT>(src[i]) * sc);
            }
            __syncthreads();
        } else if (threadIdx.x == 0) {
            ysc[t] = 0.f;
        }
        for (int c = threadIdx.x; c < KC * 16; c += blockDim.x) {
            const int kc = c >> 4, a = (c >> 3) & 1, j = c & 7;
            uint4 out = make_uint4(0u, 0u, 0u, 0u);
            if (t < M) {
                const uint4* ip = reinterpret_cast<const uint4*>(xslot + kc * 128 + 64 * a + 8 * j);
                const uint4 i0 = __ldg(ip), i1 = __ldg(ip + 1);
                const unsigned short* xr = reinterpret_cast<const unsigned short*>(xrow);
                out.x = static_cast<uint32_t>(xr[i0.x]) | (static_cast<uint32_t>(xr[i0.y]) << 16);
                out.y = static_cast<uint32_t>(xr[i0.z]) | (static_cast<uint32_t>(xr[i0.w]) << 16);
                out.z = static_cast<uint32_t>(xr[i1.x]) | (static_cast<uint32_t>(xr[i1.y]) << 16);
                out.w = static_cast<uint32_t>(xr[i1.z]) | (static_cast<uint32_t>(xr[i1.w]) << 16);
            }
            *reinterpret_cast<uint4*>(dst + (static_cast<size_t>(kc) * 2 + a) * N * 128 + ((j ^ (r & 7)) << 4)) = out;
        }
        __syncthreads();
    }
}

// Tile order (numerics-neutral): groups of GT token tiles; within a group
// the row tiles are outer and the group's token tiles inner, so the ~148
// tiles in flight share a bounded X working set (GT token tiles' images) and
// each weight row tile is read once per group (L2 reuse of both operands).
__host__ __device__ __forceinline__ void tile_coords(const GemmParams& p, int tile, int& rt, int& tt) {
    const int per = p.RT * p.GT;
    const int grp = tile / per;
    const int r = tile - grp * per;
    const int gt = min(p.GT, p.TT - grp * p.GT);
    rt = r / gt;
    tt = grp * p.GT + (r - rt * gt);
}

// Work items of this CTA: items b, b+G, b+2G, ... ; item i = (tile i / ks,
// K split i % ks), split j covering chunks [j*KC/ks, (j+1)*KC/ks).  Every role
// walks the same sequence.
struct GSeg {
    int item, tile, kc0, kc1;
};
__device__ __forceinline__ bool seg_at(const GemmParams& p, int k, GSeg& g) {
    const int item = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
    if (item >= p.items) return false;
    g.item = item;
    g.tile = item / p.ks;
    const int j = item - g.tile * p.ks;
    g.kc0 = j * p.KC / p.ks;
    g.kc1 = (j + 1) * p.KC / p.ks;
    return true;
}

// Split-K fix-up: tile's partials summed in split order (deterministic), times
// the per-token scale.  grid = (N/32, tiles); warp wi handles tokens
// j0 + wi + 4k (k < 8); lane l rows 4l..4l+3 (float4).
__global__ void __launch_bounds__(128) gemm_reduce_kernel(const GemmParams p) {
    pdl_wait();
    const int tile = blockIdx.y;
    int rt, tt;
    tile_coords(p, tile, rt, tt);
    const int N = p.N;
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = blockIdx.x * 32 + wi;
    const size_t pstride = static_cast<size_t>(N) * 128;
    const bool full = blockIdx.x * 32 + 32 <= N;
    float4 acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = 0; c < p.ks; ++c) {  // split order: deterministic
        const float4* src =
            reinterpret_cast<const float4*>(p.part + (static_cast<size_t>(tile) * p.ks + c) * pstride + static_cast<size_t>(j0) * 128) + lane;
        float4 v[8];
        if (full) {  // unconditional loads: all 8 in flight together
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldg(src + k * 4 * 32);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldg(src + (j0 + 4 * k < N ? k : 0) * 4 * 32);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (j0 + 4 * k >= N) v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc[k].x += v[k].x;
            acc[k].y += v[k].y;
            acc[k].z += v[k].z;
            acc[k].w += v[k].w;
        }
    }
    const uint64_t grow = static_cast<uint64_t>(rt) * 128 + 4 * lane;
    const bool vec = (p.out_rows % 4 == 0) && ((reinterpret_cast<uintptr_t>(p.y) & 15) == 0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int j = j0 + 4 * k, t = tt * N + j;
        if (j >= N || t >= p.M) continue;
        const float sc = p.ysc[t];
        const float4 a4 = make_float4(acc[k].x * sc, acc[k].y * sc, acc[k].z * sc, acc[k].w * sc);
        float* yp = p.y + static_cast<size_t>(t) * p.out_rows + grow;
        if (vec && grow + 4 <= p.out_rows) {
            *reinterpret_cast<float4*>(yp) = a4;
        } else {
            const float a[4] = {a4.x, a4.y, a4.z, a4.w};
            for (int e = 0; e < 4; ++e)
                if (grow + e < p.out_rows) yp[e] = a[e];
        }
    }
}

// Dequantise one 32-weight word of this thread's row into 16 f16x2.
template <int NP>
__device__ __forceinline__ void dequant_word(const uint32_t (&p)[NP], __half2 s2, __half2 z2, uint32_t (&H)[16]) {
    unpack_word<NP>(p, H);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        __half2 c = u32_as_h2(H[j]);
        if constexpr (NP <= 4) c = __hsub2(c, u32_as_h2((j & 1) ? 0x54005400u : 0x64006400u));  // exact
        H[j] = h2_as_u32(__hfma2(c, s2, z2));  // f16(s*c + z), one rounding
    }
}

template <int NP>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for the swizzled X stages
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int SX = p.SX, SW = p.SW, N = p.N;
    const uint32_t xstage = static_cast<uint32_t>(N * 128);  // one 64-column swizzle atom of X
    uint8_t* xbuf = smem;
    uint8_t* wbuf = xbuf + static_cast<size_t>(SX) * xstage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbuf + static_cast<size_t>(SW) * p.stage_w);
    uint64_t* xfull = bars;
    uint64_t* xempty = xfull + SX;
    uint64_t* wfull = xempty + SX;
    uint64_t* wempty = wfull + SW;
    uint64_t* afull = wempty + SW;     // [kNA]
    uint64_t* aempty = afull + kNA;    // [kNA]
    uint64_t* accfull = aempty + kNA;  // [1]
    uint64_t* accempty = accfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SX; ++s) {
            mbar_init(&xfull[s], 1);
            mbar_init(&xempty[s], 1);
        }
        for (int s = 0; s < SW; ++s) {
            mbar_init(&wfull[s], 1);
            mbar_init(&wempty[s], kDeqPerChunk);
        }
        for (int a = 0; a < kNA; ++a) {
            mbar_init(&afull[a], kDeqPerChunk);
            mbar_init(&aempty[a], 1);
        }
        mbar_init(accfull, 1);
        mbar_init(accempty, kEpiWarps);
        fence_mbar_init();
        fence_proxy_async();
    }
    if (warp == 1) {
        tc_alloc(smem_u32(tmem_slot), kTmemCols);
        tc_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    // the split-K fix-up (if any) may launch now; it waits for this grid
    pdl_launch_dependents();

    // Work: items (tile, K split), tile -> (rt, tt) by tile_coords, round-robin over the
    // CTAs.  A whole-tile item (ks == 1) stores y; a split item stores its
    // partial tile, summed in split order by gemm_reduce_kernel.
    const int KC = p.KC;

    if (warp == 0 || (kXW && warp == 2)) {
        // ---------------- producers ----------------
        // Lane 0 streams the weight units, lane 1 the X atoms, each gated only
        // by its own ring: the weights never wait for X slots (which free only
        // as MMAs complete), so dequantisation can run ahead.
        const uint64_t pol_w = policy_evict_first();
        if (warp == 0 && lane == 0) {
            int ws = 0, wph = 0;
            GSeg sg;
            for (int k = 0; seg_at(p, k, sg); ++k) {
                int rt, tt_unused;
                tile_coords(p, sg.tile, rt, tt_unused);
                const uint64_t* off0 = p.woff + static_cast<size_t>(rt) * KC + sg.kc0;
                uint64_t a_next = __ldg(off0);
                for (int kc = sg.kc0; kc < sg.kc1; ++kc) {
                    const uint64_t a0 = a_next;
                    a_next = __ldg(off0 + (kc - sg.kc0) + 1);
                    const uint32_t n0 = static_cast<uint32_t>(a_next - a0);
                    role_wait(&wempty[ws], wph ^ 1, 500);
                    mbar_arrive_expect_tx(&wfull[ws], n0);
                    bulk_g2s(wbuf + static_cast<size_t>(ws) * p.stage_w, p.wl + a0, n0, &wfull[ws], pol_w);
                    if (++ws == SW) { ws = 0; wph ^= 1; }
                }
            }
        } else if (kXW ? lane == 0 : lane == 1) {
            int xs = 0, xph = 0;
            pdl_wait();  // X is written by the pre-pass (programmatic dependent launch)
            GSeg sg;
            for (int k = 0; seg_at(p, k, sg); ++k) {
                int rt, tt;
                tile_coords(p, sg.tile, rt, tt);
                for (int kc = sg.kc0; kc < sg.kc1; ++kc) {
                    for (int h = 0; h < 2; ++h) {
                        role_wait(&xempty[xs], xph ^ 1, 200);
                        mbar_arrive_expect_tx(&xfull[xs], xstage);
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                smem_u32(xbuf + static_cast<size_t>(xs) * xstage)),
                            "l"(p.xs + ((static_cast<size_t>(tt) * KC + kc) * 2 + h) * xstage), "r"(xstage),
                            "r"(smem_u32(&xfull[xs]))
                            : "memory");
                        if (++xs == SX) { xs = 0; xph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // The whole warp walks the loop (warp-uniform operands stay in uniform
        // registers, no per-MMA waterfall); one elected lane issues tcgen05.
        int xs = 0, xph = 0, ab = 0, aph = 0, accph = 0;
        const uint32_t idesc = p.idesc;
        GSeg sg;
        for (int k = 0; seg_at(p, k, sg); ++k) {
            mbar_wait(accempty, accph ^ 1);
            tc_fence_after();
            for (int kc = sg.kc0; kc < sg.kc1; ++kc) {
                mbar_wait(&afull[ab], aph);
                tc_fence_after();
                const uint32_t a0 = tbase + kACol + ab * 64;
                for (int h = 0; h < 2; ++h) {
                    mbar_wait(&xfull[xs], xph);
                    tc_fence_after();
                    const uint64_t bdesc = tc_desc_sw128(smem_u32(xbuf + static_cast<size_t>(xs) * xstage));
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            tc_mma_ts(tbase + kAccCol, a0 + (h * 4 + kk) * 8, bdesc + 2 * kk, idesc,
                                      ((kc - sg.kc0) | h | kk) != 0);
                        tc_commit(&xempty[xs]);
                    }
                    __syncwarp();
                    if (++xs == SX) { xs = 0; xph ^= 1; }
                }
                if (elect_one()) tc_commit(&aempty[ab]);
                __syncwarp();
                if (++ab == kNA) { ab = 0; aph ^= 1; }
            }
            if (elect_one()) tc_commit(accfull);
            __syncwarp();
            accph ^= 1;
        }
    } else if (warp < kEpi0 + kEpiWarps) {
        // ---------------- epilogue: TMEM -> registers -> coalesced y rows ----------------
        // kEpiWarps/4 warps per TMEM lane quarter, each owning 256/(kEpiWarps/4)
        // accumulator columns, loaded 32 at a time; the accumulator is
        // released after the last load, so the last stores overlap the next
        // tile's MMAs.
        constexpr int kCols = 256 / (kEpiWarps / 4);
        const int ew = warp - kEpi0, q = warp & 3, cg = ew >> 2;
        int accph = 0;
        GSeg sg;
        for (int k = 0; seg_at(p, k, sg); ++k) {
            int rt, tt;
            tile_coords(p, sg.tile, rt, tt);
            // a whole item of MMAs away: one warp polls, the other epilogue warps
            // block on a named barrier (16 polling warps took ~45 % of the issue
            // slots from the dequant warps at small N, ncu 8192x28672 M=64)
            if (!SFMP_EPI_NAMEDBAR || ew == 0) mbar_wait_sleep(accfull, accph, 200);
            if (SFMP_EPI_NAMEDBAR) named_bar_sync(1, kEpiWarps * 32);
            accph ^= 1;
            tc_fence_after();
            const int c_begin = cg * kCols;
            const int t0 = tt * N + c_begin;
            const uint64_t row = static_cast<uint64_t>(rt) * 128 + q * 32 + lane;
            int lim = min(kCols, min(N - c_begin, p.M - t0));
            // whole-tile item -> y[t][row] * 2^e_t; else the item's partial [t][128 rows]
            const bool full = p.ks == 1;
            float* yp;
            size_t ld;
            if (full) {
                yp = p.y + static_cast<size_t>(t0) * p.out_rows + row;
                ld = p.out_rows;
                if (row >= p.out_rows) lim = 0;
            } else {
                yp = p.part + static_cast<size_t>(sg.item) * (static_cast<size_t>(N) * 128) +
                     static_cast<size_t>(c_begin) * 128 + q * 32 + lane;
                ld = 128;
            }
            // 32 columns at a time (a 64-register array would spill: 832
            // threads leave 72 registers each, and local memory misses L1);
            // the accumulator is released after the last load, before the
            // last chunk's stores
#pragma unroll
            for (int c = 0; c < kCols / 32; ++c) {
                uint32_t v[32];
                if (c_begin + 32 * c < N) {
                    tc_ld_x32(tbase + (static_cast<uint32_t>(q * 32) << 16) + kAccCol + c_begin + 32 * c, v);
                    tc_wait_ld();
                }
                if (c == kCols / 32 - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(accempty);
                }
                float sv = 1.f;
                if (full && 32 * c + lane < lim) sv = __ldg(p.ysc + t0 + 32 * c + lane);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float sj = full ? __shfl_sync(0xffffffffu, sv, j) : 1.f;
                    if (32 * c + j < lim) yp[static_cast<size_t>(32 * c + j) * ld] = __uint_as_float(v[j]) * sj;
                }
            }
        }
    } else {
        // ---------------- dequant: bit-planes -> f16 A operand in TMEM ----------------
        const int dw = warp - kEpi0 - kEpiWarps, q = warp & 3, kh = dw >> 2;
        const int r = q * 32 + lane;  // row within the unit = TMEM lane
        const uint32_t woff = SFMP_DEQ_IL ? 0u : static_cast<uint32_t>(kh * kWords * 4);  // this warp's words in a row
        int cc = 0;  // chunk counter (SFMP_DEQ_IL: this warp's chunks are cc % kKS == kh)
        int ws = 0, wph = 0, ab = 0, aph = 0;
        int pend = -1;  // A buffer whose tcgen05.st are still in flight (SFMP_DEQ_PIPE)
        (void)pend;
        GSeg sg;
        for (int k = 0; seg_at(p, k, sg); ++k) {
            for (int kc = sg.kc0; kc < sg.kc1; ++kc) {
                if (SFMP_DEQ_IL && (cc++ % kKS) != kh) {  // another group's chunk
                    if (++ws == SW) { ws = 0; wph ^= 1; }
                    if (++ab == kNA) { ab = 0; aph ^= 1; }
                    continue;
                }
                role_wait(&wfull[ws], wph, 200);
                const uint32_t u = smem_u32(wbuf + static_cast<size_t>(ws) * p.stage_w);
                const __half2 s2 = __half2half2(__ushort_as_half(lds_u16(u + 2 * r)));
                const __half2 z2 = __half2half2(__ushort_as_half(lds_u16(u + 256 + 2 * r)));
                uint32_t pl[NP][kWords];
                auto ldrow = [&](int i, uint32_t addr) {
                    if constexpr (kWords == 4) {
                        const uint4 v = lds_v4(addr);
                        pl[i][0] = v.x; pl[i][1] = v.y; pl[i][2] = v.z; pl[i][3] = v.w;
                    } else if constexpr (kWords == 2) {
                        const uint2 v = lds_v2(addr);
                        pl[i][0] = v.x; pl[i][1] = v.y;
                    } else {
                        pl[i][0] = lds_u32(addr);
                    }
                };
                if (p.has_extra) {
                    const uint4 mk = lds_v4(u + 512);
                    const uint32_t mw = q == 0 ? mk.x : q == 1 ? mk.y : q == 2 ? mk.z : mk.w;
                    const int before = (q > 0 ? __popc(mk.x) : 0) + (q > 1 ? __popc(mk.y) : 0) + (q > 2 ? __popc(mk.z) : 0);
                    const bool high = (mw >> lane) & 1u;
                    const int rank_h = before + __popc(mw & ((1u << lane) - 1u));
#pragma unroll
                    for (int i = 0; i < NP - 1; ++i) ldrow(i, u + kUnitHdr + i * kPlaneBytes + r * 16 + woff);
                    if (high) {
                        ldrow(NP - 1, u + kUnitHdr + (NP - 1) * kPlaneBytes + rank_h * 16 + woff);
                    } else {
#pragma unroll
                        for (int w = 0; w < kWords; ++w) pl[NP - 1][w] = 0u;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < NP; ++i) ldrow(i, u + kUnitHdr + i * kPlaneBytes + r * 16 + woff);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&wempty[ws]);  // shared-memory reads of this stage are done
                // 4 A buffers let dequant run ahead of the MMA, so waiting for the
                // buffer before the math costs little and keeps registers low
                mbar_wait_sleep(&aempty[ab], aph ^ 1, 300);
                tc_fence_after();
                const uint32_t ta = tbase + (static_cast<uint32_t>(q * 32) << 16) + kACol + ab * 64 + (SFMP_DEQ_IL ? 0 : kh * kWords * 16);
#if SFMP_DEQ_PIPE
                // software-pipelined: this chunk's math overlaps the previous chunk's
                // tcgen05.st, which is waited for (and its A buffer handed to the MMA)
                // only now
                uint32_t H[kWords][16];
#pragma unroll
                for (int w = 0; w < kWords; ++w) {
                    uint32_t pw[NP];
#pragma unroll
                    for (int i = 0; i < NP; ++i) pw[i] = pl[i][w];
                    dequant_word<NP>(pw, s2, z2, H[w]);
                }
                if (pend >= 0) {
                    tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&afull[pend]);
                }
#pragma unroll
                for (int w = 0; w < kWords; ++w) tc_st_x16(ta + w * 16, H[w]);
                pend = ab;
#else
#pragma unroll
                for (int w = 0; w < kWords; ++w) {
                    uint32_t pw[NP];
#pragma unroll
                    for (int i = 0; i < NP; ++i) pw[i] = pl[i][w];
                    uint32_t H[16];
                    dequant_word<NP>(pw, s2, z2, H);
                    tc_st_x16(ta + w * 16, H);
                }
                tc_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&afull[ab]);
#endif
                if (++ws == SW) { ws = 0; wph ^= 1; }
                if (++ab == kNA) { ab = 0; aph ^= 1; }
            }
        }
        if (SFMP_DEQ_PIPE && pend >= 0) {
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&afull[pend]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tc_dealloc(tbase, kTmemCols);
    }
}

int tile_n(int64_t M) { return M >= kMaxN ? kMaxN : static_cast<int>((M + 15) / 16 * 16); }

uint32_t unit_max_bytes(const DevModel& m) {
    const int F = m.floor_bits;
    const bool extra = m.ceil_bits > m.floor_bits;
    return static_cast<uint32_t>(kUnitHdr + F * kPlaneBytes + (extra ? kPlaneBytes : 0));
}

// K splits per tile: a function of the UNSHARDED matrix shape and M only
// (never of the device or the shard), so a row's accumulation order -- and its
// bits -- are the same on any B200, for any shard count.  Chosen by a cost
// model over a virtual 148-SM grid: waves x (chunks per item x MMA time per
// chunk + per-item fill/drain) + the split partials' write/read and the
// reduce launch.  Chunk-time constants: one 128-column chunk = 8 MMAs of
// K=16 at ~130 cycles each for N <= 128 and ~138 at N = 256.  That is NOT
// the MMA cost at small N (tools/mma_bench.cu with an unrolled issue loop:
// 47 / 74 / 138 cycles at N = 64 / 128 / 256) but matches the kernel's measured
// chunk time there (8192x28672, M=64: ~0.5 us per chunk, bound by the
// producer/dequant hand-offs, not the tensor pipe), so the model keeps it.
#ifndef SFMP_KSPLIT_MBPS
#define SFMP_KSPLIT_MBPS 6.0e6
#endif
constexpr int kVirtualSMs = 148;
int k_splits(const DevModel& m, int64_t M) {
    const int64_t N = tile_n(M), TT = (M + N - 1) / N;
    const int64_t KC = static_cast<int64_t>(m.cols / 128);
    const int64_t tiles_g = static_cast<int64_t>((m.global_rows + 127) / 128) * TT;
    const double chunk_us = 8.0 * (N > 128 ? 138.0 : 130.0) / 1900.0, item_us = 1.5;
    int best = 1;
    double best_t = 1e30;
    for (int64_t ks = 1; ks <= std::max<int64_t>(1, std::min<int64_t>(KC / 4, 32)); ++ks) {
        const int64_t items = tiles_g * ks;
        const double waves = static_cast<double>((items + kVirtualSMs - 1) / kVirtualSMs);
        double t = waves * (static_cast<double>((KC + ks - 1) / ks) * chunk_us + item_us);
        if (ks > 1) t += static_cast<double>(items) * N * 128 * 4 * 2 / SFMP_KSPLIT_MBPS + 3.0;  // partials via L2 + reduce
        if (t < best_t * 0.97) {  // prefer fewer splits unless clearly faster
            best_t = t;
            best = static_cast<int>(ks);
        }
    }
    return best;
}

// Token tiles per raster group: the group's X images stay within ~40 MB of L2.
int raster_group(const DevModel& m, int64_t M) {
    const int64_t N = tile_n(M), TT = (M + N - 1) / N;
    const int64_t ximg = N * static_cast<int64_t>(m.cols) * 2;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(TT, (40ll << 20) / std::max<int64_t>(ximg, 1))));
}

template <class F>
void once_per_device(std::once_flag* flags, F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(flags[dev & 63], f);
}

template <int NP>
cudaError_t launch_np(const GemmParams& p, size_t smem, int grid, cudaStream_t st) {
    auto k = gemm_kernel<NP>;
    static std::once_flag fl[64];
    once_per_device(fl, [&] { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit); });
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    note_launch();
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, p);
    if (e != cudaSuccess) return e;
    if (p.ks > 1) {  // split-K fix-up, a programmatic dependent of the GEMM
        cudaLaunchConfig_t rc{};
        rc.gridDim = dim3((p.N + 31) / 32, p.items / p.ks);
        rc.blockDim = dim3(128);
        rc.stream = st;
        rc.attrs = attr;
        rc.numAttrs = 1;
        note_launch();
        e = cudaLaunchKernelEx(&rc, gemm_reduce_kernel, p);
    }
    return e;
}

}  // namespace

// ---------------------------------------------------------------------------
// Upload-time row-tile layout (host).  For output column c of y (0..out_rows)
// the source row is the local reordered row inv[c] (or none: zero weights).
// ---------------------------------------------------------------------------
bool build_gemm_layout(DevModel& d, const std::vector<uint8_t>& payload, const std::vector<uint32_t>& out_map,
                       std::vector<uint8_t>& wl, std::vector<uint64_t>& woff) {
    if (d.n_b % 128 != 0 || d.cols % 128 != 0 || d.out_rows == 0) return false;
    const uint64_t KC = d.cols / 128, RT2 = (d.out_rows + 127) / 128;
    const uint32_t TR = d.TR, nb8 = d.n_b / 8;
    const uint64_t plane_unit = static_cast<uint64_t>(TR) * nb8;
    std::vector<uint32_t> inv(RT2 * 128, 0xFFFFFFFFu);
    for (uint64_t i = 0; i < out_map.size(); ++i)
        if (out_map[i] < inv.size()) inv[out_map[i]] = static_cast<uint32_t>(i);
    const int F = d.floor_bits, C = d.ceil_bits;
    woff.assign(RT2 * KC + 1, 0);
    wl.clear();
    wl.reserve(static_cast<size_t>(RT2 * KC) * (kUnitHdr + (F + 1) * kPlaneBytes / 2));
    std::vector<uint8_t> unit;
    for (uint64_t T = 0; T < RT2; ++T)
        for (uint64_t kc = 0; kc < KC; ++kc) {
            woff[T * KC + kc] = wl.size();
            unit.assign(kUnitHdr + F * kPlaneBytes, 0);
            std::vector<uint8_t> extra;
            const uint64_t bc = kc * 128 / d.n_b, sub = (kc * 128 % d.n_b) / 8;
            for (int r = 0; r < 128; ++r) {
                const uint32_t i = inv[T * 128 + r];
                if (i == 0xFFFFFFFFu) continue;
                const uint64_t u = (i / TR) * d.BC + bc, rr = i % TR;
                const uint64_t desc = d.h_unit_desc[u];
                const uint8_t* base = payload.data() + (desc & 0xFFFFFFFFFFFFull);
                const int bits = static_cast<int>((desc >> 48) & 0xF);
                std::memcpy(&unit[2 * r], base + 2 * rr, 2);
                std::memcpy(&unit[256 + 2 * r], base + 2ull * TR + 2 * rr, 2);
                const uint8_t* planes = base + 4ull * TR + rr * nb8 + sub;
                for (int pi = 0; pi < F; ++pi)
                    std::memcpy(&unit[kUnitHdr + pi * kPlaneBytes + r * 16], planes + pi * plane_unit, 16);
                if (bits > F) {
                    unit[512 + r / 8] |= static_cast<uint8_t>(1u << (r % 8));  // mask words: bit r%32 of word r/32
                    extra.insert(extra.end(), planes + F * plane_unit, planes + F * plane_unit + 16);
                }
            }
            wl.insert(wl.end(), unit.begin(), unit.end());
            wl.insert(wl.end(), extra.begin(), extra.end());
        }
    woff[RT2 * KC] = wl.size();
    d.gl_row_tiles = RT2;
    (void)C;
    return true;
}

std::vector<uint32_t> gemm_slot_table(const std::vector<uint32_t>& col_perm) {
    std::vector<uint32_t> t(col_perm.size());
    for (size_t kc = 0; kc + 128 <= col_perm.size(); kc += 128)
        for (int sl = 0; sl < 128; ++sl) t[kc + sl] = col_perm[kc + slot_col(sl)];
    return t;
}

bool gemm_supported(const DevModel& m) {
    return m.d_gl != nullptr && m.d_xslot != nullptr && m.cols * 2 <= 200ull * 1024 && m.ceil_bits >= 1 && m.ceil_bits <= 8 && m.cols < (1ull << 31);
}

template <sfmp_dtype DT>
void launch_xprep_rows(const void* x, const DevModel& m, uint8_t* xs, float* ysc, const GemmParams& p, int cols, int Mpad,
                       int grid, size_t smem, cudaStream_t st, const PreNorm& norm) {
    static std::once_flag fl[64];
    once_per_device(fl, [] { cudaFuncSetAttribute(xprep_gemm_rows_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
    note_launch();
    xprep_gemm_rows_kernel<DT><<<grid, 512, smem, st>>>(x, m.d_xslot, xs, ysc, p.M, p.N, p.KC, cols, Mpad, norm);
}
template <sfmp_dtype DT>
void launch_xprep_warp(const void* x, const DevModel& m, uint8_t* xs, float* ysc, const GemmParams& p, int cols, int Mpad,
                       int nw, int grid, size_t smem, cudaStream_t st, const PreNorm& norm) {
    static std::once_flag fl[64];
    once_per_device(fl, [] { cudaFuncSetAttribute(xprep_gemm_warp_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit); });
    note_launch();
    xprep_gemm_warp_kernel<DT><<<grid, 32 * nw, smem, st>>>(x, m.d_xslot, xs, ysc, p.M, p.N, p.KC, cols, Mpad, norm);
}
template <sfmp_dtype DT>
void launch_xprep_tok(const void* x, const DevModel& m, uint8_t* xs, float* ysc, const GemmParams& p, int cols, int Mpad,
                      cudaStream_t st, const PreNorm& norm) {
    static std::once_flag fl[64];
    once_per_device(fl, [] {
        cudaFuncSetAttribute(xprep_gemm_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(xprep_gemm_kernel<DT>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    });
    note_launch();
    // 512 threads: the per-token absmax, convert and gather loops need the
    // whole CTA (128 threads per 28672-column row ran at ~150 GB/s)
    xprep_gemm_kernel<DT><<<Mpad, 512, static_cast<size_t>(cols) * 2, st>>>(x, m.d_xslot, xs, ysc, p.M, p.N, p.KC, cols, Mpad,
                                                                           norm);
}

// Workspace: swizzled X images | per-token scales | split-K partial tiles [items][N][128] f32.
size_t gemm_x_bytes(const DevModel& m, int64_t M) {
    const int N = tile_n(M);
    const int64_t TT = (M + N - 1) / N;
    return (static_cast<size_t>(TT) * N * m.cols * 2 + 255) / 256 * 256;
}
size_t gemm_scale_bytes(int64_t M) {
    const int N = tile_n(M);
    const int64_t TT = (M + N - 1) / N;
    return (static_cast<size_t>(TT) * N * 4 + 255) / 256 * 256;
}
size_t gemm_workspace_bytes(const DevModel& m, int64_t M) {
    const int ks = k_splits(m, M);
    const int N = tile_n(M);
    const int64_t TT = (M + N - 1) / N;
    const size_t part = ks > 1 ? static_cast<size_t>(m.gl_row_tiles * TT * ks) * N * 128 * 4 : 0;
    return gemm_x_bytes(m, M) + gemm_scale_bytes(M) + part;
}

cudaError_t launch_gemm(const DevModel& m, const void* x, sfmp_dtype dt, int64_t M, float* y, void* ws,
                        cudaStream_t st, const PreNorm* norm_in) {
    const PreNorm norm = norm_in ? *norm_in : PreNorm{};
    GemmParams p{};
    p.N = tile_n(M);
    p.M = static_cast<int>(M);
    p.TT = static_cast<int>((M + p.N - 1) / p.N);
    p.KC = static_cast<int>(m.cols / 128);
    p.RT = static_cast<int>(m.gl_row_tiles);
    p.wl = m.d_gl;
    p.woff = m.d_gl_off;
    uint8_t* xs = static_cast<uint8_t*>(ws);
    float* ysc = reinterpret_cast<float*>(xs + gemm_x_bytes(m, M));
    p.xs = xs;
    p.ysc = ysc;
    p.part = reinterpret_cast<float*>(xs + gemm_x_bytes(m, M) + gemm_scale_bytes(M));
    p.y = y;
    p.out_rows = m.out_rows;
    p.floor_bits = m.floor_bits;
    p.has_extra = m.ceil_bits > m.floor_bits;
    p.idesc = tc_idesc_f16(128, p.N);
    p.stage_w = (unit_max_bytes(m) + 127) / 128 * 128;
    const uint32_t xstage = static_cast<uint32_t>(p.N) * 128;
    const size_t bar_bytes = 1024;
    // W ring: up to SFMP_SW_MAX units; X ring: as many 64-column atoms as the rest holds (<= SFMP_SX_MAX)
    const size_t avail = kSmemLimit - 1024 - bar_bytes;
    p.SW = SFMP_SW_MAX;
    p.SX = static_cast<int>(std::min<size_t>(SFMP_SX_MAX, (avail - p.SW * p.stage_w) / xstage));
    while (p.SX < 4 && p.SW > 4) {
        --p.SW;
        p.SX = static_cast<int>(std::min<size_t>(SFMP_SX_MAX, (avail - p.SW * p.stage_w) / xstage));
    }
    if (p.SX < 2) {
        p.SW = 2;
        p.SX = static_cast<int>(std::min<size_t>(SFMP_SX_MAX, (avail - p.SW * p.stage_w) / xstage));
    }
    if (SFMP_DEQ_IL) p.SW -= p.SW % kKS;  // a weight stage always meets the same dequant group
    if (p.SX < 2 || p.SW < kKS) return cudaErrorInvalidConfiguration;
    const size_t smem = 1024 + p.SX * xstage + p.SW * p.stage_w + bar_bytes;
    // K4 (prefill flavour): gather + scale + convert + swizzle X
    const int cols = static_cast<int>(m.cols);
    const int Mpad = p.TT * p.N;
    const size_t elem = dt == SFMP_F32 ? 4 : 2;
    // persistent pre-pass when the u16 slot table + two rows fit in one CTA's
    // shared memory (1..4 CTAs per SM)
    const size_t rsm = 16 + (static_cast<size_t>(cols) * 2 + 15) / 16 * 16 + 2 * static_cast<size_t>(cols) * elem;
    const bool rows_ok = cols < 65536 && rsm <= 200 * 1024 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    // warp-per-token pre-pass when >= 8 row buffers fit next to the slot table
    const size_t wtab = 8 * 16 + (static_cast<size_t>(cols) * 2 + 15) / 16 * 16, wrow = static_cast<size_t>(cols) * elem;
    const int nw = static_cast<int>(std::min<size_t>(16, (kSmemLimit - 1024 - wtab) / wrow));
    const size_t wsm = wtab + static_cast<size_t>(std::max(nw, 1)) * wrow;
    const int per_sm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(2048 / (32 * std::max(nw, 1)), (kSmemLimit - 1024) / wsm)));
    // ... and every token gets its own warp (a second round would wait a whole row
    // copy again: 70B q at M=2048, 1924 warps for 2048 tokens, measured 6 us slower)
    const bool warp_ok = rows_ok && cols % 8 == 0 && nw >= 8 && SFMP_XPREP_WARP &&
                         Mpad <= static_cast<int64_t>(nw) * per_sm * m.num_sms;
    cudaError_t e0 = cudaSuccess;
    if (warp_ok) {
        const int wgrid = static_cast<int>(std::min<int64_t>((Mpad + nw - 1) / nw, static_cast<int64_t>(per_sm) * m.num_sms));
        switch (dt) {
            case SFMP_F32: launch_xprep_warp<SFMP_F32>(x, m, xs, ysc, p, cols, Mpad, nw, wgrid, wsm, st, norm); break;
            case SFMP_F16: launch_xprep_warp<SFMP_F16>(x, m, xs, ysc, p, cols, Mpad, nw, wgrid, wsm, st, norm); break;
            default: launch_xprep_warp<SFMP_BF16>(x, m, xs, ysc, p, cols, Mpad, nw, wgrid, wsm, st, norm); break;
        }
    } else if (rows_ok) {
        const int per_sm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(4, (220 * 1024) / rsm)));
        const int rgrid = static_cast<int>(std::min<int64_t>(Mpad, static_cast<int64_t>(per_sm) * m.num_sms));
        switch (dt) {
            case SFMP_F32: launch_xprep_rows<SFMP_F32>(x, m, xs, ysc, p, cols, Mpad, rgrid, rsm, st, norm); break;
            case SFMP_F16: launch_xprep_rows<SFMP_F16>(x, m, xs, ysc, p, cols, Mpad, rgrid, rsm, st, norm); break;
            default: launch_xprep_rows<SFMP_BF16>(x, m, xs, ysc, p, cols, Mpad, rgrid, rsm, st, norm); break;
        }
    } else {
        switch (dt) {
            case SFMP_F32: launch_xprep_tok<SFMP_F32>(x, m, xs, ysc, p, cols, Mpad, st, norm); break;
            case SFMP_F16: launch_xprep_tok<SFMP_F16>(x, m, xs, ysc, p, cols, Mpad, st, norm); break;
            default: launch_xprep_tok<SFMP_BF16>(x, m, xs, ysc, p, cols, Mpad, st, norm); break;
        }
    }
    e0 = cudaGetLastError();
    if (e0 != cudaSuccess) return e0;
    // (Clusters of 4 sharing X by TMA multicast measured no faster and capped the
    // grid at the co-resident cluster count, 132 of 148 SMs: not used.)
    const int64_t ntiles = static_cast<int64_t>(p.RT) * p.TT;
    p.ks = k_splits(m, M);
    p.GT = raster_group(m, M);
    p.items = static_cast<int>(ntiles * p.ks);
    const int grid = static_cast<int>(std::min<int64_t>(p.items, m.num_sms));
    switch (m.ceil_bits) {
        case 1: return launch_np<1>(p, smem, grid, st);
        case 2: return launch_np<2>(p, smem, grid, st);
        case 3: return launch_np<3>(p, smem, grid, st);
        case 4: return launch_np<4>(p, smem, grid, st);
        case 5: return launch_np<5>(p, smem, grid, st);
        case 6: return launch_np<6>(p, smem, grid, st);
        case 7: return launch_np<7>(p, smem, grid, st);
        default: return launch_np<8>(p, smem, grid, st);
    }
}

}  // namespace sfmpk
