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
//  * xprep_gemm_kernel gathers x[t][col_perm[.]], converts to f16 and lays
//    every (token tile, 128-column chunk) out as the exact 128-byte-swizzled
//    K-major shared-memory image of the MMA B operand, so the GEMM fetches
//    it with one 1-D bulk copy (no tensor map).  The K order inside each
//    32-column word follows the register order the unpacker produces.
//  * Persistent warp-specialised kernel, one CTA per SM, tile = 256 output
//    rows (two M=128 MMAs) x N<=128 tokens:
//      warp 0      producer: cp.async.bulk of weight units and X tiles
//      warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//      warps 2-5   epilogue: tcgen05.ld accumulators -> coalesced y stores
//      warps 6-13  dequant: bit-planes -> codes -> f16(s*c+z) (one HFMA2 per
//                  weight pair, fp16 s/z exactly as stored) written straight
//                  into TMEM as the MMA A operand (tcgen05.st), so weights
//                  never take a shared-memory round trip.
//    TMEM (512 columns): 2 accumulators x 128 columns, 2 A buffers x 2 row
//    halves x 64 columns (128 f16 of K per row).
//  * Precision: weights are rounded once to f16 (SURVEY §7 hard part 1:
//    f16 dequant stays ~5x inside the 1e-3 bar, bf16 would not); the
//    activations are converted to f16 (exact for bf16 values in f16 range);
//    accumulation is f32 in TMEM.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ptx.cuh"
#include "sfmp_internal.h"
#include "tc.cuh"
#include "unpack.cuh"

namespace sfmpk {

namespace {

constexpr int kRowsTile = 128;            // rows per layout tile (= MMA M)
constexpr int kUnitHdr = 528;             // scales[128] | zeros[128] | highmask[4]
constexpr int kPlaneBytes = 128 * 16;     // one plane of a unit
constexpr int kThreads = 14 * 32;
constexpr int kMaxN = 128;                // tokens per tile
constexpr int kTmemCols = 512;
constexpr int kAccCol = 0;                // accumulator rh at kAccCol + rh*128
constexpr int kACol = 256;                // A buffer (ab, rh) at kACol + (ab*2+rh)*64
constexpr int kSmemLimit = 227 * 1024;

struct GemmParams {
    const uint8_t* wl;       // row-tile layout payload
    const uint64_t* woff;    // [RT2*KC + 1] unit byte offsets
    const uint8_t* xs;       // [TT][KC][2][N][128 B] swizzled f16 X
    float* y;
    int M, N, TT, KC, RP;    // tokens, tokens/tile, token tiles, 128-col chunks, row-tile pairs
    uint64_t out_rows;
    int floor_bits, has_extra;
    int SX, SW;              // X / W ring stages
    uint32_t stage_w, half_w;  // W stage bytes, offset of the bottom unit
    uint32_t idesc;
};

// x[t][col_perm[...]] -> f16, in the K order of the unpacked A operand:
// slot s of a 128-column chunk holds reordered column 32w + 4h + a + 16e
// with w = s/32, p = s%32, j = p/2 = 4a + h, e = p%2 (unpack_word register
// order: H[4a+h] = weights (4h+a, 4h+a+16) of the word, low half first).
__device__ __forceinline__ int slot_col(int s) {
    const int w = s >> 5, p = s & 31, j = p >> 1, e = p & 1;
    return 32 * w + 4 * (j & 3) + (j >> 2) + 16 * e;
}

template <sfmp_dtype DT>
__device__ __forceinline__ float ldx(const void* x, size_t i) {
    if constexpr (DT == SFMP_F32) return __ldg(static_cast<const float*>(x) + i);
    else if constexpr (DT == SFMP_F16)
        return __half2float(__ldg(static_cast<const __half*>(x) + i));
    else
        return __bfloat162float(__ldg(static_cast<const __nv_bfloat16*>(x) + i));
}

// One CTA per (token tile, 128-column chunk): 2 atoms x N rows x 8 chunks of 16 B.
template <sfmp_dtype DT>
__global__ void __launch_bounds__(256) xprep_gemm_kernel(const void* x, const uint32_t* col_perm, uint8_t* xs,
                                                         int M, int N, int KC, int cols) {
    pdl_launch_dependents();
    const int kc = blockIdx.x % KC, tt = blockIdx.x / KC;
    uint8_t* dst = xs + (static_cast<size_t>(tt) * KC + kc) * 2 * N * 128;
    const uint32_t* cp = col_perm + static_cast<size_t>(kc) * 128;
    for (int c = threadIdx.x; c < 2 * N * 8; c += blockDim.x) {
        const int a = c / (N * 8), rem = c - a * N * 8, r = rem >> 3, pc = rem & 7;
        const int j = pc ^ (r & 7);  // logical 16-byte chunk stored at physical pc
        const int t = tt * N + r;
        uint32_t packed[4] = {0u, 0u, 0u, 0u};
        if (t < M) {
            const size_t row = static_cast<size_t>(t) * cols;
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                const int s = 64 * a + 8 * j + e;
                const float v0 = ldx<DT>(x, row + __ldg(cp + slot_col(s)));
                const float v1 = ldx<DT>(x, row + __ldg(cp + slot_col(s + 1)));
                packed[e >> 1] = h2_as_u32(__floats2half2_rn(v0, v1));
            }
        }
        *reinterpret_cast<uint4*>(dst + static_cast<size_t>(a) * N * 128 + r * 128 + pc * 16) =
            make_uint4(packed[0], packed[1], packed[2], packed[3]);
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
    const uint32_t xstage = static_cast<uint32_t>(2 * N * 128);
    uint8_t* xbuf = smem;
    uint8_t* wbuf = xbuf + static_cast<size_t>(SX) * xstage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbuf + static_cast<size_t>(SW) * p.stage_w);
    uint64_t* xfull = bars;
    uint64_t* xempty = xfull + SX;
    uint64_t* wfull = xempty + SX;
    uint64_t* wempty = wfull + SW;
    uint64_t* afull = wempty + SW;   // [2]
    uint64_t* aempty = afull + 2;    // [2]
    uint64_t* accfull = aempty + 2;  // [1]
    uint64_t* accempty = accfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 1);
    uint64_t* offs = accempty + 2;  // [2*KC + 1] unit offsets of the producer's current tile

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SX; ++s) {
            mbar_init(&xfull[s], 1);
            mbar_init(&xempty[s], 1);
        }
        for (int s = 0; s < SW; ++s) {
            mbar_init(&wfull[s], 1);
            mbar_init(&wempty[s], 8);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&afull[a], 8);
            mbar_init(&aempty[a], 1);
        }
        mbar_init(accfull, 1);
        mbar_init(accempty, 4);
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

    const int ntiles = p.RP * p.TT;
    const int KC = p.KC;

    if (warp == 0) {
        // ---------------- producer ----------------
        // The unit offsets of a tile's two row tiles are staged in shared
        // memory by the whole warp, so lane 0 never waits on a global load
        // between bulk copies.
        const uint64_t pol_w = policy_evict_first();
        int xs = 0, xph = 0, ws = 0, wph = 0;
        bool waited = false;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int rp = tile / p.TT, tt = tile - rp * p.TT;
            const uint64_t* off0 = p.woff + static_cast<size_t>(2 * rp) * KC;
            __syncwarp();
            for (int i = lane; i <= 2 * KC; i += 32) offs[i] = __ldg(off0 + i);
            __syncwarp();
            if (lane == 0) {
                for (int kc = 0; kc < KC; ++kc) {
                    // weights (independent of the X pre-pass)
                    mbar_wait(&wempty[ws], wph ^ 1);
                    const uint64_t a0 = offs[kc], a1 = offs[kc + 1];
                    const uint64_t b0 = offs[KC + kc], b1 = offs[KC + kc + 1];
                    const uint32_t n0 = static_cast<uint32_t>(a1 - a0), n1 = static_cast<uint32_t>(b1 - b0);
                    mbar_arrive_expect_tx(&wfull[ws], n0 + n1);
                    uint8_t* wdst = wbuf + static_cast<size_t>(ws) * p.stage_w;
                    bulk_g2s(wdst, p.wl + a0, n0, &wfull[ws], pol_w);
                    bulk_g2s(wdst + p.half_w, p.wl + b0, n1, &wfull[ws], pol_w);
                    if (++ws == SW) { ws = 0; wph ^= 1; }
                    // activations
                    if (!waited) {
                        pdl_wait();
                        waited = true;
                    }
                    mbar_wait(&xempty[xs], xph ^ 1);
                    mbar_arrive_expect_tx(&xfull[xs], xstage);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(xbuf + static_cast<size_t>(xs) * xstage)),
                        "l"(p.xs + (static_cast<size_t>(tt) * KC + kc) * xstage), "r"(xstage), "r"(smem_u32(&xfull[xs]))
                        : "memory");
                    if (++xs == SX) { xs = 0; xph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            int xs = 0, xph = 0, ab = 0, aph = 0, accph = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                mbar_wait(accempty, accph ^ 1);
                tc_fence_after();
                for (int kc = 0; kc < KC; ++kc) {
                    mbar_wait(&afull[ab], aph);
                    mbar_wait(&xfull[xs], xph);
                    tc_fence_after();
                    const uint32_t xaddr = smem_u32(xbuf + static_cast<size_t>(xs) * xstage);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint64_t bdesc = tc_desc_sw128(xaddr + (kk >> 2) * N * 128 + (kk & 3) * 32);
#pragma unroll
                        for (int rh = 0; rh < 2; ++rh)
                            tc_mma_ts(tbase + kAccCol + rh * 128, tbase + kACol + (ab * 2 + rh) * 64 + kk * 8, bdesc,
                                      p.idesc, (kc | kk) != 0);
                    }
                    tc_commit(&aempty[ab]);
                    tc_commit(&xempty[xs]);
                    if (++ab == 2) { ab = 0; aph ^= 1; }
                    if (++xs == SX) { xs = 0; xph ^= 1; }
                }
                tc_commit(accfull);
                accph ^= 1;
            }
        }
    } else if (warp < 6) {
        // ---------------- epilogue ----------------
        const int q = warp & 3;
        int accph = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int rp = tile / p.TT, tt = tile - rp * p.TT;
            mbar_wait(accfull, accph);
            accph ^= 1;
            tc_fence_after();
            const int t0 = tt * N;
#pragma unroll 1
            for (int rh = 0; rh < 2; ++rh) {
                const uint64_t row = static_cast<uint64_t>(rp) * 256 + rh * 128 + q * 32 + lane;
                const bool row_ok = row < p.out_rows;
#pragma unroll 1
                for (int c0 = 0; c0 < N; c0 += 32) {
                    uint32_t v[32];
                    tc_ld_x32(tbase + (static_cast<uint32_t>(q * 32) << 16) + kAccCol + rh * 128 + c0, v);
                    tc_wait_ld();
                    if (row_ok) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int t = t0 + c0 + j;
                            if (c0 + j < N && t < p.M) p.y[static_cast<size_t>(t) * p.out_rows + row] = __uint_as_float(v[j]);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty);
        }
    } else {
        // ---------------- dequant ----------------
        const int dw = warp - 6, q = warp & 3, rh = dw >> 2;
        const int r = q * 32 + lane;  // row within the unit = TMEM lane
        const int F = p.floor_bits;
        int ws = 0, wph = 0, ab = 0, aph = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            for (int kc = 0; kc < KC; ++kc) {
                mbar_wait(&wfull[ws], wph);
                const uint32_t u = smem_u32(wbuf + static_cast<size_t>(ws) * p.stage_w + rh * p.half_w);
                const __half2 s2 = __half2half2(__ushort_as_half(lds_u16(u + 2 * r)));
                const __half2 z2 = __half2half2(__ushort_as_half(lds_u16(u + 256 + 2 * r)));
                uint4 pl[NP];
                if (p.has_extra) {
                    const uint4 mk = lds_v4(u + 512);
                    const uint32_t mw = q == 0 ? mk.x : q == 1 ? mk.y : q == 2 ? mk.z : mk.w;
                    const int before = (q > 0 ? __popc(mk.x) : 0) + (q > 1 ? __popc(mk.y) : 0) + (q > 2 ? __popc(mk.z) : 0);
                    const bool high = (mw >> lane) & 1u;
                    const int rank = before + __popc(mw & ((1u << lane) - 1u));
#pragma unroll
                    for (int i = 0; i < NP - 1; ++i) pl[i] = lds_v4(u + kUnitHdr + i * kPlaneBytes + r * 16);
                    pl[NP - 1] = high ? lds_v4(u + kUnitHdr + (NP - 1) * kPlaneBytes + rank * 16) : make_uint4(0, 0, 0, 0);
                } else {
#pragma unroll
                    for (int i = 0; i < NP; ++i) pl[i] = lds_v4(u + kUnitHdr + i * kPlaneBytes + r * 16);
                }
                (void)F;
                mbar_wait(&aempty[ab], aph ^ 1);
                tc_fence_after();
                const uint32_t ta = tbase + (static_cast<uint32_t>(q * 32) << 16) + kACol + (ab * 2 + rh) * 64;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    uint32_t pw[NP];
#pragma unroll
                    for (int i = 0; i < NP; ++i) pw[i] = w == 0 ? pl[i].x : w == 1 ? pl[i].y : w == 2 ? pl[i].z : pl[i].w;
                    uint32_t H[16];
                    dequant_word<NP>(pw, s2, z2, H);
                    tc_st_x16(ta + w * 16, H);
                }
                tc_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&afull[ab]);
                    mbar_arrive(&wempty[ws]);
                }
                if (++ws == SW) { ws = 0; wph ^= 1; }
                if (++ab == 2) { ab = 0; aph ^= 1; }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tc_dealloc(tbase, kTmemCols);
    }
}

int tile_n(int64_t M) {
    if (const char* e = getenv("SFMP_GEMM_N")) {
        const int n = atoi(e);
        if (n >= 16 && n <= kMaxN && n % 16 == 0) return n;
    }
    return M >= kMaxN ? kMaxN : static_cast<int>((M + 15) / 16 * 16);
}

uint32_t unit_max_bytes(const DevModel& m) {
    const int F = m.floor_bits;
    const bool extra = m.ceil_bits > m.floor_bits;
    return static_cast<uint32_t>(kUnitHdr + F * kPlaneBytes + (extra ? kPlaneBytes : 0));
}

template <int NP>
cudaError_t launch_np(const GemmParams& p, size_t smem, int grid, cudaStream_t st) {
    auto k = gemm_kernel<NP>;
    static int configured[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
        if (e != cudaSuccess) return e;
        configured[dev] = 1;
    }
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
    return cudaLaunchKernelEx(&cfg, k, p);
}

}  // namespace

// ---------------------------------------------------------------------------
// Upload-time row-tile layout (host).  For output column c of y (0..out_rows)
// the source row is the local reordered row inv[c] (or none: zero weights).
// ---------------------------------------------------------------------------
bool build_gemm_layout(DevModel& d, const std::vector<uint8_t>& payload, const std::vector<uint32_t>& out_map,
                       std::vector<uint8_t>& wl, std::vector<uint64_t>& woff) {
    if (d.n_b % 128 != 0 || d.cols % 128 != 0 || d.out_rows == 0) return false;
    const uint64_t KC = d.cols / 128, RT2 = (d.out_rows + 255) / 256 * 2;
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
    (void)C;
    return true;
}

bool gemm_supported(const DevModel& m) {
    return m.d_gl != nullptr && m.ceil_bits >= 1 && m.ceil_bits <= 8 && m.cols < (1ull << 31);
}

size_t gemm_workspace_bytes(const DevModel& m, int64_t M) {
    const int N = tile_n(M);
    const int64_t TT = (M + N - 1) / N;
    return static_cast<size_t>(TT) * N * m.cols * 2;
}

cudaError_t launch_gemm(const DevModel& m, const void* x, sfmp_dtype dt, int64_t M, float* y, void* ws,
                        cudaStream_t st) {
    GemmParams p{};
    p.N = tile_n(M);
    p.M = static_cast<int>(M);
    p.TT = static_cast<int>((M + p.N - 1) / p.N);
    p.KC = static_cast<int>(m.cols / 128);
    p.RP = static_cast<int>(m.gl_row_tiles / 2);
    p.wl = m.d_gl;
    p.woff = m.d_gl_off;
    p.xs = static_cast<const uint8_t*>(ws);
    p.y = y;
    p.out_rows = m.out_rows;
    p.floor_bits = m.floor_bits;
    p.has_extra = m.ceil_bits > m.floor_bits;
    p.idesc = tc_idesc_f16(128, p.N);
    const uint32_t ub = (unit_max_bytes(m) + 127) / 128 * 128;
    p.half_w = ub;
    p.stage_w = 2 * ub;
    const uint32_t xstage = 2u * p.N * 128;
    const size_t bar_bytes = 256 + (2 * static_cast<size_t>(p.KC) + 1) * 8;
    // X ring first (up to 4 stages), the rest of shared memory for weights
    p.SX = 4;
    const size_t avail = kSmemLimit - 1024 - bar_bytes;
    while (p.SX > 2 && p.SX * xstage + 2 * p.stage_w > avail) --p.SX;
    p.SW = static_cast<int>(std::min<size_t>(4, (avail - p.SX * xstage) / p.stage_w));
    if (p.SW < 2) return cudaErrorInvalidConfiguration;
    const size_t smem = 1024 + p.SX * xstage + p.SW * p.stage_w + bar_bytes;
    // K4 (prefill flavour): gather + convert + swizzle X
    const int xgrid = p.TT * p.KC;
    const int cols = static_cast<int>(m.cols);
    uint8_t* xs = static_cast<uint8_t*>(ws);
    switch (dt) {
        case SFMP_F32: xprep_gemm_kernel<SFMP_F32><<<xgrid, 256, 0, st>>>(x, m.d_col_perm, xs, p.M, p.N, p.KC, cols); break;
        case SFMP_F16: xprep_gemm_kernel<SFMP_F16><<<xgrid, 256, 0, st>>>(x, m.d_col_perm, xs, p.M, p.N, p.KC, cols); break;
        default: xprep_gemm_kernel<SFMP_BF16><<<xgrid, 256, 0, st>>>(x, m.d_col_perm, xs, p.M, p.N, p.KC, cols); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int ntiles = p.RP * p.TT;
    const int grid = std::max(1, std::min(ntiles, m.num_sms));
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
