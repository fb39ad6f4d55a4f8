// gemv_tc.cu -- K1: decode GEMV (M <= 16) for SFMP block-wise mixed-precision weights.
//
// Replaces sfmp::gemv (lutgemm.cpp:95-135) incl. the activation gather
// (reorder_activation_in, reorder.cpp:103-111) and the output scatter
// (reorder_activation_out, reorder.cpp:113-121).  Paths relative to
// /root/reference/proj.
//
// HBM-bound design:
//  * Work unit = 128 reordered rows x one block column (n_b columns).  The
//    unit's bytes are 2+bits contiguous spans of the SFMPPKD1 block (scales,
//    zeros, one span per bit-plane), streamed by 1-D bulk async copies
//    (cp.async.bulk, the TMA engine) into a deep shared-memory ring guarded
//    by mbarriers.  One persistent CTA per SM walks a contiguous range of
//    units (row-tile-major), balanced by bytes.
//  * The activation gather x[t][col_perm[.]] (reorder-in) runs once per call
//    in a tiny pre-pass (xprep_kernel) that writes, per block column, the f16
//    MMA B fragments plus per-token column sums; the GEMV is launched with
//    programmatic dependent launch, so its producer streams weights while the
//    pre-pass runs and bulk-copies each unit's 2-4 KB fragment record next to
//    the unit's weights.
//  * Warp roles: 1 producer warp (bulk copies), 8 compute warps (16 rows
//    each); 2 CTAs per SM.
//  * Compute: the bit-planes of a row's 32-weight word are transposed into
//    nibble codes with 4 delta-swaps, converted to exact f16 integers with the
//    0x6400 magic, and contracted against the activations on the tensor pipe
//    (mma.m16n8k16, tokens = N).  The per-row affine (s, z) of each block is
//    applied in f32 after the block column: y += s*sum(c*x) + z*sum(x), which
//    equals sum((s*c+z)*x) up to f32 rounding.  The K permutation inside a
//    128-column chunk that the unpack produces is absorbed by the gather.
//  * Deterministic split-K: a row tile spread over several CTAs is reduced by
//    the last arriving CTA in fixed segment order; the row un-permutation is
//    fused into the final store.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "ptx.cuh"
#include "sfmp_internal.h"

namespace sfmpk {

namespace {

constexpr int kTR = 128;  // rows per unit
constexpr int kNCW = 8;   // compute warps (16 rows each)
constexpr int kThreads = 32 * (1 + kNCW);
constexpr int kFirstCompute = 32;
constexpr int kCtasPerSm = 2;
constexpr int kSmemPerCta = 113 * 1024;

struct Params {
    const uint8_t* payload;
    const uint64_t* off;
    const uint8_t* bits;
    const uint32_t* out_map;
    const uint8_t* xfrag;  // [BC] records of stage_x bytes (written by xprep_kernel)
    float* y;
    float* ws;
    const int* cta_begin;
    const int* rt_nseg;
    const int* rt_slot;
    const int* rt_first;
    unsigned* counters;
    int M;
    int BC;
    int m_b;
    int n_b;
    uint64_t out_rows;
    int stages;
    uint32_t stage_w;  // bytes per weight stage (smem)
    uint32_t stage_x;  // bytes per activation record (smem and global)
};

template <sfmp_dtype DT>
__device__ __forceinline__ float load_x(const void* x, size_t i) {
    if constexpr (DT == SFMP_F32) return __ldg(static_cast<const float*>(x) + i);
    else if constexpr (DT == SFMP_F16)
        return __half2float(__ldg(static_cast<const __half*>(x) + i));
    else
        return __bfloat162float(__ldg(static_cast<const __nv_bfloat16*>(x) + i));
}

// K4 (decode flavour): gather x[t][col_perm[.]] once per call into per-block-
// column records laid out exactly as the MMA B fragments the GEMV consumes,
// plus the per-token column sums X_g used by the zero-point term
// (lutgemm.cpp:113-115).  One warp per (block column, n-tile); lane (n,q)
// owns token nt*8+n and k-slots 32q + 4h + a (+16).
template <int NT, sfmp_dtype DT>
__global__ void __launch_bounds__(256) xprep_kernel(const void* x, const uint32_t* col_perm, uint8_t* xfrag,
                                                    int M, int cols, int n_b, int BC, uint32_t rec_bytes) {
    pdl_launch_dependents();  // let the GEMV start streaming weights right away
    const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (w >= BC * NT) return;
    const int bc = w / NT, nt = w - bc * NT;
    const int lane = threadIdx.x & 31, q = lane & 3, n = lane >> 2;
    const int CH = n_b >> 7;
    const int t = nt * 8 + n;
    uint8_t* rec = xfrag + static_cast<size_t>(bc) * rec_bytes;
    float xs = 0.f;
    for (int c = 0; c < CH; ++c) {
        const uint4 idx4 = __ldg(reinterpret_cast<const uint4*>(col_perm + bc * n_b + c * 128) + lane);
        uint32_t gi[32];
#pragma unroll
        for (int s8 = 0; s8 < 8; ++s8) {
            const int a = s8 >> 1;
            const uint32_t comp = a == 0 ? idx4.x : a == 1 ? idx4.y : a == 2 ? idx4.z : idx4.w;
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int wk = 4 * (2 * (s8 & 1) + j) + a + 16 * e;
                    gi[s8 * 4 + j * 2 + e] = __shfl_sync(0xffffffffu, comp, 8 * q + (wk >> 2));
                }
        }
        float v[32];
        if (t < M) {
            const size_t rowoff = static_cast<size_t>(t) * cols;
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = load_x<DT>(x, rowoff + gi[e]);
        } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0.f;
        }
#pragma unroll
        for (int s8 = 0; s8 < 8; ++s8) {
            uint2 st;
            st.x = h2_as_u32(__floats2half2_rn(v[s8 * 4 + 0], v[s8 * 4 + 1]));
            st.y = h2_as_u32(__floats2half2_rn(v[s8 * 4 + 2], v[s8 * 4 + 3]));
            *reinterpret_cast<uint2*>(rec + ((c * NT + nt) * 8 + s8) * 256 + lane * 8) = st;
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) xs += v[e];
    }
    xs += __shfl_xor_sync(0xffffffffu, xs, 1);
    xs += __shfl_xor_sync(0xffffffffu, xs, 2);
    if (q == 0) reinterpret_cast<float*>(rec + CH * NT * 2048)[nt * 8 + n] = xs;
}

// 4x4 bit-matrix transpose of four plane words (bit j = weight j of the
// 32-weight word) into nibble words: q[a] nibble n = code of weight 4n+a.
template <int NP>
__device__ __forceinline__ void planes_to_nibbles(const uint32_t* p, uint32_t (&q)[4]) {
    uint32_t p0 = p[0], p1 = NP > 1 ? p[1] : 0u, p2 = NP > 2 ? p[2] : 0u, p3 = NP > 3 ? p[3] : 0u;
    uint32_t t;
    if (NP > 1) {
        t = ((p0 >> 1) ^ p1) & 0x55555555u;
        p1 ^= t;
        p0 ^= t << 1;
    } else {
        t = (p0 >> 1) & 0x55555555u;
        p1 = t;
        p0 ^= t << 1;
    }
    if (NP > 2) {
        if (NP > 3) {
            t = ((p2 >> 1) ^ p3) & 0x55555555u;
            p3 ^= t;
            p2 ^= t << 1;
        } else {
            t = (p2 >> 1) & 0x55555555u;
            p3 = t;
            p2 ^= t << 1;
        }
        t = ((p0 >> 2) ^ p2) & 0x33333333u;
        p2 ^= t;
        p0 ^= t << 2;
        t = ((p1 >> 2) ^ p3) & 0x33333333u;
        p3 ^= t;
        p1 ^= t << 2;
    } else {
        t = (p0 >> 2) & 0x33333333u;
        p2 = t;
        p0 ^= t << 2;
        t = (p1 >> 2) & 0x33333333u;
        p3 = t;
        p1 ^= t << 2;
    }
    q[0] = p0;
    q[1] = p1;
    q[2] = p2;
    q[3] = p3;
}

// Nibble word -> 4 half2 of exact integer codes:
// h[0]=(nib0,nib4) h[1]=(nib1,nib5) h[2]=(nib2,nib6) h[3]=(nib3,nib7).
__device__ __forceinline__ void nibbles_to_h2(uint32_t q, uint32_t* h) {
    const uint32_t kMagic = 0x64006400u;  // 1024.0 in both halves
    const __half2 k1024 = u32_as_h2(0x64006400u);
    const __half2 k16th = u32_as_h2(0x2C002C00u);  // 1/16
    const __half2 kM64 = u32_as_h2(0xD400D400u);   // -64
    const uint32_t q8 = q >> 8;
    h[0] = h2_as_u32(__hsub2(u32_as_h2(lop3_and_or(q, 0x000F000Fu, kMagic)), k1024));
    h[1] = h2_as_u32(__hfma2(u32_as_h2(lop3_and_or(q, 0x00F000F0u, kMagic)), k16th, kM64));
    h[2] = h2_as_u32(__hsub2(u32_as_h2(lop3_and_or(q8, 0x000F000Fu, kMagic)), k1024));
    h[3] = h2_as_u32(__hfma2(u32_as_h2(lop3_and_or(q8, 0x00F000F0u, kMagic)), k16th, kM64));
}

// All 32 weights of one row word as 16 half2 codes; H[4a+h] = weights
// (4h+a, 4h+a+16) of the word.
template <int B>
__device__ __forceinline__ void unpack_word(const uint32_t* p, uint32_t (&H)[16]) {
    uint32_t q[4];
    if constexpr (B <= 4) {
        planes_to_nibbles<B>(p, q);
#pragma unroll
        for (int a = 0; a < 4; ++a) nibbles_to_h2(q[a], H + 4 * a);
    } else {
        uint32_t qh[4];
        planes_to_nibbles<4>(p, q);
        planes_to_nibbles<B - 4>(p + 4, qh);
        const __half2 k16 = u32_as_h2(0x4C004C00u);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            uint32_t lo[4], hi[4];
            nibbles_to_h2(q[a], lo);
            nibbles_to_h2(qh[a], hi);
#pragma unroll
            for (int h = 0; h < 4; ++h)
                H[4 * a + h] = h2_as_u32(__hfma2(u32_as_h2(hi[h]), k16, u32_as_h2(lo[h])));
        }
    }
}

template <int B, int NT>
__device__ __forceinline__ void unit_chunk(const uint8_t* wst, const uint8_t* xst, int c, int nb8,
                                           int r0, int q, int lane, float (&cacc)[2][NT][4]) {
    const uint8_t* planes = wst + 4 * kTR;
    const int plane_stride = kTR * nb8;
    uint32_t p0[B], p1[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
        p0[i] = *reinterpret_cast<const uint32_t*>(planes + i * plane_stride + r0 * nb8 + c * 16 + q * 4);
        p1[i] = *reinterpret_cast<const uint32_t*>(planes + i * plane_stride + (r0 + 8) * nb8 + c * 16 +
                                                   q * 4);
    }
    uint32_t A0[16], A1[16];
    unpack_word<B>(p0, A0);
    unpack_word<B>(p1, A1);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const uint2 b = *reinterpret_cast<const uint2*>(xst + ((c * NT + nt) * 8 + s) * 256 + lane * 8);
            // two independent accumulator chains halve the HMMA dependency depth
            mma_16816(cacc[s & 1][nt], A0[2 * s], A1[2 * s], A0[2 * s + 1], A1[2 * s + 1], b.x, b.y);
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) gemv_kernel(const Params p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    int* flag = reinterpret_cast<int*>(empty + S);
    uint8_t* wbase = smem + 512;
    uint8_t* xbase = wbase + static_cast<size_t>(S) * p.stage_w;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNCW);
        }
        fence_mbar_init();
        fence_proxy_async();
    }
    __syncthreads();

    const int u0 = p.cta_begin[blockIdx.x], u1 = p.cta_begin[blockIdx.x + 1];
    const int nb8 = p.n_b >> 3;
    const int CH = p.n_b >> 7;
    const int tiles_per_brow = p.m_b / kTR;

    if (warp == 0) {
        // ---------------- producer: bulk copies (weights now, x after PDL wait) ----
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const uint32_t pbytes = kTR * nb8;
            const size_t plane_bytes = static_cast<size_t>(p.m_b) * nb8;
            int rt = u0 / p.BC, bc = u0 - rt * p.BC;
            auto issue_w = [&](int s, int rt_, int bc_) {
                const int br = rt_ / tiles_per_brow, ro = (rt_ - br * tiles_per_brow) * kTR;
                const size_t k = static_cast<size_t>(br) * p.BC + bc_;
                const int bits = p.bits[k];
                const uint8_t* blk = p.payload + p.off[k];
                uint8_t* dst = wbase + static_cast<size_t>(s) * p.stage_w;
                mbar_arrive_expect_tx(&full[s], 4 * kTR + bits * pbytes + p.stage_x);
                bulk_g2s(dst, blk + 2 * ro, 2 * kTR, &full[s], pol);
                bulk_g2s(dst + 2 * kTR, blk + 2 * p.m_b + 2 * ro, 2 * kTR, &full[s], pol);
                for (int b = 0; b < bits; ++b)
                    bulk_g2s(dst + 4 * kTR + b * pbytes,
                             blk + 4 * static_cast<size_t>(p.m_b) + b * plane_bytes + static_cast<size_t>(ro) * nb8,
                             pbytes, &full[s], pol);
            };
            auto issue_x = [&](int s, int bc_) {
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(xbase + static_cast<size_t>(s) * p.stage_x)),
                    "l"(p.xfrag + static_cast<size_t>(bc_) * p.stage_x), "r"(p.stage_x), "r"(smem_u32(&full[s]))
                    : "memory");
            };
            const int n = u1 - u0;
            const int pre = n < S ? n : S;
            // 1) weights of the first ring-full of units do not depend on x
            int prt = rt, pbc = bc;
            for (int i = 0; i < pre; ++i) {
                issue_w(i, prt, pbc);
                if (++pbc == p.BC) { pbc = 0; ++prt; }
            }
            // 2) wait for the x-fragment producer (programmatic dependent launch)
            pdl_wait();
            prt = rt;
            pbc = bc;
            for (int i = 0; i < pre; ++i) {
                issue_x(i, pbc);
                if (++pbc == p.BC) { pbc = 0; ++prt; }
            }
            // 3) steady state
            for (int i = pre; i < n; ++i) {
                const int s = i % S;
                mbar_wait(&empty[s], ((i / S) - 1) & 1);
                issue_w(s, prt, pbc);
                issue_x(s, pbc);
                if (++pbc == p.BC) { pbc = 0; ++prt; }
            }
        }
        return;
    }

    // ---------------- compute warps ------------------------------------------
    const int cw = warp - 1;
    const int g = lane >> 2, q = lane & 3;
    const int r0 = cw * 16 + g;  // row within the unit; second row r0+8
    const int ct = threadIdx.x - kFirstCompute;
    float yacc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) yacc[nt][e] = 0.f;

    auto flush = [&](int rt) {
        const int nseg = p.rt_nseg[rt];
        const int rowbase = rt * kTR;
        if (nseg == 1) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int t = nt * 8 + 2 * q + (e & 1);
                    const int row = r0 + (e >> 1) * 8;
                    if (t < p.M) p.y[t * p.out_rows + p.out_map[rowbase + row]] = yacc[nt][e];
                }
            return;
        }
        const int slot0 = p.rt_slot[rt];
        const int slot = slot0 + (blockIdx.x - p.rt_first[rt]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int t = nt * 8 + 2 * q + (e & 1);
                const int row = r0 + (e >> 1) * 8;
                if (t < p.M) p.ws[(static_cast<size_t>(slot) * 16 + t) * kTR + row] = yacc[nt][e];
            }
        __threadfence();
        named_bar_sync(1, kNCW * 32);
        if (ct == 0) *flag = (atomicAdd(&p.counters[rt], 1u) == static_cast<unsigned>(nseg - 1));
        named_bar_sync(1, kNCW * 32);
        if (*flag) {
            __threadfence();
            for (int idx = ct; idx < p.M * kTR; idx += kNCW * 32) {
                const int t = idx >> 7, row = idx & (kTR - 1);
                float acc = 0.f;
                for (int sg = 0; sg < nseg; ++sg)
                    acc += __ldcg(p.ws + (static_cast<size_t>(slot0 + sg) * 16 + t) * kTR + row);
                p.y[t * p.out_rows + p.out_map[rowbase + row]] = acc;
            }
            if (ct == 0) p.counters[rt] = 0u;
        }
    };

    int rt = u0 / p.BC, bc = u0 - rt * p.BC;
    int cur_rt = rt;
    int s = 0, ph = 0;
    for (int u = u0; u < u1; ++u) {
        if (rt != cur_rt) {
            flush(cur_rt);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) yacc[nt][e] = 0.f;
            cur_rt = rt;
        }
        const int bits = p.bits[static_cast<size_t>(rt / tiles_per_brow) * p.BC + bc];
        const uint8_t* wst = wbase + static_cast<size_t>(s) * p.stage_w;
        const uint8_t* xst = xbase + static_cast<size_t>(s) * p.stage_x;
        mbar_wait(&full[s], ph);
        const __half* sz = reinterpret_cast<const __half*>(wst);
        const float s0 = __half2float(sz[r0]), s1 = __half2float(sz[r0 + 8]);
        const float z0 = __half2float(sz[kTR + r0]), z1 = __half2float(sz[kTR + r0 + 8]);
        float cacc[2][NT][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) cacc[h][nt][e] = 0.f;
        for (int c = 0; c < CH; ++c) {
            switch (bits) {
                case 1: unit_chunk<1, NT>(wst, xst, c, nb8, r0, q, lane, cacc); break;
                case 2: unit_chunk<2, NT>(wst, xst, c, nb8, r0, q, lane, cacc); break;
                case 3: unit_chunk<3, NT>(wst, xst, c, nb8, r0, q, lane, cacc); break;
                case 4: unit_chunk<4, NT>(wst, xst, c, nb8, r0, q, lane, cacc); break;
                case 5: unit_chunk<5, NT>(wst, xst, c, nb8, r0, q, lane, cacc); break;
                case 6: unit_chunk<6, NT>(wst, xst, c, nb8, r0, q, lane, cacc); break;
                case 7: unit_chunk<7, NT>(wst, xst, c, nb8, r0, q, lane, cacc); break;
                default: unit_chunk<8, NT>(wst, xst, c, nb8, r0, q, lane, cacc); break;
            }
        }
        const float* xg = reinterpret_cast<const float*>(xst + CH * NT * 2048);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float xg0 = xg[nt * 8 + 2 * q], xg1 = xg[nt * 8 + 2 * q + 1];
            yacc[nt][0] += s0 * (cacc[0][nt][0] + cacc[1][nt][0]) + z0 * xg0;
            yacc[nt][1] += s0 * (cacc[0][nt][1] + cacc[1][nt][1]) + z0 * xg1;
            yacc[nt][2] += s1 * (cacc[0][nt][2] + cacc[1][nt][2]) + z1 * xg0;
            yacc[nt][3] += s1 * (cacc[0][nt][3] + cacc[1][nt][3]) + z1 * xg1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == S) { s = 0; ph ^= 1; }
        if (++bc == p.BC) { bc = 0; ++rt; }
    }
    if (u1 > u0) flush(cur_rt);
}

template <class K>
cudaError_t set_smem_once(K k, int slot) {
    static int configured[2][64] = {{0}};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[slot][dev]) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemPerCta);
        if (e != cudaSuccess) return e;
        configured[slot][dev] = 1;
    }
    return cudaSuccess;
}

template <int NT, sfmp_dtype DT>
cudaError_t launch_t(const Params& p, const void* x, const uint32_t* col_perm, int cols, int grid, size_t smem,
                     cudaStream_t st) {
    // K4: x fragments (normal launch: it overwrites the workspace the previous
    // call may still read, so it must follow it in stream order).
    const int warps = p.BC * NT;
    xprep_kernel<NT, DT><<<(warps + 7) / 8, 256, 0, st>>>(x, col_perm, const_cast<uint8_t*>(p.xfrag), p.M,
                                                          cols, p.n_b, p.BC, p.stage_x);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    auto k = gemv_kernel<NT>;
    if ((e = set_smem_once(k, NT - 1)) != cudaSuccess) return e;
    // K1 with programmatic dependent launch: its producer streams weights
    // while xprep runs and waits (griddepcontrol.wait) only before the x copies.
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

static uint32_t stage_x_bytes(const DevModel& m, int NT) {
    return static_cast<uint32_t>((static_cast<int>(m.n_b / 128) * NT * 2048 + 64 + 127) / 128 * 128);
}

size_t gemv_workspace_bytes(const DevModel& m, int M) {
    (void)M;
    const size_t partial = static_cast<size_t>(m.gemv.total_slots) * 16 * kTR * sizeof(float);
    const size_t xfrag = static_cast<size_t>(m.gemv.block_cols) * stage_x_bytes(m, 2);
    return (partial + 255) / 256 * 256 + xfrag;
}

int gemv_ctas_per_sm() { return kCtasPerSm; }

cudaError_t launch_gemv(const DevModel& m, const void* x, sfmp_dtype dt, int M, float* y, float* ws,
                        cudaStream_t st) {
    const GemvSchedule& g = m.gemv;
    Params p{};
    p.payload = m.d_payload;
    p.off = m.d_off;
    p.bits = m.d_bits;
    p.out_map = m.d_out_map;
    p.y = y;
    p.ws = ws;
    const size_t partial = static_cast<size_t>(g.total_slots) * 16 * kTR * sizeof(float);
    p.xfrag = reinterpret_cast<const uint8_t*>(ws) + (partial + 255) / 256 * 256;
    p.cta_begin = g.d_cta_begin;
    p.rt_nseg = g.d_rt_nseg;
    p.rt_slot = g.d_rt_slot;
    p.rt_first = g.d_rt_first;
    p.counters = g.d_counters;
    p.M = M;
    p.BC = g.block_cols;
    p.m_b = static_cast<int>(m.m_b);
    p.n_b = static_cast<int>(m.n_b);
    p.out_rows = m.out_rows;
    const int NT = M > 8 ? 2 : 1;
    p.stage_w = static_cast<uint32_t>((4 * kTR + m.ceil_bits * kTR * (m.n_b / 8) + 127) / 128 * 128);
    p.stage_x = stage_x_bytes(m, NT);
    const int stages = std::min<int>(16, (kSmemPerCta - 512) / static_cast<int>(p.stage_w + p.stage_x));
    if (stages < 2) return cudaErrorInvalidConfiguration;
    p.stages = stages;
    const size_t smem = 512 + static_cast<size_t>(stages) * (p.stage_w + p.stage_x);
    const int cols = static_cast<int>(m.cols);
    if (NT == 1) {
        switch (dt) {
            case SFMP_F32: return launch_t<1, SFMP_F32>(p, x, m.d_col_perm, cols, g.grid, smem, st);
            case SFMP_F16: return launch_t<1, SFMP_F16>(p, x, m.d_col_perm, cols, g.grid, smem, st);
            default: return launch_t<1, SFMP_BF16>(p, x, m.d_col_perm, cols, g.grid, smem, st);
        }
    }
    switch (dt) {
        case SFMP_F32: return launch_t<2, SFMP_F32>(p, x, m.d_col_perm, cols, g.grid, smem, st);
        case SFMP_F16: return launch_t<2, SFMP_F16>(p, x, m.d_col_perm, cols, g.grid, smem, st);
        default: return launch_t<2, SFMP_BF16>(p, x, m.d_col_perm, cols, g.grid, smem, st);
    }
}

}  // namespace sfmpk
