// gemv_tc.cu -- K1: decode GEMV (M <= 16) for SFMP block-wise mixed-precision weights.
//
// Replaces sfmp::gemv (lutgemm.cpp:95-135) incl. the activation gather
// (reorder_activation_in, reorder.cpp:103-111) and the output scatter
// (reorder_activation_out, reorder.cpp:113-121).  Paths relative to
// /root/reference/proj.
//
// HBM-bound design:
//  * Work unit = 128 reordered rows x one block column, stored unit-major in
//    HBM (sfmp_internal.h), so a unit is one contiguous span fetched by ONE
//    1-D bulk async copy (cp.async.bulk on the TMA engine) into a small
//    mbarrier ring.
//  * Each 128-row tile is split over C CTAs (split-K); CTA s streams block
//    columns [s*BC/C, (s+1)*BC/C), writes its f32 partial tile to the
//    workspace and bumps the tile's counter; the last CTA to finish sums the
//    C partials in split order and stores them un-permuted (deterministic,
//    no float atomics) and re-zeroes the counter for the next call.
//  * The activation gather x[t][col_perm[.]] runs once per call in a small
//    pre-pass (xprep_kernel) that writes, per block column, an "activation
//    record": f16 MMA B fragments + per-token column sums.  The GEMV is a
//    programmatic dependent of it: its producer streams weights while xprep
//    runs and waits (griddepcontrol.wait) only before copying the records.
//  * Compute: the bit-planes of a row's 32-weight word are transposed into
//    nibble codes with 4 delta-swaps, and each nibble pair becomes one f16x2
//    by a single LOP3 against a magic exponent (1024+c or 64+c).  The magic
//    offsets are a per-token constant folded in f32 after the MMA (bias term
//    from the record), so the tensor pipe (mma.m16n8k16, tokens = N)
//    contracts exact integer codes against f16 activations.  The per-row
//    affine (s, z) of each block is applied in f32 after the block column:
//    y += s*(C - bias) + z*sum(x) == sum((s*c+z)*x) up to f32 rounding.  The
//    K permutation inside each 128-column chunk is absorbed by the record.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "ptx.cuh"
#include "repack.cuh"
#include "unpack.cuh"
#include "sfmp_internal.h"

namespace sfmpk {

namespace {

constexpr int kTR = 128;  // rows per unit
#ifndef SFMP_GEMV_MT
#define SFMP_GEMV_MT 2
#endif
constexpr int kMT = SFMP_GEMV_MT;  // m16 tiles (16 rows each) per compute warp
constexpr int kNCW = 8 / kMT;      // compute warps per 128-row tile
#ifndef SFMP_GEMV_CTAS1
#define SFMP_GEMV_CTAS1 (SFMP_GEMV_MT == 2 ? 4 : 3)
#endif
#ifndef SFMP_GEMV_CTAS2
#define SFMP_GEMV_CTAS2 (SFMP_GEMV_MT == 2 ? 3 : 2)
#endif
constexpr int kCtasNT1 = SFMP_GEMV_CTAS1, kCtasNT2 = SFMP_GEMV_CTAS2;  // resident CTAs per SM
constexpr int kThreads = 32 * (1 + kNCW);
constexpr int kHdrBytes = 1280;  // barriers | zeros | stage bit-widths | out_map
// resident CTAs per SM: 4 for M<=8 (NT=1), 3 for M<=16 (NT=2, more registers)
__host__ __device__ constexpr int ctas_per_sm(int NT) { return NT == 1 ? kCtasNT1 : kCtasNT2; }
__host__ __device__ constexpr int smem_per_cta(int NT) { return (225 * 1024) / ctas_per_sm(NT); }

// One linear of a (possibly grouped) launch: independent matrices -- e.g. the
// seven linears of a decoder layer -- share one launch so the fixed per-call
// latencies (launch, first HBM bytes, split-K tail) are paid once.
constexpr int kMaxLin = 40;
constexpr int kMaxSplit = 32;  // CTAs that may share one row tile
struct Lin {
    const uint8_t* payload;
    const uint64_t* unit_desc;  // [RT*BC] row-tile-major
    const uint32_t* out_map;
    const uint8_t* xrec;        // [BC] activation records of rec_bytes (xprep_kernel)
    float* y;
    float* part;                // [RT][C][16][128] f32 split-K partials
    unsigned* counters;         // [RT] completion counters (zero between calls)
    uint64_t out_rows;
    int BC;
    int M;                      // tokens of this linear (problems of one launch may differ)
    uint32_t rec_bytes;         // its activation record bytes (RecGeom{M})
    int64_t unit0;              // first unit of this linear in the group's unit sequence
};
struct Params {
    Lin lin[kMaxLin];
    int nlin;
    int64_t units;  // units of all linears
    int64_t Q;      // units per CTA
    int M;          // max tokens over the linears (all <= 8 or all in 9..16)
    int n_b;
    int stages;
    uint32_t stage_w;    // bytes per weight stage (smem)
    uint32_t rec_bytes;  // max activation record bytes (shared-memory stage stride)
    int debug_mode;      // 0 normal; 5 timeline stamps
};
struct XLin {
    const void* x;
    const uint32_t* col_perm;
    uint8_t* xrec;
    int BC, cols, warp0;
    int item0;  // first pre-pass CTA of this linear (one per token x 8 block columns)
    int lo;     // floor bit-width: records carry the magic biases of lo and lo+1 bit units
    int M;      // tokens of this linear
    uint32_t rec_bytes;
};
struct XParams {
    XLin lin[kMaxLin];
    int nlin, M, n_b;
    uint32_t rec_bytes;
    int dbg;
    int wait_prev;  // launched as a programmatic dependent of the previous GEMV
};

// Activation record of one block column (n_b columns), for M tokens:
//   for chunk c (128 columns), n-tile nt (8 tokens), token n < Mnt, k-step s:
//     4 lanes x 8 B of f16 B fragments  (tokens >= M omitted)
//   then Xg[16] (f32 column sums), then for the floor-bit and the ceil-bit
//   layout the NEGATED per-token magic offset (repack.cuh) as MMA accumulator
//   fragments [nt][lane quad q][4] = {-b(2q), -b(2q+1), -b(2q), -b(2q+1)} of
//   n-tile nt: one 16-byte load initialises an accumulator, so C - bias comes
//   out of the MMA itself.
// Within a (c, nt, n) run the 8 k-steps are contiguous (stride 32 B), so a
// lane's fragment addresses are compile-time offsets from one base.  Runs are
// kRun = 288 B apart (256 B + 32 B pad): a warp's k-step load then spreads the
// 8 tokens over all 32 banks (2 wavefronts for 256 B) instead of hitting one
// bank pair 8 times (at 256 B stride the B loads were 59 % bank conflicts and
// the shared-memory pipe the M=16 bottleneck).
constexpr int kRun = 288;
// float index (from xg_off) of token t's accumulator-init slots, layout hi=0/1
__host__ __device__ __forceinline__ int bias_slot(int t, int hi) {
    return 16 + hi * 32 + ((t >> 3) * 4 + ((t & 7) >> 1)) * 4 + (t & 1);
}
struct RecGeom {
    int M;
    __host__ __device__ int mnt(int nt) const { return nt == 0 ? (M < 8 ? M : 8) : M - 8; }
    __host__ __device__ int nt_count() const { return M > 8 ? 2 : 1; }
    __host__ __device__ int chunk_bytes() const { return kRun * M; }  // all n-tiles
    __host__ __device__ int lane_off(int c, int nt, int n, int q) const {
        return c * chunk_bytes() + nt * 8 * kRun + n * kRun + q * 8;
    }
    __host__ __device__ int frag_off(int c, int nt, int s, int n, int q) const {
        return lane_off(c, nt, n, q) + s * 32;
    }
    __host__ __device__ int xg_off(int CH) const { return CH * chunk_bytes(); }
    __host__ __device__ int bytes(int CH) const { return (xg_off(CH) + 320 + 127) / 128 * 128; }
};

// Debug timeline (SFMP_GEMV_DEBUG=5): [cta][slot] globaltimer stamps for the
// first kDbgCtas CTAs: slot 0 start, 1 end, 2+3i producer issue of unit i,
// 3+3i full observed by compute warp 0, 4+3i unit done; row kDbgCtas-1 slots
// 100.. hold kernel-level stamps.
constexpr int kDbgCtas = 512, kDbgSlots = 128;
__device__ unsigned long long g_dbg_timeline[kDbgCtas * kDbgSlots];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define DBG_STAMP(slot)                                                                       \
    do {                                                                                      \
        if (dbg == 5 && blockIdx.x < kDbgCtas - 1 && (slot) < kDbgSlots)                      \
            g_dbg_timeline[blockIdx.x * kDbgSlots + (slot)] = gtimer();                       \
    } while (0)
#define DBG_KSTAMP(slot)                                                                      \
    do {                                                                                      \
        if (dbg == 5) g_dbg_timeline[(kDbgCtas - 1) * kDbgSlots + (slot)] = gtimer();         \
    } while (0)
// Per-unit stamps cost ~12 issue slots per unit even when off: compiled in
// only with -DSFMP_GEMV_TIMELINE=1 (tools/prof_group.py's timeline).
#ifndef SFMP_GEMV_TIMELINE
#define SFMP_GEMV_TIMELINE 0
#endif
#if SFMP_GEMV_TIMELINE
#define DBG_USTAMP(slot) DBG_STAMP(slot)
#else
#define DBG_USTAMP(slot) \
    do {                 \
    } while (0)
#endif

template <sfmp_dtype DT>
__device__ __forceinline__ float load_x(const void* x, size_t i) {
    if constexpr (DT == SFMP_F32) return __ldg(static_cast<const float*>(x) + i);
    else if constexpr (DT == SFMP_F16)
        return __half2float(__ldg(static_cast<const __half*>(x) + i));
    else
        return __bfloat162float(__ldg(static_cast<const __nv_bfloat16*>(x) + i));
}

template <sfmp_dtype DT>
struct XT;
template <>
struct XT<SFMP_F32> {
    using T = float;
    static __device__ __forceinline__ float f(float v) { return v; }
};
template <>
struct XT<SFMP_F16> {
    using T = __half;
    static __device__ __forceinline__ float f(__half v) { return __half2float(v); }
};
template <>
struct XT<SFMP_BF16> {
    using T = __nv_bfloat16;
    static __device__ __forceinline__ float f(__nv_bfloat16 v) { return __bfloat162float(v); }
};
constexpr int kXprepRowLimit = 192 * 1024;  // staged x row bytes (larger rows: xprep_kernel)

// K4 (decode flavour, staged): one CTA per (token t, 8 block columns of one
// linear).  It stages token t's x row and the 8 block columns' col_perm in
// shared memory with coalesced 16 B loads, then each warp writes the record
// piece of one block column for token t: lane (s, q) gathers the 4 k-slots
// 32q + 8(s&1) + 4j + 16e + (s>>1) of each 128-column chunk from shared
// memory and stores 8 B at frag_off(c, nt, s, n, q) -- the token's 256 B of a
// chunk are one contiguous warp store.  The column sum X_g (lutgemm.cpp:
// 113-115) uses the input values, the magic bias the f16-rounded ones.
template <sfmp_dtype DT>
__global__ void __launch_bounds__(256) xprep_rows_kernel(const XParams xp) {
    using T = typename XT<DT>::T;
    pdl_launch_dependents();  // let the GEMV start streaming weights right away
    extern __shared__ __align__(16) uint8_t xsm[];
    const int dbg = xp.dbg;
    if (blockIdx.x == 0 && threadIdx.x == 0 && dbg == 5) {
        // previous launch's GEMV end (complete: stream order), then this start
        g_dbg_timeline[(kDbgCtas - 1) * kDbgSlots + 104] = g_dbg_timeline[(kDbgCtas - 1) * kDbgSlots + 102];
        DBG_KSTAMP(100);
    }
    const int n_b = xp.n_b, CH = n_b >> 7;
    int it = blockIdx.x, li = 0;  // compact grid: (linear, token, 8 block columns)
    while (li + 1 < xp.nlin && it >= xp.lin[li + 1].item0) ++li;
    const XLin& XL = xp.lin[li];
    const int M = XL.M;
    it -= XL.item0;
    const int nit = (XL.BC + 7) / 8;
    const int t = it / nit;
    it -= t * nit;
    const int bc0 = it * 8, nbc = min(8, XL.BC - bc0), cols = XL.cols;
    uint32_t* cp = reinterpret_cast<uint32_t*>(xsm);  // [nbc][n_b] column indices
    T* xr = reinterpret_cast<T*>(xsm + 8 * n_b * 4);  // x[t][0..cols)
    {
        const uint4* src = reinterpret_cast<const uint4*>(XL.col_perm + static_cast<size_t>(bc0) * n_b);
        const uint64_t keep = policy_evict_last();
        for (int i = threadIdx.x; i < nbc * n_b / 4; i += 256) reinterpret_cast<uint4*>(cp)[i] = ldg_keep_v4(src + i, keep);
        const T* xrow = static_cast<const T*>(XL.x) + static_cast<size_t>(t) * cols;
        if ((reinterpret_cast<uintptr_t>(xrow) & 15) == 0) {
            const int nv = cols * static_cast<int>(sizeof(T)) / 16;  // cols % 128 == 0
            for (int i = threadIdx.x; i < nv; i += 256)
                reinterpret_cast<uint4*>(xr)[i] = __ldg(reinterpret_cast<const uint4*>(xrow) + i);
        } else {
            for (int i = threadIdx.x; i < cols; i += 256) xr[i] = xrow[i];
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp >= nbc) return;
    const int bc = bc0 + warp, s8 = lane >> 2, q = lane & 3;
    const RecGeom G{M};
    uint8_t* rec = XL.xrec + static_cast<size_t>(bc) * XL.rec_bytes;
    const uint32_t* cpw = cp + warp * n_b;
    const int lo = XL.lo;
    auto mag = [](int B, int j) { return B <= 4 ? rp_magic(B, j) : 0.f; };
    const float mlx = mag(lo, 2 * s8), mly = mag(lo, 2 * s8 + 1);
    const float mhx = mag(lo + 1, 2 * s8), mhy = mag(lo + 1, 2 * s8 + 1);
    const int kb = 32 * q + 8 * (s8 & 1) + (s8 >> 1);
    float xs = 0.f, bias_lo = 0.f, bias_hi = 0.f;
    for (int c = 0; c < CH; ++c) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) v[j * 2 + e] = XT<DT>::f(xr[cpw[c * 128 + kb + 4 * j + 16 * e]]);
        uint2 st;
        st.x = h2_as_u32(__floats2half2_rn(v[0], v[1]));  // pairs with A register 2*s8
        st.y = h2_as_u32(__floats2half2_rn(v[2], v[3]));  // ... and 2*s8+1
        *reinterpret_cast<uint2*>(rec + G.frag_off(c, t >> 3, s8, t & 7, q)) = st;
        const float sx = __low2float(u32_as_h2(st.x)) + __high2float(u32_as_h2(st.x));
        const float sy = __low2float(u32_as_h2(st.y)) + __high2float(u32_as_h2(st.y));
        bias_lo += mlx * sx + mly * sy;
        bias_hi += mhx * sx + mhy * sy;
        xs += (v[0] + v[1]) + (v[2] + v[3]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        xs += __shfl_xor_sync(0xffffffffu, xs, o);
        bias_lo += __shfl_xor_sync(0xffffffffu, bias_lo, o);
        bias_hi += __shfl_xor_sync(0xffffffffu, bias_hi, o);
    }
    if (lane == 0) {
        float* xg = reinterpret_cast<float*>(rec + G.xg_off(CH));
        xg[t] = xs;
        xg[bias_slot(t, 0)] = xg[bias_slot(t, 0) + 2] = -bias_lo;
        xg[bias_slot(t, 1)] = xg[bias_slot(t, 1) + 2] = -bias_hi;
        if (t == M - 1)  // token columns the GEMV computes but never stores
            for (int u = M; u < 8 * G.nt_count(); ++u)
                xg[u] = xg[bias_slot(u, 0)] = xg[bias_slot(u, 0) + 2] = xg[bias_slot(u, 1)] = xg[bias_slot(u, 1) + 2] = 0.f;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) DBG_KSTAMP(101);
    // When launched to overlap the previous GEMV of the same grouped call, do
    // not complete before it: this grid's completion (which the next GEMV waits
    // for) then implies the previous launch's, keeping stream order for any
    // later work.  A no-op for a normal launch.
    if (xp.wait_prev) pdl_wait();
}

// Fallback for x rows above kXprepRowLimit bytes.
// K4 (decode flavour): gather x[t][col_perm[.]] once per call into per-block-
// column records laid out exactly as the MMA B fragments the GEMV consumes,
// plus per-token column sums X_g (lutgemm.cpp:113-115) and the magic-offset
// bias.  One item per (block column, n-tile); its CH 128-column chunks go to
// CH warps of one CTA (so the col_perm -> x dependent loads of the chunks are
// in flight together), whose sums are combined in chunk order through shared
// memory.  Lane (n,q) owns token nt*8+n and k-slots 32q + 4h + a (+16).
template <sfmp_dtype DT>
__global__ void __launch_bounds__(256) xprep_kernel(const XParams xp) {
    pdl_launch_dependents();  // let the GEMV start streaming weights right away
    __shared__ float red[8][3][8];
    const int dbg = xp.dbg;
    if (blockIdx.x == 0 && threadIdx.x == 0 && dbg == 5) {
        // previous launch's GEMV end (complete: stream order), then this start
        g_dbg_timeline[(kDbgCtas - 1) * kDbgSlots + 104] = g_dbg_timeline[(kDbgCtas - 1) * kDbgSlots + 102];
        DBG_KSTAMP(100);
    }
    const int n_b = xp.n_b;
    const int NT = RecGeom{xp.M}.nt_count();  // per launch (its linears share the n-tile count)
    const int CH = n_b >> 7;  // 1..8 (host: 8 % CH == 0)
    const int warp = threadIdx.x >> 5, c = warp % CH;
    int w = blockIdx.x * (8 / CH) + warp / CH;  // item
    int li = 0;
    while (li + 1 < xp.nlin && w >= xp.lin[li + 1].warp0) ++li;
    const XLin& XL = xp.lin[li];
    w -= XL.warp0;
    const int M = XL.M;
    const uint32_t rec_bytes = XL.rec_bytes;
    const RecGeom G{M};
    const int BC = XL.BC, cols = XL.cols;
    const void* x = XL.x;
    const uint32_t* col_perm = XL.col_perm;
    uint8_t* xrec = XL.xrec;
    const int lo = XL.lo;
    const bool item_ok = w < BC * NT;
    const int bc = w / NT, nt = w - bc * NT;
    const int lane = threadIdx.x & 31, q = lane & 3, n = lane >> 2;
    const int t = nt * 8 + n;
    const bool live = item_ok && n < G.mnt(nt);
    uint8_t* rec = xrec + static_cast<size_t>(bc) * rec_bytes;
    float xs = 0.f, bias_lo = 0.f, bias_hi = 0.f;
    if (item_ok) {
        const uint4 idx4 =
            ldg_keep_v4(reinterpret_cast<const uint4*>(col_perm + bc * n_b + c * 128) + lane, policy_evict_last());
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
        if (live) {
            const size_t rowoff = static_cast<size_t>(t) * cols;
            float v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = load_x<DT>(x, rowoff + gi[e]);
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) {
                uint2 st;
                st.x = h2_as_u32(__floats2half2_rn(v[s8 * 4 + 0], v[s8 * 4 + 1]));
                st.y = h2_as_u32(__floats2half2_rn(v[s8 * 4 + 2], v[s8 * 4 + 3]));
                *reinterpret_cast<uint2*>(rec + G.frag_off(c, nt, s8, n, q)) = st;
                // st.x pairs with A register 2*s8, st.y with 2*s8+1; each carries the
                // magic of its register in the repacked layout of a lo / lo+1 bit
                // unit (0 for the exact >4-bit path).  The bias uses the f16-rounded
                // values the MMA sees.
                const float sx = __low2float(u32_as_h2(st.x)) + __high2float(u32_as_h2(st.x));
                const float sy = __low2float(u32_as_h2(st.y)) + __high2float(u32_as_h2(st.y));
                auto mag = [](int B, int j) { return B <= 4 ? rp_magic(B, j) : 0.f; };
                bias_lo += mag(lo, 2 * s8) * sx + mag(lo, 2 * s8 + 1) * sy;
                bias_hi += mag(lo + 1, 2 * s8) * sx + mag(lo + 1, 2 * s8 + 1) * sy;
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) xs += v[e];
        }
        xs += __shfl_xor_sync(0xffffffffu, xs, 1);
        xs += __shfl_xor_sync(0xffffffffu, xs, 2);
        bias_lo += __shfl_xor_sync(0xffffffffu, bias_lo, 1);
        bias_lo += __shfl_xor_sync(0xffffffffu, bias_lo, 2);
        bias_hi += __shfl_xor_sync(0xffffffffu, bias_hi, 1);
        bias_hi += __shfl_xor_sync(0xffffffffu, bias_hi, 2);
    }
    if (CH > 1) {
        if (q == 0) {
            red[warp][0][n] = xs;
            red[warp][1][n] = bias_lo;
            red[warp][2][n] = bias_hi;
        }
        __syncthreads();
        if (c != 0) return;
        if (q == 0) {
            xs = bias_lo = bias_hi = 0.f;
            for (int k = 0; k < CH; ++k) {
                xs += red[warp + k][0][n];
                bias_lo += red[warp + k][1][n];
                bias_hi += red[warp + k][2][n];
            }
        }
    }
    if (item_ok && q == 0) {
        float* xg = reinterpret_cast<float*>(rec + G.xg_off(CH));
        const int tt = nt * 8 + n;
        xg[tt] = live ? xs : 0.f;
        xg[bias_slot(tt, 0)] = xg[bias_slot(tt, 0) + 2] = live ? -bias_lo : 0.f;
        xg[bias_slot(tt, 1)] = xg[bias_slot(tt, 1) + 2] = live ? -bias_hi : 0.f;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) DBG_KSTAMP(101);
}

// One 128-column chunk of a unit for this warp's 32 rows (2 m16 tiles), four
// independent accumulator chains (m-tile x even/odd k-step).  prow / xb are
// 32-bit shared addresses; all other offsets are compile-time immediates.
template <int B, int NT, int CH>
__device__ __forceinline__ void unit_chunk(uint32_t prow, const uint32_t (&xb)[NT], int chunk_bytes, int c,
                                           float (&cacc)[kMT][NT][4]) {
    constexpr int NB8 = CH * 16;   // bytes of one row of one plane
    constexpr int PS = kTR * NB8;  // bytes of one plane of the unit
    // rows r0 + 8*r: (r0, r0+8) is m-tile 0, (r0+16, r0+24) m-tile 1
    uint32_t p[2 * kMT][B];
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
        for (int r = 0; r < 2 * kMT; ++r) p[r][i] = lds_u32(prow + i * PS + r * 8 * NB8 + c * 16);
    uint32_t A[2 * kMT][16];
#pragma unroll
    for (int r = 0; r < 2 * kMT; ++r) {
        if constexpr (B <= 4) unpack_rp<B>(p[r], A[r]);  // repacked layout (repack.cuh)
        else unpack_word<B>(p[r], A[r]);                // bit planes, exact codes
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const uint2 b = lds_v2(xb[nt] + c * chunk_bytes + s * 32);
#pragma unroll
            for (int m = 0; m < kMT; ++m)
                mma_16816(cacc[m][nt], A[2 * m][2 * s], A[2 * m + 1][2 * s], A[2 * m][2 * s + 1],
                          A[2 * m + 1][2 * s + 1], b.x, b.y);
        }
    }
}

// LO = the model's floor bit-width: every unit has LO or LO+1 bits
// (PackedModel::validate, layout.cpp:100-103), so the kernel carries exactly
// two unpack paths and its hot loop stays resident in the instruction cache.
// Work split: all units of all linears form one sequence (linear, row tile,
// block column); CTA b streams units [b*Q, (b+1)*Q) -- equal work per CTA,
// one wave.  A CTA's range is cut into segments at row-tile boundaries; a
// row tile covered by several CTAs is reduced split-K style (part k of the
// tile = the k-th CTA that touches it, summed in k order).
struct Seg {
    int li, rt, bc0, bc1;  // units [bc0, bc1) of row tile rt of linear li
    int k, C;              // this CTA is the k-th of the C CTAs touching the tile
};
__device__ __forceinline__ Seg seg_at(const Params& p, int64_t u, int64_t end) {
    int li = 0;
    while (li + 1 < p.nlin && u >= p.lin[li + 1].unit0) ++li;
    const Lin& L = p.lin[li];
    const int64_t rel = u - L.unit0;
    Seg sg;
    sg.li = li;
    sg.rt = static_cast<int>(rel / L.BC);
    sg.bc0 = static_cast<int>(rel - static_cast<int64_t>(sg.rt) * L.BC);
    const int64_t t0 = L.unit0 + static_cast<int64_t>(sg.rt) * L.BC, t1 = t0 + L.BC;  // tile's unit range
    sg.bc1 = static_cast<int>((end < t1 ? end : t1) - t0);
    const int64_t c0 = t0 / p.Q, c1 = (t1 - 1) / p.Q;
    sg.C = static_cast<int>(c1 - c0 + 1);
    sg.k = static_cast<int>(static_cast<int64_t>(blockIdx.x) - c0);
    return sg;
}

// LO = the model's floor bit-width: every unit has LO or LO+1 bits
// (PackedModel::validate, layout.cpp:100-103), so the kernel carries exactly
// two unpack paths and its hot loop stays resident in the instruction cache.
template <int NT, int CH, int LO>
__global__ void __launch_bounds__(kThreads, ctas_per_sm(NT)) gemv_kernel(const Params p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    uint8_t* zeros = smem + 256;                               // 256 B: B fragments of absent tokens
    uint32_t* sbits = reinterpret_cast<uint32_t*>(smem + 512);  // bit-width of the unit in stage s
    uint32_t* flag = reinterpret_cast<uint32_t*>(smem + 640);    // "this CTA finishes the tile"
    uint8_t* wbase = smem + kHdrBytes;
    uint8_t* xbase = wbase + static_cast<size_t>(S) * p.stage_w;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int dbg = p.debug_mode;
    // a programmatic dependent (only ever the next launch of the same grouped
    // call, whose problems are independent of ours) may start now
    pdl_launch_dependents();
    if (threadIdx.x == 0) DBG_STAMP(0);
    if (threadIdx.x == 0 && dbg == 5 && blockIdx.x < kDbgCtas - 1) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_dbg_timeline[blockIdx.x * kDbgSlots + 123] = smid;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNCW);
        }
        fence_mbar_init();
        fence_proxy_async();
    }
    if (threadIdx.x < 64) reinterpret_cast<uint32_t*>(zeros)[threadIdx.x] = 0u;
    __syncthreads();

    constexpr int nb8 = CH * 16;

    if (warp == 0) {
        // ---------------- producer: one bulk copy per unit (+ its activation record) ----
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const uint64_t keep = policy_evict_last();
            const uint32_t pbytes = kTR * nb8;
            int gi = 0;  // unit counter of this CTA (debug stamps)
            auto issue_w = [&](int s, const Lin& L, uint64_t d) {
                const int bits = static_cast<int>((d >> 48) & 0xF);
                sbits[s] = static_cast<uint32_t>(bits);  // published by the arrive below
                DBG_USTAMP(2 + 3 * gi);
                const uint32_t wbytes = 4 * kTR + bits * pbytes;
                mbar_arrive_expect_tx(&full[s], wbytes + L.rec_bytes);
                bulk_g2s(wbase + static_cast<size_t>(s) * p.stage_w, L.payload + (d & 0xFFFFFFFFFFFFull), wbytes,
                         &full[s], pol);
            };
            auto issue_x = [&](int s, const Lin& L, int bc_) {
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(xbase + static_cast<size_t>(s) * p.rec_bytes)),
                    "l"(L.xrec + static_cast<size_t>(bc_) * L.rec_bytes), "r"(L.rec_bytes), "r"(smem_u32(&full[s]))
                    : "memory");
            };
            int s = 0, ph = 0;
            bool first = true;
            const int64_t uend = min(p.units, (static_cast<int64_t>(blockIdx.x) + 1) * p.Q);
            for (int64_t u = static_cast<int64_t>(blockIdx.x) * p.Q; u < uend;) {
                const Seg I = seg_at(p, u, uend);
                u += I.bc1 - I.bc0;
                const Lin& L = p.lin[I.li];
                const uint64_t* gdesc = L.unit_desc + static_cast<size_t>(I.rt) * L.BC + I.bc0;
                const int nunits = I.bc1 - I.bc0;
                int i0 = 0;
                if (first) {
                    // weights of the first ring-full do not depend on x: issue them,
                    // then wait for the activation records (programmatic dependent launch)
                    const int pre = nunits < S ? nunits : S;
                    uint64_t dpre[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (i < pre) dpre[i] = ldg_keep_u64(gdesc + i, keep);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (i < pre) {
                            issue_w(i, L, dpre[i]);
                            ++gi;
                        }
                    pdl_wait();
                    for (int i = 0; i < pre; ++i) issue_x(i, L, I.bc0 + i);
                    s = pre % S;
                    ph = pre == S ? 1 : 0;
                    i0 = pre;
                    first = false;
                }
                uint64_t dnext = i0 < nunits ? ldg_keep_u64(gdesc + i0, keep) : 0;
                for (int i = i0; i < nunits; ++i) {
                    const uint64_t d = dnext;
                    if (i + 1 < nunits) dnext = ldg_keep_u64(gdesc + i + 1, keep);
                    mbar_wait(&empty[s], ph ^ 1);
                    issue_w(s, L, d);
                    issue_x(s, L, I.bc0 + i);
                    ++gi;
                    if (++s == S) { s = 0; ph ^= 1; }
                }
            }
        }
    } else {
        // ---------------- compute warps ------------------------------------------
        const int cw = warp - 1;
        const int g = lane >> 2, q = lane & 3;
        const int r0 = cw * 16 * kMT + g;  // rows r0 + 8*r of the tile
        const uint32_t stage_w = p.stage_w, rec_bytes = p.rec_bytes;
        // per-lane shared addresses for stage 0; a stage adds s * stage_w / rec_bytes
        const uint32_t prow0 = smem_u32(wbase) + 4 * kTR + r0 * nb8 + q * 4;
        const uint32_t sz0 = smem_u32(wbase) + 2 * r0;
        // record addresses depend on the linear's M: set per segment
        int chunk_bytes = 0, cur_li = -1;
        uint32_t xb0[NT], xstep[NT], xg0 = 0, bc_a = 0;
        const uint32_t sbits_a = smem_u32(sbits);
        const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty);
        int s = 0, ph = 0, gi = 0;
        uint32_t wo = 0, xo = 0;  // byte offsets of stage s in the weight / record rings
        const int64_t uend = min(p.units, (static_cast<int64_t>(blockIdx.x) + 1) * p.Q);
        for (int64_t u = static_cast<int64_t>(blockIdx.x) * p.Q; u < uend;) {
            const Seg I = seg_at(p, u, uend);
            u += I.bc1 - I.bc0;
            const Lin& L = p.lin[I.li];
            const int C = I.C, rt = I.rt, nunits = I.bc1 - I.bc0;
            if (I.li != cur_li) {
                cur_li = I.li;
                const RecGeom GL{L.M};
                chunk_bytes = GL.chunk_bytes();
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const bool live = g < GL.mnt(nt);
                    xb0[nt] = live ? smem_u32(xbase) + GL.lane_off(0, nt, g, q) : smem_u32(zeros) + q * 8;
                    xstep[nt] = live ? rec_bytes : 0u;
                }
                xg0 = smem_u32(xbase) + GL.xg_off(CH) + 8 * q;
                bc_a = smem_u32(xbase) + GL.xg_off(CH) + 64 + 16 * q;  // accumulator inits
            }
            float yacc[kMT][NT][4];
#pragma unroll
            for (int m = 0; m < kMT; ++m)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) yacc[m][nt][e] = 0.f;
            for (int i = 0; i < nunits; ++i, ++gi) {
                mbar_wait_a(full_a + 8 * s, ph);
                if (cw == 0 && lane == 0) DBG_USTAMP(3 + 3 * gi);
                const int bits = static_cast<int>(lds_u32(sbits_a + 4 * s));
                uint32_t xb[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) xb[nt] = xb0[nt] + (xstep[nt] ? xo : 0u);
                const uint32_t prow = prow0 + wo;
                // accumulators start at -bias (this unit's layout): C - bias from the MMA
                const uint32_t xg = xg0 + xo;
                const uint32_t binit = bc_a + xo + (bits == LO ? 0u : 128u);
                float cacc[kMT][NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const uint4 b4 = lds_v4(binit + 64 * nt);
#pragma unroll
                    for (int h = 0; h < kMT; ++h) {
                        cacc[h][nt][0] = __uint_as_float(b4.x);
                        cacc[h][nt][1] = __uint_as_float(b4.y);
                        cacc[h][nt][2] = __uint_as_float(b4.z);
                        cacc[h][nt][3] = __uint_as_float(b4.w);
                    }
                }
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    if (bits == LO) {
                        unit_chunk<LO, NT, CH>(prow, xb, chunk_bytes, c, cacc);
                    } else if constexpr (LO < 8) {
                        unit_chunk<LO + 1, NT, CH>(prow, xb, chunk_bytes, c, cacc);
                    }
                }
                // per-row affine of this block: y += s*(C - bias) + z*Xg
                const uint32_t sz = sz0 + wo;
#pragma unroll
                for (int m = 0; m < kMT; ++m) {
                    const float sa = lds_h2f(sz + 32 * m), sb = lds_h2f(sz + 32 * m + 16);
                    const float za = lds_h2f(sz + 2 * kTR + 32 * m), zb = lds_h2f(sz + 2 * kTR + 32 * m + 16);
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const float2 xg01 = lds_f2(xg + 32 * nt);
                        const float* c0 = cacc[m][nt];  // = C - bias
                        yacc[m][nt][0] = fmaf(sa, c0[0], fmaf(za, xg01.x, yacc[m][nt][0]));
                        yacc[m][nt][1] = fmaf(sa, c0[1], fmaf(za, xg01.y, yacc[m][nt][1]));
                        yacc[m][nt][2] = fmaf(sb, c0[2], fmaf(zb, xg01.x, yacc[m][nt][2]));
                        yacc[m][nt][3] = fmaf(sb, c0[3], fmaf(zb, xg01.y, yacc[m][nt][3]));
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_a(empty_a + 8 * s);
                if (cw == 0 && lane == 0) DBG_USTAMP(4 + 3 * gi);
                wo += stage_w;
                xo += rec_bytes;
                if (++s == S) { s = 0; ph ^= 1; wo = 0; xo = 0; }
            }
            if (C == 1) {
                // whole row tile in this item: un-permuted store straight to y
#pragma unroll
                for (int m = 0; m < kMT; ++m)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int t = nt * 8 + 2 * q + (e & 1);
                            if (t < L.M)
                                L.y[t * L.out_rows + __ldg(L.out_map + rt * kTR + r0 + 16 * m + 8 * (e >> 1))] =
                                    yacc[m][nt][e];
                        }
                continue;
            }
            // split-K partial tile [t][128 rows] of this item (coalesced rows)
            float* part = L.part + (static_cast<size_t>(rt) * kMaxSplit + I.k) * (16 * kTR);
#pragma unroll
            for (int m = 0; m < kMT; ++m)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int t = nt * 8 + 2 * q + (e & 1);
                        if (t < L.M) part[t * kTR + r0 + 16 * m + 8 * (e >> 1)] = yacc[m][nt][e];
                    }
            // Deterministic split-K: the last of the C items of this row tile
            // sums the partials in split order and stores them un-permuted.
            // Compute warps only (the producer streams on): named barrier 1.
            named_bar_sync(1, kNCW * 32);  // every partial store precedes the release below
            if (threadIdx.x == 32) DBG_STAMP(124);
            if (threadIdx.x == 32) {
                const unsigned old = atomic_add_acq_rel_gpu(L.counters + rt, 1u);
                *flag = (old == static_cast<unsigned>(C - 1)) ? 1u : 0u;
            }
            named_bar_sync(1, kNCW * 32);
            if (threadIdx.x == 32) DBG_STAMP(125);
            if (*flag) {
                // Acquire by thread 32 (it also invalidates this SM's L1) + the
                // barrier order these plain loads after every partial store
                // (the semaphore pattern).  Weak loads: a strong ld.cg is
                // issued one at a time.
                // One row per thread, all tokens; RB splits per round so that
                // RB*8*NT loads are in flight together (latency, not bandwidth).
                static_assert(kNCW * 32 >= kTR, "fixup maps one compute thread per row");
                constexpr int RB = NT == 1 ? 4 : 2;
                const int row = threadIdx.x - 32;
                if (row < kTR) {
                const float* pp = L.part + static_cast<size_t>(rt) * kMaxSplit * (16 * kTR) + row;
                const uint32_t orow = __ldg(L.out_map + rt * kTR + row);
                float acc[8 * NT];
#pragma unroll
                for (int t = 0; t < 8 * NT; ++t) acc[t] = 0.f;
                for (int r0 = 0; r0 < C; r0 += RB) {
                    float v[RB][8 * NT];
#pragma unroll
                    for (int r = 0; r < RB; ++r)
#pragma unroll
                        for (int t = 0; t < 8 * NT; ++t)
                            v[r][t] = (r0 + r < C && t < L.M)
                                          ? pp[static_cast<size_t>(r0 + r) * (16 * kTR) + t * kTR]
                                          : 0.f;
#pragma unroll
                    for (int r = 0; r < RB; ++r)
#pragma unroll
                        for (int t = 0; t < 8 * NT; ++t)
                            if (r0 + r < C) acc[t] += v[r][t];  // split order, as the partials were cut
                }
#pragma unroll
                for (int t = 0; t < 8 * NT; ++t)
                    if (t < L.M) L.y[t * L.out_rows + orow] = acc[t];
                }
                if (threadIdx.x == 32) L.counters[rt] = 0u;  // ready for the next call (stream-ordered)
                if (threadIdx.x == 32) DBG_STAMP(126);
            }
        }
    }
    if (threadIdx.x == 0) DBG_STAMP(1);
    if (threadIdx.x == 32) DBG_STAMP(127);
    if (dbg == 5 && threadIdx.x == 32) {  // kernel-level: max end over all CTAs (compute warps)
        atomicMax(&g_dbg_timeline[(kDbgCtas - 1) * kDbgSlots + 102], gtimer());
        if (blockIdx.x == gridDim.x - 1) g_dbg_timeline[(kDbgCtas - 1) * kDbgSlots + 103] = gridDim.x;
    }
}

template <int NT, int CH, int LO>
cudaError_t launch_k(cudaLaunchConfig_t& cfg, const Params& p) {
    auto k = gemv_kernel<NT, CH, LO>;
    static int configured[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_per_cta(NT));
        if (e != cudaSuccess) return e;
        configured[dev] = 1;
    }
    return cudaLaunchKernelEx(&cfg, k, p);
}

template <int NT, int CH>
cudaError_t launch_nc(cudaLaunchConfig_t& cfg, const Params& p, int lo) {
    switch (lo) {
        case 1: return launch_k<NT, CH, 1>(cfg, p);
        case 2: return launch_k<NT, CH, 2>(cfg, p);
        case 3: return launch_k<NT, CH, 3>(cfg, p);
        case 4: return launch_k<NT, CH, 4>(cfg, p);
        case 5: return launch_k<NT, CH, 5>(cfg, p);
        case 6: return launch_k<NT, CH, 6>(cfg, p);
        case 7: return launch_k<NT, CH, 7>(cfg, p);
        default: return launch_k<NT, CH, 8>(cfg, p);
    }
}

template <sfmp_dtype DT>
cudaError_t launch_t(const Params& p, const XParams& xp, int xwarps, int xitems, int max_cols, int grid, size_t smem, int lo,
                     cudaStream_t st, bool overlap_prev) {
    const size_t elem = DT == SFMP_F32 ? 4 : 2;
    // K4: activation records (normal launch: it overwrites the workspace the
    // previous call may still read, and x may be that call's output, so it
    // follows it in stream order).  Measured: chaining it programmatically
    // lets the next GEMV's CTAs occupy slots early and slows both calls.
    const int NT = p.M > 8 ? 2 : 1;
    {
        // Same shared-memory carveout as the GEMV: an SM running a pre-pass CTA
        // then needs no reconfiguration (which waits for the SM to drain)
        // before the GEMV's CTAs can join it.
        static int configured[64] = {0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 64 && !configured[dev]) {
            cudaFuncSetAttribute(xprep_kernel<DT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
            configured[dev] = 1;
        }
    }
    const size_t row_smem = static_cast<size_t>(8) * p.n_b * 4 + static_cast<size_t>(max_cols) * elem;
    if (row_smem <= static_cast<size_t>(kXprepRowLimit)) {
        static int configured_rows[64] = {0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 64 && !configured_rows[dev]) {
            cudaFuncSetAttribute(xprep_rows_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kXprepRowLimit);
            cudaFuncSetAttribute(xprep_rows_kernel<DT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
            configured_rows[dev] = 1;
        }
        // overlap_prev: a later launch of one grouped call (independent problems,
        // workspaces disjoint from the earlier launches'): the pre-pass may start
        // while the previous GEMV still runs (it never waits on it), and this
        // call's GEMV then fills the previous one's tail.
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = overlap_prev ? 1 : 0;
        XParams xq = xp;
        xq.wait_prev = overlap_prev ? 1 : 0;
        cudaLaunchConfig_t c{};
        c.gridDim = dim3(xitems);
        c.blockDim = dim3(256);
        c.dynamicSmemBytes = row_smem;
        c.stream = st;
        c.attrs = a;
        c.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&c, xprep_rows_kernel<DT>, xq);
        if (e != cudaSuccess) return e;
    } else {
        const int per_cta = 8 / (p.n_b / 128);  // items per pre-pass CTA
        xprep_kernel<DT><<<(xwarps + per_cta - 1) / per_cta, 256, 0, st>>>(xp);
    }
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    // K1: C CTAs per 128-row tile of every linear, programmatic dependent of xprep
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    const int CH = p.n_b / 128;
    if (NT == 1) return CH == 1 ? launch_nc<1, 1>(cfg, p, lo) : launch_nc<1, 2>(cfg, p, lo);
    return CH == 1 ? launch_nc<2, 1>(cfg, p, lo) : launch_nc<2, 2>(cfg, p, lo);
}

}  // namespace

// Not part of the ABI: copies the debug timeline (SFMP_GEMV_DEBUG=5) to the host.
extern "C" int sfmp_debug_gemv_timeline(unsigned long long* host, size_t n) {
    if (n > static_cast<size_t>(kDbgCtas) * kDbgSlots) n = static_cast<size_t>(kDbgCtas) * kDbgSlots;
    return static_cast<int>(cudaMemcpyFromSymbol(host, g_dbg_timeline, n * sizeof(unsigned long long)));
}

// Workspace: activation records | split-K partials | completion counters.
size_t gemv_rec_bytes(const DevModel& m) {
    return (static_cast<size_t>(m.BC) * RecGeom{16}.bytes(static_cast<int>(m.n_b / 128)) + 255) / 256 * 256;
}
size_t gemv_part_bytes(const DevModel& m) {
    return static_cast<size_t>(m.RT) * kMaxSplit * 16 * kTR * 4;
}
size_t gemv_workspace_bytes(const DevModel& m, int M) {
    (void)M;
    return gemv_rec_bytes(m) + gemv_part_bytes(m) + static_cast<size_t>(m.RT) * 4;
}

int gemv_ctas_per_sm(int NT) { return ctas_per_sm(NT); }

bool gemv_groupable(const DevModel& a, const DevModel& b) {
    return a.gemv_ok && b.gemv_ok && a.n_b == b.n_b && a.floor_bits == b.floor_bits && a.device == b.device;
}

cudaError_t launch_gemv_group(const DevModel* const* ms, const void* const* xs, float* const* ys, uint8_t* const* wss,
                              const int* Ms, int n, sfmp_dtype dt, cudaStream_t st, bool overlap_prev) {
    if (n < 1 || n > kMaxLin) return cudaErrorInvalidValue;
    const DevModel& m0 = *ms[0];
    int M = 0;
    for (int i = 0; i < n; ++i) {
        if (Ms[i] < 1 || Ms[i] > 16) return cudaErrorInvalidValue;
        M = std::max(M, Ms[i]);
    }
    const int NT = M > 8 ? 2 : 1;
    for (int i = 0; i < n; ++i)
        if ((Ms[i] > 8 ? 2 : 1) != NT) return cudaErrorInvalidValue;  // one n-tile count per launch
    const int CH = static_cast<int>(m0.n_b / 128);
    Params p{};
    XParams xp{};
    p.nlin = xp.nlin = n;
    p.M = xp.M = M;
    p.n_b = xp.n_b = static_cast<int>(m0.n_b);
    p.rec_bytes = xp.rec_bytes = static_cast<uint32_t>(RecGeom{M}.bytes(CH));  // stage stride: the largest
    {
        const char* dbg = getenv("SFMP_GEMV_DEBUG");
        p.debug_mode = xp.dbg = dbg ? atoi(dbg) : 0;
    }
    // split-K: every CTA gets ~U units so that all linears' CTAs fit one wave
    // of resident slots with equal work (balanced across the group)
    int ceil_bits = 0;
    int64_t units = 0;
    for (int i = 0; i < n; ++i) {
        units += static_cast<int64_t>(ms[i]->RT) * ms[i]->BC;
        ceil_bits = std::max(ceil_bits, ms[i]->ceil_bits);
    }
    const int slots = m0.num_sms * ctas_per_sm(NT);
    // One wave: G CTAs, each Q consecutive units of the group's unit sequence
    // (Q large enough that no row tile is shared by more than kMaxSplit CTAs).
    int max_bc = 1;
    for (int i = 0; i < n; ++i) max_bc = std::max(max_bc, static_cast<int>(ms[i]->BC));
    int64_t Q = std::max<int64_t>({2, (units + slots - 1) / slots, (max_bc + kMaxSplit - 2) / (kMaxSplit - 1)});
    if (const char* e = getenv("SFMP_GEMV_Q")) Q = std::max<int64_t>(Q, atoi(e));
    int64_t unit0 = 0;
    int xwarps = 0, xitems = 0, max_cols = 0;
    for (int i = 0; i < n; ++i) {
        const DevModel& m = *ms[i];
        Lin& L = p.lin[i];
        const int BC = static_cast<int>(m.BC);
        L.payload = m.d_payload;
        L.unit_desc = m.d_unit_desc;
        L.out_map = m.d_out_map;
        L.xrec = wss[i];
        L.y = ys[i];
        L.part = reinterpret_cast<float*>(wss[i] + gemv_rec_bytes(m));
        L.counters = reinterpret_cast<unsigned*>(wss[i] + gemv_rec_bytes(m) + gemv_part_bytes(m));
        L.out_rows = m.out_rows;
        L.BC = BC;
        L.M = Ms[i];
        L.rec_bytes = static_cast<uint32_t>(RecGeom{Ms[i]}.bytes(CH));
        L.unit0 = unit0;
        unit0 += static_cast<int64_t>(m.RT) * BC;
        XLin& X = xp.lin[i];
        X.x = xs[i];
        X.col_perm = m.d_col_perm;
        X.xrec = wss[i];
        X.BC = BC;
        X.cols = static_cast<int>(m.cols);
        X.warp0 = xwarps;
        X.item0 = xitems;
        X.lo = m.floor_bits;
        X.M = Ms[i];
        X.rec_bytes = L.rec_bytes;
        xwarps += BC * NT;
        xitems += (BC + 7) / 8 * Ms[i];  // pre-pass CTAs: (8 block columns) x tokens
        max_cols = std::max(max_cols, X.cols);
    }
    p.stage_w = static_cast<uint32_t>((4 * kTR + ceil_bits * kTR * (m0.n_b / 8) + 127) / 128 * 128);
    int max_stages = 4;
    if (const char* ss = getenv("SFMP_GEMV_STAGES")) max_stages = std::max(2, atoi(ss));
    const int fixed = kHdrBytes;
    const int stages = std::min<int>(max_stages, (smem_per_cta(NT) - fixed) / static_cast<int>(p.stage_w + p.rec_bytes));
    if (stages < 2) return cudaErrorInvalidConfiguration;
    p.stages = stages;
    const size_t smem = fixed + static_cast<size_t>(stages) * (p.stage_w + p.rec_bytes);
    p.units = unit0;
    p.Q = Q;
    const int grid = static_cast<int>((unit0 + Q - 1) / Q);
    switch (dt) {
        case SFMP_F32: return launch_t<SFMP_F32>(p, xp, xwarps, xitems, max_cols, grid, smem, m0.floor_bits, st, overlap_prev);
        case SFMP_F16: return launch_t<SFMP_F16>(p, xp, xwarps, xitems, max_cols, grid, smem, m0.floor_bits, st, overlap_prev);
        default: return launch_t<SFMP_BF16>(p, xp, xwarps, xitems, max_cols, grid, smem, m0.floor_bits, st, overlap_prev);
    }
}

cudaError_t launch_gemv(const DevModel& m, const void* x, sfmp_dtype dt, int M, float* y, float* ws,
                        cudaStream_t st) {
    const DevModel* ms[1] = {&m};
    const void* xs[1] = {x};
    float* ys[1] = {y};
    uint8_t* wss[1] = {reinterpret_cast<uint8_t*>(ws)};
    const int Ms[1] = {M};
    return launch_gemv_group(ms, xs, ys, wss, Ms, 1, dt, st, false);
}

}  // namespace sfmpk
