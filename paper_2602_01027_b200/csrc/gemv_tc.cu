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
//  * Canonical accumulation order ("independent of thread count,
//    deterministic merge"): every 128-row tile is cut into fixed K segments of
//    kSegCols = 1024 columns.  A segment's units are folded sequentially from
//    zero; the segment sums of a tile are added in segment order.  The cut
//    depends on the matrix alone, so a linear's output bits do not depend on
//    the grid, the SM count, the other linears of a grouped launch, the
//    number of shards or the token count M (MMA columns are independent).
//  * Work items = (linear, tile, segment), handed out by a global queue
//    (one atomic per item, claimed one item ahead by the producer), so SMs
//    that run ahead take more items and all finish together.  A segment of a
//    multi-segment tile stores its f32 partial and moves on (no barrier, no
//    fence in the GEMV); gemv_fixup_kernel, a programmatic dependent launch,
//    sums each tile's partials in segment order and stores the un-permuted
//    rows (no float atomics).
//  * The activation gather x[t][col_perm[.]] runs once per call in a small
//    pre-pass (xprep_*) that writes, per block column, an "activation
//    record": f16 MMA B fragments + per-token column sums + the per-token
//    output scale.  Each token row is first scaled by a power of two 2^-e_t
//    (max|x_t| -> [2^-10, 2^-9)), so every finite input stays in range; f32
//    inputs are split x = hi + lo into two f16 terms (22 significant bits)
//    contracted by two MMAs; y is multiplied back by 2^e_t (exact).
//    The GEMV is a programmatic dependent of the pre-pass: its producer
//    streams weights while the pre-pass runs and waits (griddepcontrol.wait)
//    only before copying the records.
//  * Compute: each unit's bit planes were re-arranged at upload (repack.cuh)
//    so every f16x2 MMA A register is one LOP3 AND of a word: the codes land
//    in mantissa bits [p, p+B) under a zero exponent, i.e. the EXACT f16
//    subnormal c * 2^(p-24).  The activation paired with that register is
//    pre-scaled by 2^(24-p) in the record (one record section per bit-width
//    layout of the matrix), so the tensor pipe (mma.m16n8k16, tokens = N)
//    contracts exact integer codes against the scaled activations with no
//    magic offset to cancel.  The per-row affine (s, z) of each block is
//    applied in f32 after the block column: y += s*C + z*sum(x)
//    == sum((s*c+z)*x) up to f32 rounding.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>

#include "prenorm.cuh"
#include "ptx.cuh"
#include "repack.cuh"
#include "unpack.cuh"
#include "sfmp_internal.h"

namespace sfmpk {

namespace {

constexpr int kTR = 128;          // rows per unit
constexpr int kMT = 2;            // m16 tiles (16 rows each) per compute warp
constexpr int kNCW = 8 / kMT;     // compute warps per 128-row tile
constexpr int kThreads = 32 * (1 + kNCW);  // producer | compute warps
#ifndef SFMP_SEG_COLS
#define SFMP_SEG_COLS 1024
#endif
constexpr int kSegCols = SFMP_SEG_COLS;  // canonical K segment (columns)
// the decode pre-pass scales x per (token, 8 block columns); a segment must
// never straddle two such groups (n_b in {128, 256})
static_assert(kSegCols == 1024 || kSegCols == 512 || kSegCols == 256, "segment inside one pre-pass scale group");
constexpr int kHdrBytes = 1024;   // barriers | stage info | pending record copies
constexpr int kSmemSM = 225 * 1024;
#ifndef SFMP_MAX_STAGES
#define SFMP_MAX_STAGES 4
#endif
#ifndef SFMP_SU
#define SFMP_SU 2  // units per pipeline stage for n_b = 128
#endif
#ifndef SFMP_UNROLL_U
#define SFMP_UNROLL_U 1
#endif
#ifndef SFMP_EXP_NOUNPACK
#define SFMP_EXP_NOUNPACK 0
#endif
#ifndef SFMP_EXP_NOMMA
#define SFMP_EXP_NOMMA 0
#endif
#ifndef SFMP_XPREP_PDL
#define SFMP_XPREP_PDL 1
#endif
#ifndef SFMP_XPREP_MINB
#define SFMP_XPREP_MINB 8
#endif
#ifndef SFMP_EXP_NOPREPASS
#define SFMP_EXP_NOPREPASS 0
#endif
#ifndef SFMP_YTOT_GLOBAL
#define SFMP_YTOT_GLOBAL 0
#endif

#ifndef SFMP_FIX_PAIRS
#define SFMP_FIX_PAIRS 1
#endif
constexpr int kFixPairs = SFMP_FIX_PAIRS;  // (tile, token) pairs per fix-up warp
#ifndef SFMP_EXP_NOFIXUP
#define SFMP_EXP_NOFIXUP 0
#endif
#ifndef SFMP_EXP_EMPTY
#define SFMP_EXP_EMPTY 0
#endif
#ifndef SFMP_EXP_NOLOAD
#define SFMP_EXP_NOLOAD 0
#endif
#ifndef SFMP_EXP_NOREC
#define SFMP_EXP_NOREC 0
#endif
#ifndef SFMP_NOCOMPUTE
#define SFMP_NOCOMPUTE 0
#endif
#ifndef SFMP_SPIN
#define SFMP_SPIN 0
#endif
#ifndef SFMP_CTAS1
#define SFMP_CTAS1 4
#endif
#ifndef SFMP_CTAS2
#define SFMP_CTAS2 3
#endif
constexpr int kCtasNT1 = SFMP_CTAS1, kCtasNT2 = SFMP_CTAS2;  // resident CTAs per SM (M <= 8 / 9..16)
// M <= 16 with floor bits <= 3 and 16-bit x fits 96 registers without spills,
// so 4 CTAs per SM (measured: M=16 launch 47.6 -> 46.0 us); wider or f32 variants keep 3.
__host__ __device__ constexpr int ctas_per_sm(int NT, int LO = 8, bool X2 = true) {
    return NT == 1 ? kCtasNT1 : (LO <= 3 && !X2 ? kCtasNT2 + 1 : kCtasNT2);
}

// One linear of a (possibly grouped) launch.
constexpr int kMaxLin = 40;
struct Lin {
    const uint8_t* payload;
    const uint64_t* unit_desc;  // [RT*BC] row-tile-major
    const uint32_t* out_map;
    const uint8_t* xrec;        // activation records: [nl sections][BC] of sec_bytes
    float* y;
    float* part;                // [RT][P][16][128] f32 segment partials
    uint64_t out_rows;
    int BC, M, P, L;            // block columns, tokens, segments per tile, units per segment
    int RT;
    uint32_t sec_bytes;         // one record section (one block column, one bit-width layout)
    uint32_t lo_off;            // offset of the lo fragments inside a 128-column chunk (f32 input)
    int item0;                  // first work item of this linear (queue order)
    int IP;                     // work items per tile: P (one per segment) or 1 (the whole K, P > 1)
    int fix0;                   // first fix-up (tile, token) pair of this linear
    int lo;                     // floor bits: units at lo use section 0, lo+1 section 1
};
struct Params {
    Lin lin[kMaxLin];
    int nlin;
    int n_items;
    int n_fix;           // fix-up (tile, token) pairs
    int item_start[kMaxLin + 1];  // first work item of each queue slot (+ total)
    int qlin[kMaxLin];            // linear of each queue slot: whole-K linears first
    int any_whole;                // some linear runs whole-K items (TMEM running sums)
    int fix_start[kMaxLin + 1];   // first fix-up pair of each linear (+ total; none if P == 1)
    unsigned* queue;     // [0] next item, [1] CTAs done (zero between calls)
    int n_b;
    int stages;
    uint32_t stage_w;    // bytes per weight stage (smem): SU units of the widest bit-width
    uint32_t sec_bytes;  // max record section bytes (shared-memory record slot stride)
};
// Index of the linear owning entry `v` of a prefix array (binary search).
__device__ __forceinline__ int owner_of(const int* start, int n, int v) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (start[mid] <= v) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

struct XLin {
    const void* x;
    const uint32_t* col_perm;
    uint8_t* xrec;
    int BC, cols;
    int item0;      // first pre-pass CTA of this linear (one per token x 8 block columns)
    int lo, nl;     // floor bit-width, number of layout sections (1 or 2)
    int M;          // tokens of this linear
    uint32_t sec_bytes;
    PreNorm norm;   // fused RMSNorm of the token rows (on = 0: x as given)
};
struct XParams {
    XLin lin[kMaxLin];
    int nlin, M, n_b;
    int wait_prev;  // launched as a programmatic dependent of the previous GEMV
    int wait_first; // programmatic dependent of whatever ran before: wait before x and the workspace
};

// Activation record section of one block column (n_b columns) for M tokens
// in one bit-width layout (floor or ceil) of the matrix; the producer copies
// the section of the unit's own bit-width.  Sections are stored [layout][BC],
// so the records of consecutive block columns in one layout are contiguous.
// A section:
//   for chunk c (128 columns): hi runs of tokens 0..M-1, then (f32 input)
//   lo runs.  A run = the token's 8 k-step B fragments (256 B) arranged so a
//   lane reads the fragments of k-steps 2j, 2j+1 with ONE 16-byte load at
//   j*64 + q*16; runs sit kRun = 320 B apart (20 x 16 B: the two tokens of
//   a quarter-warp then fall into disjoint bank quads).  Each value is the
//   scaled activation times 2^(24-p) of the register slot it pairs with.
//   Tail (floats): Xg[16] column sums of the scaled x | ysa[16], ysb[16]
//   with ysa*ysb = 2^e_t (two factors: 2^e_t may not be a normal float).
constexpr int kRun = 320;
constexpr int kTailFloats = 48;
constexpr int kYsIdx = 16;
struct RecGeom {
    int M;
    bool X2;
    __host__ __device__ int nt_count() const { return M > 8 ? 2 : 1; }
    __host__ __device__ int chunk_bytes() const { return kRun * M * (X2 ? 2 : 1); }
    __host__ __device__ int lo_off() const { return kRun * M; }
    __host__ __device__ int run_off(int c, int t, int q) const { return c * chunk_bytes() + t * kRun + q * 16; }
    __host__ __device__ static int step_off(int s8) { return (s8 >> 1) * 64 + (s8 & 1) * 8; }
    __host__ __device__ int xg_off(int CH) const { return CH * chunk_bytes(); }
    __host__ __device__ int sec_bytes(int CH) const { return (xg_off(CH) + 4 * kTailFloats + 127) / 128 * 128; }
};

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
constexpr int kXprepRowLimit = 192 * 1024;  // staged x row bytes of the fused-norm pre-pass

// Per-token power-of-two scale: e such that max|x| * 2^-e lies in
// [2^-10, 2^-9), so the largest record value (slot factor 2^24) lies in
// [2^14, 2^15): every finite input stays finite in f16.  0 for an all-zero or
// non-finite row (inf/nan then propagate as in the f32 reference).
__device__ __forceinline__ int token_exponent(float amax) {
    if (!(amax > 0.f) || !isfinite(amax)) return 0;
    return ilogbf(amax) + 10;
}
// 2^e for |e| <= 254 as a product of two normal floats
__device__ __forceinline__ float2 pow2_pair(int e) {
    const int a = e / 2;
    return make_float2(__int_as_float((a + 127) << 23), __int_as_float((e - a + 127) << 23));
}

// f16 hi (+ lo for f32 input) parts of v0*f, v1*f (f a power of two).
template <bool X2>
__device__ __forceinline__ void split2(float v0, float v1, float f, uint32_t& hi, uint32_t& lo) {
    const float a = v0 * f, b = v1 * f;
    const __half2 h = __floats2half2_rn(a, b);
    hi = h2_as_u32(h);
    if constexpr (X2) lo = h2_as_u32(__floats2half2_rn(a - __low2float(h), b - __high2float(h)));
    else lo = 0u;
}
// slot factor 2^(24-p) of register j in the layout of B-bit units
__device__ __forceinline__ float slot_factor(int B, int j) {
    return __int_as_float((24 - sub_pos(B, j) + 127) << 23);
}

// Row-wide max |x| reduction of a staged row (256 threads).
template <class T, class F>
__device__ __forceinline__ float row_absmax(const T* xr, int cols, F cvt, float* red) {
    float m = 0.f;
    for (int i = threadIdx.x; i < cols; i += blockDim.x) m = fmaxf(m, fabsf(cvt(xr[i])));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = 0.f;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
    return m;
}

// Record piece of one block column for token t from 4 gathered, scaled
// values per chunk: lane (s8, q) owns registers 2*s8, 2*s8+1 of k-step s8;
// each layout section gets them times its slot factors.  rec0 = the block
// column's layout-0 section; layout l is l * lstride further.
template <bool X2>
__device__ __forceinline__ void write_fragments(uint8_t* rec0, size_t lstride, const RecGeom& G, int c, int t, int q,
                                                int s8, const float (&v)[4], int lo, int nl) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
        if (l >= nl) break;
        const int B = lo + l;
        uint2 h, w;
        split2<X2>(v[0], v[1], slot_factor(B, 2 * s8), h.x, w.x);      // pairs with A register 2*s8
        split2<X2>(v[2], v[3], slot_factor(B, 2 * s8 + 1), h.y, w.y);  // ... and 2*s8+1
        uint8_t* dst = rec0 + l * lstride + G.run_off(c, t, q) + RecGeom::step_off(s8);
        *reinterpret_cast<uint2*>(dst) = h;
        if constexpr (X2) *reinterpret_cast<uint2*>(dst + G.lo_off()) = w;
    }
}
__device__ __forceinline__ void write_tail(uint8_t* rec0, size_t lstride, const RecGeom& G, int CH, int t, int M,
                                          float xs, int e, int nl) {
    const float2 ys = pow2_pair(e);
    for (int l = 0; l < nl; ++l) {
        float* xg = reinterpret_cast<float*>(rec0 + l * lstride + G.xg_off(CH));
        xg[t] = xs;
        xg[kYsIdx + t] = ys.x;
        xg[kYsIdx + 16 + t] = ys.y;
        if (t == M - 1)  // token columns the GEMV computes but never stores
            for (int u = M; u < 8 * G.nt_count(); ++u) xg[u] = xg[kYsIdx + u] = xg[kYsIdx + 16 + u] = 0.f;
    }
}

// K4 (decode flavour, staged): one CTA per (token t, 8 block columns of one
// linear).  It stages token t's x row and the 8 block columns' col_perm in
// shared memory with coalesced 16 B loads, finds the row's power-of-two
// scale, then each warp writes the record piece of one block column for
// token t: lane (s, q) gathers the 4 k-slots 32q + 8(s&1) + 4j + 16e + (s>>1)
// of each 128-column chunk from shared memory and stores 8 B of B fragments
// per layout (hi, and lo for f32 input).  The column sum X_g
// (lutgemm.cpp:113-115) uses the scaled input values.
template <sfmp_dtype DT>
__global__ void __launch_bounds__(256) xprep_rows_kernel(const XParams xp) {
    using T = typename XT<DT>::T;
    constexpr bool X2 = DT == SFMP_F32;
    pdl_launch_dependents();  // let the GEMV start streaming weights right away
    extern __shared__ __align__(16) uint8_t xsm[];
    __shared__ float red[8];
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
    // fused RMSNorm (prenorm.cuh): x = h * inv_rms * gamma, folded into the scale
    float inv = 1.f;
    int e;
    if (XL.norm.on) {
        __shared__ float nred[32];
        inv = row_inv_rms([&](int i) { return XT<DT>::f(xr[i]); }, cols, XL.norm.eps, nred);
        float m = 0.f;
        for (int i = threadIdx.x; i < cols; i += 256) m = fmaxf(m, fabsf(XT<DT>::f(xr[i]) * gamma_at(XL.norm, i)));
        e = token_exponent(block_reduce<true>(m, nred) * inv);
    } else {
        e = token_exponent(row_absmax(xr, cols, [](T v) { return XT<DT>::f(v); }, red));
    }
    const float2 sc = pow2_pair(-e);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp >= nbc) return;
    const int bc = bc0 + warp, s8 = lane >> 2, q = lane & 3;
    const RecGeom G{M, X2};
    const size_t lstride = static_cast<size_t>(XL.BC) * XL.sec_bytes;
    uint8_t* rec0 = XL.xrec + static_cast<size_t>(bc) * XL.sec_bytes;
    const uint32_t* cpw = cp + warp * n_b;
    const int kb = 32 * q + 8 * (s8 & 1) + (s8 >> 1);
    float xs = 0.f;
    for (int c = 0; c < CH; ++c) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
                const uint32_t col = cpw[c * 128 + kb + 4 * j + 16 * e2];
                float h = XT<DT>::f(xr[col]);
                if (XL.norm.on) h = (h * inv) * gamma_at(XL.norm, col);
                v[j * 2 + e2] = h * sc.x * sc.y;
            }
        write_fragments<X2>(rec0, lstride, G, c, t, q, s8, v, XL.lo, XL.nl);
        xs += (v[0] + v[1]) + (v[2] + v[3]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
    if (lane == 0) write_tail(rec0, lstride, G, CH, t, M, xs, e, XL.nl);
    // When launched to overlap the previous GEMV of the same grouped call, do
    // not complete before it: this grid's completion (which the next GEMV waits
    // for) then implies the previous launch's, keeping stream order for any
    // later work.  A no-op for a normal launch.
    if (xp.wait_prev) pdl_wait();
}

// K4 (decode flavour, default): one CTA per (token t, 8 block columns of one
// linear).  The 8 block columns' col_perm slices are staged in shared memory
// (coalesced), then warp w gathers its block column's activations for token
// t straight from x (x[t][col_perm[.]], reorder.cpp:103-111), lane (s, q)
// owning the 4 k-slots 32q + 8(s&1) + 4j + 16e + (s>>1) of each 128-column
// chunk.  The output scale 2^e is per (token, 8 block columns): max|x| of
// the CTA's 1024 (or 2048) values -> [2^-10, 2^-9), written into each of its
// records' tails and applied by the GEMV per unit (exact powers of two), so no
// CTA reads the whole row.  Column sums X_g (lutgemm.cpp:113-115) use the
// scaled values.
template <sfmp_dtype DT>
// 8 CTAs per SM (<= 32 registers): the step's ~1200 (linear, token, 8 block
// columns) CTAs then fit in one wave on 148 SMs
__global__ void __launch_bounds__(256, SFMP_XPREP_MINB) xprep_gather_kernel(const XParams xp) {
    using T = typename XT<DT>::T;
    constexpr bool X2 = DT == SFMP_F32;
    // let the GEMV start streaming weights right away -- unless this grid itself
    // started early (wait_first): then only once the previous grid is done, so
    // the GEMV never overlaps the previous call's GEMV (shared work queue)
    if (!xp.wait_first) pdl_launch_dependents();
    __shared__ __align__(16) uint32_t cp[8 * 256];  // [nbc][n_b] column indices
    __shared__ float red[8];
    const int n_b = xp.n_b, CH = n_b >> 7;
    int it = blockIdx.x, li = 0;  // compact grid: (linear, token, 8 block columns)
    while (li + 1 < xp.nlin && it >= xp.lin[li + 1].item0) ++li;
    const XLin& XL = xp.lin[li];
    const int M = XL.M;
    it -= XL.item0;
    const int nit = (XL.BC + 7) / 8;
    const int t = it / nit;
    it -= t * nit;
    const int bc0 = it * 8, nbc = min(8, XL.BC - bc0);
    {
        const uint4* src = reinterpret_cast<const uint4*>(XL.col_perm + static_cast<size_t>(bc0) * n_b);
        const uint64_t keep = policy_evict_last();
        for (int i = threadIdx.x; i < nbc * n_b / 4; i += 256) reinterpret_cast<uint4*>(cp)[i] = ldg_keep_v4(src + i, keep);
    }
    // prologue done (col_perm is the model's, constant): from here on x -- maybe
    // the previous kernel's output -- and the workspace the previous call's
    // GEMV may still read are touched, so wait for the previous grid
    if (xp.wait_first) {
        pdl_wait();
        pdl_launch_dependents();
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s8 = lane >> 2, q = lane & 3;
    const int kb = 32 * q + 8 * (s8 & 1) + (s8 >> 1);
    const T* xrow = static_cast<const T*>(XL.x) + static_cast<size_t>(t) * XL.cols;
    const uint32_t* cpw = cp + warp * n_b;
    float v[2][4];
    float m = 0.f;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[c][j] = 0.f;
            if (warp < nbc && c < CH) {
                v[c][j] = XT<DT>::f(xrow[cpw[c * 128 + kb + 4 * (j >> 1) + 16 * (j & 1)]]);
                m = fmaxf(m, fabsf(v[c][j]));
            }
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[warp] = m;
    __syncthreads();
    m = 0.f;
    for (int w = 0; w < 8; ++w) m = fmaxf(m, red[w]);
    if (warp < nbc) {
        const int e = token_exponent(m);
        const float2 sc = pow2_pair(-e);
        const int bc = bc0 + warp;
        const RecGeom G{M, X2};
        const size_t lstride = static_cast<size_t>(XL.BC) * XL.sec_bytes;
        uint8_t* rec0 = XL.xrec + static_cast<size_t>(bc) * XL.sec_bytes;
        float xs = 0.f;
        for (int c = 0; c < CH; ++c) {
            float u[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) u[j] = v[c][j] * sc.x * sc.y;
            write_fragments<X2>(rec0, lstride, G, c, t, q, s8, u, XL.lo, XL.nl);
            xs += (u[0] + u[1]) + (u[2] + u[3]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
        if (lane == 0) write_tail(rec0, lstride, G, CH, t, M, xs, e, XL.nl);
    }
    if (xp.wait_prev) pdl_wait();  // see xprep_rows_kernel
}

// Decode layout of a unit (upload time, sfmp_internal.h "lane-major"): a
// 512-byte s/z block [warp cw][g][r] of (s, z) fp16 pairs for row
// cw*32 + 8r + g, then the planes as [chunk c][cw][plane i][lane][r] words,
// lane = 4g + q holding word q of the 16-byte row segment of chunk c.  A
// compute lane therefore fetches its 4 rows' words of one plane with ONE
// 16-byte shared load, and its 4 rows' (s, z) with one more.
__host__ __device__ constexpr uint32_t unit_bytes(int B, int nb8) { return 512u + static_cast<uint32_t>(B) * 128u * nb8; }

// One 128-column chunk of a unit for this warp's 32 rows (2 m16 tiles).
// pw = this lane's word of plane 0 (planes 512 B apart); xb = this lane's
// B-fragment piece 0 of each n-tile (pieces 64 B apart).  X2: the lo B
// fragments (lo_off further) are contracted into the same accumulators.
template <int B, int NT, bool X2>
__device__ __forceinline__ void unit_chunk(const uint8_t* pw, const uint8_t* const (&xb)[NT], uint32_t lo_off,
                                           float (&cacc)[kMT][NT][4]) {
    // rows r0 + 8*r: (r0, r0+8) is m-tile 0, (r0+16, r0+24) m-tile 1
    uint32_t p[2 * kMT][B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
        const uint4 v = *reinterpret_cast<const uint4*>(pw + i * 512);
        p[0][i] = v.x;
        p[1][i] = v.y;
        p[2][i] = v.z;
        p[3][i] = v.w;
    }
    uint32_t A[2 * kMT][16];
#pragma unroll
    for (int r = 0; r < 2 * kMT; ++r) {
        if constexpr (SFMP_EXP_NOUNPACK) {  // experiment builds only: no unpack
#pragma unroll
            for (int j = 0; j < 16; ++j) A[r][j] = p[r][j % B];
        } else if constexpr (B <= 4) unpack_rp_sub<B>(p[r], A[r]);  // repacked layout (repack.cuh)
        else unpack_word_sub<B>(p[r], A[r]);                // bit planes (unpack.cuh)
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const uint4 b = *reinterpret_cast<const uint4*>(xb[nt] + j * 64);
            uint4 bl;
            if constexpr (X2) bl = *reinterpret_cast<const uint4*>(xb[nt] + lo_off + j * 64);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int s = 2 * j + h;
                const uint32_t b0 = h ? b.z : b.x, b1 = h ? b.w : b.y;
#pragma unroll
                for (int m = 0; m < kMT; ++m) {
                    if (SFMP_EXP_NOMMA) {  // experiment builds only: no tensor-core work
                        cacc[m][nt][0] += __uint_as_float(A[2 * m][2 * s] ^ A[2 * m + 1][2 * s + 1] ^ b0 ^ b1);
                        continue;
                    }
                    mma_16816(cacc[m][nt], A[2 * m][2 * s], A[2 * m + 1][2 * s], A[2 * m][2 * s + 1],
                              A[2 * m + 1][2 * s + 1], b0, b1);
                    if constexpr (X2)
                        mma_16816(cacc[m][nt], A[2 * m][2 * s], A[2 * m + 1][2 * s], A[2 * m][2 * s + 1],
                                  A[2 * m + 1][2 * s + 1], h ? bl.z : bl.x, h ? bl.w : bl.y);
                }
            }
        }
    }
}

// One unit (block column) of B bits: the MMA over its chunks, then the
// block's per-row affine y += s*C + z*Xg (the mirror identity of
// quantizer.cpp:57-72 without the LUT).
// NT: n-tiles of this linear (tokens <= 8 or <= 16); NTM: the launch's
// accumulator width (a launch mixing token classes runs each linear's own NT).
template <int B, int CH, int NT, int NTM, bool X2>
__device__ __forceinline__ void unit_step(const uint8_t* ub, const uint8_t* xr, const uint32_t (&xoff)[NTM],
                                          uint32_t chunk_bytes, uint32_t lo_off, uint32_t xg_off, int cw, int lane,
                                          float (&yacc)[kMT][NTM][4]) {
    float cacc[kMT][NT][4];
#pragma unroll
    for (int m = 0; m < kMT; ++m)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) cacc[m][nt][e] = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const uint8_t* xbc[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) xbc[nt] = xr + xoff[nt] + c * chunk_bytes;
        unit_chunk<B, NT, X2>(ub + 512 + c * (B * 2048) + cw * (B * 512) + lane * 16, xbc, lo_off, cacc);
    }
    const uint4 sz = *reinterpret_cast<const uint4*>(ub + cw * 128 + (lane >> 2) * 16);
    const uint32_t szw[4] = {sz.x, sz.y, sz.z, sz.w};
#pragma unroll
    for (int m = 0; m < kMT; ++m) {
        const __half2 pa = u32_as_h2(szw[2 * m]), pb = u32_as_h2(szw[2 * m + 1]);
        const float sa = __low2float(pa), za = __high2float(pa);
        const float sb = __low2float(pb), zb = __high2float(pb);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float2 xg01 = *reinterpret_cast<const float2*>(xr + xg_off + 8 * (lane & 3) + 32 * nt);
            const float* c0 = cacc[m][nt];
            yacc[m][nt][0] = fmaf(sa, c0[0], fmaf(za, xg01.x, yacc[m][nt][0]));
            yacc[m][nt][1] = fmaf(sa, c0[1], fmaf(za, xg01.y, yacc[m][nt][1]));
            yacc[m][nt][2] = fmaf(sb, c0[2], fmaf(zb, xg01.x, yacc[m][nt][2]));
            yacc[m][nt][3] = fmaf(sb, c0[3], fmaf(zb, xg01.y, yacc[m][nt][3]));
        }
    }
}

// Barrier waits that suspend the thread (woken by the phase completion)
// instead of spinning: spinning waiters took issue slots from working warps.
__device__ __forceinline__ void mbar_wait_idle(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAITI_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITI_%=;\n\t}" ::"r"(bar),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// A stage holds SU consecutive units of one work item (SU = 2 for n_b = 128,
// 1 for n_b = 256: 256 columns either way) and their record sections.
// Stage info (16 B): x = linear | bits0 << 8 | bits1 << 12 | units << 16 | flags << 20, y = row tile, z = segment.
// kFirst / kLast: first / last stage of a segment; kItemLast: last stage of the work item.
constexpr uint32_t kFirst = 1, kLast = 2, kEnd = 4, kItemLast = 8;
struct PendCopy {
    const uint8_t* src;
    uint32_t dst, bytes;
};

// NT = the widest linear's n-tile count (M <= 8: 1, M <= 16: 2); linears of
// both classes may share a launch, each running its own n-tile count.
// LO = the model's floor bit-width: every unit has LO or LO+1 bits
// (PackedModel::validate, layout.cpp:100-103), so the kernel carries exactly
// two unpack paths and its hot loop stays resident in the instruction cache.
// WH = the launch has whole-K items (only n_b = 128 with 16-bit x: the running
// sums cost registers, so launches without whole-K items use the lean build).
template <int NT, int CH, int LO, bool X2, bool WH>
__global__ void __launch_bounds__(kThreads, ctas_per_sm(NT, LO, X2)) gemv_kernel(const Params p) {
    constexpr int SU = CH == 1 ? SFMP_SU : 1;
    constexpr int nb8 = CH * 16;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 8;
    uint4* sinfo = reinterpret_cast<uint4*>(smem + 128);                  // [S]
    PendCopy* pend = reinterpret_cast<PendCopy*>(smem + 256);             // [2S] producer only
    uint8_t* wbase = smem + kHdrBytes;
    const uint32_t xstride = SU * p.sec_bytes;
    uint8_t* xbase = wbase + static_cast<size_t>(S) * p.stage_w;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (SFMP_EXP_EMPTY) {  // experiment builds only: the launch's fixed costs without the GEMV
        pdl_launch_dependents();
        return;
    }
    // a programmatic dependent (the fix-up of this launch, or the next launch
    // of the same grouped call, whose problems are independent of ours) may
    // start now: it waits for this grid's completion before it reads our data
    pdl_launch_dependents();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNCW * 32);  // every compute lane releases the stage
        }
        fence_mbar_init();
        fence_proxy_async();
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer: claims items, one bulk copy per stage (+ its record sections) ----
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const uint64_t keep = policy_evict_last();
            const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty);
            int s = 0, ph = 0;
            bool released = false;  // griddepcontrol.wait done: records may be copied
            int npend = 0, pstages = 0;
            auto issue_x = [&](const uint8_t* src, uint32_t dst, uint32_t n, int st) {
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                    "l"(src), "r"(n), "r"(full_a + 8 * st)
                    : "memory");
            };
            // The weights of the first ring-full do not depend on x: they are
            // issued before griddepcontrol.wait, their records after it.
            auto release = [&]() {
                if (released) return;
                pdl_wait();
                released = true;
                for (int i = 0; i < npend; ++i) issue_x(pend[i].src, pend[i].dst & 0x00FFFFFFu, pend[i].bytes, static_cast<int>(pend[i].dst >> 24));
                npend = 0;
            };
            unsigned item = atomicAdd(p.queue, 1u);
            while (item < static_cast<unsigned>(p.n_items)) {
                const unsigned next = atomicAdd(p.queue, 1u);  // claim ahead: latency overlaps this item
                const int li = p.qlin[owner_of(p.item_start, p.nlin, static_cast<int>(item))];
                const Lin& L = p.lin[li];
                const int rel = static_cast<int>(item) - L.item0;
                const int rt = rel / L.IP, seg0 = rel - rt * L.IP;
                // a whole-K item (IP == 1) runs all segments of its tile back to back
                const int bc0 = seg0 * L.L, bc1 = L.IP == 1 ? L.BC : min(L.BC, bc0 + L.L);
                const uint64_t* gdesc = L.unit_desc + static_cast<size_t>(rt) * L.BC;
                const uint32_t sec = L.sec_bytes;
                uint64_t d0n = ldg_keep_u64(gdesc + bc0, keep);
                uint64_t d1n = (SU == 2 && bc0 + 1 < bc1) ? ldg_keep_u64(gdesc + bc0 + 1, keep) : 0ull;
                int seg = seg0, seg_beg = bc0, seg_end = min(bc1, bc0 + L.L);
                for (int bc = bc0; bc < bc1; bc += SU) {
                    const int nu = min(SU, bc1 - bc);
                    if (bc == seg_end) {  // a stage never straddles a segment (L % SU == 0)
                        ++seg;
                        seg_beg = seg_end;
                        seg_end = min(bc1, seg_end + L.L);
                    }
                    const uint64_t d0 = d0n, d1 = d1n;
                    if (bc + SU < bc1) {
                        d0n = ldg_keep_u64(gdesc + bc + SU, keep);
                        if (SU == 2 && bc + SU + 1 < bc1) d1n = ldg_keep_u64(gdesc + bc + SU + 1, keep);
                    }
                    if (!released && pstages == S) release();  // ring full: records now
                    mbar_wait_idle(empty_a + 8 * s, ph ^ 1);
                    const int b0 = static_cast<int>((d0 >> 48) & 0xF);
                    const int b1 = nu > 1 ? static_cast<int>((d1 >> 48) & 0xF) : 0;
                    const uint32_t fl = (bc == seg_beg ? kFirst : 0u) | (bc + nu == seg_end ? kLast : 0u) |
                                        (bc + nu == bc1 ? kItemLast : 0u);
                    sinfo[s] = make_uint4(static_cast<uint32_t>(li) | (static_cast<uint32_t>(b0) << 8) |
                                              (static_cast<uint32_t>(b1) << 12) | (static_cast<uint32_t>(nu) << 16) |
                                              (fl << 20),
                                          static_cast<uint32_t>(rt), static_cast<uint32_t>(seg), 0u);
                    const uint32_t wbytes = unit_bytes(b0, nb8) + (nu > 1 ? unit_bytes(b1, nb8) : 0u);
                    if (SFMP_EXP_NOLOAD) {  // experiment builds only: compute on stale shared memory
                        mbar_arrive(&full[s]);
                        if (++s == S) { s = 0; ph ^= 1; }
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[s], wbytes + (SFMP_EXP_NOREC ? 0u : nu * sec));  // publishes sinfo[s]
                    bulk_g2s(wbase + static_cast<size_t>(s) * p.stage_w, L.payload + (d0 & 0xFFFFFFFFFFFFull), wbytes,
                             &full[s], pol);
                    // record sections of the units' bit-width layouts ([layout][BC]: one
                    // copy when both units share a layout)
                    const int l0 = b0 != L.lo, l1 = b1 != L.lo;
                    const uint32_t xd = smem_u32(xbase) + s * xstride;
                    const uint8_t* r0 = L.xrec + static_cast<size_t>(l0 * L.BC + bc) * sec;
                    const uint8_t* r1 = L.xrec + static_cast<size_t>(l1 * L.BC + bc + 1) * sec;
                    const bool one = nu == 1 || l0 == l1;
                    const uint32_t n0 = one ? nu * sec : sec;
                    if (SFMP_EXP_NOREC) {  // experiment builds only: records never copied
                    } else if (released) {
                        issue_x(r0, xd, n0, s);
                        if (!one) issue_x(r1, xd + sec, sec, s);
                    } else {
                        pend[npend++] = PendCopy{r0, xd | (static_cast<uint32_t>(s) << 24), n0};
                        if (!one) pend[npend++] = PendCopy{r1, (xd + sec) | (static_cast<uint32_t>(s) << 24), sec};
                        ++pstages;
                    }
                    if (++s == S) { s = 0; ph ^= 1; }
                }
                item = next;
            }
            release();
            // end of work: one empty stage with the END flag
            mbar_wait_idle(empty_a + 8 * s, ph ^ 1);
            sinfo[s] = make_uint4(kEnd << 20, 0u, 0u, 0u);
            mbar_arrive(&full[s]);
        }
        __syncwarp();
    } else {
        // ---------------- compute warps ------------------------------------------
        const int cw = warp - 1;
        const int g = lane >> 2, q = lane & 3;
        const int r0 = cw * 16 * kMT + g;  // rows r0 + 8*r of the tile
        const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty);
        // record geometry depends on the linear's M: set when the linear changes
        int cur_li = -1, cur_nt = NT;
        uint32_t chunk_bytes = 0, lo_off = 0, xg_off = 0, sec = 0;
        uint32_t xoff[NT];  // offset of this lane's B-fragment piece 0 of each n-tile in a record
        float yacc[kMT][NT][4];
#if !SFMP_YTOT_GLOBAL
        float ytot[WH ? kMT : 1][WH ? NT : 1][4];  // whole-K item: the segment sums added in segment order
#endif
        float ysa[NT][2], ysb[NT][2];
        int s = 0, ph = 0;
        for (;;) {
            if (SFMP_SPIN) mbar_wait_a(full_a + 8 * s, ph);
            else mbar_wait_idle(full_a + 8 * s, ph);
            // lane 0 reads the stage info and is the lane that later frees the stage
            // (the producer rewrites sinfo[s] after that arrive): broadcast it
            uint4 info = make_uint4(0u, 0u, 0u, 0u);
            if (lane == 0) info = sinfo[s];
            info.x = __shfl_sync(0xffffffffu, info.x, 0);
            info.y = __shfl_sync(0xffffffffu, info.y, 0);
            info.z = __shfl_sync(0xffffffffu, info.z, 0);
            const uint32_t fl = info.x >> 20;
            if (fl & kEnd) break;
            const int li = static_cast<int>(info.x & 0xFF);
            if (li != cur_li) {
                cur_li = li;
                const Lin& L = p.lin[li];
                const RecGeom GL{L.M, X2};
                chunk_bytes = GL.chunk_bytes();
                cur_nt = GL.nt_count();
                lo_off = L.lo_off;
                sec = L.sec_bytes;
                xg_off = GL.xg_off(CH);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)  // absent tokens read token 0's fragments (never stored)
                    xoff[nt] = GL.run_off(0, nt * 8 + g < L.M ? nt * 8 + g : 0, q);
            }
            const uint8_t* ws = wbase + static_cast<size_t>(s) * p.stage_w;
            const uint8_t* xs = xbase + static_cast<size_t>(s) * xstride;
            if (fl & kFirst) {
#pragma unroll
                for (int m = 0; m < kMT; ++m)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 4; ++e) yacc[m][nt][e] = 0.f;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {  // the segment's output scale of tokens nt*8+2q, +1
                    // (one scale per (token, 8 block columns) -- a segment never straddles two)
                    const float2 a = *reinterpret_cast<const float2*>(xs + xg_off + 4 * kYsIdx + 32 * nt + 8 * q);
                    const float2 b = *reinterpret_cast<const float2*>(xs + xg_off + 4 * (kYsIdx + 16) + 32 * nt + 8 * q);
                    ysa[nt][0] = a.x;
                    ysa[nt][1] = a.y;
                    ysb[nt][0] = b.x;
                    ysb[nt][1] = b.y;
                }
            }
#if SFMP_UNROLL_U
#pragma unroll
#else
#pragma unroll 1
#endif
            for (int u = 0; u < SU; ++u) {
                const int bits = static_cast<int>((info.x >> (8 + 4 * u)) & 0xF);
                if (u > 0 && ((info.x >> 16) & 0xF) < 2) break;
                const uint8_t* ub = ws + (u ? unit_bytes(info.x >> 8 & 0xF, nb8) : 0u);
                const uint8_t* xr = xs + u * sec;
                if (SFMP_NOCOMPUTE) {
                    if (bits == 0xF) yacc[0][0][0] += 1.f;  // experiment builds: streaming only
                } else if (NT == 2 && cur_nt == 1) {
                    if (bits == LO) {
                        unit_step<LO, CH, 1, NT, X2>(ub, xr, xoff, chunk_bytes, lo_off, xg_off, cw, lane, yacc);
                    } else if constexpr (LO < 8) {
                        unit_step<LO + 1, CH, 1, NT, X2>(ub, xr, xoff, chunk_bytes, lo_off, xg_off, cw, lane, yacc);
                    }
                } else if (bits == LO) {
                    unit_step<LO, CH, NT, NT, X2>(ub, xr, xoff, chunk_bytes, lo_off, xg_off, cw, lane, yacc);
                } else if constexpr (LO < 8) {
                    unit_step<LO + 1, CH, NT, NT, X2>(ub, xr, xoff, chunk_bytes, lo_off, xg_off, cw, lane, yacc);
                }
            }
            // every lane arrives (its own reads of the stage precede its own release)
            mbar_arrive_a(empty_a + 8 * s);
            if (++s == S) { s = 0; ph ^= 1; }
            if (!(fl & kLast)) continue;

            // ---- end of a segment: scale back by 2^e (exact), store y or the partial ----
            const Lin& L = p.lin[li];
            const int rt = static_cast<int>(info.y), seg = static_cast<int>(info.z);
            const bool whole = L.P == 1;
            if (WH && L.IP == 1 && !whole) {
                // whole-K item: ((0 + s_0) + s_1) + ... -- the same float operations
                // gemv_fixup_kernel performs on the partials, so the bits do not depend
                // on how the call was cut into items
#pragma unroll
                for (int m = 0; m < kMT; ++m)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float v = (yacc[m][nt][e] * ysa[nt][e & 1]) * ysb[nt][e & 1];  // exact
#if SFMP_YTOT_GLOBAL
                            // the running sum in this thread's own slot of the tile's partials
                            const int t = nt * 8 + 2 * q + (e & 1);
                            float* slot = L.part + static_cast<size_t>(rt) * L.P * (16 * kTR) + t * kTR + r0 + 16 * m + 8 * (e >> 1);
                            yacc[m][nt][e] = (seg == 0 ? 0.f : *slot) + v;
                            if (!(fl & kItemLast)) *slot = yacc[m][nt][e];
#else
                            ytot[m][nt][e] = (seg == 0 ? 0.f : ytot[m][nt][e]) + v;
#endif
                        }
                if (!(fl & kItemLast)) continue;
#pragma unroll
                for (int m = 0; m < kMT; ++m)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int t = nt * 8 + 2 * q + (e & 1);
                            if (t >= L.M) continue;
                            const int row = r0 + 16 * m + 8 * (e >> 1);
#if SFMP_YTOT_GLOBAL
                            L.y[t * L.out_rows + __ldg(L.out_map + rt * kTR + row)] = yacc[m][nt][e];
#else
                            L.y[t * L.out_rows + __ldg(L.out_map + rt * kTR + row)] = ytot[m][nt][e];
#endif
                        }
                continue;
            }
            float* dst = whole ? L.y : L.part + (static_cast<size_t>(rt) * L.P + seg) * (16 * kTR);
#pragma unroll
            for (int m = 0; m < kMT; ++m)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int t = nt * 8 + 2 * q + (e & 1);
                        if (t >= L.M) continue;
                        const float v = (yacc[m][nt][e] * ysa[nt][e & 1]) * ysb[nt][e & 1];  // exact
                        const int row = r0 + 16 * m + 8 * (e >> 1);
                        if (whole) dst[t * L.out_rows + __ldg(L.out_map + rt * kTR + row)] = v;  // un-permuted
                        else dst[t * kTR + row] = v;  // [t][128 rows], coalesced
                    }
        }
    }
    // the last CTA out resets the work queue for the next call (stream-ordered)
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned done = atomicAdd(p.queue + 1, 1u);
        if (done == gridDim.x - 1) {
            p.queue[0] = 0u;
            p.queue[1] = 0u;
        }
    }
}

// Split-tile fix-up (programmatic dependent of the GEMV).  One warp per
// (tile, token) pair of every multi-segment linear (fix_start prefix); lane l
// owns rows 4l..4l+3 of the tile (float4), issues all P partial loads at once
// and adds them in SEGMENT order -- the canonical order -- then stores the 4
// un-permuted outputs.  One warp per pair and 8 pairs per 256-thread CTA keep
// a whole launch's fix-up in one wave (the 128-threads-per-pair, 2-pairs-per-
// thread version took ~2.3 latency-bound passes: 11 us exposed at M=16).
__global__ void __launch_bounds__(256) gemv_fixup_kernel(const Params p) {
    pdl_launch_dependents();  // a later launch of the same grouped call may start its pre-pass
    const int lane = threadIdx.x & 31;
    // kFixPairs (tile, token) pairs per warp, all their partial loads issued before any is used
    const int w0 = (static_cast<int>(blockIdx.x) * 8 + static_cast<int>(threadIdx.x >> 5)) * kFixPairs;
    if (w0 >= p.n_fix) return;
    const float4* pp[kFixPairs];
    float* yrow[kFixPairs];
    uint4 om[kFixPairs];
    int P[kFixPairs];
#pragma unroll
    for (int h = 0; h < kFixPairs; ++h) {
        P[h] = 0;
        const int w = w0 + h;
        if (w >= p.n_fix) continue;
        const Lin& L = p.lin[owner_of(p.fix_start, p.nlin, w)];
        const int rel = w - L.fix0, rt = rel / L.M, t = rel - rt * L.M;
        P[h] = L.P;
        om[h] = __ldg(reinterpret_cast<const uint4*>(L.out_map + rt * kTR) + lane);
        pp[h] = reinterpret_cast<const float4*>(L.part + static_cast<size_t>(rt) * L.P * (16 * kTR) + t * kTR) + lane;
        yrow[h] = L.y + static_cast<size_t>(t) * L.out_rows;
    }
    pdl_wait();  // the GEMV grid has completed and its partials are visible
    int Pm = 0;
#pragma unroll
    for (int h = 0; h < kFixPairs; ++h) Pm = max(Pm, P[h]);
    float4 acc[kFixPairs];
#pragma unroll
    for (int h = 0; h < kFixPairs; ++h) acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = 0; k0 < Pm; k0 += 8) {
        float4 v[kFixPairs][8];
#pragma unroll
        for (int h = 0; h < kFixPairs; ++h)
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < P[h]) v[h][k] = __ldg(pp[h] + (k0 + k) * (16 * kTR / 4));  // previous grid's data
#pragma unroll
        for (int h = 0; h < kFixPairs; ++h)
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < P[h]) {  // segment order
                    acc[h].x += v[h][k].x;
                    acc[h].y += v[h][k].y;
                    acc[h].z += v[h][k].z;
                    acc[h].w += v[h][k].w;
                }
    }
#pragma unroll
    for (int h = 0; h < kFixPairs; ++h) {
        if (!P[h]) continue;
        yrow[h][om[h].x] = acc[h].x;
        yrow[h][om[h].y] = acc[h].y;
        yrow[h][om[h].z] = acc[h].z;
        yrow[h][om[h].w] = acc[h].w;
    }
}

// One-time (per device, thread-safe) function attribute setup.
template <class F>
void once_per_device(std::once_flag* flags, F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    std::call_once(flags[dev], f);
}

template <int NT, int CH, int LO, bool X2, bool WH>
cudaError_t launch_kw(cudaLaunchConfig_t& cfg, const Params& p) {
    auto k = gemv_kernel<NT, CH, LO, X2, WH>;
    static std::once_flag fl[64];
    static cudaError_t err[64];
    int dev = 0;
    cudaGetDevice(&dev);
    once_per_device(fl, [&] { err[dev & 63] = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024); });
    if (err[dev & 63] != cudaSuccess) return err[dev & 63];
    note_launch();
    return cudaLaunchKernelEx(&cfg, k, p);
}
template <int NT, int CH, int LO, bool X2>
cudaError_t launch_k(cudaLaunchConfig_t& cfg, const Params& p) {
    if constexpr (CH == 1 && !X2) {
        if (p.any_whole) return launch_kw<NT, CH, LO, X2, true>(cfg, p);
    }
    return launch_kw<NT, CH, LO, X2, false>(cfg, p);
}

template <int NT, int CH, bool X2>
cudaError_t launch_nc(cudaLaunchConfig_t& cfg, const Params& p, int lo) {
    switch (lo) {
        case 1: return launch_k<NT, CH, 1, X2>(cfg, p);
        case 2: return launch_k<NT, CH, 2, X2>(cfg, p);
        case 3: return launch_k<NT, CH, 3, X2>(cfg, p);
        case 4: return launch_k<NT, CH, 4, X2>(cfg, p);
        case 5: return launch_k<NT, CH, 5, X2>(cfg, p);
        case 6: return launch_k<NT, CH, 6, X2>(cfg, p);
        case 7: return launch_k<NT, CH, 7, X2>(cfg, p);
        default: return launch_k<NT, CH, 8, X2>(cfg, p);
    }
}

template <sfmp_dtype DT>
cudaError_t launch_t(const Params& p, const XParams& xp, int xitems, int max_cols, int grid, size_t smem,
                     int lo, cudaStream_t st, bool overlap_prev) {
    constexpr bool X2 = DT == SFMP_F32;
    const size_t elem = DT == SFMP_F32 ? 4 : 2;
    // K4: activation records (normal launch: it overwrites the workspace the
    // previous call may still read, and x may be that call's output, so it
    // follows it in stream order).
    int maxM = 1;
    for (int i = 0; i < xp.nlin; ++i) maxM = std::max(maxM, xp.lin[i].M);
    const int NT = maxM > 8 ? 2 : 1;
    const size_t row_smem = static_cast<size_t>(8) * p.n_b * 4 + static_cast<size_t>(max_cols) * elem;
    bool any_norm = false;
    for (int i = 0; i < xp.nlin; ++i) any_norm = any_norm || xp.lin[i].norm.on;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    // overlap_prev: a later launch of one grouped call (independent problems,
    // workspaces disjoint from the earlier launches'): the pre-pass may start
    // while the previous GEMV still runs, and this call's GEMV then fills the
    // previous one's tail.
    a[0].val.programmaticStreamSerializationAllowed = (overlap_prev || (!any_norm && SFMP_XPREP_PDL)) ? 1 : 0;
    XParams xq = xp;
    xq.wait_prev = overlap_prev ? 1 : 0;
    // the gather pre-pass is always a programmatic dependent: its launch and the
    // col_perm load overlap the previous kernel's tail, it waits before x
    xq.wait_first = (!overlap_prev && !any_norm && SFMP_XPREP_PDL) ? 1 : 0;
    cudaLaunchConfig_t c{};
    c.gridDim = dim3(xitems);
    c.blockDim = dim3(256);
    c.stream = st;
    c.attrs = a;
    c.numAttrs = 1;
    if (SFMP_EXP_NOPREPASS) {  // experiment builds only: records left as they are
    } else if (!any_norm) {
        note_launch();
        cudaError_t e = cudaLaunchKernelEx(&c, xprep_gather_kernel<DT>, xq);
        if (e != cudaSuccess) return e;
    } else {
        // the fused RMSNorm needs each token's whole row: the staged pre-pass
        if (row_smem > static_cast<size_t>(kXprepRowLimit)) return cudaErrorNotSupported;
        static std::once_flag fl[64];
        once_per_device(fl, [] {
            cudaFuncSetAttribute(xprep_rows_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kXprepRowLimit);
            // same carveout as the GEMV: an SM running a pre-pass CTA needs no
            // reconfiguration before the GEMV's CTAs can join it
            cudaFuncSetAttribute(xprep_rows_kernel<DT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        });
        c.dynamicSmemBytes = row_smem;
        note_launch();
        cudaError_t e = cudaLaunchKernelEx(&c, xprep_rows_kernel<DT>, xq);
        if (e != cudaSuccess) return e;
    }
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    // K1: persistent CTAs over the work queue, programmatic dependent of the pre-pass
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
    cudaError_t e;
    if (NT == 1) e = CH == 1 ? launch_nc<1, 1, X2>(cfg, p, lo) : launch_nc<1, 2, X2>(cfg, p, lo);
    else e = CH == 1 ? launch_nc<2, 1, X2>(cfg, p, lo) : launch_nc<2, 2, X2>(cfg, p, lo);
    if (e != cudaSuccess || p.n_fix == 0 || SFMP_EXP_NOFIXUP) return e;
    // split tiles: sum the segment partials (programmatic dependent of the GEMV)
    cudaLaunchConfig_t fc{};
    fc.gridDim = dim3((p.n_fix + 8 * kFixPairs - 1) / (8 * kFixPairs));  // kFixPairs (tile, token) pairs per warp
    fc.blockDim = dim3(256);
    fc.stream = st;
    fc.attrs = pdl;
    fc.numAttrs = 1;
    note_launch();
    return cudaLaunchKernelEx(&fc, gemv_fixup_kernel, p);
}

// Canonical K segment: kSegCols columns for every linear (measured: 512- or
// 256-column segments for small linears raised configs[0] from 10.4 to 11.7 us
// and the 8B decode launch by 5 %: more partials and fix-up work than balance gained).
int units_per_segment(const DevModel& m) { return std::max(1, kSegCols / static_cast<int>(m.n_b)); }
int segments_per_tile(const DevModel& m) {
    const int L = units_per_segment(m);
    return (static_cast<int>(m.BC) + L - 1) / L;
}

// Work items of one launch.  A multi-segment linear runs either one item per
// (tile, segment) -- partials summed by the fix-up -- or one item per tile
// that sums its segments in registers: the same float operations, so the
// choice changes no bit and is made per call for balance.  Whole-K items
// (fewer claims, no partial traffic, no fix-up) go first in the queue,
// shortest K first; the small items -- split linears and single-segment
// ones -- go last, so the dynamic queue still ends evenly: the small-item
// work per CTA slot must cover kWholeFrac of the longest whole-K item, and
// the call keeps at least two items per CTA slot.
#ifndef SFMP_WHOLE_FRAC
#define SFMP_WHOLE_FRAC 0.5
#endif
#ifndef SFMP_WHOLE_MAX
#define SFMP_WHOLE_MAX 0.35  // longest whole-K item / average units per CTA slot
#endif
void plan_items(Params& p, int slots, bool allow) {
    const int n = p.nlin;
    double small = 0.0;
    int items = 0;
    for (int i = 0; i < n; ++i) {
        small += static_cast<double>(p.lin[i].RT) * p.lin[i].BC;
        items += p.lin[i].RT * p.lin[i].P;
    }
    const double total = small;
    p.any_whole = 0;
    int order[kMaxLin];
    for (int i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order, order + n, [&](int a, int b) { return p.lin[a].BC < p.lin[b].BC; });
    int longest = 0;
    for (int k = 0; k < n; ++k) {
        Lin& L = p.lin[order[k]];
        if (L.P < 2 || !allow) continue;
        const double rest = small - static_cast<double>(L.RT) * L.BC;
        const int items_after = items - L.RT * (L.P - 1);
        const int lw = std::max(longest, L.BC);
        if (rest < SFMP_WHOLE_FRAC * slots * lw || lw > SFMP_WHOLE_MAX * total / slots || items_after < 2 * slots) break;
        L.IP = 1;
        p.any_whole = 1;
        small = rest;
        items = items_after;
        longest = std::max(longest, L.BC);
    }
    int q = 0, it = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i < n; ++i) {
            Lin& L = p.lin[i];
            if ((L.IP == 1 && L.P > 1) != (pass == 0)) continue;
            p.qlin[q] = i;
            p.item_start[q++] = it;
            L.item0 = it;
            it += L.RT * L.IP;
        }
}

// Shared-memory plan of one launch: stages and resident CTAs per SM (fewer
// CTAs when two stages of the widest unit + record section would not fit).
struct SmemPlan {
    int stages, ctas;
    size_t smem;
};
SmemPlan smem_plan(uint32_t stage_w, uint32_t rec_slot, int NT, int LO = 8, bool X2 = true) {
    for (int ctas = ctas_per_sm(NT, LO, X2); ctas >= 1; --ctas) {
        const int budget = (ctas == 1 ? 227 * 1024 : kSmemSM / ctas) - kHdrBytes;
        const int stages = std::min<int>(SFMP_MAX_STAGES, budget / static_cast<int>(stage_w + rec_slot));
        if (stages >= 2) return {stages, ctas, kHdrBytes + static_cast<size_t>(stages) * (stage_w + rec_slot)};
    }
    return {0, 0, 0};
}
int layouts_of(const DevModel& m) { return m.ceil_bits > m.floor_bits ? 2 : 1; }
int units_per_stage(const DevModel& m) { return m.n_b == 128 ? SFMP_SU : 1; }
uint32_t stage_bytes(const DevModel& m, int ceil_bits) {
    return (units_per_stage(m) * unit_bytes(ceil_bits, static_cast<int>(m.n_b / 8)) + 127) / 128 * 128;
}

}  // namespace

// Workspace: activation records | segment partials | queue | row exponents.
size_t gemv_rec_bytes(const DevModel& m) {
    const size_t rec = static_cast<size_t>(layouts_of(m)) * RecGeom{16, true}.sec_bytes(static_cast<int>(m.n_b / 128));
    return (static_cast<size_t>(m.BC) * rec + 255) / 256 * 256;
}
size_t gemv_part_bytes(const DevModel& m) {
    return segments_per_tile(m) > 1 ? static_cast<size_t>(m.RT) * segments_per_tile(m) * 16 * kTR * 4 : 0;
}
size_t gemv_workspace_bytes(const DevModel& m, int M) {
    (void)M;
    return gemv_rec_bytes(m) + gemv_part_bytes(m) + 128;  // + queue[2] | pad | exponents[16]
}

int gemv_ctas_per_sm(int NT) { return ctas_per_sm(NT); }

bool gemv_feasible(const DevModel& m) {
    return smem_plan(stage_bytes(m, m.ceil_bits),
                     units_per_stage(m) * static_cast<uint32_t>(RecGeom{16, true}.sec_bytes(static_cast<int>(m.n_b / 128))), 2)
               .stages >= 2;
}

bool gemv_groupable(const DevModel& a, const DevModel& b) {
    return a.gemv_ok && b.gemv_ok && a.n_b == b.n_b && a.floor_bits == b.floor_bits && a.device == b.device;
}

cudaError_t launch_gemv_group(const DevModel* const* ms, const void* const* xs, float* const* ys, uint8_t* const* wss,
                              const int* Ms, int n, sfmp_dtype dt, cudaStream_t st, bool overlap_prev,
                              const PreNorm* norms) {
    if (n < 1 || n > kMaxLin) return cudaErrorInvalidValue;
    const DevModel& m0 = *ms[0];
    int M = 0;
    for (int i = 0; i < n; ++i) {
        if (Ms[i] < 1 || Ms[i] > 16) return cudaErrorInvalidValue;
        M = std::max(M, Ms[i]);
    }
    const int NT = M > 8 ? 2 : 1;  // the widest linear's n-tile count
    const bool X2 = dt == SFMP_F32;
    const int CH = static_cast<int>(m0.n_b / 128);
    Params p{};
    XParams xp{};
    p.nlin = xp.nlin = n;
    xp.M = M;
    p.n_b = xp.n_b = static_cast<int>(m0.n_b);
    p.sec_bytes = static_cast<uint32_t>(RecGeom{M, X2}.sec_bytes(CH));  // stage stride: the largest
    int ceil_bits = 0, items = 0, fix = 0, xitems = 0, max_cols = 0;
    for (int i = 0; i < n; ++i) {
        const DevModel& m = *ms[i];
        ceil_bits = std::max(ceil_bits, m.ceil_bits);
        Lin& L = p.lin[i];
        const int BC = static_cast<int>(m.BC);
        const RecGeom G{Ms[i], X2};
        const int nl = layouts_of(m);
        L.payload = m.d_payload;
        L.unit_desc = m.d_unit_desc;
        L.out_map = m.d_out_map;
        L.xrec = wss[i];
        L.y = ys[i];
        L.part = reinterpret_cast<float*>(wss[i] + gemv_rec_bytes(m));
        L.out_rows = m.out_rows;
        L.BC = BC;
        L.RT = static_cast<int>(m.RT);
        L.M = Ms[i];
        L.L = units_per_segment(m);
        L.P = segments_per_tile(m);
        L.sec_bytes = static_cast<uint32_t>(G.sec_bytes(CH));
        L.lo_off = static_cast<uint32_t>(G.lo_off());
        L.lo = m.floor_bits;
        L.IP = L.P;
        XLin& X = xp.lin[i];
        X.x = xs[i];
        X.col_perm = m.d_col_perm;
        X.xrec = wss[i];
        X.BC = BC;
        X.cols = static_cast<int>(m.cols);
        X.item0 = xitems;
        X.lo = m.floor_bits;
        X.nl = nl;
        X.M = Ms[i];
        X.sec_bytes = L.sec_bytes;
        if (norms) X.norm = norms[i];
        xitems += (BC + 7) / 8 * Ms[i];  // pre-pass CTAs: (8 block columns) x tokens
        max_cols = std::max(max_cols, X.cols);
    }
    // the launch's work queue lives in the first problem's workspace (problems
    // of one launch have distinct workspaces)
    p.queue = reinterpret_cast<unsigned*>(wss[0] + gemv_rec_bytes(m0) + gemv_part_bytes(m0));
    p.stage_w = stage_bytes(m0, ceil_bits);
    const SmemPlan sp = smem_plan(p.stage_w, units_per_stage(m0) * p.sec_bytes, NT, m0.floor_bits, X2);
    if (sp.stages < 2) return cudaErrorInvalidConfiguration;  // excluded at upload (gemv_feasible)
    p.stages = sp.stages;
    plan_items(p, m0.num_sms * sp.ctas, CH == 1 && !X2);
    for (int i = 0; i < n; ++i) {
        Lin& L = p.lin[i];
        p.fix_start[i] = fix;
        L.fix0 = fix;
        if (L.IP > 1) fix += L.RT * L.M;  // (tile, token) fix-up pairs
        items += L.RT * L.IP;
    }
    p.n_items = items;
    p.n_fix = fix;
    p.item_start[n] = items;
    p.fix_start[n] = fix;
    const int grid = std::min(items, m0.num_sms * sp.ctas);
    switch (dt) {
        case SFMP_F32: return launch_t<SFMP_F32>(p, xp, xitems, max_cols, grid, sp.smem, m0.floor_bits, st, overlap_prev);
        case SFMP_F16: return launch_t<SFMP_F16>(p, xp, xitems, max_cols, grid, sp.smem, m0.floor_bits, st, overlap_prev);
        default: return launch_t<SFMP_BF16>(p, xp, xitems, max_cols, grid, sp.smem, m0.floor_bits, st, overlap_prev);
    }
}

cudaError_t launch_gemv(const DevModel& m, const void* x, sfmp_dtype dt, int M, float* y, float* ws,
                        cudaStream_t st, const PreNorm* norm) {
    const DevModel* ms[1] = {&m};
    const void* xs[1] = {x};
    float* ys[1] = {y};
    uint8_t* wss[1] = {reinterpret_cast<uint8_t*>(ws)};
    const int Ms[1] = {M};
    return launch_gemv_group(ms, xs, ys, wss, Ms, 1, dt, st, false, norm);
}

}  // namespace sfmpk
