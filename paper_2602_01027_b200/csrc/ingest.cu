// ingest.cu -- device-side ingest / repack: the SFMPPKD1 block
// region (layout.cpp:179-208) is uploaded as stored, and the two device
// layouts are built by kernels instead of host loops over every weight:
//  * unit_layout_kernel -- the decode GEMV's unit-major, lane-major layout
//    (sfmp_internal.h, repack.cuh): one thread per (unit, row, 32-weight
//    group) reads the group's B plane words, re-arranges <= 4-bit groups
//    for one-LOP3 unpacking (rp_pack) and writes them and the row's (s, z).
//  * tile_layout_kernel -- the prefill GEMM's row-tile layout
//    (gemm_tcgen05.cu): one warp per (128 output rows, 128 columns): s, z,
//    high-row mask, floor planes, and the ceil plane compacted over the high
//    rows with a warp prefix count.
// Blocks start at arbitrary byte offsets in the stream, so the kernels read
// the raw region with byte loads.  The host keeps the cheap O(blocks) and
// O(rows x column-chunks) bookkeeping (unit offsets, tile offsets).
#include <cuda_runtime.h>

#include "repack.cuh"
#include "sfmp_internal.h"

namespace sfmpk {
namespace {

__device__ __forceinline__ uint32_t ld_u32_bytes(const uint8_t* p) {
    return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
           (static_cast<uint32_t>(p[3]) << 24);
}

struct IngestGeom {
    const uint8_t* raw;        // the model's blocks as stored (local block order)
    const uint64_t* raw_off;   // [K] byte offset of each local block in raw
    const uint8_t* bits;       // [K]
    uint32_t m_b, n_b, BC, tiles;  // tiles = m_b / 128 unit rows per block row
};

// grid: (units, 128 rows / 8) ; block 8 x groups threads
__global__ void __launch_bounds__(256) unit_layout_kernel(const IngestGeom g, const uint64_t* __restrict__ unit_desc,
                                                          uint8_t* __restrict__ dst) {
    const uint32_t u = blockIdx.x;
    const uint32_t groups = g.n_b / 32;
    const uint32_t rr = blockIdx.y * 8 + threadIdx.x / groups, gi = threadIdx.x % groups;
    if (rr >= 128) return;
    const uint32_t rt = u / g.BC, bc = u % g.BC;
    const uint32_t br = rt / g.tiles, t = rt % g.tiles;
    const uint64_t k = static_cast<uint64_t>(br) * g.BC + bc;
    const int B = g.bits[k];
    const uint32_t nb8 = g.n_b / 8, row = t * 128 + rr;  // row within the block
    const uint8_t* blk = g.raw + g.raw_off[k];
    uint8_t* du = dst + (unit_desc[u] & 0xFFFFFFFFFFFFull);
    if (gi == 0) {  // (s, z) of the row, fp16 as stored
        uint8_t* sz = du + lm_sz_off(rr);
        sz[0] = blk[2 * row];
        sz[1] = blk[2 * row + 1];
        sz[2] = blk[2 * g.m_b + 2 * row];
        sz[3] = blk[2 * g.m_b + 2 * row + 1];
    }
    const uint8_t* planes = blk + 4ull * g.m_b;
    uint32_t pw[8], out[8];
    for (int i = 0; i < B; ++i)
        pw[i] = ld_u32_bytes(planes + static_cast<uint64_t>(i) * g.m_b * nb8 + static_cast<uint64_t>(row) * nb8 + gi * 4);
    if (B <= 4) {
        uint32_t codes[32];
        for (int kk = 0; kk < 32; ++kk) {
            uint32_t c = 0;
            for (int i = 0; i < B; ++i) c |= ((pw[i] >> kk) & 1u) << i;
            codes[kk] = c;
        }
        rp_pack(codes, B, out);
    } else {
        for (int i = 0; i < B; ++i) out[i] = pw[i];
    }
    for (int i = 0; i < B; ++i)
        *reinterpret_cast<uint32_t*>(du + 512 + lm_word_off(static_cast<uint32_t>(B), gi >> 2, rr, gi & 3,
                                                             static_cast<uint32_t>(i))) = out[i];
}

constexpr int kTileHdr = 528;          // scales[128] | zeros[128] | highmask[16]  (gemm_tcgen05.cu kUnitHdr)
constexpr int kTilePlane = 128 * 16;   // one plane of a 128 x 128 tile

// grid: tiles (T * KC); block 32 threads, lane owns output rows 4*lane .. +3
__global__ void __launch_bounds__(32) tile_layout_kernel(const IngestGeom g, const uint32_t* __restrict__ inv,
                                                         const uint64_t* __restrict__ woff, uint32_t KC, int F,
                                                         uint8_t* __restrict__ dst) {
    const uint32_t T = blockIdx.x / KC, kc = blockIdx.x % KC, lane = threadIdx.x;
    uint8_t* du = dst + woff[blockIdx.x];
    const uint32_t bc = kc * 128 / g.n_b, sub = (kc * 128 % g.n_b) / 8, nb8 = g.n_b / 8;
    const uint8_t* src[4];
    bool high[4];
    uint32_t hmask = 0;
    for (int j = 0; j < 4; ++j) {
        const uint32_t r = 4 * lane + j, i = inv[T * 128 + r];
        src[j] = nullptr;
        high[j] = false;
        if (i == 0xFFFFFFFFu) continue;
        const uint32_t br = i / g.m_b, rb = i % g.m_b;
        const uint64_t k = static_cast<uint64_t>(br) * g.BC + bc;
        const uint8_t* blk = g.raw + g.raw_off[k];
        src[j] = blk;
        high[j] = g.bits[k] > F;
        hmask |= (high[j] ? 1u : 0u) << j;
        // scales, zeros
        du[2 * r] = blk[2 * rb];
        du[2 * r + 1] = blk[2 * rb + 1];
        du[256 + 2 * r] = blk[2 * g.m_b + 2 * rb];
        du[256 + 2 * r + 1] = blk[2 * g.m_b + 2 * rb + 1];
        const uint8_t* planes = blk + 4ull * g.m_b + static_cast<uint64_t>(rb) * nb8 + sub;
        for (int pi = 0; pi < F; ++pi)
            for (int b = 0; b < 16; ++b) du[kTileHdr + pi * kTilePlane + r * 16 + b] = planes[static_cast<uint64_t>(pi) * g.m_b * nb8 + b];
    }
    // high-row mask: bit r%8 of byte 512 + r/8 (rows 4*lane .. +3 share one byte half)
    const uint32_t allm = __ballot_sync(0xffffffffu, hmask != 0);
    (void)allm;
    const uint32_t nib = hmask & 0xFu;
    const uint32_t other = __shfl_xor_sync(0xffffffffu, nib, 1);
    if ((lane & 1) == 0) du[512 + lane / 2] = static_cast<uint8_t>(nib | (other << 4));
    // ceil planes of the high rows, compacted in row order
    const uint32_t cnt = __popc(nib);
    uint32_t before = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, before, o);
        if (lane >= static_cast<uint32_t>(o)) before += v;
    }
    before -= cnt;  // exclusive prefix
    for (int j = 0; j < 4; ++j) {
        if (!high[j]) continue;
        const uint32_t r = 4 * lane + j, i = inv[T * 128 + r], rb = i % g.m_b;
        const uint8_t* plane = src[j] + 4ull * g.m_b + static_cast<uint64_t>(F) * g.m_b * nb8 + static_cast<uint64_t>(rb) * nb8 + sub;
        for (int b = 0; b < 16; ++b) du[kTileHdr + F * kTilePlane + before * 16 + b] = plane[b];
        ++before;
    }
}

}  // namespace

cudaError_t device_unit_layout(const uint8_t* raw, const uint64_t* raw_off, const uint8_t* bits, uint32_t m_b,
                               uint32_t n_b, uint32_t BC, uint32_t units, const uint64_t* unit_desc, uint8_t* dst,
                               cudaStream_t st) {
    IngestGeom g{raw, raw_off, bits, m_b, n_b, BC, m_b / 128};
    note_launch();
    unit_layout_kernel<<<dim3(units, 16), 8 * (n_b / 32), 0, st>>>(g, unit_desc, dst);
    return cudaGetLastError();
}

cudaError_t device_tile_layout(const uint8_t* raw, const uint64_t* raw_off, const uint8_t* bits, uint32_t m_b,
                               uint32_t n_b, uint32_t BC, const uint32_t* inv, const uint64_t* woff, uint64_t tiles,
                               uint32_t KC, int F, uint8_t* dst, cudaStream_t st) {
    IngestGeom g{raw, raw_off, bits, m_b, n_b, BC, m_b / 128};
    note_launch();
    tile_layout_kernel<<<static_cast<unsigned>(tiles), 32, 0, st>>>(g, inv, woff, KC, F, dst);
    return cudaGetLastError();
}

}  // namespace sfmpk
