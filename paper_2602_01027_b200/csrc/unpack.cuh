// unpack.cuh -- bit-plane -> f16 code conversion shared by the decode GEMV
// (K1) and the prefill GEMM (K2).  Codes follow unpack_block
// (layout.cpp:67-86): weight k of a row = bit (k mod 8) of byte k/8 of each
// plane, plane i carrying bit i of the code.
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

#include "ptx.cuh"

namespace sfmpk {

// Bit-matrix transpose of NP (<=4) plane words (bit j = weight j of the
// 32-weight word) into nibble words: q[a] nibble n = code of weight 4n+a.
// Each delta-swap half is one shift plus one LOP3 select (15 ops for 3 planes).
template <int NP>
__device__ __forceinline__ void planes_to_nibbles(const uint32_t* p, uint32_t (&q)[4]) {
    constexpr uint32_t kO = 0xAAAAAAAAu, kH = 0xCCCCCCCCu;
    uint32_t r0, r1, r2 = 0u, r3 = 0u;
    // stage 1: pairs (p0,p1), (p2,p3) -> 2-bit crumbs
    if constexpr (NP > 1) {
        r0 = lop3_sel<kO>(p[0], p[1] << 1);
        r1 = lop3_sel<kO>(p[0] >> 1, p[1]);
    } else {
        r0 = p[0] & ~kO;
        r1 = (p[0] >> 1) & ~kO;
    }
    if constexpr (NP > 3) {
        r2 = lop3_sel<kO>(p[2], p[3] << 1);
        r3 = lop3_sel<kO>(p[2] >> 1, p[3]);
    } else if constexpr (NP > 2) {
        r2 = p[2] & ~kO;
        r3 = (p[2] >> 1) & ~kO;
    }
    // stage 2: pairs (r0,r2), (r1,r3) -> nibbles
    if constexpr (NP > 2) {
        q[0] = lop3_sel<kH>(r0, r2 << 2);
        q[2] = lop3_sel<kH>(r0 >> 2, r2);
        q[1] = lop3_sel<kH>(r1, r3 << 2);
        q[3] = lop3_sel<kH>(r1 >> 2, r3);
    } else {
        q[0] = r0 & ~kH;
        q[2] = (r0 >> 2) & ~kH;
        q[1] = r1 & ~kH;
        q[3] = (r1 >> 2) & ~kH;
    }
}

// Nibble word -> 4 f16x2 with magic offsets (exact):
// h[0]=(nib0,nib4)+1024 h[1]=(nib1,nib5)+64 h[2]=(nib2,nib6)+1024 h[3]=(nib3,nib7)+64.
__device__ __forceinline__ void nibbles_to_h2_biased(uint32_t q, uint32_t* h) {
    const uint32_t q8 = q >> 8;
    h[0] = lop3_and_or(q, 0x000F000Fu, 0x64006400u);   // 1024 + c (ulp 1)
    h[1] = lop3_and_or(q, 0x00F000F0u, 0x54005400u);   // 64 + c   (ulp 1/16, bits 4-7)
    h[2] = lop3_and_or(q8, 0x000F000Fu, 0x64006400u);
    h[3] = lop3_and_or(q8, 0x00F000F0u, 0x54005400u);
}

// Exact codes (no offset), used for 5..8-bit blocks where hi*16+lo must stay exact.
__device__ __forceinline__ void nibbles_to_h2_exact(uint32_t q, uint32_t* h) {
    const __half2 k1024 = u32_as_h2(0x64006400u);
    const __half2 k64 = u32_as_h2(0x54005400u);
    uint32_t b[4];
    nibbles_to_h2_biased(q, b);
    h[0] = h2_as_u32(__hsub2(u32_as_h2(b[0]), k1024));
    h[1] = h2_as_u32(__hsub2(u32_as_h2(b[1]), k64));
    h[2] = h2_as_u32(__hsub2(u32_as_h2(b[2]), k1024));
    h[3] = h2_as_u32(__hsub2(u32_as_h2(b[3]), k64));
}

// All 32 weights of one row word as 16 f16x2; H[4a+h] = weights (4h+a,
// 4h+a+16) of the word.  B<=4: magic-biased codes; B>4: exact codes.
template <int B>
__device__ __forceinline__ void unpack_word(const uint32_t* p, uint32_t (&H)[16]) {
    uint32_t q[4];
    if constexpr (B <= 4) {
        planes_to_nibbles<B>(p, q);
#pragma unroll
        for (int a = 0; a < 4; ++a) nibbles_to_h2_biased(q[a], H + 4 * a);
    } else {
        uint32_t qh[4];
        planes_to_nibbles<4>(p, q);
        planes_to_nibbles<B - 4>(p + 4, qh);
        const __half2 k16 = u32_as_h2(0x4C004C00u);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            uint32_t lo[4], hi[4];
            nibbles_to_h2_exact(q[a], lo);
            nibbles_to_h2_exact(qh[a], hi);
#pragma unroll
            for (int h = 0; h < 4; ++h)
                H[4 * a + h] = h2_as_u32(__hfma2(u32_as_h2(hi[h]), k16, u32_as_h2(lo[h])));
        }
    }
}

// 5..8-bit units for the decode GEMV: exact codes as f16 subnormals
// c * 2^-24 (code in mantissa bits 0-7, exponent 0); H[4a+h] = weights
// (4h+a, 4h+a+16) of the word.
template <int B>
__device__ __forceinline__ void unpack_word_sub(const uint32_t* p, uint32_t (&H)[16]) {
    static_assert(B > 4 && B <= 8, "wide codes only");
    uint32_t q[4], qh[4];
    planes_to_nibbles<4>(p, q);
    planes_to_nibbles<B - 4>(p + 4, qh);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            // nibble h of q (low 4 bits) and of qh (high bits), both halves
            const uint32_t lo = (q[a] >> (4 * h)) & 0x000F000Fu;
            const uint32_t hi = h == 0 ? (qh[a] << 4) : h == 1 ? qh[a] : (qh[a] >> (4 * h - 4));
            H[4 * a + h] = lop3_and_or(hi, 0x00F000F0u, lo);
        }
}

}  // namespace sfmpk
