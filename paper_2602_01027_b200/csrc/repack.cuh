// repack.cuh -- upload-time re-arrangement of the bits of <=4-bit units for
// the decode GEMV (same bytes per weight, SURVEY §7 hard part 3(c)).
//
// SFMPPKD1 stores a 32-weight row group of a B-bit block as B bit-plane words
// (plane i = bit i of each code, weight k = bit k; layout.cpp:58-61).  The
// decode GEMV needs, for each of the 16 f16x2 MMA A registers j of the group,
// the codes of weights (lo(j), hi(j)) = (4h+a, 4h+a+16), j = 4a+h, in f16
// mantissa bits under a magic exponent.  From planes that is a bit-matrix
// transpose (~1.1 instructions/weight).  Here the same B words are refilled so
// that register j is ONE lop3 (and an occasional shift) of a word:
//   code(lo(j)) at bits [s_j + p_j, +B) of word w_j, code(hi(j)) at +16,
// which an `(t & mask) | magic` with magic = 2^(10-p_j) turns into
// f16x2(2^(10-p_j) + c_lo, 2^(10-p_j) + c_hi) exactly.  The per-slot magics
// are folded into the per-token bias of the activation record.
//   B=4: w=j/4, r=j%4: s=8*(r>>1), p=4*(r&1)            (5 ops / 8 weights)
//   B=3: w=j/5, r=j%5: s=9*(r>=3), p=3*(r%3); j=15 takes bit i of its codes
//        from bit 15 / 31 of word i                        (24 ops / 32)
//   B=2: w=j/8, r=j%8: s=10*(r>=5), p=2*(r%5)            (18 ops / 32)
//   B=1: w=0: s=10*(j>=10), p=j%10                        (17 ops / 32)
// Units with B >= 5 keep the plane layout.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace sfmpk {

__host__ __device__ constexpr int rp_word(int B, int j) {
    return B == 4 ? j / 4 : B == 3 ? (j == 15 ? -1 : j / 5) : B == 2 ? j / 8 : 0;
}
__host__ __device__ constexpr int rp_shift(int B, int j) {
    return B == 4 ? 8 * ((j % 4) >> 1) : B == 3 ? 9 * ((j % 5) >= 3) : B == 2 ? 10 * ((j % 8) >= 5) : 10 * (j >= 10);
}
__host__ __device__ constexpr int rp_pos(int B, int j) {
    return B == 4 ? 4 * ((j % 4) & 1) : B == 3 ? (j == 15 ? 0 : 3 * ((j % 5) % 3)) : B == 2 ? 2 * ((j % 8) % 5) : j % 10;
}
// f16 bits of the magic 2^(10-p) (exponent field 25-p)
__host__ __device__ constexpr uint32_t rp_magic_bits(int B, int j) {
    return static_cast<uint32_t>(25 - rp_pos(B, j)) << 10;
}
__host__ __device__ constexpr float rp_magic(int B, int j) {
    return static_cast<float>(1 << (10 - rp_pos(B, j)));
}
// weight k (0..31) of a group <-> register j and half
__host__ __device__ constexpr int rp_reg_of(int k) { return 4 * (k % 4) + (k % 16) / 4; }
__host__ __device__ constexpr int rp_half_of(int k) { return k / 16; }

// Code of weight k from the B repacked words of its group.
__host__ __device__ inline uint32_t rp_code(const uint32_t* w, int B, int k) {
    const int j = rp_reg_of(k), half = rp_half_of(k);
    if (B == 3 && j == 15) {
        uint32_t c = 0;
        for (int i = 0; i < 3; ++i) c |= ((w[i] >> (15 + 16 * half)) & 1u) << i;
        return c;
    }
    return (w[rp_word(B, j)] >> (rp_shift(B, j) + rp_pos(B, j) + 16 * half)) & ((1u << B) - 1u);
}

// Host: codes[32] of one group -> B repacked words.
__host__ __device__ inline void rp_pack(const uint32_t* codes, int B, uint32_t* out) {
    for (int i = 0; i < B; ++i) out[i] = 0u;
    for (int k = 0; k < 32; ++k) {
        const int j = rp_reg_of(k), half = rp_half_of(k);
        const uint32_t c = codes[k];
        if (B == 3 && j == 15) {
            for (int i = 0; i < 3; ++i) out[i] |= ((c >> i) & 1u) << (15 + 16 * half);
        } else {
            out[rp_word(B, j)] |= c << (rp_shift(B, j) + rp_pos(B, j) + 16 * half);
        }
    }
}

// Exponent offset of register j's codes when read as f16 SUBNORMALS: with the
// exponent field zero, mantissa bits [p, p+B) holding c give exactly
// c * 2^(p-24), so the activation paired with register j is pre-scaled by
// 2^(24-p) (the decode pre-pass) and the MMA contracts the exact codes with
// no magic offset to cancel.  Wider (5..8-bit) units put c at p = 0.
__host__ __device__ constexpr int sub_pos(int B, int j) { return B <= 4 ? rp_pos(B, j) : 0; }

// Logical right shift on the FMA pipe (IMAD.HI) instead of the ALU pipe
// (SHF), which the unpack LOP3s saturate.
#ifndef SFMP_SHR_IMAD
#define SFMP_SHR_IMAD 0
#endif
template <int K>
__device__ __forceinline__ uint32_t shr_k(uint32_t w) {
    if constexpr (SFMP_SHR_IMAD) return __umulhi(w, 1u << (32 - K));
    else return w >> K;
}

// Device: 16 f16x2 registers from the B repacked words, codes as subnormals
// (one LOP3 AND per register; no magic exponent).
template <int B>
__device__ __forceinline__ void unpack_rp_sub(const uint32_t* w, uint32_t (&H)[16]) {
    uint32_t sh[B];
#pragma unroll
    for (int i = 0; i < B; ++i) sh[i] = shr_k<(B == 4 ? 8 : B == 3 ? 9 : 10)>(w[i]);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if constexpr (B == 3) {
            if (j == 15) {
                const uint32_t t1 = shr_k<14>(w[1]) & 0x00020002u;
                const uint32_t t2 = lop3_and_or(shr_k<13>(w[2]), 0x00040004u, t1);
                H[15] = lop3_and_or(shr_k<15>(w[0]), 0x00010001u, t2);
                continue;
            }
        }
        const int wi = rp_word(B, j), s = rp_shift(B, j), p = rp_pos(B, j);
        const uint32_t src = s ? sh[wi] : w[wi];
        const uint32_t m = ((1u << B) - 1u) << p;
        H[j] = src & (m | (m << 16));
    }
}

// Device: 16 f16x2 (2^(10-p_j) + c) registers from the B repacked words.
template <int B>
__device__ __forceinline__ void unpack_rp(const uint32_t* w, uint32_t (&H)[16]) {
    constexpr int NW = B;
    uint32_t sh[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) sh[i] = w[i] >> (B == 4 ? 8 : B == 3 ? 9 : 10);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if constexpr (B == 3) {
            if (j == 15) {
                const uint32_t t1 = lop3_and_or(w[1] >> 14, 0x00020002u, 0x64006400u);
                const uint32_t t2 = lop3_and_or(w[2] >> 13, 0x00040004u, t1);
                H[15] = lop3_and_or(w[0] >> 15, 0x00010001u, t2);
                continue;
            }
        }
        const int wi = rp_word(B, j), s = rp_shift(B, j), p = rp_pos(B, j);
        const uint32_t src = s ? sh[wi] : w[wi];
        const uint32_t m = ((1u << B) - 1u) << p;
        const uint32_t mg = rp_magic_bits(B, j);
        H[j] = lop3_and_or(src, m | (m << 16), mg | (mg << 16));
    }
}

// Lane-major unit order of the decode GEMV (128-row units; gemv_tc.cu): the
// compute warp cw (rows 32cw..32cw+31) lane (g, q) = 4g + q owns rows
// 32cw + 8r + g (r = 0..3) and word q of each 16-byte row segment of a
// 128-column chunk.  s/z: [cw][g][r] (s, z) fp16 pairs, 512 B.  Planes (after
// the s/z block): [chunk c][cw][plane i][lane][r] 4-byte words.
__host__ __device__ constexpr uint32_t lm_sz_off(uint32_t row) {
    return (row >> 5) * 128 + (row & 7) * 16 + ((row >> 3) & 3) * 4;
}
__host__ __device__ constexpr uint32_t lm_word_off(uint32_t B, uint32_t c, uint32_t row, uint32_t q, uint32_t i) {
    return c * (B * 2048) + (row >> 5) * (B * 512) + i * 512 + ((row & 7) * 4 + q) * 16 + ((row >> 3) & 3) * 4;
}

}  // namespace sfmpk
