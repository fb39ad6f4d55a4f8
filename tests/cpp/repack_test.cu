// Host-side check of the repacked decode layout (csrc/repack.cuh): for every
// bit-width 1..4 and random codes, pack -> decode is the identity, the words
// hold exactly B*32 bits (same bytes as B bit planes), and the device unpack
// formula (mask | magic, shift) evaluated on the host gives 2^(10-p) + c.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../paper_2602_01027_b200/csrc/repack.cuh"

using namespace sfmpk;

static float h2f(uint16_t h) {  // exact f16 -> f32 for normal values
    const uint32_t e = (h >> 10) & 0x1F, m = h & 0x3FF;
    uint32_t u = ((e - 15 + 127) << 23) | (m << 13);
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

int main() {
    unsigned seed = 12345;
    auto rnd = [&]() { seed = seed * 1103515245u + 12345u; return seed >> 8; };
    int bad = 0;
    for (int B = 1; B <= 4; ++B)
        for (int trial = 0; trial < 2000; ++trial) {
            uint32_t codes[32], w[4];
            for (int k = 0; k < 32; ++k) codes[k] = rnd() & ((1u << B) - 1u);
            rp_pack(codes, B, w);
            int ones = 0;
            for (int k = 0; k < 32; ++k) {
                if (rp_code(w, B, k) != codes[k]) ++bad;
                ones += __builtin_popcount(codes[k]);
            }
            int wones = 0;
            for (int i = 0; i < B; ++i) wones += __builtin_popcount(w[i]);
            if (ones != wones) ++bad;  // a bijection of bits: no bit lost or duplicated
            // device formula per register j: (t & mask) | magic, t = w >> shift
            for (int j = 0; j < 16; ++j) {
                for (int half = 0; half < 2; ++half) {
                    const int k = 16 * half + 4 * (j & 3) + (j >> 2);  // weight of register j, half
                    if (!(rp_reg_of(k) == j && rp_half_of(k) == half)) ++bad;
                    uint32_t c;
                    if (B == 3 && j == 15) {
                        c = 0;
                        for (int i = 0; i < 3; ++i) c |= ((w[i] >> (15 + 16 * half)) & 1u) << i;
                        const float v = 1024.f + c;
                        if (v - rp_magic(B, j) != static_cast<float>(codes[k])) ++bad;
                        continue;
                    }
                    const uint32_t t = w[rp_word(B, j)] >> rp_shift(B, j);
                    const uint32_t m = ((1u << B) - 1u) << rp_pos(B, j);
                    const uint32_t mg = rp_magic_bits(B, j);
                    const uint32_t h2 = (t & (m | (m << 16))) | (mg | (mg << 16));
                    const uint16_t hv = half ? static_cast<uint16_t>(h2 >> 16) : static_cast<uint16_t>(h2 & 0xFFFF);
                    if (h2f(hv) - rp_magic(B, j) != static_cast<float>(codes[k])) ++bad;
                }
            }
        }
    std::printf("repack mismatches: %d\n", bad);
    return bad ? 1 : 0;
}
