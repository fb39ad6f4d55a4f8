// lut.cu -- K6: the paper-faithful LUT GEMV on the GPU, a COMPARISON line
// (PAPER.md:475-479): the reference's own algorithm
// (lutgemm.cpp:11-71) on the SFMPPKD1 block payload as stored (bit planes),
// not the product path (K1 contracts exact codes on the tensor cores).
//
//  * build_luts (lutgemm.cpp:11-36): per 8-activation group of the reordered
//    x a mirror-compressed table of 128 signed sums (sign bit 7 fixed +1),
//    entry j = ((+-x0 +- x1) ... +- x6) + x7 summed in ascending k -- the
//    same float operations as the reference's recursive doubling, so every
//    entry is bit-identical to the reference's table.
//  * lookup (lutgemm.hpp:16-27): the other half by an exact sign flip.
//  * accumulate_block (lutgemm.cpp:45-71): per row and bit plane the 16
//    lookups of a 128-column block column, planes combined as sum 2^i s_i,
//    then the mirror affine s^ = s/2, z^ = z + s^(2^b - 1) plus z^ X_g.
// B200 mapping: one CTA per (block row, chunk of block columns, token), one
// thread per row of the block row (m_b threads), so a table built in shared
// memory (16 groups x 128 entries per 128 columns) serves m_b rows; chunk
// partial sums are added to y with atomics (a comparison line: summation
// order is not canonical here).
#include <cuda_fp16.h>

#include "sfmp_internal.h"

namespace sfmpk {
namespace {

constexpr int kLutChunk = 4;  // block columns per CTA

__global__ void __launch_bounds__(1024) lut_gemv_kernel(const uint8_t* __restrict__ payload,
                                                        const uint64_t* __restrict__ boff,
                                                        const uint8_t* __restrict__ bits,
                                                        const uint32_t* __restrict__ col_perm,
                                                        const uint32_t* __restrict__ out_map,
                                                        const float* __restrict__ x, float* __restrict__ y, int m_b,
                                                        int n_b, int BC, int cols, int out_rows) {
    __shared__ float lut[16][128];  // the tables of one 128-column pass
    __shared__ float xr[128];
    __shared__ float xsum;
    const int t = blockIdx.z, br = blockIdx.x, row = threadIdx.x;
    const int bc0 = blockIdx.y * kLutChunk, bc1 = min(BC, bc0 + kLutChunk);
    const float* xt = x + static_cast<size_t>(t) * cols;
    const int row_bytes = n_b / 8;
    float acc = 0.f;
    for (int bc = bc0; bc < bc1; ++bc) {
        const uint64_t k = static_cast<uint64_t>(br) * BC + bc;
        const uint8_t* blk = payload + boff[k];
        const int b = bits[k];
        float planes_acc = 0.f, bsum = 0.f;
        for (int c0 = 0; c0 < n_b; c0 += 128) {
            __syncthreads();  // the previous pass's tables are no longer read
            for (int i = threadIdx.x; i < 128; i += blockDim.x)  // m_b may be < 128 threads
                xr[i] = __ldg(xt + __ldg(col_perm + static_cast<size_t>(bc) * n_b + c0 + i));
            __syncthreads();
            if (threadIdx.x == 0) {  // range_sum (lutgemm.cpp:73-77), ascending
                float s = 0.f;
                for (int i = 0; i < 128; ++i) s += xr[i];
                xsum = s;
            }
            for (int e = threadIdx.x; e < 16 * 128; e += blockDim.x) {  // build_luts
                const int g = e >> 7, j = e & 127;
                const float* xs = &xr[8 * g];
                float v = (j & 1) ? xs[0] : -xs[0];
#pragma unroll
                for (int kk = 1; kk < 7; ++kk) v = ((j >> kk) & 1) ? v + xs[kk] : v - xs[kk];
                lut[g][j] = v + xs[7];
            }
            __syncthreads();
            bsum += xsum;
            const uint8_t* planes = blk + 4ull * m_b + static_cast<size_t>(row) * row_bytes + c0 / 8;
            for (int i = 0; i < b; ++i) {  // accumulate_block: 16 lookups per plane row
                const uint4 w = *reinterpret_cast<const uint4*>(planes + static_cast<size_t>(i) * m_b * row_bytes);
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
                float s = 0.f;
#pragma unroll
                for (int g = 0; g < 16; ++g) {
                    const uint32_t p = (ww[g >> 2] >> (8 * (g & 3))) & 0xFFu;
                    const uint32_t neg = (p >> 7) ^ 1u;
                    const uint32_t idx = (p ^ (0x7Fu * neg)) & 0x7Fu;
                    s += __uint_as_float(__float_as_uint(lut[g][idx]) ^ (neg << 31));
                }
                planes_acc += static_cast<float>(1 << i) * s;
            }
        }
        const float sh = 0.5f * __half2float(*reinterpret_cast<const __half*>(blk + 2 * row));
        const float zh = __half2float(*reinterpret_cast<const __half*>(blk + 2 * m_b + 2 * row)) +
                         sh * static_cast<float>((1 << b) - 1);
        acc += sh * planes_acc + zh * bsum;
    }
    atomicAdd(y + static_cast<size_t>(t) * out_rows + out_map[static_cast<size_t>(br) * m_b + row], acc);
}

}  // namespace

bool lut_supported(const DevModel& m) {
    return m.d_lut != nullptr && m.m_b % 32 == 0 && m.m_b <= 1024 && m.n_b % 128 == 0 && m.num_shards == 1;
}

cudaError_t launch_lut(const DevModel& m, const float* x, int64_t M, float* y, cudaStream_t st) {
    if (M > 65535) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(y, 0, static_cast<size_t>(M) * m.out_rows * 4, st);
    if (e != cudaSuccess) return e;
    const dim3 grid(static_cast<unsigned>(m.rows / m.m_b), static_cast<unsigned>((m.BC + kLutChunk - 1) / kLutChunk),
                    static_cast<unsigned>(M));
    note_launch();
    lut_gemv_kernel<<<grid, m.m_b, 0, st>>>(m.d_lut, m.d_lut_off, m.d_lut_bits, m.d_col_perm, m.d_out_map, x, y,
                                            static_cast<int>(m.m_b), static_cast<int>(m.n_b), static_cast<int>(m.BC),
                                            static_cast<int>(m.cols), static_cast<int>(m.out_rows));
    return cudaGetLastError();
}

}  // namespace sfmpk
