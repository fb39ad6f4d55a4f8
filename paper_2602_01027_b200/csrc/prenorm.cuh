// prenorm.cuh -- RMSNorm fused into the activation pre-passes (SURVEY §8(f)1,
// "fused activation producer"): the caller passes the UNNORMALISED hidden
// state h and the norm weight gamma; the pre-pass that already stages each
// token row (gather by col_perm, reorder.cpp:103-111, scale, convert) applies
//     x[t][j] = h[t][j] / sqrt(mean_j h[t][j]^2 + eps) * gamma[j]      (f32)
// on the fly, so the separate norm kernel's read and write of x disappear.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "sfmp_internal.h"

namespace sfmpk {

__device__ __forceinline__ float gamma_at(const PreNorm& n, uint32_t j) {
    if (!n.gamma) return 1.f;
    if (n.gdt == SFMP_F32) return __ldg(static_cast<const float*>(n.gamma) + j);
    if (n.gdt == SFMP_F16) return __half2float(__ldg(static_cast<const __half*>(n.gamma) + j));
    return __bfloat162float(__ldg(static_cast<const __nv_bfloat16*>(n.gamma) + j));
}

// Block-wide sum / max over all threads (red: >= 32 floats of shared memory).
template <bool MAX>
__device__ __forceinline__ float block_reduce(float v, float* red) {
    const int NW = static_cast<int>(blockDim.x >> 5);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float u = __shfl_xor_sync(0xffffffffu, v, o);
        v = MAX ? fmaxf(v, u) : v + u;
    }
    __syncthreads();  // red[] free (previous use finished)
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = MAX ? 0.f : 0.f;
    for (int w = 0; w < NW; ++w) v = MAX ? fmaxf(v, red[w]) : v + red[w];
    return v;
}

// 1/rms of one token row (values given by f(i), i < cols).
template <class F>
__device__ __forceinline__ float row_inv_rms(F f, int cols, float eps, float* red) {
    float ss = 0.f;
    for (int i = threadIdx.x; i < cols; i += blockDim.x) {
        const float v = f(i);
        ss = fmaf(v, v, ss);
    }
    ss = block_reduce<false>(ss, red);
    return 1.f / sqrtf(ss / static_cast<float>(cols) + eps);
}

}  // namespace sfmpk
