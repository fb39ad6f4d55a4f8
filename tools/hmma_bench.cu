// hmma_bench.cu -- legacy mma.sync.m16n8k16 (f16 x f16 -> f32) throughput on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hmma_bench tools/hmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k(int iters, float* out) {
    float acc[CH][4] = {};
    unsigned a0 = threadIdx.x * 0x00010001u, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 7, a3 = a1 + 3;
    unsigned b0 = 0x3c003c00u ^ threadIdx.x, b1 = b0 + 1;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (s == 1234.5f) out[0] = s;
}

int main() {
    float* d;
    cudaMalloc(&d, 4);
    const int iters = 20000;
    for (int ch : {1, 2, 4, 8})
    for (int warps : {4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (ch == 1) k<1><<<148, 32 * warps>>>(iters, d);
            if (ch == 2) k<2><<<148, 32 * warps>>>(iters, d);
            if (ch == 4) k<4><<<148, 32 * warps>>>(iters, d);
            if (ch == 8) k<8><<<148, 32 * warps>>>(iters, d);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double mmas = 148.0 * warps * iters * ch;
            if (rep)
                printf("chains %d warps/SM %2d: %.1f TFLOP/s, %.2f ns per MMA per SM-subcore (%s)\n", ch, warps,
                       mmas * 4096 / (ms * 1e-3) / 1e12, ms * 1e6 / (mmas / 148 / 4), cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
