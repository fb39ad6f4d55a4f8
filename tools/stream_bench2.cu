// stream_bench2.cu -- the K1 unit copy pattern (128-row slices of 512x128 3-bit blocks:
// s 256 B, z 256 B, 3 planes x 2 KB) through a bulk-copy ring: vary stages, units per
// stage, CTAs per SM, and whether the two 256 B meta copies are issued.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_2602_01027_b200/csrc/ptx.cuh"
using namespace sfmpk;

template <int CPS>
__global__ void __launch_bounds__(288, CPS) unit_stream(const uint8_t* payload, int nunits, int ups, int stages,
                                                         int meta, unsigned* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + stages;
    uint8_t* ring = smem + 1024;
    const int ubytes = 512 + 3 * 2048;
    const int sbytes = ups * ubytes;
    const int per = (nunits + gridDim.x - 1) / gridDim.x;
    const int u0 = blockIdx.x * per, u1 = min(nunits, u0 + per);
    const int nst = (u1 - u0 + ups - 1) / ups;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
        fence_mbar_init();
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int s = 0, ph = 0;
            for (int i = 0; i < nst; ++i) {
                if (i >= stages) mbar_wait(&empty[s], ph ^ 1);
                int bytes = 0;
                for (int k = 0; k < ups; ++k) if (u0 + i * ups + k < u1) bytes += meta ? ubytes : 3 * 2048;
                mbar_arrive_expect_tx(&full[s], bytes);
                for (int k = 0; k < ups; ++k) {
                    const int u = u0 + i * ups + k;
                    if (u >= u1) break;
                    const int blk = u / 4, ro = (u % 4) * 128;
                    const uint8_t* b = payload + static_cast<size_t>(blk) * (2048 + 3 * 8192);
                    uint8_t* d = ring + s * sbytes + k * ubytes;
                    if (meta) {
                        bulk_g2s(d, b + 2 * ro, 256, &full[s], pol);
                        bulk_g2s(d + 256, b + 1024 + 2 * ro, 256, &full[s], pol);
                    }
                    for (int pl = 0; pl < 3; ++pl) bulk_g2s(d + 512 + pl * 2048, b + 2048 + pl * 8192 + ro * 16, 2048, &full[s], pol);
                }
                if (++s == stages) { s = 0; ph ^= 1; }
            }
        }
        return;
    }
    unsigned acc = 0;
    int s = 0, ph = 0;
    for (int i = 0; i < nst; ++i) {
        mbar_wait(&full[s], ph);
        acc += *reinterpret_cast<const unsigned*>(ring + s * sbytes + 512 + threadIdx.x * 4);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    const int nblocks = 896;  // 14336x4096 / (512x128)
    const size_t bytes = static_cast<size_t>(nblocks) * (2048 + 3 * 8192);
    const int nunits = nblocks * 4;
    const int copies = 8;
    std::vector<uint8_t*> bufs(copies);
    for (auto& b : bufs) { cudaMalloc(&b, bytes); cudaMemset(b, 1, bytes); }
    unsigned* sink; cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(unit_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    cudaFuncSetAttribute(unit_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
    auto run = [&](int cps, int ups, int stages, int meta, int grid_mult) {
        const int sb = ups * (512 + 3 * 2048);
        const size_t smem = 1024 + static_cast<size_t>(stages) * sb;
        const int grid = grid_mult * sms;
        auto launch = [&](uint8_t* b) {
            if (cps == 1) unit_stream<1><<<grid, 288, smem>>>(b, nunits, ups, stages, meta, sink);
            else unit_stream<2><<<grid, 288, smem>>>(b, nunits, ups, stages, meta, sink);
        };
        for (int w = 0; w < 3; ++w) launch(bufs[w]);
        cudaDeviceSynchronize();
        const int reps = 40;
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) launch(bufs[r % copies]);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / reps;
        printf("cps=%d ups=%d stages=%2d meta=%d grid=%d*sms smem=%6zu: %7.2f us %7.1f GB/s %s\n", cps, ups, stages, meta,
               grid_mult, smem, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    for (int meta : {1, 0}) {
        for (int st : {4, 8, 12}) run(2, 1, st, meta, 2);
        for (int st : {4, 6}) run(2, 2, st, meta, 2);
        run(2, 4, 3, meta, 2);
        for (int st : {8, 16, 24}) run(1, 1, st, meta, 1);
        for (int st : {6, 12}) run(1, 2, st, meta, 1);
        run(1, 4, 6, meta, 1);
        run(2, 1, 12, meta, 4);
    }
    return 0;
}
