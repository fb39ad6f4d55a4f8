// stream_bench.cu -- microbenchmark: how fast can one SM-resident kernel stream
// a ~26 MB weight matrix (Llama-3.1-8B gate_proj at 3.25 bits) from HBM on B200,
// with (a) 1-D bulk copies (TMA) into an mbarrier ring vs (b) plain vector loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "../paper_2602_01027_b200/csrc/ptx.cuh"

using namespace sfmpk;

constexpr int kThreads = 288;

// (a) bulk-copy ring: one producer lane, 8 consumer warps that only release.
__global__ void __launch_bounds__(kThreads, 2) bulk_stream(const uint8_t* src, size_t total, int piece,
                                                           int pieces_per_stage, int stages, unsigned* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + stages;
    uint8_t* ring = smem + 1024;
    const size_t stage_bytes = static_cast<size_t>(piece) * pieces_per_stage;
    const size_t nstage_total = total / stage_bytes;
    const size_t per_cta = (nstage_total + gridDim.x - 1) / gridDim.x;
    const size_t b0 = blockIdx.x * per_cta, b1 = min(nstage_total, b0 + per_cta);
    const int n = static_cast<int>(b1 > b0 ? b1 - b0 : 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 8);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int s = 0, ph = 0;
            for (int i = 0; i < n; ++i) {
                if (i >= stages) mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(stage_bytes));
                const uint8_t* g = src + (b0 + i) * stage_bytes;
                for (int p = 0; p < pieces_per_stage; ++p)
                    bulk_g2s(ring + s * stage_bytes + p * piece, g + p * piece, piece, &full[s], pol);
                if (++s == stages) { s = 0; ph ^= 1; }
            }
        }
        return;
    }
    unsigned acc = 0;
    int s = 0, ph = 0;
    for (int i = 0; i < n; ++i) {
        mbar_wait(&full[s], ph);
        acc += *reinterpret_cast<const unsigned*>(ring + s * stage_bytes + (threadIdx.x * 4) % stage_bytes);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678u) *sink = acc;
}

// (b) vector loads, UNROLL x 16 B in flight per thread, grid-stride.
template <int UNROLL>
__global__ void __launch_bounds__(256) ldg_stream(const uint4* src, size_t n16, unsigned* sink) {
    unsigned acc = 0;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * UNROLL;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x * UNROLL + threadIdx.x; i < n16; i += stride) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const size_t j = i + static_cast<size_t>(u) * blockDim.x;
            if (j < n16) {
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(src + j));
            } else {
                v[u] = make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    const size_t total = 26u << 20;  // 26 MiB like gate_proj @3.25 b
    const int copies = 8;            // rotate buffers so every launch reads HBM (208 MiB > L2)
    std::vector<uint8_t*> bufs(copies);
    for (auto& b : bufs) {
        cudaMalloc(&b, total);
        cudaMemset(b, 1, total);
    }
    unsigned* sink;
    cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
    auto time_it = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch(bufs[w % copies]);
        cudaDeviceSynchronize();
        const int reps = 40;
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) launch(bufs[r % copies]);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / reps;
        printf("%-44s %8.2f us/launch  %7.1f GB/s  (%s)\n", name, us, total / us / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int piece : {256, 2048, 8192, 16384}) {
        for (int pps : {1, 4}) {
            const size_t stage = static_cast<size_t>(piece) * pps;
            const int stages = static_cast<int>(std::min<size_t>(16, (113 * 1024 - 1024) / stage));
            if (stages < 2) continue;
            char name[128];
            snprintf(name, sizeof name, "bulk piece=%d x%d stages=%d grid=%d", piece, pps, stages, 2 * sms);
            time_it(name, [&](uint8_t* b) {
                bulk_stream<<<2 * sms, kThreads, 1024 + stages * stage>>>(b, total, piece, pps, stages, sink);
            });
        }
    }
    for (int gm : {1, 2, 4, 8}) {
        char name[128];
        snprintf(name, sizeof name, "ldg x4 grid=%d*sms", gm);
        time_it(name, [&](uint8_t* b) {
            ldg_stream<4><<<gm * sms, 256>>>(reinterpret_cast<const uint4*>(b), total / 16, sink);
        });
        snprintf(name, sizeof name, "ldg x8 grid=%d*sms", gm);
        time_it(name, [&](uint8_t* b) {
            ldg_stream<8><<<gm * sms, 256>>>(reinterpret_cast<const uint4*>(b), total / 16, sink);
        });
    }
    return 0;
}
