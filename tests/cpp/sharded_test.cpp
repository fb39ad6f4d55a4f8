// C++ caller of the sharded entry (include/sfmp/cuda.hpp: sfmp::cuda::gemm_sharded)
// at world size 1 on one GPU: a library-created NCCL communicator, ONE
// all-gather per call, and the result bit-identical to sfmp_gemm.
// usage: sharded_test model.sfmp   (exit 0 on success)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <vector>

#include "sfmp_cuda.h"

#define CK(x)                                                                                    \
    do {                                                                                         \
        sfmp_status s_ = (x);                                                                    \
        if (s_) {                                                                                \
            std::printf("%s -> %s: %s\n", #x, sfmp_status_string(s_), sfmp_last_error());        \
            return 1;                                                                            \
        }                                                                                        \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ifstream f(argv[1], std::ios::binary);
    const std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), {});
    sfmp_dev_model *full = nullptr, *shard = nullptr;
    CK(sfmp_model_create(bytes.data(), bytes.size(), 0, &full));
    CK(sfmp_model_create_shard(bytes.data(), bytes.size(), 0, 0, 1, &shard));
    sfmp_model_info info;
    CK(sfmp_model_get_info(full, &info));
    const int64_t Ms[2] = {1, 16};
    const size_t rows = info.rows, cols = info.cols;
    std::vector<float> xh(16 * cols);
    for (size_t i = 0; i < xh.size(); ++i) xh[i] = static_cast<float>((i * 2654435761u) % 1000) / 500.f - 1.f;
    float *x = nullptr, *y_ref = nullptr, *y = nullptr;
    cudaMalloc(&x, xh.size() * 4);
    cudaMalloc(&y_ref, 17 * rows * 4);
    cudaMalloc(&y, 17 * rows * 4);
    cudaMemcpy(x, xh.data(), xh.size() * 4, cudaMemcpyHostToDevice);
    size_t wsb = 0;
    CK(sfmp_workspace_size(shard, 16, SFMP_PATH_GEMV, &wsb));
    void *ws0 = nullptr, *ws1 = nullptr, *wsr = nullptr;
    cudaMalloc(&ws0, wsb);
    cudaMalloc(&ws1, wsb);
    cudaMalloc(&wsr, wsb);
    cudaMemset(ws0, 0, wsb);
    cudaMemset(ws1, 0, wsb);
    cudaMemset(wsr, 0, wsb);
    // reference: the unsharded model, one call per problem
    CK(sfmp_gemm(full, x, SFMP_F32, 1, y_ref, wsr, wsb, nullptr));
    CK(sfmp_gemm(full, x, SFMP_F32, 16, y_ref + rows, wsr, wsb, nullptr));
    // sharded: both problems, one all-gather
    uint8_t id[SFMP_NCCL_ID_BYTES];
    CK(sfmp_nccl_unique_id(id));
    void* comm = nullptr;
    CK(sfmp_nccl_comm_init(1, id, 0, 0, &comm));
    const sfmp_dev_model* ms[2] = {shard, shard};
    size_t gb = 0;
    CK(sfmp_sharded_gather_bytes(ms, Ms, 2, &gb));
    void* gather = nullptr;
    cudaMalloc(&gather, gb);
    const void* xs[2] = {x, x};
    float* ys[2] = {y, y + rows};
    void* wss[2] = {ws0, ws1};
    CK(sfmp_gemm_sharded(ms, xs, SFMP_F32, Ms, ys, wss, nullptr, 2, gather, gb, comm, nullptr));
    cudaDeviceSynchronize();
    std::vector<float> a(17 * rows), b(17 * rows);
    cudaMemcpy(a.data(), y_ref, a.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), y, b.size() * 4, cudaMemcpyDeviceToHost);
    const bool same = std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
    // a communicator whose size does not match the shard count is refused
    sfmp_dev_model* half = nullptr;
    CK(sfmp_model_create_shard(bytes.data(), bytes.size(), 0, 0, 2, &half));
    const sfmp_dev_model* hm[1] = {half};
    const sfmp_status bad = sfmp_gemm_sharded(hm, xs, SFMP_F32, Ms, ys, wss, nullptr, 1, gather, gb, comm, nullptr);
    CK(sfmp_nccl_comm_destroy(comm));
    std::printf("sharded_vs_unsharded_bit_equal=%d mismatched_comm=%s\n", same, sfmp_status_string(bad));
    return (same && bad == SFMP_ERR_CONFIG) ? 0 : 1;
}
