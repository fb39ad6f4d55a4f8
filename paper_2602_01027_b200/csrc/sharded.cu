// sharded.cu -- multi-GPU decode/prefill over N-sharded linears (SURVEY §8e,
// DESIGN.md §6): each rank runs its block-row shard of every problem into ONE
// packed send buffer, ONE all-gather moves every problem's shard outputs,
// ONE kernel scatters the gathered rows to their original positions.
//
// The reference has no multi-GPU code; SPEC.md:553 allows row-range
// parallelism with a deterministic merge -- the merge here is a pure
// scatter (every output row is computed by exactly one shard), so the sharded
// result is bit-identical to the unsharded one.
//
// NCCL is loaded at first use with dlopen("libnccl.so.2") (in a PyTorch
// process that is the library torch already loaded), so the product library
// has no link-time NCCL dependency and a caller's own ncclComm_t can be used.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sfmp_cuda.h"
#include "sfmp_internal.h"

namespace sfmpk {
namespace {

constexpr int kMaxProb = 64;
struct UnpermParams {
    const uint32_t* inv[kMaxProb];  // [rows] original row -> g * SR + local position
    float* y[kMaxProb];             // [M][rows] original order
    uint64_t off[kMaxProb];         // first float of each problem in one shard's packed block
    int poff[kMaxProb + 1];         // first (problem, token) pair of each problem (+ total)
    uint32_t SR[kMaxProb];
    uint32_t rows[kMaxProb];
    uint64_t total;                 // floats of one shard's packed block
    int n;
};

// y_i[t][r] = recv[g][off_i + t*SR_i + k] with g << 24 | k = inv_i[r] for
// every problem i.  CTA = (1024-row chunk, (problem, token) pair); the pair
// is found once per CTA.  Coalesced 16-byte writes; each shard's rows are in
// ascending original order, so the reads follow G sequential streams.
__global__ void __launch_bounds__(256) unpermute_grouped_kernel(const float* __restrict__ recv,
                                                                const UnpermParams p) {
    const int pair = static_cast<int>(blockIdx.y);
    int lo = 0, hi = p.n - 1;  // problem owning this (problem, token) pair
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.poff[mid] <= pair) lo = mid;
        else hi = mid - 1;
    }
    const uint64_t t = static_cast<uint64_t>(pair - p.poff[lo]);
    const uint32_t rows = p.rows[lo], SR = p.SR[lo];
    const uint64_t r0 = (static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x) * 4;
    if (r0 >= rows) return;
    const float* src = recv + p.off[lo] + t * SR;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        v[j] = 0.f;
        if (r0 + j < rows) {
            const uint32_t k = __ldg(p.inv[lo] + r0 + j);
            v[j] = __ldg(src + static_cast<uint64_t>(k >> 24) * p.total + (k & 0xFFFFFFu));
        }
    }
    float* yr = p.y[lo] + t * rows + r0;
    if (r0 + 4 <= rows && (reinterpret_cast<uintptr_t>(yr) & 15) == 0) {
        *reinterpret_cast<float4*>(yr) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
        for (int j = 0; j < 4 && r0 + j < rows; ++j) yr[j] = v[j];
    }
}

// ---- NCCL, loaded at run time -------------------------------------------------
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclCommUserRank) comm_user_rank = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("dlopen libnccl.so.2: ") + (e ? e : "not found");
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.comm_count = reinterpret_cast<decltype(api.comm_count)>(sym("ncclCommCount"));
        api.comm_user_rank = reinterpret_cast<decltype(api.comm_user_rank)>(sym("ncclCommUserRank"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count &&
                 api.comm_user_rank && api.all_gather && api.error_string;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

sfmp_status nccl_fail(const NcclApi& api, ncclResult_t r, const char* what) {
    return api_fail(SFMP_ERR_NCCL, std::string(what) + ": " + (api.error_string ? api.error_string(r) : "nccl error"));
}

// Shared validation of a sharded call: every problem a shard of the same
// partition on one device.
sfmp_status check_shards(const sfmp_dev_model* const* models, const int64_t* Ms, int count,
                         std::vector<const DevModel*>& ms) {
    if (count < 1 || !models || !Ms) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    if (count > kMaxProb) return api_fail(SFMP_ERR_CONFIG, "at most 64 problems per sharded call");
    ms.resize(count);
    for (int i = 0; i < count; ++i) {
        if (!models[i]) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null model");
        if (Ms[i] < 0) return api_fail(SFMP_ERR_SHAPE, "negative M");
        ms[i] = reinterpret_cast<const DevModel*>(models[i]);
        if (!ms[i]->d_gather_map) return api_fail(SFMP_ERR_CONFIG, "model is not a shard (sfmp_model_create_shard)");
        if (ms[i]->num_shards != ms[0]->num_shards || ms[i]->shard != ms[0]->shard || ms[i]->device != ms[0]->device)
            return api_fail(SFMP_ERR_CONFIG, "problems of one sharded call must be the same shard of one partition");
    }
    return SFMP_OK;
}

uint64_t packed_floats(const std::vector<const DevModel*>& ms, const int64_t* Ms, std::vector<uint64_t>* off) {
    uint64_t t = 0;
    if (off) off->assign(ms.size() + 1, 0);
    for (size_t i = 0; i < ms.size(); ++i) {
        if (off) (*off)[i] = t;
        t += static_cast<uint64_t>(Ms[i]) * ms[i]->shard_rows;
    }
    if (off) (*off)[ms.size()] = t;
    return t;
}

}  // namespace
}  // namespace sfmpk

using sfmpk::api_fail;
using sfmpk::DevModel;

extern "C" {

sfmp_status sfmp_sharded_gather_bytes(const sfmp_dev_model* const* models, const int64_t* Ms, int count,
                                      size_t* bytes) {
    if (!bytes) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null bytes");
    std::vector<const DevModel*> ms;
    sfmp_status s = sfmpk::check_shards(models, Ms, count, ms);
    if (s) return s;
    const uint64_t t = sfmpk::packed_floats(ms, Ms, nullptr);
    *bytes = static_cast<size_t>((1 + ms[0]->num_shards) * t * 4);
    return SFMP_OK;
}

sfmp_status sfmp_gemm_sharded_local(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                                    const int64_t* Ms, void* const* workspaces, const size_t* workspace_bytes,
                                    int count, void* gather_buf, void* stream) {
    std::vector<const DevModel*> ms;
    sfmp_status s = sfmpk::check_shards(models, Ms, count, ms);
    if (s) return s;
    if (!gather_buf || !xs || !workspaces) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    std::vector<uint64_t> off;
    sfmpk::packed_floats(ms, Ms, &off);
    std::vector<float*> ys(count);
    for (int i = 0; i < count; ++i) ys[i] = static_cast<float*>(gather_buf) + off[i];
    // y_local[M][shard_rows] of problem i at its offset of the send block
    return sfmp_gemm_grouped_v(models, xs, dtype, Ms, ys.data(), workspaces, workspace_bytes, count, stream);
}

sfmp_status sfmp_sharded_unpermute(const sfmp_dev_model* const* models, const int64_t* Ms, int count,
                                   const void* gather_buf, float* const* ys, void* stream) {
    std::vector<const DevModel*> ms;
    sfmp_status s = sfmpk::check_shards(models, Ms, count, ms);
    if (s) return s;
    if (!gather_buf || !ys) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    sfmpk::UnpermParams p{};
    std::vector<uint64_t> off;
    const uint64_t total = sfmpk::packed_floats(ms, Ms, &off);
    if (total == 0) return SFMP_OK;
    p.n = count;
    p.total = total;
    uint64_t d = 0, maxrows = 0;
    for (int i = 0; i < count; ++i) {
        if (Ms[i] && !ys[i]) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null y");
        p.inv[i] = ms[i]->d_gather_inv;
        p.y[i] = ys[i];
        p.off[i] = off[i];
        p.poff[i] = static_cast<int>(d);
        p.SR[i] = static_cast<uint32_t>(ms[i]->shard_rows);
        p.rows[i] = static_cast<uint32_t>(ms[i]->global_rows);
        d += static_cast<uint64_t>(Ms[i]);
        maxrows = std::max<uint64_t>(maxrows, ms[i]->global_rows);
    }
    p.poff[count] = static_cast<int>(d);
    if (d > 65535) return api_fail(SFMP_ERR_CONFIG, "sharded call: at most 65535 (problem, token) pairs");
    sfmpk::DeviceGuard guard(ms[0]->device);
    const float* recv = static_cast<const float*>(gather_buf) + total;  // [G][total] after the send block
    const dim3 grid(static_cast<unsigned>((maxrows + 1023) / 1024), static_cast<unsigned>(d));
    sfmpk::note_launch();
    sfmpk::unpermute_grouped_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(recv, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return api_fail(SFMP_ERR_CUDA, std::string("unpermute launch: ") + cudaGetErrorString(e));
    return SFMP_OK;
}

sfmp_status sfmp_gemm_sharded(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                              const int64_t* Ms, float* const* ys, void* const* workspaces,
                              const size_t* workspace_bytes, int count, void* gather_buf, size_t gather_bytes,
                              void* nccl_comm, void* stream) {
    std::vector<const DevModel*> ms;
    sfmp_status s = sfmpk::check_shards(models, Ms, count, ms);
    if (s) return s;
    if (!nccl_comm) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null communicator");
    const sfmpk::NcclApi& api = sfmpk::nccl_api();
    if (!api.ok) return api_fail(SFMP_ERR_NCCL, api.why);
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    int n = 0, r = 0;
    ncclResult_t nr = api.comm_count(comm, &n);
    if (nr != ncclSuccess) return sfmpk::nccl_fail(api, nr, "ncclCommCount");
    if ((nr = api.comm_user_rank(comm, &r)) != ncclSuccess) return sfmpk::nccl_fail(api, nr, "ncclCommUserRank");
    if (static_cast<uint32_t>(n) != ms[0]->num_shards || static_cast<uint32_t>(r) != ms[0]->shard)
        return api_fail(SFMP_ERR_CONFIG, "communicator size/rank must equal the shard count/index");
    const uint64_t total = sfmpk::packed_floats(ms, Ms, nullptr);
    if (!gather_buf || gather_bytes < (1 + static_cast<uint64_t>(n)) * total * 4)
        return api_fail(SFMP_ERR_CONFIG, "gather buffer too small (sfmp_sharded_gather_bytes)");
    if ((s = sfmp_gemm_sharded_local(models, xs, dtype, Ms, workspaces, workspace_bytes, count, gather_buf, stream)))
        return s;
    if (total) {
        sfmpk::DeviceGuard guard(ms[0]->device);
        float* send = static_cast<float*>(gather_buf);
        nr = api.all_gather(send, send + total, total, ncclFloat32, comm, static_cast<cudaStream_t>(stream));
        if (nr != ncclSuccess) return sfmpk::nccl_fail(api, nr, "ncclAllGather");
    }
    return sfmp_sharded_unpermute(models, Ms, count, gather_buf, ys, stream);
}

sfmp_status sfmp_nccl_unique_id(uint8_t* id) {
    if (!id) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null id");
    const sfmpk::NcclApi& api = sfmpk::nccl_api();
    if (!api.ok) return api_fail(SFMP_ERR_NCCL, api.why);
    ncclUniqueId u;
    const ncclResult_t r = api.get_unique_id(&u);
    if (r != ncclSuccess) return sfmpk::nccl_fail(api, r, "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == SFMP_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, u.internal, sizeof(u.internal));
    return SFMP_OK;
}

sfmp_status sfmp_nccl_comm_init(int nranks, const uint8_t* id, int rank, int device, void** comm) {
    if (!id || !comm) return api_fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return api_fail(SFMP_ERR_CONFIG, "bad rank / size");
    const sfmpk::NcclApi& api = sfmpk::nccl_api();
    if (!api.ok) return api_fail(SFMP_ERR_NCCL, api.why);
    sfmpk::DeviceGuard guard(device);
    ncclUniqueId u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    ncclComm_t c = nullptr;
    const ncclResult_t r = api.comm_init_rank(&c, nranks, u, rank);
    if (r != ncclSuccess) return sfmpk::nccl_fail(api, r, "ncclCommInitRank");
    *comm = c;
    return SFMP_OK;
}

sfmp_status sfmp_nccl_comm_destroy(void* comm) {
    if (!comm) return SFMP_OK;
    const sfmpk::NcclApi& api = sfmpk::nccl_api();
    if (!api.ok) return api_fail(SFMP_ERR_NCCL, api.why);
    const ncclResult_t r = api.comm_destroy(static_cast<ncclComm_t>(comm));
    if (r != ncclSuccess) return sfmpk::nccl_fail(api, r, "ncclCommDestroy");
    return SFMP_OK;
}

}  // extern "C"
