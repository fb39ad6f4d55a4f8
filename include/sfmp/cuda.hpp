// sfmp/cuda.hpp -- header-only C++ shim over the C ABI (include/sfmp_cuda.h)
// that restores the reference's calling convention and exception types.
//
// Drop-in for the reference hot path (paths relative to /root/reference/proj):
//   sfmp::gemv(const PackedModel&, const Vector&, GemvStats*)   lutgemm.hpp:57
// with the same errors: ShapeError (lutgemm.cpp:96), ConfigError,
// FormatError{bad_magic, bad_version, truncated, invariant, io} (errors.hpp:9-36).
//
// Include AFTER the reference headers ("sfmp/layout.hpp", "sfmp/lutgemm.hpp",
// "sfmp/errors.hpp") so PackedModel / Vector / GemvStats / the exception types
// are the reference's own; link libsfmp_b200.so.  See INTEGRATION.md.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../sfmp_cuda.h"

namespace sfmp {
namespace cuda {

// Map a C-ABI status to the reference exception it stands for.
inline void check(sfmp_status s) {
    if (s == SFMP_OK) return;
    const std::string msg = sfmp_last_error();
    switch (s) {
        case SFMP_ERR_SHAPE: throw ShapeError(msg);
        case SFMP_ERR_CONFIG: throw ConfigError(msg);
        case SFMP_ERR_FORMAT_BAD_MAGIC: throw FormatError(FormatErrorKind::bad_magic, msg);
        case SFMP_ERR_FORMAT_BAD_VERSION: throw FormatError(FormatErrorKind::bad_version, msg);
        case SFMP_ERR_FORMAT_TRUNCATED: throw FormatError(FormatErrorKind::truncated, msg);
        case SFMP_ERR_FORMAT_INVARIANT: throw FormatError(FormatErrorKind::invariant, msg);
        case SFMP_ERR_FORMAT_IO: throw FormatError(FormatErrorKind::io, msg);
        default: throw std::runtime_error(std::string("sfmp_cuda: ") + sfmp_status_string(s) + ": " + msg);
    }
}

// A PackedModel resident on one B200 (uploaded once, reused across calls --
// the reference re-reads the PackedModel on every gemv, lutgemm.cpp:95).
class DeviceModel {
public:
    // From SFMPPKD1 bytes (serialize(), layout.cpp:179-208).
    DeviceModel(const std::vector<uint8_t>& bytes, int device = 0) {
        sfmp_dev_model* m = nullptr;
        check(sfmp_model_create(bytes.data(), bytes.size(), device, &m));
        h_.reset(m);
        check(sfmp_model_get_info(m, &info_));
    }
    // From an in-memory PackedModel (layout.hpp:36-53).
    explicit DeviceModel(const PackedModel& pm, int device = 0) {
        std::vector<const uint16_t*> sc, ze;
        std::vector<const uint8_t*> planes;
        for (const PackedBlock& b : pm.blocks) {
            sc.push_back(b.scales.data());
            ze.push_back(b.zeros.data());
            for (const auto& pl : b.planes) planes.push_back(pl.data());
        }
        sfmp_model_parts parts{};
        parts.rows = pm.rows;
        parts.cols = pm.cols;
        parts.m_b = static_cast<uint32_t>(pm.block_rows);
        parts.n_b = static_cast<uint32_t>(pm.group_size);
        parts.floor_bits = pm.floor_bits;
        parts.ceil_bits = pm.ceil_bits;
        parts.mode = static_cast<int32_t>(pm.reorder.mode);
        parts.row_perm = pm.reorder.row_perm.forward.empty() ? nullptr : pm.reorder.row_perm.forward.data();
        parts.col_perm = pm.reorder.col_perm.forward.empty() ? nullptr : pm.reorder.col_perm.forward.data();
        parts.block_bits = pm.block_bits.data();
        parts.scales = sc.data();
        parts.zeros = ze.data();
        parts.plane_ptrs = planes.data();
        sfmp_dev_model* m = nullptr;
        check(sfmp_model_create_from_parts(&parts, device, &m));
        h_.reset(m);
        check(sfmp_model_get_info(m, &info_));
    }
    const sfmp_dev_model* handle() const { return h_.get(); }
    const sfmp_model_info& info() const { return info_; }

private:
    struct Del {
        void operator()(sfmp_dev_model* m) const { sfmp_model_destroy(m); }
    };
    std::unique_ptr<sfmp_dev_model, Del> h_;
    sfmp_model_info info_{};
};

// y = W x for host vectors (the reference signature).  GemvStats
// (lutgemm.hpp:47-52) is filled from the GPU call's own measurements:
// accumulate_us = device time of the kernels (gather, contraction and
// scatter are fused into them, so reorder_us = 0); there are no lookup tables
// (the tensor cores contract the exact codes), so lookups = 0 and
// lut_build_us = 0.
inline Vector gemv(const DeviceModel& model, const Vector& x, GemvStats* stats = nullptr) {
    if (x.data.size() != model.info().cols) throw ShapeError("gemv: x.len != model cols");
    std::vector<float> y(model.info().out_rows);
    sfmp_stats st{};
    check(sfmp_gemm_host_stats(model.handle(), x.data.data(), 1, y.data(), nullptr, stats ? &st : nullptr));
    if (stats) {
        stats->lookups = 0;
        stats->lut_build_us = 0.0;
        stats->accumulate_us = st.device_us;
        stats->reorder_us = 0.0;
    }
    return Vector(std::move(y));
}

// The full GPU statistics of one call (device / copy / wall time, bytes, path, launches).
inline Vector gemv_ex(const DeviceModel& model, const Vector& x, sfmp_stats* stats) {
    if (x.data.size() != model.info().cols) throw ShapeError("gemv: x.len != model cols");
    std::vector<float> y(model.info().out_rows);
    check(sfmp_gemm_host_stats(model.handle(), x.data.data(), 1, y.data(), nullptr, stats));
    return Vector(std::move(y));
}

// bench_gemv (lutgemm.cpp:137-179) over the GPU drop-in: the same
// repetitions, percentiles (index llround(q*(n-1)) of the sorted host
// wall times) and ConfigError for reps < 1.
inline BenchResult bench_gemv(const DeviceModel& model, const Vector& x, size_t reps) {
    if (reps < 1) throw ConfigError("bench_gemv: repetitions must be >= 1");
    std::vector<double> totals;
    totals.reserve(reps);
    for (size_t r = 0; r < reps; ++r) {
        sfmp_stats st{};
        (void)gemv_ex(model, x, &st);
        totals.push_back(st.wall_us);
    }
    std::sort(totals.begin(), totals.end());
    auto pct = [&](double q) { return totals[static_cast<size_t>(std::llround(q * static_cast<double>(totals.size() - 1)))]; };
    BenchResult res;
    res.rows = model.info().out_rows;
    res.cols = model.info().cols;
    res.reps = reps;
    res.median_us = pct(0.5);
    res.p10_us = reps > 1 ? pct(0.10) : std::nan("");
    res.p90_us = reps > 1 ? pct(0.90) : std::nan("");
    res.lut_build_us = 0.0;
    res.reorder_us = 0.0;
    res.lookups = 0;
    return res;
}

// Exact drop-in for sfmp::gemv(const PackedModel&, ...): uploads per call.
// Prefer DeviceModel + gemv(DeviceModel) on a hot path.
inline Vector gemv(const PackedModel& model, const Vector& x, GemvStats* stats = nullptr) {
    return gemv(DeviceModel(model), x, stats);
}

// M tokens at once (the reference loops gemv per token):
// x_host [M][cols] -> y_host [M][rows], both row-major host arrays.
inline void gemm_host(const DeviceModel& model, const float* x_host, int64_t M, float* y_host) {
    check(sfmp_gemm_host(model.handle(), x_host, M, y_host, nullptr));
}

// Sharded decode/prefill of several linears with ONE NCCL all-gather
// (multi-GPU).  models: this rank's shards (DeviceModel built
// with sfmp_model_create_shard); xs/ys/workspaces: device pointers;
// gather_buf: sfmp_sharded_gather_bytes() bytes of device memory;
// comm: an ncclComm_t with size/rank = shard count/index.
inline void gemm_sharded(const std::vector<const sfmp_dev_model*>& models, const std::vector<const void*>& xs,
                         sfmp_dtype dtype, const std::vector<int64_t>& Ms, const std::vector<float*>& ys,
                         const std::vector<void*>& workspaces, void* gather_buf, size_t gather_bytes, void* comm,
                         void* stream = nullptr) {
    const int n = static_cast<int>(models.size());
    if (xs.size() != models.size() || Ms.size() != models.size() || ys.size() != models.size() ||
        workspaces.size() != models.size())
        throw ShapeError("gemm_sharded: argument lists differ in length");
    check(sfmp_gemm_sharded(models.data(), xs.data(), dtype, Ms.data(), ys.data(), workspaces.data(), nullptr, n,
                            gather_buf, gather_bytes, comm, stream));
}

}  // namespace cuda
}  // namespace sfmp
