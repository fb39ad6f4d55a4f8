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

// y = W x for host vectors (the reference signature).  GemvStats::lookups has
// no GPU meaning and stays 0; the timing fields are left untouched.
inline Vector gemv(const DeviceModel& model, const Vector& x, GemvStats* stats = nullptr) {
    (void)stats;
    if (x.data.size() != model.info().cols) throw ShapeError("gemv: x.len != model cols");
    std::vector<float> y(model.info().out_rows);
    check(sfmp_gemm_host(model.handle(), x.data.data(), 1, y.data(), nullptr));
    return Vector(std::move(y));
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

}  // namespace cuda
}  // namespace sfmp
