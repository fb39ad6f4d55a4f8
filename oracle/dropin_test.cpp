// TEST INFRASTRUCTURE ONLY -- proves the C++ drop-in: the reference's own
// types and functions (compiled unmodified from /root/reference/proj/src) on
// one side, sfmp::cuda::gemv (include/sfmp/cuda.hpp -> libsfmp_b200.so) on
// the other.  usage: dropin_test model.sfmp x.f32 [M]
// exit 0 iff max|d|/max|y_ref| <= 1e-3 for every token and the shim maps a
// corrupted stream to sfmp::FormatError{bad_magic}.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <vector>

#include "sfmp/errors.hpp"
#include "sfmp/layout.hpp"
#include "sfmp/lutgemm.hpp"
#include "sfmp/cuda.hpp"

static std::vector<uint8_t> slurp(const char* path) {
    std::ifstream f(path, std::ios::binary);
    return std::vector<uint8_t>(std::istreambuf_iterator<char>(f), {});
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::vector<uint8_t> bytes = slurp(argv[1]);
    const std::vector<uint8_t> xb = slurp(argv[2]);
    const int M = argc > 3 ? std::atoi(argv[3]) : 1;
    const sfmp::PackedModel pm = sfmp::deserialize(bytes);          // reference ingest
    const sfmp::cuda::DeviceModel dm(pm);                             // shim: PackedModel -> device
    const size_t n = pm.cols;
    double worst = 0.0;
    for (int t = 0; t < M; ++t) {
        std::vector<float> xv(n);
        std::memcpy(xv.data(), xb.data() + t * n * 4, n * 4);
        const sfmp::Vector x(xv);
        const sfmp::Vector y_ref = sfmp::gemv(pm, x);                  // reference LUT path
        const sfmp::Vector y_gpu = sfmp::cuda::gemv(dm, x);            // B200 path
        double dmax = 0.0, ymax = 0.0;
        for (size_t i = 0; i < y_ref.data.size(); ++i) {
            dmax = std::fmax(dmax, std::fabs(double(y_gpu.data[i]) - y_ref.data[i]));
            ymax = std::fmax(ymax, std::fabs(double(y_ref.data[i])));
        }
        worst = std::fmax(worst, dmax / ymax);
    }
    // the exact-signature drop-in (uploads per call)
    {
        std::vector<float> xv(n);
        std::memcpy(xv.data(), xb.data(), n * 4);
        const sfmp::Vector y1 = sfmp::cuda::gemv(pm, sfmp::Vector(xv), nullptr);
        if (y1.data.size() != pm.rows) return 3;
    }
    // GemvStats filled from the GPU call (lutgemm.hpp:47-52); bench_gemv's ConfigError (lutgemm.cpp:138)
    bool ok_stats = false, ok_cfg = false;
    {
        std::vector<float> xv(n);
        std::memcpy(xv.data(), xb.data(), n * 4);
        sfmp::GemvStats st;
        (void)sfmp::cuda::gemv(dm, sfmp::Vector(xv), &st);
        ok_stats = st.accumulate_us > 0.0 && st.lookups == 0;
        const sfmp::BenchResult br = sfmp::cuda::bench_gemv(dm, sfmp::Vector(xv), 5);
        ok_stats = ok_stats && br.median_us > 0.0 && br.p10_us <= br.median_us && br.median_us <= br.p90_us &&
                   br.rows == pm.rows;
        try {
            (void)sfmp::cuda::bench_gemv(dm, sfmp::Vector(xv), 0);
        } catch (const sfmp::ConfigError&) {
            ok_cfg = true;
        }
    }
    bool ok_err = false;
    try {
        std::vector<uint8_t> bad = bytes;
        bad[0] ^= 0xFF;
        sfmp::cuda::DeviceModel broken(bad);
    } catch (const sfmp::FormatError& e) {
        ok_err = e.kind() == sfmp::FormatErrorKind::bad_magic;
    }
    bool ok_shape = false;
    try {
        sfmp::cuda::gemv(dm, sfmp::Vector(std::vector<float>(n + 1)));
    } catch (const sfmp::ShapeError&) {
        ok_shape = true;
    }
    std::printf("dropin max_rel=%.3e format_error=%d shape_error=%d stats=%d config_error=%d\n", worst, ok_err,
                ok_shape, ok_stats, ok_cfg);
    return (worst <= 1e-3 && ok_err && ok_shape && ok_stats && ok_cfg) ? 0 : 1;
}
