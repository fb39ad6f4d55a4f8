// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled
// from the sources where they lie (/root/reference/proj/src/*.cpp) by
// oracle/Makefile into oracle/_ref/libsfmpref.so.  Nothing here re-states an
// algorithm: every call forwards to the reference's own functions, so the
// golden fixtures in tests/golden/ and the `--impl reference` bench arm are
// the reference itself.  Built with -O2 -std=c++20 and no -march flags
// (SURVEY §8c caveat 2).
#include <sfmp/allocation.hpp>
#include <sfmp/errors.hpp>
#include <sfmp/fp16.hpp>
#include <sfmp/layout.hpp>
#include <sfmp/lutgemm.hpp>
#include <sfmp/matrix.hpp>
#include <sfmp/quantizer.hpp>
#include <sfmp/reorder.hpp>
#include <sfmp/salience.hpp>

#include <cstring>
#include <thread>
#include <vector>

using namespace sfmp;

namespace {

int code_of(const FormatError& e) {
    switch (e.kind()) {
        case FormatErrorKind::bad_magic: return 3;
        case FormatErrorKind::bad_version: return 4;
        case FormatErrorKind::truncated: return 5;
        case FormatErrorKind::invariant: return 6;
        case FormatErrorKind::io: return 7;
    }
    return 6;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError&) {
        return 1;
    } catch (const ConfigError&) {
        return 2;
    } catch (const FormatError& e) {
        return code_of(e);
    } catch (...) {
        return 99;
    }
}

}  // namespace

extern "C" {

uint16_t ref_fp16_from_float(float f) { return fp16_from_float(f); }
float ref_fp16_to_float(uint16_t h) { return fp16_to_float(h); }

int ref_quantize_group(const float* v, size_t n, int bits, float* scale, float* zero,
                       uint8_t* codes) {
    return guarded([&] {
        QuantGroup g = quantize_group(std::span<const float>(v, n), bits);
        *scale = g.scale;
        *zero = g.zero;
        std::memcpy(codes, g.codes.data(), n);
    });
}

// Composes the reference's offline path (pipeline.hpp's
// quantize_matrix is declared but not defined): make_reorder_spec ->
// apply_reorder -> block_salience -> make_bit_plan -> allocate_block_bits ->
// quantize_group -> pack_block -> serialize.
int ref_build_model(const float* W, const float* S, uint64_t rows, uint64_t cols, uint32_t m_b,
                    uint32_t n_b, double target_bpw, int mode, uint8_t* out, size_t* out_len) {
    return guarded([&] {
        Matrix w(rows, cols, std::vector<float>(W, W + rows * cols));
        Matrix s(rows, cols, std::vector<float>(S, S + rows * cols));
        ReorderSpec spec = make_reorder_spec(s, static_cast<ReorderMode>(mode));
        Matrix wr = apply_reorder(w, spec);
        Matrix sr = apply_reorder(s, spec);
        std::vector<BlockSalience> bs = block_salience(sr, m_b, n_b);
        BitPlan plan = make_bit_plan(target_bpw, n_b, m_b);
        BlockBitMap map = allocate_block_bits(plan, bs);

        PackedModel pm;
        pm.rows = rows;
        pm.cols = cols;
        pm.block_rows = m_b;
        pm.group_size = n_b;
        pm.floor_bits = plan.floor_bits;
        pm.ceil_bits = plan.ceil_bits;
        pm.reorder = spec;
        pm.block_bits = map.bits;
        const size_t gc = cols / n_b;
        for (size_t k = 0; k < map.bits.size(); ++k) {
            const size_t br = k / gc, bc = k % gc;
            std::vector<QuantGroup> groups;
            groups.reserve(m_b);
            for (size_t r = 0; r < m_b; ++r)
                groups.push_back(quantize_group(
                    std::span<const float>(wr.row(br * m_b + r) + bc * n_b, n_b), map.bits[k]));
            pm.blocks.push_back(pack_block(groups, n_b));
        }
        std::vector<uint8_t> bytes = serialize(pm);
        const size_t cap = *out_len;
        *out_len = bytes.size();
        if (out) {
            if (bytes.size() > cap) throw ShapeError("ref_build_model: buffer too small");
            std::memcpy(out, bytes.data(), bytes.size());
        }
    });
}

void* ref_load(const uint8_t* bytes, size_t len, int* status) {
    PackedModel* pm = nullptr;
    *status = guarded([&] { pm = new PackedModel(deserialize(std::span<const uint8_t>(bytes, len))); });
    return pm;
}

void ref_free(void* h) { delete static_cast<PackedModel*>(h); }

int ref_serialize(void* h, uint8_t* out, size_t* len) {
    return guarded([&] {
        std::vector<uint8_t> b = serialize(*static_cast<PackedModel*>(h));
        const size_t cap = *len;
        *len = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    });
}

int ref_block_offsets(void* h, uint64_t* out) {
    return guarded([&] {
        std::vector<size_t> o = compute_block_offsets(*static_cast<PackedModel*>(h));
        for (size_t i = 0; i < o.size(); ++i) out[i] = o[i];
    });
}

int ref_unpack_codes(void* h, uint8_t* codes) {
    return guarded([&] {
        const PackedModel& m = *static_cast<PackedModel*>(h);
        const size_t gc = m.block_grid_cols();
        for (size_t k = 0; k < m.block_count(); ++k) {
            const size_t br = k / gc, bc = k % gc;
            std::vector<QuantGroup> g = unpack_block(m.blocks[k], m.block_rows, m.group_size);
            for (size_t r = 0; r < m.block_rows; ++r)
                std::memcpy(codes + (br * m.block_rows + r) * m.cols + bc * m.group_size,
                            g[r].codes.data(), m.group_size);
        }
    });
}

int ref_dequantize(void* h, float* w) {
    return guarded([&] {
        Matrix d = dequantize_model(*static_cast<PackedModel*>(h));
        std::memcpy(w, d.data.data(), d.data.size() * sizeof(float));
    });
}

int ref_matmul(const float* x, const float* w, float* y, uint64_t rows, uint64_t cols) {
    return guarded([&] {
        Matrix mw(rows, cols, std::vector<float>(w, w + rows * cols));
        Vector vx(std::vector<float>(x, x + cols));
        Vector out = matmul_reference(vx, mw);
        std::memcpy(y, out.data.data(), rows * sizeof(float));
    });
}

int ref_gemv(void* h, const float* x, float* y, uint64_t* lookups) {
    return guarded([&] {
        const PackedModel& m = *static_cast<PackedModel*>(h);
        GemvStats st;
        Vector out = gemv(m, Vector(std::vector<float>(x, x + m.cols)), &st);
        std::memcpy(y, out.data.data(), m.rows * sizeof(float));
        if (lookups) *lookups = st.lookups;
    });
}

// M tokens through the reference gemv; tokens split over `threads` std::threads
// (the reference functions are pure and reentrant).
int ref_gemm_threads(void* h, const float* x, float* y, int64_t M, int threads) {
    const PackedModel& m = *static_cast<PackedModel*>(h);
    if (threads < 1) threads = 1;
    if (threads > M) threads = static_cast<int>(M > 0 ? M : 1);
    std::vector<int> rc(threads, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            rc[t] = guarded([&] {
                for (int64_t i = t; i < M; i += threads) {
                    Vector out = gemv(m, Vector(std::vector<float>(x + i * m.cols, x + (i + 1) * m.cols)));
                    std::memcpy(y + i * m.rows, out.data.data(), m.rows * sizeof(float));
                }
            });
        });
    for (auto& th : pool) th.join();
    for (int r : rc)
        if (r) return r;
    return 0;
}

int ref_bench_gemv(void* h, const float* x, uint64_t reps, double* out4) {
    return guarded([&] {
        const PackedModel& m = *static_cast<PackedModel*>(h);
        BenchResult r = bench_gemv(m, Vector(std::vector<float>(x, x + m.cols)), reps);
        out4[0] = r.median_us;
        out4[1] = r.p10_us;
        out4[2] = r.p90_us;
        out4[3] = static_cast<double>(r.lookups);
    });
}

}  // extern "C"
