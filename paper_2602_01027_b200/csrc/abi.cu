// abi.cu -- the extern "C" boundary (include/sfmp_cuda.h): SFMPPKD1 ingest,
// device model lifetime, kernel dispatch.  Host code only.
//
// Ingest restates deserialize (layout.cpp:210-279) + PackedModel::validate
// (layout.cpp:88-124) + compute_block_offsets (layout.cpp:301-314) with the
// same error kinds (errors.hpp:20-36).  Paths relative to /root/reference/proj.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/sfmp_cuda.h"
#include "sfmp_internal.h"

using sfmpk::DevModel;
using sfmpk::note_launch;

namespace {

thread_local std::string g_last_error;

sfmp_status fail(sfmp_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

sfmp_status cuda_fail(cudaError_t e, const char* what) {
    return fail(SFMP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define SFMP_CUDA_TRY(expr)                                 \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
    } while (0)

using sfmpk::DeviceGuard;

// ---------------------------------------------------------------------------
// Host ingest of SFMPPKD1
// ---------------------------------------------------------------------------
struct Parsed {
    uint64_t rows = 0, cols = 0;
    uint32_t m_b = 0, n_b = 0;
    int floor_bits = 0, ceil_bits = 0, mode = 0;
    const uint32_t* row_perm = nullptr;  // unaligned pointers into the stream
    const uint32_t* col_perm = nullptr;
    uint64_t K = 0;
    const uint8_t* bits = nullptr;
    std::vector<uint64_t> off;  // absolute offsets
    uint64_t payload_begin = 0, payload_end = 0;
};

template <class T>
T rd(const uint8_t* p) {
    T v;
    std::memcpy(&v, p, sizeof(T));
    return v;
}

sfmp_status check_perm(const uint8_t* p, uint64_t n, const char* what) {
    std::vector<uint8_t> seen(n, 0);
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t v = rd<uint32_t>(p + 4 * i);
        if (v >= n || seen[v])
            return fail(SFMP_ERR_FORMAT_INVARIANT,
                        std::string(what) + ": permutation is not a bijection on 0..n-1");
        seen[v] = 1;
    }
    return SFMP_OK;
}

sfmp_status parse(const uint8_t* b, size_t len, Parsed& m) {
    if (!b && len) return fail(SFMP_ERR_INVALID_ARGUMENT, "null byte buffer");
    size_t pos = 0;
    auto need = [&](uint64_t n, const char* what) -> sfmp_status {
        if (n > len - pos)
            return fail(SFMP_ERR_FORMAT_TRUNCATED, std::string("truncated while reading ") + what);
        return SFMP_OK;
    };
    sfmp_status s;
    if ((s = need(8, "magic"))) return s;
    if (std::memcmp(b, "SFMPPKD1", 8) != 0) return fail(SFMP_ERR_FORMAT_BAD_MAGIC, "not an SFMPPKD1 file");
    pos = 8;
    if ((s = need(2, "version"))) return s;
    const uint16_t ver = rd<uint16_t>(b + pos);
    pos += 2;
    if (ver != 1)
        return fail(SFMP_ERR_FORMAT_BAD_VERSION, "unsupported packed model version " + std::to_string(ver));
    if ((s = need(28, "header"))) return s;
    m.rows = rd<uint64_t>(b + pos);
    m.cols = rd<uint64_t>(b + pos + 8);
    m.m_b = rd<uint32_t>(b + pos + 16);
    m.n_b = rd<uint32_t>(b + pos + 20);
    m.floor_bits = b[pos + 24];
    m.ceil_bits = b[pos + 25];
    const uint8_t mode = b[pos + 26];
    pos += 28;
    if (mode > 3) return fail(SFMP_ERR_FORMAT_INVARIANT, "unknown reorder mode byte");
    m.mode = mode;
    if (m.rows < 1 || m.cols < 1 || m.m_b < 1 || m.n_b < 1 || m.rows % m.m_b || m.cols % m.n_b ||
        m.n_b % 8)
        return fail(SFMP_ERR_FORMAT_INVARIANT, "bad shape/block header fields");
    if (mode & 1) {
        if (m.rows > (len - pos) / 4) return fail(SFMP_ERR_FORMAT_TRUNCATED, "truncated while reading row permutation");
        m.row_perm = reinterpret_cast<const uint32_t*>(b + pos);
        if ((s = check_perm(b + pos, m.rows, "row permutation"))) return s;
        pos += m.rows * 4;
    }
    if (mode & 2) {
        if (m.cols > (len - pos) / 4) return fail(SFMP_ERR_FORMAT_TRUNCATED, "truncated while reading col permutation");
        m.col_perm = reinterpret_cast<const uint32_t*>(b + pos);
        if ((s = check_perm(b + pos, m.cols, "col permutation"))) return s;
        pos += m.cols * 4;
    }
    if ((s = need(8, "block count"))) return s;
    m.K = rd<uint64_t>(b + pos);
    pos += 8;
    if (m.K != (m.rows / m.m_b) * (m.cols / m.n_b))
        return fail(SFMP_ERR_FORMAT_INVARIANT, "block count does not match shape/block dims");
    if ((s = need(m.K, "block bit map"))) return s;
    m.bits = b + pos;
    pos += m.K;
    m.payload_begin = pos;
    m.off.resize(m.K);
    const uint64_t plane = static_cast<uint64_t>(m.m_b) * m.n_b / 8;
    for (uint64_t k = 0; k < m.K; ++k) {
        m.off[k] = pos;
        const uint64_t n = 4ull * m.m_b + static_cast<uint64_t>(m.bits[k]) * plane;
        if (n > len - pos) return fail(SFMP_ERR_FORMAT_TRUNCATED, "truncated while reading block payload");
        pos += n;
    }
    if (pos != len) return fail(SFMP_ERR_FORMAT_INVARIANT, "trailing bytes after model");
    m.payload_end = pos;
    if (m.floor_bits < 1 || m.ceil_bits < m.floor_bits || m.ceil_bits - m.floor_bits > 1 || m.ceil_bits > 8)
        return fail(SFMP_ERR_FORMAT_INVARIANT, "packed model: bad candidate bit-widths");
    for (uint64_t k = 0; k < m.K; ++k)
        if (m.bits[k] != m.floor_bits && m.bits[k] != m.ceil_bits)
            return fail(SFMP_ERR_FORMAT_INVARIANT, "packed model: block bit-width outside candidate set");
    return SFMP_OK;
}

void fill_info(const Parsed& p, sfmp_model_info* info) {
    std::memset(info, 0, sizeof(*info));
    info->rows = p.rows;
    info->cols = p.cols;
    info->m_b = p.m_b;
    info->n_b = p.n_b;
    info->floor_bits = p.floor_bits;
    info->ceil_bits = p.ceil_bits;
    info->mode = p.mode;
    info->block_count = p.K;
    uint64_t sum = 0, high = 0;
    for (uint64_t k = 0; k < p.K; ++k) {
        sum += p.bits[k];
        if (p.ceil_bits != p.floor_bits && p.bits[k] == p.ceil_bits) ++high;
    }
    info->blocks_high = high;
    info->avg_code_bits = p.K ? static_cast<double>(sum) / p.K : 0.0;
    info->payload_bytes = p.payload_end - p.payload_begin;
    info->num_shards = 1;
    info->out_rows = p.rows;
    info->global_rows = p.rows;
}

template <class T>
sfmp_status dev_upload(DevModel& d, T** dst, const void* src, size_t bytes) {
    void* ptr = nullptr;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(&ptr, bytes);
    if (e != cudaSuccess) return fail(SFMP_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    d.allocs.push_back(ptr);
    d.device_bytes += bytes;
    if (src) {
        e = cudaMemcpy(ptr, src, bytes, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy H2D");
    } else {
        e = cudaMemset(ptr, 0, bytes);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemset");
    }
    *dst = static_cast<T*>(ptr);
    return SFMP_OK;
}

void free_model(DevModel* d) {
    if (!d) return;
    {
        DeviceGuard g(d->device);
        for (void* p : d->allocs) cudaFree(p);
        if (d->d_host_stage) cudaFree(d->d_host_stage);
    }
    delete d;
}

// The decode GEMV (K1) needs 128-row units and n_b in {128, 256}; its cluster
// split is chosen per launch (gemv_tc.cu).
sfmp_status build_gemv_schedule(DevModel& d) {
    d.gemv_ok = d.TR == 128 && (d.n_b == 128 || d.n_b == 256) && d.cols < (1ull << 31) &&
                d.rows < (1ull << 31) && d.payload_bytes < (1ull << 48) && sfmpk::gemv_feasible(d);
    return SFMP_OK;
}

// Build a device model from a parsed stream, restricted to `brows` block rows
// (in the given order), repacked unit-major (sfmp_internal.h).  out_map:
// local reordered row -> column of y.
sfmp_status build_model(const uint8_t* bytes, const Parsed& p, int device,
                        const std::vector<uint64_t>& brows, const std::vector<uint32_t>& out_map,
                        uint64_t out_rows, DevModel** out, uint32_t flags = 0) {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(SFMP_ERR_CUDA, "no CUDA device available (no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(SFMP_ERR_INVALID_ARGUMENT, "bad device ordinal");
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (prop.major != 10)
        return fail(SFMP_ERR_CUDA, "device is not sm_100 (B200); this build targets sm_100a only");
    DeviceGuard guard(device);
    std::unique_ptr<DevModel, void (*)(DevModel*)> d(new DevModel(), free_model);
    d->device = device;
    d->num_sms = prop.multiProcessorCount;
    d->m_b = p.m_b;
    d->n_b = p.n_b;
    d->cols = p.cols;
    d->floor_bits = p.floor_bits;
    d->ceil_bits = p.ceil_bits;
    d->mode = p.mode;
    d->global_rows = p.rows;
    const uint64_t BC = p.cols / p.n_b;
    d->rows = brows.size() * p.m_b;
    d->K = brows.size() * BC;
    d->out_rows = out_rows;
    d->TR = (p.m_b % 128 == 0) ? 128 : p.m_b;
    d->BC = static_cast<uint32_t>(BC);
    d->RT = static_cast<uint32_t>(d->rows / d->TR);
    const uint32_t TR = d->TR, tiles = p.m_b / TR;
    const uint64_t rb = p.n_b / 8, pb_blk = static_cast<uint64_t>(p.m_b) * rb, pb_unit = TR * rb;
    // unit descriptors: units ordered (block row, TR-row tile, block column), each
    // scales[TR] | zeros[TR] | planes (the bytes of SFMPPKD1, re-ordered)
    uint64_t pos = 0, sum = 0;
    d->h_unit_desc.reserve(static_cast<size_t>(d->RT) * BC);
    for (uint64_t br : brows) {
        for (uint64_t bc = 0; bc < BC; ++bc) {
            sum += p.bits[br * BC + bc];
            if (p.ceil_bits != p.floor_bits && p.bits[br * BC + bc] == p.ceil_bits) ++d->blocks_high;
        }
        for (uint32_t t = 0; t < tiles; ++t)
            for (uint64_t bc = 0; bc < BC; ++bc) {
                const int bits = p.bits[br * BC + bc];
                d->h_unit_desc.push_back(pos | (static_cast<uint64_t>(bits) << 48));
                pos += 4ull * TR + bits * pb_unit;
            }
    }
    d->avg_bits = d->K ? static_cast<double>(sum) / d->K : 0.0;
    d->payload_bytes = pos;
    sfmp_status s;
    if ((s = dev_upload(*d, &d->d_unit_desc, d->h_unit_desc.data(), d->h_unit_desc.size() * 8))) return s;
    std::vector<uint32_t> cp(p.cols);
    if (p.col_perm) std::memcpy(cp.data(), p.col_perm, p.cols * 4);
    else std::iota(cp.begin(), cp.end(), 0u);
    if ((s = dev_upload(*d, &d->d_col_perm, cp.data(), cp.size() * 4))) return s;
    if ((s = dev_upload(*d, &d->d_out_map, out_map.data(), out_map.size() * 4))) return s;
    if ((s = build_gemv_schedule(*d))) return s;
    if ((flags & SFMP_MODEL_LUT_LAYOUT) && p.m_b % 32 == 0 && p.m_b <= 1024 && p.n_b % 128 == 0) {
        // K6 comparison layout: the block payloads as stored, 16-byte aligned
        std::vector<uint8_t> lp;
        std::vector<uint64_t> lo;
        std::vector<uint8_t> lb;
        for (uint64_t br : brows)
            for (uint64_t bc = 0; bc < BC; ++bc) {
                const uint64_t k = br * BC + bc;
                const uint64_t n = (k + 1 < p.K ? p.off[k + 1] : p.payload_end) - p.off[k];
                lo.push_back(lp.size());
                lb.push_back(p.bits[k]);
                lp.insert(lp.end(), bytes + p.off[k], bytes + p.off[k] + n);
                lp.resize((lp.size() + 15) / 16 * 16, 0);
            }
        if ((s = dev_upload(*d, &d->d_lut, lp.data(), lp.size()))) return s;
        if ((s = dev_upload(*d, &d->d_lut_off, lo.data(), lo.size() * 8))) return s;
        if ((s = dev_upload(*d, &d->d_lut_bits, lb.data(), lb.size()))) return s;
    }
    const bool want_gemm = !(flags & SFMP_MODEL_DECODE_ONLY) || !d->gemv_ok;
    if (d->gemv_ok) {
        // Device-side ingest (csrc/ingest.cu): the model's blocks are
        // uploaded as stored (one span per block row) and both layouts are built by
        // kernels; the host only keeps O(blocks) + O(rows x chunks) bookkeeping.
        std::vector<uint64_t> raw_off;
        std::vector<uint8_t> lbits;
        uint64_t raw_bytes = 0;
        for (uint64_t br : brows) {
            const uint64_t k0 = br * BC, k1 = k0 + BC;
            const uint64_t end = k1 < p.K ? p.off[k1] : p.payload_end;
            for (uint64_t k = k0; k < k1; ++k) {
                raw_off.push_back(raw_bytes + (p.off[k] - p.off[k0]));
                lbits.push_back(p.bits[k]);
            }
            raw_bytes += end - p.off[k0];
        }
        uint8_t* raw = nullptr;
        uint64_t* d_raw_off = nullptr;
        uint8_t* d_lbits = nullptr;
        auto release = [&]() {
            if (raw) cudaFree(raw);
            if (d_raw_off) cudaFree(d_raw_off);
            if (d_lbits) cudaFree(d_lbits);
        };
        SFMP_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&raw), raw_bytes));
        if ((e = cudaMalloc(reinterpret_cast<void**>(&d_raw_off), raw_off.size() * 8)) != cudaSuccess ||
            (e = cudaMalloc(reinterpret_cast<void**>(&d_lbits), lbits.size())) != cudaSuccess) {
            release();
            return cuda_fail(e, "ingest staging");
        }
        uint64_t at = 0;
        for (uint64_t br : brows) {
            const uint64_t k0 = br * BC, k1 = k0 + BC;
            const uint64_t n = (k1 < p.K ? p.off[k1] : p.payload_end) - p.off[k0];
            e = cudaMemcpy(raw + at, bytes + p.off[k0], n, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) break;
            at += n;
        }
        if (e == cudaSuccess) e = cudaMemcpy(d_raw_off, raw_off.data(), raw_off.size() * 8, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(d_lbits, lbits.data(), lbits.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            release();
            return cuda_fail(e, "ingest upload");
        }
        if ((s = dev_upload<uint8_t>(*d, &d->d_payload, nullptr, d->payload_bytes))) {
            release();
            return s;
        }
        e = sfmpk::device_unit_layout(raw, d_raw_off, d_lbits, p.m_b, p.n_b, static_cast<uint32_t>(BC),
                                      static_cast<uint32_t>(d->h_unit_desc.size()), d->d_unit_desc, d->d_payload, 0);
        if (e == cudaSuccess && want_gemm && p.cols % 128 == 0) {
            // row-tile layout: tile (T, kc) holds output rows 128T.. (inverse of out_map)
            const uint64_t KC = p.cols / 128, RT2 = (out_rows + 127) / 128;
            const int F = p.floor_bits;
            std::vector<uint32_t> inv(RT2 * 128, 0xFFFFFFFFu);
            for (uint64_t i = 0; i < out_map.size(); ++i)
                if (out_map[i] < inv.size()) inv[out_map[i]] = static_cast<uint32_t>(i);
            std::vector<uint64_t> woff(RT2 * KC + 1, 0);
            uint64_t w = 0;
            for (uint64_t T = 0; T < RT2; ++T)
                for (uint64_t kc = 0; kc < KC; ++kc) {
                    woff[T * KC + kc] = w;
                    const uint64_t bc = kc * 128 / p.n_b;
                    uint64_t nh = 0;
                    for (int r = 0; r < 128; ++r) {
                        const uint32_t i = inv[T * 128 + r];
                        if (i != 0xFFFFFFFFu && lbits[(i / p.m_b) * BC + bc] > F) ++nh;
                    }
                    w += 528 + static_cast<uint64_t>(F) * 2048 + nh * 16;
                }
            woff[RT2 * KC] = w;
            uint32_t* d_inv = nullptr;
            if ((s = dev_upload<uint8_t>(*d, &d->d_gl, nullptr, w)) ||
                (s = dev_upload(*d, &d->d_gl_off, woff.data(), woff.size() * 8))) {
                release();
                return s;
            }
            e = cudaMalloc(reinterpret_cast<void**>(&d_inv), inv.size() * 4);
            if (e == cudaSuccess) e = cudaMemcpy(d_inv, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice);
            if (e == cudaSuccess)
                e = sfmpk::device_tile_layout(raw, d_raw_off, d_lbits, p.m_b, p.n_b, static_cast<uint32_t>(BC), d_inv,
                                              d->d_gl_off, RT2 * KC, static_cast<uint32_t>(KC), F, d->d_gl, 0);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (d_inv) cudaFree(d_inv);
            d->gl_bytes = w;
            d->gl_row_tiles = RT2;
            if (e == cudaSuccess) {
                const std::vector<uint32_t> xslot = sfmpk::gemm_slot_table(cp);
                if ((s = dev_upload(*d, &d->d_xslot, xslot.data(), xslot.size() * 4))) {
                    release();
                    return s;
                }
            }
        }
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        release();
        if (e != cudaSuccess) return cuda_fail(e, "device ingest");
    } else {
        // other geometries: the unit-major layout in plane form, built on the host
        std::vector<uint8_t> payload(d->payload_bytes);
        uint64_t at = 0;
        for (uint64_t br : brows)
            for (uint32_t t = 0; t < tiles; ++t)
                for (uint64_t bc = 0; bc < BC; ++bc) {
                    const uint64_t k = br * BC + bc;
                    const uint8_t* blk = bytes + p.off[k];
                    const int bits = p.bits[k];
                    const uint64_t ro = static_cast<uint64_t>(t) * TR;
                    std::memcpy(&payload[at], blk + 2 * ro, 2ull * TR);                                // scales
                    std::memcpy(&payload[at + 2ull * TR], blk + 2ull * p.m_b + 2 * ro, 2ull * TR);   // zeros
                    at += 4ull * TR;
                    for (int i = 0; i < bits; ++i) {
                        std::memcpy(&payload[at], blk + 4ull * p.m_b + i * pb_blk + ro * rb, pb_unit);
                        at += pb_unit;
                    }
                }
        if (want_gemm) {
            std::vector<uint8_t> wl;
            std::vector<uint64_t> woff;
            if (sfmpk::build_gemm_layout(*d, payload, out_map, wl, woff)) {
                if ((s = dev_upload(*d, &d->d_gl, wl.data(), wl.size()))) return s;
                if ((s = dev_upload(*d, &d->d_gl_off, woff.data(), woff.size() * 8))) return s;
                d->gl_bytes = wl.size();
                const std::vector<uint32_t> xslot = sfmpk::gemm_slot_table(cp);
                if ((s = dev_upload(*d, &d->d_xslot, xslot.data(), xslot.size() * 4))) return s;
            }
        }
        if ((s = dev_upload(*d, &d->d_payload, payload.data(), payload.size()))) return s;
    }
    d->gemm_ok = sfmpk::gemm_supported(*d);
    const size_t ws = d->gemv_ok ? sfmpk::gemv_workspace_bytes(*d, 16) : 0;
    if (ws) {
        if ((s = dev_upload<float>(*d, &d->d_ws, nullptr, ws))) return s;
        d->ws_bytes = ws;
        d->device_bytes -= ws;  // device_bytes: weight layouts and indices only
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cuda_fail(e, "upload sync");
    *out = d.release();
    return SFMP_OK;
}

std::vector<uint32_t> row_order(const Parsed& p) {
    std::vector<uint32_t> r(p.rows);
    if (p.row_perm) std::memcpy(r.data(), p.row_perm, p.rows * 4);
    else std::iota(r.begin(), r.end(), 0u);
    return r;
}

// Snake (boustrophedon) block-row owner.
uint32_t snake_owner(uint64_t br, uint32_t G) {
    const uint64_t round = br / G, pos = br % G;
    return static_cast<uint32_t>((round & 1) ? G - 1 - pos : pos);
}

// Snake block-row partition + global gather map.
// Each shard's rows are held in ascending ORIGINAL row order (local position
// = rank of the row's original index among the shard's rows): the shard's
// y_local rows then map to increasing output rows, so the un-permutation of
// gathered shards reads G sequential streams and writes y coalesced.
// rank_of[g][j] = local position of the shard's j-th stored (reordered) row.
sfmp_status shard_plan(const Parsed& p, uint32_t G, std::vector<std::vector<uint64_t>>& owned,
                       std::vector<uint32_t>& gmap, uint64_t& SR,
                       std::vector<std::vector<uint32_t>>* rank_of = nullptr) {
    if (G < 1) return fail(SFMP_ERR_CONFIG, "num_shards must be >= 1");
    const uint64_t GR = p.rows / p.m_b;
    if (GR < G) return fail(SFMP_ERR_SHAPE, "fewer block rows than shards (repack with a smaller m_b)");
    owned.assign(G, {});
    for (uint64_t br = 0; br < GR; ++br) owned[snake_owner(br, G)].push_back(br);
    size_t maxb = 0;
    for (auto& v : owned) maxb = std::max(maxb, v.size());
    SR = maxb * p.m_b;
    const std::vector<uint32_t> rp = row_order(p);
    gmap.assign(G * SR, 0xFFFFFFFFu);
    if (rank_of) rank_of->assign(G, {});
    std::vector<std::pair<uint32_t, uint32_t>> rows;
    for (uint32_t g = 0; g < G; ++g) {
        rows.clear();
        for (size_t i = 0; i < owned[g].size(); ++i)
            for (uint32_t r = 0; r < p.m_b; ++r)
                rows.emplace_back(rp[owned[g][i] * p.m_b + r], static_cast<uint32_t>(i * p.m_b + r));
        std::sort(rows.begin(), rows.end());
        if (rank_of) (*rank_of)[g].assign(rows.size(), 0);
        for (size_t k = 0; k < rows.size(); ++k) {
            gmap[g * SR + k] = rows[k].first;
            if (rank_of) (*rank_of)[g][rows[k].second] = static_cast<uint32_t>(k);
        }
    }
    return SFMP_OK;
}

// Algorithmic bytes of one call: planes + fp16 s,z + perms + x + y.
uint64_t algo_bytes(const DevModel& d, int64_t M, sfmp_dtype dt) {
    const uint64_t esz = dt == SFMP_F32 ? 4 : 2;
    return d.payload_bytes + ((d.mode & 2) ? 4 * d.cols : 0) + ((d.mode & 1) ? 4 * d.rows : 0) +
           static_cast<uint64_t>(M) * d.cols * esz + 4ull * M * d.out_rows;
}

sfmp_path resolve_path(const DevModel& d, int64_t M, const void* x, sfmp_path path) {
    const bool x_aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    if (path == SFMP_PATH_AUTO)
        path = (M > 16 && d.gemm_ok && x_aligned) ? SFMP_PATH_GEMM : (d.gemv_ok ? SFMP_PATH_GEMV : SFMP_PATH_GENERIC);
    return path;
}

sfmp_status gemm_impl(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M, float* y,
                      void* workspace, size_t workspace_bytes, sfmp_path path, void* stream,
                      const sfmpk::PreNorm* norm);
sfmp_status grouped_impl(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                         const int64_t* Ms, float* const* ys, void* const* workspaces, const size_t* workspace_bytes,
                         int count, void* stream, const sfmpk::PreNorm* norms);

sfmp_status to_prenorm(const sfmp_prenorm* n, sfmpk::PreNorm& out) {
    out = sfmpk::PreNorm{};
    if (!n || !n->enabled) return SFMP_OK;
    if (n->gamma_dtype != SFMP_F32 && n->gamma_dtype != SFMP_F16 && n->gamma_dtype != SFMP_BF16)
        return fail(SFMP_ERR_INVALID_ARGUMENT, "bad gamma dtype");
    if (!(n->eps >= 0.f)) return fail(SFMP_ERR_INVALID_ARGUMENT, "eps must be >= 0");
    out.gamma = n->gamma;
    out.gdt = n->gamma_dtype;
    out.eps = n->eps;
    out.on = 1;
    return SFMP_OK;
}

double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Events around a region of one stream (the stats entry points synchronise).
struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    EventPair() {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
    }
    ~EventPair() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
    double us() const {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        return ms * 1e3;
    }
};

}  // namespace

namespace sfmpk {
sfmp_status api_fail(sfmp_status s, const std::string& msg) { return fail(s, msg); }
}  // namespace sfmpk

extern "C" {

uint64_t sfmp_launch_count(void) { return sfmpk::t_launches; }

int sfmp_abi_version(void) { return SFMP_CUDA_ABI_VERSION; }

const char* sfmp_status_string(sfmp_status s) {
    switch (s) {
        case SFMP_OK: return "ok";
        case SFMP_ERR_SHAPE: return "shape";
        case SFMP_ERR_CONFIG: return "config";
        case SFMP_ERR_FORMAT_BAD_MAGIC: return "bad_magic";
        case SFMP_ERR_FORMAT_BAD_VERSION: return "bad_version";
        case SFMP_ERR_FORMAT_TRUNCATED: return "truncated";
        case SFMP_ERR_FORMAT_INVARIANT: return "invariant";
        case SFMP_ERR_FORMAT_IO: return "io";
        case SFMP_ERR_CUDA: return "cuda";
        case SFMP_ERR_NCCL: return "nccl";
        case SFMP_ERR_INVALID_ARGUMENT: return "invalid_argument";
        case SFMP_ERR_NOMEM: return "nomem";
        case SFMP_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown";
}

const char* sfmp_last_error(void) { return g_last_error.c_str(); }

int sfmp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int ok = 0;
    for (int i = 0; i < n; ++i) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10) ++ok;
    }
    return ok;
}

sfmp_status sfmp_parse_header(const uint8_t* bytes, size_t len, sfmp_model_info* info) {
    if (!info) return fail(SFMP_ERR_INVALID_ARGUMENT, "null info");
    Parsed p;
    sfmp_status s = parse(bytes, len, p);
    if (s) return s;
    fill_info(p, info);
    return SFMP_OK;
}

sfmp_status sfmp_block_offsets(const uint8_t* bytes, size_t len, uint64_t* offsets, uint64_t count) {
    if (!offsets && count) return fail(SFMP_ERR_INVALID_ARGUMENT, "null offsets");
    Parsed p;
    sfmp_status s = parse(bytes, len, p);
    if (s) return s;
    if (count != p.K) return fail(SFMP_ERR_SHAPE, "offset buffer length != block count");
    std::memcpy(offsets, p.off.data(), p.K * 8);
    return SFMP_OK;
}

sfmp_status sfmp_model_create(const uint8_t* bytes, size_t len, int device, sfmp_dev_model** out) {
    return sfmp_model_create_ex(bytes, len, device, 0, out);
}

sfmp_status sfmp_model_create_ex(const uint8_t* bytes, size_t len, int device, uint32_t flags, sfmp_dev_model** out) {
    if (!out) return fail(SFMP_ERR_INVALID_ARGUMENT, "null out");
    if (flags & ~static_cast<uint32_t>(SFMP_MODEL_DECODE_ONLY | SFMP_MODEL_LUT_LAYOUT))
        return fail(SFMP_ERR_INVALID_ARGUMENT, "unknown model flags");
    *out = nullptr;
    Parsed p;
    sfmp_status s = parse(bytes, len, p);
    if (s) return s;
    std::vector<uint64_t> brows(p.rows / p.m_b);
    std::iota(brows.begin(), brows.end(), 0ull);
    DevModel* d = nullptr;
    s = build_model(bytes, p, device, brows, row_order(p), p.rows, &d, flags);
    if (s) return s;
    *out = reinterpret_cast<sfmp_dev_model*>(d);
    return SFMP_OK;
}

sfmp_status sfmp_model_create_from_parts(const sfmp_model_parts* pt, int device, sfmp_dev_model** out) {
    if (!pt || !out || !pt->block_bits || !pt->scales || !pt->zeros || !pt->plane_ptrs)
        return fail(SFMP_ERR_INVALID_ARGUMENT, "null parts");
    if (pt->m_b < 1 || pt->n_b < 1 || pt->rows % pt->m_b || pt->cols % pt->n_b || pt->n_b % 8 ||
        pt->mode < 0 || pt->mode > 3)
        return fail(SFMP_ERR_FORMAT_INVARIANT, "packed model: bad geometry");
    if (((pt->mode & 1) && !pt->row_perm) || ((pt->mode & 2) && !pt->col_perm))
        return fail(SFMP_ERR_FORMAT_INVARIANT, "packed model: permutation missing for mode");
    // Serialise (layout.cpp:179-208) then ingest through the same validated path.
    const uint64_t K = (pt->rows / pt->m_b) * (pt->cols / pt->n_b);
    const uint64_t pb = static_cast<uint64_t>(pt->m_b) * pt->n_b / 8;
    std::vector<uint8_t> b;
    auto put = [&](const void* src, size_t n) {
        const uint8_t* s = static_cast<const uint8_t*>(src);
        b.insert(b.end(), s, s + n);
    };
    const uint16_t ver = 1;
    const uint8_t hdr[4] = {static_cast<uint8_t>(pt->floor_bits), static_cast<uint8_t>(pt->ceil_bits),
                            static_cast<uint8_t>(pt->mode), 0};
    put("SFMPPKD1", 8);
    put(&ver, 2);
    put(&pt->rows, 8);
    put(&pt->cols, 8);
    put(&pt->m_b, 4);
    put(&pt->n_b, 4);
    put(hdr, 4);
    if (pt->mode & 1) put(pt->row_perm, pt->rows * 4);
    if (pt->mode & 2) put(pt->col_perm, pt->cols * 4);
    put(&K, 8);
    put(pt->block_bits, K);
    uint64_t pi = 0;
    for (uint64_t k = 0; k < K; ++k) {
        if (!pt->scales[k] || !pt->zeros[k]) return fail(SFMP_ERR_INVALID_ARGUMENT, "null block scales/zeros");
        put(pt->scales[k], pt->m_b * 2ull);
        put(pt->zeros[k], pt->m_b * 2ull);
        for (int i = 0; i < pt->block_bits[k]; ++i, ++pi) {
            if (!pt->plane_ptrs[pi]) return fail(SFMP_ERR_INVALID_ARGUMENT, "null plane pointer");
            put(pt->plane_ptrs[pi], pb);
        }
    }
    return sfmp_model_create(b.data(), b.size(), device, out);
}

sfmp_status sfmp_shard_plan(const uint8_t* bytes, size_t len, uint32_t num_shards, uint32_t* gather_map,
                            uint64_t* shard_rows) {
    if (!shard_rows) return fail(SFMP_ERR_INVALID_ARGUMENT, "null shard_rows");
    Parsed p;
    sfmp_status s = parse(bytes, len, p);
    if (s) return s;
    std::vector<std::vector<uint64_t>> owned;
    std::vector<uint32_t> gmap;
    uint64_t SR = 0;
    if ((s = shard_plan(p, num_shards, owned, gmap, SR))) return s;
    *shard_rows = SR;
    if (gather_map) std::memcpy(gather_map, gmap.data(), gmap.size() * 4);
    return SFMP_OK;
}

sfmp_status sfmp_shard_extract(const uint8_t* bytes, size_t len, uint32_t shard, uint32_t num_shards, uint8_t* out,
                               size_t* out_len) {
    if (!out_len) return fail(SFMP_ERR_INVALID_ARGUMENT, "null out_len");
    if (num_shards < 1 || shard >= num_shards) return fail(SFMP_ERR_CONFIG, "bad shard index/count");
    Parsed p;
    sfmp_status s = parse(bytes, len, p);
    if (s) return s;
    std::vector<std::vector<uint64_t>> owned;
    std::vector<uint32_t> gmap;
    std::vector<std::vector<uint32_t>> rank_of;
    uint64_t SR = 0;
    if ((s = shard_plan(p, num_shards, owned, gmap, SR, &rank_of))) return s;
    const std::vector<uint64_t>& br = owned[shard];
    const uint64_t BC = p.cols / p.n_b, rows = br.size() * p.m_b, K = br.size() * BC;
    // row permutation: stored row j -> its local output position (ascending original order)
    const uint8_t mode = static_cast<uint8_t>((p.mode & 2) | 1);
    uint64_t need = 38 + 4 * rows + (mode & 2 ? 4 * p.cols : 0) + 8 + K;
    for (uint64_t b : br)
        for (uint64_t bc = 0; bc < BC; ++bc) {
            const uint64_t k = b * BC + bc;
            need += (k + 1 < p.K ? p.off[k + 1] : p.payload_end) - p.off[k];
        }
    if (!out) {
        *out_len = need;
        return SFMP_OK;
    }
    if (*out_len < need) return fail(SFMP_ERR_SHAPE, "output buffer too small");
    uint8_t* o = out;
    auto put = [&](const void* src, size_t n) {
        std::memcpy(o, src, n);
        o += n;
    };
    const uint16_t ver = 1;
    const uint32_t mb = p.m_b, nb = p.n_b;
    const uint8_t hdr[4] = {static_cast<uint8_t>(p.floor_bits), static_cast<uint8_t>(p.ceil_bits), mode, 0};
    put("SFMPPKD1", 8);
    put(&ver, 2);
    put(&rows, 8);
    put(&p.cols, 8);
    put(&mb, 4);
    put(&nb, 4);
    put(hdr, 4);
    put(rank_of[shard].data(), rows * 4);
    if (mode & 2) put(p.col_perm, p.cols * 4);
    put(&K, 8);
    for (uint64_t b : br) put(p.bits + b * BC, BC);
    for (uint64_t b : br)
        for (uint64_t bc = 0; bc < BC; ++bc) {
            const uint64_t k = b * BC + bc;
            put(bytes + p.off[k], (k + 1 < p.K ? p.off[k + 1] : p.payload_end) - p.off[k]);
        }
    *out_len = need;
    return SFMP_OK;
}

sfmp_status sfmp_model_create_shard(const uint8_t* bytes, size_t len, int device, uint32_t shard,
                                    uint32_t num_shards, sfmp_dev_model** out) {
    return sfmp_model_create_shard_ex(bytes, len, device, shard, num_shards, 0, out);
}

sfmp_status sfmp_model_create_shard_ex(const uint8_t* bytes, size_t len, int device, uint32_t shard,
                                       uint32_t num_shards, uint32_t flags, sfmp_dev_model** out) {
    if (!out) return fail(SFMP_ERR_INVALID_ARGUMENT, "null out");
    if (flags & ~static_cast<uint32_t>(SFMP_MODEL_DECODE_ONLY | SFMP_MODEL_LUT_LAYOUT))
        return fail(SFMP_ERR_INVALID_ARGUMENT, "unknown model flags");
    *out = nullptr;
    if (num_shards < 1 || shard >= num_shards) return fail(SFMP_ERR_CONFIG, "bad shard index/count");
    Parsed p;
    sfmp_status s = parse(bytes, len, p);
    if (s) return s;
    std::vector<std::vector<uint64_t>> owned;
    std::vector<uint32_t> gmap;
    std::vector<std::vector<uint32_t>> rank_of;
    uint64_t SR = 0;
    if ((s = shard_plan(p, num_shards, owned, gmap, SR, &rank_of))) return s;
    DevModel* d = nullptr;
    s = build_model(bytes, p, device, owned[shard], rank_of[shard], SR, &d, flags);
    if (s) return s;
    d->shard = shard;
    d->num_shards = num_shards;
    d->shard_rows = SR;
    {
        // inverse map: original row -> shard g << 24 | local position (SR < 2^24)
        if (SR >= (1ull << 24) || num_shards > 255) {
            free_model(d);
            return fail(SFMP_ERR_UNSUPPORTED, "sharding supports < 2^24 rows per shard and < 256 shards");
        }
        std::vector<uint32_t> inv(p.rows, 0xFFFFFFFFu);
        for (uint64_t k = 0; k < gmap.size(); ++k)
            if (gmap[k] != 0xFFFFFFFFu) inv[gmap[k]] = static_cast<uint32_t>(((k / SR) << 24) | (k % SR));
        DeviceGuard guard(device);
        s = dev_upload(*d, &d->d_gather_map, gmap.data(), gmap.size() * 4);
        if (!s) s = dev_upload(*d, &d->d_gather_inv, inv.data(), inv.size() * 4);
    }
    if (s) {
        free_model(d);
        return s;
    }
    *out = reinterpret_cast<sfmp_dev_model*>(d);
    return SFMP_OK;
}

sfmp_status sfmp_model_destroy(sfmp_dev_model* model) {
    free_model(reinterpret_cast<DevModel*>(model));
    return SFMP_OK;
}

sfmp_status sfmp_model_get_info(const sfmp_dev_model* model, sfmp_model_info* info) {
    if (!model || !info) return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    const DevModel& d = *reinterpret_cast<const DevModel*>(model);
    std::memset(info, 0, sizeof(*info));
    info->rows = d.rows;
    info->cols = d.cols;
    info->m_b = d.m_b;
    info->n_b = d.n_b;
    info->floor_bits = d.floor_bits;
    info->ceil_bits = d.ceil_bits;
    info->mode = d.mode;
    info->block_count = d.K;
    info->blocks_high = d.blocks_high;
    info->avg_code_bits = d.avg_bits;
    info->payload_bytes = d.payload_bytes;
    info->device_bytes = d.device_bytes;
    info->shard = d.shard;
    info->num_shards = d.num_shards;
    info->out_rows = d.out_rows;
    info->global_rows = d.global_rows;
    return SFMP_OK;
}

sfmp_status sfmp_workspace_size(const sfmp_dev_model* model, int64_t M, sfmp_path path, size_t* bytes) {
    if (!model || !bytes) return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    const DevModel& d = *reinterpret_cast<const DevModel*>(model);
    size_t b = 0;
    // (AUTO may still pick the GEMV for M > 16 when x is misaligned: size for both)
    const bool gemm = (path == SFMP_PATH_GEMM) || (path == SFMP_PATH_AUTO && M > 16 && d.gemm_ok);
    if (gemm) b = sfmpk::gemm_workspace_bytes(d, M);
    if (path != SFMP_PATH_GENERIC && path != SFMP_PATH_GEMM && d.gemv_ok)
        b = std::max(b, sfmpk::gemv_workspace_bytes(d, 16));
    *bytes = b;
    return SFMP_OK;
}

sfmp_status sfmp_gemm_ex(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M,
                         float* y, void* workspace, size_t workspace_bytes, sfmp_path path,
                         void* stream) {
    return gemm_impl(model, x, dtype, M, y, workspace, workspace_bytes, path, stream, nullptr);
}

sfmp_status sfmp_gemm_norm(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M, float* y,
                           void* workspace, size_t workspace_bytes, const sfmp_prenorm* norm, void* stream) {
    sfmpk::PreNorm pn;
    sfmp_status s = to_prenorm(norm, pn);
    if (s) return s;
    return gemm_impl(model, x, dtype, M, y, workspace, workspace_bytes, SFMP_PATH_AUTO, stream, norm ? &pn : nullptr);
}

}  // extern "C"

namespace {
sfmp_status gemm_impl(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M, float* y,
                      void* workspace, size_t workspace_bytes, sfmp_path path, void* stream,
                      const sfmpk::PreNorm* norm) {
    if (!model) return fail(SFMP_ERR_INVALID_ARGUMENT, "null model");
    if (M < 0) return fail(SFMP_ERR_SHAPE, "negative M");
    if (M == 0) return SFMP_OK;
    if (!x || !y) return fail(SFMP_ERR_INVALID_ARGUMENT, "null x/y");
    if (dtype != SFMP_F32 && dtype != SFMP_F16 && dtype != SFMP_BF16)
        return fail(SFMP_ERR_INVALID_ARGUMENT, "bad dtype");
    const DevModel& d = *reinterpret_cast<const DevModel*>(model);
    if (workspace && (reinterpret_cast<uintptr_t>(workspace) & 127))
        return fail(SFMP_ERR_INVALID_ARGUMENT, "workspace must be 128-byte aligned");
    DeviceGuard guard(d.device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the tensor-core pre-pass reads x rows with 16-byte vector loads
    const bool x_aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    path = resolve_path(d, M, x, path);
    if (path == SFMP_PATH_GEMM && !x_aligned)
        return fail(SFMP_ERR_INVALID_ARGUMENT, "GEMM path needs x 16-byte aligned");
    cudaError_t e = cudaSuccess;
    const size_t esz = dtype == SFMP_F32 ? 4 : 2;
    switch (path) {
        case SFMP_PATH_GEMV: {
            if (!d.gemv_ok) return fail(SFMP_ERR_UNSUPPORTED, "decode GEMV needs m_b%128==0 and n_b in {128,256}");
            float* ws = static_cast<float*>(workspace);
            const size_t need = sfmpk::gemv_workspace_bytes(d, 16);
            if (!ws) ws = d.d_ws;
            else if (workspace_bytes < need) return fail(SFMP_ERR_CONFIG, "workspace too small");
            for (int64_t t0 = 0; t0 < M && e == cudaSuccess; t0 += 16) {
                const int mt = static_cast<int>(std::min<int64_t>(16, M - t0));
                e = sfmpk::launch_gemv(d, static_cast<const uint8_t*>(x) + t0 * d.cols * esz, dtype, mt,
                                       y + t0 * d.out_rows, ws, st, norm);
            }
            break;
        }
        case SFMP_PATH_GEMM: {
            if (!d.gemm_ok) return fail(SFMP_ERR_UNSUPPORTED, "tcgen05 GEMM unsupported for this geometry");
            const size_t need = sfmpk::gemm_workspace_bytes(d, M);
            if (need && (!workspace || workspace_bytes < need))
                return fail(SFMP_ERR_CONFIG, "GEMM path needs a workspace (sfmp_workspace_size)");
            e = sfmpk::launch_gemm(d, x, dtype, M, y, workspace, st, norm);
            break;
        }
        case SFMP_PATH_LUT:
            if (!sfmpk::lut_supported(d))
                return fail(SFMP_ERR_UNSUPPORTED, "LUT path needs SFMP_MODEL_LUT_LAYOUT, m_b % 32 == 0 (<= 1024), n_b % 128 == 0");
            if (dtype != SFMP_F32 || (norm && norm->on))
                return fail(SFMP_ERR_UNSUPPORTED, "the LUT comparison path takes f32 x without a fused norm");
            e = sfmpk::launch_lut(d, static_cast<const float*>(x), M, y, st);
            break;
        case SFMP_PATH_GENERIC:
            if (norm && norm->on) return fail(SFMP_ERR_UNSUPPORTED, "fused RMSNorm needs the GEMV or GEMM path");
            e = sfmpk::launch_generic(d, x, dtype, M, y, st);
            break;
        default: return fail(SFMP_ERR_INVALID_ARGUMENT, "bad path");
    }
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(SFMP_ERR_UNSUPPORTED, "fused RMSNorm: the x row does not fit the staged pre-pass");
    }
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return SFMP_OK;
}
}  // namespace

extern "C" {

sfmp_status sfmp_gemm_grouped(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                              int64_t M, float* const* ys, void* const* workspaces, const size_t* workspace_bytes,
                              int count, void* stream) {
    if (count < 0) return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    if (M < 0) return fail(SFMP_ERR_SHAPE, "negative M");
    std::vector<int64_t> Ms(count > 0 ? count : 1, M);
    return sfmp_gemm_grouped_v(models, xs, dtype, Ms.data(), ys, workspaces, workspace_bytes, count, stream);
}

sfmp_status sfmp_gemm_grouped_v(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                                const int64_t* Ms, float* const* ys, void* const* workspaces,
                                const size_t* workspace_bytes, int count, void* stream) {
    return grouped_impl(models, xs, dtype, Ms, ys, workspaces, workspace_bytes, count, stream, nullptr);
}

sfmp_status sfmp_gemm_grouped_v_norm(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                                     const int64_t* Ms, float* const* ys, void* const* workspaces,
                                     const size_t* workspace_bytes, int count, const sfmp_prenorm* norms,
                                     void* stream) {
    if (count < 0 || (count && !norms)) return fail(SFMP_ERR_INVALID_ARGUMENT, "null norms");
    std::vector<sfmpk::PreNorm> pn(count > 0 ? count : 1);
    for (int i = 0; i < count; ++i) {
        sfmp_status s = to_prenorm(&norms[i], pn[i]);
        if (s) return s;
    }
    return grouped_impl(models, xs, dtype, Ms, ys, workspaces, workspace_bytes, count, stream, pn.data());
}

}  // extern "C"

namespace {
sfmp_status grouped_impl(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                         const int64_t* Ms, float* const* ys, void* const* workspaces, const size_t* workspace_bytes,
                         int count, void* stream, const sfmpk::PreNorm* norms) {
    if (count < 0 || (count && (!models || !xs || !ys || !workspaces || !Ms)))
        return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    if (count == 0) return SFMP_OK;
    if (dtype != SFMP_F32 && dtype != SFMP_F16 && dtype != SFMP_BF16)
        return fail(SFMP_ERR_INVALID_ARGUMENT, "bad dtype");
    std::vector<const DevModel*> ms(count);
    for (int i = 0; i < count; ++i) {
        if (Ms[i] < 0) return fail(SFMP_ERR_SHAPE, "negative M");
        if (!models[i] || (Ms[i] && (!xs[i] || !ys[i]))) return fail(SFMP_ERR_INVALID_ARGUMENT, "null model/x/y");
        ms[i] = reinterpret_cast<const DevModel*>(models[i]);
    }
    // Runs of groupable decode problems go out as one launch; anything else
    // (prefill M, odd geometry) falls to the per-model entry point.
    for (int k = 0; k < count; ++k)
        if (workspaces[k] && (reinterpret_cast<uintptr_t>(workspaces[k]) & 127))
            return fail(SFMP_ERR_INVALID_ARGUMENT, "workspaces must be 128-byte aligned");
    auto decode_ok = [&](int k) {
        if (Ms[k] < 1 || Ms[k] > 16 || !ms[k]->gemv_ok || !workspaces[k]) return false;
        return !workspace_bytes || workspace_bytes[k] >= sfmpk::gemv_workspace_bytes(*ms[k], 16);
    };
    // A later decode launch of this call may overlap the previous one when its
    // workspaces are not used by any earlier launch of the call (the problems
    // themselves are independent by contract).
    std::vector<const void*> used_ws;
    bool prev_decode = false;
    int i = 0;
    while (i < count) {
        int j = i + 1;
        if (Ms[i] == 0) {
            i = j;
            continue;
        }
        if (Ms[i] <= 16 && ms[i]->gemv_ok) {
            if (!decode_ok(i))
                return fail(SFMP_ERR_CONFIG, "grouped decode needs a workspace per model (sfmp_workspace_size)");
            // groupable geometry and a workspace of its own (the records / partials /
            // counters of one launch must not alias); token counts 1..16 mix freely
            while (j < count && j - i < 40 && decode_ok(j) && sfmpk::gemv_groupable(*ms[i], *ms[j])) {
                bool distinct = true;
                for (int k = i; k < j; ++k) distinct = distinct && workspaces[k] != workspaces[j];
                if (!distinct) break;
                ++j;
            }
            DeviceGuard guard(ms[i]->device);
            std::vector<uint8_t*> wss(j - i);
            std::vector<int> mi(j - i);
            for (int k = i; k < j; ++k) {
                wss[k - i] = static_cast<uint8_t*>(workspaces[k]);
                mi[k - i] = static_cast<int>(Ms[k]);
            }
            bool disjoint = true;
            for (int k = i; k < j; ++k)
                for (const void* w : used_ws) disjoint = disjoint && w != workspaces[k];
            const bool overlap = prev_decode && disjoint;
            cudaError_t e = sfmpk::launch_gemv_group(ms.data() + i, xs + i, ys + i, wss.data(), mi.data(), j - i, dtype,
                                                     static_cast<cudaStream_t>(stream), overlap,
                                                     norms ? norms + i : nullptr);
            if (e == cudaErrorNotSupported) {
                cudaGetLastError();
                return fail(SFMP_ERR_UNSUPPORTED, "fused RMSNorm: the x row does not fit the staged pre-pass");
            }
            if (e != cudaSuccess) return cuda_fail(e, "grouped GEMV launch");
            for (int k = i; k < j; ++k) used_ws.push_back(workspaces[k]);
            prev_decode = true;
        } else {
            // workspace_bytes == NULL: the caller vouches for the sizes
            sfmp_status s = gemm_impl(models[i], xs[i], dtype, Ms[i], ys[i], workspaces[i],
                                      workspace_bytes ? workspace_bytes[i] : (workspaces[i] ? SIZE_MAX : 0),
                                      SFMP_PATH_AUTO, stream, norms ? norms + i : nullptr);
            if (s) return s;
            prev_decode = false;  // the next decode launch follows a non-grouped kernel
        }
        i = j;
    }
    return SFMP_OK;
}
}  // namespace

extern "C" {

sfmp_status sfmp_gemm(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M, float* y,
                      void* workspace, size_t workspace_bytes, void* stream) {
    return sfmp_gemm_ex(model, x, dtype, M, y, workspace, workspace_bytes, SFMP_PATH_AUTO, stream);
}

sfmp_status sfmp_gemm_host_stats(const sfmp_dev_model* model, const float* x_host, int64_t M, float* y_host,
                                 void* stream, sfmp_stats* stats) {
    if (!model || (!x_host && M) || (!y_host && M)) return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    const double w0 = now_us();
    const uint64_t l0 = sfmpk::t_launches;
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (M == 0) return SFMP_OK;
    DevModel& d = *const_cast<DevModel*>(reinterpret_cast<const DevModel*>(model));
    std::lock_guard<std::mutex> lock(d.host_mu);  // the staging buffers are per model
    DeviceGuard guard(d.device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    size_t wsb = 0;
    sfmp_status s = sfmp_workspace_size(model, M, SFMP_PATH_AUTO, &wsb);
    if (s) return s;
    const size_t xb = (M * d.cols * 4 + 255) / 256 * 256, yb = (M * d.out_rows * 4 + 255) / 256 * 256;
    const size_t need = xb + yb + wsb;
    if (need > d.host_stage_bytes) {
        if (d.d_host_stage) cudaFree(d.d_host_stage);
        d.d_host_stage = nullptr;
        d.host_stage_bytes = 0;
        SFMP_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&d.d_host_stage), need));
        SFMP_CUDA_TRY(cudaMemset(d.d_host_stage, 0, need));  // workspaces start zeroed
        d.host_stage_bytes = need;
    }
    float* dx = reinterpret_cast<float*>(d.d_host_stage);
    float* dy = reinterpret_cast<float*>(d.d_host_stage + xb);
    void* ws = wsb ? d.d_host_stage + xb + yb : nullptr;
    EventPair e_h2d, e_dev, e_d2h;
    if (stats) cudaEventRecord(e_h2d.a, st);
    SFMP_CUDA_TRY(cudaMemcpyAsync(dx, x_host, M * d.cols * 4, cudaMemcpyHostToDevice, st));
    if (stats) {
        cudaEventRecord(e_h2d.b, st);
        cudaEventRecord(e_dev.a, st);
    }
    s = sfmp_gemm(model, dx, SFMP_F32, M, dy, ws, wsb, stream);
    if (s) return s;
    if (stats) {
        cudaEventRecord(e_dev.b, st);
        cudaEventRecord(e_d2h.a, st);
    }
    SFMP_CUDA_TRY(cudaMemcpyAsync(y_host, dy, M * d.out_rows * 4, cudaMemcpyDeviceToHost, st));
    if (stats) cudaEventRecord(e_d2h.b, st);
    SFMP_CUDA_TRY(cudaStreamSynchronize(st));
    if (stats) {
        stats->h2d_us = e_h2d.us();
        stats->device_us = e_dev.us();
        stats->d2h_us = e_d2h.us();
        stats->bytes = algo_bytes(d, M, SFMP_F32);
        stats->flops = 2.0 * M * d.rows * d.cols;
        stats->path = resolve_path(d, M, dx, SFMP_PATH_AUTO);
        stats->launches = static_cast<int32_t>(sfmpk::t_launches - l0);
        stats->wall_us = now_us() - w0;
    }
    return SFMP_OK;
}

sfmp_status sfmp_gemm_host(const sfmp_dev_model* model, const float* x_host, int64_t M, float* y_host,
                           void* stream) {
    return sfmp_gemm_host_stats(model, x_host, M, y_host, stream, nullptr);
}

sfmp_status sfmp_gemm_stats(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M, float* y,
                            void* workspace, size_t workspace_bytes, sfmp_path path, void* stream,
                            sfmp_stats* stats) {
    if (!stats) return sfmp_gemm_ex(model, x, dtype, M, y, workspace, workspace_bytes, path, stream);
    std::memset(stats, 0, sizeof(*stats));
    if (!model) return fail(SFMP_ERR_INVALID_ARGUMENT, "null model");
    const DevModel& d = *reinterpret_cast<const DevModel*>(model);
    DeviceGuard guard(d.device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const double w0 = now_us();
    const uint64_t l0 = sfmpk::t_launches;
    EventPair ev;
    cudaEventRecord(ev.a, st);
    sfmp_status s = sfmp_gemm_ex(model, x, dtype, M, y, workspace, workspace_bytes, path, stream);
    if (s) return s;
    cudaEventRecord(ev.b, st);
    SFMP_CUDA_TRY(cudaEventSynchronize(ev.b));
    stats->device_us = ev.us();
    stats->bytes = M > 0 ? algo_bytes(d, M, dtype) : 0;
    stats->flops = 2.0 * M * d.rows * d.cols;
    stats->path = resolve_path(d, M, x, path);
    stats->launches = static_cast<int32_t>(sfmpk::t_launches - l0);
    stats->wall_us = now_us() - w0;
    return SFMP_OK;
}

sfmp_status sfmp_gemv_block(const sfmp_dev_model* model, uint64_t block, const float* x_reordered, float* out,
                            void* stream) {
    if (!model || !x_reordered || !out) return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    const DevModel& d = *reinterpret_cast<const DevModel*>(model);
    if (block >= d.K) return fail(SFMP_ERR_SHAPE, "gemv_block: block index out of range");
    DeviceGuard guard(d.device);
    cudaError_t e = sfmpk::launch_gemv_block(d, block, x_reordered, out, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "gemv_block launch");
    return SFMP_OK;
}

sfmp_status sfmp_dequantize(const sfmp_dev_model* model, float* w, void* stream) {
    if (!model || !w) return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    const DevModel& d = *reinterpret_cast<const DevModel*>(model);
    DeviceGuard guard(d.device);
    cudaError_t e = sfmpk::launch_dequant(d, w, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "dequant launch");
    return SFMP_OK;
}

sfmp_status sfmp_unpack_codes(const sfmp_dev_model* model, uint8_t* codes, void* stream) {
    if (!model || !codes) return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    const DevModel& d = *reinterpret_cast<const DevModel*>(model);
    DeviceGuard guard(d.device);
    cudaError_t e = sfmpk::launch_unpack(d, codes, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "unpack launch");
    return SFMP_OK;
}

sfmp_status sfmp_unpermute_gathered(const sfmp_dev_model* model, const float* gathered, int64_t M, float* y,
                                    void* stream) {
    if (!model || (M && (!gathered || !y))) return fail(SFMP_ERR_INVALID_ARGUMENT, "null argument");
    const DevModel& d = *reinterpret_cast<const DevModel*>(model);
    if (!d.d_gather_map) return fail(SFMP_ERR_CONFIG, "model is not a shard");
    DeviceGuard guard(d.device);
    cudaError_t e = sfmpk::launch_unpermute_gathered(d, gathered, M, y, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "unpermute launch");
    return SFMP_OK;
}

}  // extern "C"
