/*
 * sfmp_oracle.c -- TEST INFRASTRUCTURE ONLY (see sfmp_oracle.h).
 *
 * A plain-C restatement of the reference's CPU algorithms for the SFMP
 * mixed-precision GEMM path.  Compile with -O2 -ffp-contract=off and no
 * -march flags so float arithmetic rounds exactly like the reference built
 * with `g++ -std=c++20 -O2` on baseline x86-64 (SURVEY §8c caveat 2).
 * All paths below are relative to /root/reference/proj.
 */
#include "sfmp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* binary16 conversions: include/sfmp/fp16.hpp:14-56 and :58-83        */
/* ------------------------------------------------------------------ */

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

uint16_t sfmpo_fp16_from_float(float f) {
    const uint32_t x = f2u(f);
    const uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
    const uint32_t mag = x & 0x7FFFFFFFu;
    if (mag >= 0x7F800000u) /* inf -> max finite, NaN -> quiet NaN (fp16.hpp:20-24) */
        return (uint16_t)(sign | (mag > 0x7F800000u ? 0x7E00u : 0x7BFFu));
    if (mag >= 0x477FF000u) return (uint16_t)(sign | 0x7BFFu); /* saturate (:25-28) */
    if (mag < 0x33000001u) return sign;                        /* to zero (:29-32) */
    const int32_t e = (int32_t)(mag >> 23) - 127;
    const uint32_t sig = (mag & 0x007FFFFFu) | 0x00800000u;
    if (e < -14) { /* subnormal result, RNE (:37-46) */
        const int32_t sh = 13 + (-14 - e);
        uint32_t hm = sig >> sh;
        const uint32_t rem = sig & ((1u << sh) - 1u), half = 1u << (sh - 1);
        if (rem > half || (rem == half && (hm & 1u))) hm += 1;
        return (uint16_t)(sign | hm);
    }
    uint32_t hm = sig >> 13; /* normal result, RNE with carry (:48-55) */
    const uint32_t rem = sig & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (hm & 1u))) hm += 1;
    uint32_t b = ((uint32_t)(e + 15) << 10) + hm - (1u << 10);
    if (b >= 0x7C00u) b = 0x7BFFu;
    return (uint16_t)(sign | b);
}

float sfmpo_fp16_to_float(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1Fu;
    uint32_t m = h & 0x3FFu;
    if (e == 0) {
        if (m == 0) return u2f(sign);
        int sh = -1; /* normalise the subnormal (fp16.hpp:66-75) */
        do { m <<= 1; ++sh; } while ((m & 0x400u) == 0);
        return u2f(sign | ((uint32_t)(127 - 15 - sh) << 23) | ((m & 0x3FFu) << 13));
    }
    if (e == 0x1Fu) return u2f(sign | 0x7F800000u | (m << 13));
    return u2f(sign | ((e - 15 + 127) << 23) | (m << 13));
}

static inline float fp16_round(float f) { return sfmpo_fp16_to_float(sfmpo_fp16_from_float(f)); }

/* ------------------------------------------------------------------ */
/* SFMPPKD1 ingest: layout.cpp:210-279 (+ validate :88-124)            */
/* ------------------------------------------------------------------ */

typedef struct { const uint8_t* p; size_t len, pos; } rd_t;

static int rd(rd_t* r, void* dst, size_t n) {
    if (n > r->len - r->pos) return SFMPO_ERR_TRUNCATED; /* ByteReader::raw :154-159 */
    if (dst) memcpy(dst, r->p + r->pos, n);
    r->pos += n;
    return SFMPO_OK;
}

/* Permutation bijection check (reorder.cpp:10-17). */
static int check_perm(const uint32_t* fwd, uint64_t n) {
    uint8_t* seen = (uint8_t*)calloc(n ? n : 1, 1);
    if (!seen) return SFMPO_ERR_NOMEM;
    int rc = SFMPO_OK;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t v;
        memcpy(&v, fwd + i, 4);
        if (v >= n || seen[v]) { rc = SFMPO_ERR_INVARIANT; break; }
        seen[v] = 1;
    }
    free(seen);
    return rc;
}

int sfmpo_parse(const uint8_t* bytes, size_t len, sfmpo_model* m) {
    static const char magic_ref[8] = {'S', 'F', 'M', 'P', 'P', 'K', 'D', '1'};
    memset(m, 0, sizeof(*m));
    rd_t r = {bytes, len, 0};
    char magic[8];
    int rc;
    if ((rc = rd(&r, magic, 8))) return rc;
    if (memcmp(magic, magic_ref, 8) != 0) return SFMPO_ERR_BAD_MAGIC;
    if ((rc = rd(&r, &m->version, 2))) return rc;
    if (m->version != 1) return SFMPO_ERR_BAD_VERSION;
    uint8_t fb, cb, mode, resv;
    if ((rc = rd(&r, &m->rows, 8)) || (rc = rd(&r, &m->cols, 8)) || (rc = rd(&r, &m->m_b, 4)) ||
        (rc = rd(&r, &m->n_b, 4)) || (rc = rd(&r, &fb, 1)) || (rc = rd(&r, &cb, 1)) ||
        (rc = rd(&r, &mode, 1)) || (rc = rd(&r, &resv, 1)))
        return rc;
    m->floor_bits = fb;
    m->ceil_bits = cb;
    if (mode > 3) return SFMPO_ERR_INVARIANT;
    m->mode = mode;
    if (m->rows < 1 || m->cols < 1 || m->m_b < 1 || m->n_b < 1 || m->rows % m->m_b != 0 ||
        m->cols % m->n_b != 0 || m->n_b % 8 != 0)
        return SFMPO_ERR_INVARIANT;
    if (mode & 1) {
        if (m->rows > (len - r.pos) / 4) return SFMPO_ERR_TRUNCATED;
        m->row_perm = (const uint32_t*)(bytes + r.pos);
        r.pos += m->rows * 4;
        if ((rc = check_perm(m->row_perm, m->rows))) return rc;
    }
    if (mode & 2) {
        if (m->cols > (len - r.pos) / 4) return SFMPO_ERR_TRUNCATED;
        m->col_perm = (const uint32_t*)(bytes + r.pos);
        r.pos += m->cols * 4;
        if ((rc = check_perm(m->col_perm, m->cols))) return rc;
    }
    if ((rc = rd(&r, &m->K, 8))) return rc;
    const uint64_t expect = (m->rows / m->m_b) * (m->cols / m->n_b);
    if (m->K != expect) return SFMPO_ERR_INVARIANT;
    if (m->K > len - r.pos) return SFMPO_ERR_TRUNCATED;
    m->block_bits = bytes + r.pos;
    r.pos += m->K;
    m->block_off = (uint64_t*)malloc((m->K ? m->K : 1) * sizeof(uint64_t));
    if (!m->block_off) return SFMPO_ERR_NOMEM;
    const uint64_t plane_bytes = (uint64_t)m->m_b * m->n_b / 8;
    for (uint64_t k = 0; k < m->K; ++k) {
        m->block_off[k] = r.pos;
        const uint64_t need = 4ull * m->m_b + (uint64_t)m->block_bits[k] * plane_bytes;
        if (need > len - r.pos) { sfmpo_free(m); return SFMPO_ERR_TRUNCATED; }
        r.pos += need;
    }
    if (r.pos != len) { sfmpo_free(m); return SFMPO_ERR_INVARIANT; } /* trailing bytes :274-275 */
    /* PackedModel::validate (layout.cpp:88-124) */
    if (m->floor_bits < 1 || m->ceil_bits < m->floor_bits || m->ceil_bits - m->floor_bits > 1 ||
        m->ceil_bits > 8) { sfmpo_free(m); return SFMPO_ERR_INVARIANT; }
    for (uint64_t k = 0; k < m->K; ++k)
        if (m->block_bits[k] != m->floor_bits && m->block_bits[k] != m->ceil_bits) {
            sfmpo_free(m);
            return SFMPO_ERR_INVARIANT;
        }
    m->base = bytes;
    return SFMPO_OK;
}

void sfmpo_free(sfmpo_model* m) {
    free(m->block_off);
    m->block_off = NULL;
}

int sfmpo_block_offsets(const uint8_t* bytes, size_t len, uint64_t* out, uint64_t K) {
    sfmpo_model m;
    int rc = sfmpo_parse(bytes, len, &m);
    if (rc) return rc;
    if (K != m.K) { sfmpo_free(&m); return SFMPO_ERR_SHAPE; }
    memcpy(out, m.block_off, K * sizeof(uint64_t));
    sfmpo_free(&m);
    return SFMPO_OK;
}

/* ------------------------------------------------------------------ */
/* unpack / dequant: layout.cpp:67-86, :316-332; quantizer.cpp:50-55   */
/* ------------------------------------------------------------------ */

static inline uint16_t ld16(const uint8_t* p) { uint16_t v; memcpy(&v, p, 2); return v; }

void sfmpo_unpack_codes(const sfmpo_model* m, uint8_t* codes) {
    const uint64_t gc = m->cols / m->n_b, rb = m->n_b / 8, pb = (uint64_t)m->m_b * rb;
    for (uint64_t k = 0; k < m->K; ++k) {
        const uint64_t br = k / gc, bc = k % gc;
        const int bits = m->block_bits[k];
        const uint8_t* planes = m->base + m->block_off[k] + 4ull * m->m_b;
        for (uint64_t r = 0; r < m->m_b; ++r) {
            uint8_t* dst = codes + (br * m->m_b + r) * m->cols + bc * m->n_b;
            for (uint64_t j = 0; j < m->n_b; ++j) {
                uint8_t c = 0;
                for (int i = 0; i < bits; ++i)
                    c |= (uint8_t)(((planes[i * pb + r * rb + j / 8] >> (j % 8)) & 1u) << i);
                dst[j] = c;
            }
        }
    }
}

void sfmpo_dequantize(const sfmpo_model* m, float* w) {
    const uint64_t cols = m->cols;
    const uint64_t gc = cols / m->n_b, rb = m->n_b / 8, pb = (uint64_t)m->m_b * rb;
    /* Inverse permutations: apply_reorder_inverse gathers by inverse(perm), i.e.
     * the reordered row i lands at original row row_perm[i]. */
    for (uint64_t k = 0; k < m->K; ++k) {
        const uint64_t br = k / gc, bc = k % gc;
        const int bits = m->block_bits[k];
        const uint8_t* blk = m->base + m->block_off[k];
        const uint8_t* planes = blk + 4ull * m->m_b;
        for (uint64_t r = 0; r < m->m_b; ++r) {
            const float s = sfmpo_fp16_to_float(ld16(blk + 2 * r));
            const float z = sfmpo_fp16_to_float(ld16(blk + 2ull * m->m_b + 2 * r));
            const uint64_t rr = br * m->m_b + r;
            uint32_t orow_idx;
            if (m->row_perm) memcpy(&orow_idx, m->row_perm + rr, 4); else orow_idx = (uint32_t)rr;
            float* orow = w + (uint64_t)orow_idx * cols;
            for (uint64_t j = 0; j < m->n_b; ++j) {
                uint8_t c = 0;
                for (int i = 0; i < bits; ++i)
                    c |= (uint8_t)(((planes[i * pb + r * rb + j / 8] >> (j % 8)) & 1u) << i);
                const float v = s * (float)c + z; /* quantizer.cpp:53, two roundings */
                const uint64_t cj = bc * m->n_b + j;
                uint32_t oc;
                if (m->col_perm) memcpy(&oc, m->col_perm + cj, 4); else oc = (uint32_t)cj;
                orow[oc] = v;
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* matmul_reference: matrix.cpp:5-17                                   */
/* ------------------------------------------------------------------ */

static void matmul_rows(const float* x, const float* w, float* y, int64_t M, int64_t rows,
                        int64_t cols, int64_t r0, int64_t r1) {
    for (int64_t t = 0; t < M; ++t) {
        const float* xt = x + t * cols;
        for (int64_t i = r0; i < r1; ++i) {
            const float* wr = w + i * cols;
            float acc = 0.0f;
            for (int64_t k = 0; k < cols; ++k) acc += xt[k] * wr[k];
            y[t * rows + i] = acc;
        }
    }
}

void sfmpo_matmul_reference(const float* x, const float* w, float* y, int64_t M, int64_t rows,
                            int64_t cols) {
    matmul_rows(x, w, y, M, rows, cols, 0, rows);
}

typedef struct {
    const float *x, *w;
    float* y;
    int64_t M, rows, cols, r0, r1;
} mm_job;

static void* mm_thread(void* p) {
    mm_job* j = (mm_job*)p;
    matmul_rows(j->x, j->w, j->y, j->M, j->rows, j->cols, j->r0, j->r1);
    return NULL;
}

void sfmpo_matmul_reference_mt(const float* x, const float* w, float* y, int64_t M, int64_t rows,
                               int64_t cols, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    mm_job jobs[256];
    const int64_t per = (rows + threads - 1) / threads;
    int n = 0;
    for (int t = 0; t < threads; ++t) {
        const int64_t r0 = t * per, r1 = r0 + per < rows ? r0 + per : rows;
        if (r0 >= r1) break;
        jobs[n] = (mm_job){x, w, y, M, rows, cols, r0, r1};
        pthread_create(&th[n], NULL, mm_thread, &jobs[n]);
        ++n;
    }
    for (int t = 0; t < n; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------ */
/* LUT GEMV: lutgemm.cpp:11-36 (tables), lutgemm.hpp:21-26 (lookup),   */
/* lutgemm.cpp:45-71 (accumulate_block), :95-135 (gemv)                */
/* ------------------------------------------------------------------ */

static void build_tables(const float* xr, uint64_t n, float* tab /* n/8 x 128 */) {
    for (uint64_t t = 0; t < n / 8; ++t) {
        const float* xs = xr + t * 8;
        float* a = tab + t * 128;
        a[0] = -xs[0];
        a[1] = xs[0];
        for (int k = 1; k < 7; ++k) { /* recursive doubling, ascending k */
            const float xv = xs[k];
            const int half = 1 << k;
            for (int j = 0; j < half; ++j) {
                const float b = a[j];
                a[j + half] = b + xv;
                a[j] = b - xv;
            }
        }
        for (int j = 0; j < 128; ++j) a[j] += xs[7]; /* stored half: bit 7 = +1 */
    }
}

static inline float table_lookup(const float* e, uint8_t p) {
    const uint32_t neg = ((uint32_t)p >> 7) ^ 1u;
    const uint32_t idx = ((uint32_t)p ^ (0x7Fu * neg)) & 0x7Fu;
    return u2f(f2u(e[idx]) ^ (neg << 31));
}

int sfmpo_gemv_lut(const sfmpo_model* m, const float* x, float* y, uint64_t* lookups) {
    const uint64_t rows = m->rows, cols = m->cols, m_b = m->m_b, n_b = m->n_b;
    const uint64_t gc = cols / n_b, rb = n_b / 8, pb = m_b * rb;
    float* xr = (float*)malloc(cols * sizeof(float));
    float* tab = (float*)malloc((cols / 8) * 128 * sizeof(float));
    float* yr = (float*)calloc(rows, sizeof(float));
    float* csum = (float*)malloc(gc * sizeof(float));
    if (!xr || !tab || !yr || !csum) { free(xr); free(tab); free(yr); free(csum); return SFMPO_ERR_NOMEM; }
    for (uint64_t j = 0; j < cols; ++j) { /* reorder_activation_in (reorder.cpp:103-111) */
        uint32_t src = (uint32_t)j;
        if (m->col_perm) memcpy(&src, m->col_perm + j, 4);
        xr[j] = x[src];
    }
    build_tables(xr, cols, tab);
    for (uint64_t bc = 0; bc < gc; ++bc) { /* range_sum, ascending (lutgemm.cpp:73-77) */
        float s = 0.0f;
        for (uint64_t i = 0; i < n_b; ++i) s += xr[bc * n_b + i];
        csum[bc] = s;
    }
    uint64_t lk = 0;
    for (uint64_t k = 0; k < m->K; ++k) {
        const uint64_t br = k / gc, bc = k % gc;
        const int bits = m->block_bits[k];
        const uint8_t* blk = m->base + m->block_off[k];
        const uint8_t* planes = blk + 4 * m_b;
        const float* luts = tab + (bc * n_b / 8) * 128;
        const float levels = (float)((1 << bits) - 1);
        float* out = yr + br * m_b;
        for (uint64_t r = 0; r < m_b; ++r) {
            float pacc = 0.0f;
            for (int i = 0; i < bits; ++i) {
                const uint8_t* pbp = planes + i * pb + r * rb;
                float s = 0.0f;
                for (uint64_t g = 0; g < rb; ++g) s += table_lookup(luts + g * 128, pbp[g]);
                pacc += (float)(1 << i) * s;
            }
            const float sh = 0.5f * sfmpo_fp16_to_float(ld16(blk + 2 * r));
            const float zh = sfmpo_fp16_to_float(ld16(blk + 2 * m_b + 2 * r)) + sh * levels;
            const float t1 = sh * pacc, t2 = zh * csum[bc];
            out[r] += t1 + t2;
        }
        lk += (uint64_t)bits * m_b * rb;
    }
    for (uint64_t i = 0; i < rows; ++i) { /* reorder_activation_out (reorder.cpp:113-121) */
        uint32_t dst = (uint32_t)i;
        if (m->row_perm) memcpy(&dst, m->row_perm + i, 4);
        y[dst] = yr[i];
    }
    if (lookups) *lookups = lk;
    free(xr); free(tab); free(yr); free(csum);
    return SFMPO_OK;
}

typedef struct {
    const sfmpo_model* m;
    const float* x;
    float* y;
    int64_t t0, t1;
    int rc;
} lut_job;

static void* lut_thread(void* p) {
    lut_job* j = (lut_job*)p;
    for (int64_t t = j->t0; t < j->t1 && !j->rc; ++t)
        j->rc = sfmpo_gemv_lut(j->m, j->x + t * j->m->cols, j->y + t * j->m->rows, NULL);
    return NULL;
}

int sfmpo_gemm_lut(const sfmpo_model* m, const float* x, float* y, int64_t M, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (threads > M) threads = (int)(M > 0 ? M : 1);
    pthread_t th[256];
    lut_job jobs[256];
    const int64_t per = (M + threads - 1) / threads;
    int n = 0;
    for (int t = 0; t < threads; ++t) {
        const int64_t a = t * per, b = a + per < M ? a + per : M;
        if (a >= b) break;
        jobs[n] = (lut_job){m, x, y, a, b, 0};
        pthread_create(&th[n], NULL, lut_thread, &jobs[n]);
        ++n;
    }
    int rc = 0;
    for (int t = 0; t < n; ++t) { pthread_join(th[t], NULL); if (jobs[t].rc) rc = jobs[t].rc; }
    return rc;
}

/* ------------------------------------------------------------------ */
/* Offline fixture path                                  */
/* ------------------------------------------------------------------ */

int sfmpo_quantize_group(const float* v, size_t n, int bits, float* scale, float* zero,
                         uint8_t* codes) {
    if (bits < 1 || bits > 8) return SFMPO_ERR_CONFIG; /* quantizer.cpp:12-13 */
    if (n == 0) return SFMPO_ERR_SHAPE;
    float lo = v[0], hi = v[0];
    for (size_t i = 1; i < n; ++i) { if (v[i] < lo) lo = v[i]; if (v[i] > hi) hi = v[i]; }
    const int levels = (1 << bits) - 1;
    float s = (hi > lo) ? (hi - lo) / (float)levels : 1.0f;
    float z = lo;
    s = fp16_round(s); /* parameters through fp16 before coding (:28-31) */
    z = fp16_round(z);
    if (!(s > 0.0f)) { /* degenerate range (:32-39) */
        *scale = 1.0f;
        *zero = z;
        memset(codes, 0, n);
        return SFMPO_OK;
    }
    *scale = s;
    *zero = z;
    for (size_t i = 0; i < n; ++i) {
        float q = roundf((v[i] - z) / s);
        if (q < 0.0f) q = 0.0f;
        if (q > (float)levels) q = (float)levels;
        codes[i] = (uint8_t)q;
    }
    return SFMPO_OK;
}

typedef struct { float v; uint32_t i; } kv_f;
typedef struct { double v; uint64_t i; } kv_d;

/* argsort_desc (reorder.cpp:40-48): stable, so ties keep ascending index;
 * equivalently order by (value desc, index asc). */
static int cmp_desc_f(const void* a, const void* b) {
    const kv_f *x = (const kv_f*)a, *y = (const kv_f*)b;
    if (x->v > y->v) return -1;
    if (x->v < y->v) return 1;
    return (x->i > y->i) - (x->i < y->i);
}
/* quantile_threshold ordering (allocation.cpp:70-75). */
static int cmp_desc_d(const void* a, const void* b) {
    const kv_d *x = (const kv_d*)a, *y = (const kv_d*)b;
    if (x->v != y->v) return x->v > y->v ? -1 : 1;
    return (x->i > y->i) - (x->i < y->i);
}

static void argsort_desc_f(const float* v, uint64_t n, uint32_t* out) {
    kv_f* t = (kv_f*)malloc(n * sizeof(kv_f));
    for (uint64_t i = 0; i < n; ++i) { t[i].v = v[i]; t[i].i = (uint32_t)i; }
    qsort(t, n, sizeof(kv_f), cmp_desc_f);
    for (uint64_t i = 0; i < n; ++i) out[i] = t[i].i;
    free(t);
}

typedef struct { uint8_t* p; size_t cap, pos; } wr_t;
static void wr(wr_t* w, const void* src, size_t n) {
    if (w->p && w->pos + n <= w->cap) memcpy(w->p + w->pos, src, n);
    w->pos += n;
}

int sfmpo_build_model(const float* W, const float* S, uint64_t rows, uint64_t cols, uint32_t m_b,
                      uint32_t n_b, double target_bpw, int mode, uint8_t* out, size_t* out_len) {
    if (m_b < 1 || n_b < 1 || n_b % 8 || rows % m_b || cols % n_b) return SFMPO_ERR_SHAPE;
    if (mode < 0 || mode > 3) return SFMPO_ERR_CONFIG;
    /* make_bit_plan: effective_weight_bits (allocation.cpp:18-29) + candidate_bits (:9-16) */
    const double overhead = 32.0 / (double)n_b;
    if (!(target_bpw > overhead)) return SFMPO_ERR_CONFIG;
    const double eff = target_bpw - overhead;
    if (!(eff >= 1.0)) return SFMPO_ERR_CONFIG;
    const int fb = (int)floor(eff);
    const double alpha = eff - fb;
    const int cb = (alpha == 0.0) ? fb : fb + 1;
    if (cb > 8) return SFMPO_ERR_CONFIG;

    uint32_t* rp = (uint32_t*)malloc(rows * 4);
    uint32_t* cp = (uint32_t*)malloc(cols * 4);
    for (uint64_t i = 0; i < rows; ++i) rp[i] = (uint32_t)i;
    for (uint64_t j = 0; j < cols; ++j) cp[j] = (uint32_t)j;
    if (mode != 0) { /* make_reorder_spec (reorder.cpp:50-62) via row_col_salience (salience.cpp:31-45) */
        float* rs = (float*)malloc(rows * 4);
        float* cs = (float*)calloc(cols, 4);
        for (uint64_t i = 0; i < rows; ++i) {
            const float* r = S + i * cols;
            double acc = 0.0;
            for (uint64_t j = 0; j < cols; ++j) { acc += r[j]; cs[j] += r[j]; }
            rs[i] = (float)acc;
        }
        if (mode & 1) argsort_desc_f(rs, rows, rp);
        if (mode & 2) argsort_desc_f(cs, cols, cp);
        free(rs); free(cs);
    }
    /* apply_reorder (reorder.cpp:75-93): out[i][j] = w[rp[i]][cp[j]] */
    float* Wr = (float*)malloc(rows * cols * 4);
    float* Sr = (float*)malloc(rows * cols * 4);
    if (!Wr || !Sr) { free(rp); free(cp); free(Wr); free(Sr); return SFMPO_ERR_NOMEM; }
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) {
            Wr[i * cols + j] = W[(uint64_t)rp[i] * cols + cp[j]];
            Sr[i * cols + j] = S[(uint64_t)rp[i] * cols + cp[j]];
        }
    /* block_salience (salience.cpp:47-75) + allocate_block_bits (allocation.cpp:85-103) */
    const uint64_t gr = rows / m_b, gc = cols / n_b, K = gr * gc;
    kv_d* bs = (kv_d*)malloc(K * sizeof(kv_d));
    for (uint64_t br = 0; br < gr; ++br)
        for (uint64_t bc = 0; bc < gc; ++bc) {
            double s = 0.0;
            for (uint64_t i = br * m_b; i < (br + 1) * m_b; ++i)
                for (uint64_t j = bc * n_b; j < (bc + 1) * n_b; ++j) s += Sr[i * cols + j];
            bs[br * gc + bc] = (kv_d){s, br * gc + bc};
        }
    uint8_t* bits = (uint8_t*)malloc(K);
    memset(bits, fb, K);
    const uint64_t nhigh = (uint64_t)floor(alpha * (double)K + 0.5); /* high_block_count :51-57 */
    if (nhigh > 0) {
        qsort(bs, K, sizeof(kv_d), cmp_desc_d);
        for (uint64_t t = 0; t < nhigh && t < K; ++t) bits[bs[t].i] = (uint8_t)cb;
    }
    free(bs);

    /* serialize (layout.cpp:179-208) with pack_block (:29-65) inline */
    wr_t w = {out, out ? *out_len : 0, 0};
    static const char magic[8] = {'S', 'F', 'M', 'P', 'P', 'K', 'D', '1'};
    const uint16_t ver = 1;
    const uint32_t mb32 = m_b, nb32 = n_b;
    const uint8_t hdr[4] = {(uint8_t)fb, (uint8_t)cb, (uint8_t)mode, 0};
    wr(&w, magic, 8); wr(&w, &ver, 2); wr(&w, &rows, 8); wr(&w, &cols, 8);
    wr(&w, &mb32, 4); wr(&w, &nb32, 4); wr(&w, hdr, 4);
    if (mode & 1) wr(&w, rp, rows * 4);
    if (mode & 2) wr(&w, cp, cols * 4);
    wr(&w, &K, 8);
    wr(&w, bits, K);
    const uint64_t rb = n_b / 8, pbytes = (uint64_t)m_b * rb;
    uint16_t* sc = (uint16_t*)malloc(m_b * 2);
    uint16_t* zr = (uint16_t*)malloc(m_b * 2);
    uint8_t* pl = (uint8_t*)malloc(8 * pbytes);
    uint8_t* codes = (uint8_t*)malloc(n_b);
    for (uint64_t k = 0; k < K; ++k) {
        const uint64_t br = k / gc, bc = k % gc;
        const int b = bits[k];
        memset(pl, 0, (size_t)b * pbytes);
        for (uint64_t r = 0; r < m_b; ++r) {
            float s, z;
            sfmpo_quantize_group(Wr + (br * m_b + r) * cols + bc * n_b, n_b, b, &s, &z, codes);
            sc[r] = sfmpo_fp16_from_float(s);
            zr[r] = sfmpo_fp16_from_float(z);
            for (uint64_t j = 0; j < n_b; ++j)
                for (int i = 0; i < b; ++i)
                    if ((codes[j] >> i) & 1u) pl[i * pbytes + r * rb + j / 8] |= (uint8_t)(1u << (j % 8));
        }
        wr(&w, sc, m_b * 2);
        wr(&w, zr, m_b * 2);
        wr(&w, pl, (size_t)b * pbytes);
    }
    free(sc); free(zr); free(pl); free(codes); free(bits);
    free(Wr); free(Sr); free(rp); free(cp);
    const size_t cap = out ? *out_len : 0;
    *out_len = w.pos;
    if (out && w.pos > cap) return SFMPO_ERR_SHAPE;
    return SFMPO_OK;
}

/* ------------------------------------------------------------------ */
/* Deterministic synthetic inputs                                      */
/* ------------------------------------------------------------------ */

static inline uint64_t splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline double unif(uint64_t* s) { /* (0,1] */
    return ((double)(splitmix64(s) >> 11) + 1.0) * (1.0 / 9007199254740992.0);
}
static inline double gauss(uint64_t* s) {
    const double u1 = unif(s), u2 = unif(s);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

void sfmpo_gen_normal(float* out, size_t n, uint64_t seed, float mean, float std) {
    uint64_t s = seed * 0x2545F4914F6CDD1Dull + 1;
    for (size_t i = 0; i < n; ++i) out[i] = (float)(mean + std * gauss(&s));
}

void sfmpo_gen_salience(float* out, uint64_t rows, uint64_t cols, uint64_t seed) {
    uint64_t s = seed * 0x2545F4914F6CDD1Dull + 7;
    double* r = (double*)malloc(rows * sizeof(double));
    double* c = (double*)malloc(cols * sizeof(double));
    for (uint64_t i = 0; i < rows; ++i) r[i] = exp(gauss(&s));
    for (uint64_t j = 0; j < cols; ++j) c[j] = exp(gauss(&s));
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) out[i * cols + j] = (float)(r[i] * c[j] * -log(unif(&s)));
    free(r); free(c);
}

static float to_bf16(float f) { /* RNE to bf16, kept in f32 */
    uint32_t u = f2u(f);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return u2f(u & 0xFFFF0000u);
}

void sfmpo_gen_activation(float* out, size_t n, uint64_t seed) {
    uint64_t s = seed * 0x2545F4914F6CDD1Dull + 13;
    for (size_t i = 0; i < n; ++i) {
        float v = to_bf16((float)gauss(&s));
        if (fabsf(v) < 7.62939453125e-06f) v = 0.0f; /* 2^-17 */
        out[i] = v;
    }
}
