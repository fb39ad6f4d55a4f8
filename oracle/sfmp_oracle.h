/*
 * sfmp_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C99) of the reference SFMP algorithms on the
 * mixed-precision GEMM hot path, used as the parity checker for the CUDA
 * product library.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this; the product path
 * (paper_2602_01027_b200/) never does.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function below
 * against golden vectors produced by the unmodified reference compiled from
 * /root/reference/proj/src (oracle/ref_shim.cpp -> oracle/_ref/), and against
 * the spec's known-answer examples.
 *
 * Reference file:line anchors are relative to /root/reference/proj.
 */
#ifndef SFMP_ORACLE_H
#define SFMP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes mirror include/sfmp_cuda.h (and errors.hpp:9-36). */
enum {
    SFMPO_OK = 0,
    SFMPO_ERR_SHAPE = 1,
    SFMPO_ERR_CONFIG = 2,
    SFMPO_ERR_BAD_MAGIC = 3,
    SFMPO_ERR_BAD_VERSION = 4,
    SFMPO_ERR_TRUNCATED = 5,
    SFMPO_ERR_INVARIANT = 6,
    SFMPO_ERR_IO = 7,
    SFMPO_ERR_NOMEM = 11
};

/* fp16.hpp:14-56 / :58-83 */
uint16_t sfmpo_fp16_from_float(float f);
float sfmpo_fp16_to_float(uint16_t h);

/* Parsed SFMPPKD1 model (layout.cpp:210-279).  Block payloads are pointers
 * into the caller's byte buffer (not copied). */
typedef struct {
    uint16_t version;
    uint64_t rows, cols;
    uint32_t m_b, n_b;
    int floor_bits, ceil_bits;
    int mode; /* 0 none, 1 row, 2 col, 3 rowcol (reorder.hpp:25-30) */
    const uint32_t* row_perm; /* rows entries or NULL */
    const uint32_t* col_perm; /* cols entries or NULL */
    uint64_t K;
    const uint8_t* block_bits; /* K entries */
    uint64_t* block_off;       /* K offsets into the byte stream (malloc'd) */
    const uint8_t* base;
} sfmpo_model;

int sfmpo_parse(const uint8_t* bytes, size_t len, sfmpo_model* out);
void sfmpo_free(sfmpo_model* m);

/* compute_block_offsets (layout.cpp:301-314): offsets from the header alone. */
int sfmpo_block_offsets(const uint8_t* bytes, size_t len, uint64_t* out, uint64_t K);

/* unpack_block (layout.cpp:67-86) over the whole model: codes in REORDERED
 * order, row-major [rows x cols]. */
void sfmpo_unpack_codes(const sfmpo_model* m, uint8_t* codes);

/* dequantize_model (layout.cpp:316-332): dense f32 [rows x cols] in the
 * ORIGINAL row/col order (dequantize_group quantizer.cpp:50-55, then
 * apply_reorder_inverse reorder.cpp:95-101). */
void sfmpo_dequantize(const sfmpo_model* m, float* w);

/* matmul_reference (matrix.cpp:5-17), looped over M tokens:
 * y[t][i] = sum_k x[t][k] * w[i][k], f32, ascending k. */
void sfmpo_matmul_reference(const float* x, const float* w, float* y, int64_t M,
                            int64_t rows, int64_t cols);

/* Multithreaded variant for large shapes (row ranges, same per-row order,
 * bit-identical to the single-threaded result). */
void sfmpo_matmul_reference_mt(const float* x, const float* w, float* y, int64_t M,
                               int64_t rows, int64_t cols, int threads);

/* gemv (lutgemm.cpp:95-135): the reference LUT path incl. reorder in/out.
 * x: [cols], y: [rows].  lookups (may be NULL) receives GemvStats.lookups. */
int sfmpo_gemv_lut(const sfmpo_model* m, const float* x, float* y, uint64_t* lookups);

/* M tokens through gemv, token-parallel over `threads` host threads. */
int sfmpo_gemm_lut(const sfmpo_model* m, const float* x, float* y, int64_t M, int threads);

/* ---- fixture generation (offline path) ---- */

/* quantize_group (quantizer.cpp:11-48). */
int sfmpo_quantize_group(const float* v, size_t n, int bits, float* scale, float* zero,
                         uint8_t* codes);

/* Whole offline pipeline on caller-provided weights W and salience S
 * (both [rows x cols] f32): make_reorder_spec (reorder.cpp:50-62) ->
 * apply_reorder (:75-93) -> block_salience (salience.cpp:47-75) ->
 * make_bit_plan (allocation.cpp:31-49) -> allocate_block_bits (:85-103) ->
 * quantize_group per row-group -> pack_block (layout.cpp:29-65) ->
 * serialize (:179-208).  out==NULL queries the size into *out_len. */
int sfmpo_build_model(const float* W, const float* S, uint64_t rows, uint64_t cols,
                      uint32_t m_b, uint32_t n_b, double target_bpw, int mode,
                      uint8_t* out, size_t* out_len);

/* Deterministic synthetic inputs: splitmix64 + Box-Muller. */
void sfmpo_gen_normal(float* out, size_t n, uint64_t seed, float mean, float std);
/* S_ij = r_i * c_j * e_ij with r,c ~ LogNormal(0,1), e ~ Exp(1). */
void sfmpo_gen_salience(float* out, uint64_t rows, uint64_t cols, uint64_t seed);
/* x ~ N(0,1) rounded to bf16 (RNE), |x| < 2^-17 flushed to 0. */
void sfmpo_gen_activation(float* out, size_t n, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
