/*
 * sfmp_cuda.h -- C ABI of the B200-native (sm_100a) SFMP mixed-precision GEMM.
 *
 * This is the drop-in boundary for the reference's hot path
 *   sfmp::gemv(const PackedModel&, const Vector&, GemvStats*)   lutgemm.hpp:57
 * (definition lutgemm.cpp:95-135), together with the packed-model ingest it
 * depends on (deserialize layout.cpp:210-279, compute_block_offsets
 * layout.cpp:301-314) and the dequant oracle it is validated against
 * (dequantize_model layout.cpp:316-332).  Paths are relative to
 * /root/reference/proj.  Plain C: pointers, sizes and integer status codes;
 * no torch or C++ types cross this boundary.  A header-only C++ shim that
 * restores the reference's exception types is in include/sfmp/cuda.hpp.
 *
 * Semantics
 *  - Weights are ingested as the exact SFMPPKD1 bytes.  The
 *    block payload region is uploaded verbatim; no re-quantisation.
 *  - sfmp_gemm computes, for every token t < M,
 *        y[t] = gemv(model, x[t])          (M>1 loops the GEMV)
 *    i.e. y = x * dequantize_model(model)^T with x and y in the ORIGINAL
 *    column/row order: the col_perm gather (reorder_activation_in,
 *    reorder.cpp:103-111) and row_perm scatter (reorder_activation_out,
 *    reorder.cpp:113-121) happen inside the kernels.
 *  - Results are deterministic and independent of the parallel
 *    decomposition: every output element is summed in a
 *    canonical order fixed by the matrix shape alone (decode GEMV: fixed
 *    1024-column K segments added in segment order; prefill GEMM: fixed
 *    K chunks), so the bits do not depend on the grid, the SM count, the
 *    stream, the other problems of a grouped call, the shard count, or M.
 *    No floating-point atomics.
 *  - Everything is stream-ordered on the caller's stream.  Calls on distinct
 *    streams are safe when each passes its own workspace (or workspace=NULL
 *    is used from one stream at a time).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns SFMP_ERR_CUDA.
 */
#ifndef SFMP_CUDA_H
#define SFMP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFMP_CUDA_ABI_VERSION 2
#define SFMP_NCCL_ID_BYTES 128

/* Status codes, 1:1 with the reference exception kinds (errors.hpp:9-36). */
typedef enum sfmp_status {
    SFMP_OK = 0,
    SFMP_ERR_SHAPE = 1,               /* sfmp::ShapeError   (e.g. x.len != cols, lutgemm.cpp:96) */
    SFMP_ERR_CONFIG = 2,              /* sfmp::ConfigError  (e.g. reps < 1, lutgemm.cpp:138)     */
    SFMP_ERR_FORMAT_BAD_MAGIC = 3,    /* FormatError{bad_magic}   layout.cpp:216-217             */
    SFMP_ERR_FORMAT_BAD_VERSION = 4,  /* FormatError{bad_version} layout.cpp:220-222             */
    SFMP_ERR_FORMAT_TRUNCATED = 5,    /* FormatError{truncated}   layout.cpp:154-159             */
    SFMP_ERR_FORMAT_INVARIANT = 6,    /* FormatError{invariant}   layout.cpp:88-124, :229-275    */
    SFMP_ERR_FORMAT_IO = 7,           /* FormatError{io}          layout.cpp:281-299             */
    SFMP_ERR_CUDA = 8,                /* CUDA runtime / launch failure, or no sm_100 device      */
    SFMP_ERR_NCCL = 9,                /* collective failure (sharded path)                        */
    SFMP_ERR_INVALID_ARGUMENT = 10,   /* NULL pointer / bad enum                                  */
    SFMP_ERR_NOMEM = 11,              /* host or device allocation failed                         */
    SFMP_ERR_UNSUPPORTED = 12         /* valid request this build does not implement             */
} sfmp_status;

/* Activation element type.  Accumulation is always f32; y is always f32. */
typedef enum sfmp_dtype { SFMP_F32 = 0, SFMP_F16 = 1, SFMP_BF16 = 2 } sfmp_dtype;

/* Kernel selection (SFMP_PATH_AUTO picks by M: decode GEMV for M<=16,
 * tcgen05 GEMM for larger M). Forcing a path is for tests and benches. */
typedef enum sfmp_path {
    SFMP_PATH_AUTO = 0,
    SFMP_PATH_GEMV = 1,     /* K1: decode GEMV, M <= 16, HBM-bound            */
    SFMP_PATH_GEMM = 2,     /* K2: tcgen05/TMEM prefill GEMM                   */
    SFMP_PATH_GENERIC = 3,  /* any m_b/n_b/M; simple CUDA-core kernel          */
    SFMP_PATH_LUT = 4       /* the paper's LUT GEMV (lutgemm.cpp:11-71) on the GPU: a comparison
                               line, f32 x only, needs SFMP_MODEL_LUT_LAYOUT   */
} sfmp_path;

/* Opaque device-resident model (owns payload, offsets, perms, bit map). */
typedef struct sfmp_dev_model sfmp_dev_model;

/* Header / geometry summary (PackedModel fields, layout.hpp:36-53). */
typedef struct sfmp_model_info {
    uint64_t rows, cols;           /* m (output features), n (input features)            */
    uint32_t m_b, n_b;             /* block_rows, group_size                              */
    int32_t floor_bits, ceil_bits; /* candidate bit-widths                                */
    int32_t mode;                  /* ReorderMode: 0 none, 1 row, 2 col, 3 rowcol        */
    uint64_t block_count;          /* K = (m/m_b)(n/n_b)                                  */
    uint64_t blocks_high;          /* blocks at ceil_bits (when ceil != floor)            */
    double avg_code_bits;          /* sum_k bits_k / K                                    */
    uint64_t payload_bytes;        /* bytes of the block region (scales+zeros+planes)     */
    uint64_t device_bytes;         /* device memory of the weight layouts + indices (the
                                      model's default workspace is not counted)           */
    uint32_t shard, num_shards;    /* (0,1) for an unsharded model                        */
    uint64_t out_rows;             /* length of one output row of y written by sfmp_gemm  */
    uint64_t global_rows;          /* rows of the whole (unsharded) matrix                */
} sfmp_model_info;

/* A PackedModel (layout.hpp:36-53) given field by field.  plane_ptrs holds
 * sum_k block_bits[k] pointers in block order, planes least-significant
 * first, each m_b*n_b/8 bytes (PackedBlock::planes, layout.hpp:22-27). */
typedef struct sfmp_model_parts {
    uint64_t rows, cols;
    uint32_t m_b, n_b;
    int32_t floor_bits, ceil_bits, mode;
    const uint32_t* row_perm;           /* rows entries, NULL unless mode has row */
    const uint32_t* col_perm;           /* cols entries, NULL unless mode has col */
    const uint8_t* block_bits;          /* K entries                               */
    const uint16_t* const* scales;      /* K pointers, m_b fp16 payloads each      */
    const uint16_t* const* zeros;       /* K pointers, m_b fp16 payloads each      */
    const uint8_t* const* plane_ptrs;   /* sum(block_bits) pointers                */
} sfmp_model_parts;

/* ---- library ---------------------------------------------------------- */
int sfmp_abi_version(void);
const char* sfmp_status_string(sfmp_status s);
/* Message of the last failing call on this host thread ("" if none). */
const char* sfmp_last_error(void);
/* Number of usable sm_100 devices (0 on a host without a B200). */
int sfmp_device_count(void);

/* ---- host-only ingest (no device needed) -------------------------------- */
/* Full SFMPPKD1 validation (deserialize + PackedModel::validate). */
sfmp_status sfmp_parse_header(const uint8_t* bytes, size_t len, sfmp_model_info* info);
/* compute_block_offsets (layout.cpp:301-314): absolute byte offset of each
 * block in the serialized stream. */
sfmp_status sfmp_block_offsets(const uint8_t* bytes, size_t len, uint64_t* offsets,
                               uint64_t count);

/* ---- model lifetime ------------------------------------------------------ */
/* Ingest SFMPPKD1 bytes (read_packed_file/deserialize equivalent) onto `device`. */
sfmp_status sfmp_model_create(const uint8_t* bytes, size_t len, int device,
                              sfmp_dev_model** out);
/* Ingest an in-memory PackedModel (already validated by its owner). */
sfmp_status sfmp_model_create_from_parts(const sfmp_model_parts* parts, int device,
                                         sfmp_dev_model** out);
/* Ingest only the block rows owned by `shard` of `num_shards` under the snake
 * (boustrophedon) block-row partition.  The shard's
 * sfmp_gemm writes y_local[M][out_rows] in shard-local reordered row order;
 * sfmp_unpermute_gathered() turns the all-gathered shards into y. */
/* Host-only shard plan: gather_map[num_shards*shard_rows] maps (shard g,
 * local row i) to the ORIGINAL output row (0xFFFFFFFF for padding);
 * *shard_rows receives the per-shard row count (padded to the largest). Pass
 * gather_map=NULL to query *shard_rows only. */
sfmp_status sfmp_shard_plan(const uint8_t* bytes, size_t len, uint32_t num_shards,
                            uint32_t* gather_map, uint64_t* shard_rows);
/* Host-only: the shard's block rows as a stand-alone SFMPPKD1 stream (rows in
 * shard-local order, so the row permutation is dropped; col_perm kept).  Its
 * gemv equals the shard's sfmp_gemm output without padding.  Pass out=NULL to
 * query *out_len. */
sfmp_status sfmp_shard_extract(const uint8_t* bytes, size_t len, uint32_t shard, uint32_t num_shards,
                               uint8_t* out, size_t* out_len);
sfmp_status sfmp_model_create_shard(const uint8_t* bytes, size_t len, int device,
                                    uint32_t shard, uint32_t num_shards, sfmp_dev_model** out);
/* Model creation flags.  Default (0): both device layouts -- the decode
 * GEMV's unit-major layout and the prefill GEMM's row-tile layout (~2x the
 * SFMPPKD1 payload).  SFMP_MODEL_DECODE_ONLY keeps only the decode layout
 * (~1.0x): M > 16 then runs the decode GEMV in 16-token chunks. */
#define SFMP_MODEL_DECODE_ONLY 1u
/* Also keep the SFMPPKD1 block payloads as stored, for SFMP_PATH_LUT. */
#define SFMP_MODEL_LUT_LAYOUT 2u
sfmp_status sfmp_model_create_ex(const uint8_t* bytes, size_t len, int device, uint32_t flags,
                                 sfmp_dev_model** out);
sfmp_status sfmp_model_create_shard_ex(const uint8_t* bytes, size_t len, int device, uint32_t shard,
                                       uint32_t num_shards, uint32_t flags, sfmp_dev_model** out);
sfmp_status sfmp_model_destroy(sfmp_dev_model* model);
sfmp_status sfmp_model_get_info(const sfmp_dev_model* model, sfmp_model_info* info);

/* ---- compute (device pointers, stream-ordered) ------------------------- */
/* Bytes of scratch sfmp_gemm needs for this M (0 if none).  A workspace must
 * be zero-filled once before its first use; every call leaves it re-zeroed
 * (it holds the grid-wide completion counters of the decode GEMV). */
sfmp_status sfmp_workspace_size(const sfmp_dev_model* model, int64_t M, sfmp_path path,
                                size_t* bytes);
/* y[M][out_rows] (f32) = x[M][cols] (dtype) . W^T.  workspace may be NULL
 * (the model's own scratch is used; then calls must not overlap). */
sfmp_status sfmp_gemm(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M,
                      float* y, void* workspace, size_t workspace_bytes, void* stream);
sfmp_status sfmp_gemm_ex(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype,
                         int64_t M, float* y, void* workspace, size_t workspace_bytes,
                         sfmp_path path, void* stream);
/* Several independent linears (e.g. the q/k/v/o/gate/up/down of a decoder
 * layer, each with its own x) in one call.  For M <= 16 consecutive models
 * with the same n_b and floor bits share ONE activation pre-pass and ONE GEMV
 * launch, so launch and first-byte latencies are paid once per group; other
 * cases run model by model.  workspaces[i] as for sfmp_gemm on models[i]
 * (required for the decode path); workspace_bytes may be NULL. */
sfmp_status sfmp_gemm_grouped(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                              int64_t M, float* const* ys, void* const* workspaces, const size_t* workspace_bytes,
                              int count, void* stream);
/* Same with a token count per problem (Ms[i] rows of xs[i] / ys[i]), e.g. the
 * experts of a mixture-of-experts layer.  Consecutive decode problems (M <= 16)
 * that are groupable, fall in the same class (M <= 8 or 9..16) and use distinct
 * workspaces share one launch (up to 40 per launch).  The problems of one call
 * must be independent (no ys[i] aliasing an xs[j]): a later launch of the call
 * may start while an earlier one finishes. */
sfmp_status sfmp_gemm_grouped_v(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                                const int64_t* Ms, float* const* ys, void* const* workspaces,
                                const size_t* workspace_bytes, int count, void* stream);
/* RMSNorm fused into the activation pre-pass (the "fused activation producer"
 * of SURVEY §8(f)1): x is the UNNORMALISED hidden state h and the GEMM uses
 *     x[t][j] = h[t][j] / sqrt(mean_j h[t][j]^2 + eps) * gamma[j]   (f32)
 * (the Llama pre-attention / pre-MLP norm).  The pre-pass already stages
 * every token row to gather it by col_perm, so the norm costs no extra pass
 * over x.  gamma = NULL means 1.  SFMP_ERR_UNSUPPORTED for the generic path
 * and for rows too wide for the staged decode pre-pass (> 192 KB). */
typedef struct sfmp_prenorm {
    const void* gamma;       /* [cols] device pointer, or NULL */
    sfmp_dtype gamma_dtype;
    float eps;
    int32_t enabled;         /* 0: x is used as given (lets a grouped call mix normed and plain inputs) */
} sfmp_prenorm;
sfmp_status sfmp_gemm_norm(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M, float* y,
                           void* workspace, size_t workspace_bytes, const sfmp_prenorm* norm, void* stream);
/* sfmp_gemm_grouped_v with one norm per problem (norms[count]). */
sfmp_status sfmp_gemm_grouped_v_norm(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                                     const int64_t* Ms, float* const* ys, void* const* workspaces,
                                     const size_t* workspace_bytes, int count, const sfmp_prenorm* norms,
                                     void* stream);
/* Host-buffer convenience with the reference's calling convention: x and y
 * are HOST arrays; copies, kernel and synchronisation happen inside. */
sfmp_status sfmp_gemm_host(const sfmp_dev_model* model, const float* x_host, int64_t M,
                           float* y_host, void* stream);

/* ---- call statistics (GemvStats, lutgemm.hpp:47-52; filled at lutgemm.cpp:127-132) ---- */
typedef struct sfmp_stats {
    double device_us;       /* kernel time of the call on its stream (CUDA events)              */
    double h2d_us, d2h_us;  /* host-buffer entry only: copy times (CUDA events)                 */
    double wall_us;         /* host wall-clock time of the whole call                           */
    uint64_t bytes;         /* algorithmic HBM bytes: planes + s,z + perms + x + y  */
    double flops;           /* 2 * M * rows * cols                                              */
    int32_t path;           /* kernel path taken (sfmp_path)                                     */
    int32_t launches;       /* kernels the call enqueued                                         */
} sfmp_stats;
/* sfmp_gemm_ex that also fills *stats; with stats != NULL the call
 * synchronises its stream (as the reference's GemvStats timing is blocking). */
sfmp_status sfmp_gemm_stats(const sfmp_dev_model* model, const void* x, sfmp_dtype dtype, int64_t M,
                            float* y, void* workspace, size_t workspace_bytes, sfmp_path path,
                            void* stream, sfmp_stats* stats);
/* sfmp_gemm_host that also fills *stats (NULL allowed). */
sfmp_status sfmp_gemm_host_stats(const sfmp_dev_model* model, const float* x_host, int64_t M,
                                 float* y_host, void* stream, sfmp_stats* stats);
/* Kernels enqueued by this host thread so far (every entry point counts its
 * launches; a CUDA-graph capture counts the captured launches once). */
uint64_t sfmp_launch_count(void);

/* gemv_block (lutgemm.hpp:44-45, lutgemm.cpp:87-93): out[m_b] = the
 * contribution of block k (block-row-major, as PackedModel::blocks) to its
 * m_b rows in STORED row order, from the REORDERED activation x_reordered
 * (device f32, cols entries: x[col_perm[j]], reorder.cpp:103-111). */
sfmp_status sfmp_gemv_block(const sfmp_dev_model* model, uint64_t block, const float* x_reordered,
                            float* out, void* stream);

/* K3 (debug/parity): dense f32 W[rows][cols] in ORIGINAL order, bit-exact
 * with dequantize_model (layout.cpp:316-332; quantizer.cpp:50-55). */
sfmp_status sfmp_dequantize(const sfmp_dev_model* model, float* w, void* stream);
/* Integer codes [rows][cols] in REORDERED (stored) order, bit-exact with
 * unpack_block (layout.cpp:67-86). */
sfmp_status sfmp_unpack_codes(const sfmp_dev_model* model, uint8_t* codes, void* stream);

/* ---- sharded output assembly (multi-GPU) ---------------------- */
/* gathered: [num_shards][M][shard_rows] f32 as produced by an all-gather of
 * each shard's y_local.  Writes y[M][rows] in ORIGINAL row order.  `model`
 * may be any shard of the same matrix (all shards carry the global map). */
sfmp_status sfmp_unpermute_gathered(const sfmp_dev_model* model, const float* gathered,
                                    int64_t M, float* y, void* stream);

/* ---- sharded calls: many problems, ONE collective -------- */
/* models[i] are shards (sfmp_model_create_shard) with the same shard index and
 * count on one device; problem i has Ms[i] tokens.  Each rank writes its
 * problems' shard outputs y_local[Ms[i]][shard_rows_i] back to back into the
 * send block of gather_buf; an all-gather of that block (total floats) into
 * the receive block that follows it ([num_shards][total]) gives every rank
 * every row; one kernel scatters them to ys[i][Ms[i]][global rows] in the
 * ORIGINAL row order.  Bit-identical to the unsharded sfmp_gemm. */
/* Bytes of gather_buf: (1 + num_shards) * sum_i Ms[i] * shard_rows_i * 4. */
sfmp_status sfmp_sharded_gather_bytes(const sfmp_dev_model* const* models, const int64_t* Ms, int count,
                                      size_t* bytes);
/* Step 1: the shard GEMMs into the send block (one grouped call). */
sfmp_status sfmp_gemm_sharded_local(const sfmp_dev_model* const* models, const void* const* xs,
                                    sfmp_dtype dtype, const int64_t* Ms, void* const* workspaces,
                                    const size_t* workspace_bytes, int count, void* gather_buf,
                                    void* stream);
/* Step 3 (after the caller's all-gather of the send block into the receive
 * block): scatter every problem's rows to ys in original order (one launch). */
sfmp_status sfmp_sharded_unpermute(const sfmp_dev_model* const* models, const int64_t* Ms, int count,
                                   const void* gather_buf, float* const* ys, void* stream);
/* Steps 1-3 with NCCL: nccl_comm is an ncclComm_t whose size/rank equal the
 * shard count/index.  NCCL failures return SFMP_ERR_NCCL.  Stream-ordered and
 * CUDA-graph capturable. */
sfmp_status sfmp_gemm_sharded(const sfmp_dev_model* const* models, const void* const* xs, sfmp_dtype dtype,
                              const int64_t* Ms, float* const* ys, void* const* workspaces,
                              const size_t* workspace_bytes, int count, void* gather_buf,
                              size_t gather_bytes, void* nccl_comm, void* stream);
/* NCCL helpers for callers without a communicator (libnccl.so.2 is loaded at
 * run time; in a PyTorch process that is torch's NCCL). id: SFMP_NCCL_ID_BYTES. */
sfmp_status sfmp_nccl_unique_id(uint8_t* id);
sfmp_status sfmp_nccl_comm_init(int nranks, const uint8_t* id, int rank, int device, void** comm);
sfmp_status sfmp_nccl_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* SFMP_CUDA_H */
