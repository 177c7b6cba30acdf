/*
 * anyq_b200.h — C-ABI of the B200-native any4 quantize + LUT-GEMM path.
 *
 * This is the drop-in boundary for the reference library `anyq`
 * (/root/reference/proj). The reference has no FFI of its own: its boundary is
 * the C++ headers proj/include/anyq/{core,learner,pack,quantize,qgemm}.hpp.
 * Every entry point below replaces one of those functions (cited per entry)
 * with the same argument meaning and the same error classes (returned as
 * anyq_status, see core.hpp:27-74). All compute runs on the GPU; there is no
 * CPU fallback. The library fails with ANYQ_ERR_CUDA when no device is usable.
 *
 * Two call styles:
 *   - anyq_*      : host buffers in, host buffers out (value semantics, like
 *                   the reference). H2D/D2H staging happens inside the call.
 *   - anyq_dev_*  : device pointers + cudaStream_t (passed as void*), stream
 *                   ordered, no host synchronisation; used for timed paths.
 *
 * Layout conventions follow the reference exactly: row-major fp32 matrices,
 * packed codes little-end-first with rows padded to a byte boundary
 * (pack.hpp:45-51), one LUT of 2^bits fp32 values per row (pack.hpp:27),
 * group scales indexed by ScaleSet::group_of (scaling.hpp:36-45).
 */
#ifndef ANYQ_B200_H
#define ANYQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; one per exception class of core.hpp:27-74. */
typedef enum anyq_status {
  ANYQ_OK = 0,
  ANYQ_ERR_SHAPE = 1,       /* ShapeError */
  ANYQ_ERR_CONFIG = 2,      /* ConfigError */
  ANYQ_ERR_CODE_RANGE = 3,  /* CodeRangeError */
  ANYQ_ERR_NONFINITE = 4,   /* NonFiniteError */
  ANYQ_ERR_STATS = 5,       /* StatsError */
  ANYQ_ERR_IO = 6,          /* IoError */
  ANYQ_ERR_MAGIC = 7,       /* MagicError */
  ANYQ_ERR_VERSION = 8,     /* VersionError */
  ANYQ_ERR_TRUNCATED = 9,   /* TruncatedError */
  ANYQ_ERR_INVARIANT = 10,  /* InvariantError */
  ANYQ_ERR_INTERNAL = 11,   /* anyq::Error (internal assertion) */
  ANYQ_ERR_CUDA = 12,       /* device / driver failure (no reference twin) */
} anyq_status;

/* Message of the last error raised on the calling thread ("" if none). */
const char* anyq_last_error(void);

/* Enums mirror core.hpp:78-96 and pack.hpp:17-19 value for value. */
enum { ANYQ_CB_INT = 0, ANYQ_CB_FP4 = 1, ANYQ_CB_NF4 = 2, ANYQ_CB_ANY = 3 };
enum {
  ANYQ_G_TENSOR = 0,
  ANYQ_G_ROW = 1,
  ANYQ_G_COLUMN = 2,
  ANYQ_G_GROUP = 3,
  ANYQ_G_BLOCK = 4
};
enum { ANYQ_INIT_KMPP = 0, ANYQ_INIT_RANDOM = 1, ANYQ_INIT_GRID = 2, ANYQ_INIT_NF4 = 3 };
enum { ANYQ_W_WEIGHTS = 0, ANYQ_W_ACTS = 1, ANYQ_W_FULL = 2 };
enum { ANYQ_LAYOUT_ROWMAJOR = 0, ANYQ_LAYOUT_KTILED = 1 };
enum { ANYQ_STORE_FP16 = 0, ANYQ_STORE_BF16 = 1, ANYQ_STORE_FP32 = 2 };

/* QuantConfig + LearnerConfig (core.hpp:98-121), flattened. */
typedef struct anyq_config {
  int32_t bits;               /* 2,3,4,8 */
  int32_t codebook;           /* ANYQ_CB_* */
  int32_t granularity;        /* ANYQ_G_* */
  int32_t group_size;
  int32_t block_size;
  int32_t symmetric;
  int32_t int_range_shifted;
  int32_t init;               /* ANYQ_INIT_* */
  int32_t max_iters;
  float rel_tol;
  int32_t restarts;
  int32_t weighting;          /* ANYQ_W_* */
  int32_t check_invariants;
  int32_t reserved;
  uint64_t seed;
} anyq_config;

/* Defaults of core.hpp:98-121 (IntGrid, 4 bits, groupwise 128, kmeans++...). */
void anyq_config_default(anyq_config* cfg);

/* QuantizedTensor (pack.hpp:21-39) as flat host arrays. */
typedef struct anyq_qtensor {
  int64_t rows, cols;
  anyq_config cfg;
  int32_t layout;      /* ANYQ_LAYOUT_* */
  int32_t tile_k;
  int32_t lut_store;   /* ANYQ_STORE_* */
  int32_t scale_store; /* ANYQ_STORE_* */
  uint8_t* codes;      /* rows * packed_bytes_per_row(cols, bits) */
  float* luts;         /* rows * 2^bits for ANYQ_CB_ANY, else NULL */
  float* alphas;       /* num_groups */
  float* betas;        /* num_groups */
  int64_t num_groups;
} anyq_qtensor;

/* Sizes the caller must allocate for an anyq_qtensor of this shape/config. */
int64_t anyq_packed_bytes_per_row(int64_t cols, int32_t bits); /* pack.hpp:45 */
int64_t anyq_num_groups(const anyq_config* cfg, int64_t rows, int64_t cols);
int64_t anyq_lut_entries(const anyq_config* cfg);

/* ---------------------------------------------------------------------------
 * Quantization (host buffers)
 * ------------------------------------------------------------------------- */

/* learner.hpp:74 quantize_any(w, cfg, exj, threads). exj may be NULL.
 * `row_offset` is added to the local row index when keying the per-row RNG
 * (rng_for_row(seed, row_offset + i)); pass 0 for reference semantics on a
 * whole matrix, or the first global row when a matrix is split across GPUs.
 * out must have codes/luts/alphas/betas allocated with the sizes above. */
anyq_status anyq_quantize_any(const float* w, int64_t rows, int64_t cols,
                              const anyq_config* cfg, const float* exj,
                              int64_t row_offset, anyq_qtensor* out);

/* quantize.hpp:17 quantize_fixed(w, cfg): RTN onto int/fp4/nf4 tables. */
anyq_status anyq_quantize_fixed(const float* w, int64_t rows, int64_t cols,
                                const anyq_config* cfg, anyq_qtensor* out);

/* ---------------------------------------------------------------------------
 * Packing / layout / dequant (host buffers, computed on device)
 * ------------------------------------------------------------------------- */

/* pack.hpp:50 pack_codes / pack.hpp:51 unpack_codes. */
anyq_status anyq_pack_codes(const uint8_t* codes, int64_t rows, int64_t cols,
                            int32_t bits, uint8_t* packed);
anyq_status anyq_unpack_codes(const uint8_t* packed, int64_t rows, int64_t cols,
                              int32_t bits, uint8_t* codes);

/* pack.hpp:86-87 to_ktiled / from_ktiled on the packed codes of a tensor. */
anyq_status anyq_ktile_codes(const uint8_t* packed, int64_t rows, int64_t cols,
                             int32_t bits, int32_t tile_k, int32_t inverse,
                             uint8_t* out);

/* pack.hpp:68 narrowed(qt): LUT/scales rounded to their 16-bit stores and
 * widened back, in place on the host arrays of qt. */
anyq_status anyq_narrow_inplace(anyq_qtensor* qt);

/* pack.hpp:98 dequantize(qt) -> rows x cols fp32. */
anyq_status anyq_dequantize(const anyq_qtensor* qt, float* w_out);

/* ---------------------------------------------------------------------------
 * Scaling (host buffers). Group map: cfg->granularity / group_size / block_size
 * (ScaleSet::group_of, scaling.hpp:36-45); alphas/betas hold num_groups entries.
 * ------------------------------------------------------------------------- */
/* scaling.hpp:52 compute_scales(w, cfg, qmin, qmax): per-group min/max -> alpha, beta. */
anyq_status anyq_compute_scales(const float* w, int64_t rows, int64_t cols, const anyq_config* cfg,
                                float qmin, float qmax, float* alphas, float* betas);
/* scaling.hpp:56 scale_weights(w, s): ws = (w - beta_g) / alpha_g. */
anyq_status anyq_scale_weights(const float* w, int64_t rows, int64_t cols, const anyq_config* cfg,
                               const float* alphas, const float* betas, float* ws);
/* scaling.hpp:60 dequantize(values, s): out = alpha_g * v + beta_g. */
anyq_status anyq_dequantize_values(const float* v, int64_t rows, int64_t cols,
                                   const anyq_config* cfg, const float* alphas,
                                   const float* betas, float* out);

/* calibration.cpp:62-67, the per-layer statistic of collect_stats
 * (calibration.hpp:43): exj[j] = float(sum_{m in order} |double(x[m][j])| / M)
 * over the M x K row-major activations x, bit-identical to the reference.
 * ShapeError when M < 1, NonFiniteError on NaN/Inf inputs (require_finite). */
anyq_status anyq_column_mean_abs(const float* x, int64_t m, int64_t k, float* exj);

/* eval.cpp:11-29 weight_error(w, qt) -> (mse, relative Frobenius error) and
 * eval.cpp:31-46 output_error(w, qt, x) -> mean squared output error of
 * gemm_reference(x, qt) against gemm_dense(x, w). Both GEMMs and the
 * dequantisation are the bit-identical device paths; the double sums are a
 * deterministic tree (equal to the reference's sequential sums up to
 * reassociation). ShapeError on mismatched shapes, CodeRangeError from
 * dequantize. */
anyq_status anyq_weight_error(const float* w, int64_t rows, int64_t cols, const anyq_qtensor* qt,
                              double* mse, double* rel);
anyq_status anyq_output_error(const float* w, int64_t rows, int64_t cols, const anyq_qtensor* qt,
                              const float* x, int64_t m, int64_t x_cols, double* mse);

/* eval.cpp:48-61 eval_activations(rows, cols, exj, seed): channel j drawn from
 * N(0, E|x_j| sqrt(pi/2)) (standard normal when exj is NULL), row r from
 * rng_for_row(seed, r) (Box-Muller in double on the host, like the reference:
 * synthetic data is not generated on the device). out: rows x cols fp32. */
anyq_status anyq_eval_activations(int64_t rows, int64_t cols, const float* exj, uint64_t seed,
                                  float* out);

/* eval.cpp:62-86 compare_formats(w, formats, base, stats, module, opts):
 * `formats` comma-separated names of quantize.cpp:34-54; exj = the module's
 * E|x_j| (NULL = no stats); eval_rows / eval_seed = CompareOptions. Per
 * format i, out[4i..4i+3] = weight_mse, weight_rel_frobenius, output_mse,
 * bits_per_entry. Quantization, dequantization and both GEMMs of the errors
 * run on the GPU; n_formats receives the row count. */
anyq_status anyq_compare_formats(const float* w, int64_t rows, int64_t cols, const char* formats,
                                 const anyq_config* base, const float* exj, int64_t eval_rows,
                                 uint64_t eval_seed, double* out, int32_t* n_formats);

/* ANYQ v1 files (pack.hpp write_file / read_file, pack.cpp:293-471).
 * anyq_write_file is byte-identical to write_file (lut_store / scale_store of
 * qt choose the stored precision). anyq_read_file_header parses and validates
 * the header and section table and fills the scalar fields of hdr (rows, cols,
 * cfg, layout, tile_k, stores, num_groups; LUT entries = anyq_lut_entries);
 * the caller then allocates the arrays and calls anyq_read_file, which runs
 * every check of read_file in its order (MagicError, VersionError,
 * TruncatedError, InvariantError, CodeRangeError). Host only: no device. */
anyq_status anyq_write_file(const anyq_qtensor* qt, const char* path);
anyq_status anyq_read_file_header(const char* path, anyq_qtensor* hdr);
anyq_status anyq_read_file(const char* path, anyq_qtensor* qt);

/* ---------------------------------------------------------------------------
 * GEMM (host buffers)
 * ------------------------------------------------------------------------- */

/* qgemm.hpp:36 gemm_fused(x, qt, plan): y[m x rows] = x[m x cols] * W^T with
 * W = dequant(qt). Reduction over k ascending in fp32 exactly as the
 * reference, so the result is bit-identical to gemm_fused / gemm_reference.
 * plan_layout/plan_tile_k reproduce GemmPlan's layout check (qgemm.cpp:75). */
anyq_status anyq_gemm_fused(const float* x, int64_t m, const anyq_qtensor* qt,
                            int32_t plan_layout, int32_t plan_tile_k, float* y);

/* qgemm.hpp:28 gemm_dense(x, w). */
anyq_status anyq_gemm_dense(const float* x, int64_t m, const float* w, int64_t n,
                            int64_t k, float* y);

/* ---------------------------------------------------------------------------
 * Device-resident path (timed). All pointers are device pointers; `stream`
 * is a cudaStream_t. Calls are asynchronous and stream ordered.
 * ------------------------------------------------------------------------- */

/* Opaque prepacked weight tensor living in HBM (codes in the fragment-
 * ordered tile layout, LUT + alpha/beta narrowed to fp16). */
typedef struct anyq_dev_tensor anyq_dev_tensor;

/* Build a device tensor from a host QuantizedTensor (narrowing the LUT and
 * scales to fp16 exactly like narrowed(); pack.cpp:159-169). */
anyq_status anyq_dev_tensor_create(const anyq_qtensor* qt, anyq_dev_tensor** out);
void anyq_dev_tensor_destroy(anyq_dev_tensor* t);
/* The inverse of the prepack: the device tensor back in the reference layout
 * (pack.hpp:21-39; row-major codes packed at cfg.bits, LUT and alpha/beta as
 * the fp32 values of their fp16 stores, i.e. narrowed(qt) of the tensor it was
 * created from). out sized like any anyq_qtensor of (rows, cols, cfg). */
anyq_status anyq_dev_tensor_export(const anyq_dev_tensor* t, anyq_qtensor* out);
/* The config a device tensor was created (or loaded) from. */
void anyq_dev_tensor_config(const anyq_dev_tensor* t, anyq_config* out);
/* Bytes the GEMM must stream per call (codes + scales + LUT). */
int64_t anyq_dev_tensor_weight_bytes(const anyq_dev_tensor* t);
int64_t anyq_dev_tensor_rows(const anyq_dev_tensor* t);
int64_t anyq_dev_tensor_cols(const anyq_dev_tensor* t);

/* y[m x rows] (bf16) = x[m x cols] (bf16) * dequant(W)^T (fp32 accumulation),
 * any m >= 1; the kernel is chosen by m (ANYQ_PATH_AUTO below). y_f32 may be
 * NULL. Device pointers. */
anyq_status anyq_dev_gemm_bf16(const anyq_dev_tensor* t, const void* x_bf16,
                               int64_t m, void* y_bf16, float* y_f32,
                               void* stream);

/* Same, with the kernel chosen explicitly (tests and the M sweep):
 *   ANYQ_PATH_GEMV  CUDA-core LUT GEMV, m <= 4 (gemv.cu)
 *   ANYQ_PATH_TC    tensor-core (tcgen05, A in TMEM) LUT GEMM, m <= 16
 *   ANYQ_PATH_DEQUANT  bf16 dequantization + cuBLAS GEMM, any m (large-M path)
 *   ANYQ_PATH_MMA   fused dequant-to-shared-memory + mma.sync, m <= 64 (lutmma.cu)
 *   ANYQ_PATH_GEMV_TC  K1t: the persistent GEMV chain with the products on
 *                   tcgen05 (pair-table lookups -> TMEM A operand), m <= 16 (gemv.cu)
 *   ANYQ_PATH_K2    large M: dequantise to bf16 in shared memory, tcgen05
 *                   (A and B from shared memory, x by TMA), lutgemm2.cu
 *   ANYQ_PATH_AUTO  GEMV for m <= 4 when its shared-memory plan fits (else
 *                   tcgen05), fused mma for 5 <= m <= 32, dequant above
 *                   (measured crossovers; what anyq_dev_gemm_bf16 uses) */
enum { ANYQ_PATH_AUTO = 0, ANYQ_PATH_GEMV = 1, ANYQ_PATH_TC = 2, ANYQ_PATH_DEQUANT = 3, ANYQ_PATH_MMA = 4,
       ANYQ_PATH_GEMV_TC = 5, ANYQ_PATH_K2 = 6 };
anyq_status anyq_dev_gemm_bf16_path(const anyq_dev_tensor* t, const void* x_bf16, int64_t m,
                                    void* y_bf16, float* y_f32, int32_t path, void* stream);
/* The path ANYQ_PATH_AUTO takes for this tensor at m rows of x. */
int32_t anyq_dev_gemm_auto_path(const anyq_dev_tensor* t, int64_t m);

/* A chain of small-M GEMMs in ONE persistent launch (e.g. the projections of a
 * decoder layer): y_i[m x rows_i] = x_i[m x cols_i] * dequant(W_i)^T for
 * i < n (n <= 8, the same 1 <= m <= 4 for all; CUDA-core GEMV path). Problem
 * i > 0 with wait_prev[i] != 0 reads x_i only after every earlier problem has
 * completed grid-wide, so x_i may be (or depend on) an earlier y_j; the
 * weights of later problems stream in while it waits. y32 may be NULL (or any
 * entry of it). A tensor may appear once per chain. */
anyq_status anyq_dev_gemm_chain(int32_t n, const anyq_dev_tensor* const* t,
                                const void* const* x_bf16, void* const* y_bf16,
                                float* const* y_f32, const int32_t* wait_prev, int64_t m,
                                void* stream);
/* Same, with one dependency per problem: deps[i] = index of the earlier
 * problem whose y problem i reads as its x (it starts once every CTA finished
 * that problem), or -1. Independent problems (e.g. k/v next to o in a decoder
 * layer) run while others wait. */
anyq_status anyq_dev_gemm_chain_deps(int32_t n, const anyq_dev_tensor* const* t,
                                     const void* const* x_bf16, void* const* y_bf16,
                                     float* const* y_f32, const int32_t* deps, int64_t m,
                                     void* stream);

/* Same, with the chain engine chosen explicitly: ANYQ_PATH_GEMV (CUDA-core,
 * m <= 4), ANYQ_PATH_GEMV_TC (tcgen05, m <= 16) or ANYQ_PATH_AUTO (what
 * anyq_dev_gemm_chain_deps uses). */
anyq_status anyq_dev_gemm_chain_path(int32_t n, const anyq_dev_tensor* const* t,
                                     const void* const* x_bf16, void* const* y_bf16,
                                     float* const* y_f32, const int32_t* deps, int64_t m,
                                     int32_t path, void* stream);

/* ---------------------------------------------------------------------------
 * Tensor parallelism: W sharded by output rows over `world`
 * ranks (one GPU each); y is all-gathered. The gather is fused into the GEMV
 * writer: every y value of this rank's shard is stored straight into every
 * rank's full-width y buffer (NVLink peer stores to buffers mapped with
 * anyq_ipc_open), and each CTA then bumps flags[r][rank] on every rank r
 * (system-scope release). anyq_dev_tp_wait makes `stream` wait until every
 * rank's contribution of call number `epoch` (1, 2, ...) has landed here.
 * ------------------------------------------------------------------------- */
typedef struct anyq_tp_peers {
  int32_t world;        /* ranks, 1..8 */
  int32_t rank;         /* this rank */
  int64_t rows_total;   /* rows of the unsharded weight (= columns of y) */
  int64_t row0;         /* first row of this rank's shard */
  void* y[8];           /* every rank's y (bf16, m x rows_total), valid on this device */
  int32_t* flags[8];    /* every rank's flag words (int32[world], zero at start), valid here */
} anyq_tp_peers;
anyq_status anyq_dev_gemm_allgather(const anyq_dev_tensor* shard, const void* x_bf16, int64_t m,
                                    const anyq_tp_peers* tp, void* stream);
anyq_status anyq_dev_tp_wait(const anyq_dev_tensor* shard, const anyq_tp_peers* tp, int32_t epoch,
                             void* stream);
/* CUDA IPC for the peer buffers: a 64-byte handle of a device allocation, and
 * its mapping in another process (close with anyq_ipc_close). */
anyq_status anyq_ipc_handle(const void* dev_ptr, uint8_t handle[64]);
anyq_status anyq_ipc_open(const uint8_t handle[64], void** dev_ptr);
anyq_status anyq_ipc_close(void* dev_ptr);

/* read_file straight into the prepacked device layout. */
anyq_status anyq_dev_tensor_load(const char* path, anyq_dev_tensor** out);

/* Device quantize: rows [row_offset, row_offset+rows) of a matrix, fp32 in,
 * reference-layout outputs (packed codes, fp32 LUT/alpha/beta) on device.
 * Fully stream ordered (no host synchronisation; capturable into a CUDA
 * graph). Argument/config errors return at once; the data checks of the
 * reference (require_finite: NonFiniteError, the stats and KmProblem weight
 * checks: StatsError) run on the device and are reported by
 * anyq_dev_stream_status(stream). */
anyq_status anyq_dev_quantize_any(const float* w_dev, int64_t rows, int64_t cols,
                                  const anyq_config* cfg, const float* exj_dev,
                                  int64_t row_offset, uint8_t* codes_dev,
                                  float* luts_dev, float* alphas_dev,
                                  float* betas_dev, void* stream);

/* Synchronises `stream` and returns the first data error recorded on the
 * device by the stream-ordered entries issued on it since the last call (in
 * the reference's check order), clearing it; ANYQ_OK if none. */
anyq_status anyq_dev_stream_status(void* stream);

/* anyq_column_mean_abs on device buffers, stream ordered; a non-finite input
 * is reported by anyq_dev_stream_status. */
anyq_status anyq_dev_column_mean_abs(const float* x_dev, int64_t m, int64_t k, float* exj_dev,
                                     void* stream);

/* ---------------------------------------------------------------------------
 * The per-row learner API, codebooks, scalar narrowing, accounting (host
 * buffers). With these the C++ drop-in (host/anyq_host.cpp) serves every
 * function of the reference's hot-path headers from this library.
 * ------------------------------------------------------------------------- */

/* learner.hpp:55 kmeans_pp_init (mode 2), learner.hpp:61 weighted_kmeans
 * (mode 1) and learner.hpp:66 learn_row_lut (mode 0: centroids = the sorted
 * LUT widened to double, assignments = the rank-remapped codes, loss) on the
 * GPU, for `rows` independent KmProblems of n samples each
 * (samples / weights row-major). rng_key[r], rng_counter[r] are problem r's
 * Rng state (core.hpp:164-192); the counter is advanced in place exactly as
 * the reference advances its Rng&. Every reduction runs in the reference's
 * sample-index order, so results are bit-identical by construction.
 * Outputs: centroids [rows][k] (learner order, double); mode 1 also
 * assignments [rows][n] (centroid indices), loss [rows], iters [rows].
 * cfg supplies the LearnerConfig fields (init, max_iters, rel_tol, restarts).
 * Errors as KmProblem::validate + the k checks (learner.cpp:11-23, 133, 318-319). */
anyq_status anyq_kmeans_problems(const float* samples, const float* weights, int64_t rows,
                                 int64_t n, int32_t k, const anyq_config* cfg, int32_t mode,
                                 const uint64_t* rng_key, uint64_t* rng_counter,
                                 double* centroids, uint8_t* assignments, double* loss,
                                 int32_t* iters);

/* learner.hpp:45 build_sample_weights(s, row, stats, mode) for the scale set
 * (cfg granularity, rows x cols, alphas[num_groups]); stats may be NULL
 * (E|x_j| = 1). StatsError on a stats length mismatch or a negative /
 * non-finite entry (learner.cpp:27-34). out: cols floats. */
anyq_status anyq_build_sample_weights(const anyq_config* cfg, int64_t rows, int64_t cols,
                                      const float* alphas, int64_t num_groups, int64_t row,
                                      const float* stats, int64_t stats_len, int32_t weighting,
                                      float* out);

/* codebooks.hpp:44 round_to_codebook(ws, cb): nearest of the n sorted table
 * values, ties to the smaller index (NonFiniteError on non-finite ws). */
anyq_status anyq_round_to_table(const float* ws, int64_t rows, int64_t cols, const float* table,
                                int32_t n, uint8_t* codes);

/* pack.hpp:95 scaled_values(qt): the table value of every code (rows x cols). */
anyq_status anyq_scaled_values(const anyq_qtensor* qt, float* out);

/* codebooks.hpp:27-38 int_grid(bits, shifted) / fp4_table() / nf4_table():
 * the nominal table of a fixed codebook kind (values[<= 256], *n entries). */
anyq_status anyq_fixed_table(int32_t codebook, int32_t bits, int32_t shifted, float* values,
                             int32_t* n);

/* pack.hpp:57-60 RNE narrowing: NonFiniteError on non-finite input, IoError on
 * overflow to infinity; widening is exact. */
anyq_status anyq_f32_to_f16(float f, uint16_t* out);
float anyq_f16_to_f32(uint16_t h);
anyq_status anyq_f32_to_bf16(float f, uint16_t* out);
float anyq_bf16_to_f32(uint16_t h);

/* codebooks.hpp:50 storage_bits_per_entry(cfg, rows, cols). */
anyq_status anyq_storage_bits_per_entry(const anyq_config* cfg, int64_t rows, int64_t cols,
                                        double* bits);

/* qgemm.hpp:55 bench's timing loop on the device: `repeats` runs (after one
 * warm-up) of one GEMM with operands resident in HBM, each timed with CUDA
 * events; ns[r] = run r in nanoseconds. kind 0: fp32 gemm_dense(x, w) (w is
 * n x k, qt unused); 1: the bit-exact gemm_fused kernel on qt; 2: the A16W4
 * LUT GEMM on the prepacked tensor (bf16 x, the AUTO kernel for m). */
anyq_status anyq_bench_gemm(int32_t kind, const anyq_qtensor* qt, const float* w, int64_t n,
                            int64_t k, const float* x, int64_t m, int32_t repeats, double* ns);

/* Number of kernel launches issued by this library since load (for the
 * bench's gpu_launches accounting). */
uint64_t anyq_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* ANYQ_B200_H */
