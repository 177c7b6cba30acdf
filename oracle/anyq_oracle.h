/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the any4 hot path.
 *
 * A plain-C restatement of the reference algorithms (cited per function in
 * anyq_oracle.c). Same extern "C" signatures as oracle/ref_capi.cpp with an
 * "orc_" prefix instead of "ref_", so the tests drive both through one
 * Python front end (oracle/refpy.py) and pin the restatement against the
 * reference build and the committed golden vectors (tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. The product never links or calls it.
 */
#ifndef ANYQ_ORACLE_H
#define ANYQ_ORACLE_H

#include <stdint.h>

#include "anyq_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
int orc_quantize(const float* w, int64_t rows, int64_t cols, const anyq_config* c,
                 const float* exj, int threads, anyq_qtensor* out);
int orc_time_quantize(const float* w, int64_t rows, int64_t cols, const anyq_config* c,
                      const float* exj, int threads, double* secs);
int orc_narrowed(anyq_qtensor* qt);
int orc_dequantize(const anyq_qtensor* qt, float* w);
int orc_gemm_reference(const float* x, int64_t m, const anyq_qtensor* qt, float* y);
int orc_gemm_fused(const float* x, int64_t m, int64_t k, const anyq_qtensor* qt, int plan_layout,
                   int plan_tile_k, float* y);
int orc_time_gemm_fused(const float* x, int64_t m, const anyq_qtensor* qt, int repeats,
                        double* secs);
int orc_gemm_dense(const float* x, int64_t m, const float* w, int64_t n, int64_t k, float* y);
int orc_column_mean_abs(const float* x, int64_t m, int64_t k, float* out);
int orc_weight_error(const float* w, const anyq_qtensor* qt, double* mse, double* rel);
int orc_output_error(const float* w, const anyq_qtensor* qt, const float* x, int64_t m, double* mse);
int orc_pack_codes(const uint8_t* codes, int64_t rows, int64_t cols, int bits, uint8_t* out);
int orc_unpack_codes(const uint8_t* packed, int64_t rows, int64_t cols, int bits, uint8_t* out);
int orc_to_ktiled(const anyq_qtensor* qt, int tile_k, uint8_t* codes_out);
int orc_from_ktiled(const anyq_qtensor* qt, uint8_t* codes_out);
int orc_f32_to_f16(float f, uint16_t* out);
float orc_f16_to_f32(uint16_t h);
int orc_f32_to_bf16(float f, uint16_t* out);
float orc_bf16_to_f32(uint16_t h);
double orc_storage_bits_per_entry(const anyq_config* c, int64_t rows, int64_t cols);
int orc_kmeans_pp_init(const float* x, const float* w, int64_t n, int k, uint64_t seed,
                       int64_t row, double* centroids);
int orc_weighted_kmeans(const float* x, const float* w, int64_t n, int k, const anyq_config* c,
                        uint64_t seed, int64_t row, double* centroids, uint8_t* assignments,
                        double* loss, int* iters);
int orc_learn_row_lut(const float* x, const float* w, int64_t n, int bits, const anyq_config* c,
                      uint64_t seed, int64_t row, float* lut, uint8_t* codes, double* loss);
void orc_gaussian(int64_t rows, int64_t cols, uint64_t seed, float scale, float* out);
void orc_uniform(int64_t rows, int64_t cols, uint64_t seed, float lo, float hi, float* out);
void orc_dyadic(int64_t rows, int64_t cols, uint64_t seed, int span, float step, float* out);
void orc_heavy_tailed(int64_t rows, int64_t cols, uint64_t seed, float rate, float gain,
                      float* out);
void orc_synthetic_stats(int64_t cols, uint64_t seed, float* out);
void orc_rng_u64(uint64_t seed, int64_t row, int64_t n, uint64_t* out);
void orc_rng_double(uint64_t seed, int64_t row, int64_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif
