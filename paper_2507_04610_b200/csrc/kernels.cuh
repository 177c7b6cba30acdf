// Launcher declarations shared by the C-ABI layer (capi.cu) and the kernels.
#pragma once

#include <float.h>

#include <algorithm>

#include "common.cuh"

namespace anyq_b200 {

void launch_check_finite(const float* p, int64_t n, int* err, int status, cudaStream_t s);
// out2 = {sum (a-b)^2, sum a^2} in double, deterministic tree; part: 2 * 592 doubles
void launch_sqdiff_sums(const float* a, const float* b, int64_t n, double* part, double* out2,
                        cudaStream_t s);
// E|x_j| of collect_stats (calibration.cpp:62-67), bit-identical (quant_kernels.cu)
// (non-finite inputs set *err = ANYQ_ERR_NONFINITE; the output is then undefined)
void launch_col_mean_abs(const float* x, int64_t m, int64_t k, float* out, int* err, cudaStream_t s);
void launch_check_stats(const float* p, int64_t n, int* err, cudaStream_t s);
void launch_scales(const float* w, int64_t rows, int64_t cols, const anyq_config& cfg, float qmin,
                   float qmax, float* alphas, float* betas, cudaStream_t s);
void launch_scale_rows(const float* w, int64_t rows, int64_t cols, const anyq_config& cfg,
                       const float* alphas, const float* betas, const float* exj, float* ws,
                       float* sw, int* err, cudaStream_t s);
void launch_affine(const float* in, int64_t rows, int64_t cols, const anyq_config& cfg,
                   const float* alphas, const float* betas, int inverse, float* out,
                   cudaStream_t s);
void launch_round(const float* ws, int64_t n, const Table& t, uint8_t* codes, cudaStream_t s);
// build_sample_weights (learner.cpp:25-51) of one row: out[cols]
void launch_sample_weights(const anyq_config& cfg, int64_t row, int64_t cols, const float* alphas,
                           const float* stats, int weighting, float* out, cudaStream_t s);
void launch_pack(const uint8_t* codes, int64_t rows, int64_t cols, int bits, uint8_t* out,
                 int* err, cudaStream_t s);
void launch_unpack(const uint8_t* packed, int64_t rows, int64_t cols, int bits, uint8_t* codes,
                   cudaStream_t s);
void launch_ktile(const uint8_t* in, int64_t rows, int64_t cols, int64_t tile_k, int inverse,
                  uint8_t* out, cudaStream_t s);
void launch_narrow(float* v, int64_t n, int store, int is_alpha, int* err, cudaStream_t s);
void launch_dequant(const uint8_t* packed, int64_t rows, int64_t cols, int bits, int ktiled,
                    int64_t tile_k, const float* luts, const Table& fixed, const anyq_config& cfg,
                    const float* alphas, const float* betas, float* w, int* err, cudaStream_t s);
void launch_gemm_exact(const float* x, int64_t m, int64_t k, const uint8_t* packed, int64_t n,
                       int bits, int ktiled, int64_t tile_k, const float* luts, const Table& fixed,
                       const anyq_config& cfg, const float* alphas, const float* betas, float* y,
                       int* err, cudaStream_t s);
void launch_gemm_dense(const float* x, int64_t m, const float* w, int64_t n, int64_t k, float* y,
                       cudaStream_t s);

// k-means learner (kmeans.cu): ws/sw are rows x cols on device; writes the
// row LUTs (rows x 2^bits fp32) and logical codes (rows x cols uint8).
void launch_kmeans(const float* ws, const float* sw, int64_t rows, int64_t cols,
                   const anyq_config& cfg, int64_t row_offset, float* luts, uint8_t* codes,
                   int* err, cudaStream_t s);

// The per-row learner API (learner.hpp:52-61) on `rows` independent problems
// of n samples (row-major, original order), every reduction in the
// reference's order: mode 0 = learn_row_lut (sorted LUT [rows][k] as float,
// rank codes [rows][n], loss), 1 = weighted_kmeans (centroids [rows][k],
// assignments [rows][n], loss, iters), 2 = kmeans_pp_init (centroids only).
// rng_key / rng_ctr: each problem's Rng state, counters advanced in place.
void launch_kmeans_problems(const float* x, const float* w, int64_t rows, int64_t n, int k,
                            const anyq_config& cfg, int mode, const uint64_t* rng_key,
                            uint64_t* rng_ctr, double* centroids, uint8_t* assignments, double* loss,
                            int* iters, float* luts, uint8_t* codes, int* err, cudaStream_t s);

}  // namespace anyq_b200
