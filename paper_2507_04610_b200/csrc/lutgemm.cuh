// Tensor-core LUT GEMM (small M): device-resident prepacked weight tensor.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"

namespace anyq_b200 {

// Prepacked 4-bit LUT tensor resident in HBM (see lutgemm.cu for layouts).
struct LutTensor {
  int64_t rows = 0, cols = 0;
  int RB = 0;   // 32-row blocks
  int C = 0;    // 128-wide k chunks (K padded up)
  int GC = 0;   // chunks per scale group
  int GR = 0;   // scale groups per row
  int64_t weight_bytes = 0;  // algorithmic bytes streamed per GEMM (codes+scales+LUT)
  uint8_t* codes = nullptr;  // [RB][C][4 quarters][32 rows][16 B]
  __half* lut = nullptr;     // [RB*32][16]
  __half2* ab = nullptr;     // [RB][GR][32] (alpha, beta)
  int cmax = 0;  // tcgen05 path: most chunk ranges a row block is split into
  int sms = 148;
  anyq_config cfg{};  // the quantisation config it was created from (for export)
  // CUDA-core GEMV (gemv.cu) work split (its counters live per stream)
  int gv_ncta = 0, gv_gshift = -1;
};

LutTensor* lutgemm_create(const anyq_qtensor* qt);
// prepack^-1: the device layout back to the reference arrays (row-major packed
// codes at cfg.bits, LUT / alpha / beta widened from their fp16 stores) into
// host buffers sized for (rows, cols, cfg) (lutgemm.cu)
void lutgemm_export(const LutTensor* t, anyq_qtensor* out);
LutTensor* load_device_tensor(const char* path);  // ANYQ v1 file -> prepacked (anyq_file.cu)
void lutgemm_destroy(LutTensor* t);
void lutgemm_set_trace(long long* dev);  // debug timeline ([ncta][16] int64), or null
// K1a CUDA-core GEMV (m <= 4) over the same prepacked tensor (gemv.cu).
void lutgemv_setup(LutTensor* t);
void lutgemv_set_trace(long long* dev);  // debug timeline ([ncta][16] int64), or null
// A chain of n <= 8 GEMMs (same m <= 4) in one launch. deps[i]: index of the
// earlier problem whose y problem i reads as x, or -1 (null = no dependencies).
void lutgemv_chain_run(int n, const LutTensor* const* ts, const void* const* xs, void* const* ys,
                       float* const* y32s, const int32_t* deps, int64_t m, cudaStream_t s);
bool lutgemv_fits(const LutTensor* t, int64_t m);  // GEMV applies (m <= 4, shared memory)
// Row-sharded tensor-parallel GEMM with the all-gather fused into the GEMV
// writer (peer stores + per-CTA system-scope flags), and the stream wait for a
// full y (gemv.cu).
void lutgemv_tp_run(const LutTensor* t, const void* x_bf16, int64_t m, const anyq_tp_peers* tp, cudaStream_t s);
int lutgemv_tp_ctas(const LutTensor* t);
void lutgemv_tp_wait(const anyq_tp_peers* tp, int expect, cudaStream_t s);
void lutgemv_run(const LutTensor* t, const void* x_bf16, int64_t m, void* y_bf16, float* y_f32,
                 cudaStream_t s);
// K1t: the same chain with the products on tcgen05 (m <= 16; gemv.cu).
void lutgemv_tc_chain_run(int n, const LutTensor* const* ts, const void* const* xs, void* const* ys,
                          float* const* y32s, const int32_t* deps, int64_t m, cudaStream_t s);
bool lutgemv_tc_fits(const LutTensor* t, int64_t m);  // with up to 8 K-slices
// K-slices a single K1t GEMM at m x rows needs (1: whole; 0: does not fit)
int lutgemv_tc_slices(const LutTensor* t, int64_t m);
void lutgemv_chain_run_auto(int n, const LutTensor* const* ts, const void* const* xs, void* const* ys,
                            float* const* y32s, const int32_t* deps, int64_t m, cudaStream_t s);
void lutgemv_tc_run(const LutTensor* t, const void* x_bf16, int64_t m, void* y_bf16, float* y_f32,
                    cudaStream_t s);
// 1 <= M <= 64: fused dequant-to-shared-memory + mma.sync LUT GEMM (lutmma.cu).
bool lutmma_supports(const LutTensor* t, int64_t m);
void lutmma_run(const LutTensor* t, const void* x_bf16, int64_t m, void* y_bf16, float* y_f32,
                cudaStream_t s);
// K2, large M: dequantise to bf16 in shared memory -> tcgen05 (lutgemm2.cu).
bool lutgemm_k2_supports(const LutTensor* t, int64_t m);
bool lutgemm_k2_long_k(const LutTensor* t, int64_t m);  // AUTO: K2 split stream-K pays (few row tiles, long K)
void lutgemm_k2_run(const LutTensor* t, const void* x_bf16, int64_t m, void* y_bf16, float* y_f32,
                    cudaStream_t s);
// Large M: bf16 dequantization in row slices + cuBLAS GEMM (dequant_gemm.cu).
void dequant_gemm_run(const LutTensor* t, const void* x_bf16, int64_t m, void* y_bf16, float* y_f32,
                      cudaStream_t s);
void lutgemm_run(const LutTensor* t, const void* x_bf16, int64_t m, void* y_bf16, float* y_f32,
                 cudaStream_t s);

}  // namespace anyq_b200
