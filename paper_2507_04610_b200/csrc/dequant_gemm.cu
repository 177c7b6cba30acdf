// Large-M path (M > 16, compute-bound): dequantize the prepacked weight to
// bf16 in row-block slices and run a cuBLAS bf16 GEMM (fp32 accumulation) per
// slice. W = alpha_g * T[c] + beta_g is formed in fp32 from the fp16 LUT and
// scales (pack.cpp:205-236 with the narrowed stores) and rounded once to bf16;
// the error bound is the tensor-core tolerance 2^-8 * sum|x*w|
// (tests/test_gpu_gemm.py). This is the library-GEMM baseline the fused
// tcgen05 large-M kernel is measured against.
#include <cublas_v2.h>
#include <cuda_bf16.h>

#include <mutex>

#include "kernels.cuh"
#include "lutgemm.cuh"

namespace anyq_b200 {

namespace {

constexpr int64_t kSliceRows = 4096;  // row-block slice dequantized per GEMM (bounded workspace)

// One thread per (row, slab): 16 code bytes -> 32 bf16 weights at
// k = 128c + 64h + 16q + 2j (+1), h = byte/8, j = byte%8 (layout of lutgemm.cu).
__global__ void k_dequant_bf16(const uint4* __restrict__ codes, const uint4* __restrict__ lut,
                               const __half2* __restrict__ ab, int rb0, int nrb, int C, int GR,
                               int gshift_chunks, int64_t K, __nv_bfloat16* __restrict__ w) {
  const int64_t total = (int64_t)nrb * C * 4 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(i & 31);
    const int q = (int)((i >> 5) & 3);
    const int64_t cc = i >> 7;  // (row block, chunk)
    const int c = (int)(cc % C);
    const int rbl = (int)(cc / C);
    const int rb = rb0 + rbl;
    const uint4 w4 = codes[((int64_t)rb * C + c) * 128 + q * 32 + lane];
    const int64_t row = (int64_t)rb * 32 + lane;
    __half t[16];
    {
      const uint4 l0 = lut[row * 2], l1 = lut[row * 2 + 1];
      const uint32_t lw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const __half2 h2 = *reinterpret_cast<const __half2*>(&lw[j]);
        t[2 * j] = __low2half(h2);
        t[2 * j + 1] = __high2half(h2);
      }
    }
    const int g = gshift_chunks >= 30 ? 0 : (c >> gshift_chunks);
    const float2 s = __half22float2(ab[((int64_t)rb * GR + g) * 32 + lane]);
    const uint32_t wd[4] = {w4.x, w4.y, w4.z, w4.w};
    __nv_bfloat16 out[32];
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const uint32_t byte = (wd[b >> 2] >> (8 * (b & 3))) & 0xffu;
      // fp32 alpha * T + beta, no contraction (qgemm.cpp:98-111 order)
      out[2 * b] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(s.x, __half2float(t[byte & 15])), s.y));
      out[2 * b + 1] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(s.x, __half2float(t[byte >> 4])), s.y));
    }
    __nv_bfloat16* dst = w + (int64_t)rbl * 32 * K + (int64_t)lane * K + (int64_t)c * 128 + q * 16;
    // bytes 0..7 -> k = 128c + 16q + [0,16); bytes 8..15 -> k = 128c + 64 + 16q + [0,16)
    const int64_t k0 = (int64_t)c * 128 + q * 16;
    const bool vec = (K & 7) == 0;  // 16-B aligned rows
    if (vec && k0 + 16 <= K) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&out[0]);
      *reinterpret_cast<uint4*>(dst + 8) = *reinterpret_cast<const uint4*>(&out[8]);
    } else {
      for (int j = 0; j < 16; ++j)
        if (k0 + j < K) dst[j] = out[j];
    }
    if (vec && k0 + 64 + 16 <= K) {
      *reinterpret_cast<uint4*>(dst + 64) = *reinterpret_cast<const uint4*>(&out[16]);
      *reinterpret_cast<uint4*>(dst + 72) = *reinterpret_cast<const uint4*>(&out[24]);
    } else {
      for (int j = 0; j < 16; ++j)
        if (k0 + 64 + j < K) dst[64 + j] = out[16 + j];
    }
  }
}

__global__ void k_f32_to_outputs(const float* __restrict__ src, int64_t m, int64_t n_slice,
                                 int64_t N, int64_t col0, __nv_bfloat16* __restrict__ y,
                                 float* __restrict__ y32) {
  const int64_t total = m * n_slice;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n_slice, c = i % n_slice;
    const float v = src[i];
    y[r * N + col0 + c] = __float2bfloat16_rn(v);
    if (y32) y32[r * N + col0 + c] = v;
  }
}

struct Blas {
  cublasHandle_t h = nullptr;
  std::mutex mu;
};
Blas& blas() {
  static Blas b;
  return b;
}

void check_blas(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS)
    fail(ANYQ_ERR_CUDA, std::string(what) + ": cuBLAS status " + std::to_string((int)st));
}

}  // namespace

void dequant_gemm_run(const LutTensor* t, const void* x, int64_t m, void* y, float* y32,
                      cudaStream_t s) {
  if (!t) fail(ANYQ_ERR_SHAPE, "null device tensor");
  if (m < 1) fail(ANYQ_ERR_SHAPE, "dequant GEMM needs m >= 1");
  if (t->GR != 1 && (t->GC & (t->GC - 1)) != 0)
    fail(ANYQ_ERR_CONFIG, "dequant GEMM needs rowwise scales or group_size = 128 * 2^j");
  const int gshift = t->GR == 1 ? 30 : __builtin_ctz((unsigned)t->GC);
  const int64_t K = t->cols, N = t->rows;
  const int slice_rb = (int)(kSliceRows / 32);
  const int64_t srows = std::min<int64_t>(kSliceRows, (int64_t)t->RB * 32);
  // workspace kept on the tensor (first use sizes it; later calls are graph-capturable)
  LutTensor* mt = const_cast<LutTensor*>(t);
  if (!mt->dq_w) ANYQ_CUDA(cudaMalloc(&mt->dq_w, sizeof(__nv_bfloat16) * srows * K));
  if (m * srows > mt->dq_acc_n) {
    if (mt->dq_acc) ANYQ_CUDA(cudaFree(mt->dq_acc));
    ANYQ_CUDA(cudaMalloc(&mt->dq_acc, sizeof(float) * m * srows));
    mt->dq_acc_n = m * srows;
  }
  __nv_bfloat16* wbuf = reinterpret_cast<__nv_bfloat16*>(mt->dq_w);
  float* accbuf = mt->dq_acc;
  Blas& B = blas();
  std::lock_guard<std::mutex> lock(B.mu);
  if (!B.h) check_blas(cublasCreate(&B.h), "cublasCreate");
  check_blas(cublasSetStream(B.h, s), "cublasSetStream");
  const float one = 1.0f, zero = 0.0f;
  for (int rb0 = 0; rb0 < t->RB; rb0 += slice_rb) {
    const int nrb = std::min(slice_rb, t->RB - rb0);
    const int64_t row0 = (int64_t)rb0 * 32;
    const int64_t nrows = std::min<int64_t>((int64_t)nrb * 32, N - row0);
    const int64_t items = (int64_t)nrb * t->C * 128;
    k_dequant_bf16<<<(unsigned)std::min<int64_t>((items + 255) / 256, 148 * 16), 256, 0, s>>>(
        reinterpret_cast<const uint4*>(t->codes), reinterpret_cast<const uint4*>(t->lut), t->ab,
        rb0, nrb, t->C, t->GR, gshift, K, wbuf);
    ANYQ_LAUNCHED();
    // column-major view: acc^T[nrows x m] = W[nrows x K] (row-major = col-major K x nrows)^T * x^T
    check_blas(cublasGemmEx(B.h, CUBLAS_OP_T, CUBLAS_OP_N, (int)nrows, (int)m, (int)K, &one, wbuf,
                            CUDA_R_16BF, (int)K, x, CUDA_R_16BF, (int)K, &zero, accbuf, CUDA_R_32F,
                            (int)nrows, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
               "cublasGemmEx");
    note_launch();
    k_f32_to_outputs<<<(unsigned)std::min<int64_t>((m * nrows + 255) / 256, 148 * 8), 256, 0, s>>>(
        accbuf, m, nrows, N, row0, reinterpret_cast<__nv_bfloat16*>(y), y32);
    ANYQ_LAUNCHED();
  }
}

}  // namespace anyq_b200
