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

constexpr int64_t kSliceRows = 16384;  // row-block slice dequantized per GEMM (bounded workspace)

// One warp per (row block, 128-k chunk) item, lane L = row L. The lane's 16
// dequantised values alpha_g * T[i] + beta_g (fp32, no contraction:
// qgemm.cpp:98-111, rounded once to bf16) go to a per-warp table tbl[i][lane]
// (bank = lane: conflict free); the chunk's 128 codes become 128 table reads.
// Byte b of slab q holds k = 128c + 16q + 2b (+1) for b < 8 and
// 128c + 64 + 16q + 2(b-8) (+1) for b >= 8 (layout of lutgemm.cu). The 32 x 128
// bf16 tile is staged in shared memory (rows padded to 272 B: conflict free)
// and written out as whole 256-B row segments (coalesced).
constexpr int kDqWarps = 4;
constexpr int kTileStride = 136;  // bf16 per staged row (128 + 8 pad)
__global__ void __launch_bounds__(kDqWarps * 32) k_dequant_bf16(
    const uint4* __restrict__ codes, const uint4* __restrict__ lut, const __half2* __restrict__ ab,
    int rb0, int nrb, int C, int GR, int gshift_chunks, int64_t K, __nv_bfloat16* __restrict__ w) {
  __shared__ uint32_t tbl_all[kDqWarps][16][32];
  __shared__ __align__(16) __nv_bfloat16 tile_all[kDqWarps][32 * kTileStride];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t(*tbl)[32] = tbl_all[warp];
  __nv_bfloat16* tile = tile_all[warp];
  const bool vec = (K & 7) == 0;  // 16-B aligned rows
  int cur_rb = -1;
  float t[16];
  for (int it = blockIdx.x * kDqWarps + warp; it < nrb * C; it += gridDim.x * kDqWarps) {
    const int rbl = it / C, c = it - rbl * C;
    const int rb = rb0 + rbl;
    const int64_t row = (int64_t)rb * 32 + lane;
    if (rb != cur_rb) {
      const uint4 l0 = lut[row * 2], l1 = lut[row * 2 + 1];
      const uint32_t lw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&lw[j]));
        t[2 * j] = f.x;
        t[2 * j + 1] = f.y;
      }
      cur_rb = rb;
    }
    const int g = gshift_chunks >= 30 ? 0 : (c >> gshift_chunks);
    const float2 s = __half22float2(ab[((int64_t)rb * GR + g) * 32 + lane]);
    const uint4* cp = codes + ((int64_t)rb * C + c) * 128 + lane;
    uint4 w4[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w4[q] = cp[q * 32];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; ++i)
      tbl[i][lane] = (uint32_t)__bfloat16_as_ushort(
          __float2bfloat16_rn(__fadd_rn(__fmul_rn(s.x, t[i]), s.y)));
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t wd[4] = {w4[q].x, w4[q].y, w4[q].z, w4[q].w};
      uint32_t o[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const uint32_t byte = (wd[b >> 2] >> (8 * (b & 3))) & 0xffu;
        o[b] = tbl[byte & 15][lane] | (tbl[byte >> 4][lane] << 16);
      }
      uint4* trow = reinterpret_cast<uint4*>(tile + lane * kTileStride + q * 16);
      trow[0] = make_uint4(o[0], o[1], o[2], o[3]);
      trow[1] = make_uint4(o[4], o[5], o[6], o[7]);
      trow[8] = make_uint4(o[8], o[9], o[10], o[11]);    // k + 64
      trow[9] = make_uint4(o[12], o[13], o[14], o[15]);
    }
    __syncwarp();
    // write-out: 16 lanes per row (16 B each) -> 2 rows per instruction
    const int64_t k0 = (int64_t)c * 128;
    const int half = lane >> 4, seg = lane & 15;
#pragma unroll 4
    for (int r = 0; r < 32; r += 2) {
      const int rr = r + half;
      const uint4 v = *reinterpret_cast<const uint4*>(tile + rr * kTileStride + seg * 8);
      __nv_bfloat16* dst = w + ((int64_t)rbl * 32 + rr) * K + k0 + seg * 8;
      if (vec && k0 + seg * 8 + 8 <= K) {
        *reinterpret_cast<uint4*>(dst) = v;
      } else {
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
        for (int j = 0; j < 8; ++j)
          if (k0 + seg * 8 + j < K)
            dst[j] = __ushort_as_bfloat16((unsigned short)(vv[j / 2] >> (16 * (j & 1))));
      }
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
  // stream-ordered workspace from the retained pool: no allocation on the hot
  // path after the first call, and capturable into CUDA graphs (memory nodes)
  DevBuf<__nv_bfloat16> wws(srows * K, s);
  __nv_bfloat16* wbuf = wws.p;
  DevBuf<float> accw;
  if (y32) accw.alloc(m * srows, s);
  Blas& B = blas();
  std::lock_guard<std::mutex> lock(B.mu);
  if (!B.h) check_blas(cublasCreate(&B.h), "cublasCreate");
  check_blas(cublasSetStream(B.h, s), "cublasSetStream");
  const float one = 1.0f, zero = 0.0f;
  for (int rb0 = 0; rb0 < t->RB; rb0 += slice_rb) {
    const int nrb = std::min(slice_rb, t->RB - rb0);
    const int64_t row0 = (int64_t)rb0 * 32;
    const int64_t nrows = std::min<int64_t>((int64_t)nrb * 32, N - row0);
    const int items = nrb * t->C;
    k_dequant_bf16<<<(unsigned)std::max(1, std::min((items + kDqWarps - 1) / kDqWarps, t->sms * 16)),
                     kDqWarps * 32, 0, s>>>(
        reinterpret_cast<const uint4*>(t->codes), reinterpret_cast<const uint4*>(t->lut), t->ab,
        rb0, nrb, t->C, t->GR, gshift, K, wbuf);
    ANYQ_LAUNCHED();
    // column-major view: y^T[nrows x m] (ld N, starting at column row0 of y) =
    // W[nrows x K] (row-major = col-major K x nrows)^T * x^T; bf16 output
    // straight from the GEMM (fp32 accumulation) unless fp32 y is requested
    if (!y32) {
      check_blas(cublasGemmEx(B.h, CUBLAS_OP_T, CUBLAS_OP_N, (int)nrows, (int)m, (int)K, &one, wbuf,
                              CUDA_R_16BF, (int)K, x, CUDA_R_16BF, (int)K, &zero,
                              reinterpret_cast<__nv_bfloat16*>(y) + row0, CUDA_R_16BF, (int)N,
                              CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
                 "cublasGemmEx");
      note_launch();
    } else {
      check_blas(cublasGemmEx(B.h, CUBLAS_OP_T, CUBLAS_OP_N, (int)nrows, (int)m, (int)K, &one, wbuf,
                              CUDA_R_16BF, (int)K, x, CUDA_R_16BF, (int)K, &zero, accw.p, CUDA_R_32F,
                              (int)nrows, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
                 "cublasGemmEx");
      note_launch();
      k_f32_to_outputs<<<(unsigned)std::min<int64_t>((m * nrows + 255) / 256, 148 * 8), 256, 0, s>>>(
          accw.p, m, nrows, N, row0, reinterpret_cast<__nv_bfloat16*>(y), y32);
      ANYQ_LAUNCHED();
    }
  }
}

}  // namespace anyq_b200
