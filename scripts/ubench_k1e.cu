// Microbenchmark for the planned K1e: the inner loop of a LUT GEMM
// at M = 8 tokens, shared memory only (no HBM), 148 CTAs x 16 warps.
//   A) GEMV style (K1a): lane = row, one pair-table LDS per code byte, 2 FHFMA per
//      byte per token (16 per byte at M = 8).
//   B) MMA fragments: a code byte is one fp16x2 A register of mma.m16n8k16 (looked
//      up in a 16-row pair table laid out [entry][row]); one HMMA per 16 rows x 16 k
//      x 8 tokens.
// Reports weights x tokens per second per SM. Codes come from a register LCG
// (same cost in every variant).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_k1e scripts/ubench_k1e.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

constexpr int kWarps = 16, kIters = 4096;

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float fhfma_lo(uint32_t a, uint32_t b, float c) {
  float d;
  asm("{.reg .f16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, al, bl, %3;}"
      : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fhfma_hi(uint32_t a, uint32_t b, float c) {
  float d;
  asm("{.reg .f16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2; fma.rn.f32.f16 %0, ah, bh, %3;}"
      : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}

template <int M>
__global__ void __launch_bounds__(kWarps * 32, 1) k_gemv(float* out, uint32_t seed) {
  __shared__ uint32_t tbl[256 * 32];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) tbl[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tbl) + lane * 4;
  uint32_t x[M];
  float acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    x[m] = 0x3c003c00u + m;
    acc[m] = 0.0f;
  }
  uint32_t s = seed ^ threadIdx.x;
  for (int it = 0; it < kIters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t t[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) t[b] = lds32(base + (((s >> (8 * b)) & 0xff) << 7));
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int m = 0; m < M; ++m) {
        acc[m] = fhfma_lo(t[b], x[m], acc[m]);
        acc[m] = fhfma_hi(t[b], x[m], acc[m]);
      }
  }
  float r = 0;
#pragma unroll
  for (int m = 0; m < M; ++m) r += acc[m];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int REP>
__global__ void __launch_bounds__(kWarps * 32, 1) k_mma8(float* out, uint32_t seed) {
  // pair table of 16 rows: word (copy, entry, row) at copy*4096 + entry*16 + row
  __shared__ uint32_t tbl[REP * 256 * 16];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int i = threadIdx.x; i < REP * 256 * 16; i += blockDim.x) tbl[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
  __syncthreads();
  const int copy = REP == 2 ? (t >> 1) : 0;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tbl) + (uint32_t)(copy * 4096 + g) * 4 +
                        (REP == 2 ? (uint32_t)copy * 32 : 0u);  // copy 1 shifted by 8 banks
  const uint32_t b0 = 0x3c003c00u + lane, b1 = 0x3c003c01u + lane;  // x^T fragment (8 tokens)
  float c[4] = {0, 0, 0, 0};
  uint32_t s = seed ^ threadIdx.x;
  for (int it = 0; it < kIters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t a[4];
    // a0: row g, a1: row g+8, a2: row g, a3: row g+8 (k pairs t and t+4)
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r] = lds32(base + (((s >> (8 * r)) & 0xff) << 6) + (r & 1) * 32);
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0] + c[1] + c[2] + c[3];
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * kWarps * 32 * sizeof(float));
  const double per_sm = 1.0 / 148;
  // A: per lane per iteration 4 code bytes = 8 weights, x 8 tokens
  float ms = time_it([&] { k_gemv<8><<<148, kWarps * 32>>>(out, 1); });
  double wt = 148.0 * kWarps * 32 * kIters * 8 * 8;
  printf("A gemv-style M=8 : %.3f ms  %.1f G weight*token/s per SM\n", ms, wt / (ms * 1e-3) * per_sm / 1e9);
  ms = time_it([&] { k_gemv<1><<<148, kWarps * 32>>>(out, 1); });
  wt = 148.0 * kWarps * 32 * kIters * 8;
  printf("A gemv-style M=1 : %.3f ms  %.1f G weight*token/s per SM (x in registers: no broadcast loads)\n",
         ms, wt / (ms * 1e-3) * per_sm / 1e9);
  // B/C: per warp per iteration one MMA = 16 rows x 16 k weights x 8 tokens
  wt = 148.0 * kWarps * kIters * 256 * 8;
  ms = time_it([&] { k_mma8<1><<<148, kWarps * 32>>>(out, 1); });
  printf("B mma-fragment   : %.3f ms  %.1f G weight*token/s per SM\n", ms, wt / (ms * 1e-3) * per_sm / 1e9);
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
