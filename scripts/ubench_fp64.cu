// Microbenchmark: fp64 DADD latency / throughput and F2F.F64.F32 throughput on one SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, int iters) {
  double a = out[threadIdx.x], b = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void thr(double* out, long long* cyc, int iters) {
  double a0 = out[threadIdx.x], a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7, b = 1.0000001;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = __dadd_rn(a0, b); a1 = __dadd_rn(a1, b); a2 = __dadd_rn(a2, b); a3 = __dadd_rn(a3, b);
    a4 = __dadd_rn(a4, b); a5 = __dadd_rn(a5, b); a6 = __dadd_rn(a6, b); a7 = __dadd_rn(a7, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void cvt(float* in, double* out, long long* cyc, int iters) {
  float f0 = in[threadIdx.x], f1 = f0 * 2, f2 = f0 * 3, f3 = f0 * 4;
  double s = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double d0 = (double)f0, d1 = (double)f1, d2 = (double)f2, d3 = (double)f3;
    f0 = __double2float_rn(d1); f1 = __double2float_rn(d2); f2 = __double2float_rn(d3); f3 = __double2float_rn(d0);
  }
  long long t1 = clock64();
  out[threadIdx.x] = f0 + f1 + f2 + f3 + s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  float* in;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&in, 1024 * 4);
  cudaMemset(out, 0, 1024 * 8);
  cudaMemset(in, 0, 1024 * 4);
  cudaMallocManaged(&cyc, 8);
  const int it = 4096;
  lat<<<1, 32>>>(out, cyc, it);
  cudaDeviceSynchronize();
  printf("DADD dependent latency: %.1f cycles\n", (double)*cyc / (4.0 * it));
  for (int warps : {1, 4, 8, 16, 32}) {
    thr<<<1, 32 * warps>>>(out, cyc, it);
    cudaDeviceSynchronize();
    printf("DADD throughput, %2d warps: %.2f cycles per warp-instr per SM (%.1f lanes/clk/SM)\n", warps,
           (double)*cyc / (8.0 * it * warps), 32.0 * 8.0 * it * warps / (double)*cyc);
  }
  for (int warps : {1, 4, 8, 16}) {
    cvt<<<1, 32 * warps>>>(in, out, cyc, it);
    cudaDeviceSynchronize();
    printf("F2F f32<->f64 pairs, %2d warps: %.2f cycles per warp-conversion per SM\n", warps,
           (double)*cyc / (8.0 * it * warps));
  }
  return 0;
}
