// Microbenchmark: HBM read bandwidth of a persistent LDG.128 streaming kernel
// vs. loads in flight per warp (D) and warps per SM (W), at the GEMV's sizes.
// Each warp reads contiguous 512-B slabs (one uint4 per lane) like the LUT GEMV.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_stream ubench_stream.cu
#include <cstdint>
#include <cstdio>
#include <vector>

template <int D>
__global__ void k_stream(const uint4* __restrict__ p, size_t nslab, unsigned* out) {
  const int lane = threadIdx.x & 31;
  const size_t warps = (size_t)gridDim.x * (blockDim.x >> 5);
  const size_t w = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // contiguous range of slabs per warp
  const size_t s0 = w * nslab / warps, s1 = (w + 1) * nslab / warps;
  unsigned acc = 0;
  size_t s = s0;
  for (; s + D <= s1; s += D) {
    uint4 r[D];
#pragma unroll
    for (int j = 0; j < D; ++j) r[j] = __ldcs(p + (s + j) * 32 + lane);
#pragma unroll
    for (int j = 0; j < D; ++j) acc ^= r[j].x ^ r[j].y ^ r[j].z ^ r[j].w;
  }
  for (; s < s1; ++s) {
    uint4 r = __ldcs(p + s * 32 + lane);
    acc ^= r.x ^ r.y ^ r.z ^ r.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int D>
float run(const uint4* p, size_t bytes, int ctas, int threads, unsigned* out, int ncopy,
          size_t stride) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i)
    k_stream<D><<<ctas, threads>>>(p + (i % ncopy) * stride / 16, bytes / 512, out);
  const int reps = 40;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i)
    k_stream<D><<<ctas, threads>>>(p + (i % ncopy) * stride / 16, bytes / 512, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;  // us per kernel
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint4* p;
  unsigned* out;
  cudaMalloc(&p, total);
  cudaMalloc(&out, 4);
  cudaMemset(p, 1, total);
  const size_t sizes[] = {(size_t)9 << 20, (size_t)32 << 20, (size_t)128 << 20};
  for (size_t bytes : sizes) {
    const int ncopy = (int)(total / bytes) > 8 ? 8 : (int)(total / bytes);
    for (int W : {8, 16, 32}) {
      for (int cps : {1, 2}) {
        const int threads = W * 32 / cps;
        if (threads > 1024 || threads < 32) continue;
        const int ctas = 148 * cps;
        float t1 = run<1>(p, bytes, ctas, threads, out, ncopy, bytes);
        float t4 = run<4>(p, bytes, ctas, threads, out, ncopy, bytes);
        float t8 = run<8>(p, bytes, ctas, threads, out, ncopy, bytes);
        float t16 = run<16>(p, bytes, ctas, threads, out, ncopy, bytes);
        printf("%4zu MB  warps/SM %2d (%d CTA/SM)  us: D1 %7.2f  D4 %7.2f  D8 %7.2f  D16 %7.2f   "
               "GB/s: %6.0f %6.0f %6.0f %6.0f\n",
               bytes >> 20, W, cps, t1, t4, t8, t16, bytes / t1 / 1e3, bytes / t4 / 1e3,
               bytes / t8 / 1e3, bytes / t16 / 1e3);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
