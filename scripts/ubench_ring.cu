// Microbenchmark: per-warp weight streaming transports for the LUT GEMV.
// 148 persistent CTAs x W warps; each warp streams a contiguous range of 2-KB
// chunks either with LDG.128 (4 per lane per chunk, D chunks in flight in
// registers) or with cp.async.bulk into a private R-slot shared-memory ring
// (mbarrier per slot), then reads the chunk (LDS.128) and xors it.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ring ubench_ring.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(ph)
        : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(n), "r"(bar)
      : "memory");
}

template <int R, int CH>  // R slots of CH bytes per warp
__global__ void k_tma(const uint8_t* __restrict__ p, size_t nchunk, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[32 * R];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const size_t gw = (size_t)blockIdx.x * nw + warp, W = (size_t)gridDim.x * nw;
  const size_t c0 = gw * nchunk / W, c1 = (gw + 1) * nchunk / W;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(sm) + warp * R * CH;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp * R]);
  if (lane == 0)
    for (int j = 0; j < R; ++j) mbar_init(bar + 8 * j, 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  size_t ci = c0;
  for (int j = 0; j < R && ci < c1; ++j, ++ci)
    if (lane == 0) {
      mbar_expect_tx(bar + 8 * j, CH);
      bulk(ring + j * CH, p + ci * CH, CH, bar + 8 * j);
    }
  unsigned acc = 0;
  for (size_t c = c0, n = 0; c < c1; ++c, ++n) {
    const int s = (int)(n % R);
    mbar_wait(bar + 8 * s, (uint32_t)((n / R) & 1));
    for (int q = 0; q < CH / 512; ++q) {
      uint4 v;
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "r"(ring + s * CH + q * 512 + lane * 16));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncwarp();
    if (ci < c1) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar + 8 * s, CH);
        bulk(ring + s * CH, p + ci * CH, CH, bar + 8 * s);
      }
      ++ci;
    }
  }
  if (acc == 0x1234567u) out[0] = acc;
}

template <int D>
__global__ void k_ldg(const uint8_t* __restrict__ p, size_t nchunk, unsigned* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const size_t gw = (size_t)blockIdx.x * nw + warp, W = (size_t)gridDim.x * nw;
  const size_t c0 = gw * nchunk / W, c1 = (gw + 1) * nchunk / W;
  const uint4* q = reinterpret_cast<const uint4*>(p);
  unsigned acc = 0;
  size_t c = c0;
  for (; c + D <= c1; c += D) {
    uint4 r[D][4];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int k = 0; k < 4; ++k) r[d][k] = __ldcs(q + (c + d) * 128 + k * 32 + lane);
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc ^= r[d][k].x ^ r[d][k].y ^ r[d][k].z ^ r[d][k].w;
  }
  for (; c < c1; ++c)
    for (int k = 0; k < 4; ++k) {
      uint4 v = __ldcs(q + c * 128 + k * 32 + lane);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x1234567u) out[0] = acc;
}

template <typename K>
float timeit(K kern, int threads, size_t smem, const uint8_t* p, size_t bytes, size_t stride, int ncopy,
             unsigned* out, size_t chunk) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int i = 0; i < 3; ++i) kern<<<148, threads, smem>>>(p + (i % ncopy) * stride, bytes / chunk, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 40;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) kern<<<148, threads, smem>>>(p + (i % ncopy) * stride, bytes / chunk, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t* p;
  unsigned* out;
  cudaMalloc(&p, total);
  cudaMalloc(&out, 4);
  cudaMemset(p, 1, total);
  for (size_t mb : {32, 128}) {
    const size_t bytes = mb << 20;
    const int ncopy = (int)(total / bytes);
    for (int W : {8, 16}) {
      const int th = W * 32;
      float t;
      t = timeit(k_ldg<2>, th, 0, p, bytes, bytes, ncopy, out, 2048);
      printf("%4zu MB W=%2d LDG D=2          %7.2f us %6.0f GB/s\n", mb, W, t, bytes / t / 1e3);
      t = timeit(k_ldg<4>, th, 0, p, bytes, bytes, ncopy, out, 2048);
      printf("%4zu MB W=%2d LDG D=4          %7.2f us %6.0f GB/s\n", mb, W, t, bytes / t / 1e3);
      t = timeit(k_tma<2, 2048>, th, (size_t)W * 2 * 2048, p, bytes, bytes, ncopy, out, 2048);
      printf("%4zu MB W=%2d TMA R=2 x 2KB    %7.2f us %6.0f GB/s\n", mb, W, t, bytes / t / 1e3);
      t = timeit(k_tma<4, 2048>, th, (size_t)W * 4 * 2048, p, bytes, bytes, ncopy, out, 2048);
      printf("%4zu MB W=%2d TMA R=4 x 2KB    %7.2f us %6.0f GB/s\n", mb, W, t, bytes / t / 1e3);
      t = timeit(k_tma<2, 4096>, th, (size_t)W * 2 * 4096, p, bytes, bytes, ncopy, out, 4096);
      printf("%4zu MB W=%2d TMA R=2 x 4KB    %7.2f us %6.0f GB/s\n", mb, W, t, bytes / t / 1e3);
      t = timeit(k_tma<3, 4096>, th, (size_t)W * 3 * 4096, p, bytes, bytes, ncopy, out, 4096);
      printf("%4zu MB W=%2d TMA R=3 x 4KB    %7.2f us %6.0f GB/s\n", mb, W, t, bytes / t / 1e3);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
