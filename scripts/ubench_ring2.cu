// Microbenchmark: the GEMV-style transport alone. 148 persistent CTAs, one
// producer lane streams items (row blocks of IB bytes, dealt round-robin to
// the CTAs) as S-byte cp.async.bulk stages into an R-slot shared-memory ring;
// C consumer warps wait for each stage, read it (LDS.128 per lane, one slice
// per warp) and release it. Reports GB/s for a gate-sized (29.4 MB of codes)
// and a 1 GB stream.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ring2 ubench_ring2.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(ph), "r"(0x989680)
        : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(n), "r"(bar)
      : "memory");
}

constexpr int kC = 16;  // consumer warps
__global__ void __launch_bounds__((kC + 1) * 32, 1)
    k_stream(const uint8_t* __restrict__ p, int nitems, uint32_t IB, uint32_t S, int R, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t full = (uint32_t)__cvta_generic_to_shared(&bars[0]), empty = full + 8 * 32;
  if (threadIdx.x == 0) {
    for (int j = 0; j < R; ++j) {
      mbar_init(full + 8 * j, 1);
      mbar_init(empty + 8 * j, kC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int per = (int)(IB / S);
  if (warp == kC) {
    if (lane == 0) {
      int slot = 0;
      uint32_t round = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x)
        for (int s = 0; s < per; ++s) {
          if (round > 0) mbar_wait(empty + 8 * slot, (round - 1) & 1);
          mbar_expect_tx(full + 8 * slot, S);
          bulk(ring + slot * S, p + (size_t)it * IB + (size_t)s * S, S, full + 8 * slot);
          if (++slot == R) {
            slot = 0;
            ++round;
          }
        }
    }
    return;
  }
  unsigned acc = 0;
  int slot = 0;
  uint32_t round = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x)
    for (int s = 0; s < per; ++s) {
      mbar_wait(full + 8 * slot, round & 1);
      for (uint32_t o = warp * 512; o < S; o += kC * 512) {
        uint4 v;
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(ring + slot * S + o + lane * 16));
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + 8 * slot);
      if (++slot == R) {
        slot = 0;
        ++round;
      }
    }
  if (acc == 0x1234567u) out[0] = acc;
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t* p;
  unsigned* out;
  cudaMalloc(&p, total);
  cudaMalloc(&out, 4);
  cudaMemset(p, 1, total);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { uint32_t S; int R; };
  const Cfg cfgs[] = {{32768, 2}, {32768, 3}, {32768, 4}, {32768, 6}, {16384, 4}, {16384, 8}, {16384, 12},
                      {8192, 8}, {8192, 16}, {8192, 24}, {65536, 3}};
  for (uint32_t IB : {65536u, 229376u}) {
    for (size_t bytes : {(size_t)29360128, (size_t)1 << 29}) {
      const int nitems = (int)(bytes / IB);
      const int ncopy = (int)(total / (nitems * (size_t)IB));
      for (const Cfg& c : cfgs) {
        if (IB % c.S) continue;
        const size_t smem = (size_t)c.S * c.R;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int i = 0; i < 3; ++i)
          k_stream<<<148, (kC + 1) * 32, smem>>>(p + (size_t)(i % ncopy) * nitems * IB, nitems, IB, c.S, c.R, out);
        const int reps = bytes > 100000000 ? 10 : 100;
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i)
          k_stream<<<148, (kC + 1) * 32, smem>>>(p + (size_t)(i % ncopy) * nitems * IB, nitems, IB, c.S, c.R, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const float us = ms * 1e3f / reps;
        printf("item %6u B  total %9zu B  stage %6u x %2d (%4zu KB)  %8.2f us  %6.0f GB/s\n", IB,
               (size_t)nitems * IB, c.S, c.R, smem >> 10, us, nitems * (double)IB / us / 1e3);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
