// Microbenchmark: tcgen05.mma issue throughput for the shapes the LUT GEMM
// uses (M=128, K=16, f16) — A from TMEM (.kind::f16 [a_tmem]) vs A from SMEM,
// N in {16, 32, 64, 128, 256}, 16 MMAs into 8 independent accumulators per
// commit (the GEMM's per-stage pattern). Reports cycles per MMA for issue
// (clock64 around the issue loop) and for completion (commit -> mbarrier).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_mma_issue ubench_mma_issue.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(pred));
  return pred != 0;
}

template <bool kTmemA, int N, int NMMA>
__global__ void k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t bb = (uint32_t)__cvta_generic_to_shared(&bar);
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bb), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tslot;
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm);
  const uint64_t bdesc0 = (uint64_t)(((sa + 32768) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
                          ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
  const uint64_t adesc0 = (uint64_t)((sa >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
                          ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  constexpr int NACC = (448 / N) < 8 ? (448 / N) : 8;
  if (threadIdx.x < 32) {
    uint32_t phase = 0;
    long long iss = 0, tot = 0;
    for (int it = 0; it < 40; ++it) {
      __syncwarp();
      long long t0 = clock64();
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < NMMA; ++j) {
          const uint32_t d = t + 64 + (uint32_t)((j >> 1) % NACC) * N;
          const uint64_t bd = bdesc0 + (uint64_t)((j & 7) * 128);
          if (kTmemA) {
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], "
                "%2, %3, p; }" ::"r"(d),
                "r"(t + (j & 7) * 8), "l"(bd), "r"(idesc), "r"(j & 1)
                : "memory");
          } else {
            const uint64_t ad = adesc0 + (uint64_t)((j & 7) * 256);
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, "
                "%2, %3, p; }" ::"r"(d),
                "l"(ad), "l"(bd), "r"(idesc), "r"(j & 1)
                : "memory");
          }
        }
      }
      __syncwarp();
      long long t1 = clock64();
      if (elect_one())
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bb)
                     : "memory");
      __syncwarp();
      mbar_wait(bb, phase);
      phase ^= 1;
      long long t2 = clock64();
      if (it >= 8) {
        iss += t1 - t0;
        tot += t2 - t0;
      }
    }
    if (threadIdx.x == 0) {
      out[0] = iss / 32;
      out[1] = tot / 32;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512));
}

template <bool A, int N, int NM>
void run(long long* d) {
  cudaFuncSetAttribute(k<A, N, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<A, N, NM><<<1, 128, 65536>>>(d);
  long long h[2];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  printf("A=%s N=%3d mmas=%2d: issue %5lld cyc (%5.1f/mma)  issue->complete %5lld cyc (%5.1f/mma)\n",
         A ? "tmem" : "smem", N, NM, h[0], (double)h[0] / NM, h[1], (double)h[1] / NM);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  // warm the clocks up
  cudaFuncSetAttribute(k<true, 64, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int w = 0; w < 400; ++w) k<true, 64, 16><<<148, 128, 65536>>>(d);
  cudaDeviceSynchronize();
  run<true, 16, 2>(d); run<true, 16, 16>(d); run<true, 16, 64>(d);
  run<true, 64, 16>(d); run<true, 64, 64>(d);
  run<true, 256, 16>(d); run<true, 256, 64>(d);
  run<false, 16, 16>(d); run<false, 16, 64>(d);
  run<false, 64, 64>(d); run<false, 256, 64>(d);
  return 0;
}
