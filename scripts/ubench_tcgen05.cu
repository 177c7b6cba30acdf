// Microbenchmark: latencies of the tcgen05 primitives the LUT GEMM chains
// per chunk (A-from-TMEM MMA issue -> commit -> mbarrier completion,
// tcgen05.st + wait::st, tcgen05.ld + wait::ld). One CTA, clock64 deltas.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench_tcgen05.cu
#include <cstdint>
#include <cstdio>

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

__global__ void k(long long* out, int n_mma_per_commit, int N) {
  __shared__ __align__(1024) uint8_t bsm[8192];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t bb = (uint32_t)__cvta_generic_to_shared(&bar);
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) bsm[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bb), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tslot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tslot;
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(bsm);
  uint64_t desc = (uint64_t)((sa >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) |
                  (1ull << 46);
  uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  // 1) MMA round trip
  if (threadIdx.x == 0) {
    uint32_t phase = 0;
    long long tot = 0, mn = 1ll << 60;
    for (int it = 0; it < 64; ++it) {
      long long t0 = clock64();
      for (int j = 0; j < n_mma_per_commit; ++j)
        asm volatile(
            "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, "
            "%3, p; }" ::"r"(t + 128),
            "r"(t), "l"(desc), "r"(idesc), "r"(j)
            : "memory");
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bb)
                   : "memory");
      mbar_wait(bb, phase);
      phase ^= 1;
      long long dt = clock64() - t0;
      if (it >= 8) {
        tot += dt;
        mn = dt < mn ? dt : mn;
      }
    }
    out[0] = tot / 56;
    out[1] = mn;
  }
  __syncthreads();
  // 2) STTM x16 + wait::st, 3) LDTM x4 + wait::ld (warp 0, lanes 0..31)
  if (threadIdx.x < 32) {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = i;
    long long tot = 0, tot2 = 0;
    for (int it = 0; it < 64; ++it) {
      long long t0 = clock64();
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(t),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
          "r"(v[15])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      long long t1 = clock64();
      uint32_t r0, r1, r2, r3;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                   : "r"(t + 128)
                   : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      long long t2 = clock64();
      v[0] += r0 & 1;
      if (it >= 8) {
        tot += t1 - t0;
        tot2 += t2 - t1;
      }
    }
    if (threadIdx.x == 0) {
      out[2] = tot / 56;
      out[3] = tot2 / 56;
      out[4] = v[0];
    }
  }
  // 4) mbarrier arrive -> wait wake-up between two warps (ping-pong)
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(256));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  for (int N : {16, 64, 256}) {
    for (int per : {1, 2, 8}) {
      k<<<1, 128>>>(d, per, N);
      long long h[8];
      cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      printf("N=%3d mma/commit=%d: MMA round trip avg %lld min %lld cycles; STTM.x16+wait %lld; "
             "LDTM.x4+wait %lld\n",
             N, per, h[0], h[1], h[2], h[3]);
    }
  }
  return 0;
}
