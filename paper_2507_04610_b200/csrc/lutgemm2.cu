// K2 — large-M any4 LUT GEMM on tcgen05, sm_100a: the weights are dequantised
// to bf16 in shared memory and fed to the tensor cores; no weight copy in HBM.
//
//   y[m][n] = sum_k x[m][k] * bf16(alpha[n][g(k)] * T_n[c[n][k]] + beta[n][g(k)])
//
// (qgemm.cpp:98-111 with the weight rounded once to bf16, as the dequant +
// cuBLAS path K1c; fp32 accumulation in TMEM; bound 2^-8 * sum|x*w|,
// tests/test_gpu_k2.py).
//
// A CTA computes 128 W rows x NT tokens tiles (persistent, round-robin over the
// tiles, tokens innermost so concurrently running CTAs share the weight rows in
// L2). When the tiles are one token tile wide and leave SMs idle in the last
// wave (14336 rows = 112 tiles on 148 SMs; 4096 rows = 32), the launch is split
// stream-K: every CTA takes an equal run of the tiles' k-steps; a segment that
// starts past a tile's step 0 stores its fp32 partial and raises a ready flag
// per epilogue warp (release), and the CTA whose segment holds step 0 adds the
// later CTAs' partials in k order (acquire) before storing y — deterministic,
// and every CTA is co-resident (cooperative launch, one CTA per SM). A pipeline step covers kK2Cps = 2 chunks of 128 k (one step per chunk
// measured 15% slower: the per-step barriers and waits dominate). Per step:
//  * an x producer lane issues the x tile as TMA tensor loads (box 64 k x
//    NT tokens, SWIZZLE_128B: the canonical UMMA K-major layout) into a 2-4
//    stage ring; a code producer lane streams the step's codes (4 row blocks x
//    2 x 2 KB, contiguous per row block in the prepacked layout) and
//    alpha/beta lines by bulk copies into a 4-stage ring;
//  * 16 dequant warps (row block q = warp & 3 = TMEM lane quarter, k quarter
//    j = warp >> 2; lane = row) build a private 16-entry bf16 table
//    bf16(alpha * T[i] + beta) of their row for the step, look each code up
//    (one LDS.U16 per weight) and store the bf16 pairs straight into TMEM as
//    the A operand (tcgen05.st; 2 A stages of 128 columns);
//  * one thread issues 16 tcgen05.mma kind::f16 (bf16 x bf16, M = 128, N = NT,
//    K = 16; A from TMEM, B from shared memory, D in TMEM) and commits;
//  * 4 epilogue warps read the finished tile from TMEM (two accumulator
//    buffers, so the next tile's MMAs overlap) and store y (bf16, optionally
//    fp32).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <mutex>

#include "kernels.cuh"
#include "lutgemm.cuh"

namespace anyq_b200 {

namespace {

constexpr int kK2Dq = 16;       // dequant warps: 4 row blocks (TMEM lane quarters) x 4 k quarters
constexpr int kK2Epi0 = 16;     // epilogue warps 16..19 (TMEM lane quarter = warp & 3)
constexpr int kK2Mma = 20;
constexpr int kK2ProdX = 21;    // x tiles (TMA tensor loads)
constexpr int kK2ProdC = 22;    // codes + alpha/beta (bulk copies)
constexpr int kK2T = 23 * 32;
#ifndef K2_CPS
#define K2_CPS 2
#endif
constexpr int kK2Cps = K2_CPS;                     // 128-k chunks per pipeline step
constexpr int kK2CStages = 8 / kK2Cps;             // code ring
constexpr int kK2AStages = 4 / kK2Cps;             // A stages in TMEM (64 columns per chunk)
constexpr uint32_t kK2Codes = 4 * kK2Cps * 2048;   // codes of one step: 4 row blocks x kK2Cps chunks
constexpr uint32_t kK2Ab = 4 * kK2Cps * 128;       // alpha/beta lines of one step (at most one per chunk)
constexpr uint32_t kK2CStage = kK2Codes + kK2Ab;
constexpr int kK2SkStage = 4;  // stream-K contributors staged per round (4 KB each per epilogue warp)
constexpr uint32_t kK2Tbl = 16 * 64;      // one chunk's table of a row block: 16 entries x 32 rows x bf16

template <int NT>
struct K2Cfg {
  static constexpr int kXStages = kK2Cps == 1 ? (NT >= 128 ? 4 : 6) : (NT >= 128 ? 2 : 4);
  static constexpr uint32_t kBox = NT * 128;           // one 64-k x NT box of x (bf16), 1024-aligned
  static constexpr uint32_t kB = 2 * kK2Cps * kBox;    // x of one step
  static constexpr uint32_t kOffB = 0;
  static constexpr uint32_t kOffC = kOffB + kXStages * kB;
  static constexpr uint32_t kOffTbl = kOffC + kK2CStages * kK2CStage;
  static constexpr uint32_t kOffBars = kOffTbl + 4 * 2 * kK2Cps * kK2Tbl;
  static constexpr uint32_t kSmem = kOffBars + 512;
  static constexpr uint32_t kACol0 = 2 * NT;            // D buffers at columns [0, 2 NT), A after
  static constexpr int kTmemCols = 512;
  static_assert(kACol0 + kK2AStages * 64 * kK2Cps <= kTmemCols, "TMEM budget");
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static_assert(4u * kK2SkStage * 4096u <= kXStages * kB, "stream-K staging fits the x ring");
  // kind::f16 instruction descriptor: D f32 (bit 4), A and B bf16 (format 1 at
  // bits 7 and 10), both K-major, N >> 3 at bit 17, M >> 4 at bit 24
  static constexpr uint32_t kIdesc =
      (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) | ((128u >> 4) << 24);
};
// mbarrier offsets (from kOffBars): x full/empty [6], codes full/empty [8],
// A full/empty [4], D full/empty [2], TMEM slot
constexpr uint32_t kQXFull = 0, kQXEmpty = 48, kQCFull = 96, kQCEmpty = 160, kQAFull = 224, kQAEmpty = 256,
                   kQDFull = 288, kQDEmpty = 304, kQTmem = 320;

struct K2Params {
  const uint8_t* codes;   // [RB][C][4][32][16 B]
  const uint4* lut;       // [RB*32][16] fp16
  const __half2* ab;      // [RB][GR][32]
  __nv_bfloat16* y;
  float* y32;
  int64_t M, N;
  int RB, C, GR, gshift, rtiles, ttiles;
  // stream-K (one token tile): CTA b takes the steps [b U / G, (b+1) U / G)
  // of the U = tiles x steps units; a tile split over CTAs is finished by the
  // CTA holding its step 0, which adds the later CTAs' fp32 partials in k order
  int sk;
  float* part;            // [G][NT][128] partial tiles (stream-K)
  int* flags;             // [G][kK2FlagStride] partial-ready flags of the 4 epilogue warps (self-resetting)
};

// A segment: steps [s0, s1) of one tile.
struct Seg {
  int tile, s0, s1;
};
struct SegIt {
  int u, uend;  // stream-K units
  int t;        // round-robin tile
};
__device__ __forceinline__ int sk_begin(long long U, int b, int G) { return (int)(U * b / G); }
__device__ __forceinline__ SegIt seg_begin(const K2Params& P, int S, int ntiles) {
  SegIt it;
  const long long U = (long long)ntiles * S;
  it.u = sk_begin(U, blockIdx.x, gridDim.x);
  it.uend = sk_begin(U, blockIdx.x + 1, gridDim.x);
  it.t = blockIdx.x;
  return it;
}
__device__ __forceinline__ bool seg_next(const K2Params& P, int S, int ntiles, SegIt& it, Seg& sg) {
  if (P.sk) {
    if (it.u >= it.uend) return false;
    sg.tile = it.u / S;
    sg.s0 = it.u - sg.tile * S;
    sg.s1 = min(S, sg.s0 + (it.uend - it.u));
    it.u += sg.s1 - sg.s0;
    return true;
  }
  if (it.t >= ntiles) return false;
  sg.tile = it.t;
  sg.s0 = 0;
  sg.s1 = S;
  it.t += gridDim.x;
  return true;
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(0x989680)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(pred));
  return pred != 0;
}
// UMMA shared-memory descriptor of B (version 1): K-major SWIZZLE_128B
// (layout type 2), SBO 1024 B between 8-row groups.
__device__ __forceinline__ uint64_t desc_b(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
      "%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int NT>
__global__ void __launch_bounds__(kK2T, 1) k_lutgemm_k2(const __grid_constant__ CUtensorMap xmap,
                                                         const __grid_constant__ K2Params P) {
  using CF = K2Cfg<NT>;
  constexpr int XS = CF::kXStages;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bars = sbase + CF::kOffBars;
  if (threadIdx.x == 0) {
    for (int j = 0; j < XS; ++j) {
      mbar_init(bars + kQXFull + 8 * j, 1);
      mbar_init(bars + kQXEmpty + 8 * j, 1);
    }
    for (int j = 0; j < kK2CStages; ++j) {
      mbar_init(bars + kQCFull + 8 * j, 1);
      mbar_init(bars + kQCEmpty + 8 * j, kK2Dq);
    }
    for (int j = 0; j < kK2AStages; ++j) {
      mbar_init(bars + kQAFull + 8 * j, kK2Dq);
      mbar_init(bars + kQAEmpty + 8 * j, 1);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(bars + kQDFull + 8 * j, 1);
      mbar_init(bars + kQDEmpty + 8 * j, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kK2Mma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(bars + kQTmem),
                 "r"(CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<const uint32_t*>(smem + CF::kOffBars + kQTmem);
  const int ntiles = P.rtiles * P.ttiles;
  const int C = P.C;

  const int S = (C + kK2Cps - 1) / kK2Cps;  // steps per tile

  if (warp == kK2ProdX) {
    // ------------------------------------------------------------ x producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
      int st = 0;
      uint32_t round = 0;
      SegIt it = seg_begin(P, S, ntiles);
      Seg sg;
      while (seg_next(P, S, ntiles, it, sg)) {
        const int tt = sg.tile % P.ttiles;
        for (int sp = sg.s0; sp < sg.s1; ++sp) {
          const int c0 = sp * kK2Cps, nc = min(kK2Cps, C - c0);
          if (round > 0) mbar_wait(bars + kQXEmpty + 8 * st, (round - 1) & 1);
          const uint32_t full = bars + kQXFull + 8 * st;
          mbar_expect_tx(full, (uint32_t)nc * 2 * CF::kBox);
          const uint32_t b = sbase + CF::kOffB + st * CF::kB;
          for (int h = 0; h < nc; ++h) {
            tma_load_2d(b + 2 * h * CF::kBox, &xmap, (c0 + h) * 128, tt * NT, full);
            tma_load_2d(b + (2 * h + 1) * CF::kBox, &xmap, (c0 + h) * 128 + 64, tt * NT, full);
          }
          if (++st == XS) {
            st = 0;
            ++round;
          }
        }
      }
    }
  } else if (warp == kK2ProdC) {
    // ------------------------------------------------------------ code producer
    if (lane == 0) {
      int st = 0;
      uint32_t round = 0;
      SegIt it = seg_begin(P, S, ntiles);
      Seg sg;
      while (seg_next(P, S, ntiles, it, sg)) {
        const int rt = sg.tile / P.ttiles;
        const int nrb = min(4, P.RB - 4 * rt);
        for (int sp = sg.s0; sp < sg.s1; ++sp) {
          const int c0 = sp * kK2Cps, nc = min(kK2Cps, C - c0);
          const int g0 = c0 >> P.gshift, ng = ((c0 + nc - 1) >> P.gshift) - g0 + 1;
          if (round > 0) mbar_wait(bars + kQCEmpty + 8 * st, (round - 1) & 1);
          const uint32_t full = bars + kQCFull + 8 * st;
          mbar_expect_tx(full, (uint32_t)nrb * (nc * 2048 + ng * 128));
          const uint32_t cs = sbase + CF::kOffC + st * kK2CStage;
          for (int q = 0; q < nrb; ++q) {
            const int rb = 4 * rt + q;
            // a row block's chunks are contiguous in the prepacked layout
            bulk_g2s(cs + q * kK2Cps * 2048, P.codes + ((size_t)rb * C + c0) * 2048, nc * 2048, full);
            bulk_g2s(cs + kK2Codes + q * kK2Cps * 128, P.ab + ((size_t)rb * P.GR + g0) * 32, ng * 128, full);
          }
          if (++st == kK2CStages) {
            st = 0;
            ++round;
          }
        }
      }
    }
  } else if (warp == kK2Mma) {
    // ------------------------------------------------------------ MMA issue
    int xs = 0, as = 0, tl = 0;
    uint32_t xround = 0, around = 0;
    SegIt it = seg_begin(P, S, ntiles);
    Seg sg;
    for (; seg_next(P, S, ntiles, it, sg); ++tl) {
      const int db = tl & 1;
      if (tl >= 2) mbar_wait(bars + kQDEmpty + 8 * db, (uint32_t)(((tl >> 1) - 1) & 1));
      const uint32_t d = tmem + (uint32_t)db * NT;
      for (int sp = sg.s0; sp < sg.s1; ++sp) {
        const int nc = min(kK2Cps, C - sp * kK2Cps);
        mbar_wait(bars + kQXFull + 8 * xs, xround & 1);
        mbar_wait(bars + kQAFull + 8 * as, around & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = tmem + CF::kACol0 + (uint32_t)as * (64 * kK2Cps);
          const uint32_t b = sbase + CF::kOffB + xs * CF::kB;
#pragma unroll
          for (int h = 0; h < kK2Cps; ++h) {
            if (h < nc) {  // a missing last chunk: its A and B are stale, skip its MMAs
#pragma unroll
              for (int s = 0; s < 8; ++s)
                tc_mma_ts(d, a + h * 64 + s * 8, desc_b(b + (2 * h + (s >> 2)) * CF::kBox + (s & 3) * 32),
                          CF::kIdesc, (sp > sg.s0 || h > 0 || s > 0) ? 1u : 0u);
            }
          }
          tc_commit(bars + kQXEmpty + 8 * xs);
          tc_commit(bars + kQAEmpty + 8 * as);
          if (sp == sg.s1 - 1) tc_commit(bars + kQDFull + 8 * db);
        }
        __syncwarp();
        if (++xs == XS) {
          xs = 0;
          ++xround;
        }
        if (++as == kK2AStages) {
          as = 0;
          ++around;
        }
      }
    }
  } else if (warp >= kK2Epi0) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    int tl = 0;
    const long long U = (long long)ntiles * S;
    const int b = blockIdx.x, G = gridDim.x;
    SegIt it = seg_begin(P, S, ntiles);
    Seg sg;
    for (; seg_next(P, S, ntiles, it, sg); ++tl) {
      const int rt = sg.tile / P.ttiles, tt = sg.tile - rt * P.ttiles;
      const int db = tl & 1;
      // stream-K: a segment past the tile's step 0 leaves an fp32 partial; the
      // segment holding step 0 (and not the last step) adds the partials of the
      // CTAs b+1.. whose ranges start inside the tile, in k order
      const bool partial = sg.s0 > 0;
      const bool finish = sg.s0 == 0 && sg.s1 < S;
      int cend = b + 1;
      if (finish) {
        const int tend = (sg.tile + 1) * S;
        while (cend < G && sk_begin(U, cend, G) < tend) ++cend;
        // partial rows 32q.. of CTA c are epilogue warp q's: one flag per (c, q)
        if (lane == 0)
          for (int c = b + 1; c < cend; ++c) {
            int v;
            do {
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];"
                           : "=r"(v)
                           : "l"(P.flags + kK2FlagStride * c + q)
                           : "memory");
              if (!v) __nanosleep(32);
            } while (!v);
          }
        __syncwarp();
      }
      mbar_wait(bars + kQDFull + 8 * db, (uint32_t)((tl >> 1) & 1));
      tc_fence_after();
      const int64_t row = (int64_t)rt * 128 + 32 * q + lane;
      const int64_t t0 = (int64_t)tt * NT;
      for (int c0 = 0; c0 < NT; c0 += 32) {
        if (t0 + c0 >= P.M) break;  // no token of this column block (warp-uniform)
        // finisher: this warp's 32 x 32 block of every contributor's partial is
        // staged in the x ring (idle once the CTA's last segment is committed)
        // by cp.async, all contributors in flight at once (a register load per
        // contributor costs one L2 round trip each); 4 contributors per round
        float* stg = reinterpret_cast<float*>(smem + CF::kOffB) + q * (kK2SkStage * 1024);
        int cs0 = b + 1;
        if (finish) {
          const int n0 = min(cend - cs0, kK2SkStage);
          for (int cc = 0; cc < n0; ++cc) {
            const float* src = P.part + ((size_t)(cs0 + cc) * NT + c0) * 128 + 32 * q;
#pragma unroll
            for (int i = 0; i < 8; ++i) {  // 256 16-B pieces: column (i*32+lane)/8, piece %8
              const int idx = i * 32 + lane, col = idx >> 3, pc = idx & 7;
              cp_async16(stg + cc * 1024 + col * 32 + pc * 4, src + (size_t)col * 128 + pc * 4);
            }
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)db * NT + c0, r);
        // partials move whole 32-column blocks, unpredicated (a load under a
        // per-column branch would wait one round trip per column); columns past
        // M are never stored
        if (partial) {
          float* pp = P.part + ((size_t)b * NT + c0) * 128 + 32 * q + lane;
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcg(pp + j * 128, __uint_as_float(r[j]));
        } else {
          while (cs0 < cend) {  // in k order
            const int n0 = min(cend - cs0, kK2SkStage);
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
            for (int cc = 0; cc < n0; ++cc)
#pragma unroll
              for (int j = 0; j < 32; ++j)
                r[j] = __float_as_uint(__uint_as_float(r[j]) + stg[cc * 1024 + j * 32 + lane]);
            cs0 += n0;
            if (cs0 < cend) {  // more than kK2SkStage contributors: next round
              __syncwarp();
              const int n1 = min(cend - cs0, kK2SkStage);
              for (int cc = 0; cc < n1; ++cc) {
                const float* src = P.part + ((size_t)(cs0 + cc) * NT + c0) * 128 + 32 * q;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const int idx = i * 32 + lane, col = idx >> 3, pc = idx & 7;
                  cp_async16(stg + cc * 1024 + col * 32 + pc * 4, src + (size_t)col * 128 + pc * 4);
                }
              }
              asm volatile("cp.async.commit_group;" ::: "memory");
            }
          }
          __syncwarp();
          if (row < P.N) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int64_t m = t0 + c0 + j;
            if (m < P.M) {
              const float v = __uint_as_float(r[j]);
              P.y[m * P.N + row] = __float2bfloat16_rn(v);
              if (P.y32) P.y32[m * P.N + row] = v;
            }
          }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bars + kQDEmpty + 8 * db);
        if (partial) {  // this warp's rows of the partial are out (release)
          __threadfence();
          asm volatile("st.relaxed.gpu.global.s32 [%0], 1;" ::"l"(P.flags + kK2FlagStride * b + q) : "memory");
        }
        for (int c = b + 1; c < cend; ++c)  // consumed: reset for the next launch (kernel-ordered)
          asm volatile("st.relaxed.gpu.global.s32 [%0], 0;" ::"l"(P.flags + kK2FlagStride * c + q) : "memory");
      }
    }
  } else {
    // ------------------------------------------------------------ dequant
    // the row block's 4 warps share its per-chunk tables (two sets by step
    // parity): warp j builds entries 4j..4j+3, a 128-thread named barrier
    // (one per row block) publishes them
    const int q = warp & 3, j = warp >> 2;
    uint16_t* tbl0 = reinterpret_cast<uint16_t*>(smem + CF::kOffTbl + q * 2 * kK2Cps * kK2Tbl);
    const uint32_t tblw0 = sbase + CF::kOffTbl + q * 2 * kK2Cps * kK2Tbl + lane * 2;
    int par = 0;
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + CF::kACol0;
    int cs = 0, as = 0;
    uint32_t cround = 0, around = 0;
    SegIt it = seg_begin(P, S, ntiles);
    Seg sg;
    while (seg_next(P, S, ntiles, it, sg)) {
      const int rt = sg.tile / P.ttiles;
      const int rb = 4 * rt + q;
      const bool live = rb < P.RB;
      // the row's 16 fp16 LUT values
      // this warp builds table entries 4j..4j+3 only: the row's fp16 LUT
      // entries 8(j/2)..+7 are one 16-B load, the half picked by selects (a
      // runtime index into a register array would go through local memory)
      float T[4];
      {
        uint4 l = make_uint4(0, 0, 0, 0);
        if (live) l = P.lut[((size_t)rb * 32 + lane) * 2 + (j >> 1)];
        const uint32_t w0 = (j & 1) ? l.z : l.x, w1 = (j & 1) ? l.w : l.y;
        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&w0));
        const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&w1));
        T[0] = f0.x;
        T[1] = f0.y;
        T[2] = f1.x;
        T[3] = f1.y;
      }
      for (int sp = sg.s0; sp < sg.s1; ++sp) {
        const int c0 = sp * kK2Cps, nc = min(kK2Cps, C - c0);
        mbar_wait(bars + kQCFull + 8 * cs, cround & 1);
        uint32_t v[16 * kK2Cps];
        if (live) {
          const uint8_t* cst = smem + CF::kOffC + cs * kK2CStage;
          const int g0 = c0 >> P.gshift;
          float2 ab[kK2Cps];
          uint4 w4[kK2Cps];
#pragma unroll
          for (int h = 0; h < kK2Cps; ++h) {
            if (h < nc) {
              const int gl = ((c0 + h) >> P.gshift) - g0;
              ab[h] = __half22float2(
                  *reinterpret_cast<const __half2*>(cst + kK2Codes + (q * kK2Cps + gl) * 128 + lane * 4));
              w4[h] = *reinterpret_cast<const uint4*>(cst + (q * kK2Cps + h) * 2048 + j * 512 + lane * 16);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(bars + kQCEmpty + 8 * cs);  // codes and scales are in registers
          // bf16(alpha * T[i] + beta) for this row and chunk (fp32, one rounding)
#pragma unroll
          for (int h = 0; h < kK2Cps; ++h) {
            if (h < nc) {
              uint16_t* tbl = tbl0 + (par * kK2Cps + h) * (kK2Tbl / 2);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                tbl[(4 * j + i) * 32 + lane] = __bfloat16_as_ushort(
                    __float2bfloat16_rn(__fadd_rn(__fmul_rn(ab[h].x, T[i]), ab[h].y)));
            }
          }
          asm volatile("bar.sync %0, 128;" ::"r"(1 + q) : "memory");
          // entry i of row `lane` at tbl + i * 64 + lane * 2, the table 1024-B aligned: the
          // address of nibble n of a code word is ((w >> (4n - 6)) & 0x3C0) | (tbl + lane * 2)
#pragma unroll
          for (int h = 0; h < kK2Cps; ++h) {
            if (h < nc) {
              const uint32_t tblw = tblw0 + (par * kK2Cps + h) * kK2Tbl;
              const uint32_t wd[4] = {w4[h].x, w4[h].y, w4[h].z, w4[h].w};
#pragma unroll
              for (int bb = 0; bb < 16; ++bb) {
                const uint32_t w = wd[bb >> 2];
                const int nlo = 8 * (bb & 3), nhi = nlo + 4;  // bit offsets of the two nibbles
                const uint32_t alo = ((nlo >= 6 ? (w >> (nlo - 6)) : (w << (6 - nlo))) & 0x3C0u) | tblw;
                const uint32_t ahi = ((nhi >= 6 ? (w >> (nhi - 6)) : (w << (6 - nhi))) & 0x3C0u) | tblw;
                uint32_t lo, hi;
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(lo) : "r"(alo));
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(hi) : "r"(ahi));
                v[16 * h + bb] = __byte_perm(lo, hi, 0x5410);
              }
            }
          }
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(bars + kQCEmpty + 8 * cs);
        }
        par ^= 1;
        // chunk h, bytes 0..7: k = 16j + 2b (+1) -> slice j (A columns 64h + 8j..); bytes 8..15:
        // k = 64 + 16j + ... -> slice 4 + j (columns 64h + 32 + 8j..)
        if (around > 0) mbar_wait(bars + kQAEmpty + 8 * as, (around - 1) & 1);
        tc_fence_after();
        if (live) {
          const uint32_t ta = tq + (uint32_t)as * (64 * kK2Cps);
#pragma unroll
          for (int h = 0; h < kK2Cps; ++h) {
            if (h < nc) {
              tc_st8(ta + 64 * h + 8 * j, v + 16 * h);
              tc_st8(ta + 64 * h + 32 + 8 * j, v + 16 * h + 8);
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bars + kQAFull + 8 * as);
        if (++cs == kK2CStages) {
          cs = 0;
          ++cround;
        }
        if (++as == kK2AStages) {
          as = 0;
          ++around;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kK2Mma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::kTmemCols));
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_tiled() {
  static std::mutex mu;
  static EncodeTiled fn = nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    ANYQ_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) fail(ANYQ_ERR_CUDA, "cuTensorMapEncodeTiled not available");
    fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

// Stream-K when the tiles are one token tile wide and do not fill the SMs in
// whole waves. Its cost is one fp32 partial (128 x NT) per split tile, so at
// NT = 128 only for at most half a wave of tiles or >= 24 steps per CTA (gate,
// m = 128, 12 steps per CTA: round-robin 38.6 us against 39.6 us split; down,
// 32 tiles: 95 -> 46 us; 70B gate, 224 tiles x 32 steps: 116 -> 100 us).
bool k2_stream_k(int ntiles, int ttiles, int S, int NT, int sms) {
  const long long U = (long long)ntiles * S;
  return ttiles == 1 && ntiles % sms != 0 && U >= sms && U <= INT32_MAX &&
         (NT == 64 || 2 * ntiles <= sms || U >= 24LL * sms);
}

template <int NT>
void launch_k2(const LutTensor* t, const void* x, int64_t m, void* y, float* y32, cudaStream_t s) {
  using CF = K2Cfg<NT>;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)t->cols, (cuuint64_t)m};
  const cuuint64_t strides[1] = {(cuuint64_t)t->cols * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)NT};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ANYQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  K2Params P;
  P.codes = t->codes;
  P.lut = reinterpret_cast<const uint4*>(t->lut);
  P.ab = t->ab;
  P.y = reinterpret_cast<__nv_bfloat16*>(y);
  P.y32 = y32;
  P.M = m;
  P.N = t->rows;
  P.RB = t->RB;
  P.C = t->C;
  P.GR = t->GR;
  P.gshift = t->gv_gshift;
  P.rtiles = (t->RB + 3) / 4;
  P.ttiles = (int)((m + NT - 1) / NT);
  const int ntiles = P.rtiles * P.ttiles;
  const int S = (P.C + kK2Cps - 1) / kK2Cps;
  P.sk = k2_stream_k(ntiles, P.ttiles, S, NT, t->sms);
  const int grid = P.sk ? t->sms : std::min(ntiles, t->sms);
  P.part = P.sk ? stream_scratch_f32(s, (size_t)grid * NT * 128) : nullptr;
  P.flags = P.sk ? stream_ws(s).k2flags : nullptr;
  ensure_dyn_smem((const void*)k_lutgemm_k2<NT>, (int)CF::kSmem);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 0;
  attr[1].id = cudaLaunchAttributeCooperative;  // stream-K: finishers wait on other CTAs
  attr[1].val.cooperative = 1;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3(kK2T);
  lc.dynamicSmemBytes = CF::kSmem;
  lc.stream = s;
  lc.attrs = attr;
  lc.numAttrs = P.sk ? 2 : 1;
  ANYQ_CUDA(cudaLaunchKernelEx(&lc, k_lutgemm_k2<NT>, map, P));
  ANYQ_LAUNCHED();
}

}  // namespace

bool lutgemm_k2_long_k(const LutTensor* t, int64_t m) {
  if (!t || m < 1 || m > 128) return false;
  const int NT = m <= 64 ? 64 : 128, ntiles = (t->RB + 3) / 4, S = (t->C + kK2Cps - 1) / kK2Cps;
  return k2_stream_k(ntiles, 1, S, NT, t->sms) && (long long)ntiles * S >= 8LL * t->sms;
}

bool lutgemm_k2_supports(const LutTensor* t, int64_t m) {
  return t && m >= 1 && t->gv_gshift >= 0 && (t->cols % 8) == 0 && m <= (int64_t)INT32_MAX;
}

void lutgemm_k2_run(const LutTensor* t, const void* x, int64_t m, void* y, float* y32, cudaStream_t s) {
  if (!t) fail(ANYQ_ERR_SHAPE, "null device tensor");
  if (!lutgemm_k2_supports(t, m))
    fail(ANYQ_ERR_CONFIG, "tcgen05 large-M GEMM needs K % 8 == 0 and rowwise scales or group_size = 128 * 2^j");
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) fail(ANYQ_ERR_SHAPE, "tcgen05 large-M GEMM needs 16-B aligned x");
  if (m <= 64) launch_k2<64>(t, x, m, y, y32, s);
  else launch_k2<128>(t, x, m, y, y32, s);
}

}  // namespace anyq_b200
