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
// L2). Per 128-k step:
//  * a producer lane issues the x tile as two TMA tensor loads (box 64 k x NT
//    tokens, SWIZZLE_128B: the canonical UMMA K-major layout) and the step's
//    codes (4 row blocks x 2 KB of the prepacked layout) and alpha/beta lines
//    as bulk copies, all on one mbarrier, into a 2-stage ring;
//  * 16 dequant warps (row block q = warp & 3, k quarter j = warp >> 2; lane =
//    row) build a private 16-entry bf16 table bf16(alpha * T[i] + beta) of
//    their row for the step, then look each code up (one LDS.U16 per weight)
//    and store the bf16 pairs as the A operand in the canonical K-major
//    no-swizzle layout (per 16-k slice [8-row group][k half][8 rows][16 B]);
//  * one thread issues 8 tcgen05.mma kind::f16 (bf16 x bf16, M = 128, N = NT,
//    K = 16; A and B from shared memory, D in TMEM) and commits the stage;
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

constexpr int kK2Dq = 16;       // dequant warps: 4 row blocks x 4 k quarters
constexpr int kK2Epi0 = 16;     // epilogue warps 16..19 (TMEM lane quarter = warp & 3)
constexpr int kK2Mma = 20;
constexpr int kK2Prod = 21;
constexpr int kK2T = 22 * 32;
constexpr int kK2Stages = 2;
constexpr uint32_t kK2A = 8 * 4096;       // A of one step: 8 slices x (16 groups x 256 B)
constexpr uint32_t kK2Codes = 4 * 2048;   // codes of one step: 4 row blocks x one chunk
constexpr uint32_t kK2Ab = 4 * 128;       // alpha/beta lines of one step
constexpr uint32_t kK2Tbl = 16 * 64;      // a dequant warp's table: 16 entries x 32 lanes x bf16

template <int NT>
struct K2Cfg {
  static constexpr uint32_t kBox = NT * 128;           // one 64-k x NT box of x (bf16), 1024-aligned
  static constexpr uint32_t kB = 2 * kBox;             // x of one 128-k step
  static constexpr uint32_t kOffB = 0;
  static constexpr uint32_t kOffA = kOffB + kK2Stages * kB;
  static constexpr uint32_t kOffCodes = kOffA + kK2Stages * kK2A;
  static constexpr uint32_t kOffAb = kOffCodes + kK2Stages * kK2Codes;
  static constexpr uint32_t kOffTbl = kOffAb + kK2Stages * kK2Ab;
  static constexpr uint32_t kOffBars = kOffTbl + kK2Dq * kK2Tbl;
  static constexpr uint32_t kSmem = kOffBars + 256;
  static constexpr int kTmemCols = 2 * NT <= 256 ? 256 : 512;
  // kind::f16 instruction descriptor: D f32 (bit 4), A and B bf16 (format 1 at
  // bits 7 and 10), both K-major, N >> 3 at bit 17, M >> 4 at bit 24
  static constexpr uint32_t kIdesc =
      (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) | ((128u >> 4) << 24);
};
// mbarrier offsets (from kOffBars)
constexpr uint32_t kQFull = 0, kQEmpty = 16, kQAFull = 32, kQDFull = 48, kQDEmpty = 64, kQTmem = 80;

struct K2Params {
  const uint8_t* codes;   // [RB][C][4][32][16 B]
  const uint4* lut;       // [RB*32][16] fp16
  const __half2* ab;      // [RB][GR][32]
  __nv_bfloat16* y;
  float* y32;
  int64_t M, N;
  int RB, C, GR, gshift, rtiles, ttiles;
};

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
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(pred));
  return pred != 0;
}
// UMMA shared-memory descriptors (version 1): A — K-major, no swizzle, LBO
// 128 B between the two 8-k halves, SBO 256 B between 8-row groups; B —
// K-major SWIZZLE_128B (layout type 2), SBO 1024 B between 8-row groups.
__device__ __forceinline__ uint64_t desc_a(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46);
}
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
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bars = sbase + CF::kOffBars;
  if (threadIdx.x == 0) {
    for (int j = 0; j < kK2Stages; ++j) {
      mbar_init(bars + kQFull + 8 * j, 1);
      mbar_init(bars + kQEmpty + 8 * j, 1);
      mbar_init(bars + kQAFull + 8 * j, kK2Dq);
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

  if (warp == kK2Prod) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
      int st = 0;
      uint32_t round = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int rt = tile / P.ttiles, tt = tile - rt * P.ttiles;
        const int nrb = min(4, P.RB - 4 * rt);
        for (int c = 0; c < C; ++c) {
          if (round > 0) mbar_wait(bars + kQEmpty + 8 * st, (round - 1) & 1);
          const uint32_t full = bars + kQFull + 8 * st;
          mbar_expect_tx(full, CF::kB + (uint32_t)nrb * (2048 + 128));
          const uint32_t b = sbase + CF::kOffB + st * CF::kB;
          tma_load_2d(b, &xmap, c * 128, tt * NT, full);
          tma_load_2d(b + CF::kBox, &xmap, c * 128 + 64, tt * NT, full);
          const int g = c >> P.gshift;
          for (int q = 0; q < nrb; ++q) {
            const int rb = 4 * rt + q;
            bulk_g2s(sbase + CF::kOffCodes + st * kK2Codes + q * 2048,
                     P.codes + ((size_t)rb * C + c) * 2048, 2048, full);
            bulk_g2s(sbase + CF::kOffAb + st * kK2Ab + q * 128, P.ab + ((size_t)rb * P.GR + g) * 32, 128, full);
          }
          if (++st == kK2Stages) {
            st = 0;
            ++round;
          }
        }
      }
    }
  } else if (warp == kK2Mma) {
    // ------------------------------------------------------------ MMA issue
    int st = 0, tl = 0;
    uint32_t round = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
      const int db = tl & 1;
      if (tl >= 2) mbar_wait(bars + kQDEmpty + 8 * db, (uint32_t)(((tl >> 1) - 1) & 1));
      const uint32_t d = tmem + (uint32_t)db * NT;
      for (int c = 0; c < C; ++c) {
        mbar_wait(bars + kQFull + 8 * st, round & 1);
        mbar_wait(bars + kQAFull + 8 * st, round & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = sbase + CF::kOffA + st * kK2A;
          const uint32_t b = sbase + CF::kOffB + st * CF::kB;
#pragma unroll
          for (int s = 0; s < 8; ++s)
            tc_mma_ss(d, desc_a(a + s * 4096), desc_b(b + (s >> 2) * CF::kBox + (s & 3) * 32), CF::kIdesc,
                      (c > 0 || s > 0) ? 1u : 0u);
          tc_commit(bars + kQEmpty + 8 * st);
          if (c == C - 1) tc_commit(bars + kQDFull + 8 * db);
        }
        __syncwarp();
        if (++st == kK2Stages) {
          st = 0;
          ++round;
        }
      }
    }
  } else if (warp >= kK2Epi0) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    int tl = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
      const int rt = tile / P.ttiles, tt = tile - rt * P.ttiles;
      const int db = tl & 1;
      mbar_wait(bars + kQDFull + 8 * db, (uint32_t)((tl >> 1) & 1));
      tc_fence_after();
      const int64_t row = (int64_t)rt * 128 + 32 * q + lane;
      const int64_t t0 = (int64_t)tt * NT;
      for (int c0 = 0; c0 < NT; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)db * NT + c0, r);
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
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bars + kQDEmpty + 8 * db);
    }
  } else {
    // ------------------------------------------------------------ dequant
    const int q = warp & 3, j = warp >> 2;
    uint16_t* tbl = reinterpret_cast<uint16_t*>(smem + CF::kOffTbl + warp * kK2Tbl);
    const uint32_t tblw = sbase + CF::kOffTbl + warp * kK2Tbl + lane * 2;
    int st = 0;
    uint32_t round = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int rt = tile / P.ttiles;
      const int rb = 4 * rt + q;
      const bool live = rb < P.RB;
      // the row's 16 fp16 LUT values
      float T[16];
      {
        uint4 l0 = make_uint4(0, 0, 0, 0), l1 = l0;
        if (live) {
          l0 = P.lut[((size_t)rb * 32 + lane) * 2];
          l1 = P.lut[((size_t)rb * 32 + lane) * 2 + 1];
        }
        const uint32_t lw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&lw[i]));
          T[2 * i] = f.x;
          T[2 * i + 1] = f.y;
        }
      }
      for (int c = 0; c < C; ++c) {
        // the stage's A buffer is free once its previous MMAs completed
        if (round > 0) mbar_wait(bars + kQEmpty + 8 * st, (round - 1) & 1);
        mbar_wait(bars + kQFull + 8 * st, round & 1);
        if (live) {
          // bf16(alpha * T[i] + beta) for this row and step (fp32, one rounding)
          const float2 ab = __half22float2(*reinterpret_cast<const __half2*>(
              smem + CF::kOffAb + st * kK2Ab + q * 128 + lane * 4));
#pragma unroll
          for (int i = 0; i < 16; ++i)
            tbl[i * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(__fadd_rn(__fmul_rn(ab.x, T[i]), ab.y)));
          __syncwarp();
          const uint4 w4 = *reinterpret_cast<const uint4*>(smem + CF::kOffCodes + st * kK2Codes + q * 2048 +
                                                           j * 512 + lane * 16);
          const uint32_t wd[4] = {w4.x, w4.y, w4.z, w4.w};
          uint32_t v[16];
#pragma unroll
          for (int bb = 0; bb < 16; ++bb) {
            const uint32_t byte = (wd[bb >> 2] >> (8 * (bb & 3))) & 0xFFu;
            uint16_t lo, hi;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(lo) : "r"(tblw + ((byte & 15u) << 6)));
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(hi) : "r"(tblw + ((byte >> 4) << 6)));
            v[bb] = (uint32_t)lo | ((uint32_t)hi << 16);
          }
          // bytes 0..7: k = 16j + 2b (+1) -> slice j; bytes 8..15: k = 64 + 16j + ... -> slice 4 + j.
          // Row r = 32q + lane: [slice][r / 8][k half][r % 8][16 B]
          const uint32_t rowoff = (uint32_t)(4 * q + (lane >> 3)) * 256 + (uint32_t)(lane & 7) * 16;
          uint8_t* a = smem + CF::kOffA + st * kK2A + rowoff;
          *reinterpret_cast<uint4*>(a + j * 4096) = make_uint4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<uint4*>(a + j * 4096 + 128) = make_uint4(v[4], v[5], v[6], v[7]);
          *reinterpret_cast<uint4*>(a + (4 + j) * 4096) = make_uint4(v[8], v[9], v[10], v[11]);
          *reinterpret_cast<uint4*>(a + (4 + j) * 4096 + 128) = make_uint4(v[12], v[13], v[14], v[15]);
        }
        // generic-proxy writes of A -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(bars + kQAFull + 8 * st);
        if (++st == kK2Stages) {
          st = 0;
          ++round;
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
  const int grid = std::min(ntiles, t->sms);
  ensure_dyn_smem((const void*)k_lutgemm_k2<NT>, (int)CF::kSmem);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3(kK2T);
  lc.dynamicSmemBytes = CF::kSmem;
  lc.stream = s;
  lc.attrs = attr;
  lc.numAttrs = 1;
  ANYQ_CUDA(cudaLaunchKernelEx(&lc, k_lutgemm_k2<NT>, map, P));
  ANYQ_LAUNCHED();
}

}  // namespace

bool lutgemm_k2_supports(const LutTensor* t, int64_t m) {
  return t && m >= 1 && t->gv_gshift >= 0 && (t->cols % 8) == 0 && m <= (int64_t)INT32_MAX;
}

void lutgemm_k2_run(const LutTensor* t, const void* x, int64_t m, void* y, float* y32, cudaStream_t s) {
  if (!t) fail(ANYQ_ERR_SHAPE, "null device tensor");
  if (!lutgemm_k2_supports(t, m))
    fail(ANYQ_ERR_CONFIG, "tcgen05 large-M GEMM needs K % 8 == 0 and rowwise scales or group_size = 128 * 2^j");
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) fail(ANYQ_ERR_SHAPE, "tcgen05 large-M GEMM needs 16-B aligned x");
  if (m <= 64) launch_k2<64>(t, x, m, y, y32, s);
  else if (m <= 128) launch_k2<128>(t, x, m, y, y32, s);
  else launch_k2<256>(t, x, m, y, y32, s);
}

}  // namespace anyq_b200
