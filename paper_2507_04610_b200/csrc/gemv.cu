// K1a — CUDA-core any4 LUT GEMV for M <= 4 (the memory-bound decode path), sm_100a.
//
//   y[m][n] = sum_k x[m][k] * (alpha[n][g(k)] * T_n[c[n][k]] + beta[n][g(k)])
//
// is the reference's gemm_fused (qgemm.cpp:71-128) with the per-group scale
// factored out of the k loop. Per 128-k chunk c:
//   y[m][n] += alpha_g * 2^-e * sum_{k in c} xh[m][k] * T_n[c[n][k]] + beta_g * sum_{k in c} x[m][k]
// where xh = fp16(x * 2^e), e putting max|x| of the chunk in [2^14, 2^15),
// is exact for every |x| >= 2^-32 max|x| (bf16 has 8 significant bits; fp16
// keeps them down to 2^-17, inside its subnormal range); smaller values round
// to the fp16 subnormal grid (error <= 2^-40 max|x| per element, far inside
// the tolerance; tests/test_gpu_headline.py::test_gemv_wide_dynamic_range_x).
// Every product xh * T
// (fp16 x fp16) is formed exactly by FHFMA (fma.rn.f32.f16) and accumulated in
// fp32, so the result differs from the fp32 reference only by summation order
// (tolerance 1e-5 * sum|x*w|, tests/test_gpu_gemm.py).
//
// One persistent CTA per SM: 16 compute warps, 1 writer warp, 1 producer warp
// (two lanes, one per half ring), 1 builder warp (each item's pair table, one
// item ahead), 1 dependency warp (the x hand-offs).
//  * Work items are whole 32-row blocks. A launch runs a chain of up to 8
//    GEMMs; problem i may depend on one earlier problem dep[i] (its x is that
//    problem's y). The chain's row blocks, concatenated in problem order, are
//    dealt round-robin to the CTAs and every CTA walks its items in order, so
//    independent problems fill the time other CTAs spend waiting on a
//    dependency. An item is computed by one CTA only, so y needs no cross-CTA
//    combine and the result is deterministic.
//  * The producer warp streams every item of the CTA: its 32 LUT rows (1 KB)
//    and its codes in STAGES of 16 consecutive 128-k chunks (32 rows x 128 k
//    = 2 KB each, contiguous in the prepacked layout [RB][C][4 slabs][32
//    rows][16 B]) plus their (alpha, beta) lines into a 2..4-deep
//    shared-memory ring. Compute warp w takes chunk w of every stage; lane L
//    owns row L, so compute warps read weights from shared memory only. The
//    ring is two half rings (chunks 0-7 of a stage for warps 0-7, 8-15 for
//    warps 8-15; one producer lane and one cp.async.bulk per half and stage),
//    so one half's refills do not wait for the other half's slowest warp.
//  * LUT lookup: the row's 16 fp16 values are expanded once per row block into
//    a 256-entry pair table T2[byte] = (T[lo], T[hi]); entry e of lane L lives
//    at shared address 0x10000 + e*256 + buf*128 + L*4. Every lookup of a warp
//    hits bank L (conflict free), the address is ONE prmt of the code byte into
//    the lane word (no add: the table is 64 KB aligned in the shared window),
//    and ONE LDS dequantises two weights. Two buffers, handed between warps
//    with mbarriers (warps drift by up to one item instead of meeting at a CTA
//    barrier).
//  * x enters once per image: each compute warp loads the bf16 x of exactly
//    the chunks it reads straight from global memory (L2) and converts it into
//    the permuted fp16 image the code bytes index, plus per-chunk (2^-e, sum x),
//    so no CTA barrier follows. Consecutive problems that read the same x share
//    the image; images alternate between two banks.
//  * The writer warp reduces the 16 warp partials of an item in a fixed order,
//    stores y, and after its items of a problem releases that problem
//    grid-wide (done[p], in problem order). A dependency warp releases x to
//    the compute warps (bar_x): for a dependent problem it first waits until
//    every CTA released the problem x comes from, while the weights already
//    stream in. The grid is co-resident (cooperative launch) and dependencies
//    point backwards, so the waits cannot deadlock.
#include <cuda_bf16.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>

#include "kernels.cuh"
#include "lutgemm.cuh"

namespace anyq_b200 {

namespace {

constexpr int kW = 16;                // compute warps per CTA (one table slice each)
constexpr int kWriterWarp = kW;
constexpr int kProducerWarp = kW + 1;
constexpr int kBuilderWarp = kW + 2;  // every item's pair table, one item ahead
constexpr int kDepWarp = kW + 3;      // the x hand-offs (dependency waits), off the writer
constexpr int kT = (kW + 4) * 32;
constexpr int kMaxMP = 4;  // MP in {1, 2, 3, 4}: one template instance per x-row count
constexpr int kStageChunks = kW;      // chunks per ring stage: one per compute warp
constexpr uint32_t kStageBytes = kStageChunks * 2048u;
constexpr uint32_t kStageAb = kStageChunks * 128u;
constexpr int kMaxRing = 4;
constexpr int kTcStageGroups = 4;     // K1t: 4 chunk groups (one per team) per ring stage
constexpr uint32_t kTcGroupBytes = 4 * 2048u;                      // codes of one group
constexpr uint32_t kTcStageBytes = kTcStageGroups * kTcGroupBytes;  // 32 KB
constexpr uint32_t kTcGroupAb = 4 * 128u;                          // alpha/beta lines of one group
constexpr uint32_t kTcStageAb = kTcStageGroups * kTcGroupAb;
constexpr int kTcMaxRing = 6;
constexpr int kMaxProb = 8;
constexpr int kMaxTp = 8;  // ranks of the fused tensor-parallel gather
constexpr uint32_t kTblAddr = 0x10000;  // shared-window address of the pair table
constexpr uint32_t kDynBase = 0x400;    // shared-window address of dynamic smem (sm_100)
constexpr uint32_t kPre = kTblAddr - kDynBase;  // bytes of dynamic smem before the table
constexpr uint32_t kTblBytes = 0x10000;
constexpr uint32_t kSmemMax = 227u * 1024u;
constexpr uint32_t kParamOff = 0;     // dynamic-smem copy of the parameter block

// mbarriers (8 B each) at GvParams::bars
constexpr uint32_t kBarRedFull = 0;    // [2] partials of an item ready (kW arrivals)
constexpr uint32_t kBarRedEmpty = 16;  // [2] partials consumed by the writer (1)
constexpr uint32_t kBarX = 32;         // x rows of a batch landed (writer + tx)
constexpr uint32_t kBarTReady = 40;    // [2] pair-table buffer written (kW)
constexpr uint32_t kBarTFree = 56;     // [2] pair-table buffer no longer read (kW)
constexpr uint32_t kBarLFull = 72;     // [2] LUT rows of an item landed (producer + tx)
constexpr uint32_t kBarLFree = 88;     // [2] LUT rows consumed (kW)
#ifndef GV_RING_PARTS
#define GV_RING_PARTS 2
#endif
constexpr int kRingParts = GV_RING_PARTS;           // independent part rings of a stage
constexpr int kPartChunks = kStageChunks / kRingParts;  // chunks (= compute warps) per part
constexpr uint32_t kBarSFull = 104;    // [kRingParts][kMaxRing] part of a stage landed (producer + tx)
constexpr uint32_t kBarSEmpty = kBarSFull + 8 * kRingParts * kMaxRing;  // [..] part consumed
// compute warps consume kRingParts independent part rings (each 32-KB stage
// buffer holds every part's chunks; barriers per part): a lagging part no
// longer holds back the other parts' refills (2 parts: gate 14.1 -> 13.85 us)
constexpr uint32_t kBarBytes = kBarSEmpty + 8 * kRingParts * kMaxRing;

struct GvProb {
  const uint4* codes;    // [RB][C][4][32] uint4
  const uint4* lut;      // [RB*32][2] uint4 (16 fp16)
  const uint32_t* ab;    // [RB][GR][32] half2 (alpha, beta)
  const __nv_bfloat16* x;
  __nv_bfloat16* y;
  float* y32;
  uint32_t xh, xs;       // dynamic-smem offsets of this problem's x image / chunk scales
  int N, K, C, GR, RB;
  int gshift;            // chunk -> scale group: g = c >> gshift
  int dep;               // problem whose output x is (must be complete first), or -1
  int img;               // x image index (problems in a row with the same x share one)
  int newimg;            // first problem of its image
  int tma;               // x rows 16-B aligned with K % 128 == 0: 16-B loads (K1a, K1t)
  int rboff;             // first item of this problem in the chain's item sequence
  // K1t K-slices of one GEMM (lutgemv_tc_run when the whole x image does not
  // fit): chunks [c0, c0 + C) of the tensor; codes/ab/x point at chunk c0
  int cstride;           // chunks per row block in the code layout (the tensor's C)
  int xstride;           // elements between x rows (the tensor's K)
  const float* acc_in;   // y32 partial of the previous slice (added first), or null
  float* acc_out;        // this slice's partial (y32 of the running sum), or null: final slice
};

struct GvParams {
  GvProb p[kMaxProb];
  int np, M, ncta;
  int tot;               // items (row blocks) of the whole chain
  int nring;             // code ring stages (2..kMaxRing)
  uint32_t red;          // dynamic-smem offset of the reduction buffer [2][kW][MP][32]
  uint32_t bars;         // dynamic-smem offset of the mbarriers
  uint32_t ring[kTcMaxRing];  // dynamic-smem offsets of the code ring stages [chunks][2048]
  uint32_t abring;       // dynamic-smem offset of the (alpha, beta) ring [nring][16][128]
  uint32_t lutbuf;       // dynamic-smem offset of the LUT rows [2][32][32 B]
  int* done;             // [kMaxProb] per-problem release counters (self-resetting)
  int* err;              // device error word
  long long* trace;      // debug: [ncta][64] globaltimer stamps, or null
  // tensor-parallel gather fused into the writer (single-problem launches):
  // y also goes to every rank's full-width y buffer (NVLink peer stores), then
  // each CTA bumps tp_flags[r][tp_rank] on every rank r (release, system scope)
  int tp_world, tp_rank;
  long long tp_row0, tp_N;
  __nv_bfloat16* tp_y[kMaxTp];
  int* tp_flags[kMaxTp];
};

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float fhfma_lo(uint32_t a, uint32_t b, float c) {
  float r;
  asm("{ .reg .f16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2;"
      " fma.rn.f32.f16 %0, al, bl, %3; }"
      : "=f"(r)
      : "r"(a), "r"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fhfma_hi(uint32_t a, uint32_t b, float c) {
  float r;
  asm("{ .reg .f16 al, ah, bl, bh; mov.b32 {al, ah}, %1; mov.b32 {bl, bh}, %2;"
      " fma.rn.f32.f16 %0, ah, bh, %3; }"
      : "=f"(r)
      : "r"(a), "r"(b), "f"(c));
  return r;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds64f(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: the waiting warp is parked until the
// phase completes instead of re-polling, so waiting warps (the highest warp
// ids, which the scheduler favours) do not take issue slots from the warps
// sharing their SMSP.
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
#ifdef GV_SPIN_WAIT  // experiment build: poll without the hint
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
#else
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(0x989680)
        : "memory");
#endif
  }
}
// Same, backing off between polls (for waits that are usually long).
__device__ __forceinline__ void mbar_wait_sleep(uint32_t a, uint32_t parity) {
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(200);
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin until *p >= target, then acquire (one fence, not an L1 invalidation per poll).
__device__ __forceinline__ void wait_geq(const int* p, int target) {
  while (ld_relaxed(p) < target) __nanosleep(32);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GV_TRACE(slot)                                                             \
  do {                                                                             \
    if (P.trace && threadIdx.x == 0) P.trace[blockIdx.x * 64 + (slot)] = gtimer(); \
  } while (0)
#define GV_TRACE_W(slot)                                        \
  do {                                                          \
    if (P.trace) P.trace[blockIdx.x * 64 + (slot)] = gtimer(); \
  } while (0)

// ---------------------------------------------------------------------------
// Work items: (problem, row block). The chain's row blocks, concatenated in
// problem order, are dealt round-robin to the CTAs (item j -> CTA j % ncta);
// every CTA walks its items in sequence order, so a problem's dependency
// (always an earlier problem) can never wait on a later item.
// ---------------------------------------------------------------------------
struct Item {
  int p, rb, j;  // p == np: end; j = item index in the chain sequence
};

__device__ __forceinline__ void locate(const GvParams& P, Item& it) {
  if (it.j >= P.tot) {
    it.p = P.np;
    return;
  }
  while (it.j >= P.p[it.p].rboff + P.p[it.p].RB) ++it.p;
  it.rb = it.j - P.p[it.p].rboff;
}
__device__ __forceinline__ Item item_begin(const GvParams& P, int b) {
  Item it{0, 0, b};
  locate(P, it);
  return it;
}
__device__ __forceinline__ void item_next(const GvParams& P, int /*b*/, Item& it) {
  it.j += P.ncta;
  locate(P, it);
}
struct Chunk {
  uint4 w[4];
  uint32_t ab;
};

// Pair table for row `lane` into buffer buf: entry e = 16*hi + lo holds
// (T[lo], T[hi]); call `warp` = w writes the slice hi = w (the builder warps
// of K1a and K1t call it for w = 0..15).
__device__ __forceinline__ void build_table(const uint4 l0, const uint4 l1, int warp, int buf,
                                            uint32_t laneoff) {
  static_assert(kW >= 16, "one high nibble per compute warp");
  if (warp >= 16) return;
  const uint32_t t[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
  const int h = warp >> 1;  // word of T[warp] (selects, not a local-memory index)
  const uint32_t s0 = (h & 1) ? l0.y : l0.x, s1 = (h & 1) ? l0.w : l0.z;
  const uint32_t s2 = (h & 1) ? l1.y : l1.x, s3 = (h & 1) ? l1.w : l1.z;
  const uint32_t u0 = (h & 2) ? s1 : s0, u1 = (h & 2) ? s3 : s2;
  const uint32_t th = (h & 4) ? u1 : u0;
  const uint32_t hsel = (warp & 1) ? 0x76u : 0x54u;
#pragma unroll
  for (int lo = 0; lo < 16; ++lo) {
    const uint32_t sel = ((lo & 1) ? 0x32u : 0x10u) | (hsel << 8);
    sts32(kTblAddr + (16 * warp + lo) * 256 + buf * 128 + laneoff, __byte_perm(t[lo >> 1], th, sel));
  }
}

// One chunk: 128 codes of row `lane` against the x image of the chunk.
// tb = table word (0x10000 | buf << 7 | lane << 2); xa/xsa = shared addresses of
// the (m = 0) x image / (2^-e, sum x) of this chunk; per-m strides follow.
template <int MP>
__device__ __forceinline__ void consume(const Chunk& ch, const uint32_t tb, const uint32_t xa,
                                        const uint32_t xsa, const uint32_t xstride,
                                        const uint32_t xsstride, float (&y)[MP]) {
  float a0[MP], a1[MP], a2[MP], a3[MP];
#pragma unroll
  for (int m = 0; m < MP; ++m) a0[m] = a1[m] = a2[m] = a3[m] = 0.0f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t wd[4] = {ch.w[q].x, ch.w[q].y, ch.w[q].z, ch.w[q].w};
    uint32_t t[16];
#pragma unroll
    for (int b = 0; b < 16; ++b)
#ifdef GV_NOLOOKUP  // experiment build: the table address without the shared-memory read
      t[b] = __byte_perm(wd[b >> 2], tb, 0x7604u | ((uint32_t)(b & 3) << 4));
#else
      t[b] = lds32(__byte_perm(wd[b >> 2], tb, 0x7604u | ((uint32_t)(b & 3) << 4)));
#endif
#pragma unroll
    for (int m = 0; m < MP; ++m) {
      const uint32_t xq = xa + m * xstride + q * 64;
      const uint4 x0 = lds128(xq), x1 = lds128(xq + 16), x2 = lds128(xq + 32), x3 = lds128(xq + 48);
      const uint32_t xw[16] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w,
                               x2.x, x2.y, x2.z, x2.w, x3.x, x3.y, x3.z, x3.w};
#pragma unroll
      for (int b = 0; b < 16; b += 2) {
        a0[m] = fhfma_lo(t[b], xw[b], a0[m]);
        a1[m] = fhfma_hi(t[b], xw[b], a1[m]);
        a2[m] = fhfma_lo(t[b + 1], xw[b + 1], a2[m]);
        a3[m] = fhfma_hi(t[b + 1], xw[b + 1], a3[m]);
      }
    }
  }
  const float2 ab = __half22float2(*reinterpret_cast<const __half2*>(&ch.ab));
#pragma unroll
  for (int m = 0; m < MP; ++m) {
    const float2 sc = lds64f(xsa + m * xsstride);
    y[m] = fmaf(ab.x, sc.x * ((a0[m] + a1[m]) + (a2[m] + a3[m])), fmaf(ab.y, sc.y, y[m]));
  }
}

// x of problem q -> permuted fp16 image + per-chunk (2^-e, sum x) for chunk c
// of x row m: the 8 lanes of a lane group own 16 consecutive k each
// (k = 128c + 16*sub + t), so the max/sum trees are 3 shuffles deep. Image position of k = 128c + 64h + 16s + 2j (+1): slab s,
// pair 8h + j -> a lane's 16 values are pairs 8*(sub/4) .. +7 of slab sub%4.
template <int MP>
__device__ __forceinline__ void prep_x(const GvProb& q, int M, uint8_t* smem, int m, int c, int lane) {
  const int sub = lane & 7;
  const int k0 = c * 128 + sub * 16;
  float v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) v[t] = 0.0f;
  const bool live = m < M && c < q.C;
  if (live && q.tma && k0 + 16 <= q.K) {
    // 16-B loads straight from global (L2; x may be another CTA's y, released
    // to this CTA by the writer's acquire and bar_x)
    const uint4* src = reinterpret_cast<const uint4*>(q.x + (size_t)m * q.K + k0);
    const uint4 r0 = __ldcg(src), r1 = __ldcg(src + 1);
    const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const __nv_bfloat162 p2 = *reinterpret_cast<const __nv_bfloat162*>(&w[t]);
      v[2 * t] = __low2float(p2);
      v[2 * t + 1] = __high2float(p2);
    }
  } else if (live) {  // direct loads (K not a multiple of 128 or unaligned x)
    const unsigned short* xr = reinterpret_cast<const unsigned short*>(q.x + (size_t)m * q.K);
    unsigned short r[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) r[t] = (k0 + t < q.K) ? __ldcg(xr + k0 + t) : (unsigned short)0;
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = __bfloat162float(__ushort_as_bfloat16(r[t]));
  }
  float amax = 0.0f, sum = 0.0f;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    amax = fmaxf(amax, fabsf(v[t]));
    sum += v[t];
  }
#pragma unroll
  for (int off = 4; off; off >>= 1) {
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    sum += __shfl_xor_sync(0xffffffffu, sum, off);
  }
  // e puts max|x| in [2^14, 2^15): exponent arithmetic on the bits (ldexpf /
  // ilogbf are library calls, many times the instructions of this block)
  const int ex = (__float_as_int(amax) >> 23) & 0xff;  // biased exponent (amax >= 0)
  const int e = (amax > 0.0f && ex < 255) ? min(141 - ex, 126) : 0;
  const float sc = __int_as_float((127 + e) << 23), isc = __int_as_float((127 - e) << 23);
  uint32_t h[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const __half2 p2 = __floats2half2_rn(v[2 * t] * sc, v[2 * t + 1] * sc);
    h[t] = *reinterpret_cast<const uint32_t*>(&p2);
  }
  __syncwarp();
  if (live) {
    uint8_t* dst = smem + q.xh + (size_t)m * q.C * 256 + c * 256 + ((sub & 3) * 16 + 8 * (sub >> 2)) * 4;
    *reinterpret_cast<uint4*>(dst) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(dst + 16) = make_uint4(h[4], h[5], h[6], h[7]);
    if (sub == 0)
      *reinterpret_cast<float2*>(smem + q.xs + ((size_t)m * q.C + c) * 8) = make_float2(isc, sum);
  }
}

// Writer warp, per problem in order: reduces the kW warp partials of each
// item in a fixed order and stores y, then releases the problem grid-wide
// (done[p]; in order, so done[p] == ncta implies every earlier problem is
// complete too). The x hand-offs are the dependency warp's.
template <int MP>
__device__ __forceinline__ void writer_loop(const GvParams& P, const float* red, uint32_t bars,
                                            uint32_t sbase, int b, int lane) {
  const uint32_t bar_full = bars + kBarRedFull, bar_empty = bars + kBarRedEmpty;
  Item it = item_begin(P, b);
  int g = 0;
  for (int p = 0; p < P.np; ++p) {
    const GvProb& q = P.p[p];
    while (it.p == p) {
      const int par = g & 1;
      mbar_wait_sleep(bar_full + 8 * par, (uint32_t)((g >> 1) & 1));
      const float* rp = red + (size_t)par * kW * MP * 32;
      float acc[MP];
#pragma unroll
      for (int m = 0; m < MP; ++m) {
        float t = 0.0f;
#pragma unroll
        for (int w = 0; w < kW; ++w) t += rp[(w * MP + m) * 32 + lane];
        acc[m] = t;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + 8 * par);
      const int row = it.rb * 32 + lane;
      if (row < q.N) {
#pragma unroll
        for (int m = 0; m < MP; ++m) {
          if (m < P.M) {
            const __nv_bfloat16 v = __float2bfloat16_rn(acc[m]);
            if (P.tp_world == 0) {
              q.y[(size_t)m * q.N + row] = v;
              if (q.y32) q.y32[(size_t)m * q.N + row] = acc[m];
            }
            // the fused all-gather: this rank's slice straight into every rank's y
            for (int r = 0; r < P.tp_world; ++r) P.tp_y[r][(size_t)m * P.tp_N + P.tp_row0 + row] = v;
          }
        }
      }
      item_next(P, b, it);
      ++g;
    }
    __syncwarp();
    if (P.tp_world > 0) __threadfence_system();  // every lane's peer stores before the flags
    __syncwarp();
    if (P.tp_world > 0 && lane < P.tp_world) {
      asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(P.tp_flags[lane] + P.tp_rank) : "memory");
    }
    if (lane == 0) {
      if (p < P.np - 1) {  // fire-and-forget release (this warp's y stores ordered by __syncwarp)
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&P.done[p]) : "memory");
      } else {  // the last problem's release also finds the last CTA, which resets the counters
        __threadfence();
        const int old = atomicAdd(&P.done[p], 1);
        if (old == P.ncta - 1)
          for (int r = 0; r < P.np; ++r) P.done[r] = 0;
      }
    }
    __syncwarp();
  }
}

// Producer (lanes 0 and 1, one per half ring): per item lane 0 loads its LUT
// rows into lutbuf[g & 1]; each lane copies its half's 8 chunks of every stage
// (and their alpha/beta lines) into its half ring. Weights do not depend on
// the previous kernel, so this runs before griddepcontrol.wait.
__device__ __forceinline__ void producer_loop(const GvParams& P, uint32_t bars, uint32_t sbase,
                                              int b, int half) {
  const uint32_t lfull = bars + kBarLFull, lfree = bars + kBarLFree;
  const uint32_t sfull = bars + kBarSFull + 8u * kMaxRing * half;
  const uint32_t sempty = bars + kBarSEmpty + 8u * kMaxRing * half;
  const uint32_t abring = sbase + P.abring, lutbuf = sbase + P.lutbuf;
  Item it = item_begin(P, b);
  int g = 0, slot = 0;
  uint32_t round = 0;
  while (it.p < P.np) {
    const GvProb& q = P.p[it.p];
    const int lb = g & 1;
    if (half == 0) {  // the item's LUT rows (half A's lane)
      if (g >= 2) mbar_wait(lfree + 8 * lb, (uint32_t)(((g >> 1) - 1) & 1));
      mbar_expect_tx(lfull + 8 * lb, 1024);
      bulk_g2s(lutbuf + lb * 1024, reinterpret_cast<const uint8_t*>(q.lut) + (size_t)it.rb * 1024, 1024,
               lfull + 8 * lb);
    }
    const uint8_t* cg = reinterpret_cast<const uint8_t*>(q.codes) + (size_t)it.rb * q.C * 2048;
    const uint8_t* ag = reinterpret_cast<const uint8_t*>(q.ab) + (size_t)it.rb * q.GR * 128;
    for (int cs = 0; cs < q.C; cs += kStageChunks) {
      // this half's 8 chunks of the stage (possibly none: the slot still turns)
      const int c0 = cs + kPartChunks * half;
      const int n = max(0, min(kPartChunks, q.C - c0));
      const uint32_t hoff = (uint32_t)half * kPartChunks * 2048u, aoff = (uint32_t)half * (kStageAb / kRingParts);
      if (n == 0) {
        if (round > 0) mbar_wait(sempty + 8 * slot, (round - 1) & 1);
        mbar_arrive(sfull + 8 * slot);
        if (++slot == P.nring) {
          slot = 0;
          ++round;
        }
        continue;
      }
      const int g0 = c0 >> q.gshift, g1 = (c0 + n - 1) >> q.gshift;
      if (round > 0) mbar_wait(sempty + 8 * slot, (round - 1) & 1);
#ifdef GV_NOLOAD  // compute-only experiment build: the ring keeps stale codes
      mbar_expect_tx(sfull + 8 * slot, (uint32_t)(g1 - g0 + 1) * 128);
#else
      mbar_expect_tx(sfull + 8 * slot, (uint32_t)n * 2048 + (uint32_t)(g1 - g0 + 1) * 128);
      bulk_g2s(sbase + P.ring[slot] + hoff, cg + (size_t)c0 * 2048, (uint32_t)n * 2048, sfull + 8 * slot);
#endif
      bulk_g2s(abring + slot * kStageAb + aoff, ag + (size_t)g0 * 128, (uint32_t)(g1 - g0 + 1) * 128,
               sfull + 8 * slot);
      if (++slot == P.nring) {
        slot = 0;
        ++round;
      }
    }
    item_next(P, b, it);
    ++g;
  }
}

template <int MP>
__global__ void __launch_bounds__(kT, 1) k_lutgemv(const __grid_constant__ GvParams Pk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  asm volatile("griddepcontrol.launch_dependents;");
  // The parameter block (indexed by problem) is copied to shared memory in one
  // parallel pass: register-indexed constant loads would otherwise miss the
  // constant cache one dependent round trip at a time.
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&Pk);
    uint32_t* dst = reinterpret_cast<uint32_t*>(smem + kParamOff);
    for (int i = threadIdx.x; i < (int)(sizeof(GvParams) / 4); i += kT) dst[i] = src[i];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x;
  const uint32_t laneoff = (uint32_t)lane << 2;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const GvParams& P = *reinterpret_cast<const GvParams*>(smem + kParamOff);
  __syncthreads();
  const uint32_t bars = sbase + P.bars;
  GV_TRACE(0);
  if (sbase != kDynBase) {  // the table must sit at shared address 0x10000
    if (threadIdx.x == 0) atomicMax(P.err, (int)ANYQ_ERR_INTERNAL);
    return;
  }
  if (threadIdx.x == 0) {
    for (int j = 0; j < 2; ++j) {
      mbar_init(bars + kBarRedFull + 8 * j, kW);
      mbar_init(bars + kBarRedEmpty + 8 * j, 1);
      mbar_init(bars + kBarTReady + 8 * j, 1);  // the builder warp
      mbar_init(bars + kBarTFree + 8 * j, kW);
      mbar_init(bars + kBarLFull + 8 * j, 1);
      mbar_init(bars + kBarLFree + 8 * j, 1);
    }
    mbar_init(bars + kBarX, 1);
    for (int j = 0; j < kMaxRing; ++j) {
      for (int h = 0; h < kRingParts; ++h) {
        mbar_init(bars + kBarSFull + 8 * (h * kMaxRing + j), 1);
        mbar_init(bars + kBarSEmpty + 8 * (h * kMaxRing + j), kW / kRingParts);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem + P.red);
  if (warp == kProducerWarp) {
    if (lane < kRingParts) producer_loop(P, bars, sbase, b, lane);  // lane h feeds part ring h
    return;
  }
  if (warp == kWriterWarp) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    writer_loop<MP>(P, red, bars, sbase, b, lane);
    return;
  }
  // Builder warp: item g's pair table into buffer g & 1 once the compute warps
  // released item g - 2's (tfree) and the LUT rows landed; the compute warps no
  // longer build slices between items, so they never wait for each other there
  // (chain 51.6 -> 50.2 us, gate 15.0 -> 14.7 us)
  // Dependency warp: the compute warps' x hand-offs (bar_x), one per image that
  // needs one — the CTA's first image (earlier kernels' memory, after
  // griddepcontrol.wait) and every image that is another problem's y (after
  // every CTA released that problem); an input x needs none, the compute warps
  // apply the same rule. In its own warp the wait no longer queues behind the
  // writer's last items (8B chain 47.0 -> 42.9 us).
  if (warp == kDepWarp) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    Item it = item_begin(P, b);
    int staged = -1;
    for (int p = 0; p < P.np; ++p) {
      const GvProb& q = P.p[p];
      if (it.p == p && q.img != staged) {
        if (q.dep >= 0 || staged < 0) {
          if (lane == 0) {
            if (q.dep >= 0) wait_geq(&P.done[q.dep], P.ncta);
            mbar_arrive(bars + kBarX);
          }
          __syncwarp();
        }
        staged = q.img;
      }
      while (it.p == p) item_next(P, b, it);
    }
    return;
  }
  if (warp == kBuilderWarp) {
    const uint32_t lutrow = sbase + P.lutbuf + (uint32_t)lane * 32;
    Item it = item_begin(P, b);
    for (int gi = 0; it.p < P.np; ++gi) {
      const int nb = gi & 1;
      if (gi >= 2) mbar_wait(bars + kBarTFree + 8 * nb, (uint32_t)(((gi - 2) >> 1) & 1));
      mbar_wait(bars + kBarLFull + 8 * nb, (uint32_t)((gi >> 1) & 1));
      const uint4 l0 = lds128(lutrow + nb * 1024), l1 = lds128(lutrow + nb * 1024 + 16);
#pragma unroll 4
      for (int hi = 0; hi < 16; ++hi) build_table(l0, l1, hi, nb, laneoff);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bars + kBarLFree + 8 * nb);
        mbar_arrive(bars + kBarTReady + 8 * nb);
      }
      item_next(P, b, it);
    }
    return;
  }

  // ---- compute warps: shared memory only ------------------------------------
  const uint32_t tready = bars + kBarTReady, tfree = bars + kBarTFree;
  const int half = warp / kPartChunks;  // part ring
  const uint32_t sfull = bars + kBarSFull + 8u * kMaxRing * half, sempty = bars + kBarSEmpty + 8u * kMaxRing * half;
  const uint32_t abring = sbase + P.abring + laneoff + (uint32_t)half * (kStageAb / kRingParts);
  const uint32_t bar_full = bars + kBarRedFull, bar_empty = bars + kBarRedEmpty;
  const uint32_t ring = sbase + (uint32_t)warp * 2048 + lane * 16;
  Item s = item_begin(P, b);
  Item nx = s;
  item_next(P, b, nx);

  GV_TRACE(1);

  int xbatch = 0;     // x images staged so far (parity of bar_x)
  int cur_img = -1;   // x image the compute warps hold
  int g = 0;          // items processed by this CTA
  int slot = 0;       // ring stage
  uint32_t round = 0;
  while (s.p < P.np) {
    const int p = s.p;
    const GvProb& q = P.p[p];
    if (q.img != cur_img) {  // first item on a new x image: load and convert it
      if (q.dep >= 0 || cur_img < 0) {  // the writer's hand-off (see writer_loop)
        mbar_wait(bars + kBarX, (uint32_t)(xbatch & 1));
        ++xbatch;
      }
      // each warp converts exactly the chunks it reads (c = warp + 16 i, lane
      // group i % 4 per pass): the image needs no CTA barrier
      const int nmine = (q.C - warp + kW - 1) / kW;  // chunks of this warp
      for (int m = 0; m < MP; ++m)
        for (int i0 = 0; i0 < nmine; i0 += 4)
          prep_x<MP>(q, P.M, smem, m, warp + kW * (i0 + (lane >> 3)), lane);
      cur_img = q.img;
      GV_TRACE(2 + (q.img & 7));
    }
    const uint32_t tb = kTblAddr | ((uint32_t)(g & 1) << 7) | laneoff;
    mbar_wait(tready + 8 * (g & 1), (uint32_t)((g >> 1) & 1));
    float y[MP];
#pragma unroll
    for (int m = 0; m < MP; ++m) y[m] = 0.0f;
    const uint32_t xstride = (uint32_t)q.C * 256, xsstride = (uint32_t)q.C * 8;
    const uint32_t xa0 = sbase + q.xh + (uint32_t)warp * 256, xsa0 = sbase + q.xs + (uint32_t)warp * 8;
    for (int c0 = 0; c0 < q.C; c0 += kStageChunks) {
      mbar_wait(sfull + 8 * slot, round & 1);
      const int c = c0 + warp;
      Chunk ch;
      if (c < q.C) {
        const uint32_t a = ring + P.ring[slot];
#pragma unroll
        for (int j = 0; j < 4; ++j) ch.w[j] = lds128(a + j * 512);
        ch.ab = lds32(abring + slot * kStageAb +
                      (uint32_t)(((c >> q.gshift) - ((c0 + kPartChunks * half) >> q.gshift)) << 7));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty + 8 * slot);  // release orders the reads above
#ifdef GV_SKIPCOMPUTE  // transport-only experiment build (never the shipped library)
      if (c < q.C) y[0] += __uint_as_float((ch.w[0].x ^ ch.w[1].y ^ ch.w[2].z ^ ch.w[3].w ^ ch.ab) & 0x3fffffff) * 1e-30f;
#else
      if (c < q.C)
        consume<MP>(ch, tb, xa0 + (uint32_t)c0 * 256, xsa0 + (uint32_t)c0 * 8, xstride, xsstride, y);
#endif
      if (++slot == P.nring) {
        slot = 0;
        ++round;
      }
    }
    // partial sums to the writer warp
    const int par = g & 1;
    if (g >= 2) mbar_wait(bar_empty + 8 * par, (uint32_t)(((g >> 1) - 1) & 1));
    float* rp = red + (size_t)par * kW * MP * 32;
#pragma unroll
    for (int m = 0; m < MP; ++m) rp[(warp * MP + m) * 32 + lane] = y[m];
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(bar_full + 8 * par);
      mbar_arrive(tfree + 8 * (g & 1));  // done reading this item's table
    }
    // the next item's table goes into the other buffer

    if (g < 31) GV_TRACE(32 + g);
    s = nx;
    item_next(P, b, nx);
    ++g;
  }
  GV_TRACE(63);
}

// ===========================================================================
// K1t — the same persistent chain, with the products on the tensor cores.
//
// The CUDA-core compute warps above spend ~2 FHFMA per code byte per x row,
// so they are issue bound at M = 1 and scale linearly in M. Here the 16
// "dequant" warps only look weights up (one PRMT + one LDS per two weights,
// the same pair table) and store the fp16 pairs straight into tensor memory
// (tcgen05.st); one thread issues tcgen05.mma kind::f16 (M = 128, K = 16,
// A from TMEM, B = the x image in shared memory, fp32 accumulators in TMEM),
// so the cost per weight no longer depends on M (1..16).
//
//  * A chunk group = 4 consecutive 128-k chunks of one 32-row block. TMEM
//    lane quarter q (warps q, q+4, q+8, q+12) holds chunk 4g+q: warp (q, j)
//    dequantises slab j of that chunk, i.e. k in {16j..16j+15} (MMA step 2j)
//    and {64+16j..} (step 2j+1), into A columns 16j..16j+15. 8 MMAs (K = 16)
//    cover the group; B step t holds, in column block q' (MP columns = x
//    rows), x of chunk 4g+q' at the step's k, so D[(q, row), (q', m)] is the
//    chunk-q dot product when q' = q (the other blocks are never read).
//  * 4 epilogue warps (quarter q each) read their MP accumulator columns per
//    group (tcgen05.ld), apply alpha * 2^-e and beta * sum x per chunk
//    exactly as K1a does, and hand per-item quarter partials to the writer.
//  * x images are converted by the dequant warps straight from global
//    memory (ld.cg, after the writer saw the dependency released) into the
//    UMMA K-major no-swizzle layout: per 64-k MMA step [rowgroup][k half]
//    [8 rows][16 B], LBO 128 B, SBO 256 B, row n = q'*MP + m.
//  * Producer, writer, item schedule, dependencies, pair table and its
//    buffers are those of K1a; alpha/beta come through their own ring so
//    the code ring is released as soon as the dequant warps read it.
//  * A single GEMM whose x image does not fit (m x K too large) runs as up to
//    8 K-slices in one launch: slice s is a problem over chunks [c0, c0 + nc)
//    (codes, scales and x offset, row strides of the whole tensor) that waits
//    for slice s - 1 and adds its fp32 partial (the caller's y32, else stream
//    scratch) before its own: deterministic. Image rows m >= M are zero.
// ===========================================================================
// debug trace of K1t: [ncta][8 events][64 chunk groups] behind K1a's [ncta][64]
#ifdef TC_TRACE_ON  // experiment builds only: the stamps perturb the pipeline
#define TC_TRACE(ev, i)                                                                        \
  do {                                                                                         \
    if (P.trace && (i) < 64) P.trace[148 * 64 + (blockIdx.x * 8 + (ev)) * 64 + (i)] = gtimer(); \
  } while (0)
#else
#define TC_TRACE(ev, i) \
  do {                  \
  } while (0)
#endif
constexpr int kTcDq = 16;                 // dequant warps
constexpr int kTcEpi0 = 16;               // epilogue warps 16..19 (quarter = warp & 3)
constexpr int kTcMma = 20;
constexpr int kTcWriter = 21;
constexpr int kTcProducer = 22;
constexpr int kTcBuilder = 23;            // builds every item's pair table, one item ahead
constexpr int kTcT = 24 * 32;
constexpr int kTcNA = 8;                  // A-slot barriers (one chunk group = 64 TMEM columns each)
constexpr int kTcND = 8;                  // accumulator-slot barriers
constexpr int kTcAbRing = 4;              // alpha/beta ring stages (2 KB each)
constexpr int kTcTmemCols = 512;
constexpr int kTcMaxMP = 16;
// mbarriers (8 B each) of K1t
constexpr uint32_t kTbRedFull = 0, kTbRedEmpty = 16, kTbX = 32, kTbXReady = 40, kTbTReady = 48,
                   kTbTFree = 64, kTbLFull = 80, kTbLFree = 96, kTbSFull = 112,
                   kTbSEmpty = kTbSFull + 8 * kTcMaxRing, kTbAbFull = kTbSEmpty + 8 * kTcMaxRing,
                   kTbAbEmpty = kTbAbFull + 8 * kTcAbRing, kTbAFull = kTbAbEmpty + 8 * kTcAbRing,
                   kTbAFree = kTbAFull + 8 * kTcNA, kTbDFull = kTbAFree + 8 * kTcNA,
                   kTbDFree = kTbDFull + 8 * kTcND, kTbTmemSlot = kTbDFree + 8 * kTcND,
                   kTbBytes = kTbTmemSlot + 16;

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, "
      "p; }" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
template <int MP>
__device__ __forceinline__ void tc_ld(uint32_t taddr, float (&r)[MP]) {
  uint32_t u[MP];
  if constexpr (MP == 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                 : "=r"(u[0]), "=r"(u[1])
                 : "r"(taddr)
                 : "memory");
  } else if constexpr (MP == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3])
                 : "r"(taddr)
                 : "memory");
  } else if constexpr (MP == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]),
                   "=r"(u[6]), "=r"(u[7])
                 : "r"(taddr)
                 : "memory");
  } else {
    static_assert(MP == 16, "MP in {2, 4, 8, 16}");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
          "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
          "=r"(u[14]), "=r"(u[15])
        : "r"(taddr)
        : "memory");
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < MP; ++i) r[i] = __uint_as_float(u[i]);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(pred));
  return pred != 0;
}
// UMMA shared-memory descriptor: K-major, no swizzle, LBO 128 B (k halves),
// SBO 256 B (8-row groups), version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}

// x of problem q -> the K1t B image: lane group (lane >> 3) of the warp owns
// (m, c), lane sub = lane & 7 the 16 consecutive k = 128c + 16 sub + t; chunk
// scale 2^e and sum x per (m, c) as in prep_x. Reads x from global (L2).
template <int MP>
__device__ __forceinline__ void prep_x_tc(const GvProb& q, int M, uint8_t* smem, int idx, int lane) {
  const int sub = lane & 7;
  const int m = idx / q.C, c = idx - m * q.C;
  const bool live = idx < M * q.C;   // a real x row: load it
  const bool img = idx < MP * q.C;   // an image row (rows m >= M are written as zeros)
  const int k0 = c * 128 + sub * 16;
  float v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) v[t] = 0.0f;
  if (live) {
    const __nv_bfloat16* xr = q.x + (size_t)m * q.xstride;
    if (q.tma && k0 + 16 <= q.K) {  // 16-B aligned rows (K % 128 == 0, x 16-B aligned)
      const uint4 r0 = __ldcg(reinterpret_cast<const uint4*>(xr + k0));
      const uint4 r1 = __ldcg(reinterpret_cast<const uint4*>(xr + k0 + 8));
      const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const __nv_bfloat162 p2 = *reinterpret_cast<const __nv_bfloat162*>(&w[t]);
        v[2 * t] = __low2float(p2);
        v[2 * t + 1] = __high2float(p2);
      }
    } else {
      const unsigned short* xs = reinterpret_cast<const unsigned short*>(xr);
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (k0 + t < q.K) v[t] = __bfloat162float(__ushort_as_bfloat16(__ldcg(xs + k0 + t)));
    }
  }
  float amax = 0.0f, sum = 0.0f;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    amax = fmaxf(amax, fabsf(v[t]));
    sum += v[t];
  }
#pragma unroll
  for (int off = 4; off; off >>= 1) {
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    sum += __shfl_xor_sync(0xffffffffu, sum, off);
  }
  const int ex = (__float_as_int(amax) >> 23) & 0xff;
  const int e = (amax > 0.0f && ex < 255) ? min(141 - ex, 126) : 0;
  const float sc = __int_as_float((127 + e) << 23), isc = __int_as_float((127 - e) << 23);
  uint32_t h[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const __half2 p2 = __floats2half2_rn(v[2 * t] * sc, v[2 * t + 1] * sc);
    h[t] = *reinterpret_cast<const uint32_t*>(&p2);
  }
  if (img) {
    // k = 16 sub + t: MMA step 2 sub (sub < 4) or 2 (sub - 4) + 1, row n = q' MP + m
    const int st = sub < 4 ? 2 * sub : 2 * (sub - 4) + 1;
    const int n = (c & 3) * MP + m;
    uint8_t* dst = smem + q.xh + (size_t)(c >> 2) * (1024 * MP) + st * (128 * MP) + (n >> 3) * 256 +
                   (n & 7) * 16;
    *reinterpret_cast<uint4*>(dst) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(dst + 128) = make_uint4(h[4], h[5], h[6], h[7]);
    if (sub == 0) *reinterpret_cast<float2*>(smem + q.xs + ((size_t)m * q.C + c) * 8) = make_float2(isc, sum);
  }
}

// Writer of K1t: K1a's writer with 4 quarter partials per item and no x
// staging (the dequant warps read x themselves once bar_x is released).
template <int MP>
__device__ __forceinline__ void writer_loop_tc(const GvParams& P, const float* red, uint32_t bars,
                                               int b, int lane) {
  const uint32_t bar_full = bars + kTbRedFull, bar_empty = bars + kTbRedEmpty;
  Item it = item_begin(P, b);
  int g = 0, staged = -1;
  for (int p = 0; p < P.np; ++p) {
    const GvProb& q = P.p[p];
    if (it.p == p && q.img != staged) {
      if (lane == 0) {
        if (q.dep >= 0) wait_geq(&P.done[q.dep], P.ncta);
        mbar_arrive(bars + kTbX);
      }
      __syncwarp();
      staged = q.img;
    }
    // K-slices: every lane acquires the earlier slices' partials it adds
    if (it.p == p && q.acc_in) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    while (it.p == p) {
      const int par = g & 1;
      mbar_wait_sleep(bar_full + 8 * par, (uint32_t)((g >> 1) & 1));
      const float* rp = red + (size_t)par * 4 * MP * 32;
      float acc[MP];
#pragma unroll
      for (int m = 0; m < MP; ++m)
        acc[m] = ((rp[(0 * MP + m) * 32 + lane] + rp[(1 * MP + m) * 32 + lane]) +
                  rp[(2 * MP + m) * 32 + lane]) +
                 rp[(3 * MP + m) * 32 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + 8 * par);
      const int row = it.rb * 32 + lane;
      if (row < q.N) {
#pragma unroll
        for (int m = 0; m < MP; ++m) {
          if (m < P.M) {
            const size_t o = (size_t)m * q.N + row;
            // K-slices: the earlier slices' sum first (written by the problem this
            // one waits for), then this slice's
            if (q.acc_in) acc[m] = __fadd_rn(__ldcg(q.acc_in + o), acc[m]);
            if (q.acc_out) {
              q.acc_out[o] = acc[m];
            } else {
              q.y[o] = __float2bfloat16_rn(acc[m]);
              if (q.y32) q.y32[o] = acc[m];
            }
          }
        }
      }
      item_next(P, b, it);
      ++g;
    }
    __syncwarp();
    if (lane == 0) {
      if (p < P.np - 1) {
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&P.done[p]) : "memory");
      } else {
        __threadfence();
        const int old = atomicAdd(&P.done[p], 1);
        if (old == P.ncta - 1)
          for (int r = 0; r < P.np; ++r) P.done[r] = 0;
      }
    }
    __syncwarp();
  }
}

// Producer of K1t: K1a's, with alpha/beta through their own ring.
__device__ __forceinline__ void producer_loop_tc(const GvParams& P, uint32_t bars, uint32_t sbase,
                                                 int b) {
  // A stage = the next 4 chunk groups of the CTA's sequence (group p of the
  // stage goes to team p), possibly from different items: one empty wait,
  // one expect_tx and up to 4 bulk copies per stage for the codes and for
  // the alpha/beta lines each. An item's LUT rows go out with its first group.
  const uint32_t lfull = bars + kTbLFull, lfree = bars + kTbLFree;
  const uint32_t sfull = bars + kTbSFull, sempty = bars + kTbSEmpty;
  const uint32_t abfull = bars + kTbAbFull, abempty = bars + kTbAbEmpty;
  const uint32_t abring = sbase + P.abring, lutbuf = sbase + P.lutbuf;
  Item it = item_begin(P, b);
  int g = 0, gi = 0, slot = 0, aslot = 0;
  uint32_t round = 0, around = 0;
  // L2 prefetch of a whole item (codes + alpha/beta), one item ahead of the
  // ring: the ring's shared memory bounds the bytes in flight, the L2 does not
  auto prefetch_item = [&](const Item& x) {
#ifndef TC_NOPREFETCH
    if (x.p >= P.np) return;
    const GvProb& q = P.p[x.p];
    const uint8_t* c = reinterpret_cast<const uint8_t*>(q.codes) + (size_t)x.rb * q.cstride * 2048;
    for (uint32_t o = 0, n = (uint32_t)q.C * 2048; o < n; o += 32768) prefetch_l2(c + o, min(32768u, n - o));
    prefetch_l2(reinterpret_cast<const uint8_t*>(q.ab) + (size_t)x.rb * q.GR * 128, (uint32_t)q.GR * 128);
#endif
  };
  prefetch_item(it);
  while (it.p < P.np) {
    const uint8_t* src[kTcStageGroups];
    const uint8_t* asrc[kTcStageGroups];
    uint32_t nb[kTcStageGroups], anb[kTcStageGroups];
    int ng = 0;
    uint32_t tot = 0, atot = 0;
    while (ng < kTcStageGroups && it.p < P.np) {
      const GvProb& q = P.p[it.p];
      if (gi == 0) {  // the item's LUT rows; the next item into L2
        Item nx2 = it;
        item_next(P, b, nx2);
        prefetch_item(nx2);
        const int lb = g & 1;
        if (g >= 2) mbar_wait(lfree + 8 * lb, (uint32_t)(((g >> 1) - 1) & 1));
        mbar_expect_tx(lfull + 8 * lb, 1024);
        bulk_g2s(lutbuf + lb * 1024, reinterpret_cast<const uint8_t*>(q.lut) + (size_t)it.rb * 1024, 1024,
                 lfull + 8 * lb);
      }
      const int c0 = 4 * gi, n = min(4, q.C - c0);
      const int g0 = c0 >> q.gshift, g1 = (c0 + n - 1) >> q.gshift;
      src[ng] = reinterpret_cast<const uint8_t*>(q.codes) + ((size_t)it.rb * q.cstride + c0) * 2048;
      nb[ng] = (uint32_t)n * 2048;
      asrc[ng] = reinterpret_cast<const uint8_t*>(q.ab) + ((size_t)it.rb * q.GR + g0) * 128;
      anb[ng] = (uint32_t)(g1 - g0 + 1) * 128;
      tot += nb[ng];
      atot += anb[ng];
      ++ng;
      if (4 * ++gi >= q.C) {
        gi = 0;
        ++g;
        item_next(P, b, it);
      }
    }
    if (round > 0) mbar_wait(sempty + 8 * slot, (round - 1) & 1);
    mbar_expect_tx(sfull + 8 * slot, tot);
    for (int p = 0; p < ng; ++p)
      bulk_g2s(sbase + P.ring[slot] + p * kTcGroupBytes, src[p], nb[p], sfull + 8 * slot);
    if (around > 0) mbar_wait(abempty + 8 * aslot, (around - 1) & 1);
    mbar_expect_tx(abfull + 8 * aslot, atot);
    for (int p = 0; p < ng; ++p)
      bulk_g2s(abring + aslot * kTcStageAb + p * kTcGroupAb, asrc[p], anb[p], abfull + 8 * aslot);
    if (++slot == P.nring) {
      slot = 0;
      ++round;
    }
    if (++aslot == kTcAbRing) {
      aslot = 0;
      ++around;
    }
  }
}

template <int MP>
__global__ void __launch_bounds__(kTcT, 1) k_lutgemv_tc(const __grid_constant__ GvParams Pk) {
  constexpr int NB = 4 * MP;  // MMA N: 4 column blocks (one per chunk of the group) of MP x rows
  constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(NB >> 3) << 17) | ((128u >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem[];
  asm volatile("griddepcontrol.launch_dependents;");
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&Pk);
    uint32_t* dst = reinterpret_cast<uint32_t*>(smem + kParamOff);
    for (int i = threadIdx.x; i < (int)(sizeof(GvParams) / 4); i += kTcT) dst[i] = src[i];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x;
  const uint32_t laneoff = (uint32_t)lane << 2;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const GvParams& P = *reinterpret_cast<const GvParams*>(smem + kParamOff);
  __syncthreads();
  const uint32_t bars = sbase + P.bars;
  if (sbase != kDynBase) {
    if (threadIdx.x == 0) atomicMax(P.err, (int)ANYQ_ERR_INTERNAL);
    return;
  }
  if (threadIdx.x == 0) {
    for (int j = 0; j < 2; ++j) {
      mbar_init(bars + kTbRedFull + 8 * j, 4);
      mbar_init(bars + kTbRedEmpty + 8 * j, 1);
      mbar_init(bars + kTbTReady + 8 * j, 1);
      mbar_init(bars + kTbTFree + 8 * j, kTcDq);
      mbar_init(bars + kTbLFull + 8 * j, 1);
      mbar_init(bars + kTbLFree + 8 * j, 1);
    }
    mbar_init(bars + kTbX, 1);
    mbar_init(bars + kTbXReady, kTcDq);
    for (int j = 0; j < kTcMaxRing; ++j) {
      mbar_init(bars + kTbSFull + 8 * j, 1);
      mbar_init(bars + kTbSEmpty + 8 * j, kTcDq);
    }
    for (int j = 0; j < kTcAbRing; ++j) {
      mbar_init(bars + kTbAbFull + 8 * j, 1);
      mbar_init(bars + kTbAbEmpty + 8 * j, 4);  // the epilogue warps
    }
    for (int j = 0; j < kTcNA; ++j) {
      mbar_init(bars + kTbAFull + 8 * j, 4);   // team j's 4 warps
      mbar_init(bars + kTbAFree + 8 * j, 1);
    }
    for (int j = 0; j < kTcND; ++j) {
      mbar_init(bars + kTbDFull + 8 * j, 1);
      mbar_init(bars + kTbDFree + 8 * j, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P.bars + kTbTmemSlot);
  if (warp == kTcMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     sbase + P.bars + kTbTmemSlot),
                 "r"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // A slots: as many 64-column slots as TMEM leaves next to the accumulator
  // slots (MP 2: 7, MP 4: 6, MP 8: 6, MP 16: 4), round-robin over the CTA's
  // groups, so a team starts its next group while the MMA still reads its last
  // accumulator slots: 8 where they are narrow (MP <= 4: the MMA runs further
  // ahead of the epilogue, 1-2 % faster), else 4
  constexpr int ND = NB <= 16 ? 8 : 4;
  constexpr int NA = (512 - ND * NB) / 64 > 7 ? 7 : (512 - ND * NB) / 64;
  static_assert(NA >= 4 && NA <= kTcNA, "A slots");
  constexpr uint32_t kDCol0 = NA * 64;
  float* red = reinterpret_cast<float*>(smem + P.red);

  if (warp == kTcProducer) {
    if (lane == 0) producer_loop_tc(P, bars, sbase, b);
    return;
  }
  if (warp == kTcBuilder) {
    // pair table of item g into buffer g & 1 (lane L = row L, all 16 high nibbles)
    const uint32_t lutrow = sbase + P.lutbuf + (uint32_t)lane * 32;
    Item it = item_begin(P, b);
    for (int g = 0; it.p < P.np; ++g) {
      const int nb = g & 1;
      if (g >= 2) mbar_wait(bars + kTbTFree + 8 * nb, (uint32_t)(((g - 2) >> 1) & 1));
      mbar_wait(bars + kTbLFull + 8 * nb, (uint32_t)((g >> 1) & 1));
      const uint4 l0 = lds128(lutrow + nb * 1024), l1 = lds128(lutrow + nb * 1024 + 16);
#pragma unroll 4
      for (int hi = 0; hi < 16; ++hi) build_table(l0, l1, hi, nb, laneoff);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bars + kTbLFree + 8 * nb);
        mbar_arrive(bars + kTbTReady + 8 * nb);
      }
      item_next(P, b, it);
    }
    return;
  }
  if (warp == kTcWriter) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    writer_loop_tc<MP>(P, red, bars, b, lane);
    return;
  }

  if (warp == kTcMma) {
    // ------------------------------------------------------------ MMA issue
    Item s = item_begin(P, b);
    int cg = 0, cur_img = -1, xr = 0;
    while (s.p < P.np) {
      const GvProb& q = P.p[s.p];
      bool need_x = q.img != cur_img;
      cur_img = q.img;
      const int ngrp = (q.C + 3) >> 2;
      const uint32_t xb = sbase + q.xh;
      for (int gi = 0; gi < ngrp; ++gi, ++cg) {
        const int a = cg % NA, d = cg % ND;
        mbar_wait(bars + kTbAFull + 8 * a, (uint32_t)((cg / NA) & 1));
        if (lane == 0) TC_TRACE(4, cg);
        if (cg >= ND) mbar_wait(bars + kTbDFree + 8 * d, (uint32_t)(((cg / ND) - 1) & 1));
        if (need_x) {
          mbar_wait(bars + kTbXReady, (uint32_t)(xr & 1));
          ++xr;
          need_x = false;
        }
        tc_fence_after();
        if (elect_one()) {
          const uint32_t bg = xb + (uint32_t)gi * (1024u * MP);
#ifdef TC_NOMMA  // experiment build: hand the slots on without the tensor core
          (void)bg;
          mbar_arrive(bars + kTbAFree + 8 * a);
          mbar_arrive(bars + kTbDFull + 8 * d);
#else
#pragma unroll
          for (int t = 0; t < 8; ++t)
            tc_mma(tmem + kDCol0 + d * NB, tmem + a * 64 + 8 * t, umma_desc(bg + t * (128u * MP)), kIdesc,
                   t > 0 ? 1u : 0u);
          tc_commit(bars + kTbAFree + 8 * a);
          tc_commit(bars + kTbDFull + 8 * d);
#endif
          TC_TRACE(5, cg);
        }
        __syncwarp();
      }
      item_next(P, b, s);
    }
  } else if (warp >= kTcEpi0) {
    // ------------------------------------------------------------ epilogue
    const int qq = warp & 3;
    const uint32_t tq = tmem + ((uint32_t)(32 * qq) << 16) + kDCol0 + qq * MP;
    const uint32_t abring = sbase + P.abring + laneoff;
    Item s = item_begin(P, b);
    int cg = 0, aslot = 0, gpar = 0;
    uint32_t around = 0;
    while (s.p < P.np) {
      const GvProb& q = P.p[s.p];
      float y[MP];
#pragma unroll
      for (int m = 0; m < MP; ++m) y[m] = 0.0f;
      const int ngrp = (q.C + 3) >> 2;
      const float2* xs = reinterpret_cast<const float2*>(smem + q.xs);
      for (int gi = 0; gi < ngrp; ++gi, ++cg) {
        const int c0 = 4 * gi;
        if ((cg & 3) == 0) mbar_wait(bars + kTbAbFull + 8 * aslot, around & 1);
        const int d = cg % ND;
        mbar_wait(bars + kTbDFull + 8 * d, (uint32_t)((cg / ND) & 1));
        if (qq == 0 && lane == 0) TC_TRACE(6, cg);
        tc_fence_after();
        float r[MP];
#ifdef TC_NOEPI  // experiment build: accumulators are not read
#pragma unroll
        for (int m = 0; m < MP; ++m) r[m] = 0.0f;
#else
        tc_ld<MP>(tq + d * NB, r);
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bars + kTbDFree + 8 * d);
        const int c = 4 * gi + qq;
        if (c < q.C) {
          const uint32_t abw =
              lds32(abring + aslot * kTcStageAb + (uint32_t)(cg & 3) * kTcGroupAb +
                    (uint32_t)(((c >> q.gshift) - (c0 >> q.gshift)) << 7));
          const float2 ab = __half22float2(*reinterpret_cast<const __half2*>(&abw));
#pragma unroll
          for (int m = 0; m < MP; ++m) {
            const float2 sc = xs[m * q.C + c];
            y[m] = fmaf(ab.x, sc.x * r[m], fmaf(ab.y, sc.y, y[m]));
          }
        }
        if ((cg & 3) == 3) {
          __syncwarp();
          if (lane == 0) mbar_arrive(bars + kTbAbEmpty + 8 * aslot);
          if (++aslot == kTcAbRing) {
            aslot = 0;
            ++around;
          }
        }
      }
      const int par = gpar & 1;
      if (gpar >= 2) mbar_wait(bars + kTbRedEmpty + 8 * par, (uint32_t)(((gpar >> 1) - 1) & 1));
      float* rp = red + (size_t)par * 4 * MP * 32;
#pragma unroll
      for (int m = 0; m < MP; ++m) rp[(qq * MP + m) * 32 + lane] = y[m];
      __syncwarp();
      if (lane == 0) mbar_arrive(bars + kTbRedFull + 8 * par);
      ++gpar;
      item_next(P, b, s);
    }
  } else {
    // ------------------------------------------------------------ dequant
    // 4 teams of 4 warps; team t = warp >> 2 takes the chunk groups cg = t
    // (mod 4) of the CTA's sequence (its own A slot t, ring slots = t mod 4),
    // so four groups are in flight and each hand-off covers 64 lookups per
    // warp. Warp (t, q) dequantises chunk 4 gi + q of a group: its 4 slabs
    // (k in {16j..16j+15, 64+16j..}) into A columns 16j..16j+15 of TMEM lane
    // quarter q. Every warp still builds its slice of every item's table.
    const int qq = warp & 3, team = warp >> 2;
    const uint32_t tq0 = tmem + ((uint32_t)(32 * qq) << 16);
    const uint32_t tready = bars + kTbTReady, tfree = bars + kTbTFree;
    Item s = item_begin(P, b);
    int xbatch = 0, cur_img = -1, g = 0, base = 0, slot = 0, k = 0;
    uint32_t round = 0;
    while (s.p < P.np) {
      const GvProb& q = P.p[s.p];
      if (q.img != cur_img) {  // convert the new x image (x may be an earlier problem's y)
        mbar_wait_sleep(bars + kTbX, (uint32_t)(xbatch & 1));
        ++xbatch;
        for (int i0 = warp * 4; i0 < MP * q.C; i0 += kTcDq * 4)  // padding rows m >= M as zeros
          prep_x_tc<MP>(q, P.M, smem, i0 + (lane >> 3), lane);
        // generic-proxy writes of the image -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(bars + kTbXReady);
        cur_img = q.img;
      }
      const int ngrp = (q.C + 3) >> 2;
      // this team's first group of the item: the CTA-wide group index ≡ team (mod 4)
      int gi = (team - base) & 3;
      if (gi < ngrp) {
        const uint32_t tb = kTblAddr | ((uint32_t)(g & 1) << 7) | laneoff;
        mbar_wait(tready + 8 * (g & 1), (uint32_t)((g >> 1) & 1));
        for (; gi < ngrp; gi += 4, ++k) {
          const int cga = team + 4 * k;  // this group's CTA-wide index
          const int as = cga % NA;
          const uint32_t tq = tq0 + (uint32_t)as * 64;
          mbar_wait(bars + kTbSFull + 8 * slot, round & 1);
          const bool live = 4 * gi + qq < q.C;
          if (live) {
            const uint32_t ra = sbase + P.ring[slot] + (uint32_t)team * kTcGroupBytes + (uint32_t)qq * 2048 + lane * 16;
            uint4 w[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) w[jj] = lds128(ra + jj * 512);
            __syncwarp();
            if (lane == 0) mbar_arrive(bars + kTbSEmpty + 8 * slot);  // codes are in registers
            if (cga >= NA) mbar_wait(bars + kTbAFree + 8 * as, (uint32_t)(((cga / NA) - 1) & 1));
            tc_fence_after();
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const uint32_t wd[4] = {w[jj].x, w[jj].y, w[jj].z, w[jj].w};
              uint32_t t[16];
#pragma unroll
              for (int bb = 0; bb < 16; ++bb)
#ifdef TC_NOLOOKUP  // experiment build: addresses without the table reads
                t[bb] = __byte_perm(wd[bb >> 2], tb, 0x7604u | ((uint32_t)(bb & 3) << 4));
#else
                t[bb] = lds32(__byte_perm(wd[bb >> 2], tb, 0x7604u | ((uint32_t)(bb & 3) << 4)));
#endif
#ifdef TC_NOST  // experiment build: no TMEM stores (the MMAs read stale A)
              asm volatile("" ::"r"(t[0] ^ t[5] ^ t[10] ^ t[15]));
#else
              tc_st16(tq + 16 * jj, t);
#endif
            }
#ifndef TC_NOST
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#endif
          } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(bars + kTbSEmpty + 8 * slot);
            if (cga >= NA) mbar_wait(bars + kTbAFree + 8 * as, (uint32_t)(((cga / NA) - 1) & 1));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bars + kTbAFull + 8 * as);
          if (++slot == P.nring) {
            slot = 0;
            ++round;
          }
        }
      }
      base += ngrp;
      __syncwarp();
      if (lane == 0) mbar_arrive(tfree + 8 * (g & 1));
      item_next(P, b, s);
      ++g;
    }
  }
  // every TMEM user is done (the producer and writer returned above)
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"r"((kTcMma + 1) * 32) : "memory");
  if (warp == kTcMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcTmemCols));
  }
}

long long* g_gv_trace = nullptr;

// Per-problem parameters, batches and shared-memory placement; returns the
// dynamic shared memory bytes. TC: the K1t layout (x images in the UMMA
// layout, 4 quarter partials, the alpha/beta ring).
struct KSlice {   // one K-slice of a sliced single GEMM (K1t)
  int c0, nc;      // chunks [c0, c0 + nc)
  const float* acc_in;
  float* acc_out;
};

template <int MP, bool TC = false>
uint32_t plan_chain(int n, const LutTensor* const* ts, const void* const* xs, void* const* ys,
                    float* const* y32s, const int32_t* deps, int64_t m, GvParams& P,
                    const KSlice* slices = nullptr) {
  if (n < 1 || n > kMaxProb) fail(ANYQ_ERR_SHAPE, "LUT GEMV chain: 1..8 problems");
  P.np = n;
  P.M = (int)m;
  P.ncta = ts[0]->gv_ncta;
  P.err = nullptr;  // set per launch (stream workspace)
  P.done = nullptr;
  P.tp_world = 0;
  P.tp_rank = 0;
  P.tp_row0 = 0;
  P.tp_N = 0;
  P.trace = g_gv_trace;
  // dependencies, x images and the chain's item sequence
  int tot = 0;
  for (int i = 0; i < n; ++i) {
    const LutTensor* t = ts[i];
    if (!t) fail(ANYQ_ERR_SHAPE, "null device tensor");
    if (t->gv_gshift < 0)
      fail(ANYQ_ERR_CONFIG, "LUT GEMV needs rowwise scales or group_size = 128 * 2^j");
    if (t->gv_ncta != P.ncta) fail(ANYQ_ERR_SHAPE, "chain tensors were prepared for different devices");
    GvProb& q = P.p[i];
    q.codes = reinterpret_cast<const uint4*>(t->codes);
    q.lut = reinterpret_cast<const uint4*>(t->lut);
    q.ab = reinterpret_cast<const uint32_t*>(t->ab);
    q.x = reinterpret_cast<const __nv_bfloat16*>(xs[i]);
    q.y = reinterpret_cast<__nv_bfloat16*>(ys[i]);
    q.y32 = y32s ? y32s[i] : nullptr;
    q.N = (int)t->rows;
    q.K = (int)t->cols;
    q.C = t->C;
    q.GR = t->GR;
    q.RB = t->RB;
    q.gshift = t->gv_gshift;
    q.cstride = t->C;
    q.xstride = (int)t->cols;
    q.acc_in = nullptr;
    q.acc_out = nullptr;
    if (slices) {
      const KSlice& sl = slices[i];
      q.codes += (size_t)sl.c0 * 128;  // 2048-B chunks of uint4
      if (t->GR > 1) q.ab += (size_t)(sl.c0 >> q.gshift) * 32;
      q.x += (size_t)sl.c0 * 128;
      q.K = std::min((int)t->cols - sl.c0 * 128, sl.nc * 128);
      q.C = sl.nc;
      q.acc_in = sl.acc_in;
      q.acc_out = sl.acc_out;
    }
    q.dep = deps ? deps[i] : -1;
    if (q.dep < -1 || q.dep >= i) fail(ANYQ_ERR_SHAPE, "chain dependency must name an earlier problem");
    // raw x rows are staged in place of their image: needs K = 128 * C
    q.tma = (q.K % 128 == 0) && ((reinterpret_cast<uintptr_t>(q.x) & 15) == 0);
    // a problem shares the previous problem's x image when it reads the same x
    // after the same dependency
    q.newimg = !(i > 0 && P.p[i - 1].x == q.x && P.p[i - 1].K == q.K && P.p[i - 1].dep == q.dep);
    q.img = i == 0 ? 0 : P.p[i - 1].img + q.newimg;
    q.rboff = tot;
    tot += q.RB;
  }
  P.tot = tot;
  // x images alternate between two banks: image i+2 is staged only after this
  // CTA's items on image i are done, so nobody still reads it
  auto img_bytes = [&](const GvProb& q) {
    // K1t: the image covers whole chunk groups (4 chunks)
    const uint32_t cimg = TC ? (uint32_t)((q.C + 3) & ~3) : (uint32_t)q.C;
    return (((uint32_t)MP * q.C * 8 + 255u) & ~255u) + (((uint32_t)MP * cimg * 256 + 255u) & ~255u);
  };
  uint32_t bank_need[2] = {0, 0};
  for (int i = 0; i < n; ++i)
    if (P.p[i].newimg) bank_need[P.p[i].img & 1] = std::max(bank_need[P.p[i].img & 1], img_bytes(P.p[i]));
  // placement: pieces go in front of the 64-KB table while they fit, else behind it
  uint32_t front = kParamOff + (((uint32_t)sizeof(GvParams) + 255u) & ~255u);
  uint32_t back = kPre + kTblBytes;
  auto place = [&](uint32_t bytes) {
    bytes = (bytes + 255u) & ~255u;
    if (front + bytes <= kPre) {
      const uint32_t o = front;
      front += bytes;
      return o;
    }
    const uint32_t o = back;
    back += bytes;
    return o;
  };
  P.bars = place(TC ? kTbBytes : kBarBytes);
  P.lutbuf = place(2048);
  P.red = place(2u * (TC ? 4 : kW) * MP * 32 * 4);
  uint32_t bank_off[2];
  for (int k = 0; k < 2; ++k) bank_off[k] = bank_need[k] ? place(bank_need[k]) : 0;
  for (int i = 0; i < n; ++i) {
    GvProb& q = P.p[i];
    if (q.newimg) {
      q.xs = bank_off[q.img & 1];
      q.xh = q.xs + (((uint32_t)MP * q.C * 8 + 255u) & ~255u);
    } else {
      q.xs = P.p[i - 1].xs;
      q.xh = P.p[i - 1].xh;
    }
  }
  // the code ring takes what is left: as many 32-KB stages as fit (2..4),
  // each stage in front of the table if it still fits there
  P.nring = 0;
  const int rmax = TC ? kTcMaxRing : kMaxRing;
  const uint32_t sbytes = TC ? kTcStageBytes : kStageBytes;
  for (int r = rmax; r >= 2 && !P.nring; --r) {
    const uint32_t f0 = front, b0 = back;
    uint32_t ro[kTcMaxRing] = {};
    for (int j = 0; j < r; ++j) ro[j] = place(sbytes);
    const uint32_t ao = place(TC ? (uint32_t)kTcAbRing * kTcStageAb : (uint32_t)r * kStageAb);
    if (back <= kSmemMax) {
      P.nring = r;
      for (int j = 0; j < kTcMaxRing; ++j) P.ring[j] = ro[j];
      P.abring = ao;
    } else {
      front = f0;
      back = b0;
    }
  }
  if (!P.nring)
    fail(ANYQ_ERR_SHAPE, "LUT GEMV chain: x images leave no room for the weight ring (" +
                             std::to_string(back + 2 * (kStageBytes + kStageAb)) + " > " +
                             std::to_string(kSmemMax) + " B)");
  return back;
}

template <int MP, bool TC = false>
void launch_gv(int n, const LutTensor* const* ts, const void* const* xs, void* const* ys,
               float* const* y32s, const int32_t* deps, int64_t m, cudaStream_t s,
               const KSlice* slices = nullptr) {
  GvParams P;
  const uint32_t smem_bytes = plan_chain<MP, TC>(n, ts, xs, ys, y32s, deps, m, P, slices);
  // release counters of this stream: launches on one stream are ordered and
  // leave them at zero; launches on other streams use their own
  const StreamWs ws = stream_ws(s);
  P.done = ws.done;
  P.err = ws.err + kErrGemv;
  const void* kfn;
  if constexpr (TC) kfn = (const void*)k_lutgemv_tc<MP>;
  else kfn = (const void*)k_lutgemv<MP>;
  ensure_dyn_smem(kfn, (int)smem_bytes);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // co-residency for the chain waits
  attr[1].val.cooperative = 1;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)P.ncta);
  lc.blockDim = dim3(TC ? kTcT : kT);
  lc.dynamicSmemBytes = smem_bytes;
  lc.stream = s;
  lc.attrs = attr;
  lc.numAttrs = 2;
  // Co-residency is only needed when a problem waits for another grid-wide;
  // an independent launch skips the cooperative attribute (measured 1-2 us
  // less launch latency). 1 CTA per SM and grid = SM count either way.
  bool waits = false;
  for (int i = 0; i < n; ++i) waits |= P.p[i].dep >= 0;
  if (!waits) lc.numAttrs = 1;
  if constexpr (TC) {
    ANYQ_CUDA(cudaLaunchKernelEx(&lc, k_lutgemv_tc<MP>, P));
  } else {
    ANYQ_CUDA(cudaLaunchKernelEx(&lc, k_lutgemv<MP>, P));
  }
  ANYQ_LAUNCHED();
}

// K1t instance for m x rows: MP = 2, 4, 8 or 16 (MMA N = 4 MP).
template <typename F>
auto tc_dispatch(int64_t m, F&& f) {
  if (m <= 2) return f(std::integral_constant<int, 2>{});
  if (m <= 4) return f(std::integral_constant<int, 4>{});
  if (m <= 8) return f(std::integral_constant<int, 8>{});
  return f(std::integral_constant<int, 16>{});
}

// The pair table's address trick needs the dynamic shared-memory window to
// start at kDynBase; probed once per device with a kernel of the same shape
// (no static shared memory), so a toolchain or driver that moves it turns the
// GEMV off (AUTO picks another path) instead of failing inside the kernel.
__global__ void k_sbase_probe(uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0) *out = (uint32_t)__cvta_generic_to_shared(smem);
}

bool gv_sbase_ok() {
  static std::mutex mu;
  static std::map<int, bool> ok;
  int dev = 0;
  ANYQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = ok.find(dev);
  if (it != ok.end()) return it->second;
  uint32_t* d = nullptr;
  uint32_t h = 0;
  // the first GEMV may be issued while another stream is being captured:
  // probe on a private stream in relaxed capture mode
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  ANYQ_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
  cudaStream_t z = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&z, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&d, sizeof(uint32_t));
  if (e == cudaSuccess) {
    k_sbase_probe<<<1, 32, 4096, z>>>(d);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, z);
  if (e == cudaSuccess) e = cudaStreamSynchronize(z);
  if (d) cudaFree(d);
  if (z) cudaStreamDestroy(z);
  cudaThreadExchangeStreamCaptureMode(&mode);
  ANYQ_CUDA(e);
  return ok[dev] = (h == kDynBase);
}

}  // namespace

void lutgemv_set_trace(long long* dev) { g_gv_trace = dev; }

// GEMV settings of a tensor (called once from lutgemm_create).
void lutgemv_setup(LutTensor* t) {
  t->gv_ncta = t->sms;
  // chunk -> scale-group index as a shift (rowwise: always group 0)
  t->gv_gshift = -1;
  if (t->GR == 1) t->gv_gshift = 30;
  else if ((t->GC & (t->GC - 1)) == 0) t->gv_gshift = __builtin_ctz((unsigned)t->GC);
}

void lutgemv_chain_run(int n, const LutTensor* const* ts, const void* const* xs, void* const* ys,
                       float* const* y32s, const int32_t* deps, int64_t m, cudaStream_t s) {
  if (m < 1 || m > kMaxMP) fail(ANYQ_ERR_SHAPE, "LUT GEMV supports 1 <= m <= 4");
  if (n < 1 || !ts) fail(ANYQ_ERR_SHAPE, "empty GEMM chain");
  if (!gv_sbase_ok())
    fail(ANYQ_ERR_CONFIG, "LUT GEMV: dynamic shared memory does not start at 0x400 on this device");
  if (m == 1) launch_gv<1>(n, ts, xs, ys, y32s, deps, m, s);
  else if (m == 2) launch_gv<2>(n, ts, xs, ys, y32s, deps, m, s);
  else if (m == 3) launch_gv<3>(n, ts, xs, ys, y32s, deps, m, s);
  else launch_gv<4>(n, ts, xs, ys, y32s, deps, m, s);
}

bool lutgemv_fits(const LutTensor* t, int64_t m) {
  if (!t || m < 1 || m > kMaxMP || t->gv_gshift < 0 || !gv_sbase_ok()) return false;
  const LutTensor* ts[1] = {t};
  const void* xs[1] = {nullptr};
  void* ys[1] = {nullptr};
  GvParams P;
  try {
    if (m == 1) plan_chain<1>(1, ts, xs, ys, nullptr, nullptr, m, P);
    else if (m == 2) plan_chain<2>(1, ts, xs, ys, nullptr, nullptr, m, P);
    else if (m == 3) plan_chain<3>(1, ts, xs, ys, nullptr, nullptr, m, P);
    else plan_chain<4>(1, ts, xs, ys, nullptr, nullptr, m, P);
  } catch (const Failure&) {
    return false;
  }
  return true;
}

void lutgemv_tc_chain_run(int n, const LutTensor* const* ts, const void* const* xs, void* const* ys,
                          float* const* y32s, const int32_t* deps, int64_t m, cudaStream_t s) {
  if (m < 1 || m > kTcMaxMP) fail(ANYQ_ERR_SHAPE, "tcgen05 LUT GEMV supports 1 <= m <= 16");
  if (n < 1 || !ts) fail(ANYQ_ERR_SHAPE, "empty GEMM chain");
  if (!gv_sbase_ok())
    fail(ANYQ_ERR_CONFIG, "LUT GEMV: dynamic shared memory does not start at 0x400 on this device");
  tc_dispatch(m, [&](auto mp) {
    launch_gv<decltype(mp)::value, true>(n, ts, xs, ys, y32s, deps, m, s);
    return 0;
  });
}

// AUTO engine of a chain (measured, profiles/round2_k1t.md): the CUDA-core
// GEMV at m <= 2, K1t from m = 3 while its shared-memory plan fits.
void lutgemv_chain_run_auto(int n, const LutTensor* const* ts, const void* const* xs, void* const* ys,
                            float* const* y32s, const int32_t* deps, int64_t m, cudaStream_t s) {
  if (m >= 3 && m <= kTcMaxMP && gv_sbase_ok()) {
    bool fits = true;
    try {
      GvParams P;
      tc_dispatch(m, [&](auto mp) { return plan_chain<decltype(mp)::value, true>(n, ts, xs, ys, y32s, deps, m, P); });
    } catch (const Failure&) {
      fits = false;
    }
    if (fits || m > kMaxMP) {
      lutgemv_tc_chain_run(n, ts, xs, ys, y32s, deps, m, s);
      return;
    }
  }
  lutgemv_chain_run(n, ts, xs, ys, y32s, deps, m, s);
}

// K-slices of one K1t GEMM whose x image does not fit: the fewest slices (of
// whole chunk groups and whole scale groups, at most kMaxProb) whose plan
// fits, run as a chain in which slice s waits for slice s - 1 and adds its
// fp32 partial to the running sum (fixed order: deterministic). Returns the
// slice count (0: none fits); sl[] gets the chunk ranges.
int tc_slices(const LutTensor* t, int64_t m, KSlice* sl) {
  const int unit = t->GR > 1 ? std::max(4, 1 << std::min(t->gv_gshift, 20)) : 4;
  const LutTensor* ts[kMaxProb];
  const void* xs[kMaxProb];
  void* ys[kMaxProb];
  int32_t deps[kMaxProb];
  for (int S = 1; S <= kMaxProb; ++S) {
    const int nc = (((t->C + S - 1) / S) + unit - 1) / unit * unit;
    const int ns = (t->C + nc - 1) / nc;
    if (ns != S && S > 1) continue;  // rounding to whole groups made it another count
    for (int i = 0; i < ns; ++i) {
      sl[i] = KSlice{i * nc, std::min(nc, t->C - i * nc), nullptr, nullptr};
      ts[i] = t;
      xs[i] = nullptr;
      ys[i] = nullptr;
      deps[i] = i - 1;
    }
    GvParams P;
    try {
      tc_dispatch(m, [&](auto mp) {
        return plan_chain<decltype(mp)::value, true>(ns, ts, xs, ys, nullptr, deps, m, P, sl);
      });
      return ns;
    } catch (const Failure&) {
    }
  }
  return 0;
}

bool lutgemv_tc_fits(const LutTensor* t, int64_t m) {
  if (!t || m < 1 || m > kTcMaxMP || t->gv_gshift < 0 || !gv_sbase_ok()) return false;
  KSlice sl[kMaxProb];
  return tc_slices(t, m, sl) > 0;
}

int lutgemv_tc_slices(const LutTensor* t, int64_t m) {
  if (!t || m < 1 || m > kTcMaxMP || t->gv_gshift < 0 || !gv_sbase_ok()) return 0;
  KSlice sl[kMaxProb];
  return tc_slices(t, m, sl);
}

void lutgemv_tc_run(const LutTensor* t, const void* x, int64_t m, void* y, float* y32,
                    cudaStream_t s) {
  if (!t) fail(ANYQ_ERR_SHAPE, "null device tensor");
  if (m < 1 || m > kTcMaxMP) fail(ANYQ_ERR_SHAPE, "tcgen05 LUT GEMV supports 1 <= m <= 16");
  if (t->gv_gshift < 0) fail(ANYQ_ERR_CONFIG, "LUT GEMV needs rowwise scales or group_size = 128 * 2^j");
  if (!gv_sbase_ok())
    fail(ANYQ_ERR_CONFIG, "LUT GEMV: dynamic shared memory does not start at 0x400 on this device");
  KSlice sl[kMaxProb];
  const int ns = tc_slices(t, m, sl);
  if (ns == 0) fail(ANYQ_ERR_SHAPE, "tcgen05 LUT GEMV: the x image does not fit in 8 K-slices");
  const LutTensor* ts[kMaxProb];
  const void* xs[kMaxProb];
  void* ys[kMaxProb];
  float* y32s[kMaxProb];
  int32_t deps[kMaxProb];
  // the running sum lives in y32 when the caller wants it, else in stream scratch
  float* acc = ns > 1 ? (y32 ? y32 : stream_scratch_f32(s, (size_t)m * t->rows)) : nullptr;
  for (int i = 0; i < ns; ++i) {
    ts[i] = t;
    xs[i] = x;
    ys[i] = y;
    y32s[i] = y32;
    deps[i] = i - 1;
    sl[i].acc_in = i > 0 ? acc : nullptr;
    sl[i].acc_out = i + 1 < ns ? acc : nullptr;
  }
  tc_dispatch(m, [&](auto mp) {
    constexpr int MP = decltype(mp)::value;
    launch_gv<MP, true>(ns, ts, xs, ys, y32s, ns > 1 ? deps : nullptr, m, s, sl);
    return 0;
  });
}

// ---------------------------------------------------------------------------
// Tensor-parallel GEMM with the all-gather fused into the writer
// ---------------------------------------------------------------------------
namespace {
__global__ void k_tp_wait(int* const* flags, int rank, int world, int expect) {
  const int r = threadIdx.x;
  if (r < world) {
    const int* f = flags[rank] + r;
    int v;
    do {
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (v < expect) __nanosleep(64);
    } while (v < expect);
  }
  __syncwarp();
}
}  // namespace

void lutgemv_tp_run(const LutTensor* t, const void* x, int64_t m, const anyq_tp_peers* tp, cudaStream_t s) {
  if (!t || !tp) fail(ANYQ_ERR_SHAPE, "tp gemm: null argument");
  if (tp->world < 1 || tp->world > kMaxTp || tp->rank < 0 || tp->rank >= tp->world)
    fail(ANYQ_ERR_SHAPE, "tp gemm: 1 <= world <= 8 and 0 <= rank < world");
  if (m < 1 || m > kMaxMP) fail(ANYQ_ERR_SHAPE, "tp gemm: the fused gather runs on the GEMV (1 <= m <= 4)");
  if (tp->row0 < 0 || tp->row0 + t->rows > tp->rows_total) fail(ANYQ_ERR_SHAPE, "tp gemm: shard outside y");
  if (!gv_sbase_ok())
    fail(ANYQ_ERR_CONFIG, "LUT GEMV: dynamic shared memory does not start at 0x400 on this device");
  for (int r = 0; r < tp->world; ++r)
    if (!tp->y[r] || !tp->flags[r]) fail(ANYQ_ERR_SHAPE, "tp gemm: every rank's y and flags must be mapped");
  const LutTensor* ts[1] = {t};
  const void* xs[1] = {x};
  void* ys[1] = {tp->y[tp->rank]};  // unused: the writer stores through tp_y
  GvParams P;
  auto go = [&](auto mp) {
    constexpr int MP = decltype(mp)::value;
    const uint32_t smem_bytes = plan_chain<MP>(1, ts, xs, ys, nullptr, nullptr, m, P);
    P.tp_world = tp->world;
    P.tp_rank = tp->rank;
    P.tp_row0 = tp->row0;
    P.tp_N = tp->rows_total;
    for (int r = 0; r < tp->world; ++r) {
      P.tp_y[r] = static_cast<__nv_bfloat16*>(tp->y[r]);
      P.tp_flags[r] = tp->flags[r];
    }
    const StreamWs ws = stream_ws(s);
    P.done = ws.done;
    P.err = ws.err + kErrGemv;
    ensure_dyn_smem((const void*)k_lutgemv<MP>, (int)smem_bytes);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)P.ncta);
    lc.blockDim = dim3(kT);
    lc.dynamicSmemBytes = smem_bytes;
    lc.stream = s;
    lc.attrs = attr;
    lc.numAttrs = 1;
    ANYQ_CUDA(cudaLaunchKernelEx(&lc, k_lutgemv<MP>, P));
    ANYQ_LAUNCHED();
    return 0;
  };
  if (m == 1) go(std::integral_constant<int, 1>{});
  else if (m == 2) go(std::integral_constant<int, 2>{});
  else if (m == 3) go(std::integral_constant<int, 3>{});
  else go(std::integral_constant<int, 4>{});
}

int lutgemv_tp_ctas(const LutTensor* t) { return t ? t->gv_ncta : 0; }

void lutgemv_tp_wait(const anyq_tp_peers* tp, int expect, cudaStream_t s) {
  if (!tp || tp->world < 1 || tp->world > kMaxTp) fail(ANYQ_ERR_SHAPE, "tp wait: bad peers");
  DevBuf<int*> f(tp->world, s);
  ANYQ_CUDA(cudaMemcpyAsync(f.p, tp->flags, sizeof(int*) * tp->world, cudaMemcpyHostToDevice, s));
  k_tp_wait<<<1, 32, 0, s>>>(f.p, tp->rank, tp->world, expect);
  ANYQ_LAUNCHED();
}

void lutgemv_run(const LutTensor* t, const void* x, int64_t m, void* y, float* y32,
                 cudaStream_t s) {
  if (!t) fail(ANYQ_ERR_SHAPE, "null device tensor");
  const LutTensor* ts[1] = {t};
  const void* xs[1] = {x};
  void* ys[1] = {y};
  float* y32s[1] = {y32};
  lutgemv_chain_run(1, ts, xs, ys, y32s, nullptr, m, s);
}

}  // namespace anyq_b200
