// K1a — CUDA-core any4 LUT GEMV for M <= 4 (the memory-bound decode path), sm_100a.
//
//   y[m][n] = sum_k x[m][k] * (alpha[n][g(k)] * T_n[c[n][k]] + beta[n][g(k)])
//
// is the reference's gemm_fused (qgemm.cpp:71-128) with the per-group scale
// factored out of the k loop. Per 128-k chunk c:
//   y[m][n] += alpha_g * 2^-e * sum_{k in c} xh[m][k] * T_n[c[n][k]] + beta_g * sum_{k in c} x[m][k]
// where xh = fp16(x * 2^e) is EXACT (bf16 has 8 significant bits, fp16 11;
// e puts max|x| of the chunk in [2^14, 2^15)). Every product xh * T
// (fp16 x fp16) is formed exactly by FHFMA (fma.rn.f32.f16) and accumulated in
// fp32, so the result differs from the fp32 reference only by summation order
// (tolerance 1e-5 * sum|x*w|, tests/test_gpu_gemm.py).
//
// Data path (one persistent CTA of 16 warps per SM):
//  * lane L of every warp owns row L of a 32-row block. The unit of work is a
//    chunk = 32 rows x 128 k = 2 KB contiguous in the prepacked code tensor
//    (layout of lutgemm.cu: [RB][C][4 slabs][32 rows][16 B]); a warp reads it
//    with 4 coalesced LDG.128 (512 B each) and keeps two chunks in flight in
//    registers (no shared-memory staging: the smem crossbar is the second
//    tightest resource after HBM).
//  * LUT lookup: the row's 16 fp16 values are expanded once per row block into
//    a 256-entry pair table T2[byte] = (T[lo], T[hi]); entry e of lane L lives
//    at shared address 0x10000 + e*256 + buf*128 + L*4. Every lookup of a warp
//    hits bank L (conflict free), the address is ONE prmt of the code byte into
//    the lane word (no add: the table is 64 KB aligned in the shared window),
//    and ONE LDS dequantises two weights. buf 0/1 double-buffer consecutive
//    row blocks.
//  * x enters once per CTA as the permuted fp16 image the code bytes index,
//    plus per-chunk (2^-e, sum x), in shared memory.
//  * Work split: whole row blocks round-robin over CTAs ("phase A"); the
//    remaining RB mod ncta row blocks are split by chunk over all CTAs ("phase
//    B", each CTA range spans <= 2 row blocks). Inside a CTA each row-block
//    segment is divided evenly over the 16 warps; warp partials are reduced in
//    shared memory in a fixed order and row blocks split over CTAs are combined
//    in slot order by the last-arriving CTA: deterministic.
//  * Programmatic dependent launch: codes, LUT and the first table are fetched
//    before griddepcontrol.wait, overlapping the previous kernel's tail.
#include <cuda_bf16.h>

#include "kernels.cuh"
#include "lutgemm.cuh"

namespace anyq_b200 {

namespace {

constexpr int kW = 16;  // warps per CTA (piece split uses >> 4)
constexpr int kT = kW * 32;
constexpr int kMaxMP = 4;
constexpr uint32_t kTblAddr = 0x10000;  // shared-window address of the pair table
constexpr uint32_t kDynBase = 0x400;    // shared-window address of dynamic smem (sm_100)
constexpr uint32_t kPre = kTblAddr - kDynBase;  // bytes of dynamic smem before the table
constexpr uint32_t kTblBytes = 0x10000;

// Shared-memory layout (offsets into dynamic smem). The small arrays live in
// the 63 KB in front of the table when they fit, else behind it.
template <int MP>
struct GvLayout {
  uint32_t red, xs, xh, total;
  __host__ __device__ GvLayout(int C) {
    const uint32_t nred = 2u * kW * MP * 32 * 4;
    const uint32_t nxs = (uint32_t)MP * C * 8;
    const uint32_t nxh = (uint32_t)MP * C * 256;
    red = 0;
    xs = nred;
    if (nred + nxs + nxh <= kPre) {
      xh = nred + nxs;
      total = kPre + kTblBytes;
    } else {
      xh = kPre + kTblBytes;
      total = xh + nxh;
    }
  }
};

struct GvParams {
  const uint4* codes;    // [RB][C][4][32] uint4
  const uint4* lut;      // [RB*32][2] uint4 (16 fp16)
  const uint32_t* ab;    // [RB][GR][32] half2 (alpha, beta)
  const __nv_bfloat16* x;
  __nv_bfloat16* y;
  float* y32;
  float* part;           // [RB - rbA][cmax][MP][32]
  int* counters;         // [RB - rbA]
  int* err;              // device error word
  uint32_t UB;           // phase-B chunks
  int N, K, M, RB, C, GR;
  int gshift;            // chunk -> scale group: g = c >> gshift
  int fullA, rbA, ncta, cmax;
  long long* trace;      // debug: [ncta][16] globaltimer stamps, or null
};

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
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GV_TRACE(slot)                                                             \
  do {                                                                             \
    if (P.trace && threadIdx.x == 0) P.trace[blockIdx.x * 16 + (slot)] = gtimer(); \
  } while (0)

// CTA whose phase-B range holds chunk u (all products fit 32 bits: the host
// checks UB * ncta < 2^32).
__device__ __forceinline__ int cta_of(uint32_t u, uint32_t U, uint32_t ncta) {
  return (int)(((u + 1) * ncta + U - 1) / U) - 1;
}

// Segment of a CTA: row block and chunk range [c0, c1).
struct Seg {
  int rb, c0, c1;
};

// This CTA's segments: fullA whole row blocks (phase A), then at most two
// pieces of the phase-B range (its length is <= C because RB - rbA < ncta).
struct Work {
  int fullA, ncta, b, C, nseg;
  int rb0, c0a, c0b, c1b;  // phase B: rb0 [c0a, c0b), then rb0 + 1 [0, c1b)
  __device__ __forceinline__ Seg get(int i) const {
    Seg g;
    if (i < fullA) {
      g.rb = i * ncta + b;
      g.c0 = 0;
      g.c1 = C;
    } else if (i == fullA) {
      g.rb = rb0;
      g.c0 = c0a;
      g.c1 = c0b;
    } else {
      g.rb = rb0 + 1;
      g.c0 = 0;
      g.c1 = c1b;
    }
    return g;
  }
};

__device__ __forceinline__ Work make_work(uint32_t UB, int C, int ncta, int fullA, int rbA, int b) {
  Work w;
  w.fullA = fullA;
  w.ncta = ncta;
  w.b = b;
  w.C = C;
  w.nseg = fullA;
  w.rb0 = rbA;
  w.c0a = w.c0b = w.c1b = 0;
  const uint32_t lo = (uint32_t)b * UB / (uint32_t)ncta, hi = (uint32_t)(b + 1) * UB / (uint32_t)ncta;
  if (lo < hi) {
    const int len = (int)(hi - lo);
    w.rb0 = rbA + (int)(lo / (uint32_t)C);
    w.c0a = (int)(lo % (uint32_t)C);
    w.c0b = min(C, w.c0a + len);
    w.nseg += 1;
    if (w.c0a + len > C) {
      w.c1b = w.c0a + len - C;
      w.nseg += 1;
    }
  }
  return w;
}

// Load cursor of one warp: segment li, chunk lc of its piece [.., le); cp is
// this lane's first uint4 of chunk lc, abrow the lane's (alpha, beta) row.
struct Cursor {
  int li, lc, le;
  const uint4* cp;
  const uint32_t* abrow;
};

__device__ __forceinline__ void piece_of(const Seg& sg, int warp, int& a, int& e) {
  const int n = sg.c1 - sg.c0;
  a = sg.c0 + ((warp * n) >> 4);
  e = sg.c0 + (((warp + 1) * n) >> 4);
}

// Advance to the next segment whose piece for this warp is non-empty.
__device__ __forceinline__ void next_piece(const Work& W, const uint4* codes, const uint32_t* ab,
                                           int GR, int warp, int lane, Cursor& c) {
  while (true) {
    ++c.li;
    if (c.li >= W.nseg) return;
    const Seg sg = W.get(c.li);
    piece_of(sg, warp, c.lc, c.le);
    c.cp = codes + ((size_t)sg.rb * W.C + c.lc) * 128 + lane;
    c.abrow = ab + (size_t)sg.rb * GR * 32 + lane;
    if (c.lc < c.le) return;
  }
}

struct Chunk {
  uint4 w[4];
  uint32_t ab;
};

// Pair table for row `lane` into buffer buf; warp w writes the 16 entries
// whose high nibble is w.
__device__ __forceinline__ void build_table(const uint4 l0, const uint4 l1, int warp, int buf,
                                            uint32_t laneoff) {
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
      t[b] = lds32(__byte_perm(wd[b >> 2], tb, 0x7604u | ((uint32_t)(b & 3) << 4)));
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

template <int MP>
__global__ void __launch_bounds__(kT, 1) k_lutgemv(GvParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  asm volatile("griddepcontrol.launch_dependents;");
  GV_TRACE(0);
  if (P.trace && threadIdx.x == 0) P.trace[blockIdx.x * 16 + 12] = clock64();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x;
  const uint32_t laneoff = (uint32_t)lane << 2;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  if (sbase != kDynBase) {  // the table must sit at shared address 0x10000
    if (threadIdx.x == 0) atomicMax(P.err, (int)ANYQ_ERR_INTERNAL);
    return;
  }
  const GvLayout<MP> lay(P.C);
  float* red = reinterpret_cast<float*>(smem + lay.red);
  const uint32_t xbase = sbase + lay.xh, xstride = (uint32_t)P.C * 256;
  const uint32_t xsbase = sbase + lay.xs, xsstride = (uint32_t)P.C * 8;
  const Work W = make_work(P.UB, P.C, P.ncta, P.fullA, P.rbA, b);
  const int nseg = W.nseg;
  const uint4* const codes = P.codes;
  const uint32_t* const abp = P.ab;
  const int GR = P.GR, gshift = P.gshift;

  // ---- load cursor over this warp's pieces of all segments; 2-chunk ring
  Cursor cur;
  cur.li = -1;
  cur.lc = cur.le = 0;
  cur.cp = P.codes;
  cur.abrow = P.ab;
  if (nseg > 0) next_piece(W, codes, abp, GR, warp, lane, cur);
  auto load = [&](Chunk& ch) {
    if (cur.li < nseg) {
#pragma unroll
      for (int q = 0; q < 4; ++q) ch.w[q] = __ldcs(cur.cp + q * 32);
      ch.ab = __ldg(cur.abrow + ((cur.lc >> gshift) << 5));
      cur.cp += 128;
      if (++cur.lc >= cur.le) next_piece(W, codes, abp, GR, warp, lane, cur);
    }
  };
  Chunk r0, r1;
  load(r0);
  load(r1);
  GV_TRACE(1);

  // ---- LUT of segment 0 -> table 0; LUT of segment 1 prefetched
  uint4 nl0 = make_uint4(0, 0, 0, 0), nl1 = nl0;
  if (nseg > 0) {
    const uint4* lp = P.lut + ((size_t)W.get(0).rb * 32 + lane) * 2;
    build_table(__ldg(lp), __ldg(lp + 1), warp, 0, laneoff);
  }
  if (nseg > 1) {
    const uint4* lp = P.lut + ((size_t)W.get(1).rb * 32 + lane) * 2;
    nl0 = __ldg(lp);
    nl1 = __ldg(lp + 1);
  }
  GV_TRACE(2);

  // ---- x: permuted fp16 image + per-chunk (2^-e, sum x); depends on the
  // previous kernel in the stream
  asm volatile("griddepcontrol.wait;" ::: "memory");
  GV_TRACE(3);
  for (int task = warp; task < MP * P.C; task += kW) {
    const int m = task / P.C, c = task % P.C;
    const int k0 = c * 128 + lane * 4;
    float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (m < P.M) {
      const __nv_bfloat16* xr = P.x + (size_t)m * P.K;
      if ((P.K & 3) == 0 && k0 + 3 < P.K) {
        const uint2 raw = *reinterpret_cast<const uint2*>(xr + k0);
        const __nv_bfloat162 p0 = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
        const __nv_bfloat162 p1 = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
        v[0] = __low2float(p0);
        v[1] = __high2float(p0);
        v[2] = __low2float(p1);
        v[3] = __high2float(p1);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (k0 + j < P.K) v[j] = __bfloat162float(xr[k0 + j]);
      }
    }
    float amax = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
    float sum = (v[0] + v[1]) + (v[2] + v[3]);
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
      sum += __shfl_xor_sync(0xffffffffu, sum, off);
    }
    const int e = (amax > 0.0f && isfinite(amax)) ? 14 - ilogbf(amax) : 0;
    // k = 128c + 4L + j  <->  slab q = (L%16)/4, pair b = 8(L/16) + 2(L%4) + j/2
    const int q = (lane & 15) >> 2, bp = 8 * (lane >> 4) + 2 * (lane & 3);
    const __half2 h01 = __floats2half2_rn(ldexpf(v[0], e), ldexpf(v[1], e));
    const __half2 h23 = __floats2half2_rn(ldexpf(v[2], e), ldexpf(v[3], e));
    uint2 pk;
    pk.x = *reinterpret_cast<const uint32_t*>(&h01);
    pk.y = *reinterpret_cast<const uint32_t*>(&h23);
    *reinterpret_cast<uint2*>(smem + lay.xh + (size_t)m * P.C * 256 + c * 256 + (q * 16 + bp) * 4) = pk;
    if (lane == 0)
      *reinterpret_cast<float2*>(smem + lay.xs + ((size_t)m * P.C + c) * 8) =
          make_float2(ldexpf(1.0f, -e), sum);
  }
  GV_TRACE(4);
  __syncthreads();
  GV_TRACE(5);

  // ---- main loop over segments
  for (int i = 0; i < nseg; ++i) {
    const Seg sg = W.get(i);
    int a, e;
    piece_of(sg, warp, a, e);
    const uint32_t tb = kTblAddr | ((uint32_t)(i & 1) << 7) | laneoff;
    float y[MP];
#pragma unroll
    for (int m = 0; m < MP; ++m) y[m] = 0.0f;
    uint32_t xa = xbase + (uint32_t)a * 256, xsa = xsbase + (uint32_t)a * 8;
    int c = a;
    for (; c + 2 <= e; c += 2) {
      consume<MP>(r0, tb, xa, xsa, xstride, xsstride, y);
      load(r0);
      consume<MP>(r1, tb, xa + 256, xsa + 8, xstride, xsstride, y);
      load(r1);
      xa += 512;
      xsa += 16;
    }
    if (c < e) {
      consume<MP>(r0, tb, xa, xsa, xstride, xsstride, y);
      load(r0);
      const Chunk t = r0;  // rotate: r1 is the next chunk to consume
      r0 = r1;
      r1 = t;
    }
    // next row block's table (its buffer was last read in segment i-1)
    if (i + 1 < nseg) {
      build_table(nl0, nl1, warp, (i + 1) & 1, laneoff);
      if (i + 2 < nseg) {
        const uint4* lp = P.lut + ((size_t)W.get(i + 2).rb * 32 + lane) * 2;
        nl0 = __ldg(lp);
        nl1 = __ldg(lp + 1);
      }
    }
    float* rp = red + (size_t)(i & 1) * kW * MP * 32;
#pragma unroll
    for (int m = 0; m < MP; ++m) rp[(warp * MP + m) * 32 + lane] = y[m];
    if (i < 3) GV_TRACE(6 + 2 * i);
    __syncthreads();
    if (i < 3) GV_TRACE(7 + 2 * i);
    if (warp == 0) {
      const int rb = sg.rb;
      float acc[MP];
#pragma unroll
      for (int m = 0; m < MP; ++m) {
        float t = 0.0f;
#pragma unroll
        for (int w = 0; w < kW; ++w) t += rp[(w * MP + m) * 32 + lane];
        acc[m] = t;
      }
      bool write = true;
      if (rb >= P.rbA) {
        const uint32_t ub0 = (uint32_t)(rb - P.rbA) * P.C;
        const int first = cta_of(ub0, P.UB, P.ncta);
        const int last = cta_of(ub0 + P.C - 1, P.UB, P.ncta);
        if (last > first) {
          // CTAs first..last share this row block. When UB < ncta some CTAs
          // have empty ranges; the others hold exactly one chunk each, so the
          // contributors are the C chunks of the row block (slot = chunk).
          const bool sparse = P.UB < P.ncta;
          const int ncontrib = sparse ? P.C : last - first + 1;
          const int slot = sparse ? (int)((uint32_t)b * P.UB / (uint32_t)P.ncta - ub0) : b - first;
          float* pp = P.part + ((size_t)(rb - P.rbA) * P.cmax + slot) * MP * 32;
#pragma unroll
          for (int m = 0; m < MP; ++m) pp[m * 32 + lane] = acc[m];
          __threadfence();
          __syncwarp();
          int old = 0;
          if (lane == 0) old = atomicAdd(&P.counters[rb - P.rbA], 1);
          old = __shfl_sync(0xffffffffu, old, 0);
          write = old == ncontrib - 1;
          if (write) {
            __threadfence();
#pragma unroll
            for (int m = 0; m < MP; ++m) {
              float t = 0.0f;
              for (int sl = 0; sl < ncontrib; ++sl)
                t += __ldcg(P.part + ((size_t)(rb - P.rbA) * P.cmax + sl) * MP * 32 + m * 32 + lane);
              acc[m] = t;
            }
            if (lane == 0) P.counters[rb - P.rbA] = 0;
          }
        }
      }
      const int row = rb * 32 + lane;
      if (write && row < P.N) {
#pragma unroll
        for (int m = 0; m < MP; ++m) {
          if (m < P.M) {
            P.y[(size_t)m * P.N + row] = __float2bfloat16_rn(acc[m]);
            if (P.y32) P.y32[(size_t)m * P.N + row] = acc[m];
          }
        }
      }
    }
  }
  GV_TRACE(15);
  if (P.trace && threadIdx.x == 0) P.trace[blockIdx.x * 16 + 13] = clock64();
}

long long* g_gv_trace = nullptr;

template <int MP>
void launch_gv(const LutTensor* t, const void* x, int64_t m, void* y, float* y32, cudaStream_t s) {
  GvParams P;
  P.codes = reinterpret_cast<const uint4*>(t->codes);
  P.lut = reinterpret_cast<const uint4*>(t->lut);
  P.ab = reinterpret_cast<const uint32_t*>(t->ab);
  P.x = reinterpret_cast<const __nv_bfloat16*>(x);
  P.y = reinterpret_cast<__nv_bfloat16*>(y);
  P.y32 = y32;
  P.part = t->gv_part;
  P.counters = t->gv_counters;
  P.err = t->gv_err;
  P.N = (int)t->rows;
  P.K = (int)t->cols;
  P.M = (int)m;
  P.RB = t->RB;
  P.C = t->C;
  P.GR = t->GR;
  P.gshift = t->gv_gshift;
  P.ncta = t->gv_ncta;
  P.fullA = t->gv_fullA;
  P.rbA = t->gv_rbA;
  P.UB = (uint32_t)((t->RB - t->gv_rbA) * P.C);
  P.cmax = t->gv_cmax;
  P.trace = g_gv_trace;
  const GvLayout<MP> lay(P.C);
  if (lay.total > 227u * 1024u) fail(ANYQ_ERR_SHAPE, "LUT GEMV: x image too large for shared memory");
  static uint32_t configured = 0;
  if (lay.total > configured) {
    ANYQ_CUDA(cudaFuncSetAttribute(k_lutgemv<MP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)lay.total));
    configured = lay.total;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)P.ncta);
  lc.blockDim = dim3(kT);
  lc.dynamicSmemBytes = lay.total;
  lc.stream = s;
  lc.attrs = attr;
  lc.numAttrs = 1;
  ANYQ_CUDA(cudaLaunchKernelEx(&lc, k_lutgemv<MP>, P));
  ANYQ_LAUNCHED();
}

}  // namespace

void lutgemv_set_trace(long long* dev) { g_gv_trace = dev; }

// Work split + workspace of the GEMV (called once from lutgemm_create).
void lutgemv_setup(LutTensor* t) {
  const int ncta = t->sms;
  t->gv_ncta = ncta;
  t->gv_fullA = t->RB / ncta;
  t->gv_rbA = t->gv_fullA * ncta;
  const int rbB = t->RB - t->gv_rbA;
  const int C = t->C;
  int cmax = 1;
  if (rbB > 0) {
    const long long UB = (long long)rbB * C;
    auto cta = [&](long long u) { return ((u + 1) * ncta + UB - 1) / UB - 1; };
    for (int r = 0; r < rbB; ++r)
      cmax = std::max<int>(cmax, (int)(cta((long long)(r + 1) * C - 1) - cta((long long)r * C) + 1));
  }
  t->gv_cmax = cmax;
  if ((unsigned long long)rbB * C * (ncta + 1) >= (1ull << 32))
    fail(ANYQ_ERR_SHAPE, "LUT GEMV: tensor too large for the 32-bit work split");
  // chunk -> scale-group index as a shift (rowwise: always group 0)
  t->gv_gshift = -1;
  if (t->GR == 1) t->gv_gshift = 30;
  else if ((t->GC & (t->GC - 1)) == 0) t->gv_gshift = __builtin_ctz((unsigned)t->GC);
  const int nb = std::max(rbB, 1);
  ANYQ_CUDA(cudaMalloc(&t->gv_part, sizeof(float) * (size_t)nb * cmax * kMaxMP * 32));
  ANYQ_CUDA(cudaMalloc(&t->gv_counters, sizeof(int) * nb));
  ANYQ_CUDA(cudaMemset(t->gv_counters, 0, sizeof(int) * nb));
  ANYQ_CUDA(cudaMalloc(&t->gv_err, sizeof(int)));
  ANYQ_CUDA(cudaMemset(t->gv_err, 0, sizeof(int)));
}

void lutgemv_run(const LutTensor* t, const void* x, int64_t m, void* y, float* y32,
                 cudaStream_t s) {
  if (!t) fail(ANYQ_ERR_SHAPE, "null device tensor");
  if (m < 1 || m > kMaxMP) fail(ANYQ_ERR_SHAPE, "LUT GEMV supports 1 <= m <= 4");
  if (t->gv_gshift < 0)
    fail(ANYQ_ERR_CONFIG, "LUT GEMV needs rowwise scales or group_size = 128 * 2^j");
  if (m == 1) launch_gv<1>(t, x, m, y, y32, s);
  else if (m == 2) launch_gv<2>(t, x, m, y, y32, s);
  else launch_gv<4>(t, x, m, y, y32, s);
}

}  // namespace anyq_b200
