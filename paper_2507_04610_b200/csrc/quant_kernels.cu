// Element-wise / per-group kernels of the quantize and layout path:
//   scales (scaling.cpp:29-70), scaled weights (scaling.cpp:72-83), sample
//   weights (learner.cpp:25-51, 379-380), RTN onto fixed tables
//   (codebooks.cpp:75-97), bit packing (pack.cpp:15-55), k-tiling
//   (pack.cpp:175-199), 16-bit narrowing (pack.cpp:159-169), dequantisation
//   (pack.cpp:205-238) and the bit-exact fp32 LUT GEMM (qgemm.cpp:71-128).
//
// Every arithmetic step that the reference performs in fp32 is written with
// explicit round-to-nearest intrinsics (__fadd_rn/__fmul_rn/__fdiv_rn) so the
// compiler cannot contract or reassociate it: these kernels are bit-identical
// to the reference by construction.
#include "kernels.cuh"

namespace anyq_b200 {

// ---------------------------------------------------------------------------
// finite check (core.hpp:145-147)
// ---------------------------------------------------------------------------
__global__ void k_check_finite(const float* __restrict__ p, int64_t n, int* err, int status) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int bad = 0;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) bad |= !isfinite(p[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) dev_fail(err, status);
}

// stats entries must be >= 0 and finite (learner.cpp:33-35)
__global__ void k_check_stats(const float* __restrict__ p, int64_t n, int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int bad = 0;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) bad |= !(p[i] >= 0.0f) || !isfinite(p[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) dev_fail(err, ANYQ_ERR_STATS);
}

// ---------------------------------------------------------------------------
// Scales. The reference scans elements in row-major order with strict < / >,
// so among equal extreme values the first encountered wins (this matters for
// -0.0 vs +0.0). Both paths reduce (value, flat index) pairs with the same
// tie rule, which reproduces that exactly.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void alpha_beta(float mn, float mx, bool symmetric, float qmin,
                                           float qmax, float* a, float* b) {
  if (symmetric) {
    float x = fabsf(mn), y = fabsf(mx);
    float absmax = (x < y) ? y : x;  // std::max(x, y)
    *a = absmax > 0.0f ? __fdiv_rn(absmax, qmax) : 1.0f;
    *b = 0.0f;
  } else {
    float range = __fsub_rn(mx, mn);
    *a = range > 0.0f ? __fdiv_rn(range, __fsub_rn(qmax, qmin)) : 1.0f;
    *b = mn;
  }
}

// One warp per (row, group) for rowwise / groupwise granularity.
__global__ void k_scales_rowgroup(const float* __restrict__ w, int64_t rows, int64_t cols,
                                  int64_t gsize, int64_t gpr, bool symmetric, float qmin,
                                  float qmax, float* __restrict__ alphas,
                                  float* __restrict__ betas) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= rows * gpr) return;
  int64_t i = warp / gpr, g = warp % gpr;
  int64_t j0 = g * gsize, j1 = min(cols, j0 + gsize);
  const float* row = w + i * cols;
  float mn = FLT_MAX, mx = -FLT_MAX;
  int64_t imn = INT64_MAX, imx = INT64_MAX;
  for (int64_t j = j0 + lane; j < j1; j += 32) {
    float v = row[j];
    if (v < mn) { mn = v; imn = j; }
    if (v > mx) { mx = v; imx = j; }
  }
  for (int off = 16; off; off >>= 1) {
    float omn = __shfl_xor_sync(0xffffffffu, mn, off);
    int64_t oimn = __shfl_xor_sync(0xffffffffu, imn, off);
    float omx = __shfl_xor_sync(0xffffffffu, mx, off);
    int64_t oimx = __shfl_xor_sync(0xffffffffu, imx, off);
    if (omn < mn || (omn == mn && oimn < imn)) { mn = omn; imn = oimn; }
    if (omx > mx || (omx == mx && oimx < imx)) { mx = omx; imx = oimx; }
  }
  if (lane == 0) {
    // The reference starts from FLT_MAX / lowest() and only replaces on
    // strict comparison, so a group whose values are all FLT_MAX keeps it.
    float a, b;
    alpha_beta(mn, mx, symmetric, qmin, qmax, &a, &b);
    alphas[warp] = a;
    betas[warp] = b;
  }
}

// Column / block / tensor granularity: atomic min/max over an order-preserving
// 32-bit key of the value (-0.0 and +0.0 share a key, as the reference's
// float comparisons treat them equal). Only the two zeros are distinct floats
// with one key, so a second pass finds the FIRST zero (64-bit flat index) of
// groups whose extreme is zero: the reference keeps the first of equal values.
__device__ __forceinline__ uint32_t ordered(float v) {
  uint32_t u = __float_as_uint(v == 0.0f ? 0.0f : v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unordered(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

__global__ void k_scales_atomic(const float* __restrict__ w, int64_t rows, int64_t cols,
                                GroupMap gm, uint32_t* __restrict__ kmin,
                                uint32_t* __restrict__ kmax) {
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    const int64_t g = gm(i, j);
    const uint32_t o = ordered(w[e]);
    atomicMin(&kmin[g], o);
    atomicMax(&kmax[g], o);
  }
}

__global__ void k_scales_first_zero(const float* __restrict__ w, int64_t rows, int64_t cols,
                                    GroupMap gm, const uint32_t* __restrict__ kmin,
                                    const uint32_t* __restrict__ kmax,
                                    unsigned long long* __restrict__ zmin,
                                    unsigned long long* __restrict__ zmax) {
  const int64_t n = rows * cols;
  const uint32_t kz = ordered(0.0f);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (w[e] != 0.0f) continue;
    const int64_t g = gm(e / cols, e % cols);
    if (kmin[g] == kz) atomicMin(&zmin[g], (unsigned long long)e);
    if (kmax[g] == kz) atomicMin(&zmax[g], (unsigned long long)e);
  }
}

__global__ void k_scales_finish(const float* __restrict__ w, int64_t ng,
                                const uint32_t* __restrict__ kmin, const uint32_t* __restrict__ kmax,
                                const unsigned long long* __restrict__ zmin,
                                const unsigned long long* __restrict__ zmax, bool symmetric,
                                float qmin, float qmax, float* alphas, float* betas) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const uint32_t kz = ordered(0.0f);
  const float mn = kmin[g] == kz ? w[zmin[g]] : unordered(kmin[g]);
  const float mx = kmax[g] == kz ? w[zmax[g]] : unordered(kmax[g]);
  float a, b;
  alpha_beta(mn, mx, symmetric, qmin, qmax, &a, &b);
  alphas[g] = a;
  betas[g] = b;
}

// ---------------------------------------------------------------------------
// Scaled weights + per-row sample weights (one block per row).
// ---------------------------------------------------------------------------
__global__ void k_scale_rows(const float* __restrict__ w, int64_t rows, int64_t cols, GroupMap gm,
                             const float* __restrict__ alphas, const float* __restrict__ betas,
                             const float* __restrict__ exj, int weighting,
                             float* __restrict__ ws, float* __restrict__ sw, int* err) {
  int64_t i = blockIdx.x;
  if (i >= rows) return;
  const float* wr = w + i * cols;
  float* wsr = ws + i * cols;
  float* swr = sw ? sw + i * cols : nullptr;
  int any_pos = 0, bad = 0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    int64_t g = gm(i, j);
    float x = __fdiv_rn(__fsub_rn(wr[j], betas[g]), alphas[g]);
    wsr[j] = x;
    bad |= !isfinite(x);
    if (swr) {
      float e = exj ? exj[j] : 1.0f;
      float v = weighting == ANYQ_W_WEIGHTS ? 1.0f
                : weighting == ANYQ_W_ACTS  ? e
                                            : __fmul_rn(alphas[g], e);
      swr[j] = v;
      any_pos |= v > 0.0f;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) dev_fail(err, ANYQ_ERR_NONFINITE);
  if (swr && !__syncthreads_or(any_pos)) {  // fully dead channels (learner.cpp:380)
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) swr[j] = 1.0f;
  }
}

// ---------------------------------------------------------------------------
// RTN onto a sorted table, ties toward the lower index (codebooks.cpp:75-97).
// ---------------------------------------------------------------------------
__global__ void k_round_to_table(const float* __restrict__ ws, int64_t n, Table t,
                                 uint8_t* __restrict__ codes) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float x = ws[e];
    int lo = 0, hi = t.n;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (t.v[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    uint8_t q;
    if (lo == 0) q = 0;
    else if (lo == t.n) q = (uint8_t)(t.n - 1);
    else q = (__fsub_rn(x, t.v[lo - 1]) <= __fsub_rn(t.v[lo], x)) ? (uint8_t)(lo - 1) : (uint8_t)lo;
    codes[e] = q;
  }
}

// ---------------------------------------------------------------------------
// Packing (pack.cpp:15-55): one thread per output byte / per code.
// ---------------------------------------------------------------------------
__global__ void k_pack(const uint8_t* __restrict__ codes, int64_t rows, int64_t cols, int bits,
                       uint8_t* __restrict__ out, int* err) {
  int64_t bpr = (cols * bits + 7) / 8;
  int64_t total = rows * bpr;
  uint32_t limit = 1u << bits;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / bpr, b = e % bpr;
    int64_t j0 = (8 * b) / bits, j1 = min(cols - 1, (8 * b + 7) / bits);
    uint32_t byte = 0;
    for (int64_t j = j0; j <= j1; ++j) {
      uint32_t c = codes[i * cols + j];
      if (c >= limit) dev_fail(err, ANYQ_ERR_CODE_RANGE);
      int64_t bit = j * bits;
      if ((bit >> 3) == b) byte |= (c << (bit & 7)) & 0xFFu;
      else if ((bit & 7) + bits > 8 && (bit >> 3) + 1 == b) byte |= (c >> (8 - (bit & 7))) & 0xFFu;
    }
    out[e] = (uint8_t)byte;
  }
}

__device__ __forceinline__ uint32_t code_at(const uint8_t* __restrict__ row, int64_t j, int bits) {
  int64_t bit = j * bits;
  uint32_t v = (uint32_t)row[bit >> 3] >> (bit & 7);
  if ((bit & 7) + bits > 8) v |= (uint32_t)row[(bit >> 3) + 1] << (8 - (bit & 7));
  return v & ((1u << bits) - 1u);
}

__global__ void k_unpack(const uint8_t* __restrict__ packed, int64_t rows, int64_t cols, int bits,
                         uint8_t* __restrict__ codes) {
  int64_t bpr = (cols * bits + 7) / 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols, j = e % cols;
    codes[e] = (uint8_t)code_at(packed + i * bpr, j, bits);
  }
}

// Logical codes -> k-tiled logical codes (inverse=0), or back (inverse=1).
__global__ void k_ktile(const uint8_t* __restrict__ in, int64_t rows, int64_t cols, int64_t tile_k,
                        int inverse, uint8_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols, j = e % cols;
    int64_t p = ktiled_pos(j, cols, tile_k);
    if (inverse) out[e] = in[i * cols + p];
    else out[i * cols + p] = in[e];
  }
}

// ---------------------------------------------------------------------------
// narrowed() (pack.cpp:159-169)
// ---------------------------------------------------------------------------
__global__ void k_narrow(float* __restrict__ v, int64_t n, int store, int is_alpha, int* err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int st = ANYQ_OK;
    float r = narrow_widen(v[e], store, &st);
    if (st != ANYQ_OK) dev_fail(err, st);
    else if (is_alpha && !(r > 0.0f)) dev_fail(err, ANYQ_ERR_INVARIANT);
    v[e] = r;
  }
}

// ---------------------------------------------------------------------------
// dequantize(qt) (pack.cpp:205-238 + scaling.cpp:85-96)
// ---------------------------------------------------------------------------
__global__ void k_dequant(const uint8_t* __restrict__ packed, int64_t rows, int64_t cols, int bits,
                          int ktiled, int64_t tile_k, const float* __restrict__ luts, Table fixed,
                          GroupMap gm, const float* __restrict__ alphas,
                          const float* __restrict__ betas, float* __restrict__ w, int* err) {
  int64_t bpr = (cols * bits + 7) / 8;
  int lut_n = 1 << bits;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols, j = e % cols;
    int64_t pos = ktiled ? ktiled_pos(j, cols, tile_k) : j;
    uint32_t c = code_at(packed + i * bpr, pos, bits);
    float v;
    if (luts) {
      v = luts[i * lut_n + c];
    } else {
      if ((int)c >= fixed.n) {
        dev_fail(err, ANYQ_ERR_CODE_RANGE);
        v = 0.0f;
      } else {
        v = fixed.v[c];
      }
    }
    if (alphas) {
      int64_t g = gm(i, j);
      w[e] = __fadd_rn(__fmul_rn(alphas[g], v), betas[g]);
    } else {
      w[e] = v;  // scaled_values (pack.cpp:205-236): the table value itself
    }
  }
}

// build_sample_weights (learner.cpp:25-51) for one row of a scale set.
__global__ void k_sample_weights(int64_t row, int64_t cols, GroupMap gm,
                                 const float* __restrict__ alphas, const float* __restrict__ stats,
                                 int weighting, float* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cols;
       j += (int64_t)gridDim.x * blockDim.x) {
    const float e = stats ? stats[j] : 1.0f;
    out[j] = weighting == ANYQ_W_WEIGHTS ? 1.0f
             : weighting == ANYQ_W_ACTS  ? e
                                         : __fmul_rn(alphas[gm(row, j)], e);
  }
}

// ---------------------------------------------------------------------------
// Bit-exact LUT GEMM, gemm_fused semantics (qgemm.cpp:71-128): per output
// element, k ascending, fp32 accumulate, no contraction. One thread per
// (row of W, row of x). Used for arbitrary configs (any bits, codebook,
// granularity, layout, ragged K) and as the exact mode of the C-ABI.
// ---------------------------------------------------------------------------
__global__ void k_gemm_exact(const float* __restrict__ x, int64_t m, int64_t k,
                             const uint8_t* __restrict__ packed, int64_t n, int bits, int ktiled,
                             int64_t tile_k, const float* __restrict__ luts, Table fixed,
                             GroupMap gm, const float* __restrict__ alphas,
                             const float* __restrict__ betas, float* __restrict__ y, int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // row of W
  int64_t r = blockIdx.y;                                         // row of x
  if (i >= n || r >= m) return;
  int64_t bpr = (k * bits + 7) / 8;
  const uint8_t* row = packed + i * bpr;
  const float* xr = x + r * k;
  const float* table = luts ? luts + i * (int64_t(1) << bits) : fixed.v;
  int tsize = luts ? (1 << bits) : fixed.n;
  float acc = 0.0f;
  for (int64_t j = 0; j < k; ++j) {
    int64_t pos = ktiled ? ktiled_pos(j, k, tile_k) : j;
    uint32_t c = code_at(row, pos, bits);
    if ((int)c >= tsize) {
      dev_fail(err, ANYQ_ERR_CODE_RANGE);
      c = 0;
    }
    int64_t g = gm(i, j);
    float wv = __fadd_rn(__fmul_rn(alphas[g], table[c]), betas[g]);
    acc = __fadd_rn(acc, __fmul_rn(xr[j], wv));
  }
  y[r * n + i] = acc;
}

// The same bit-exact semantics, fast path (<= 4-bit codes, tensorwise /
// rowwise / groupwise scales). Each output is ONE k-ascending chain of fadd
// (no contraction) — the reference's — and only that chain is sequential:
// the weights alpha*T[c]+beta and the products x*w are independent per k.
// The codes are first rewritten as one byte per weight in 1-KB tiles
// [row block][k tile][32 rows][32 k] (k_tile_codes) and x as 1-KB tiles
// [x chunk][k tile][8 rows][32 k], so each tile is ONE cp.async.bulk into an
// 8-stage shared-memory ring. A CTA owns 32 W rows and up to 8 x rows: 4
// producer warps turn tile t + 1 into products ([x row][k][W row], warp w:
// k = 8w..8w+7, lane = W row) while the adder warp (lane = W row) folds tile
// t into its accumulators in k order; one CTA barrier per tile.
constexpr int kExRows = 32, kExKT = 32, kExMC = 8, kExProd = 4, kExStages = 8;
constexpr int kExThreads = (kExProd + 1) * 32;
constexpr uint32_t kExTile = 1024;  // bytes of a code tile, and of an x tile (8 x 32 fp32)

__global__ void k_tile_codes(const uint8_t* __restrict__ packed, int64_t rows, int64_t cols, int bits,
                             int ktiled, int64_t tile_k, uint8_t* __restrict__ out) {
  // one thread per (row, 32-k tile): 32 logical codes of the row
  const int64_t nt = (cols + kExKT - 1) / kExKT, rb_n = (rows + kExRows - 1) / kExRows;
  const int64_t bpr = (cols * bits + 7) / 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rb_n * kExRows * nt;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e % nt, rr = e / nt;  // rr = global row (incl. padding)
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (rr < rows) {
      const uint8_t* row = packed + rr * bpr;
      for (int kk = 0; kk < kExKT; ++kk) {
        const int64_t j = t * kExKT + kk;
        if (j < cols) {
          const int64_t pos = ktiled ? ktiled_pos(j, cols, tile_k) : j;
          w[kk >> 2] |= code_at(row, pos, bits) << (8 * (kk & 3));
        }
      }
    }
    uint4* d = reinterpret_cast<uint4*>(out + (((rr / kExRows) * nt + t) * kExRows + rr % kExRows) * kExKT);
    d[0] = make_uint4(w[0], w[1], w[2], w[3]);
    d[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

__global__ void k_tile_x(const float* __restrict__ x, int64_t m, int64_t k, float* __restrict__ out) {
  const int64_t nt = (k + kExKT - 1) / kExKT, mch = (m + kExMC - 1) / kExMC;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mch * nt * kExMC * kExKT;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int kk = (int)(e % kExKT), q = (int)((e / kExKT) % kExMC);
    const int64_t t = (e / (kExKT * kExMC)) % nt, c = e / (kExKT * kExMC * nt);
    const int64_t r = c * kExMC + q, j = t * kExKT + kk;
    out[e] = (r < m && j < k) ? x[r * k + j] : 0.0f;
  }
}

template <int MCT>  // x rows this instance carries (1, 2, 4 or 8; the chunk's rows beyond m are zero)
__global__ void __launch_bounds__(kExThreads) k_gemm_exact_fast(
    const float* __restrict__ xt, int64_t m, int64_t k, const uint8_t* __restrict__ ctile, int64_t n,
    const float* __restrict__ luts, int lut_n, Table fixed, GroupMap gm, const float* __restrict__ alphas,
    const float* __restrict__ betas, float* __restrict__ y, int* err) {
  extern __shared__ __align__(128) uint8_t ex_smem[];
  float* prod = reinterpret_cast<float*>(ex_smem);                            // [2][kExMC][kExKT][32]
  uint8_t* ring = ex_smem + 2 * kExMC * kExKT * 32 * 4;                        // [stages][codes 1 KB | x 1 KB]
  float* st = reinterpret_cast<float*>(ring + kExStages * 2 * kExTile);        // [32][17]
  uint64_t* full = reinterpret_cast<uint64_t*>(st + 32 * 17);                  // [stages]
  uint64_t* empty = full + kExStages;                                          // [stages]
  float2* sab = reinterpret_cast<float2*>(empty + kExStages);                  // [32][gloc] (alpha, beta)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = (int64_t)blockIdx.x * kExRows, i = i0 + lane;
  const int64_t mchunk = blockIdx.y, r0 = mchunk * kExMC;
  const int mc = (int)(m - r0 < kExMC ? m - r0 : kExMC);
  const int tsize = luts ? lut_n : fixed.n;
  const bool live = i < n;
  const int ntiles = (int)((k + kExKT - 1) / kExKT);
  const bool tile_groups = gm.granularity != ANYQ_G_GROUP || gm.group_size % kExKT == 0;
  const uint8_t* cbase = ctile + (int64_t)blockIdx.x * ntiles * kExTile;
  const uint8_t* xbase = reinterpret_cast<const uint8_t*>(xt) + mchunk * ntiles * kExTile;
  const uint32_t sring = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t sfull = (uint32_t)__cvta_generic_to_shared(full), sempty = (uint32_t)__cvta_generic_to_shared(empty);
  for (int e = threadIdx.x; e < kExRows * 16; e += kExThreads) {
    const int rr = e >> 4, c = e & 15;
    float v = 0.0f;
    if (c < tsize) v = luts ? (i0 + rr < n ? luts[(i0 + rr) * lut_n + c] : 0.0f) : fixed.v[c];
    st[rr * 17 + c] = v;
  }
  // the rows' scale groups (tensorwise / rowwise: 1, groupwise: ceil(K / g)) in shared memory
  const int gloc = gm.granularity == ANYQ_G_GROUP ? (int)gm.gpr : 1;
  for (int e = threadIdx.x; e < kExRows * gloc; e += kExThreads) {
    const int rr = e / gloc, gg = e % gloc;
    float2 v = make_float2(1.0f, 0.0f);
    if (i0 + rr < n) {
      const int64_t g = gm.granularity == ANYQ_G_GROUP ? (i0 + rr) * gm.gpr + gg : gm(i0 + rr, 0);
      v = make_float2(alphas[g], betas[g]);
    }
    sab[e] = v;
  }
  if (threadIdx.x == 0) {
    for (int j = 0; j < kExStages; ++j) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sfull + 8 * j), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sempty + 8 * j), "r"(kExProd));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int t) {  // one thread: tile t's codes and x into stage t % stages
    const int s2 = t % kExStages;
    const uint32_t bar = sfull + 8 * s2, dst = sring + s2 * 2 * kExTile;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * kExTile) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(cbase + (int64_t)t * kExTile), "r"(kExTile), "r"(bar)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst + kExTile),
                 "l"(xbase + (int64_t)t * kExTile), "r"(kExTile), "r"(bar)
                 : "memory");
  };
  auto wait = [&](uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok)
                   : "r"(bar), "r"(parity), "r"(0x989680)
                   : "memory");
  };
  uint32_t bad = 0;
  auto produce = [&](int t) {
    const int s2 = t % kExStages;
    wait(sfull + 8 * s2, (uint32_t)((t / kExStages) & 1));
    const uint8_t* sc = ring + s2 * 2 * kExTile;
    const float* sx = reinterpret_cast<const float*>(sc + kExTile);
    float* pb = prod + (t & 1) * kExMC * kExKT * 32;
    const int64_t k0 = (int64_t)t * kExKT;
    if (live) {
      const uint32_t w0 = *reinterpret_cast<const uint32_t*>(sc + lane * kExKT + warp * 8);
      const uint32_t w1 = *reinterpret_cast<const uint32_t*>(sc + lane * kExKT + warp * 8 + 4);
      float2 ab = make_float2(1.0f, 0.0f);
      if (tile_groups) ab = sab[lane * gloc + (gloc > 1 ? (int)(k0 / gm.group_size) : 0)];
      // all loads of the 8 k first (table values, x broadcasts), then the arithmetic
      float tv[8], wv[8];
      float2 abk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t j = k0 + warp * 8 + u;
        uint32_t c = ((u < 4 ? w0 : w1) >> (8 * (u & 3))) & 0xFFu;
        bad |= (uint32_t)(j < k && (int)c >= tsize);
        c = (int)c >= tsize ? 0u : c;
        tv[u] = st[lane * 17 + c];
        abk[u] = tile_groups ? ab : sab[lane * gloc + (j < k ? (int)(j / gm.group_size) : 0)];
      }
      float xv[MCT][8];
#pragma unroll
      for (int q = 0; q < MCT; ++q) {
        const float4 x0 = *reinterpret_cast<const float4*>(sx + q * kExKT + warp * 8);
        const float4 x1 = *reinterpret_cast<const float4*>(sx + q * kExKT + warp * 8 + 4);
        xv[q][0] = x0.x; xv[q][1] = x0.y; xv[q][2] = x0.z; xv[q][3] = x0.w;
        xv[q][4] = x1.x; xv[q][5] = x1.y; xv[q][6] = x1.z; xv[q][7] = x1.w;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) wv[u] = __fadd_rn(__fmul_rn(abk[u].x, tv[u]), abk[u].y);
#pragma unroll
      for (int q = 0; q < MCT; ++q)
#pragma unroll
        for (int u = 0; u < 8; ++u) pb[(q * kExKT + warp * 8 + u) * 32 + lane] = __fmul_rn(xv[q][u], wv[u]);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sempty + 8 * s2) : "memory");
    // the issuing thread refills this stage with tile t + stages once all 4 producers read it
    if (threadIdx.x == 0 && t + kExStages < ntiles) {
      wait(sempty + 8 * s2, (uint32_t)((t / kExStages) & 1));
      issue(t + kExStages);
    }
  };
  float acc[kExMC];
#pragma unroll
  for (int q = 0; q < kExMC; ++q) acc[q] = 0.0f;
  if (threadIdx.x == 0)
    for (int t = 0; t < kExStages && t < ntiles; ++t) issue(t);
  if (warp < kExProd) produce(0);
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    if (warp < kExProd) {
      if (t + 1 < ntiles) produce(t + 1);
    } else {
      const float* pb = prod + (t & 1) * kExMC * kExKT * 32;
      const int kt = (int)(k - (int64_t)t * kExKT < kExKT ? k - (int64_t)t * kExKT : kExKT);
      if (kt == kExKT) {
#pragma unroll
        for (int kk = 0; kk < kExKT; ++kk)
#pragma unroll
          for (int q = 0; q < MCT; ++q) acc[q] = __fadd_rn(acc[q], pb[(q * kExKT + kk) * 32 + lane]);
      } else {  // the ragged last tile: the chain stops at k (no +0 terms)
        for (int q = 0; q < mc; ++q)
          for (int kk = 0; kk < kt; ++kk) acc[q] = __fadd_rn(acc[q], pb[(q * kExKT + kk) * 32 + lane]);
      }
    }
    __syncthreads();
  }
  if (warp < kExProd) {
    if (bad) dev_fail(err, ANYQ_ERR_CODE_RANGE);
  } else if (live) {
    for (int q = 0; q < mc; ++q) y[(r0 + q) * n + i] = acc[q];
  }
}

// gemm_dense (qgemm.cpp:22-34), same order and rounding.
__global__ void k_gemm_dense(const float* __restrict__ x, int64_t m, const float* __restrict__ w,
                             int64_t n, int64_t k, float* __restrict__ y) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t r = blockIdx.y;
  if (i >= n || r >= m) return;
  float acc = 0.0f;
  for (int64_t j = 0; j < k; ++j) acc = __fadd_rn(acc, __fmul_rn(x[r * k + j], w[i * k + j]));
  y[r * n + i] = acc;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int grid_for(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

void launch_check_finite(const float* p, int64_t n, int* err, int status, cudaStream_t s) {
  if (n <= 0) return;
  k_check_finite<<<grid_for(n), 256, 0, s>>>(p, n, err, status);
  ANYQ_LAUNCHED();
}

void launch_check_stats(const float* p, int64_t n, int* err, cudaStream_t s) {
  if (n <= 0) return;
  k_check_stats<<<grid_for(n), 256, 0, s>>>(p, n, err);
  ANYQ_LAUNCHED();
}

void launch_scales(const float* w, int64_t rows, int64_t cols, const anyq_config& cfg, float qmin,
                   float qmax, float* alphas, float* betas, cudaStream_t s) {
  GroupMap gm = make_group_map(cfg, cols);
  if (cfg.granularity == ANYQ_G_GROUP || cfg.granularity == ANYQ_G_ROW) {
    int64_t gsize = cfg.granularity == ANYQ_G_ROW ? cols : cfg.group_size;
    int64_t gpr = (cols + gsize - 1) / gsize;
    int64_t warps = rows * gpr;
    int64_t blocks = (warps * 32 + 255) / 256;
    k_scales_rowgroup<<<(unsigned)blocks, 256, 0, s>>>(w, rows, cols, gsize, gpr, cfg.symmetric != 0,
                                                       qmin, qmax, alphas, betas);
    ANYQ_LAUNCHED();
    return;
  }
  int64_t ng = group_count(cfg, rows, cols);
  DevBuf<uint32_t> kmin(ng, s), kmax(ng, s);
  DevBuf<unsigned long long> zmin(ng, s), zmax(ng, s);
  ANYQ_CUDA(cudaMemsetAsync(kmin.p, 0xFF, sizeof(uint32_t) * ng, s));
  ANYQ_CUDA(cudaMemsetAsync(kmax.p, 0x00, sizeof(uint32_t) * ng, s));
  ANYQ_CUDA(cudaMemsetAsync(zmin.p, 0xFF, sizeof(unsigned long long) * ng, s));
  ANYQ_CUDA(cudaMemsetAsync(zmax.p, 0xFF, sizeof(unsigned long long) * ng, s));
  k_scales_atomic<<<grid_for(rows * cols), 256, 0, s>>>(w, rows, cols, gm, kmin.p, kmax.p);
  ANYQ_LAUNCHED();
  k_scales_first_zero<<<grid_for(rows * cols), 256, 0, s>>>(w, rows, cols, gm, kmin.p, kmax.p,
                                                            zmin.p, zmax.p);
  ANYQ_LAUNCHED();
  k_scales_finish<<<(unsigned)((ng + 255) / 256), 256, 0, s>>>(w, ng, kmin.p, kmax.p, zmin.p, zmax.p,
                                                              cfg.symmetric != 0, qmin, qmax,
                                                              alphas, betas);
  ANYQ_LAUNCHED();
  // scratch is released stream-ordered on return (no host synchronisation)
}

void launch_scale_rows(const float* w, int64_t rows, int64_t cols, const anyq_config& cfg,
                       const float* alphas, const float* betas, const float* exj, float* ws,
                       float* sw, int* err, cudaStream_t s) {
  GroupMap gm = make_group_map(cfg, cols);
  k_scale_rows<<<(unsigned)rows, 256, 0, s>>>(w, rows, cols, gm, alphas, betas, exj, cfg.weighting,
                                              ws, sw, err);
  ANYQ_LAUNCHED();
}

// scale_weights (inverse = 1, scaling.cpp:72-83) / dequantize(values, s)
// (inverse = 0, scaling.cpp:85-96), element-wise in the reference's order of
// operations (no contraction).
__global__ void k_affine(const float* __restrict__ in, int64_t rows, int64_t cols, GroupMap gm,
                         const float* __restrict__ alphas, const float* __restrict__ betas,
                         int inverse, float* __restrict__ out) {
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e - i * cols;
    const int64_t g = gm(i, j);
    out[e] = inverse ? __fdiv_rn(__fsub_rn(in[e], betas[g]), alphas[g])
                     : __fadd_rn(__fmul_rn(alphas[g], in[e]), betas[g]);
  }
}

void launch_affine(const float* in, int64_t rows, int64_t cols, const anyq_config& cfg,
                   const float* alphas, const float* betas, int inverse, float* out,
                   cudaStream_t s) {
  GroupMap gm = make_group_map(cfg, cols);
  k_affine<<<grid_for(rows * cols), 256, 0, s>>>(in, rows, cols, gm, alphas, betas, inverse, out);
  ANYQ_LAUNCHED();
}

void launch_sample_weights(const anyq_config& cfg, int64_t row, int64_t cols, const float* alphas,
                           const float* stats, int weighting, float* out, cudaStream_t s) {
  k_sample_weights<<<grid_for(cols), 256, 0, s>>>(row, cols, make_group_map(cfg, cols), alphas, stats,
                                                 weighting, out);
  ANYQ_LAUNCHED();
}

void launch_round(const float* ws, int64_t n, const Table& t, uint8_t* codes, cudaStream_t s) {
  k_round_to_table<<<grid_for(n), 256, 0, s>>>(ws, n, t, codes);
  ANYQ_LAUNCHED();
}

void launch_pack(const uint8_t* codes, int64_t rows, int64_t cols, int bits, uint8_t* out,
                 int* err, cudaStream_t s) {
  int64_t total = rows * packed_bpr(cols, bits);
  k_pack<<<grid_for(total), 256, 0, s>>>(codes, rows, cols, bits, out, err);
  ANYQ_LAUNCHED();
}

void launch_unpack(const uint8_t* packed, int64_t rows, int64_t cols, int bits, uint8_t* codes,
                   cudaStream_t s) {
  k_unpack<<<grid_for(rows * cols), 256, 0, s>>>(packed, rows, cols, bits, codes);
  ANYQ_LAUNCHED();
}

void launch_ktile(const uint8_t* in, int64_t rows, int64_t cols, int64_t tile_k, int inverse,
                  uint8_t* out, cudaStream_t s) {
  k_ktile<<<grid_for(rows * cols), 256, 0, s>>>(in, rows, cols, tile_k, inverse, out);
  ANYQ_LAUNCHED();
}

void launch_narrow(float* v, int64_t n, int store, int is_alpha, int* err, cudaStream_t s) {
  if (n <= 0 || store == ANYQ_STORE_FP32) {
    if (is_alpha && n > 0) {  // fp32 store still requires alpha > 0 after narrowing (identity)
      k_narrow<<<grid_for(n), 256, 0, s>>>(v, n, ANYQ_STORE_FP32, is_alpha, err);
      ANYQ_LAUNCHED();
    }
    return;
  }
  k_narrow<<<grid_for(n), 256, 0, s>>>(v, n, store, is_alpha, err);
  ANYQ_LAUNCHED();
}

void launch_dequant(const uint8_t* packed, int64_t rows, int64_t cols, int bits, int ktiled,
                    int64_t tile_k, const float* luts, const Table& fixed, const anyq_config& cfg,
                    const float* alphas, const float* betas, float* w, int* err, cudaStream_t s) {
  GroupMap gm = make_group_map(cfg, cols);
  k_dequant<<<grid_for(rows * cols), 256, 0, s>>>(packed, rows, cols, bits, ktiled, tile_k, luts,
                                                  fixed, gm, alphas, betas, w, err);
  ANYQ_LAUNCHED();
}

void launch_gemm_exact(const float* x, int64_t m, int64_t k, const uint8_t* packed, int64_t n,
                       int bits, int ktiled, int64_t tile_k, const float* luts, const Table& fixed,
                       const anyq_config& cfg, const float* alphas, const float* betas, float* y,
                       int* err, cudaStream_t s) {
  GroupMap gm = make_group_map(cfg, k);
  const int lut_n = 1 << bits;
  const bool fast_gran = cfg.granularity == ANYQ_G_TENSOR || cfg.granularity == ANYQ_G_ROW ||
                         cfg.granularity == ANYQ_G_GROUP;
  const int64_t gl = cfg.granularity == ANYQ_G_GROUP ? gm.gpr : 1;
  if (bits <= 4 && fast_gran && n > 0 && m > 0 && k > 0 && gl <= 512) {
    // codes and x in 1-KB tiles (zero padded; the adder stops at k), then the fast kernel
    const int64_t nt = (k + kExKT - 1) / kExKT, rbn = (n + kExRows - 1) / kExRows;
    const int64_t mch = (m + kExMC - 1) / kExMC;
    DevBuf<uint8_t> ct((size_t)(rbn * nt * kExTile), s);
    DevBuf<float> xt((size_t)(mch * nt * kExMC * kExKT), s);
    k_tile_codes<<<grid_for(rbn * kExRows * nt), 256, 0, s>>>(packed, n, k, bits, ktiled, tile_k, ct.p);
    ANYQ_LAUNCHED();
    k_tile_x<<<grid_for(mch * nt * kExMC * kExKT), 256, 0, s>>>(x, m, k, xt.p);
    ANYQ_LAUNCHED();
    dim3 grid((unsigned)rbn, (unsigned)mch);
    const int gloc = cfg.granularity == ANYQ_G_GROUP ? (int)gm.gpr : 1;
    const int smem = (int)(2 * kExMC * kExKT * 32 * 4 + kExStages * 2 * kExTile + 32 * 17 * 4 + 2 * kExStages * 8 +
                           32 * gloc * 8);
    auto go = [&](auto kern) {
      ensure_dyn_smem((const void*)kern, smem);
      kern<<<grid, kExThreads, smem, s>>>(xt.p, m, k, ct.p, n, luts, lut_n, fixed, gm, alphas, betas, y, err);
    };
    if (m == 1) go(k_gemm_exact_fast<1>);
    else if (m == 2) go(k_gemm_exact_fast<2>);
    else if (m <= 4) go(k_gemm_exact_fast<4>);
    else go(k_gemm_exact_fast<8>);
    ANYQ_LAUNCHED();
    return;
  }
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)m);
  k_gemm_exact<<<grid, 128, 0, s>>>(x, m, k, packed, n, bits, ktiled, tile_k, luts, fixed, gm,
                                    alphas, betas, y, err);
  ANYQ_LAUNCHED();
}

void launch_gemm_dense(const float* x, int64_t m, const float* w, int64_t n, int64_t k, float* y,
                       cudaStream_t s) {
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)m);
  k_gemm_dense<<<grid, 128, 0, s>>>(x, m, w, n, k, y);
  ANYQ_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Activation statistics E|x_j| (collect_stats, calibration.cpp:62-67): per
// channel j, sum over the samples m = 0..M-1 IN ORDER of |x(m, j)| in double,
// divided by M in double, rounded once to float. The sum stays sequential per
// channel (bit-identical to the reference); what is parallel is the memory:
// a CTA owns 32 channels, its 8 warps load the next 256-sample x 32-channel
// tile (one 128-B row segment per load, 32 loads in flight per lane) while
// warp 0 runs the 32 sequential double sums over the current tile in shared
// memory. HBM-bound when M is large and the DADD chain (M deep) otherwise.
// ---------------------------------------------------------------------------
constexpr int kStatCols = 32, kStatRows = 256, kStatThreads = 256;

__global__ void __launch_bounds__(kStatThreads) k_col_mean_abs(const float* __restrict__ x, int64_t m,
                                                               int64_t k, float* __restrict__ out,
                                                               int* __restrict__ err) {
  __shared__ float tile[kStatRows][kStatCols + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * kStatCols + lane;
  const bool col = j < k;
  constexpr int kPer = kStatRows / (kStatThreads / 32);  // rows per warp and tile
  float v[kPer];
  auto load = [&](int64_t r0) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int64_t r = r0 + warp * kPer + i;
      v[i] = (col && r < m) ? __ldg(x + r * k + j) : 0.0f;
    }
  };
  double acc = 0.0;
  bool finite = true;  // require_finite(inputs) (calibration.cpp:52), fused into the one pass
  load(0);
  for (int64_t r0 = 0; r0 < m; r0 += kStatRows) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      finite &= isfinite(v[i]);
      tile[warp * kPer + i][lane] = v[i];
    }
    __syncthreads();
    if (r0 + kStatRows < m) load(r0 + kStatRows);  // next tile in flight during the sums
    if (warp == 0) {
      const int n = (int)(m - r0 < kStatRows ? m - r0 : kStatRows);
      if (n == kStatRows) {  // shared-memory reads run ahead of the dependent adds
#pragma unroll 32
        for (int i = 0; i < kStatRows; ++i) acc += fabs((double)tile[i][lane]);
      } else {
        for (int i = 0; i < n; ++i) acc += fabs((double)tile[i][lane]);
      }
    }
    __syncthreads();
  }
  if (!finite) atomicExch(err, (int)ANYQ_ERR_NONFINITE);
  if (warp == 0 && col) out[j] = (float)(acc / (double)m);
}

void launch_col_mean_abs(const float* x, int64_t m, int64_t k, float* out, int* err, cudaStream_t s) {
  if (k <= 0 || m <= 0) return;
  k_col_mean_abs<<<(unsigned)((k + kStatCols - 1) / kStatCols), kStatThreads, 0, s>>>(x, m, k, out,
                                                                                       err);
  ANYQ_LAUNCHED();
}

// ---------------------------------------------------------------------------
// eval.cpp:11-46 (weight_error / output_error): sum (a - b)^2 and sum a^2 in
// double, products and sums rounded separately like the reference's
// `sq += e * e` (no FMA contraction). The reference sums sequentially; here a
// fixed-shape two-level tree (kRedBlocks x kRedThreads strided partials, then
// one block) -- deterministic on any device, equal to the reference up to
// reassociation of the double sums.
// ---------------------------------------------------------------------------
constexpr int kRedBlocks = 592, kRedThreads = 256;

__device__ __forceinline__ void tree2(double* r1, double* r2, double& s1, double& s2) {
  const int t = threadIdx.x;
  r1[t] = s1;
  r2[t] = s2;
  __syncthreads();
  for (int w = kRedThreads / 2; w > 0; w >>= 1) {
    if (t < w) {
      r1[t] = __dadd_rn(r1[t], r1[t + w]);
      r2[t] = __dadd_rn(r2[t], r2[t + w]);
    }
    __syncthreads();
  }
  s1 = r1[0];
  s2 = r2[0];
}

__global__ void __launch_bounds__(kRedThreads) k_sqdiff_partial(const float* __restrict__ a,
                                                                const float* __restrict__ b, int64_t n,
                                                                double* __restrict__ part) {
  __shared__ double r1[kRedThreads], r2[kRedThreads];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; e < n;
       e += (int64_t)kRedBlocks * kRedThreads) {
    const double av = (double)a[e];
    const double d = __dsub_rn(av, (double)b[e]);
    s1 = __dadd_rn(s1, __dmul_rn(d, d));
    s2 = __dadd_rn(s2, __dmul_rn(av, av));
  }
  tree2(r1, r2, s1, s2);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s1;
    part[kRedBlocks + blockIdx.x] = s2;
  }
}

__global__ void __launch_bounds__(kRedThreads) k_sum_partials(const double* __restrict__ part,
                                                              double* __restrict__ out) {
  __shared__ double r1[kRedThreads], r2[kRedThreads];
  double s1 = 0.0, s2 = 0.0;
  for (int i = threadIdx.x; i < kRedBlocks; i += kRedThreads) {
    s1 = __dadd_rn(s1, part[i]);
    s2 = __dadd_rn(s2, part[kRedBlocks + i]);
  }
  tree2(r1, r2, s1, s2);
  if (threadIdx.x == 0) {
    out[0] = s1;
    out[1] = s2;
  }
}

void launch_sqdiff_sums(const float* a, const float* b, int64_t n, double* part, double* out2,
                        cudaStream_t s) {
  k_sqdiff_partial<<<kRedBlocks, kRedThreads, 0, s>>>(a, b, n, part);
  ANYQ_LAUNCHED();
  k_sum_partials<<<1, kRedThreads, 0, s>>>(part, out2);
  ANYQ_LAUNCHED();
}

}  // namespace anyq_b200
