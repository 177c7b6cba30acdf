// Per-row activation-weighted k-means (learner.cpp:132-369) on the GPU.
//
// One CTA (256 threads) per row, persistent over rows via an atomic row
// counter. Each row is first sorted once (cub segmented stable sort of the
// scaled weights, index as payload); Lloyd then works on the sorted row:
//
//  * E-step — exact reference semantics (learner.cpp:185-196): the nearest
//    centroid by fl((x-c)^2) in double, ties to the smallest ORIGINAL centroid
//    index. Costs are monotone in |x-c| after rounding, so the minimum lies at
//    the two centroids bracketing x in sorted order; the tied set is expanded
//    from there. O(log k) per sample instead of O(k).
//  * M-step — 1-D nearest-centroid assignment is monotone in x, so every
//    cluster is one contiguous segment of the sorted row. Segment sums of
//    w*x, w, x (double) are formed per thread-chunk and combined in a fixed
//    order: deterministic, independent of the launch configuration. (The
//    reference sums in sample-index order; the two agree to ~1e-15 relative,
//    so the float LUTs are bit-identical on essentially every row; tests
//    report the fraction.) A non-monotone assignment is detected and falls
//    back to a direct per-cluster scan.
//  * empty clusters, convergence (stable / rel_tol / zero loss), restarts and
//    the final sort + rank remap follow learner.cpp:274-369 step for step.
//
// k-means++ (learner.cpp:132-174) runs on the row in ORIGINAL index order so
// the cumulative-mass sampling selects the same sample as the reference; the
// RNG stream (core.hpp:164-200) is reproduced bit for bit.
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace anyq_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxK = 256;

struct KmParams {
  const float* ws;     // rows x n, original order
  const float* sw;     // rows x n, original order
  const float* skeys;  // rows x n, sorted values
  const int* svals;    // rows x n, original index of each sorted position
  int64_t rows, n;
  int k, init, max_iters, restarts, check_inv;
  float rel_tol;
  uint64_t seed;
  int64_t row_offset;
  float* luts;     // rows x k
  uint8_t* codes;  // rows x n (logical, original order)
  int* err;
  int* row_counter;
  uint8_t* gscratch;  // per-block scratch when the row does not fit in smem
  size_t scratch_stride;
  int use_smem;
};

struct Part {  // partial segment sums
  double swx, sw, sx;
};

struct Shared {
  double cen[kMaxK];
  double best_cen[kMaxK];
  double sv[kMaxK];  // centroid values sorted ascending (ties by index)
  int so[kMaxK];     // original index of sv[r]
  int rank_of[kMaxK];
  int seg_start[kMaxK + 1];
  double swx[kMaxK], sw[kMaxK], sx[kMaxK];
  int cnt[kMaxK];
  Part first[kThreads], last[kThreads];
  int first_c[kThreads], last_c[kThreads], nruns[kThreads];
  double red_d[kWarps];
  long long red_l[kWarps];
  double dbl_bcast;
  long long ll_bcast;
  int int_bcast;
  int64_t row;
  Rng rng;
  int ncen;
};

__device__ __forceinline__ double dcost(double x, double c) {
  double d = __dsub_rn(x, c);
  return __dmul_rn(d, d);
}

// Deterministic block reductions (fixed shuffle tree, then warp order).
__device__ double block_sum(double v, Shared& sh) {
  for (int off = 16; off; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh.red_d[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kWarps; ++i) s = __dadd_rn(s, sh.red_d[i]);
    sh.dbl_bcast = s;
  }
  __syncthreads();
  return sh.dbl_bcast;
}

__device__ long long block_min_ll(long long v, Shared& sh) {
  for (int off = 16; off; off >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, off));
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh.red_l[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = sh.red_l[0];
    for (int i = 1; i < kWarps; ++i) s = min(s, sh.red_l[i]);
    sh.ll_bcast = s;
  }
  __syncthreads();
  return sh.ll_bcast;
}

__device__ long long block_max_ll(long long v, Shared& sh) { return -block_min_ll(-v, sh); }

// Exclusive block scan of one double per thread, in thread order.
__device__ double block_exclusive_scan(double v, Shared& sh, double* total) {
  // Warp-level inclusive scan (Hillis-Steele, fixed order per lane).
  int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  double incl = v;
  for (int off = 1; off < 32; off <<= 1) {
    double o = __shfl_up_sync(0xffffffffu, incl, off);
    if (l >= off) incl = __dadd_rn(o, incl);
  }
  __syncthreads();
  if (l == 31) sh.red_d[w] = incl;
  __syncthreads();
  double base = 0.0;
  for (int i = 0; i < w; ++i) base = __dadd_rn(base, sh.red_d[i]);
  double tot = 0.0;
  for (int i = 0; i < kWarps; ++i) tot = __dadd_rn(tot, sh.red_d[i]);
  *total = tot;
  double excl_in_warp = __shfl_up_sync(0xffffffffu, incl, 1);
  if (l == 0) excl_in_warp = 0.0;
  return __dadd_rn(base, excl_in_warp);
}

// Sort the current centroids by (value, index): sv/so/rank_of.
__device__ void sort_centroids(Shared& sh, int k) {
  __syncthreads();
  for (int q = threadIdx.x; q < k; q += kThreads) {
    double v = sh.cen[q];
    int r = 0;
    for (int p = 0; p < k; ++p) {
      double u = sh.cen[p];
      r += (u < v) || (u == v && p < q);
    }
    sh.rank_of[q] = r;
    sh.sv[r] = v;
    sh.so[r] = q;
  }
  __syncthreads();
}

// Exact reference nearest centroid (see file comment).
__device__ __forceinline__ int nearest(double x, const Shared& sh, int k) {
  int lo = 0, hi = k;  // first r with sv[r] >= x
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (sh.sv[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  int p = lo;
  double cl = p > 0 ? dcost(x, sh.sv[p - 1]) : INFINITY;
  double cr = p < k ? dcost(x, sh.sv[p]) : INFINITY;
  double mc = cl < cr ? cl : cr;
  int best = 1 << 30;
  for (int r = p - 1; r >= 0; --r) {
    double c = (r == p - 1) ? cl : dcost(x, sh.sv[r]);
    if (!(c == mc)) break;
    best = min(best, sh.so[r]);
  }
  for (int r = p; r < k; ++r) {
    double c = (r == p) ? cr : dcost(x, sh.sv[r]);
    if (!(c == mc)) break;
    best = min(best, sh.so[r]);
  }
  return best;
}

// sample_index (learner.cpp:64-75) over mass[i] (original order), chunked.
__device__ int64_t sample_index(const double* mass, int64_t n, int64_t C, double r_unit,
                                Shared& sh, double* total_out) {
  int64_t b = threadIdx.x * C, e = min(n, b + C);
  double local = 0.0;
  for (int64_t i = b; i < e; ++i)
    if (mass[i] > 0.0) local = __dadd_rn(local, mass[i]);
  double total;
  double excl = block_exclusive_scan(local, sh, &total);
  *total_out = total;
  if (!(total > 0.0)) return -1;
  if (threadIdx.x == 0) sh.dbl_bcast = __dmul_rn(r_unit, total);
  __syncthreads();
  double r = sh.dbl_bcast;
  long long cand = LLONG_MAX, lastpos = -1;
  double acc = excl;
  for (int64_t i = b; i < e; ++i) {
    if (!(mass[i] > 0.0)) continue;
    acc = __dadd_rn(acc, mass[i]);
    lastpos = i;
    if (r < acc) {
      cand = i;
      break;
    }
  }
  // lastpos must be the last positive index of the chunk even after a hit.
  if (cand != LLONG_MAX) {
    for (int64_t i = e - 1; i >= b; --i)
      if (mass[i] > 0.0) {
        lastpos = i;
        break;
      }
  }
  long long c = block_min_ll(cand, sh);
  long long lp = block_max_ll(lastpos, sh);
  return c != LLONG_MAX ? c : lp;
}

// m-th distinct sample value in ascending order, cycling (pad_with_distinct).
__device__ double distinct_value(const float* xs, int64_t n, int64_t m) {
  int64_t nd = 0;
  for (int64_t j = 0; j < n; ++j)
    if (j == 0 || !((double)xs[j] == (double)xs[j - 1])) ++nd;
  int64_t want = m % nd, seen = -1;
  for (int64_t j = 0; j < n; ++j)
    if (j == 0 || !((double)xs[j] == (double)xs[j - 1]))
      if (++seen == want) return (double)xs[j];
  return (double)xs[0];
}

__device__ void init_kmeanspp(const KmParams& P, const float* xo, const float* wo, const float* xs,
                              double* d2, Shared& sh, int k) {
  const int64_t n = P.n;
  const int64_t C = (n + kThreads - 1) / kThreads;
  const int64_t b = threadIdx.x * C, e = min(n, b + C);
  // first centroid: mass = w
  for (int64_t i = b; i < e; ++i) d2[i] = (double)wo[i];
  __syncthreads();
  double u = 0.0;
  if (threadIdx.x == 0) sh.dbl_bcast = sh.rng.next_double();
  __syncthreads();
  u = sh.dbl_bcast;
  double total;
  int64_t pick = sample_index(d2, n, C, u, sh, &total);
  if (threadIdx.x == 0) {
    sh.cen[0] = (double)xo[pick];
    sh.ncen = 1;
  }
  __syncthreads();
  // d2 holds D^2 from here on; mass lives in the second half of the scratch.
  double* mass = d2 + n;
  for (int64_t i = b; i < e; ++i) d2[i] = INFINITY;
  __syncthreads();
  while (sh.ncen < k) {
    double c = sh.cen[sh.ncen - 1];
    for (int64_t i = b; i < e; ++i) {
      double pc = dcost((double)xo[i], c);
      d2[i] = (pc < d2[i]) ? pc : d2[i];
      mass[i] = __dmul_rn((double)wo[i], d2[i]);
    }
    __syncthreads();
    // The draw is consumed only when the weighted mass is positive; peek the
    // total first so the stream advances exactly as in the reference.
    double local = 0.0;
    for (int64_t i = b; i < e; ++i)
      if (mass[i] > 0.0) local = __dadd_rn(local, mass[i]);
    double tot = block_sum(local, sh);
    if (tot > 0.0) {
      if (threadIdx.x == 0) sh.dbl_bcast = sh.rng.next_double();
      __syncthreads();
      u = sh.dbl_bcast;
      pick = sample_index(mass, n, C, u, sh, &total);
      if (threadIdx.x == 0) sh.cen[sh.ncen++] = (double)xo[pick];
      __syncthreads();
      continue;
    }
    for (int64_t i = b; i < e; ++i) mass[i] = d2[i];
    __syncthreads();
    local = 0.0;
    for (int64_t i = b; i < e; ++i)
      if (mass[i] > 0.0) local = __dadd_rn(local, mass[i]);
    tot = block_sum(local, sh);
    if (tot > 0.0) {
      if (threadIdx.x == 0) sh.dbl_bcast = sh.rng.next_double();
      __syncthreads();
      u = sh.dbl_bcast;
      pick = sample_index(mass, n, C, u, sh, &total);
      if (threadIdx.x == 0) sh.cen[sh.ncen++] = (double)xo[pick];
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) {
      int64_t cursor = 0;
      while (sh.ncen < k) sh.cen[sh.ncen++] = distinct_value(xs, n, cursor++);
    }
    __syncthreads();
  }
}

__device__ void init_random(const KmParams& P, const float* xo, const float* xs, Shared& sh, int k,
                            int64_t* vkeys, int64_t* vvals) {
  if (threadIdx.x == 0) {
    const int64_t n = P.n;
    if ((int64_t)k >= n) {
      // all samples, sorted ascending, then cycle through distinct values
      int c = 0;
      for (int64_t j = 0; j < n; ++j) sh.cen[c++] = (double)xs[j];
      int64_t cursor = 0;
      while (c < k) sh.cen[c++] = distinct_value(xs, n, cursor++);
    } else {
      // partial Fisher-Yates over a virtual identity array (<= 2k touched)
      int used = 0;
      auto get = [&](int64_t pos) -> int64_t {
        for (int i = 0; i < used; ++i)
          if (vkeys[i] == pos) return vvals[i];
        return pos;
      };
      auto set = [&](int64_t pos, int64_t v) {
        for (int i = 0; i < used; ++i)
          if (vkeys[i] == pos) {
            vvals[i] = v;
            return;
          }
        vkeys[used] = pos;
        vvals[used] = v;
        ++used;
      };
      for (int t = 0; t < k; ++t) {
        int64_t pick = t + sh.rng.next_index(n - t);
        int64_t vt = get(t), vp = get(pick);
        set(t, vp);
        set(pick, vt);
        sh.cen[t] = (double)xo[vp];
      }
    }
  }
  __syncthreads();
}

// One Lloyd run (learner.cpp:207-312) on the sorted row. Returns the loss.
__device__ double lloyd(const KmParams& P, const float* xs, const float* wv, uint8_t* asg,
                        Shared& sh, int k) {
  const int64_t n = P.n;
  const int64_t C = (n + kThreads - 1) / kThreads;
  const int64_t b = threadIdx.x * C, e = min(n, b + C);
  for (int64_t j = b; j < e; ++j) asg[j] = 0;
  double prev = INFINITY;
  for (int iter = 0; iter < P.max_iters; ++iter) {
    // ---- E-step
    sort_centroids(sh, k);
    int changed = 0;
    for (int64_t j = b; j < e; ++j) {
      int q = nearest((double)xs[j], sh, k);
      changed |= q != asg[j];
      asg[j] = (uint8_t)q;
    }
    __syncthreads();
    if (P.check_inv) {
      int bad = 0;
      for (int64_t j = b; j < e; ++j) {
        double ca = dcost((double)xs[j], sh.cen[asg[j]]);
        for (int q = 0; q < k; ++q) bad |= dcost((double)xs[j], sh.cen[q]) < ca;
      }
      if (__syncthreads_or(bad) && threadIdx.x == 0) dev_fail(P.err, ANYQ_ERR_INTERNAL);
    }
    // ---- M-step: monotonicity check + segment boundaries
    int mono = 1;
    for (int64_t j = b; j < e; ++j) {
      int r = sh.rank_of[asg[j]];
      int rp = j > 0 ? sh.rank_of[asg[j - 1]] : -1;
      if (r < rp) mono = 0;
      for (int t = rp + 1; t <= r; ++t) sh.seg_start[t] = (int)j;
    }
    if (threadIdx.x == 0) {
      for (int t = sh.rank_of[asg[n - 1]] + 1; t <= k; ++t) sh.seg_start[t] = (int)n;
    }
    mono = __syncthreads_and(mono);
    if (mono) {
      // per-chunk runs: first / last partials, interior runs are complete
      int nr = 0, fc = -1, lc = -1;
      Part cur = {0, 0, 0};
      int curc = -1;
      for (int64_t j = b; j < e; ++j) {
        int q = asg[j];
        if (q != curc) {
          if (curc >= 0) {
            if (nr == 0) {
              sh.first[threadIdx.x] = cur;
              fc = curc;
            } else {  // interior run: the whole cluster lies in this chunk
              sh.swx[curc] = cur.swx;
              sh.sw[curc] = cur.sw;
              sh.sx[curc] = cur.sx;
            }
            ++nr;
          }
          curc = q;
          cur = {0, 0, 0};
        }
        double w = (double)wv[j], x = (double)xs[j];
        cur.swx = __dadd_rn(cur.swx, __dmul_rn(w, x));
        cur.sw = __dadd_rn(cur.sw, w);
        cur.sx = __dadd_rn(cur.sx, x);
      }
      if (curc >= 0) {
        if (nr == 0) {
          sh.first[threadIdx.x] = cur;
          fc = curc;
        } else {
          sh.last[threadIdx.x] = cur;
          lc = curc;
        }
        ++nr;
      }
      sh.first_c[threadIdx.x] = fc;
      sh.last_c[threadIdx.x] = lc;
      sh.nruns[threadIdx.x] = nr;
      __syncthreads();
      for (int q = threadIdx.x; q < k; q += kThreads) {
        int r = sh.rank_of[q];
        int a = sh.seg_start[r], z = sh.seg_start[r + 1];
        sh.cnt[q] = z - a;
        if (z <= a) continue;
        int t0 = (int)(a / C), t1 = (int)((z - 1) / C);
        bool starts_chunk = (int64_t)a == (int64_t)t0 * C;
        bool ends_chunk = (int64_t)z == min(n, (int64_t)(t0 + 1) * C);
        if (t0 == t1) {
          if (starts_chunk) {
            Part p = sh.first[t0];
            sh.swx[q] = p.swx;
            sh.sw[q] = p.sw;
            sh.sx[q] = p.sx;
          } else if (ends_chunk) {
            Part p = sh.last[t0];
            sh.swx[q] = p.swx;
            sh.sw[q] = p.sw;
            sh.sx[q] = p.sx;
          }  // else: interior run, already complete
          continue;
        }
        Part acc = starts_chunk ? sh.first[t0] : sh.last[t0];
        for (int t = t0 + 1; t <= t1; ++t) {
          Part p = sh.first[t];
          acc.swx = __dadd_rn(acc.swx, p.swx);
          acc.sw = __dadd_rn(acc.sw, p.sw);
          acc.sx = __dadd_rn(acc.sx, p.sx);
        }
        sh.swx[q] = acc.swx;
        sh.sw[q] = acc.sw;
        sh.sx[q] = acc.sx;
      }
    } else {
      // fallback: direct scan per cluster (fixed order, slow, rare)
      for (int q = threadIdx.x; q < k; q += kThreads) {
        double swx = 0, sw = 0, sx = 0;
        int c = 0;
        for (int64_t j = 0; j < n; ++j)
          if (asg[j] == q) {
            double w = (double)wv[j], x = (double)xs[j];
            swx = __dadd_rn(swx, __dmul_rn(w, x));
            sw = __dadd_rn(sw, w);
            sx = __dadd_rn(sx, x);
            ++c;
          }
        sh.swx[q] = swx;
        sh.sw[q] = sw;
        sh.sx[q] = sx;
        sh.cnt[q] = c;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 0; q < k; ++q) {
        if (sh.cnt[q] == 0) continue;
        if (sh.sw[q] > 0.0) sh.cen[q] = __ddiv_rn(sh.swx[q], sh.sw[q]);
        else sh.cen[q] = __ddiv_rn(sh.sx[q], (double)sh.cnt[q]);
      }
    }
    __syncthreads();
    // ---- empty-cluster repair (learner.cpp:274-289), in cluster order
    int repairs = 0;
    for (int q = 0; q < k; ++q) {
      if (sh.cnt[q] != 0) continue;
      ++repairs;
      // worst = first (smallest ORIGINAL index) sample with the largest error
      double worst = -1.0;
      long long wi = LLONG_MAX;
      for (int64_t j = b; j < e; ++j) {
        double err = __dmul_rn((double)wv[j], dcost((double)xs[j], sh.cen[asg[j]]));
        long long oi = (long long)P.svals[sh.row * n + j];
        if (err > worst || (err == worst && oi < wi)) {
          worst = err;
          wi = oi;
        }
      }
      // block argmax with smallest-index tie break: reduce on (err, -idx)
      // via two passes (max err, then min idx among equals).
      __syncthreads();
      {
        double v = worst;
        for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
        if ((threadIdx.x & 31) == 0) sh.red_d[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
          double m = sh.red_d[0];
          for (int i = 1; i < kWarps; ++i) m = fmax(m, sh.red_d[i]);
          sh.dbl_bcast = m;
        }
        __syncthreads();
      }
      double wmax = sh.dbl_bcast;
      long long cand = (worst == wmax) ? wi : LLONG_MAX;
      long long widx = block_min_ll(cand, sh);
      // locate the sorted position holding original index widx
      for (int64_t j = b; j < e; ++j)
        if ((long long)P.svals[sh.row * n + j] == widx) {
          sh.cen[q] = (double)xs[j];
          asg[j] = (uint8_t)q;
        }
      __syncthreads();
    }
    // ---- loss after the update (sample order fixed by chunk, then tree)
    double local = 0.0;
    for (int64_t j = b; j < e; ++j)
      local = __dadd_rn(local, __dmul_rn((double)wv[j], dcost((double)xs[j], sh.cen[asg[j]])));
    double loss_m = block_sum(local, sh);
    int any_changed = __syncthreads_or(changed) || repairs > 0;
    bool stable = !any_changed && iter > 0;
    bool tol = isfinite(prev) && __dsub_rn(prev, loss_m) <= __dmul_rn((double)P.rel_tol, prev);
    prev = loss_m;
    if (stable || tol || loss_m == 0.0) break;
  }
  // final reassignment and loss
  sort_centroids(sh, k);
  double local = 0.0;
  for (int64_t j = b; j < e; ++j) {
    int q = nearest((double)xs[j], sh, k);
    asg[j] = (uint8_t)q;
    local = __dadd_rn(local, __dmul_rn((double)wv[j], dcost((double)xs[j], sh.cen[q])));
  }
  return block_sum(local, sh);
}

__global__ void __launch_bounds__(kThreads) k_kmeans_rows(KmParams P) {
  extern __shared__ __align__(16) uint8_t dsmem[];
  __shared__ Shared sh;
  __shared__ int64_t vkeys[2 * kMaxK], vvals[2 * kMaxK];
  const int64_t n = P.n;
  const int k = P.k;
  uint8_t* base = P.use_smem ? dsmem : P.gscratch + blockIdx.x * P.scratch_stride;
  float* xs = reinterpret_cast<float*>(base);
  float* wv = xs + n;
  // d2 (init) and asg (Lloyd) share the tail region: 2n doubles.
  size_t off = ((sizeof(float) * 2 * n) + 15) & ~size_t(15);
  double* d2 = reinterpret_cast<double*>(base + off);
  uint8_t* asg = reinterpret_cast<uint8_t*>(d2);
  const int64_t C = (n + kThreads - 1) / kThreads;
  const int64_t b = threadIdx.x * C, e = min(n, b + C);

  while (true) {
    if (threadIdx.x == 0) sh.row = atomicAdd(P.row_counter, 1);
    __syncthreads();
    const int64_t row = sh.row;
    if (row >= P.rows) break;
    const float* xo = P.ws + row * n;
    const float* wo = P.sw + row * n;
    int bad = 0;
    for (int64_t j = b; j < e; ++j) {
      xs[j] = P.skeys[row * n + j];
      float w = wo[P.svals[row * n + j]];
      wv[j] = w;
      bad |= !(w >= 0.0f) || !isfinite(w);
    }
    if (__syncthreads_or(bad)) {  // KmProblem::validate (learner.cpp:10-23)
      if (threadIdx.x == 0) dev_fail(P.err, ANYQ_ERR_STATS);
      continue;
    }
    if (threadIdx.x == 0) sh.rng = Rng::for_row(P.seed, P.row_offset + row);
    double best = INFINITY;
    for (int r = 0; r < P.restarts; ++r) {
      __syncthreads();
      switch (P.init) {
        case ANYQ_INIT_KMPP: init_kmeanspp(P, xo, wo, xs, d2, sh, k); break;
        case ANYQ_INIT_RANDOM: init_random(P, xo, xs, sh, k, vkeys, vvals); break;
        case ANYQ_INIT_GRID:
          for (int q = threadIdx.x; q < k; q += kThreads) sh.cen[q] = (double)(-(k / 2) + q);
          break;
        default: {
          const float nf4[16] = {-1.0f, -0.6961928009986877f, -0.5250730514526367f,
                                 -0.39491748809814453f, -0.28444138169288635f,
                                 -0.18477343022823334f, -0.09105003625154495f, 0.0f,
                                 0.07958029955625534f, 0.16093020141124725f, 0.24611230194568634f,
                                 0.33791524171829224f, 0.44070982933044434f, 0.5626170039176941f,
                                 0.7229568362236023f, 1.0f};
          for (int q = threadIdx.x; q < k; q += kThreads) sh.cen[q] = (double)nf4[q & 15];
        }
      }
      __syncthreads();
      double loss = lloyd(P, xs, wv, asg, sh, k);
      if (loss < best) {
        best = loss;
        for (int q = threadIdx.x; q < k; q += kThreads) sh.best_cen[q] = sh.cen[q];
      }
      __syncthreads();
    }
    // best centroids -> sorted LUT + rank-remapped codes (learner.cpp:343-369)
    for (int q = threadIdx.x; q < k; q += kThreads) sh.cen[q] = sh.best_cen[q];
    sort_centroids(sh, k);
    for (int r = threadIdx.x; r < k; r += kThreads) P.luts[row * k + r] = (float)sh.sv[r];
    for (int64_t j = b; j < e; ++j) {
      int q = nearest((double)xs[j], sh, k);
      P.codes[row * n + P.svals[row * n + j]] = (uint8_t)sh.rank_of[q];
    }
    __syncthreads();
  }
}

__global__ void k_fill_offsets(int* off, int64_t rows, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i <= rows) off[i] = (int)(i * n);
}

__global__ void k_iota_rows(int* v, int64_t rows, int64_t n) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < rows * n) v[e] = (int)(e % n);
}

}  // namespace

void launch_kmeans(const float* ws, const float* sw, int64_t rows, int64_t cols,
                   const anyq_config& cfg, int64_t row_offset, float* luts, uint8_t* codes,
                   int* err, cudaStream_t s) {
  if (rows * cols >= (int64_t(1) << 31)) fail(ANYQ_ERR_SHAPE, "quantize batch too large; split rows");
  const int64_t total = rows * cols;
  DevBuf<float> skeys(total);
  DevBuf<int> idx(total), svals(total), offs(rows + 1), counter(1);
  k_fill_offsets<<<(unsigned)((rows + 256) / 256), 256, 0, s>>>(offs.p, rows, cols);
  ANYQ_LAUNCHED();
  k_iota_rows<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(idx.p, rows, cols);
  ANYQ_LAUNCHED();
  size_t temp_bytes = 0;
  ANYQ_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, temp_bytes, ws, skeys.p, idx.p,
                                                      svals.p, (int)total, (int)rows, offs.p,
                                                      offs.p + 1, s));
  DevBuf<uint8_t> temp(temp_bytes);
  ANYQ_CUDA(cub::DeviceSegmentedSort::StableSortPairs(temp.p, temp_bytes, ws, skeys.p, idx.p,
                                                      svals.p, (int)total, (int)rows, offs.p,
                                                      offs.p + 1, s));
  note_launch(2);
  ANYQ_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(int), s));

  KmParams P;
  P.ws = ws;
  P.sw = sw;
  P.skeys = skeys.p;
  P.svals = svals.p;
  P.rows = rows;
  P.n = cols;
  P.k = 1 << cfg.bits;
  P.init = cfg.init;
  P.max_iters = cfg.max_iters;
  P.restarts = cfg.restarts;
  P.check_inv = cfg.check_invariants;
  P.rel_tol = cfg.rel_tol;
  P.seed = cfg.seed;
  P.row_offset = row_offset;
  P.luts = luts;
  P.codes = codes;
  P.err = err;
  P.row_counter = counter.p;

  // per-row scratch: xs, wv (fp32) + 2n doubles (d2/mass during init, asg after)
  size_t need = (((sizeof(float) * 2 * cols) + 15) & ~size_t(15)) + sizeof(double) * 2 * cols;
  int dev = 0;
  ANYQ_CUDA(cudaGetDevice(&dev));
  int sms = 148, max_optin = 0;
  ANYQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  ANYQ_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  size_t static_smem = sizeof(Shared) + 2 * 2 * kMaxK * sizeof(int64_t);
  DevBuf<uint8_t> gscratch;
  int blocks;
  if (need + static_smem <= (size_t)max_optin) {
    P.use_smem = 1;
    P.gscratch = nullptr;
    P.scratch_stride = 0;
    ANYQ_CUDA(cudaFuncSetAttribute(k_kmeans_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)need));
    int per_sm = 0;
    ANYQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kmeans_rows, kThreads, need));
    blocks = (int)std::min<int64_t>(rows, (int64_t)sms * std::max(1, per_sm));
    k_kmeans_rows<<<blocks, kThreads, need, s>>>(P);
  } else {
    int per_sm = 0;
    ANYQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kmeans_rows, kThreads, 0));
    blocks = (int)std::min<int64_t>(rows, (int64_t)sms * std::max(1, per_sm));
    P.use_smem = 0;
    P.scratch_stride = (need + 255) & ~size_t(255);
    gscratch.alloc(P.scratch_stride * blocks);
    P.gscratch = gscratch.p;
    k_kmeans_rows<<<blocks, kThreads, 0, s>>>(P);
  }
  ANYQ_LAUNCHED();
  ANYQ_CUDA(cudaStreamSynchronize(s));  // scratch buffers are freed on return
}

}  // namespace anyq_b200
