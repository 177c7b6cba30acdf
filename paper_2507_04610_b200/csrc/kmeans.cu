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
#include <cstdio>
#include <cstdlib>

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
  const int* row_list;  // if set: process rows row_list[0 .. *row_list_n)
  const int* row_list_n;
  // Problem mode (the per-row learner API, learner.hpp:52-68): caller RNG
  // state per row, raw k-means results, every double reduction in the
  // reference's sample-index order (sequential), so results are bit-identical
  // by construction. mode: 0 = LUT + codes (quantize), 1 = weighted_kmeans,
  // 2 = kmeans_pp_init only.
  int mode;
  int exact;
  const uint64_t* rng_key;  // [rows] or null (rng_for_row(seed, row_offset + row))
  uint64_t* rng_ctr;        // [rows] in/out counters (with rng_key)
  double* out_cen;          // [rows][k] centroids in the learner's order
  uint8_t* out_asg;         // [rows][n] assignments, original sample order
  double* out_loss;         // [rows]
  int* out_iters;           // [rows]
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
  int iters;
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
  const double r = sh.dbl_bcast;
  __syncthreads();  // the slot is rewritten by the next broadcast
  return r;
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
  const long long r = sh.ll_bcast;
  __syncthreads();  // the slot is rewritten by the next broadcast
  return r;
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

// Exact mode: sum of the positive masses in sample-index order (thread 0,
// broadcast), as the reference's sequential `total += mass[i]` (mass >= 0).
__device__ double seq_sum_pos(const double* mass, int64_t n, Shared& sh) {
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int64_t i = 0; i < n; ++i)
      if (mass[i] > 0.0) t = __dadd_rn(t, mass[i]);
    sh.dbl_bcast = t;
  }
  __syncthreads();
  const double r = sh.dbl_bcast;
  __syncthreads();
  return r;
}

// Exact mode: sample_index (learner.cpp:64-75) sequentially in thread 0.
__device__ int64_t seq_sample_index(const double* mass, int64_t n, double r_unit, Shared& sh,
                                    double* total_out) {
  __syncthreads();
  if (threadIdx.x == 0) {
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total = __dadd_rn(total, mass[i]);
    const double r = __dmul_rn(r_unit, total);
    double acc = 0.0;
    long long pick = -1, last = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (mass[i] <= 0.0) continue;
      acc = __dadd_rn(acc, mass[i]);
      last = i;
      if (r < acc) {
        pick = i;
        break;
      }
    }
    sh.ll_bcast = pick >= 0 ? pick : last;
    sh.dbl_bcast = total;
  }
  __syncthreads();
  const long long pick = sh.ll_bcast;
  *total_out = sh.dbl_bcast;
  __syncthreads();
  return pick;
}

// Exact mode: sum_i w_i (x_i - c_{a_i})^2 in sample-index order (total_cost,
// learner.cpp:198-204); asg_o holds original-order assignments.
__device__ double seq_loss(const float* xo, const float* wo, const uint8_t* asg_o, int64_t n,
                           Shared& sh) {
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int64_t i = 0; i < n; ++i)
      l = __dadd_rn(l, __dmul_rn((double)wo[i], dcost((double)xo[i], sh.cen[asg_o[i]])));
    sh.dbl_bcast = l;
  }
  __syncthreads();
  const double r = sh.dbl_bcast;
  __syncthreads();
  return r;
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
  int64_t pick = P.exact ? seq_sample_index(d2, n, u, sh, &total) : sample_index(d2, n, C, u, sh, &total);
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
    double tot = P.exact ? seq_sum_pos(mass, n, sh) : block_sum(local, sh);
    if (tot > 0.0) {
      if (threadIdx.x == 0) sh.dbl_bcast = sh.rng.next_double();
      __syncthreads();
      u = sh.dbl_bcast;
      pick = P.exact ? seq_sample_index(mass, n, u, sh, &total) : sample_index(mass, n, C, u, sh, &total);
      if (threadIdx.x == 0) sh.cen[sh.ncen++] = (double)xo[pick];
      __syncthreads();
      continue;
    }
    for (int64_t i = b; i < e; ++i) mass[i] = d2[i];
    __syncthreads();
    local = 0.0;
    for (int64_t i = b; i < e; ++i)
      if (mass[i] > 0.0) local = __dadd_rn(local, mass[i]);
    tot = P.exact ? seq_sum_pos(mass, n, sh) : block_sum(local, sh);
    if (tot > 0.0) {
      if (threadIdx.x == 0) sh.dbl_bcast = sh.rng.next_double();
      __syncthreads();
      u = sh.dbl_bcast;
      pick = P.exact ? seq_sample_index(mass, n, u, sh, &total) : sample_index(mass, n, C, u, sh, &total);
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

// One Lloyd run (learner.cpp:207-312) on the sorted row. Returns the loss;
// sh.iters = iterations run. Exact mode (P.exact) forms the M-step sums and
// the losses in sample-index order from the original-order row (xo, wo).
__device__ double lloyd(const KmParams& P, const float* xs, const float* wv, uint8_t* asg,
                        Shared& sh, int k, const float* xo, const float* wo, uint8_t* asg_o) {
  const int64_t n = P.n;
  const int64_t C = (n + kThreads - 1) / kThreads;
  const int64_t b = threadIdx.x * C, e = min(n, b + C);
  const int* sv = P.svals + sh.row * n;
  auto original_order = [&]() {
    __syncthreads();
    for (int64_t j = b; j < e; ++j) asg_o[sv[j]] = asg[j];
    __syncthreads();
  };
  for (int64_t j = b; j < e; ++j) asg[j] = 0;
  double prev = INFINITY;
  if (threadIdx.x == 0) sh.iters = P.max_iters;
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
    if (P.exact) {
      // M-step in sample-index order (learner.cpp:245-253), one thread per cluster
      original_order();
      for (int q = threadIdx.x; q < k; q += kThreads) {
        double swx = 0, sw = 0, sx = 0;
        int c = 0;
        for (int64_t i = 0; i < n; ++i)
          if (asg_o[i] == q) {
            const double w = (double)wo[i], x = (double)xo[i];
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
    if (P.exact) {
      // sums formed above
    } else if (mono) {
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
    double loss_m;
    if (P.exact) {
      original_order();
      loss_m = seq_loss(xo, wo, asg_o, n, sh);
    } else {
      double local = 0.0;
      for (int64_t j = b; j < e; ++j)
        local = __dadd_rn(local, __dmul_rn((double)wv[j], dcost((double)xs[j], sh.cen[asg[j]])));
      loss_m = block_sum(local, sh);
    }
    int any_changed = __syncthreads_or(changed) || repairs > 0;
    bool stable = !any_changed && iter > 0;
    bool tol = isfinite(prev) && __dsub_rn(prev, loss_m) <= __dmul_rn((double)P.rel_tol, prev);
    prev = loss_m;
    if (stable || tol || loss_m == 0.0) {
      if (threadIdx.x == 0) sh.iters = iter + 1;
      break;
    }
  }
  // final reassignment and loss
  sort_centroids(sh, k);
  double local = 0.0;
  for (int64_t j = b; j < e; ++j) {
    int q = nearest((double)xs[j], sh, k);
    asg[j] = (uint8_t)q;
    local = __dadd_rn(local, __dmul_rn((double)wv[j], dcost((double)xs[j], sh.cen[q])));
  }
  if (P.exact) {
    original_order();
    return seq_loss(xo, wo, asg_o, n, sh);
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
    if (threadIdx.x == 0) {
      const int64_t i = atomicAdd(P.row_counter, 1);
      if (P.row_list) sh.row = i < *P.row_list_n ? P.row_list[i] : P.rows;
      else sh.row = i;
    }
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
    if (threadIdx.x == 0) {
      if (P.rng_key) {  // the caller's stream (learner API): key + counter
        sh.rng.key = P.rng_key[row];
        sh.rng.counter = P.rng_ctr[row];
      } else {
        sh.rng = Rng::for_row(P.seed, P.row_offset + row);
      }
    }
    if (P.mode == 2) {  // kmeans_pp_init only (learner.cpp:132-174)
      __syncthreads();
      init_kmeanspp(P, xo, wo, xs, d2, sh, k);
      for (int q = threadIdx.x; q < k; q += kThreads) P.out_cen[row * k + q] = sh.cen[q];
      if (threadIdx.x == 0) P.rng_ctr[row] = sh.rng.counter;
      __syncthreads();
      continue;
    }
    uint8_t* asg_o = asg + n;  // exact mode: original-order assignments
    double best = INFINITY;
    int best_iters = 0;
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
      double loss = lloyd(P, xs, wv, asg, sh, k, xo, wo, asg_o);
      if (loss < best) {
        best = loss;
        best_iters = sh.iters;
        for (int q = threadIdx.x; q < k; q += kThreads) sh.best_cen[q] = sh.cen[q];
      }
      __syncthreads();
    }
    if (P.mode == 1) {  // weighted_kmeans (learner.cpp:316-341): raw best run
      for (int q = threadIdx.x; q < k; q += kThreads) sh.cen[q] = sh.best_cen[q];
      sort_centroids(sh, k);
      for (int q = threadIdx.x; q < k; q += kThreads) P.out_cen[row * k + q] = sh.best_cen[q];
      // the best run's returned assignments are nearest(best centroids) (learner.cpp:302-305)
      for (int64_t j = b; j < e; ++j)
        P.out_asg[row * n + P.svals[row * n + j]] = (uint8_t)nearest((double)xs[j], sh, k);
      if (threadIdx.x == 0) {
        P.out_loss[row] = best;
        P.out_iters[row] = best_iters;
        P.rng_ctr[row] = sh.rng.counter;
      }
      __syncthreads();
      continue;
    }
    // best centroids -> sorted LUT + rank-remapped codes (learner.cpp:343-369)
    for (int q = threadIdx.x; q < k; q += kThreads) sh.cen[q] = sh.best_cen[q];
    sort_centroids(sh, k);
    for (int r = threadIdx.x; r < k; r += kThreads) P.luts[row * k + r] = (float)sh.sv[r];
    for (int64_t j = b; j < e; ++j) {
      int q = nearest((double)xs[j], sh, k);
      P.codes[row * n + P.svals[row * n + j]] = (uint8_t)sh.rank_of[q];
    }
    if (threadIdx.x == 0 && P.rng_ctr) {  // learn_row_lut (learner.cpp:343-369)
      P.out_loss[row] = best;
      P.rng_ctr[row] = sh.rng.counter;
    }
    __syncthreads();
  }
}

// ===========================================================================
// Warp-per-row Lloyd (k <= 16): one warp learns one row at a time, no block
// barriers. Same semantics as k_kmeans_rows (learner.cpp:132-369), with the
// E-step done as a search for the k-1 segment boundaries of the sorted row:
// for distinct centroid values the exact-rounded nearest rank is monotone in
// x (costs are monotone in |x - c| after rounding and a tie between the two
// bracketing centroids picks the same index across the whole tie zone), so
// seg[t] = first sorted position whose nearest rank is >= t is found by
// binary search with the reference predicate itself — O(k log n) per
// iteration instead of O(n k). Rows where two centroids come within 2^-40 of
// the data range (where a 3-way rounding tie could break monotonicity), k > 16
// or check_invariants go to k_kmeans_rows instead (bail list).
// The M-step and the loss scan each lane's contiguous chunk of the sorted
// row (stored lane-interleaved in shared memory: conflict free) and combine
// chunks in a fixed order; empty-cluster repairs, the changed test against
// the repaired assignment, convergence and restarts follow the reference.
// ===========================================================================
constexpr int kWK = 16;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxG = 8;
constexpr int kCmdDone = 0, kCmdRepair = 1, kCmdLoss = 2;  // w_lloyd's collective steps
// named barrier 1 over the row group: warp 0's command hand-off and the other
// warps' wait meet at this one instruction (one call site for both sides)
__device__ __noinline__ void km_bar1(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Per-row state of one row group (one CTA of G warps works one row at a time).
struct WarpKm {
  double cen[kWK], best_cen[kWK], sv[kWK];
  double swx[kWK], sw[kWK], sx[kWK];
  int so[kWK], rank_of[kWK], cnt[kWK];
  int seg[kWK + 1], pseg[kWK + 1], pso[kWK], prank[kWK];
  int exc_pos[kWK], exc_q[kWK], pexc_pos[kWK], pexc_q[kWK];
  int nexc, pnexc;
  long long vkeys[2 * kWK], vvals[2 * kWK];
  Rng rng;
  int ncen;
  double closs[kWK];      // per-cluster loss under the updated centroid
  unsigned empties;       // clusters to repair (command kCmdRepair)
  int cmd;                // warp 0 -> the row group's other warps
  int bailf;              // the E-step found near-duplicate centroids
  double redd[kMaxG];  // cross-warp reduction slots
  long long redl[kMaxG], redl2[kMaxG];
  int redi[kMaxG];
  double bcd;  // broadcasts from thread 0
  int bci;
  int chg;     // changed flag of the current iteration
};

struct WkParams {
  const float* ws;     // rows x n, original order
  const float* sw;     // rows x n, original order
  const float* skeys;  // rows x n, sorted values
  const int* svals;    // rows x n, original index of each sorted position
  int64_t rows;
  int n, C, k, init, max_iters, restarts;
  float rel_tol;
  uint64_t seed;
  int64_t row_offset;
  float* luts;
  uint8_t* codes;
  int* err;
  int* row_counter;
  double* d2scr;        // [CTAs][C * T] k-means++ D^2, thread-interleaved
  int* bail_rows;       // rows handed to k_kmeans_rows
  int* bail_n;
  uint32_t state_bytes;  // dynamic smem: WarpKm + fpart/lpart
  long long* dbg;        // debug counters [8] (ANYQ_KM_DEBUG), or null
};

// The row group: thread t of T = 32*G owns the contiguous chunk [t*C, t*C + C)
// of the row; element j of chunk t lives at j*(T+1) + t in shared memory (bank
// (j + t) % 32: conflict free for a warp walking its chunks in step and for
// coalesced whole-row loads; linear in j).
struct Grp {
  int t, lane, warp, G, T;
};

struct WRow {
  const float* xs;  // sorted samples (Lloyd) / original order (k-means++)
  const float* wv;  // their weights
  int n, C, T, lo, hi, nch;
  __device__ __forceinline__ int idx(int t, int j) const { return j * (T + 1) + t; }
  __device__ __forceinline__ float x_at(int p) const {
    const int t = p / C;
    return xs[idx(t, p - t * C)];
  }
};

// Deterministic group reductions (fixed shuffle tree, then warp order).
__device__ __forceinline__ double g_sum(double v, WarpKm& S, const Grp& g) {
  for (int off = 16; off; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(kFull, v, off));
  if (g.G == 1) return __shfl_sync(kFull, v, 0);
  if (g.lane == 0) S.redd[g.warp] = v;
  __syncthreads();
  double s = S.redd[0];
  for (int w = 1; w < g.G; ++w) s = __dadd_rn(s, S.redd[w]);
  __syncthreads();
  return s;
}
// g_scan_excl, and the next RNG draw (thread 0, broadcast) when the total is
// positive or `always`: the draw rides on the scan's barriers
__device__ __forceinline__ double g_scan_excl_draw(double v, WarpKm& S, const Grp& g, double* total,
                                                   double* u, bool always) {
  double incl = v;
  for (int off = 1; off < 32; off <<= 1) {
    const double o = __shfl_up_sync(kFull, incl, off);
    if (g.lane >= off) incl = __dadd_rn(o, incl);
  }
  const double wtot = __shfl_sync(kFull, incl, 31);
  double ex = __shfl_up_sync(kFull, incl, 1);
  if (g.lane == 0) ex = 0.0;
  if (g.G == 1) {
    double d = 0.0;
    if (g.lane == 0 && (always || wtot > 0.0)) d = S.rng.next_double();
    *u = __shfl_sync(kFull, d, 0);
    *total = wtot;
    return ex;
  }
  if (g.lane == 0) S.redd[g.warp] = wtot;
  __syncthreads();
  double base = 0.0, tot = S.redd[0];
  for (int w = 1; w < g.G; ++w) tot = __dadd_rn(tot, S.redd[w]);
  if (g.warp > 0) {
    base = S.redd[0];
    for (int w = 1; w < g.warp; ++w) base = __dadd_rn(base, S.redd[w]);
  }
  if (g.t == 0 && (always || tot > 0.0)) S.bcd = S.rng.next_double();
  __syncthreads();
  *total = tot;
  *u = S.bcd;
  return g.warp > 0 ? __dadd_rn(base, ex) : ex;
}
// min of a and max of b over the group in one barrier round
__device__ __forceinline__ void g_minmax_ll(long long a, long long b, WarpKm& S, const Grp& g,
                                            long long* mn, long long* mx) {
  for (int off = 16; off; off >>= 1) {
    a = min(a, __shfl_xor_sync(kFull, a, off));
    b = max(b, __shfl_xor_sync(kFull, b, off));
  }
  if (g.G == 1) {
    *mn = a;
    *mx = b;
    return;
  }
  if (g.lane == 0) {
    S.redl[g.warp] = a;
    S.redl2[g.warp] = b;
  }
  __syncthreads();
  long long m = S.redl[0], x = S.redl2[0];
  for (int w = 1; w < g.G; ++w) {
    m = min(m, S.redl[w]);
    x = max(x, S.redl2[w]);
  }
  __syncthreads();
  *mn = m;
  *mx = x;
}

__device__ __forceinline__ void w_sort(WarpKm& S, int k, const Grp& g) {
  __syncthreads();
  if (g.t < k) {
    const double v = S.cen[g.t];
    int r = 0;
#pragma unroll
    for (int p = 0; p < kWK; ++p) {  // independent loads (k <= kWK)
      if (p < k) {
        const double u = S.cen[p];
        r += (u < v) || (u == v && p < g.t);
      }
    }
    S.rank_of[g.t] = r;
    S.sv[r] = v;
    S.so[r] = g.t;
  }
  __syncthreads();
}

// Exact reference nearest centroid (ties to the smallest original index).
__device__ __forceinline__ int w_nearest(double x, const WarpKm& S, int k) {
  int lo = 0, hi = k;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S.sv[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  const int p = lo;
  const double cl = p > 0 ? dcost(x, S.sv[p - 1]) : INFINITY;
  const double cr = p < k ? dcost(x, S.sv[p]) : INFINITY;
  const double mc = cl < cr ? cl : cr;
  int best = 1 << 30;
  for (int r = p - 1; r >= 0; --r) {
    const double c = (r == p - 1) ? cl : dcost(x, S.sv[r]);
    if (!(c == mc)) break;
    best = min(best, S.so[r]);
  }
  for (int r = p; r < k; ++r) {
    const double c = (r == p) ? cr : dcost(x, S.sv[r]);
    if (!(c == mc)) break;
    best = min(best, S.so[r]);
  }
  return best;
}

// Whole-row load into the chunked layout (coalesced global reads).
template <typename F>
__device__ __forceinline__ void w_load_row(const WRow& R, const Grp& g, F&& put) {
  int t = g.t / R.C, j = g.t - (g.t / R.C) * R.C;
  for (int p = g.t; p < R.n; p += R.T) {
    put(p, R.idx(t, j));
    j += R.T;
    while (j >= R.C) {
      j -= R.C;
      ++t;
    }
  }
}

// Whole-row load xs[.] = xa[p], wv[.] = wa[perm ? perm[p] : p] in batches of
// 8 per thread: all global loads of a batch (the permutation first, then the
// gathers) are issued before any shared-memory store. One load-store pair at
// a time serialised 2 x 32 global round trips per thread and row.
__device__ __forceinline__ void w_load_row_batched(const WRow& R, const Grp& g, float* xs, float* wv,
                                                   const float* __restrict__ xa,
                                                   const float* __restrict__ wa,
                                                   const int* __restrict__ perm) {
  constexpr int B = 8;
  int t = g.t / R.C, j = g.t - (g.t / R.C) * R.C;
  for (int p0 = g.t; p0 < R.n; p0 += B * R.T) {
    int si[B], wi[B];
    float xv[B], wq[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      si[u] = R.idx(t, j);
      j += R.T;
      while (j >= R.C) {
        j -= R.C;
        ++t;
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int p = p0 + u * R.T;
      wi[u] = p < R.n ? (perm ? __ldg(perm + p) : p) : 0;
      xv[u] = p < R.n ? __ldg(xa + p) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) wq[u] = p0 + u * R.T < R.n ? __ldg(wa + wi[u]) : 0.0f;
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (p0 + u * R.T < R.n) {
        xs[si[u]] = xv[u];
        wv[si[u]] = wq[u];
      }
  }
}

// label of sorted position p under segments seg/so
__device__ __forceinline__ int w_label_seg(const int* seg, const int* so, int k, int p) {
  int r = 0;
  while (r < k - 1 && seg[r + 1] <= p) ++r;
  return so[r];
}

// m-th distinct sorted sample value, cycling (pad_with_distinct); global sorted row
__device__ double w_distinct_value(const float* sk, int n, int64_t m) {
  int64_t nd = 0;
  for (int j = 0; j < n; ++j)
    if (j == 0 || !((double)sk[j] == (double)sk[j - 1])) ++nd;
  int64_t want = m % nd, seen = -1;
  for (int j = 0; j < n; ++j)
    if (j == 0 || !((double)sk[j] == (double)sk[j - 1]))
      if (++seen == want) return (double)sk[j];
  return (double)sk[0];
}

// Cumulative-mass sampling (learner.cpp:64-75) over this thread's chunk of
// ORIGINAL indices: first hit over the group, else the last positive index.
// Thread t's running mass goes from excl (the group scan) up by its chunk's
// masses (part = their sum); only a chunk whose range can hold r is walked:
// below it (r < excl) the hit is the chunk's first positive sample, above it
// (r beyond excl + part with a margin far wider than the walk's rounding)
// there is none. The last positive index is only looked for when no chunk hit.
template <int kMode>  // 0: mass = w, 1: mass = w * d2, 2: mass = d2
__device__ __forceinline__ long long w_sample(const WRow& R, const double* d2, WarpKm& S,
                                              const Grp& g, double excl, double part, double r) {
  long long cand = LLONG_MAX;
  const int cnt = R.hi - R.lo;
  auto mass = [&](int j) {
    if (kMode == 0) return (double)R.wv[R.idx(g.t, j)];
    if (kMode == 1) return __dmul_rn((double)R.wv[R.idx(g.t, j)], d2[j * R.T + g.t]);
    return d2[j * R.T + g.t];
  };
  if (r < excl) {
    for (int j = 0; j < cnt; ++j)
      if (mass(j) > 0.0) {
        cand = R.lo + j;
        break;
      }
  } else if (!(r > __dmul_rn(__dadd_rn(excl, part), 1.0 + 0x1p-30))) {
    double acc = excl;
    for (int j0 = 0; j0 < cnt && cand == LLONG_MAX; j0 += 8) {
      double mv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mv[u] = (j0 + u < cnt) ? mass(j0 + u) : 0.0;  // loads first
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (cand != LLONG_MAX || !(mv[u] > 0.0)) continue;
        acc = __dadd_rn(acc, mv[u]);
        if (r < acc) cand = R.lo + j0 + u;
      }
    }
  }
  long long c, lp;
  g_minmax_ll(cand, -1, S, g, &c, &lp);
  if (c != LLONG_MAX) return c;
  long long lastpos = -1;  // no hit anywhere: the last positive index of the row
  for (int j = cnt - 1; j >= 0; --j)
    if (mass(j) > 0.0) {
      lastpos = R.lo + j;
      break;
    }
  g_minmax_ll(LLONG_MAX, lastpos, S, g, &c, &lp);
  return lp >= 0 ? lp : 0;
}

// k-means++ (learner.cpp:132-174): R holds the row in ORIGINAL order; D^2 in
// global scratch (thread-interleaved, coalesced).
__device__ void w_init_kmpp(const WRow& R, const float* sk, double* d2, WarpKm& S, int k,
                            const Grp& g) {
  const int cnt = R.hi - R.lo;
  double part = 0.0, total;
  for (int j = 0; j < cnt; ++j) {
    const double m = (double)R.wv[R.idx(g.t, j)];
    if (m > 0.0) part = __dadd_rn(part, m);
  }
  double u;
  double excl = g_scan_excl_draw(part, S, g, &total, &u, true);
  long long pick = w_sample<0>(R, d2, S, g, excl, part, __dmul_rn(u, total));
  for (int j = 0; j < cnt; ++j) d2[j * R.T + g.t] = INFINITY;
  if (g.t == 0) {
    S.cen[0] = (double)R.x_at((int)pick);
    S.ncen = 1;
  }
  __syncthreads();
  while (S.ncen < k) {
    const double c = S.cen[S.ncen - 1];
    part = 0.0;
    for (int j0 = 0; j0 < cnt; j0 += 8) {
      double dv[8];
#pragma unroll
      for (int uu = 0; uu < 8; ++uu) dv[uu] = d2[min(j0 + uu, cnt - 1) * R.T + g.t];  // loads first
#pragma unroll
      for (int uu = 0; uu < 8; ++uu) {
        if (j0 + uu >= cnt) break;
        const int si = R.idx(g.t, j0 + uu);
        const double pc = dcost((double)R.xs[si], c);
        const double d = (pc < dv[uu]) ? pc : dv[uu];
        d2[(j0 + uu) * R.T + g.t] = d;
        const double m = __dmul_rn((double)R.wv[si], d);
        if (m > 0.0) part = __dadd_rn(part, m);
      }
    }
    excl = g_scan_excl_draw(part, S, g, &total, &u, false);  // draws iff total > 0
    if (total > 0.0) {
      pick = w_sample<1>(R, d2, S, g, excl, part, __dmul_rn(u, total));
      if (g.t == 0) S.cen[S.ncen++] = (double)R.x_at((int)pick);
      __syncthreads();
      continue;
    }
    part = 0.0;
    for (int j = 0; j < cnt; ++j) {
      const double m = d2[j * R.T + g.t];
      if (m > 0.0) part = __dadd_rn(part, m);
    }
    excl = g_scan_excl_draw(part, S, g, &total, &u, false);  // draws iff total > 0
    if (total > 0.0) {
      pick = w_sample<2>(R, d2, S, g, excl, part, __dmul_rn(u, total));
      if (g.t == 0) S.cen[S.ncen++] = (double)R.x_at((int)pick);
      __syncthreads();
      continue;
    }
    if (g.t == 0) {
      int64_t cursor = 0;
      while (S.ncen < k) S.cen[S.ncen++] = w_distinct_value(sk, R.n, cursor++);
    }
    __syncthreads();
  }
}

// random_init (learner.cpp:86-103); R holds the row in ORIGINAL order.
__device__ void w_init_random(const WRow& R, const float* sk, WarpKm& S, int k, const Grp& g) {
  if (g.t == 0) {
    const int64_t n = R.n;
    if ((int64_t)k >= n) {
      int c = 0;
      for (int64_t j = 0; j < n; ++j) S.cen[c++] = (double)sk[j];
      int64_t cursor = 0;
      while (c < k) S.cen[c++] = w_distinct_value(sk, R.n, cursor++);
    } else {
      int used = 0;
      auto get = [&](long long pos) -> long long {
        for (int i = 0; i < used; ++i)
          if (S.vkeys[i] == pos) return S.vvals[i];
        return pos;
      };
      auto set = [&](long long pos, long long v) {
        for (int i = 0; i < used; ++i)
          if (S.vkeys[i] == pos) {
            S.vvals[i] = v;
            return;
          }
        S.vkeys[used] = pos;
        S.vvals[used] = v;
        ++used;
      };
      for (int t = 0; t < k; ++t) {
        const long long pick = t + S.rng.next_index(n - t);
        const long long vt = get(t), vp = get(pick);
        set(t, vp);
        set(pick, vt);
        S.cen[t] = (double)R.x_at((int)vp);
      }
    }
  }
  __syncthreads();
}

#define KM_PHASE(slot)                                                                  \
  do {                                                                                  \
    if (P.dbg && g.t == 0) {                                                            \
      const long long tt = clock64();                                                   \
      atomicAdd((unsigned long long*)&P.dbg[slot], (unsigned long long)(tt - tph));     \
      tph = tt;                                                                         \
    }                                                                                   \
  } while (0)

// One Lloyd run (learner.cpp:207-312). Returns the final loss (or 0 when
// not needed); *bail = 1 when the row must go to the CTA kernel.
//
// Iteration i: M-step sums of the E-step segments seg_i -> centroid update ->
// empty-cluster repair -> changed_i -> loss_i -> stop test. loss_i needs the
// updated centroids and the repaired labels of iteration i, so it shares one
// pass over the row with the M-step sums of iteration i+1: the E-step of
// iteration i+1 (a pure function of the updated centroids) runs first,
// speculatively; when the stop test then fires, its results are simply not
// used. Rows with repairs in the iteration take separate passes.
__device__ double w_lloyd(const WkParams& P, const WRow& R, WarpKm& S, double* CT,
                          const int* svals_row, const Grp& g, bool need_loss, int* bail) {
  const int n = R.n, C = R.C, k = P.k, lo = R.lo, hi = R.hi;
  const double xmax = fmax(fabs((double)R.x_at(0)), fabs((double)R.x_at(n - 1)));
  // ---- E-step: segment boundaries of the sorted row by the exact predicate
  auto estep = [&]() -> bool {
    long long tph = clock64();
    // rank the centroids (lanes < k; ties to the smaller index) on order-
    // preserving integer keys of the (finite) values, -0 folded onto +0 so that
    // key equality is double equality: integer compares and shuffles instead
    // of FP64 compares on shared-memory loads
    __syncwarp();
    {
      const double v = g.lane < k ? S.cen[g.lane] : 0.0;
      long long key = __double_as_longlong(__dadd_rn(v, 0.0));
      key ^= (key >> 63) & 0x7fffffffffffffffLL;
      int r = 0;
#pragma unroll
      for (int p = 0; p < kWK; ++p) {
        const long long kp = __shfl_sync(kFull, key, p);
        r += p < k && (kp < key || (kp == key && p < g.lane));
      }
      if (g.lane < k) {
        S.rank_of[g.lane] = r;
        S.sv[r] = v;
        S.so[r] = g.lane;
      }
    }
    __syncwarp();
    KM_PHASE(8);
    {
      double svr[kWK];
#pragma unroll
      for (int r = 0; r < kWK; ++r) svr[r] = r < k ? S.sv[r] : 0.0;  // independent loads
      double cmax = 0.0;
      bool near_dup = false;
#pragma unroll
      for (int r = 0; r < kWK; ++r) cmax = fmax(cmax, fabs(svr[r]));
      const double thresh = ldexp(xmax + cmax, -40);
#pragma unroll
      for (int r = 0; r + 1 < kWK; ++r) {
        if (r + 1 < k) {
          const double gap = __dsub_rn(svr[r + 1], svr[r]);
          near_dup |= (gap > 0.0 && gap < thresh) || !(gap >= 0.0);
        }
      }
      if (near_dup) {  // uniform: every lane sees the same centroids
        if (g.lane == 0) S.bailf = 1;
        __syncwarp();
        return false;
      }
    }
    if (g.t >= 1 && g.t < k) {
      // seg[t] = first sorted position whose nearest rank is >= t
      const int t = g.t;
      auto rank_at = [&](int p) { return S.rank_of[w_nearest((double)R.x_at(p), S, k)]; };
      int a = 0, b = n;
      bool done = false;
      if (S.sv[t - 1] < S.sv[t]) {
        // distinct neighbours: the switch sits at the midpoint up to rounding;
        // locate it by value (chunk starts, then inside the chunk), then settle
        // it with the exact predicate
        const double mid = 0.5 * S.sv[t - 1] + 0.5 * S.sv[t];
        // float x < mid  <=>  x < (the smallest float >= mid): float compares
        const float midf = __double2float_ru(mid);
        int la = 0, lb = R.nch;
        while (la < lb) {
          const int m = (la + lb) >> 1;
          if (R.xs[R.idx(m, 0)] < midf) la = m + 1;
          else lb = m;
        }
        int p = 0;
        if (la > 0) {
          const int c0 = la - 1, cntc = min(C, n - c0 * C);
          int ja = 0, jb = cntc;
          while (ja < jb) {
            const int m = (ja + jb) >> 1;
            if (R.xs[R.idx(c0, m)] < midf) ja = m + 1;
            else jb = m;
          }
          p = c0 * C + ja;
        }
        // with no near-duplicate centroids only the bracketing pair can win,
        // so "nearest rank >= t" is the reference predicate on that pair alone
        // (fl((x - c)^2), ties to the smaller original index)
        const double clo = S.sv[t - 1], chi = S.sv[t];
        const bool hi_wins_ties = S.so[t] < S.so[t - 1];
        auto at_least_t = [&](int pp) {
          const double x = (double)R.x_at(pp);
          const double dl = dcost(x, clo), dh = dcost(x, chi);
          return dh < dl || (dh == dl && hi_wins_ties);
        };
        int steps = 0;
        while (p > 0 && steps < 8 && at_least_t(p - 1)) --p, ++steps;
        while (p < n && steps < 8 && !at_least_t(p)) ++p, ++steps;
        if (steps < 8) {
          a = p;
          done = true;
        }
      }
      if (!done) {
        while (a < b) {
          const int mid = (a + b) >> 1;
          if (rank_at(mid) >= t) b = mid;
          else a = mid + 1;
        }
      }
      S.seg[t] = a;
    }
    if (g.t == 0) {
      S.seg[0] = 0;
      S.seg[k] = n;
    }
    __syncwarp();
    KM_PHASE(4);
    return true;
  };
  // ---- loss of the labels pseg/pso (+ the exceptions pexc) under the current
  // centroids (chunk order, then fixed tree)
  auto losspass = [&]() -> double {
    double lb[4] = {0.0, 0.0, 0.0, 0.0};
    const int nexc = S.pnexc;
    int r = 0;
    for (int p = lo; p < hi;) {
      while (r < k - 1 && S.pseg[r + 1] <= p) ++r;
      const int pend = min(hi, S.pseg[r + 1]);
      const double c = S.cen[S.pso[r]];
      int j = p - lo;
      const int je = pend - lo;
      if (nexc == 0) {
        for (; j + 8 <= je; j += 8) {
          float xv[8], wq[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            xv[u] = R.xs[R.idx(g.t, j + u)];
            wq[u] = R.wv[R.idx(g.t, j + u)];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            lb[u & 3] = __dadd_rn(lb[u & 3], __dmul_rn((double)wq[u], dcost((double)xv[u], c)));
        }
      }
      for (; j < je; ++j) {  // remainder / exception path into the first partial
        double cc = c;
        for (int e = 0; e < nexc; ++e)
          if (S.pexc_pos[e] == lo + j) cc = S.cen[S.pexc_q[e]];
        lb[0] = __dadd_rn(lb[0], __dmul_rn((double)R.wv[R.idx(g.t, j)],
                                           dcost((double)R.xs[R.idx(g.t, j)], cc)));
      }
      p = pend;
    }
    return __dadd_rn(__dadd_rn(lb[0], lb[1]), __dadd_rn(lb[2], lb[3]));
  };

  // ---- M-step sums without a pass over the row: a cluster is one segment
  // [a, z) of the sorted row, i.e. a head run in chunk a / C, whole chunks, and
  // a tail run in chunk (z - 1) / C. Whole-chunk sums (CT, once per row) and
  // the head / tail runs are formed exactly as the per-thread run sums of a
  // full pass (four interleaved partials per quantity from the run start,
  // folded), and combined in chunk order: the same values as summing every
  // run of the row each iteration, at O(C + T) per cluster instead of O(n).
  // w x x rides along for the cluster loss.
  auto runsum = [&](int t, int j0, int j1, double (&o)[4]) {
    double b0[4] = {0.0, 0.0, 0.0, 0.0}, b1[4] = {0.0, 0.0, 0.0, 0.0}, b2[4] = {0.0, 0.0, 0.0, 0.0};
    double b3[4] = {0.0, 0.0, 0.0, 0.0};
    int j = j0;
    for (; j + 8 <= j1; j += 8) {
      float xv[8], wq[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xv[u] = R.xs[R.idx(t, j + u)];
        wq[u] = R.wv[R.idx(t, j + u)];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double w = (double)wq[u], x = (double)xv[u];
        const double wx = __dmul_rn(w, x);
        b0[u & 3] = __dadd_rn(b0[u & 3], wx);
        b1[u & 3] = __dadd_rn(b1[u & 3], w);
        b2[u & 3] = __dadd_rn(b2[u & 3], x);
        b3[u & 3] = __fma_rn(wx, x, b3[u & 3]);
      }
    }
    for (; j < j1; ++j) {
      const double w = (double)R.wv[R.idx(t, j)], x = (double)R.xs[R.idx(t, j)];
      const double wx = __dmul_rn(w, x);
      b0[0] = __dadd_rn(b0[0], wx);
      b1[0] = __dadd_rn(b1[0], w);
      b2[0] = __dadd_rn(b2[0], x);
      b3[0] = __fma_rn(wx, x, b3[0]);
    }
    o[0] = __dadd_rn(__dadd_rn(b0[0], b0[1]), __dadd_rn(b0[2], b0[3]));
    o[1] = __dadd_rn(__dadd_rn(b1[0], b1[1]), __dadd_rn(b1[2], b1[3]));
    o[2] = __dadd_rn(__dadd_rn(b2[0], b2[1]), __dadd_rn(b2[2], b2[3]));
    o[3] = __dadd_rn(__dadd_rn(b3[0], b3[1]), __dadd_rn(b3[2], b3[3]));
  };
  {
    double o[4];
    runsum(g.t, 0, hi - lo, o);
#pragma unroll
    for (int i = 0; i < 4; ++i) CT[g.t * 4 + i] = o[i];
    if (g.t == 0) S.bailf = 0;
    __syncthreads();
  }
  // ---- collective steps (every warp of the row group): empty-cluster repair
  // and the loss over repaired labels; the other warps wait for warp 0's
  // command at named barrier 1 while warp 0 runs the iterations alone
  auto repair_all = [&]() {
    const unsigned empties = S.empties;
    for (unsigned em = empties; em; em &= em - 1) {
      const int q = __ffs(em) - 1;
      double worst = -1.0;
      int wp = -1;
      long long wo_i = LLONG_MAX;
      int r = 0;
      for (int p = lo, j = 0; p < hi; ++p, ++j) {
        while (r < k - 1 && S.seg[r + 1] <= p) ++r;
        int lab = S.so[r];
        for (int e = 0; e < S.nexc; ++e)
          if (S.exc_pos[e] == p) lab = S.exc_q[e];
        const double err = __dmul_rn((double)R.wv[R.idx(g.t, j)], dcost((double)R.xs[R.idx(g.t, j)], S.cen[lab]));
        if (err > worst) {
          worst = err;
          wp = p;
          wo_i = LLONG_MAX;
        } else if (err == worst) {
          if (wo_i == LLONG_MAX) wo_i = svals_row[wp];
          const long long oi = svals_row[p];
          if (oi < wo_i) {
            wp = p;
            wo_i = oi;
          }
        }
      }
      if (wp >= 0 && wo_i == LLONG_MAX) wo_i = svals_row[wp];
      // argmax (err), ties to the smallest original index: warp tree, then warps in order
      for (int off = 16; off; off >>= 1) {
        const double oe = __shfl_down_sync(kFull, worst, off);
        const long long oo = __shfl_down_sync(kFull, wo_i, off);
        const int op = __shfl_down_sync(kFull, wp, off);
        if (g.lane + off < 32 && (oe > worst || (oe == worst && oo < wo_i))) {
          worst = oe;
          wo_i = oo;
          wp = op;
        }
      }
      if (g.lane == 0) {
        S.redd[g.warp] = worst;
        S.redl[g.warp] = wo_i;
        S.redi[g.warp] = wp;
      }
      __syncthreads();
      if (g.t == 0) {
        double be = S.redd[0];
        long long bo = S.redl[0];
        int bp = S.redi[0];
        for (int w = 1; w < g.G; ++w)
          if (S.redd[w] > be || (S.redd[w] == be && S.redl[w] < bo)) {
            be = S.redd[w];
            bo = S.redl[w];
            bp = S.redi[w];
          }
        S.cen[q] = (double)R.x_at(bp);
        int e = 0;
        while (e < S.nexc && S.exc_pos[e] != bp) ++e;
        S.exc_pos[e] = bp;
        S.exc_q[e] = q;
        if (e == S.nexc) ++S.nexc;
      }
      __syncthreads();
    }
  };
  auto signal = [&](int cmd) {
    __syncwarp();
    if (g.lane == 0) S.cmd = cmd;
    __syncwarp();
    if (g.G > 1) km_bar1(g.T);
  };
  if (g.warp > 0) {
    while (true) {
      km_bar1(g.T);
      const int cmd = S.cmd;
      if (cmd == kCmdDone) break;
      if (cmd == kCmdRepair) repair_all();
      else (void)g_sum(losspass(), S, g);
    }
  } else {
  if (!estep()) {
    signal(kCmdDone);
  } else {
  double prev = INFINITY;
  for (int iter = 0; iter < P.max_iters; ++iter) {
    long long tph = clock64();
    // ---- M-step; each cluster's loss under its updated centroid (used by the
    // stop test when the iteration has no repairs)
    {
      // warp 0: lane q < k sums cluster q's head run and whole chunks, lane
      // 16 + q its tail run (k <= 16), added last as in chunk order
      if (g.warp == 0) {
        const int q = g.lane & 15;
        const bool tail_lane = g.lane >= 16;
        int a = 0, z = 0, t0 = 0, t1 = 0;
        double d[4] = {0.0, 0.0, 0.0, 0.0};
        // one run per lane (head or tail), one runsum call for the whole warp
        int rt = 0, rj0 = 0, rj1 = 0;
        if (q < k) {
          const int rq = S.rank_of[q];
          a = S.seg[rq];
          z = S.seg[rq + 1];
          t0 = a / C;
          t1 = z > a ? (z - 1) / C : t0;
          if (z > a) {
            if (t0 == t1) {
              if (!tail_lane) {
                rt = t0;
                rj0 = a - t0 * C;
                rj1 = z - t0 * C;
              }
            } else if (tail_lane) {
              rt = t1;
              rj1 = z - t1 * C;
            } else {
              rt = t0;
              rj0 = a - t0 * C;
              rj1 = min(C, n - t0 * C);
            }
          }
        }
        runsum(rt, rj0, rj1, d);
        if (!tail_lane && q < k && z > a) {
          for (int t = t0 + 1; t < t1; ++t) {
#pragma unroll
            for (int i = 0; i < 4; ++i) d[i] = __dadd_rn(d[i], CT[t * 4 + i]);
          }
        }
        double e[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) e[i] = __shfl_down_sync(kFull, d[i], 16);
        if (!tail_lane && q < k) {
          double cl = 0.0;
          S.cnt[q] = z - a;
          if (z > a) {
            if (t1 > t0) {
#pragma unroll
              for (int i = 0; i < 4; ++i) d[i] = __dadd_rn(d[i], e[i]);
            }
            S.swx[q] = d[0];
            S.sw[q] = d[1];
            S.sx[q] = d[2];
            const double c = d[1] > 0.0 ? __ddiv_rn(d[0], d[1]) : __ddiv_rn(d[2], (double)(z - a));
            S.cen[q] = c;
            const double xa = (double)R.x_at(a), xz = (double)R.x_at(z - 1);
            if (xa == xz) {
              cl = __dmul_rn(d[1], dcost(xa, c));  // exactly 0 iff every sample sits on c
            } else {
              // sum w (x - c)^2 = swxx - 2 c swx + c^2 sw; its rounding only reaches the
              // rel_tol test (relative error ~1e-12 against rel_tol 1e-6)
              cl = fmax(0.0, __dadd_rn(__dsub_rn(d[3], __dmul_rn(2.0 * c, d[0])),
                                       __dmul_rn(__dmul_rn(c, c), d[1])));
            }
          }
          S.closs[q] = cl;
        }
      }
      if (g.t == 0) S.nexc = 0;
      __syncwarp();
    }
    KM_PHASE(5);
    // ---- empty-cluster repair (learner.cpp:260-274), in cluster order: every warp
    const unsigned empties = __ballot_sync(kFull, g.lane < k && S.cnt[g.lane] == 0);
    if (empties) {
      if (g.lane == 0) S.empties = empties;
      signal(kCmdRepair);
      repair_all();
    }
    KM_PHASE(6);
    // ---- changed: this iteration's E-step labels vs the previous iteration's
    // repaired assignment (warp 0). Without repairs the labelings are equal iff
    // every cluster keeps the same sample range (one lane per cluster); after
    // repairs thread 0 walks the segment breakpoints (O(k^2)).
    if (g.warp == 0) {
      int changed = empties != 0;  // repairs count as changes
      if (iter > 0 && !changed) {
        if (S.pnexc == 0) {
          bool diff = false;
          if (g.lane < k) {
            const int rn = S.rank_of[g.lane], ro = S.prank[g.lane];
            const int an = S.seg[rn], bn = S.seg[rn + 1], ao = S.pseg[ro], bo = S.pseg[ro + 1];
            diff = !((an == bn && ao == bo) || (an == ao && bn == bo));
          }
          changed = __ballot_sync(kFull, diff) != 0;
        } else {
          if (g.lane == 0) {
            for (int e = 0; e < S.pnexc && !changed; ++e)
              if (w_label_seg(S.seg, S.so, k, S.pexc_pos[e]) != S.pexc_q[e]) changed = 1;
            int ro = 0, rn = 0, pos = 0;
            while (pos < n && !changed) {
              while (ro < k - 1 && S.pseg[ro + 1] <= pos) ++ro;
              while (rn < k - 1 && S.seg[rn + 1] <= pos) ++rn;
              const int end = min(S.pseg[ro + 1], S.seg[rn + 1]);
              if (S.pso[ro] != S.so[rn]) {
                if (end - pos > S.pnexc) {
                  changed = 1;
                } else {
                  for (int p = pos; p < end && !changed; ++p) {
                    bool isexc = false;
                    for (int e = 0; e < S.pnexc; ++e) isexc |= S.pexc_pos[e] == p;
                    if (!isexc) changed = 1;
                  }
                }
              }
              pos = end;
            }
          }
          changed = __shfl_sync(kFull, changed, 0);
        }
      }
      __syncwarp();
      // this iteration's (repaired) assignment becomes the previous one: the
      // labels of this iteration's loss and of the next changed test
      if (g.lane == 0) {
        S.chg = changed;
        S.pnexc = S.nexc;
        for (int e = 0; e < S.nexc; ++e) {
          S.pexc_pos[e] = S.exc_pos[e];
          S.pexc_q[e] = S.exc_q[e];
        }
        if (P.dbg) {
          atomicAdd((unsigned long long*)&P.dbg[2], 1ull);
          if (empties) atomicAdd((unsigned long long*)&P.dbg[3], (unsigned long long)__popc(empties));
        }
      }
      if (g.lane <= k) S.pseg[g.lane] = S.seg[g.lane];
      if (g.lane < k) {
        S.pso[g.lane] = S.so[g.lane];
        S.prank[g.lane] = S.rank_of[g.lane];
      }
    }
    __syncwarp();
    KM_PHASE(10);
    // ---- loss of this iteration: per-cluster sums when nothing was repaired,
    // else a pass over the repaired labels (pseg/pso + exceptions)
    double loss_m;
    if (S.pnexc == 0) {
      // fixed tree over the clusters (lane r holds the cluster of rank r)
      loss_m = g.lane < k ? S.closs[S.so[g.lane]] : 0.0;
      for (int off = 16; off; off >>= 1) loss_m = __dadd_rn(loss_m, __shfl_xor_sync(kFull, loss_m, off));
    } else {
      signal(kCmdLoss);
      loss_m = g_sum(losspass(), S, g);
    }
    KM_PHASE(7);
    const bool stable = !S.chg && iter > 0;
    const bool tol = isfinite(prev) && __dsub_rn(prev, loss_m) <= __dmul_rn((double)P.rel_tol, prev);
    prev = loss_m;
    if (stable || tol || loss_m == 0.0) break;
    if (iter + 1 < P.max_iters && !estep()) break;
  }
  signal(kCmdDone);
  }
  }
  __syncthreads();
  if (S.bailf) {
    *bail = 1;
    return 0.0;
  }
  if (!need_loss) return 0.0;
  // final reassignment and loss (learner.cpp:305-311)
  w_sort(S, k, g);
  double local = 0.0;
  for (int p = lo, j = 0; p < hi; ++p, ++j) {
    const double x = (double)R.xs[R.idx(g.t, j)];
    const int q = w_nearest(x, S, k);
    local = __dadd_rn(local, __dmul_rn((double)R.wv[R.idx(g.t, j)], dcost(x, S.cen[q])));
  }
  return g_sum(local, S, g);
}

// One CTA = one row group of G warps (blockDim.x = 32 G), persistent over rows.
// MINB = 3 (<= 85 registers) for row groups of <= 4 warps: 5 row groups per SM
// (shared-memory bound) instead of 4 (register bound) for 4096-sample rows,
// +13 % rows/s; 8-warp groups (one per SM) keep the looser bound.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_kmeans_warp(WkParams P) {
  extern __shared__ __align__(16) uint8_t dsmem[];
  Grp g;
  g.t = threadIdx.x;
  g.lane = threadIdx.x & 31;
  g.warp = threadIdx.x >> 5;
  g.G = blockDim.x >> 5;
  g.T = blockDim.x;
  WarpKm& S = *reinterpret_cast<WarpKm*>(dsmem);
  double* CT = reinterpret_cast<double*>(dsmem + ((sizeof(WarpKm) + 15) & ~size_t(15)));
  float* xs = reinterpret_cast<float*>(dsmem + P.state_bytes);
  const int n = P.n, C = P.C, k = P.k;
  float* wv = xs + (size_t)C * (g.T + 1);
  double* d2 = P.d2scr + (size_t)blockIdx.x * C * g.T;
  const WRow R{xs, wv, n, C, g.T, g.t * C, min(n, g.t * C + C), (n + C - 1) / C};
  while (true) {
    __syncthreads();
    if (g.t == 0) S.bci = atomicAdd(P.row_counter, 1);
    __syncthreads();
    const int row = S.bci;
    if (row >= P.rows) break;
    const int* sv_row = P.svals + (size_t)row * n;
    const float* sk_row = P.skeys + (size_t)row * n;
    const float* xo = P.ws + (size_t)row * n;
    const float* wo = P.sw + (size_t)row * n;
    int bad = 0;
    for (int p = g.t; p < n; p += g.T) {
      const float w = wo[p];
      bad |= !(w >= 0.0f) || !isfinite(w);
    }
    if (__syncthreads_or(bad)) {  // KmProblem::validate (learner.cpp:10-23)
      if (g.t == 0) dev_fail(P.err, ANYQ_ERR_STATS);
      continue;
    }
    if (g.t == 0) {
      S.rng = Rng::for_row(P.seed, P.row_offset + row);
      S.pnexc = 0;
      S.nexc = 0;
    }
    __syncthreads();
    double best = INFINITY;
    int bail = 0;
    for (int r = 0; r < P.restarts && !bail; ++r) {
      const long long t0 = clock64();
      if (P.init == ANYQ_INIT_KMPP || P.init == ANYQ_INIT_RANDOM) {
        // seeding works on the row in ORIGINAL order
        w_load_row_batched(R, g, xs, wv, xo, wo, nullptr);
        __syncthreads();
        if (P.init == ANYQ_INIT_KMPP) w_init_kmpp(R, sk_row, d2, S, k, g);
        else w_init_random(R, sk_row, S, k, g);
      } else if (P.init == ANYQ_INIT_GRID) {
        if (g.t < k) S.cen[g.t] = (double)(-(k / 2) + g.t);
      } else {
        const float nf4[16] = {-1.0f, -0.6961928009986877f, -0.5250730514526367f,
                               -0.39491748809814453f, -0.28444138169288635f,
                               -0.18477343022823334f, -0.09105003625154495f, 0.0f,
                               0.07958029955625534f, 0.16093020141124725f, 0.24611230194568634f,
                               0.33791524171829224f, 0.44070982933044434f, 0.5626170039176941f,
                               0.7229568362236023f, 1.0f};
        if (g.t < k) S.cen[g.t] = (double)nf4[g.t & 15];
      }
      __syncthreads();
      // Lloyd works on the sorted row
      w_load_row_batched(R, g, xs, wv, sk_row, wo, sv_row);
      __syncthreads();
      const long long t1 = clock64();
      const double loss = w_lloyd(P, R, S, CT, sv_row, g, P.restarts > 1, &bail);
      if (P.dbg && g.t == 0) {
        atomicAdd((unsigned long long*)&P.dbg[0], (unsigned long long)(t1 - t0));
        atomicAdd((unsigned long long*)&P.dbg[1], (unsigned long long)(clock64() - t1));
      }
      if (!bail && (P.restarts == 1 || loss < best)) {
        best = loss;
        if (g.t < k) S.best_cen[g.t] = S.cen[g.t];
      }
      __syncthreads();
    }
    if (bail) {
      if (g.t == 0) P.bail_rows[atomicAdd(P.bail_n, 1)] = row;
      continue;
    }
    // best centroids -> sorted LUT + rank-remapped codes (learner.cpp:343-369)
    if (g.t < k) S.cen[g.t] = S.best_cen[g.t];
    w_sort(S, k, g);
    if (g.t < k) P.luts[(size_t)row * k + g.t] = (float)S.sv[g.t];
    for (int p0 = R.lo; p0 < R.hi; p0 += 8) {  // original positions loaded 8 at a time, then stores
      int ov[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) ov[u] = p0 + u < R.hi ? __ldg(sv_row + p0 + u) : 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (p0 + u >= R.hi) break;
        const int q = w_nearest((double)xs[R.idx(g.t, p0 + u - R.lo)], S, k);
        P.codes[(size_t)row * n + ov[u]] = (uint8_t)S.rank_of[q];
      }
    }
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

namespace {

// Stable ascending sort of every row (value, original index), stream ordered.
void sort_rows(const float* ws, int64_t rows, int64_t cols, float* skeys, int* svals,
               cudaStream_t s) {
  const int64_t total = rows * cols;
  DevBuf<int> idx(total, s), offs(rows + 1, s);
  k_fill_offsets<<<(unsigned)((rows + 256) / 256), 256, 0, s>>>(offs.p, rows, cols);
  ANYQ_LAUNCHED();
  k_iota_rows<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(idx.p, rows, cols);
  ANYQ_LAUNCHED();
  size_t temp_bytes = 0;
  ANYQ_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, temp_bytes, ws, skeys, idx.p, svals,
                                                      (int)total, (int)rows, offs.p, offs.p + 1, s));
  DevBuf<uint8_t> temp(temp_bytes, s);
  ANYQ_CUDA(cub::DeviceSegmentedSort::StableSortPairs(temp.p, temp_bytes, ws, skeys, idx.p, svals,
                                                      (int)total, (int)rows, offs.p, offs.p + 1, s));
  note_launch(2);
}

// Dynamic shared memory of k_kmeans_rows for rows of n samples: xs, wv (fp32)
// + 2n doubles (d2 / mass during k-means++, then the two assignment arrays).
size_t rows_kernel_smem(int64_t n) {
  return (((sizeof(float) * 2 * n) + 15) & ~size_t(15)) + sizeof(double) * 2 * n;
}

// Launches k_kmeans_rows over P.rows rows (shared memory or global scratch).
void launch_rows_kernel(KmParams& P, int64_t cta_rows, cudaStream_t s) {
  int dev = 0, sms = 148, max_optin = 0;
  ANYQ_CUDA(cudaGetDevice(&dev));
  ANYQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  ANYQ_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t need = rows_kernel_smem(P.n);
  const size_t static_smem = sizeof(Shared) + 2 * 2 * kMaxK * sizeof(int64_t);
  DevBuf<uint8_t> gscratch;
  int blocks;
  if (need + static_smem <= (size_t)max_optin) {
    P.use_smem = 1;
    P.gscratch = nullptr;
    P.scratch_stride = 0;
    ensure_dyn_smem((const void*)k_kmeans_rows, (int)need);
    int per_sm = 0;
    ANYQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kmeans_rows, kThreads, need));
    blocks = (int)std::min<int64_t>(cta_rows, (int64_t)sms * std::max(1, per_sm));
    k_kmeans_rows<<<blocks, kThreads, need, s>>>(P);
  } else {
    int per_sm = 0;
    ANYQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kmeans_rows, kThreads, 0));
    blocks = (int)std::min<int64_t>(cta_rows, (int64_t)sms * std::max(1, per_sm));
    P.use_smem = 0;
    P.scratch_stride = (need + 255) & ~size_t(255);
    gscratch.alloc(P.scratch_stride * blocks, s);
    P.gscratch = gscratch.p;
    k_kmeans_rows<<<blocks, kThreads, 0, s>>>(P);
  }
  ANYQ_LAUNCHED();
  // scratch is released stream-ordered on return
}

}  // namespace

void launch_kmeans_problems(const float* x, const float* w, int64_t rows, int64_t n, int k,
                            const anyq_config& cfg, int mode, const uint64_t* rng_key,
                            uint64_t* rng_ctr, double* centroids, uint8_t* assignments, double* loss,
                            int* iters, float* luts, uint8_t* codes, int* err, cudaStream_t s) {
  if (rows * n >= (int64_t(1) << 31)) fail(ANYQ_ERR_SHAPE, "k-means batch too large; split rows");
  if (k < 1 || k > kMaxK) fail(ANYQ_ERR_CONFIG, "k must be in [1, 256]");
  DevBuf<float> skeys(rows * n, s);
  DevBuf<int> svals(rows * n, s), counter(1, s);
  sort_rows(x, rows, n, skeys.p, svals.p, s);
  ANYQ_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(int), s));
  KmParams P{};
  P.ws = x;
  P.sw = w;
  P.skeys = skeys.p;
  P.svals = svals.p;
  P.rows = rows;
  P.n = n;
  P.k = k;
  P.init = mode == 2 ? ANYQ_INIT_KMPP : cfg.init;
  P.max_iters = cfg.max_iters;
  P.restarts = cfg.restarts;
  P.check_inv = cfg.check_invariants;
  P.rel_tol = cfg.rel_tol;
  P.err = err;
  P.row_counter = counter.p;
  P.mode = mode;
  P.exact = 1;
  P.rng_key = rng_key;
  P.rng_ctr = rng_ctr;
  P.out_cen = centroids;
  P.out_asg = assignments;
  P.out_loss = loss;
  P.out_iters = iters;
  P.luts = luts;
  P.codes = codes;
  launch_rows_kernel(P, rows, s);
}

void launch_kmeans(const float* ws, const float* sw, int64_t rows, int64_t cols,
                   const anyq_config& cfg, int64_t row_offset, float* luts, uint8_t* codes,
                   int* err, cudaStream_t s) {
  if (rows * cols >= (int64_t(1) << 31)) fail(ANYQ_ERR_SHAPE, "quantize batch too large; split rows");
  const int64_t total = rows * cols;
  DevBuf<float> skeys(total, s);
  DevBuf<int> svals(total, s), counter(1, s);
  sort_rows(ws, rows, cols, skeys.p, svals.p, s);
  ANYQ_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(int), s));

  KmParams P{};
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

  int dev = 0;
  ANYQ_CUDA(cudaGetDevice(&dev));
  int sms = 148, max_optin = 0;
  ANYQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  ANYQ_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  P.row_list = nullptr;
  P.row_list_n = nullptr;

  // Warp-per-row kernel for k <= 16 when a warp's row fits in shared memory;
  // rows it cannot take (near-duplicate centroids) are finished by the CTA
  // kernel below from the bail list.
  DevBuf<double> d2scr;
  DevBuf<int> bail(rows, s), bail_n(1, s), counter2(1, s);
  // row group size: ~32 samples per thread (more warps per row for long rows;
  // measured best on B200 for 4096-sample rows), ANYQ_KM_G overrides (1..8)
  int G = (int)std::min<int64_t>(kMaxG, std::max<int64_t>(1, (cols + 1023) / 1024));
  if (const char* e = std::getenv("ANYQ_KM_G")) G = std::max(1, std::min(kMaxG, std::atoi(e)));
  const int T = 32 * G;
  const int64_t Cw = (cols + T - 1) / T;
  const uint32_t state_bytes =
      (uint32_t)(((sizeof(WarpKm) + 15) & ~size_t(15)) + 4 * sizeof(double) * T);
  const size_t cta_smem = state_bytes + ((2 * sizeof(float) * Cw * (T + 1) + 15) & ~size_t(15));
  const bool use_warp = P.k <= kWK && !P.check_inv && cta_smem <= (size_t)max_optin &&
                        cols < (int64_t(1) << 30);
  if (use_warp) {
    WkParams W;
    W.ws = ws;
    W.sw = sw;
    W.skeys = skeys.p;
    W.svals = svals.p;
    W.rows = rows;
    W.n = (int)cols;
    W.C = (int)Cw;
    W.k = P.k;
    W.init = P.init;
    W.max_iters = P.max_iters;
    W.restarts = P.restarts;
    W.rel_tol = P.rel_tol;
    W.seed = P.seed;
    W.row_offset = row_offset;
    W.luts = luts;
    W.codes = codes;
    W.err = err;
    W.row_counter = counter.p;
    W.state_bytes = state_bytes;
    static const bool km_debug = std::getenv("ANYQ_KM_DEBUG") != nullptr;
    DevBuf<long long> dbg;
    W.dbg = nullptr;
    if (km_debug) {
      dbg.alloc(16, s);
      ANYQ_CUDA(cudaMemsetAsync(dbg.p, 0, 16 * sizeof(long long), s));
      W.dbg = dbg.p;
    }
    const int smem = (int)cta_smem;
    const auto kfn = G <= 4 ? k_kmeans_warp<3> : k_kmeans_warp<2>;
    ANYQ_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    ANYQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, T, smem));
    const int blocks = (int)std::min<int64_t>(rows, (int64_t)sms * std::max(1, per_sm));
    d2scr.alloc((size_t)blocks * Cw * T, s);
    W.d2scr = d2scr.p;
    W.bail_rows = bail.p;
    W.bail_n = bail_n.p;
    ANYQ_CUDA(cudaMemsetAsync(bail_n.p, 0, sizeof(int), s));
    kfn<<<blocks, T, smem, s>>>(W);
    ANYQ_LAUNCHED();
    if (km_debug) {
      long long h[16];
      ANYQ_CUDA(cudaMemcpyAsync(h, dbg.p, sizeof h, cudaMemcpyDeviceToHost, s));
      int nb = 0;
      ANYQ_CUDA(cudaMemcpyAsync(&nb, bail_n.p, sizeof nb, cudaMemcpyDeviceToHost, s));
      ANYQ_CUDA(cudaStreamSynchronize(s));
      std::fprintf(stderr,
                   "[kmeans group] rows %lld n %lld warps/row %d blocks %d: init %.0f cyc/row, lloyd %.0f "
                   "cyc/row, iters/row %.2f, repairs %lld, bailed %d; per iter: E %.0f M %.0f rep %.0f loss %.0f "
                   "[sort %.0f, M-runs %.0f, changed+stop %.0f]\n",
                   (long long)rows, (long long)cols, G, blocks, (double)h[0] / rows,
                   (double)h[1] / rows, (double)h[2] / rows, h[3], nb, (double)h[4] / h[2], (double)h[5] / h[2],
                   (double)h[6] / h[2], (double)h[7] / h[2], (double)h[8] / h[2], (double)h[9] / h[2],
                   (double)h[10] / h[2]);
    }
    // the CTA kernel takes the bailed rows (exits at once when there are none)
    ANYQ_CUDA(cudaMemsetAsync(counter2.p, 0, sizeof(int), s));
    P.row_counter = counter2.p;
    P.row_list = bail.p;
    P.row_list_n = bail_n.p;
  }

  launch_rows_kernel(P, use_warp ? std::min<int64_t>(rows, (int64_t)sms) : rows, s);
}

}  // namespace anyq_b200
