// K1d — fused LUT GEMM for 3 <= M <= 64: dequantise into shared-memory tiles,
// multiply on the tensor cores (mma.sync m16n8k16, bf16 x bf16 -> fp32), no
// bf16 weight copy in HBM.
//
//   y[m][n] = sum_k x[m][k] * bf16(alpha[n][g(k)] * T_n[c[n][k]] + beta[n][g(k)])
//
// i.e. the dequant + GEMM path (dequant_gemm.cu) without its round trip of a
// bf16 weight copy through HBM; same weight rounding (fp32 alpha*T+beta, no
// contraction, qgemm.cpp:98-111, rounded once to bf16) and the same tolerance
// (2^-8 * sum |x*w|, tests/test_gpu_gemm.py).
//
// A CTA is 4 warps = 4 row blocks (128 weight rows) over a contiguous range of
// 128-k chunks (split-K over the grid when the row blocks alone do not fill
// the GPU). Per chunk:
//  * the CTA stages the chunk's x rows (M x 128 bf16) in shared memory in the
//    PHYSICAL k order of the prepacked codes (byte b of slab q holds k =
//    128c + 16q + 2b (+1) for b < 8 and 128c + 64 + 16q + 2(b-8) (+1) for
//    b >= 8), so weights and x never need re-permuting;
//  * each warp expands its row block: lane L = row L builds the 16 dequantised
//    values of its row for the chunk's scale group in a per-warp table
//    (tbl[i][lane], bank = lane), reads its 64 code bytes, and writes its 128
//    bf16 weights as one row of a 32 x 128 shared tile;
//  * ldmatrix -> mma.sync: A = weight tile (2 m16 tiles), B = x tile
//    (M/8 n8 tiles), 8 k16 steps, fp32 accumulators in registers.
// Split-K partials go to a [S][M][N] fp32 scratch and are summed in a fixed
// order by a second kernel: deterministic.
#include <cuda_bf16.h>

#include "kernels.cuh"
#include "lutgemm.cuh"

namespace anyq_b200 {

namespace {

// warps (row blocks) per CTA: 4, or 8 for the widest x tiles (M > 16), where
// the register-heavy accumulators leave few CTAs per SM
template <int NT>
constexpr int mma_warps() {
  return NT >= 4 ? 8 : 4;
}
constexpr int kTileStride = 136;  // bf16 per shared row (128 + 8 pad: conflict-free ldmatrix)

struct MmaArgs {
  const uint4* codes;  // [RB][C][4][32] uint4
  const uint4* lut;    // [RB*32][2] uint4
  const __half2* ab;   // [RB][GR][32]
  const __nv_bfloat16* x;
  __nv_bfloat16* y;
  float* y32;
  float* part;  // [S][M][N] when S > 1
  int64_t N, K;
  int M, RB, C, GR, gshift, S, cps;  // cps: chunks per split
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2,
                                        uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& b0, uint32_t& b1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
               : "=r"(b0), "=r"(b1)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NT>
constexpr uint32_t mma_smem_bytes() {  // xs + weight tiles + tables
  constexpr int kMmaWarps = mma_warps<NT>();
  return (uint32_t)(NT * 8 * kTileStride * 2 + kMmaWarps * 32 * kTileStride * 2 + kMmaWarps * 16 * 32 * 4);
}

template <int NT>  // n8 tiles of x rows: M <= 8 * NT
__global__ void __launch_bounds__(mma_warps<NT>() * 32) k_lutmma(const MmaArgs A) {
  constexpr int kMmaWarps = mma_warps<NT>();
  extern __shared__ __align__(16) uint8_t smem[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* wt_base_ptr = xs + NT * 8 * kTileStride;
  uint32_t* tbl_base = reinterpret_cast<uint32_t*>(wt_base_ptr + kMmaWarps * 32 * kTileStride);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups = (A.RB + kMmaWarps - 1) / kMmaWarps;
  const int grp = blockIdx.x % groups, split = blockIdx.x / groups;
  const int rb = grp * kMmaWarps + warp;
  const bool live = rb < A.RB;
  const int c0 = split * A.cps, c1 = min(A.C, c0 + A.cps);
  __nv_bfloat16* wt = wt_base_ptr + warp * 32 * kTileStride;
  uint32_t(*tbl)[32] = reinterpret_cast<uint32_t(*)[32]>(tbl_base + warp * 16 * 32);
  const int64_t row = (int64_t)rb * 32 + lane;

  float t[16];
  if (live) {
    const uint4 l0 = A.lut[row * 2], l1 = A.lut[row * 2 + 1];
    const uint32_t lw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&lw[j]));
      t[2 * j] = f.x;
      t[2 * j + 1] = f.y;
    }
  }
  float acc[2][NT][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0f;

  const uint32_t xs_base = (uint32_t)__cvta_generic_to_shared(xs);
  const uint32_t wt_base = (uint32_t)__cvta_generic_to_shared(wt);
  // codes of the next chunk are loaded one iteration ahead (global latency)
  uint4 wn[4] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0),
                 make_uint4(0, 0, 0, 0)};
  __half2 abn = __floats2half2_rn(0.0f, 0.0f);
  auto ab_of = [&](int c) {
    const int g = A.gshift >= 30 ? 0 : (c >> A.gshift);
    return A.ab[((int64_t)rb * A.GR + g) * 32 + lane];
  };
  if (live && c0 < c1) {
    const uint4* cp = A.codes + ((int64_t)rb * A.C + c0) * 128 + lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) wn[q] = cp[q * 32];
    abn = ab_of(c0);
  }
  // x chunk staging: this thread's 16-bf16 runs, loaded one chunk ahead
  constexpr int kXTasks = (NT * 8 * 8 + kMmaWarps * 32 - 1) / (kMmaWarps * 32);
  uint4 xv[kXTasks][2];
  auto load_x = [&](int c) {
#pragma unroll
    for (int u = 0; u < kXTasks; ++u) {
      const int task = threadIdx.x + u * kMmaWarps * 32;
      uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
      const int n = task >> 3, run = task & 7;
      const int q = run >> 1, h = run & 1;
      const int64_t k0 = (int64_t)c * 128 + 16 * q + 64 * h;
      if (task < NT * 64 && n < A.M) {
        const __nv_bfloat16* src = A.x + (int64_t)n * A.K + k0;
        if (((A.K & 7) == 0) && k0 + 16 <= A.K) {
          v0 = *reinterpret_cast<const uint4*>(src);
          v1 = *reinterpret_cast<const uint4*>(src + 8);
        } else {
          unsigned short s[16];
          for (int j = 0; j < 16; ++j)
            s[j] = k0 + j < A.K ? __bfloat16_as_ushort(src[j]) : (unsigned short)0;
          v0 = make_uint4(s[0] | (s[1] << 16), s[2] | (s[3] << 16), s[4] | (s[5] << 16), s[6] | (s[7] << 16));
          v1 = make_uint4(s[8] | (s[9] << 16), s[10] | (s[11] << 16), s[12] | (s[13] << 16),
                          s[14] | (s[15] << 16));
        }
      }
      xv[u][0] = v0;
      xv[u][1] = v1;
    }
  };
  if (c0 < c1) load_x(c0);
  for (int c = c0; c < c1; ++c) {
    // ---- x chunk -> xs[n][physical k] (rows >= M and k >= K are zero)
    __syncthreads();  // previous chunk's B reads are done
#pragma unroll
    for (int u = 0; u < kXTasks; ++u) {
      const int task = threadIdx.x + u * kMmaWarps * 32;
      if (task < NT * 64) {
        const int n = task >> 3, run = task & 7;
        const int q = run >> 1, h = run & 1;
        uint4* dst = reinterpret_cast<uint4*>(xs + n * kTileStride + 32 * q + 16 * h);
        dst[0] = xv[u][0];
        dst[1] = xv[u][1];
      }
    }
    if (c + 1 < c1) load_x(c + 1);
    // ---- this warp's 32 x 128 weight tile
    if (live) {
      const float2 s = __half22float2(abn);
      uint4 w4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w4[q] = wn[q];
      if (c + 1 < c1) {
        const uint4* cp = A.codes + ((int64_t)rb * A.C + c + 1) * 128 + lane;
#pragma unroll
        for (int q = 0; q < 4; ++q) wn[q] = cp[q * 32];
        abn = ab_of(c + 1);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i)
        tbl[i][lane] = (uint32_t)__bfloat16_as_ushort(
            __float2bfloat16_rn(__fadd_rn(__fmul_rn(s.x, t[i]), s.y)));
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t wd[4] = {w4[q].x, w4[q].y, w4[q].z, w4[q].w};
        uint32_t o[16];
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          const uint32_t byte = (wd[b >> 2] >> (8 * (b & 3))) & 0xffu;
          o[b] = __byte_perm(tbl[byte & 15][lane], tbl[byte >> 4][lane], 0x5410);
        }
        uint4* trow = reinterpret_cast<uint4*>(wt + lane * kTileStride + 32 * q);
        trow[0] = make_uint4(o[0], o[1], o[2], o[3]);
        trow[1] = make_uint4(o[4], o[5], o[6], o[7]);
        trow[2] = make_uint4(o[8], o[9], o[10], o[11]);
        trow[3] = make_uint4(o[12], o[13], o[14], o[15]);
      }
    }
    __syncthreads();  // x chunk and weight tiles visible
    if (live) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t a[2][4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = 16 * i + (lane & 15), col = 16 * ks + 8 * (lane >> 4);
          ldsm_x4(wt_base + (uint32_t)(r * kTileStride + col) * 2, a[i][0], a[i][1], a[i][2], a[i][3]);
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          uint32_t b0, b1;
          const int r = 8 * j + (lane & 7), col = 16 * ks + 8 * ((lane >> 3) & 1);
          ldsm_x2(xs_base + (uint32_t)(r * kTileStride + col) * 2, b0, b1);
#pragma unroll
          for (int i = 0; i < 2; ++i) mma_bf16(acc[i][j], a[i][0], a[i][1], a[i][2], a[i][3], b0, b1);
        }
      }
    }
  }
  if (!live) return;
  // ---- epilogue: acc[i][j][e]: weight row 16i + lane/4 (+8 for e >= 2),
  // x row 8j + 2(lane%4) + (e & 1)
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t n = (int64_t)rb * 32 + 16 * i + (lane >> 2) + 8 * (e >> 1);
        const int m = 8 * j + 2 * (lane & 3) + (e & 1);
        if (n >= A.N || m >= A.M) continue;
        const float v = acc[i][j][e];
        if (A.S > 1) {
          A.part[((int64_t)split * A.M + m) * A.N + n] = v;
        } else {
          A.y[(int64_t)m * A.N + n] = __float2bfloat16_rn(v);
          if (A.y32) A.y32[(int64_t)m * A.N + n] = v;
        }
      }
}

// y = sum over splits in a fixed order (deterministic split-K combine)
__global__ void k_lutmma_combine(const float* __restrict__ part, int S, int64_t MN,
                                 __nv_bfloat16* __restrict__ y, float* __restrict__ y32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < MN;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = part[i];
    for (int s = 1; s < S; ++s) v += part[(int64_t)s * MN + i];
    y[i] = __float2bfloat16_rn(v);
    if (y32) y32[i] = v;
  }
}

template <int NT>
void launch_mma(const MmaArgs& A, int blocks, cudaStream_t s) {
  constexpr uint32_t smem = mma_smem_bytes<NT>();
  ensure_dyn_smem((const void*)k_lutmma<NT>, (int)smem);
  k_lutmma<NT><<<blocks, mma_warps<NT>() * 32, smem, s>>>(A);
  ANYQ_LAUNCHED();
}

}  // namespace

bool lutmma_supports(const LutTensor* t, int64_t m) {
  return t && m >= 1 && m <= 64 && t->gv_gshift >= 0;
}

void lutmma_run(const LutTensor* t, const void* x, int64_t m, void* y, float* y32, cudaStream_t s) {
  if (!lutmma_supports(t, m))
    fail(ANYQ_ERR_CONFIG, "fused LUT MMA needs 1 <= m <= 64 and rowwise scales or group 128*2^j");
  MmaArgs A;
  A.codes = reinterpret_cast<const uint4*>(t->codes);
  A.lut = reinterpret_cast<const uint4*>(t->lut);
  A.ab = t->ab;
  A.x = reinterpret_cast<const __nv_bfloat16*>(x);
  A.y = reinterpret_cast<__nv_bfloat16*>(y);
  A.y32 = y32;
  A.N = t->rows;
  A.K = t->cols;
  A.M = (int)m;
  A.RB = t->RB;
  A.C = t->C;
  A.GR = t->GR;
  A.gshift = t->gv_gshift;
  const int nt = m <= 8 ? 1 : m <= 16 ? 2 : m <= 32 ? 4 : 8;
  const int warps_per_cta = nt >= 4 ? 8 : 4;  // mma_warps<NT>()
  // split K until the grid covers ~2 CTAs per SM (at least 2 chunks per split)
  const int groups = (t->RB + warps_per_cta - 1) / warps_per_cta;
  int S = std::max(1, std::min((2 * t->sms + groups - 1) / groups, std::max(1, t->C / 2)));
  A.cps = (t->C + S - 1) / S;
  S = (t->C + A.cps - 1) / A.cps;
  A.S = S;
  DevBuf<float> part;
  if (S > 1) {
    part.alloc((size_t)S * m * t->rows, s);
    A.part = part.p;
  } else {
    A.part = nullptr;
  }
  const int blocks = groups * S;
  if (nt == 1) launch_mma<1>(A, blocks, s);
  else if (nt == 2) launch_mma<2>(A, blocks, s);
  else if (nt == 4) launch_mma<4>(A, blocks, s);
  else launch_mma<8>(A, blocks, s);
  if (S > 1) {
    const int64_t MN = m * t->rows;
    k_lutmma_combine<<<(unsigned)std::min<int64_t>((MN + 255) / 256, (int64_t)t->sms * 8), 256, 0, s>>>(
        part.p, S, MN, A.y, y32);
    ANYQ_LAUNCHED();
  }
}

}  // namespace anyq_b200
