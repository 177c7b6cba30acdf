// Shared helpers for the B200 any4 library: status/error plumbing for the
// C-ABI, launch accounting, and bit-exact device restatements of the
// reference's scalar primitives (RNG core.hpp:154-200, fp16/bf16 narrowing
// pack.cpp:61-128, ktiled_pos pack.hpp:79-84, group_of scaling.hpp:36-45).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "anyq_b200.h"

namespace anyq_b200 {

// ---------------------------------------------------------------------------
// Host-side error plumbing
// ---------------------------------------------------------------------------
struct Failure {
  anyq_status status;
  std::string msg;
};

[[noreturn]] void fail(anyq_status s, const std::string& msg);
void set_last_error(const std::string& msg);
void note_launch(int n = 1);

#define ANYQ_CUDA(call)                                                             \
  do {                                                                              \
    cudaError_t e__ = (call);                                                       \
    if (e__ != cudaSuccess)                                                         \
      ::anyq_b200::fail(ANYQ_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)

// Raises a kernel's dynamic shared-memory limit to `bytes` once per (kernel,
// device) — the attribute is per device, so a process driving several GPUs
// configures each (capi.cu).
void ensure_dyn_smem(const void* kernel, int bytes);

#define ANYQ_LAUNCHED()                 \
  do {                                  \
    ::anyq_b200::note_launch();         \
    ANYQ_CUDA(cudaGetLastError());      \
  } while (0)

// Per-(device, stream) workspace (capi.cu): GEMV release counters and the
// stage error words of the stream-ordered entries.
constexpr int kWsDone = 8;  // GEMV chain release counters (one per problem)
constexpr int kWsErr = 8;   // stage error words, checked in index order
constexpr int kK2FlagStride = 32;  // one K2 stream-K counter per 128-B line
constexpr int kWsK2 = 256 * kK2FlagStride;  // K2 stream-K partial-ready counters (one per CTA, self-resetting)
constexpr int kErrFinite = 0, kErrStats = 1, kErrRows = 2, kErrLearn = 3, kErrPack = 4,
              kErrGemv = 5;
struct StreamWs {
  int* done;
  int* err;
  int* k2flags;
};
StreamWs stream_ws(cudaStream_t s);
// Per-(device, stream) fp32 scratch of at least n floats (grow-only; a grown
// buffer keeps the old one alive, so graphs captured earlier stay valid).
float* stream_scratch_f32(cudaStream_t s, size_t n);
// Synchronises s; raises the first recorded stage error (and clears the words).
void check_stream_errors(cudaStream_t s, const char* what);

// Device-side error word: kernels atomicMax an anyq_status into it.
__device__ __forceinline__ void dev_fail(int* err, int status) {
  if (err) atomicMax(err, status);
}

// ---------------------------------------------------------------------------
// RNG (core.hpp:154-200): pure 64-bit integer math + double conversion, so it
// is bit-identical on device.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct Rng {
  uint64_t key;
  uint64_t counter;
  __host__ __device__ static Rng for_row(uint64_t seed, int64_t row) {
    Rng r;
    r.key = splitmix64(seed) ^ splitmix64(0x9E3779B97F4A7C15ull * (static_cast<uint64_t>(row) + 1));
    r.counter = 0;
    return r;
  }
  __host__ __device__ uint64_t next_u64() { return splitmix64(key + 0xD1B54A32D192ED03ull * ++counter); }
  __host__ __device__ double next_double() {
    return static_cast<double>(next_u64() >> 11) * 0x1.0p-53;
  }
  __host__ __device__ int64_t next_index(int64_t bound) {
    double u = next_double();
    int64_t i = static_cast<int64_t>(__dmul_rn_hd(u, static_cast<double>(bound)));
    return i >= bound ? bound - 1 : i;
  }
  __host__ __device__ static double __dmul_rn_hd(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
  }
};

// ---------------------------------------------------------------------------
// fp16 / bf16 narrowing, bit-identical to pack.cpp:61-128 (RNE; overflow and
// non-finite inputs are reported instead of producing inf).
// Return value: the 16-bit pattern; *status set to a non-OK code on error.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint32_t f2u(float f) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(f);
#else
  uint32_t u;
  __builtin_memcpy(&u, &f, 4);
  return u;
#endif
}
__host__ __device__ __forceinline__ float u2f(uint32_t u) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  __builtin_memcpy(&f, &u, 4);
  return f;
#endif
}

__host__ __device__ __forceinline__ uint16_t f32_to_f16_exact(float f, int* status) {
  uint32_t x = f2u(f);
  uint16_t sign = static_cast<uint16_t>((x >> 16) & 0x8000u);
  uint32_t a = x & 0x7FFFFFFFu;
  if (a >= 0x7F800000u) {
    *status = ANYQ_ERR_NONFINITE;
    return 0;
  }
  if (a >= 0x477FF000u) {
    *status = ANYQ_ERR_IO;
    return 0;
  }
  uint32_t out;
  if (a < 0x38800000u) {
    uint32_t e32 = a >> 23;
    uint32_t shift = 113u - e32;
    if (a == 0 || shift > 24u) {
      out = 0;
    } else {
      uint32_t mant = (a & 0x7FFFFFu) | 0x800000u;
      uint32_t q = mant >> (shift + 13u);
      uint32_t rem = mant & ((1u << (shift + 13u)) - 1u);
      uint32_t half = 1u << (shift + 12u);
      if (rem > half || (rem == half && (q & 1u))) ++q;
      out = q;
    }
  } else {
    uint32_t e = (a >> 23) - 112u;
    uint32_t mant = a & 0x7FFFFFu;
    uint32_t q = (e << 10) | (mant >> 13);
    uint32_t rem = mant & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) ++q;
    out = q;
  }
  return static_cast<uint16_t>(sign | out);
}

__host__ __device__ __forceinline__ float f16_to_f32_exact(uint16_t h) {
  uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1Fu;
  uint32_t mant = h & 0x3FFu;
  uint32_t out;
  if (e == 0) {
    if (mant == 0) {
      out = sign;
    } else {
      uint32_t shift = 0;
      while (!(mant & 0x400u)) {
        mant <<= 1;
        ++shift;
      }
      out = sign | ((113u - shift) << 23) | ((mant & 0x3FFu) << 13);
    }
  } else if (e == 0x1Fu) {
    out = sign | 0x7F800000u | (mant << 13);
  } else {
    out = sign | ((e + 112u) << 23) | (mant << 13);
  }
  return u2f(out);
}

__host__ __device__ __forceinline__ uint16_t f32_to_bf16_exact(float f, int* status) {
  uint32_t x = f2u(f);
  if ((x & 0x7F800000u) == 0x7F800000u) {
    *status = ANYQ_ERR_NONFINITE;
    return 0;
  }
  uint32_t lsb = (x >> 16) & 1u;
  uint32_t r = x + 0x7FFFu + lsb;
  if ((r & 0x7F800000u) == 0x7F800000u) {
    *status = ANYQ_ERR_IO;
    return 0;
  }
  return static_cast<uint16_t>(r >> 16);
}

__host__ __device__ __forceinline__ float bf16_to_f32_exact(uint16_t h) {
  return u2f(static_cast<uint32_t>(h) << 16);
}

// Narrow-then-widen of narrowed() (pack.cpp:146-155).
__host__ __device__ __forceinline__ float narrow_widen(float v, int store, int* status) {
  if (store == ANYQ_STORE_FP16) return f16_to_f32_exact(f32_to_f16_exact(v, status));
  if (store == ANYQ_STORE_BF16) return bf16_to_f32_exact(f32_to_bf16_exact(v, status));
  return v;
}

// ---------------------------------------------------------------------------
// Index maps
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t ktiled_pos(int64_t k, int64_t cols, int64_t tile_k) {
  int64_t num_full = cols / tile_k;
  int64_t full_end = num_full * tile_k;
  if (k >= full_end) return k;
  return (k % tile_k) * num_full + k / tile_k;
}

struct GroupMap {
  int granularity;
  int64_t cols;
  int64_t group_size;  // groupwise
  int64_t block_size;  // blockwise
  int64_t gpr;         // groups (or blocks) per row

  __host__ __device__ int64_t operator()(int64_t i, int64_t j) const {
    switch (granularity) {
      case ANYQ_G_TENSOR: return 0;
      case ANYQ_G_ROW: return i;
      case ANYQ_G_COLUMN: return j;
      case ANYQ_G_GROUP: return i * gpr + j / group_size;
      default: return (i / block_size) * gpr + j / block_size;
    }
  }
};

inline GroupMap make_group_map(const anyq_config& c, int64_t cols) {
  GroupMap g;
  g.granularity = c.granularity;
  g.cols = cols;
  g.group_size = c.group_size > 0 ? c.group_size : 1;
  g.block_size = c.block_size > 0 ? c.block_size : 1;
  if (c.granularity == ANYQ_G_GROUP) g.gpr = (cols + g.group_size - 1) / g.group_size;
  else if (c.granularity == ANYQ_G_BLOCK) g.gpr = (cols + g.block_size - 1) / g.block_size;
  else g.gpr = 0;
  return g;
}

inline int64_t packed_bpr(int64_t cols, int bits) { return (cols * bits + 7) / 8; }

// Fixed value tables (codebooks.cpp:21-55), as host data.
extern const float kFp4Table[15];
extern const float kNf4Table[16];

// A value table for RTN / fixed-format dequantisation (<= 256 entries).
struct Table {
  int n;
  float v[256];
};

Table fixed_table(const anyq_config& c);            // codebooks.cpp:57-65
Table effective_table(Table t, bool symmetric);     // codebooks.cpp:67-73
Table int_grid_table(int bits, bool shifted);       // codebooks.cpp:8-19
void validate_config(const anyq_config& c, int64_t rows, int64_t cols);  // core.hpp:124-142
int64_t group_count(const anyq_config& c, int64_t rows, int64_t cols);   // scaling.cpp:8-24

// Keep freed stream-ordered allocations cached in the device's default pool
// (no cudaFree / unmap on the hot path).
void keep_default_pool();

// Device scratch buffers with RAII. With a stream, allocation and release are
// stream-ordered (cudaMallocAsync / cudaFreeAsync from the cached pool).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  bool async = false;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(size_t count, cudaStream_t s) { alloc(count, s); }
  void alloc(size_t count) {
    n = count;
    if (count) ANYQ_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void alloc(size_t count, cudaStream_t s) {
    n = count;
    st = s;
    async = true;
    keep_default_pool();
    if (count) ANYQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, s));
  }
  ~DevBuf() {
    if (p) {
      if (async) cudaFreeAsync(p, st);
      else cudaFree(p);
    }
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void upload(const T* h, size_t count) {
    if (count) ANYQ_CUDA(cudaMemcpy(p, h, sizeof(T) * count, cudaMemcpyHostToDevice));
  }
  void download(T* h, size_t count) const {
    if (count) ANYQ_CUDA(cudaMemcpy(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost));
  }
  void zero() {
    if (n) ANYQ_CUDA(cudaMemset(p, 0, sizeof(T) * n));
  }
};

// Reads the device error word and converts it to a Failure.
void check_device_error(const int* d_err, const char* what);

}  // namespace anyq_b200
