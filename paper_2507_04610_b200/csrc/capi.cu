// C-ABI entry points (include/anyq_b200.h). Host-side orchestration only:
// argument validation with the reference's error classes, H2D/D2H staging for
// the host-buffer calls, and kernel launches. All compute is on the device.
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "lutgemm.cuh"

namespace anyq_b200 {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

[[noreturn]] void fail(anyq_status s, const std::string& msg) { throw Failure{s, msg}; }
void set_last_error(const std::string& msg) { g_last_error = msg; }

void ensure_dyn_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  ANYQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  int& cur = done[{kernel, dev}];
  if (bytes > cur) {
    ANYQ_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    cur = bytes;
  }
}
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

const float kFp4Table[15] = {-6.0f, -4.0f, -3.0f, -2.0f, -1.5f, -1.0f, -0.5f, 0.0f,
                             0.5f,  1.0f,  1.5f,  2.0f,  3.0f,  4.0f,  6.0f};
const float kNf4Table[16] = {-1.0f,
                             -0.6961928009986877f,
                             -0.5250730514526367f,
                             -0.39491748809814453f,
                             -0.28444138169288635f,
                             -0.18477343022823334f,
                             -0.09105003625154495f,
                             0.0f,
                             0.07958029955625534f,
                             0.16093020141124725f,
                             0.24611230194568634f,
                             0.33791524171829224f,
                             0.44070982933044434f,
                             0.5626170039176941f,
                             0.7229568362236023f,
                             1.0f};

Table int_grid_table(int bits, bool shifted) {
  if (bits != 2 && bits != 3 && bits != 4 && bits != 8)
    fail(ANYQ_ERR_CONFIG, "int_grid: bits must be one of {2,3,4,8}");
  Table t;
  int lo = -(1 << (bits - 1)) + (shifted ? 1 : 0);
  t.n = 1 << bits;
  for (int q = 0; q < t.n; ++q) t.v[q] = (float)(lo + q);
  return t;
}

Table fixed_table(const anyq_config& c) {
  Table t;
  switch (c.codebook) {
    case ANYQ_CB_INT: return int_grid_table(c.bits, c.int_range_shifted != 0);
    case ANYQ_CB_FP4:
      t.n = 15;
      std::memcpy(t.v, kFp4Table, sizeof kFp4Table);
      return t;
    case ANYQ_CB_NF4:
      t.n = 16;
      std::memcpy(t.v, kNf4Table, sizeof kNf4Table);
      return t;
    case ANYQ_CB_ANY: fail(ANYQ_ERR_CONFIG, "AnyN has no fixed codebook");
  }
  fail(ANYQ_ERR_CONFIG, "unknown codebook kind");
}

Table effective_table(Table t, bool symmetric) {
  if (symmetric) return t;
  float lo = t.v[0];
  for (int q = 0; q < t.n; ++q) t.v[q] -= lo;  // host fp32, same as codebooks.cpp:70
  return t;
}

void validate_config(const anyq_config& c, int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) fail(ANYQ_ERR_SHAPE, "tensor must be at least 1x1");
  if (c.bits != 2 && c.bits != 3 && c.bits != 4 && c.bits != 8)
    fail(ANYQ_ERR_CONFIG, "bits must be one of {2,3,4,8}");
  if ((c.codebook == ANYQ_CB_FP4 || c.codebook == ANYQ_CB_NF4) && c.bits != 4)
    fail(ANYQ_ERR_CONFIG, "fp4/nf4 require bits == 4");
  if (c.granularity == ANYQ_G_GROUP && c.group_size < 2)
    fail(ANYQ_ERR_CONFIG, "group_size must be >= 2");
  if (c.granularity == ANYQ_G_BLOCK && c.block_size < 1)
    fail(ANYQ_ERR_CONFIG, "block_size must be >= 1");
  if (c.max_iters < 1) fail(ANYQ_ERR_CONFIG, "learner.max_iters must be >= 1");
  if (!(c.rel_tol >= 0)) fail(ANYQ_ERR_CONFIG, "learner.rel_tol must be >= 0");
  if (c.restarts < 1) fail(ANYQ_ERR_CONFIG, "learner.restarts must be >= 1");
  if (c.codebook == ANYQ_CB_ANY && c.granularity != ANYQ_G_ROW && c.granularity != ANYQ_G_GROUP)
    fail(ANYQ_ERR_CONFIG, "learned lookup tables are per-row; use rowwise or groupwise scaling");
  if (c.init == ANYQ_INIT_NF4 && c.bits != 4)
    fail(ANYQ_ERR_CONFIG, "nf4 seeding needs a 16-entry table (bits == 4)");
  if (c.granularity < 0 || c.granularity > 4) fail(ANYQ_ERR_CONFIG, "unknown granularity");
  if (c.codebook < 0 || c.codebook > 3) fail(ANYQ_ERR_CONFIG, "unknown codebook kind");
  if (c.codebook == ANYQ_CB_ANY && (c.init < 0 || c.init > 3)) fail(ANYQ_ERR_CONFIG, "unknown init");
  if (c.codebook == ANYQ_CB_ANY && (c.weighting < 0 || c.weighting > 2))
    fail(ANYQ_ERR_CONFIG, "unknown weighting mode");
}

int64_t group_count(const anyq_config& c, int64_t rows, int64_t cols) {
  switch (c.granularity) {
    case ANYQ_G_TENSOR: return 1;
    case ANYQ_G_ROW: return rows;
    case ANYQ_G_COLUMN: return cols;
    case ANYQ_G_GROUP: return rows * ((cols + c.group_size - 1) / c.group_size);
    case ANYQ_G_BLOCK:
      return ((rows + c.block_size - 1) / c.block_size) * ((cols + c.block_size - 1) / c.block_size);
  }
  fail(ANYQ_ERR_CONFIG, "unknown granularity");
}

// Per-(device, stream) workspace, allocated and zeroed once and never freed:
// the GEMV chain's release counters (self-resetting, so launches on one stream
// reuse them and launches on different streams never share them) and the
// sticky stage error words of the stream-ordered entries (anyq_dev_*), read
// and cleared by anyq_dev_stream_status.
StreamWs stream_ws(cudaStream_t s) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, StreamWs> table;
  int dev = 0;
  ANYQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = table.find({dev, s});
  if (it != table.end()) return it->second;
  StreamWs w{};
  int* block = nullptr;
  // The first call on a stream may come while it is being captured into a
  // graph: allocate in relaxed capture mode (cudaMalloc is otherwise refused
  // during a global-mode capture) and zero on a private stream.
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  ANYQ_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
  cudaError_t e = cudaMalloc(&block, sizeof(int) * (kWsDone + kWsErr + kWsK2));
  cudaStream_t z = nullptr;
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&z, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemsetAsync(block, 0, sizeof(int) * (kWsDone + kWsErr + kWsK2), z);
  if (e == cudaSuccess) e = cudaStreamSynchronize(z);
  if (z) cudaStreamDestroy(z);
  cudaThreadExchangeStreamCaptureMode(&mode);
  ANYQ_CUDA(e);
  w.done = block;
  w.err = block + kWsDone;
  w.k2flags = block + kWsDone + kWsErr;
  table.emplace(std::make_pair(dev, s), w);
  return w;
}

float* stream_scratch_f32(cudaStream_t s, size_t n) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<float*, size_t>> table;
  int dev = 0;
  ANYQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto& e = table[{dev, s}];
  if (e.second >= n) return e.first;
  // grow: allocate in relaxed capture mode (the call may come while s is being
  // captured); the previous buffer is not freed (graphs may still use it)
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  ANYQ_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
  float* p = nullptr;
  const size_t want = std::max(n, e.second * 2);
  const cudaError_t err = cudaMalloc(&p, want * sizeof(float));
  cudaThreadExchangeStreamCaptureMode(&mode);
  ANYQ_CUDA(err);
  e = {p, want};
  return p;
}

// First recorded stage error of the stream (stage order = the reference's
// check order), cleared; synchronises the stream.
void check_stream_errors(cudaStream_t s, const char* what) {
  const StreamWs w = stream_ws(s);
  int h[kWsErr];
  ANYQ_CUDA(cudaMemcpyAsync(h, w.err, sizeof h, cudaMemcpyDeviceToHost, s));
  ANYQ_CUDA(cudaStreamSynchronize(s));
  int first = ANYQ_OK;
  for (int i = 0; i < kWsErr && first == ANYQ_OK; ++i) first = h[i];
  if (first == ANYQ_OK) return;
  ANYQ_CUDA(cudaMemsetAsync(w.err, 0, sizeof(int) * kWsErr, s));
  ANYQ_CUDA(cudaStreamSynchronize(s));
  const char* kind = first == ANYQ_ERR_NONFINITE  ? "non-finite value"
                     : first == ANYQ_ERR_STATS    ? "negative, non-finite or all-zero weights/stats"
                     : first == ANYQ_ERR_CODE_RANGE ? "code exceeds its value table"
                                                    : "internal invariant violated";
  fail((anyq_status)first, std::string(what) + ": " + kind);
}

void keep_default_pool() {
  static int done_dev = -1;
  int dev = 0;
  ANYQ_CUDA(cudaGetDevice(&dev));
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  ANYQ_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = UINT64_MAX;
  ANYQ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  done_dev = dev;
}

void check_device_error(const int* d_err, const char* what) {
  int h = 0;
  ANYQ_CUDA(cudaMemcpy(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (h != ANYQ_OK) {
    const char* kind = h == ANYQ_ERR_NONFINITE  ? "non-finite value"
                       : h == ANYQ_ERR_STATS    ? "negative, non-finite or all-zero weights/stats"
                       : h == ANYQ_ERR_CODE_RANGE ? "code exceeds its value table"
                       : h == ANYQ_ERR_IO         ? "value overflows its 16-bit storage format"
                       : h == ANYQ_ERR_INVARIANT  ? "scale underflows its 16-bit storage format"
                                                  : "internal invariant violated";
    fail((anyq_status)h, std::string(what) + ": " + kind);
  }
}

static void ensure_device() {
  static std::once_flag once;
  static cudaError_t st = cudaSuccess;
  std::call_once(once, [] {
    int n = 0;
    st = cudaGetDeviceCount(&n);
    if (st == cudaSuccess && n == 0) st = cudaErrorNoDevice;
  });
  if (st != cudaSuccess)
    fail(ANYQ_ERR_CUDA, std::string("no usable CUDA device: ") + cudaGetErrorString(st));
}

template <typename F>
static anyq_status guard(F&& f) {
  try {
    ensure_device();
    f();
    g_last_error.clear();
    return ANYQ_OK;
  } catch (const Failure& e) {
    g_last_error = e.msg;
    return e.status;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ANYQ_ERR_INTERNAL;
  }
}

// Host-only helpers (tables, scalar narrowing, accounting) need no device.
template <typename F>
static anyq_status host_only(F&& f) {
  try {
    f();
    g_last_error.clear();
    return ANYQ_OK;
  } catch (const Failure& e) {
    g_last_error = e.msg;
    return e.status;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ANYQ_ERR_INTERNAL;
  }
}

// qmin/qmax of the quantizer (learner.cpp:401, quantize.cpp:12)
static void table_range(const anyq_config& c, float* qmin, float* qmax) {
  Table t = c.codebook == ANYQ_CB_ANY ? int_grid_table(c.bits, c.int_range_shifted != 0)
                                      : fixed_table(c);
  *qmin = t.v[0];
  *qmax = t.v[t.n - 1];
  if (!(*qmax > *qmin)) fail(ANYQ_ERR_CONFIG, "qmax must exceed qmin");
  if (c.symmetric && !(*qmax > 0)) fail(ANYQ_ERR_CONFIG, "symmetric scaling needs qmax > 0");
}

// Device-side quantize of rows (shared by the host and device entry points).
// Stream ordered, no host synchronisation (graph capturable): the data checks
// of the reference (require_finite, the stats check of build_sample_weights,
// KmProblem::validate) record their status in the stream's stage error words,
// one word per stage so the first failing stage wins as in the reference;
// later stages run on whatever the failed stage left and their results are
// discarded by the caller that checks (check_stream_errors).
static void quantize_device(const float* w, int64_t rows, int64_t cols, const anyq_config& cfg,
                            const float* exj, int64_t row_offset, uint8_t* packed, float* luts,
                            float* alphas, float* betas, cudaStream_t s) {
  validate_config(cfg, rows, cols);
  float qmin, qmax;
  table_range(cfg, &qmin, &qmax);
  int* err = stream_ws(s).err;
  launch_check_finite(w, rows * cols, err + kErrFinite, ANYQ_ERR_NONFINITE, s);
  launch_scales(w, rows, cols, cfg, qmin, qmax, alphas, betas, s);
  DevBuf<float> ws(rows * cols, s), sw;
  DevBuf<uint8_t> codes(rows * cols, s);
  if (cfg.codebook == ANYQ_CB_ANY) {
    if (exj) launch_check_stats(exj, cols, err + kErrStats, s);
    sw.alloc(rows * cols, s);
    launch_scale_rows(w, rows, cols, cfg, alphas, betas, exj, ws.p, sw.p, err + kErrRows, s);
    launch_kmeans(ws.p, sw.p, rows, cols, cfg, row_offset, luts, codes.p, err + kErrLearn, s);
  } else {
    launch_scale_rows(w, rows, cols, cfg, alphas, betas, nullptr, ws.p, nullptr, err + kErrRows, s);
    Table eff = effective_table(fixed_table(cfg), cfg.symmetric != 0);
    launch_round(ws.p, rows * cols, eff, codes.p, s);
  }
  launch_pack(codes.p, rows, cols, cfg.bits, packed, err + kErrPack, s);
}

static void fill_header(anyq_qtensor* out, int64_t rows, int64_t cols, const anyq_config& cfg) {
  out->rows = rows;
  out->cols = cols;
  out->cfg = cfg;
  out->layout = ANYQ_LAYOUT_ROWMAJOR;
  out->tile_k = 1;
  out->lut_store = ANYQ_STORE_FP16;
  out->scale_store = ANYQ_STORE_FP16;
  out->num_groups = group_count(cfg, rows, cols);
}

static void check_qt(const anyq_qtensor* qt) {
  if (!qt) fail(ANYQ_ERR_SHAPE, "null tensor");
  validate_config(qt->cfg, qt->rows, qt->cols);
  if (qt->num_groups != group_count(qt->cfg, qt->rows, qt->cols))
    fail(ANYQ_ERR_SHAPE, "tensor group count does not match its granularity");
  if (qt->cfg.codebook == ANYQ_CB_ANY && !qt->luts) fail(ANYQ_ERR_SHAPE, "AnyN tensor without LUTs");
  if (qt->layout == ANYQ_LAYOUT_KTILED && qt->tile_k < 1) fail(ANYQ_ERR_CONFIG, "tile_k must be >= 1");
}

// Uploads a host tensor; LUT null for fixed formats.
struct DevTensorArrays {
  DevBuf<uint8_t> codes;
  DevBuf<float> luts, alphas, betas;
  void upload(const anyq_qtensor* qt) {
    int64_t nb = qt->rows * packed_bpr(qt->cols, qt->cfg.bits);
    codes.alloc(nb);
    codes.upload(qt->codes, nb);
    if (qt->cfg.codebook == ANYQ_CB_ANY) {
      int64_t nl = qt->rows * (int64_t(1) << qt->cfg.bits);
      luts.alloc(nl);
      luts.upload(qt->luts, nl);
    }
    alphas.alloc(qt->num_groups);
    alphas.upload(qt->alphas, qt->num_groups);
    betas.alloc(qt->num_groups);
    betas.upload(qt->betas, qt->num_groups);
  }
};

}  // namespace anyq_b200

using namespace anyq_b200;

extern "C" {

const char* anyq_last_error(void) { return g_last_error.c_str(); }

uint64_t anyq_launch_count(void) { return g_launches.load(); }

void anyq_config_default(anyq_config* c) {
  std::memset(c, 0, sizeof *c);
  c->bits = 4;
  c->codebook = ANYQ_CB_INT;
  c->granularity = ANYQ_G_GROUP;
  c->group_size = 128;
  c->block_size = 1;
  c->init = ANYQ_INIT_KMPP;
  c->max_iters = 100;
  c->rel_tol = 1e-6f;
  c->restarts = 1;
  c->weighting = ANYQ_W_FULL;
}

int64_t anyq_packed_bytes_per_row(int64_t cols, int32_t bits) { return packed_bpr(cols, bits); }

int64_t anyq_num_groups(const anyq_config* cfg, int64_t rows, int64_t cols) {
  try {
    return group_count(*cfg, rows, cols);
  } catch (const Failure&) {
    return -1;
  }
}

int64_t anyq_lut_entries(const anyq_config* cfg) {
  return cfg->codebook == ANYQ_CB_ANY ? (int64_t(1) << cfg->bits) : 0;
}

anyq_status anyq_quantize_any(const float* w, int64_t rows, int64_t cols, const anyq_config* cfg,
                              const float* exj, int64_t row_offset, anyq_qtensor* out) {
  return guard([&] {
    if (cfg->codebook != ANYQ_CB_ANY) fail(ANYQ_ERR_CONFIG, "quantize_any requires the learned codebook");
    validate_config(*cfg, rows, cols);
    cudaStream_t s = 0;
    DevBuf<float> dw(rows * cols), dexj;
    dw.upload(w, rows * cols);
    if (exj) {
      dexj.alloc(cols);
      dexj.upload(exj, cols);
    }
    int64_t ng = group_count(*cfg, rows, cols);
    int64_t nb = rows * packed_bpr(cols, cfg->bits);
    int64_t nl = rows * (int64_t(1) << cfg->bits);
    DevBuf<uint8_t> packed(nb);
    DevBuf<float> luts(nl), alphas(ng), betas(ng);
    quantize_device(dw.p, rows, cols, *cfg, dexj.p, row_offset, packed.p, luts.p, alphas.p,
                    betas.p, s);
    check_stream_errors(s, "quantize_any");
    fill_header(out, rows, cols, *cfg);
    packed.download(out->codes, nb);
    luts.download(out->luts, nl);
    alphas.download(out->alphas, ng);
    betas.download(out->betas, ng);
  });
}

anyq_status anyq_quantize_fixed(const float* w, int64_t rows, int64_t cols, const anyq_config* cfg,
                                anyq_qtensor* out) {
  return guard([&] {
    if (cfg->codebook == ANYQ_CB_ANY) fail(ANYQ_ERR_CONFIG, "quantize_fixed handles fixed codebooks only");
    validate_config(*cfg, rows, cols);
    cudaStream_t s = 0;
    DevBuf<float> dw(rows * cols);
    dw.upload(w, rows * cols);
    int64_t ng = group_count(*cfg, rows, cols);
    int64_t nb = rows * packed_bpr(cols, cfg->bits);
    DevBuf<uint8_t> packed(nb);
    DevBuf<float> alphas(ng), betas(ng);
    quantize_device(dw.p, rows, cols, *cfg, nullptr, 0, packed.p, nullptr, alphas.p, betas.p, s);
    check_stream_errors(s, "quantize_fixed");
    fill_header(out, rows, cols, *cfg);
    packed.download(out->codes, nb);
    alphas.download(out->alphas, ng);
    betas.download(out->betas, ng);
  });
}

anyq_status anyq_dev_quantize_any(const float* w_dev, int64_t rows, int64_t cols,
                                  const anyq_config* cfg, const float* exj_dev, int64_t row_offset,
                                  uint8_t* codes_dev, float* luts_dev, float* alphas_dev,
                                  float* betas_dev, void* stream) {
  return guard([&] {
    if (cfg->codebook != ANYQ_CB_ANY) fail(ANYQ_ERR_CONFIG, "quantize_any requires the learned codebook");
    quantize_device(w_dev, rows, cols, *cfg, exj_dev, row_offset, codes_dev, luts_dev, alphas_dev,
                    betas_dev, (cudaStream_t)stream);
  });
}

anyq_status anyq_dev_stream_status(void* stream) {
  return guard([&] { check_stream_errors((cudaStream_t)stream, "stream-ordered call"); });
}

anyq_status anyq_pack_codes(const uint8_t* codes, int64_t rows, int64_t cols, int32_t bits,
                            uint8_t* packed) {
  return guard([&] {
    if (bits != 2 && bits != 3 && bits != 4 && bits != 8)
      fail(ANYQ_ERR_CONFIG, "pack_codes: bits must be one of {2,3,4,8}");
    int64_t nb = rows * packed_bpr(cols, bits);
    DevBuf<uint8_t> dc(rows * cols), dp(nb);
    DevBuf<int> err(1);
    err.zero();
    dc.upload(codes, rows * cols);
    if (rows * cols > 0) launch_pack(dc.p, rows, cols, bits, dp.p, err.p, 0);
    check_device_error(err.p, "pack_codes");
    dp.download(packed, nb);
  });
}

anyq_status anyq_unpack_codes(const uint8_t* packed, int64_t rows, int64_t cols, int32_t bits,
                              uint8_t* codes) {
  return guard([&] {
    if (bits != 2 && bits != 3 && bits != 4 && bits != 8)
      fail(ANYQ_ERR_CONFIG, "unpack_codes: bits must be one of {2,3,4,8}");
    int64_t nb = rows * packed_bpr(cols, bits);
    DevBuf<uint8_t> dp(nb), dc(rows * cols);
    dp.upload(packed, nb);
    if (rows * cols > 0) launch_unpack(dp.p, rows, cols, bits, dc.p, 0);
    dc.download(codes, rows * cols);
  });
}

anyq_status anyq_ktile_codes(const uint8_t* packed, int64_t rows, int64_t cols, int32_t bits,
                             int32_t tile_k, int32_t inverse, uint8_t* out) {
  return guard([&] {
    if (tile_k < 1) fail(ANYQ_ERR_CONFIG, "tile_k must be >= 1");
    int64_t nb = rows * packed_bpr(cols, bits);
    DevBuf<uint8_t> dp(nb), c0(rows * cols), c1(rows * cols), dq(nb);
    DevBuf<int> err(1);
    err.zero();
    dp.upload(packed, nb);
    launch_unpack(dp.p, rows, cols, bits, c0.p, 0);
    launch_ktile(c0.p, rows, cols, tile_k, inverse, c1.p, 0);
    launch_pack(c1.p, rows, cols, bits, dq.p, err.p, 0);
    check_device_error(err.p, "ktile");
    dq.download(out, nb);
  });
}

anyq_status anyq_narrow_inplace(anyq_qtensor* qt) {
  return guard([&] {
    check_qt(qt);
    DevBuf<int> err(1);
    err.zero();
    DevBuf<float> l, a(qt->num_groups), b(qt->num_groups);
    int64_t nl = 0;
    if (qt->cfg.codebook == ANYQ_CB_ANY) {
      nl = qt->rows * (int64_t(1) << qt->cfg.bits);
      l.alloc(nl);
      l.upload(qt->luts, nl);
      launch_narrow(l.p, nl, qt->lut_store, 0, err.p, 0);
    }
    a.upload(qt->alphas, qt->num_groups);
    b.upload(qt->betas, qt->num_groups);
    // reference order: alpha then beta per group; errors: overflow/non-finite (IoError /
    // NonFiniteError) dominate the alpha-underflow invariant.
    launch_narrow(a.p, qt->num_groups, qt->scale_store, 1, err.p, 0);
    launch_narrow(b.p, qt->num_groups, qt->scale_store, 0, err.p, 0);
    check_device_error(err.p, "narrowed");
    if (nl) l.download(qt->luts, nl);
    a.download(qt->alphas, qt->num_groups);
    b.download(qt->betas, qt->num_groups);
  });
}

anyq_status anyq_compute_scales(const float* w, int64_t rows, int64_t cols, const anyq_config* cfg,
                                float qmin, float qmax, float* alphas, float* betas) {
  return guard([&] {
    validate_config(*cfg, rows, cols);
    if (!(qmax > qmin)) fail(ANYQ_ERR_CONFIG, "qmax must exceed qmin");
    if (cfg->symmetric && !(qmax > 0)) fail(ANYQ_ERR_CONFIG, "symmetric scaling needs qmax > 0");
    const int64_t ng = group_count(*cfg, rows, cols);
    DevBuf<float> dw(rows * cols), da(ng), db(ng);
    DevBuf<int> err(1);
    err.zero();
    dw.upload(w, rows * cols);
    launch_check_finite(dw.p, rows * cols, err.p, ANYQ_ERR_NONFINITE, 0);
    ANYQ_CUDA(cudaDeviceSynchronize());
    check_device_error(err.p, "compute_scales");
    launch_scales(dw.p, rows, cols, *cfg, qmin, qmax, da.p, db.p, 0);
    da.download(alphas, ng);
    db.download(betas, ng);
  });
}

static anyq_status affine_host(const float* in, int64_t rows, int64_t cols, const anyq_config* cfg,
                               const float* alphas, const float* betas, int inverse, float* out) {
  return guard([&] {
    const int64_t ng = group_count(*cfg, rows, cols);
    DevBuf<float> din(rows * cols), dout(rows * cols), da(ng), db(ng);
    din.upload(in, rows * cols);
    da.upload(alphas, ng);
    db.upload(betas, ng);
    if (rows * cols > 0) launch_affine(din.p, rows, cols, *cfg, da.p, db.p, inverse, dout.p, 0);
    dout.download(out, rows * cols);
  });
}

anyq_status anyq_scale_weights(const float* w, int64_t rows, int64_t cols, const anyq_config* cfg,
                               const float* alphas, const float* betas, float* ws) {
  return affine_host(w, rows, cols, cfg, alphas, betas, 1, ws);
}

anyq_status anyq_dequantize_values(const float* v, int64_t rows, int64_t cols,
                                   const anyq_config* cfg, const float* alphas,
                                   const float* betas, float* out) {
  return affine_host(v, rows, cols, cfg, alphas, betas, 0, out);
}

// Stream ordered; a non-finite input (require_finite: NonFiniteError) is
// recorded in the stream's stage error words.
static void column_mean_abs_device(const float* x, int64_t m, int64_t k, float* exj, cudaStream_t s) {
  if (m < 1) fail(ANYQ_ERR_SHAPE, "need at least one input sample");
  if (k < 0) fail(ANYQ_ERR_SHAPE, "negative channel count");
  launch_col_mean_abs(x, m, k, exj, stream_ws(s).err + kErrFinite, s);
}

anyq_status anyq_column_mean_abs(const float* x, int64_t m, int64_t k, float* exj) {
  return guard([&] {
    if (m < 1) fail(ANYQ_ERR_SHAPE, "need at least one input sample");
    DevBuf<float> dx(m * k), de(k);
    dx.upload(x, m * k);
    column_mean_abs_device(dx.p, m, k, de.p, 0);
    check_stream_errors(0, "collect_stats inputs");
    de.download(exj, k);
  });
}

anyq_status anyq_dev_column_mean_abs(const float* x_dev, int64_t m, int64_t k, float* exj_dev,
                                     void* stream) {
  return guard([&] { column_mean_abs_device(x_dev, m, k, exj_dev, (cudaStream_t)stream); });
}

// dequantize(qt) into a device buffer (shared by dequantize and the eval metrics)
// (values_only: the scaled-domain table values, scaled_values pack.cpp:205-236)
static void dequant_to_device(const anyq_qtensor* qt, DevTensorArrays& t, float* w_dev,
                              bool values_only = false) {
  t.upload(qt);
  Table fixed{};
  if (qt->cfg.codebook != ANYQ_CB_ANY)
    fixed = effective_table(fixed_table(qt->cfg), qt->cfg.symmetric != 0);
  DevBuf<int> err(1);
  err.zero();
  launch_dequant(t.codes.p, qt->rows, qt->cols, qt->cfg.bits, qt->layout == ANYQ_LAYOUT_KTILED,
                 qt->tile_k, t.luts.p, fixed, qt->cfg, values_only ? nullptr : t.alphas.p,
                 t.betas.p, w_dev, err.p, 0);
  check_device_error(err.p, "dequantize");
}

static void sqdiff_sums(const float* a, const float* b, int64_t n, double out[2]) {
  DevBuf<double> part(2 * 592), sums(2);
  launch_sqdiff_sums(a, b, n, part.p, sums.p, 0);
  sums.download(out, 2);
}

anyq_status anyq_weight_error(const float* w, int64_t rows, int64_t cols, const anyq_qtensor* qt,
                              double* mse, double* rel) {
  return guard([&] {
    check_qt(qt);
    if (rows != qt->rows || cols != qt->cols) fail(ANYQ_ERR_SHAPE, "weight_error: shapes differ");
    const int64_t n = rows * cols;
    DevBuf<float> dw(n), dq(n);
    dw.upload(w, n);
    DevTensorArrays t;
    dequant_to_device(qt, t, dq.p);
    double s[2] = {0.0, 0.0};
    if (n > 0) sqdiff_sums(dw.p, dq.p, n, s);
    *mse = s[0] / ((double)rows * (double)cols);
    *rel = s[1] > 0 ? std::sqrt(s[0]) / std::sqrt(s[1]) : std::sqrt(s[0]);
  });
}

anyq_status anyq_output_error(const float* w, int64_t rows, int64_t cols, const anyq_qtensor* qt,
                              const float* x, int64_t m, int64_t x_cols, double* mse) {
  return guard([&] {
    check_qt(qt);
    if (rows != qt->rows || cols != qt->cols)
      fail(ANYQ_ERR_SHAPE, "output_error: weight shapes differ");
    if (x_cols != cols) fail(ANYQ_ERR_SHAPE, "output_error: activation width mismatch");
    DevBuf<float> dw(rows * cols), dq(rows * cols), dx(m * cols), y(m * rows), yq(m * rows);
    dw.upload(w, rows * cols);
    dx.upload(x, m * cols);
    DevTensorArrays t;
    dequant_to_device(qt, t, dq.p);
    double s[2] = {0.0, 0.0};
    if (m > 0 && rows > 0) {
      launch_gemm_dense(dx.p, m, dw.p, rows, cols, y.p, 0);   // gemm_dense(x, w)
      launch_gemm_dense(dx.p, m, dq.p, rows, cols, yq.p, 0);  // gemm_reference(x, qt)
      sqdiff_sums(yq.p, y.p, m * rows, s);
    }
    *mse = s[0] / ((double)m * (double)rows);
  });
}

anyq_status anyq_dequantize(const anyq_qtensor* qt, float* w_out) {
  return guard([&] {
    check_qt(qt);
    DevTensorArrays t;
    DevBuf<float> w(qt->rows * qt->cols);
    dequant_to_device(qt, t, w.p);
    w.download(w_out, qt->rows * qt->cols);
  });
}

anyq_status anyq_gemm_fused(const float* x, int64_t m, const anyq_qtensor* qt, int32_t plan_layout,
                            int32_t plan_tile_k, float* y) {
  return guard([&] {
    check_qt(qt);
    if (plan_layout != qt->layout || (qt->layout == ANYQ_LAYOUT_KTILED && plan_tile_k != qt->tile_k))
      fail(ANYQ_ERR_CONFIG, "gemm_fused: plan layout does not match tensor layout");
    if (m < 0) fail(ANYQ_ERR_SHAPE, "gemm_fused: negative m");
    if (m == 0) return;
    DevTensorArrays t;
    t.upload(qt);
    Table fixed{};
    if (qt->cfg.codebook != ANYQ_CB_ANY)
      fixed = effective_table(fixed_table(qt->cfg), qt->cfg.symmetric != 0);
    DevBuf<float> dx(m * qt->cols), dy(m * qt->rows);
    dx.upload(x, m * qt->cols);
    DevBuf<int> err(1);
    err.zero();
    launch_gemm_exact(dx.p, m, qt->cols, t.codes.p, qt->rows, qt->cfg.bits,
                      qt->layout == ANYQ_LAYOUT_KTILED, qt->tile_k, t.luts.p, fixed, qt->cfg,
                      t.alphas.p, t.betas.p, dy.p, err.p, 0);
    check_device_error(err.p, "gemm_fused");
    dy.download(y, m * qt->rows);
  });
}

anyq_status anyq_gemm_dense(const float* x, int64_t m, const float* w, int64_t n, int64_t k,
                            float* y) {
  return guard([&] {
    if (m <= 0 || n <= 0) return;
    DevBuf<float> dx(m * k), dw(n * k), dy(m * n);
    dx.upload(x, m * k);
    dw.upload(w, n * k);
    launch_gemm_dense(dx.p, m, dw.p, n, k, dy.p, 0);
    ANYQ_CUDA(cudaDeviceSynchronize());
    dy.download(y, m * n);
  });
}

// ---------------------------------------------------------------------------
// device-resident tensors + tensor-core GEMM (lutgemm.cu)
// ---------------------------------------------------------------------------
anyq_status anyq_dev_tensor_load(const char* path, anyq_dev_tensor** out) {
  return guard([&] { *out = reinterpret_cast<anyq_dev_tensor*>(load_device_tensor(path)); });
}

anyq_status anyq_dev_tensor_create(const anyq_qtensor* qt, anyq_dev_tensor** out) {
  return guard([&] {
    check_qt(qt);
    *out = reinterpret_cast<anyq_dev_tensor*>(lutgemm_create(qt));
  });
}

anyq_status anyq_dev_tensor_export(const anyq_dev_tensor* t, anyq_qtensor* out) {
  return guard([&] { lutgemm_export(reinterpret_cast<const LutTensor*>(t), out); });
}

void anyq_dev_tensor_config(const anyq_dev_tensor* t, anyq_config* out) {
  if (t && out) *out = reinterpret_cast<const LutTensor*>(t)->cfg;
}

void anyq_dev_tensor_destroy(anyq_dev_tensor* t) {
  lutgemm_destroy(reinterpret_cast<LutTensor*>(t));
}

int64_t anyq_dev_tensor_weight_bytes(const anyq_dev_tensor* t) {
  return reinterpret_cast<const LutTensor*>(t)->weight_bytes;
}
int64_t anyq_dev_tensor_rows(const anyq_dev_tensor* t) {
  return reinterpret_cast<const LutTensor*>(t)->rows;
}
int64_t anyq_dev_tensor_cols(const anyq_dev_tensor* t) {
  return reinterpret_cast<const LutTensor*>(t)->cols;
}

int32_t anyq_dev_gemm_auto_path(const anyq_dev_tensor* t, int64_t m) {
  // measured crossovers on B200 (profiles/round2_k1t.md,
  // profiles/round2_k2_stream_k.md): the CUDA-core GEMV at m = 1 (and m = 2
  // for fewer than 2 row blocks per SM); K1t (tcgen05 GEMV) for 3 <= m <= 4,
  // and up to m = 8 with at least 2 row blocks per SM, while its shared-memory
  // plan fits; K2 up to m = 128 on tall tensors (from m = 9, or m = 5 with
  // K >= 8192) and on long-K tensors it splits stream-K (from m = 8); the fused
  // dequant-to-shared-memory mma.sync kernel up to m = 32 (it splits K over
  // every SM, which wins on small N); dequant + cuBLAS above
  const LutTensor* lt = reinterpret_cast<const LutTensor*>(t);
  const bool many_rows = lt->RB >= 2 * lt->sms;
  // K2's cost is flat in m up to its 64-token tile, so it takes over below
  // m = 16 where the GEMV kernels' per-row cost has grown past it: from m = 9
  // on tall tensors (gate m = 12: 30.4 us against K1t's 32.0), from m = 5 on
  // tall tensors with K >= 8192 (70B gate m = 8: 85 against 110), from m = 8 on
  // long-K tensors it splits stream-K (70B q / down m = 12: 32.7 / 32.0 us
  // against 35.9 / 34.8)
  if (m >= 5 && m < 16 && lutgemm_k2_supports(lt, m) &&
      (many_rows ? (m >= 9 || lt->C >= 64) : (m >= 8 && lutgemm_k2_long_k(lt, m))))
    return ANYQ_PATH_K2;
  try {
    // K1t only when one x image fits: its K-sliced form (a grid-wide wait per
    // slice) measured slower than the fallbacks below (gate m = 9: 65 vs 31 us)
    if (m >= 2 && m <= 16 && (many_rows || (m >= 3 && m <= 4)) && lutgemv_tc_slices(lt, m) == 1)
      return ANYQ_PATH_GEMV_TC;
    if (lutgemv_fits(lt, m)) return ANYQ_PATH_GEMV;
  } catch (...) {
  }
  if (m <= 4) return ANYQ_PATH_TC;
  // K2 (tcgen05, bf16 dequantisation in shared memory) for 16 <= m <= 128 on
  // tensors with >= 2 row blocks per SM (its tiles are 128 rows; at m = 16 on
  // gate 29.7 us against the fused mma kernel's 32.5 us), and on long-K
  // tensors with few row tiles, split stream-K over every SM with >= 8 steps
  // per CTA (down, m = 32 / 64: 32.9 / 38.9 us against 43.2 / 57.1 us)
  if (m >= 16 && m <= 128 && (many_rows || lutgemm_k2_long_k(lt, m)) && lutgemm_k2_supports(lt, m))
    return ANYQ_PATH_K2;
  if (m <= 32 && lutmma_supports(lt, m)) return ANYQ_PATH_MMA;
  return m <= 8 ? ANYQ_PATH_TC : ANYQ_PATH_DEQUANT;
}

anyq_status anyq_dev_gemm_bf16_path(const anyq_dev_tensor* t, const void* x_bf16, int64_t m,
                                    void* y_bf16, float* y_f32, int32_t path, void* stream) {
  return guard([&] {
    const LutTensor* lt = reinterpret_cast<const LutTensor*>(t);
    if (path == ANYQ_PATH_AUTO) path = anyq_dev_gemm_auto_path(t, m);
    if (path == ANYQ_PATH_GEMV)
      lutgemv_run(lt, x_bf16, m, y_bf16, y_f32, (cudaStream_t)stream);
    else if (path == ANYQ_PATH_TC)
      lutgemm_run(lt, x_bf16, m, y_bf16, y_f32, (cudaStream_t)stream);
    else if (path == ANYQ_PATH_DEQUANT)
      dequant_gemm_run(lt, x_bf16, m, y_bf16, y_f32, (cudaStream_t)stream);
    else if (path == ANYQ_PATH_MMA)
      lutmma_run(lt, x_bf16, m, y_bf16, y_f32, (cudaStream_t)stream);
    else if (path == ANYQ_PATH_GEMV_TC)
      lutgemv_tc_run(lt, x_bf16, m, y_bf16, y_f32, (cudaStream_t)stream);
    else if (path == ANYQ_PATH_K2)
      lutgemm_k2_run(lt, x_bf16, m, y_bf16, y_f32, (cudaStream_t)stream);
    else
      fail(ANYQ_ERR_CONFIG, "unknown GEMM path");
  });
}

anyq_status anyq_dev_gemm_chain(int32_t n, const anyq_dev_tensor* const* t,
                                const void* const* x_bf16, void* const* y_bf16,
                                float* const* y_f32, const int32_t* wait_prev, int64_t m,
                                void* stream) {
  return guard([&] {
    if (n < 1 || n > 8 || !t || !x_bf16 || !y_bf16) fail(ANYQ_ERR_SHAPE, "gemm chain: bad arguments");
    // "after every earlier problem" == after problem i-1 (problems are released in order)
    int32_t deps[8];
    for (int i = 0; i < n; ++i) deps[i] = (wait_prev && i > 0 && wait_prev[i]) ? i - 1 : -1;
    lutgemv_chain_run_auto(n, reinterpret_cast<const LutTensor* const*>(t), x_bf16, y_bf16, y_f32, deps,
                           m, (cudaStream_t)stream);
  });
}

anyq_status anyq_dev_gemm_chain_deps(int32_t n, const anyq_dev_tensor* const* t,
                                     const void* const* x_bf16, void* const* y_bf16,
                                     float* const* y_f32, const int32_t* deps, int64_t m,
                                     void* stream) {
  return guard([&] {
    if (n < 1 || n > 8 || !t || !x_bf16 || !y_bf16) fail(ANYQ_ERR_SHAPE, "gemm chain: bad arguments");
    lutgemv_chain_run_auto(n, reinterpret_cast<const LutTensor* const*>(t), x_bf16, y_bf16, y_f32, deps,
                           m, (cudaStream_t)stream);
  });
}

anyq_status anyq_dev_gemm_chain_path(int32_t n, const anyq_dev_tensor* const* t,
                                     const void* const* x_bf16, void* const* y_bf16,
                                     float* const* y_f32, const int32_t* deps, int64_t m,
                                     int32_t path, void* stream) {
  return guard([&] {
    if (n < 1 || n > 8 || !t || !x_bf16 || !y_bf16) fail(ANYQ_ERR_SHAPE, "gemm chain: bad arguments");
    const auto* ts = reinterpret_cast<const LutTensor* const*>(t);
    if (path == ANYQ_PATH_AUTO)
      lutgemv_chain_run_auto(n, ts, x_bf16, y_bf16, y_f32, deps, m, (cudaStream_t)stream);
    else if (path == ANYQ_PATH_GEMV)
      lutgemv_chain_run(n, ts, x_bf16, y_bf16, y_f32, deps, m, (cudaStream_t)stream);
    else if (path == ANYQ_PATH_GEMV_TC)
      lutgemv_tc_chain_run(n, ts, x_bf16, y_bf16, y_f32, deps, m, (cudaStream_t)stream);
    else
      fail(ANYQ_ERR_CONFIG, "gemm chain: path must be AUTO, GEMV or GEMV_TC");
  });
}

anyq_status anyq_dev_gemm_allgather(const anyq_dev_tensor* shard, const void* x_bf16, int64_t m,
                                    const anyq_tp_peers* tp, void* stream) {
  return guard([&] {
    lutgemv_tp_run(reinterpret_cast<const LutTensor*>(shard), x_bf16, m, tp, (cudaStream_t)stream);
  });
}

anyq_status anyq_dev_tp_wait(const anyq_dev_tensor* shard, const anyq_tp_peers* tp, int32_t epoch,
                             void* stream) {
  return guard([&] {
    if (epoch < 1) fail(ANYQ_ERR_SHAPE, "tp wait: epoch counts calls from 1");
    // every rank's launch has one CTA per SM of its (identical) device
    lutgemv_tp_wait(tp, epoch * lutgemv_tp_ctas(reinterpret_cast<const LutTensor*>(shard)), (cudaStream_t)stream);
  });
}

anyq_status anyq_ipc_handle(const void* dev_ptr, uint8_t handle[64]) {
  return guard([&] {
    cudaIpcMemHandle_t h;
    static_assert(sizeof h == 64, "CUDA IPC handles are 64 bytes");
    ANYQ_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    std::memcpy(handle, &h, 64);
  });
}

anyq_status anyq_ipc_open(const uint8_t handle[64], void** dev_ptr) {
  return guard([&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    ANYQ_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

anyq_status anyq_ipc_close(void* dev_ptr) {
  return guard([&] { ANYQ_CUDA(cudaIpcCloseMemHandle(dev_ptr)); });
}

anyq_status anyq_dev_gemm_bf16(const anyq_dev_tensor* t, const void* x_bf16, int64_t m,
                               void* y_bf16, float* y_f32, void* stream) {
  return anyq_dev_gemm_bf16_path(t, x_bf16, m, y_bf16, y_f32, ANYQ_PATH_AUTO, stream);
}

// ---------------------------------------------------------------------------
// The per-row learner API, codebooks, scalar narrowing and accounting
// (learner.hpp:45-68, codebooks.hpp:27-50, pack.hpp:57-96): the entry points
// the C++ drop-in (host/anyq_host.cpp) serves the rest of the reference API with.
// ---------------------------------------------------------------------------

anyq_status anyq_kmeans_problems(const float* samples, const float* weights, int64_t rows, int64_t n,
                                 int32_t k, const anyq_config* cfg, int32_t mode,
                                 const uint64_t* rng_key, uint64_t* rng_counter, double* centroids,
                                 uint8_t* assignments, double* loss, int32_t* iters) {
  return guard([&] {
    if (mode < 0 || mode > 2) fail(ANYQ_ERR_CONFIG, "k-means mode must be 0, 1 or 2");
    if (rows < 1) return;
    // KmProblem::validate (learner.cpp:11-23), then the k checks, in order
    if (n < 1) fail(ANYQ_ERR_SHAPE, "KmProblem: empty problem");
    for (int64_t r = 0; r < rows; ++r) {
      const float* w = weights + r * n;
      bool any_positive = false;
      for (int64_t i = 0; i < n; ++i) {
        if (!(w[i] >= 0) || !std::isfinite(w[i])) fail(ANYQ_ERR_STATS, "KmProblem: weights must be >= 0");
        any_positive |= w[i] > 0;
      }
      if (!any_positive) fail(ANYQ_ERR_STATS, "KmProblem: all sample weights are zero");
      for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(samples[r * n + i])) fail(ANYQ_ERR_NONFINITE, "KmProblem: non-finite sample");
    }
    if (k < 1) fail(ANYQ_ERR_CONFIG, "k must be >= 1");
    if (mode != 2 && k > 256) fail(ANYQ_ERR_CONFIG, "k must fit an 8-bit code");
    if (mode == 2 && k > 256) fail(ANYQ_ERR_CONFIG, "k-means++ seeding supports k <= 256");
    if (mode != 2 && cfg->init == ANYQ_INIT_NF4 && k != 16)
      fail(ANYQ_ERR_CONFIG, "nf4 seeding needs exactly 16 centroids");
    if (mode != 2 && (cfg->max_iters < 1 || cfg->restarts < 1))
      fail(ANYQ_ERR_CONFIG, "learner needs max_iters >= 1 and restarts >= 1");
    cudaStream_t s = 0;
    DevBuf<float> dx(rows * n), dw(rows * n), dlut(mode == 0 ? rows * k : 0);
    DevBuf<uint64_t> dkey(rows), dctr(rows);
    DevBuf<double> dcen(rows * k), dloss(rows);
    DevBuf<uint8_t> dasg(mode != 2 ? rows * n : 0);
    DevBuf<int> diters(rows);
    dx.upload(samples, rows * n);
    dw.upload(weights, rows * n);
    dkey.upload(rng_key, rows);
    dctr.upload(rng_counter, rows);
    int* err = stream_ws(s).err;
    launch_kmeans_problems(dx.p, dw.p, rows, n, k, *cfg, mode, dkey.p, dctr.p, dcen.p, dasg.p,
                           dloss.p, diters.p, dlut.p, dasg.p, err + kErrLearn, s);
    check_stream_errors(s, "weighted_kmeans");
    dctr.download(rng_counter, rows);
    if (mode == 0) {  // learn_row_lut: sorted LUT (as float) + rank codes + loss
      std::vector<float> lut(rows * k);
      dlut.download(lut.data(), rows * k);
      for (int64_t i = 0; i < rows * k; ++i) centroids[i] = lut[i];
      dasg.download(assignments, rows * n);
      dloss.download(loss, rows);
      return;
    }
    dcen.download(centroids, rows * k);
    if (mode == 1) {
      dasg.download(assignments, rows * n);
      dloss.download(loss, rows);
      std::vector<int> it(rows);
      diters.download(it.data(), rows);
      for (int64_t r = 0; r < rows; ++r) iters[r] = it[r];
    }
  });
}

anyq_status anyq_build_sample_weights(const anyq_config* cfg, int64_t rows, int64_t cols,
                                      const float* alphas, int64_t num_groups, int64_t row,
                                      const float* stats, int64_t stats_len, int32_t weighting,
                                      float* out) {
  return guard([&] {
    // the stats checks of learner.cpp:27-34, in order
    if (stats) {
      if (stats_len != cols)
        fail(ANYQ_ERR_STATS, "sample weights: stats length " + std::to_string(stats_len) +
                                 " does not match row length " + std::to_string(cols));
      for (int64_t j = 0; j < cols; ++j)
        if (!(stats[j] >= 0) || !std::isfinite(stats[j]))
          fail(ANYQ_ERR_STATS, "sample weights: negative or non-finite stats entry");
    }
    if (weighting < 0 || weighting > 2) fail(ANYQ_ERR_CONFIG, "unknown weighting mode");
    if (cols < 1) return;
    if (row < 0 || row >= rows) fail(ANYQ_ERR_SHAPE, "sample weights: row out of range");
    if (weighting == ANYQ_W_FULL && num_groups != group_count(*cfg, rows, cols))
      fail(ANYQ_ERR_SHAPE, "sample weights: scale set does not match its granularity");
    DevBuf<float> da(weighting == ANYQ_W_FULL ? num_groups : 0), ds(stats ? cols : 0), dout(cols);
    if (weighting == ANYQ_W_FULL) da.upload(alphas, num_groups);
    if (stats) ds.upload(stats, cols);
    launch_sample_weights(*cfg, row, cols, da.p, ds.p, weighting, dout.p, 0);
    dout.download(out, cols);
  });
}

anyq_status anyq_round_to_table(const float* ws, int64_t rows, int64_t cols, const float* table,
                                int32_t n, uint8_t* codes) {
  return guard([&] {
    if (n < 1 || n > 256) fail(ANYQ_ERR_CONFIG, "codebook must hold 1..256 values");
    const int64_t total = rows * cols;
    if (total <= 0) return;
    Table t{};
    t.n = n;
    std::memcpy(t.v, table, sizeof(float) * n);
    DevBuf<float> dws(total);
    DevBuf<uint8_t> dc(total);
    dws.upload(ws, total);
    launch_check_finite(dws.p, total, stream_ws(0).err + kErrFinite, ANYQ_ERR_NONFINITE, 0);
    check_stream_errors(0, "round_to_codebook");  // require_finite (codebooks.cpp:76)
    launch_round(dws.p, total, t, dc.p, 0);
    dc.download(codes, total);
  });
}

anyq_status anyq_scaled_values(const anyq_qtensor* qt, float* out) {
  return guard([&] {
    check_qt(qt);
    DevTensorArrays t;
    DevBuf<float> w(qt->rows * qt->cols);
    dequant_to_device(qt, t, w.p, true);
    w.download(out, qt->rows * qt->cols);
  });
}

anyq_status anyq_fixed_table(int32_t codebook, int32_t bits, int32_t shifted, float* values,
                             int32_t* n) {
  return host_only([&] {
    if (codebook == ANYQ_CB_INT && bits != 2 && bits != 3 && bits != 4 && bits != 8)
      fail(ANYQ_ERR_CONFIG, "int_grid: bits must be one of {2,3,4,8}");
    anyq_config c;
    anyq_config_default(&c);
    c.codebook = codebook;
    c.bits = bits;
    c.int_range_shifted = shifted;
    const Table t = fixed_table(c);
    std::memcpy(values, t.v, sizeof(float) * t.n);
    *n = t.n;
  });
}

anyq_status anyq_f32_to_f16(float f, uint16_t* out) {
  return host_only([&] {
    int st = ANYQ_OK;
    const uint16_t h = f32_to_f16_exact(f, &st);
    if (st == ANYQ_ERR_NONFINITE) fail(ANYQ_ERR_NONFINITE, "fp16 narrowing: non-finite value");
    if (st != ANYQ_OK) fail((anyq_status)st, "fp16 narrowing: value overflows to infinity");
    *out = h;
  });
}
float anyq_f16_to_f32(uint16_t h) { return f16_to_f32_exact(h); }
anyq_status anyq_f32_to_bf16(float f, uint16_t* out) {
  return host_only([&] {
    int st = ANYQ_OK;
    const uint16_t h = f32_to_bf16_exact(f, &st);
    if (st == ANYQ_ERR_NONFINITE) fail(ANYQ_ERR_NONFINITE, "bf16 narrowing: non-finite value");
    if (st != ANYQ_OK) fail((anyq_status)st, "bf16 narrowing: value overflows to infinity");
    *out = h;
  });
}
float anyq_bf16_to_f32(uint16_t h) { return bf16_to_f32_exact(h); }

namespace {
// rethrow a nested C-ABI call's failure (its message is the last error)
void check_status(anyq_status st) {
  if (st != ANYQ_OK) fail(st, anyq_last_error());
}
}  // namespace

anyq_status anyq_eval_activations(int64_t rows, int64_t cols, const float* exj, uint64_t seed,
                                  float* out) {
  return host_only([&] {
    if (rows < 0 || cols < 0) fail(ANYQ_ERR_SHAPE, "eval_activations: negative shape");
    constexpr double kSqrtHalfPi = 1.2533141373155003;  // E|N(0, s)| = s sqrt(2/pi)
    for (int64_t r = 0; r < rows; ++r) {
      Rng rng = Rng::for_row(seed, r);
      for (int64_t j = 0; j < cols; ++j) {
        const double sigma = exj ? (double)exj[j] * kSqrtHalfPi : 1.0;
        // core.hpp:183-187 Box-Muller
        const double u1 = (double)((rng.next_u64() >> 11) + 1) * 0x1.0p-53;
        const double u2 = rng.next_double();
        const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
        out[r * cols + j] = (float)(sigma * g);
      }
    }
  });
}

anyq_status anyq_compare_formats(const float* w, int64_t rows, int64_t cols, const char* formats,
                                 const anyq_config* base, const float* exj, int64_t eval_rows,
                                 uint64_t eval_seed, double* out, int32_t* n_formats) {
  return guard([&] {
    if (!w || !formats || !base || !out) fail(ANYQ_ERR_SHAPE, "compare_formats: null argument");
    struct Fmt {
      const char* name;
      int32_t codebook, bits;
    };
    static const Fmt kFmts[] = {{"int2", ANYQ_CB_INT, 2}, {"int3", ANYQ_CB_INT, 3}, {"int4", ANYQ_CB_INT, 4},
                                {"int8", ANYQ_CB_INT, 8}, {"fp4", ANYQ_CB_FP4, 4},  {"nf4", ANYQ_CB_NF4, 4},
                                {"any2", ANYQ_CB_ANY, 2}, {"any3", ANYQ_CB_ANY, 3}, {"any4", ANYQ_CB_ANY, 4},
                                {"any8", ANYQ_CB_ANY, 8}};
    std::vector<std::string> names;
    {
      std::string cur;
      for (const char* c = formats;; ++c) {
        if (*c == ',' || *c == 0) {
          names.push_back(cur);
          cur.clear();
          if (!*c) break;
        } else {
          cur += *c;
        }
      }
    }
    // eval.cpp:68-70: the stats lookup happens before the activations are drawn
    std::vector<float> x((size_t)eval_rows * cols);
    check_status(anyq_eval_activations(eval_rows, cols, exj, eval_seed, x.data()));
    int32_t nf = 0;
    for (const std::string& nm : names) {
      const Fmt* f = nullptr;
      for (const Fmt& e : kFmts)
        if (nm == e.name) f = &e;
      if (!f) fail(ANYQ_ERR_CONFIG, "unknown format '" + nm + "'");
      anyq_config c = *base;
      c.codebook = f->codebook;
      c.bits = f->bits;
      validate_config(c, rows, cols);
      const int64_t ng = group_count(c, rows, cols);
      std::vector<uint8_t> codes((size_t)(rows * packed_bpr(cols, c.bits)));
      std::vector<float> luts(c.codebook == ANYQ_CB_ANY ? (size_t)rows << c.bits : 0), al(ng), be(ng);
      anyq_qtensor qt{};
      qt.rows = rows;
      qt.cols = cols;
      qt.cfg = c;
      qt.codes = codes.data();
      qt.luts = luts.empty() ? nullptr : luts.data();
      qt.alphas = al.data();
      qt.betas = be.data();
      qt.num_groups = ng;
      // quantize.cpp:25-32 (quantize): learned formats see the module's stats
      check_status(c.codebook == ANYQ_CB_ANY ? anyq_quantize_any(w, rows, cols, &c, exj, 0, &qt)
                                             : anyq_quantize_fixed(w, rows, cols, &c, &qt));
      double* o = out + 4 * nf;
      check_status(anyq_weight_error(w, rows, cols, &qt, &o[0], &o[1]));
      check_status(anyq_output_error(w, rows, cols, &qt, x.data(), eval_rows, cols, &o[2]));
      check_status(anyq_storage_bits_per_entry(&c, rows, cols, &o[3]));
      ++nf;
    }
    if (n_formats) *n_formats = nf;
  });
}

anyq_status anyq_storage_bits_per_entry(const anyq_config* cfg, int64_t rows, int64_t cols,
                                        double* bits) {
  return host_only([&] {
    validate_config(*cfg, rows, cols);
    const double entries = (double)rows * (double)cols;
    const double groups = (double)group_count(*cfg, rows, cols);
    // n code bits + 2 x 16-bit (scale, offset) per group + 2^n x 16-bit LUT per row for AnyN
    const double meta = 32.0 * groups +
                        (cfg->codebook == ANYQ_CB_ANY ? 16.0 * (double)rows * (double)(1 << cfg->bits) : 0.0);
    *bits = (double)cfg->bits + meta / entries;
  });
}

// qgemm.cpp:134-207 bench's timing loop, on the device: operands resident in
// HBM, one warm-up run, then `repeats` runs each bracketed by CUDA events.
anyq_status anyq_bench_gemm(int32_t kind, const anyq_qtensor* qt, const float* w, int64_t n,
                            int64_t k, const float* x, int64_t m, int32_t repeats, double* ns) {
  return guard([&] {
    if (repeats < 1) fail(ANYQ_ERR_CONFIG, "bench: repeats must be >= 1");
    if (m < 1 || n < 1 || k < 1) fail(ANYQ_ERR_SHAPE, "bench: empty GEMM");
    if (kind != 0) {
      check_qt(qt);
      if (qt->rows != n || qt->cols != k) fail(ANYQ_ERR_SHAPE, "bench: tensor shape mismatch");
    }
    cudaStream_t s = 0;
    DevBuf<float> dx(m * k), dy(m * n), dw(kind == 0 ? n * k : 0);
    dx.upload(x, m * k);
    DevTensorArrays t;
    Table fixed{};
    DevBuf<int> err(1);
    err.zero();
    LutTensor* lt = nullptr;
    DevBuf<uint16_t> xb(kind == 2 ? m * k : 0), yb(kind == 2 ? m * n : 0);
    if (kind == 0) {
      dw.upload(w, n * k);
    } else if (kind == 1) {
      t.upload(qt);
      if (qt->cfg.codebook != ANYQ_CB_ANY)
        fixed = effective_table(fixed_table(qt->cfg), qt->cfg.symmetric != 0);
    } else if (kind == 2) {
      lt = lutgemm_create(qt);
      std::vector<uint16_t> hb(m * k);
      int st = ANYQ_OK;
      for (int64_t i = 0; i < m * k; ++i) hb[i] = f32_to_bf16_exact(x[i], &st);
      xb.upload(hb.data(), m * k);
    } else {
      fail(ANYQ_ERR_CONFIG, "bench: kind must be 0 (dense), 1 (exact fused) or 2 (A16W4)");
    }
    struct Guard {
      LutTensor* t;
      ~Guard() { lutgemm_destroy(t); }
    } g{lt};
    auto run = [&] {
      if (kind == 0) {
        launch_gemm_dense(dx.p, m, dw.p, n, k, dy.p, s);
      } else if (kind == 1) {
        launch_gemm_exact(dx.p, m, qt->cols, t.codes.p, qt->rows, qt->cfg.bits,
                          qt->layout == ANYQ_LAYOUT_KTILED, qt->tile_k, t.luts.p, fixed, qt->cfg,
                          t.alphas.p, t.betas.p, dy.p, err.p, s);
      } else {
        const int path = anyq_dev_gemm_auto_path(reinterpret_cast<anyq_dev_tensor*>(lt), m);
        if (path == ANYQ_PATH_GEMV) lutgemv_run(lt, xb.p, m, yb.p, dy.p, s);
        else if (path == ANYQ_PATH_GEMV_TC) lutgemv_tc_run(lt, xb.p, m, yb.p, dy.p, s);
        else if (path == ANYQ_PATH_K2) lutgemm_k2_run(lt, xb.p, m, yb.p, dy.p, s);
        else if (path == ANYQ_PATH_MMA) lutmma_run(lt, xb.p, m, yb.p, dy.p, s);
        else if (path == ANYQ_PATH_TC) lutgemm_run(lt, xb.p, m, yb.p, dy.p, s);
        else dequant_gemm_run(lt, xb.p, m, yb.p, dy.p, s);
      }
    };
    run();
    check_device_error(err.p, "bench");
    cudaEvent_t e0, e1;
    ANYQ_CUDA(cudaEventCreate(&e0));
    ANYQ_CUDA(cudaEventCreate(&e1));
    for (int r = 0; r < repeats; ++r) {
      ANYQ_CUDA(cudaEventRecord(e0, s));
      run();
      ANYQ_CUDA(cudaEventRecord(e1, s));
      ANYQ_CUDA(cudaEventSynchronize(e1));
      float ms = 0.0f;
      ANYQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      ns[r] = (double)ms * 1e6;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

// Debug hook (not part of the reference interface): record a per-CTA
// globaltimer timeline of the tensor-core GEMM into dev ([ncta][16] int64).
void anyq_debug_set_trace(long long* dev) { lutgemm_set_trace(dev); }
void anyq_debug_set_gemv_trace(long long* dev) { lutgemv_set_trace(dev); }

}  // extern "C"
