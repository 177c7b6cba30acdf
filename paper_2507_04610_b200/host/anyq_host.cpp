// C++ host layer of the drop-in: the reference's hot-path API (declared in
// proj/include/anyq/{learner,quantize,pack,qgemm}.hpp, compiled against those
// headers in place) implemented on the B200 library through its C-ABI
// (include/anyq_b200.h). Same signatures, value semantics and exception
// classes as the reference; every computation runs on the GPU — a host with no
// device gets anyq::Error from the first call, never a CPU result.
//
//   quantize_any    learner.hpp:74     quantize_fixed  quantize.hpp:17
//   pack_codes      pack.hpp:50        unpack_codes    pack.hpp:51
//   narrowed        pack.hpp:68        to_ktiled / from_ktiled  pack.hpp:86-87
//   dequantize(qt)  pack.hpp:98        gemm_dense / gemm_reference / gemm_fused
//                                                      qgemm.hpp:28-37
//   compute_scales  scaling.hpp:52     scale_weights   scaling.hpp:56
//   dequantize(values, s)  scaling.hpp:60
//   write_file / read_file  pack.hpp (pack.cpp:293-471, ANYQ v1 files)
//
// Linking this object before the reference objects (tests/reftests/Makefile
// weakens the latter) swaps the hot path of an unmodified reference build —
// including its CLI and own unit tests — onto the GPU.
#include <cstring>
#include <string>
#include <vector>

#include "anyq/learner.hpp"
#include "anyq/pack.hpp"
#include "anyq/qgemm.hpp"
#include "anyq/quantize.hpp"
#include "anyq/scaling.hpp"
#include "anyq_b200.h"

namespace anyq {

namespace {

[[noreturn]] void rethrow(anyq_status s) {
  const std::string m = anyq_last_error();
  switch (s) {
    case ANYQ_ERR_SHAPE: throw ShapeError(m);
    case ANYQ_ERR_CONFIG: throw ConfigError(m);
    case ANYQ_ERR_CODE_RANGE: throw CodeRangeError(m);
    case ANYQ_ERR_NONFINITE: throw NonFiniteError(m);
    case ANYQ_ERR_STATS: throw StatsError(m);
    case ANYQ_ERR_IO: throw IoError(m);
    case ANYQ_ERR_MAGIC: throw MagicError(m);
    case ANYQ_ERR_VERSION: throw VersionError(m);
    case ANYQ_ERR_TRUNCATED: throw TruncatedError(m);
    case ANYQ_ERR_INVARIANT: throw InvariantError(m);
    default: throw Error("B200 library: " + m);
  }
}

void check(anyq_status s) {
  if (s != ANYQ_OK) rethrow(s);
}

anyq_config to_c(const QuantConfig& q) {
  anyq_config c;
  anyq_config_default(&c);
  c.bits = q.bits;
  c.codebook = static_cast<int32_t>(q.codebook);
  c.granularity = static_cast<int32_t>(q.granularity);
  c.group_size = q.group_size;
  c.block_size = q.block_size;
  c.symmetric = q.symmetric ? 1 : 0;
  c.int_range_shifted = q.int_range_shifted ? 1 : 0;
  c.init = static_cast<int32_t>(q.learner.init);
  c.max_iters = q.learner.max_iters;
  c.rel_tol = q.learner.rel_tol;
  c.restarts = q.learner.restarts;
  c.weighting = static_cast<int32_t>(q.learner.weighting);
  c.check_invariants = q.learner.check_invariants ? 1 : 0;
  c.seed = q.seed;
  return c;
}

// Contiguous row-major copy of an Eigen view (the C-ABI takes plain pointers).
std::vector<float> flat(const Eigen::Ref<const Matf>& m) {
  std::vector<float> v(static_cast<size_t>(m.rows() * m.cols()));
  for (Index i = 0; i < m.rows(); ++i)
    for (Index j = 0; j < m.cols(); ++j) v[static_cast<size_t>(i * m.cols() + j)] = m(i, j);
  return v;
}

// A C view of a QuantizedTensor; the C-ABI reads (or, for in-place calls,
// writes) the tensor's own vectors.
struct CView {
  anyq_qtensor t;
  explicit CView(const QuantizedTensor& qt) {
    std::memset(&t, 0, sizeof t);
    t.rows = qt.rows;
    t.cols = qt.cols;
    t.cfg = to_c(qt.cfg);
    t.layout = static_cast<int32_t>(qt.layout);
    t.tile_k = qt.tile_k;
    t.lut_store = static_cast<int32_t>(qt.lut_store);
    t.scale_store = static_cast<int32_t>(qt.scale_store);
    t.codes = const_cast<uint8_t*>(qt.codes.data());
    t.luts = qt.luts.empty() ? nullptr : const_cast<float*>(qt.luts.data());
    t.alphas = const_cast<float*>(qt.scales.alphas.data());
    t.betas = const_cast<float*>(qt.scales.betas.data());
    t.num_groups = qt.scales.num_groups();
  }
};

ScaleSet empty_scales(const QuantConfig& cfg, Index rows, Index cols, int64_t ng) {
  ScaleSet s;
  s.granularity = cfg.granularity;
  s.rows = rows;
  s.cols = cols;
  s.group_size = cfg.granularity == Granularity::Groupwise ? cfg.group_size : 0;
  s.block_size = cfg.granularity == Granularity::Blockwise ? cfg.block_size : 0;
  s.symmetric = cfg.symmetric;
  s.alphas = Vecf::Zero(static_cast<Index>(ng));
  s.betas = Vecf::Zero(static_cast<Index>(ng));
  return s;
}

QuantizedTensor quantize_impl(const Eigen::Ref<const Matf>& w, const QuantConfig& cfg,
                              const Vecf* exj) {
  const anyq_config c = to_c(cfg);
  const Index rows = w.rows(), cols = w.cols();
  if (exj && exj->size() != cols)
    throw StatsError("activation statistics length does not match the tensor's columns");
  QuantizedTensor qt;
  qt.rows = rows;
  qt.cols = cols;
  qt.cfg = cfg;
  const int64_t ng = anyq_num_groups(&c, rows, cols);
  if (ng < 0) throw ConfigError("unknown granularity");
  qt.codes.assign(static_cast<size_t>(rows * anyq_packed_bytes_per_row(cols, cfg.bits)), 0);
  if (cfg.codebook == CodebookKind::AnyN)
    qt.luts.assign(static_cast<size_t>(rows * anyq_lut_entries(&c)), 0.0f);
  qt.scales = empty_scales(cfg, rows, cols, ng);
  const std::vector<float> wf = flat(w);
  CView v(qt);
  if (cfg.codebook == CodebookKind::AnyN)
    check(anyq_quantize_any(wf.data(), rows, cols, &c, exj ? exj->data() : nullptr, 0, &v.t));
  else
    check(anyq_quantize_fixed(wf.data(), rows, cols, &c, &v.t));
  return qt;
}

// The group map of a ScaleSet as a C config (granularity, group/block sizes).
anyq_config group_cfg(const ScaleSet& s) {
  anyq_config c;
  anyq_config_default(&c);
  c.granularity = static_cast<int32_t>(s.granularity);
  if (s.group_size > 0) c.group_size = s.group_size;
  if (s.block_size > 0) c.block_size = s.block_size;
  c.symmetric = s.symmetric ? 1 : 0;
  return c;
}

Matf affine(const Eigen::Ref<const Matf>& in, const ScaleSet& s, bool inverse) {
  const anyq_config c = group_cfg(s);
  const std::vector<float> f = flat(in);
  Matf out(in.rows(), in.cols());
  if (inverse)
    check(anyq_scale_weights(f.data(), in.rows(), in.cols(), &c, s.alphas.data(), s.betas.data(),
                             out.data()));
  else
    check(anyq_dequantize_values(f.data(), in.rows(), in.cols(), &c, s.alphas.data(),
                                 s.betas.data(), out.data()));
  return out;
}

}  // namespace

ScaleSet compute_scales(const Eigen::Ref<const Matf>& w, const QuantConfig& cfg, Real qmin,
                        Real qmax) {
  const anyq_config c = to_c(cfg);
  const int64_t ng = anyq_num_groups(&c, w.rows(), w.cols());
  if (ng < 0) throw ConfigError("unknown granularity");
  ScaleSet s = empty_scales(cfg, w.rows(), w.cols(), ng);
  s.group_size = cfg.group_size;  // compute_scales records both sizes (scaling.cpp:40-41)
  s.block_size = cfg.block_size;
  const std::vector<float> f = flat(w);
  check(anyq_compute_scales(f.data(), w.rows(), w.cols(), &c, qmin, qmax, s.alphas.data(),
                            s.betas.data()));
  return s;
}

Matf scale_weights(const Eigen::Ref<const Matf>& w, const ScaleSet& s) {
  if (w.rows() != s.rows || w.cols() != s.cols)
    throw ShapeError("scale_weights: matrix shape does not match scale set");
  return affine(w, s, true);
}

Matf dequantize(const Eigen::Ref<const Matf>& values, const ScaleSet& s) {
  if (values.rows() != s.rows || values.cols() != s.cols)
    throw ShapeError("dequantize: matrix shape does not match scale set");
  return affine(values, s, false);
}

QuantizedTensor quantize_any(const Eigen::Ref<const Matf>& w, const QuantConfig& cfg,
                             const Vecf* exj, int /*threads: the GPU ignores it; results are
                                                     identical for any count*/) {
  if (cfg.codebook != CodebookKind::AnyN)
    throw ConfigError("quantize_any requires the learned codebook");
  return quantize_impl(w, cfg, exj);
}

QuantizedTensor quantize_fixed(const Eigen::Ref<const Matf>& w, const QuantConfig& cfg) {
  if (cfg.codebook == CodebookKind::AnyN)
    throw ConfigError("quantize_fixed handles fixed codebooks only");
  return quantize_impl(w, cfg, nullptr);
}

std::vector<uint8_t> pack_codes(const CodeMat& codes, int bits) {
  std::vector<uint8_t> out(static_cast<size_t>(codes.rows() * packed_bytes_per_row(codes.cols(), bits)));
  std::vector<uint8_t> in(static_cast<size_t>(codes.rows() * codes.cols()));
  for (Index i = 0; i < codes.rows(); ++i)
    for (Index j = 0; j < codes.cols(); ++j) in[static_cast<size_t>(i * codes.cols() + j)] = codes(i, j);
  check(anyq_pack_codes(in.data(), codes.rows(), codes.cols(), bits, out.data()));
  return out;
}

CodeMat unpack_codes(std::span<const uint8_t> packed, Index rows, Index cols, int bits) {
  if (static_cast<Index>(packed.size()) < rows * packed_bytes_per_row(cols, bits))
    throw ShapeError("unpack_codes: buffer too small for the requested shape");
  std::vector<uint8_t> out(static_cast<size_t>(rows * cols));
  check(anyq_unpack_codes(packed.data(), rows, cols, bits, out.data()));
  CodeMat codes(rows, cols);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) codes(i, j) = out[static_cast<size_t>(i * cols + j)];
  return codes;
}

QuantizedTensor from_ktiled(const QuantizedTensor& qt) {
  if (qt.layout == Layout::RowMajor) return qt;
  QuantizedTensor out = qt;
  check(anyq_ktile_codes(qt.codes.data(), qt.rows, qt.cols, qt.cfg.bits, qt.tile_k, 1,
                         out.codes.data()));
  out.layout = Layout::RowMajor;
  out.tile_k = 1;
  return out;
}

QuantizedTensor to_ktiled(const QuantizedTensor& qt, int tile_k) {
  if (tile_k < 1) throw ConfigError("tile_k must be >= 1");
  QuantizedTensor out = from_ktiled(qt);
  std::vector<uint8_t> tiled(out.codes.size());
  check(anyq_ktile_codes(out.codes.data(), out.rows, out.cols, out.cfg.bits, tile_k, 0,
                         tiled.data()));
  out.codes = std::move(tiled);
  out.layout = Layout::KTiled;
  out.tile_k = tile_k;
  return out;
}

QuantizedTensor narrowed(const QuantizedTensor& qt) {
  QuantizedTensor out = qt;
  CView v(out);
  check(anyq_narrow_inplace(&v.t));
  return out;
}

void write_file(const QuantizedTensor& qt, const std::string& path) {
  validate(qt.cfg, qt.rows, qt.cols);
  if (static_cast<Index>(qt.codes.size()) != qt.rows * packed_bytes_per_row(qt.cols, qt.cfg.bits))
    throw ShapeError("write_file: packed code size does not match shape");
  CView v(qt);
  check(anyq_write_file(&v.t, path.c_str()));
}

QuantizedTensor read_file(const std::string& path) {
  anyq_qtensor h;
  std::memset(&h, 0, sizeof h);
  check(anyq_read_file_header(path.c_str(), &h));
  QuantizedTensor qt;  // fields the file does not store keep their defaults (pack.cpp:356)
  qt.rows = h.rows;
  qt.cols = h.cols;
  qt.cfg.bits = h.cfg.bits;
  qt.cfg.codebook = static_cast<CodebookKind>(h.cfg.codebook);
  qt.cfg.granularity = static_cast<Granularity>(h.cfg.granularity);
  qt.cfg.symmetric = h.cfg.symmetric != 0;
  qt.cfg.int_range_shifted = h.cfg.int_range_shifted != 0;
  qt.cfg.group_size = h.cfg.group_size;
  qt.cfg.block_size = h.cfg.block_size;
  qt.cfg.seed = h.cfg.seed;
  qt.cfg.learner.init = static_cast<LutInit>(h.cfg.init);
  qt.cfg.learner.weighting = static_cast<Weighting>(h.cfg.weighting);
  qt.cfg.learner.max_iters = h.cfg.max_iters;
  qt.cfg.learner.rel_tol = h.cfg.rel_tol;
  qt.cfg.learner.restarts = h.cfg.restarts;
  qt.layout = static_cast<Layout>(h.layout);
  qt.tile_k = h.tile_k;
  qt.lut_store = static_cast<Store16>(h.lut_store);
  qt.scale_store = static_cast<Store16>(h.scale_store);
  qt.codes.resize(static_cast<size_t>(qt.rows * packed_bytes_per_row(qt.cols, qt.cfg.bits)));
  if (qt.cfg.codebook == CodebookKind::AnyN)
    qt.luts.resize(static_cast<size_t>(qt.rows) << qt.cfg.bits);
  qt.scales.granularity = qt.cfg.granularity;
  qt.scales.rows = qt.rows;
  qt.scales.cols = qt.cols;
  qt.scales.group_size = qt.cfg.group_size;
  qt.scales.block_size = qt.cfg.block_size;
  qt.scales.symmetric = qt.cfg.symmetric;
  qt.scales.alphas.resize(static_cast<Index>(h.num_groups));
  qt.scales.betas.resize(static_cast<Index>(h.num_groups));
  CView v(qt);  // the C-ABI fills qt's own arrays
  check(anyq_read_file(path.c_str(), &v.t));
  return qt;
}

Matf dequantize(const QuantizedTensor& qt) {
  Matf w(qt.rows, qt.cols);
  CView v(qt);
  check(anyq_dequantize(&v.t, w.data()));
  return w;
}

Matf gemm_dense(const Eigen::Ref<const Matf>& x, const Eigen::Ref<const Matf>& w) {
  if (x.cols() != w.cols()) throw ShapeError("gemm: reduction dimensions differ");
  const std::vector<float> xf = flat(x), wf = flat(w);
  Matf y(x.rows(), w.rows());
  check(anyq_gemm_dense(xf.data(), x.rows(), wf.data(), w.rows(), w.cols(), y.data()));
  return y;
}

Matf gemm_reference(const Eigen::Ref<const Matf>& x, const QuantizedTensor& qt) {
  if (x.cols() != qt.cols) throw ShapeError("gemm_reference: reduction dimensions differ");
  const Matf w = dequantize(qt);
  return gemm_dense(x, w);
}

Matf gemm_fused(const Eigen::Ref<const Matf>& x, const QuantizedTensor& qt, const GemmPlan& plan) {
  if (x.cols() != qt.cols) throw ShapeError("gemm_fused: reduction dimensions differ");
  if (plan.m != x.rows() || plan.n != qt.rows || plan.k != qt.cols)
    throw ShapeError("gemm_fused: plan does not match operands");
  const std::vector<float> xf = flat(x);
  Matf y(x.rows(), qt.rows);
  CView v(qt);
  check(anyq_gemm_fused(xf.data(), x.rows(), &v.t, static_cast<int32_t>(plan.layout), plan.tile_k,
                        y.data()));
  return y;
}

}  // namespace anyq
