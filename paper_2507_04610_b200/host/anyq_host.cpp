// C++ host layer of the drop-in: the reference's hot-path API (declared in
// proj/include/anyq/{learner,quantize,pack,qgemm,codebooks,scaling,calibration}.hpp,
// compiled against those headers in place) implemented on the B200 library
// through its C-ABI (include/anyq_b200.h). Same signatures, value semantics and
// exception classes as the reference; every computation runs on the GPU — a
// host with no device gets anyq::Error from the first compute call, never a
// CPU result. What stays on the host is argument checking, the fixed-table
// bookkeeping (effective_codebook's 16 subtractions), scalar fp16/bf16
// conversions (through the library's bit-exact converters), the ANYQ file
// size arithmetic and string tables.
//
//   quantize_any / learn_row_lut / weighted_kmeans / kmeans_pp_init /
//     build_sample_weights / KmProblem::validate        learner.hpp:30-75
//   quantize / quantize_fixed / apply_format / format and enum names
//                                                       quantize.hpp:17-45
//   int_grid / fp4_table / nf4_table / fixed_codebook / effective_codebook /
//     round_to_codebook / storage_bits_per_entry / codebook_json
//                                                       codebooks.hpp:27-55
//   pack_codes / unpack_codes / f32_to_f16 ... / narrow_lut / widen_lut /
//     narrowed / to_ktiled / from_ktiled / scaled_values / dequantize /
//     file_sizes / write_file / read_file               pack.hpp:50-121
//   compute_scales / scale_weights / dequantize(values, s)  scaling.hpp:52-60
//   make_plan / gemm_dense / gemm_reference / gemm_fused / bench / bench_csv
//                                                       qgemm.hpp:24-59
//   ActivationStats::for_module                         calibration.hpp:21
//   weight_error / output_error / eval_activations / compare_formats /
//     EvalReport::to_csv / to_json                      eval.hpp:33-70
//
// This object alone (plus libanyq_b200.so) is the drop-in: no reference
// object is linked into libanyq_host.so or the B200 test binary.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include "anyq/calibration.hpp"
#include "anyq/codebooks.hpp"
#include "anyq/eval.hpp"
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


// ---------------------------------------------------------------------------
// calibration.hpp:21
// ---------------------------------------------------------------------------
const Vecf& ActivationStats::for_module(const std::string& name, Index cols) const {
  const auto it = entries.find(name);
  if (it == entries.end()) throw StatsError("no activation stats for module '" + name + "'");
  if (it->second.size() != cols)
    throw StatsError("activation stats for '" + name + "' have " + std::to_string(it->second.size()) +
                     " channels, matrix has " + std::to_string(cols));
  return it->second;
}

// ---------------------------------------------------------------------------
// Evaluation (eval.hpp:33-70): the error metrics' dequantisations, GEMMs and
// double sums run on the GPU (anyq_weight_error / anyq_output_error); the
// activations are drawn on the host by the reference's Box-Muller.
// ---------------------------------------------------------------------------
std::pair<double, double> weight_error(const Eigen::Ref<const Matf>& w, const QuantizedTensor& qt) {
  if (w.rows() != qt.rows || w.cols() != qt.cols) throw ShapeError("weight_error: shapes differ");
  const std::vector<float> wf = flat(w);
  CView v(qt);
  double mse = 0, rel = 0;
  check(anyq_weight_error(wf.data(), w.rows(), w.cols(), &v.t, &mse, &rel));
  return {mse, rel};
}

double output_error(const Eigen::Ref<const Matf>& w, const QuantizedTensor& qt,
                    const Eigen::Ref<const Matf>& x) {
  if (w.rows() != qt.rows || w.cols() != qt.cols) throw ShapeError("output_error: weight shapes differ");
  if (x.cols() != w.cols()) throw ShapeError("output_error: activation width mismatch");
  const std::vector<float> wf = flat(w), xf = flat(x);
  CView v(qt);
  double mse = 0;
  check(anyq_output_error(wf.data(), w.rows(), w.cols(), &v.t, xf.data(), x.rows(), x.cols(), &mse));
  return mse;
}

Matf eval_activations(Index rows, Index cols, const Vecf* exj, uint64_t seed) {
  if (exj && exj->size() != cols) throw StatsError("eval_activations: stats length mismatch");
  Matf x(rows, cols);
  check(anyq_eval_activations(rows, cols, exj ? exj->data() : nullptr, seed, x.data()));
  return x;
}

EvalReport compare_formats(const Eigen::Ref<const Matf>& w, const std::vector<std::string>& formats,
                           const QuantConfig& base, const ActivationStats* stats,
                           const std::string& module_name, const CompareOptions& opts) {
  const Vecf* exj = stats ? &stats->for_module(module_name, w.cols()) : nullptr;
  const Matf x = eval_activations(opts.eval_rows, w.cols(), exj, opts.eval_seed);
  EvalReport report;
  for (const auto& fmt : formats) {
    QuantConfig cfg = base;
    apply_format(cfg, fmt);
    const QuantizedTensor qt = quantize(w, cfg, stats, module_name, opts.threads);
    const auto [mse, rel] = weight_error(w, qt);
    EvalRow row;
    row.module = module_name;
    row.format = fmt;
    row.weight_mse = mse;
    row.weight_rel_frobenius = rel;
    row.output_mse = output_error(w, qt, x);
    row.bits_per_entry = storage_bits_per_entry(cfg, w.rows(), w.cols());
    report.rows.push_back(std::move(row));
  }
  return report;
}

// the report schema (v1): CSV header + one line per row, 9 significant digits
std::string EvalReport::to_csv() const {
  std::ostringstream os;
  os.precision(9);
  os << "schema_version,module,format,weight_mse,weight_rel_frobenius,output_mse,bits_per_entry\n";
  for (const auto& r : rows)
    os << kSchemaVersion << ',' << r.module << ',' << r.format << ',' << r.weight_mse << ','
       << r.weight_rel_frobenius << ',' << r.output_mse << ',' << r.bits_per_entry << '\n';
  return os.str();
}

std::string EvalReport::to_json() const {
  std::ostringstream os;
  os.precision(9);
  os << "{\"schema_version\":\"" << kSchemaVersion << "\",\"rows\":[";
  for (size_t i = 0; i < rows.size(); ++i) {
    const auto& r = rows[i];
    os << (i ? "," : "") << "{\"module\":\"" << r.module << "\",\"format\":\"" << r.format
       << "\",\"weight_mse\":" << r.weight_mse << ",\"weight_rel_frobenius\":" << r.weight_rel_frobenius
       << ",\"output_mse\":" << r.output_mse << ",\"bits_per_entry\":" << r.bits_per_entry << '}';
  }
  os << "]}";
  return os.str();
}

// ---------------------------------------------------------------------------
// Codebooks (codebooks.hpp:27-55). The fixed tables come from the library.
// ---------------------------------------------------------------------------
namespace {

Codebook table_of(CodebookKind kind, int bits, bool shifted) {
  float v[256];
  int32_t n = 0;
  check(anyq_fixed_table(static_cast<int32_t>(kind), bits, shifted ? 1 : 0, v, &n));
  Codebook cb;
  cb.kind = kind;
  cb.bits = bits;
  cb.values.assign(v, v + n);
  return cb;
}

}  // namespace

Codebook int_grid(int bits, bool shifted) { return table_of(CodebookKind::IntGrid, bits, shifted); }
Codebook fp4_table() { return table_of(CodebookKind::Fp4, 4, false); }
Codebook nf4_table() { return table_of(CodebookKind::Nf4, 4, false); }

Codebook fixed_codebook(const QuantConfig& cfg) {
  if (cfg.codebook == CodebookKind::AnyN) throw ConfigError("AnyN has no fixed codebook");
  if (cfg.codebook == CodebookKind::IntGrid) return int_grid(cfg.bits, cfg.int_range_shifted);
  if (cfg.codebook == CodebookKind::Fp4) return fp4_table();
  if (cfg.codebook == CodebookKind::Nf4) return nf4_table();
  throw ConfigError("unknown codebook kind");
}

Codebook effective_codebook(const Codebook& cb, bool symmetric) {
  Codebook out = cb;
  if (!symmetric) {
    const Real lo = cb.values.front();
    std::transform(cb.values.begin(), cb.values.end(), out.values.begin(),
                   [lo](Real v) { return v - lo; });
  }
  return out;
}

CodeMat round_to_codebook(const Eigen::Ref<const Matf>& ws, const Codebook& cb) {
  const std::vector<float> f = flat(ws);
  std::vector<uint8_t> c(f.size());
  check(anyq_round_to_table(f.data(), ws.rows(), ws.cols(), cb.values.data(),
                            static_cast<int32_t>(cb.values.size()), c.data()));
  CodeMat codes(ws.rows(), ws.cols());
  std::memcpy(codes.data(), c.data(), c.size());
  return codes;
}

double storage_bits_per_entry(const QuantConfig& cfg, Index rows, Index cols) {
  validate(cfg, rows, cols);
  const anyq_config c = to_c(cfg);
  double bits = 0;
  check(anyq_storage_bits_per_entry(&c, rows, cols, &bits));
  return bits;
}

std::string codebook_json(const Codebook& cb) {
  static const char* const kNames[] = {"int", "fp4", "nf4", "any"};
  std::ostringstream os;
  os.precision(9);
  os << "{\"kind\":\"" << kNames[static_cast<int>(cb.kind) & 3] << "\",\"bits\":" << cb.bits
     << ",\"values\":[";
  const char* sep = "";
  for (Real v : cb.values) {
    os << sep << v;
    sep = ",";
  }
  os << "]}";
  return os.str();
}

// ---------------------------------------------------------------------------
// Scalar narrowing (pack.hpp:57-66) and whole-tensor helpers
// ---------------------------------------------------------------------------
uint16_t f32_to_f16(Real f) {
  uint16_t h = 0;
  check(anyq_f32_to_f16(f, &h));
  return h;
}
Real f16_to_f32(uint16_t h) { return anyq_f16_to_f32(h); }
uint16_t f32_to_bf16(Real f) {
  uint16_t h = 0;
  check(anyq_f32_to_bf16(f, &h));
  return h;
}
Real bf16_to_f32(uint16_t h) { return anyq_bf16_to_f32(h); }

std::vector<uint16_t> narrow_lut(std::span<const Real> values, Store16 target) {
  if (target == Store16::Fp32) throw ConfigError("narrow_lut targets fp16 or bf16");
  std::vector<uint16_t> out;
  out.reserve(values.size());
  for (Real v : values) out.push_back(target == Store16::Fp16 ? f32_to_f16(v) : f32_to_bf16(v));
  return out;
}

std::vector<Real> widen_lut(std::span<const uint16_t> bits, Store16 source) {
  if (source == Store16::Fp32) throw ConfigError("widen_lut sources fp16 or bf16");
  std::vector<Real> out;
  out.reserve(bits.size());
  for (uint16_t b : bits) out.push_back(source == Store16::Fp16 ? f16_to_f32(b) : bf16_to_f32(b));
  return out;
}

Matf scaled_values(const QuantizedTensor& qt) {
  Matf v(qt.rows, qt.cols);
  CView view(qt);
  check(anyq_scaled_values(&view.t, v.data()));
  return v;
}

SizeBreakdown file_sizes(const QuantizedTensor& qt) {
  // ANYQ v1 layout (pack.cpp:240-291): 120-byte header, packed codes, alphas
  // then betas, row LUTs; 16-bit stores take 2 bytes per value, fp32 4
  auto width = [](Store16 s) -> uint64_t { return s == Store16::Fp32 ? 4 : 2; };
  SizeBreakdown b;
  b.header = 120;
  b.codes = qt.codes.size();
  b.scales = 2ull * static_cast<uint64_t>(qt.scales.num_groups()) * width(qt.scale_store);
  b.luts = static_cast<uint64_t>(qt.luts.size()) * width(qt.lut_store);
  return b;
}

// ---------------------------------------------------------------------------
// The per-row learner (learner.hpp:30-68) on the GPU
// ---------------------------------------------------------------------------
namespace {

// Rng (core.hpp:164-192) is {key, counter}; the library takes and returns
// that state so the caller's stream advances exactly as in the reference.
static_assert(sizeof(Rng) == 2 * sizeof(uint64_t) && std::is_standard_layout_v<Rng>,
              "Rng is expected to hold {key, counter}");
void rng_get(const Rng& r, uint64_t* key, uint64_t* ctr) {
  uint64_t st[2];
  std::memcpy(st, &r, sizeof st);
  *key = st[0];
  *ctr = st[1];
}
void rng_set(Rng& r, uint64_t ctr) {
  uint64_t st[2];
  std::memcpy(st, &r, sizeof st);
  st[1] = ctr;
  std::memcpy(&r, st, sizeof st);
}

anyq_config learner_cfg(const LearnerConfig& l) {
  anyq_config c;
  anyq_config_default(&c);
  c.init = static_cast<int32_t>(l.init);
  c.max_iters = l.max_iters;
  c.rel_tol = l.rel_tol;
  c.restarts = l.restarts;
  c.weighting = static_cast<int32_t>(l.weighting);
  c.check_invariants = l.check_invariants ? 1 : 0;
  return c;
}

// One KmProblem through anyq_kmeans_problems (mode 0: learn_row_lut, 1:
// weighted_kmeans, 2: kmeans_pp_init).
void run_problem(const std::vector<Real>& x, const std::vector<Real>& w, int k,
                 const LearnerConfig& l, Rng& rng, int mode, std::vector<double>& cen,
                 std::vector<uint8_t>& asg, double& loss, int& iters) {
  uint64_t key = 0, ctr = 0;
  rng_get(rng, &key, &ctr);
  const anyq_config c = learner_cfg(l);
  const int64_t n = static_cast<int64_t>(x.size());
  cen.assign(k > 0 ? k : 0, 0.0);
  asg.assign(mode == 2 ? 0 : x.size(), 0);
  int32_t it = 0;
  if (w.size() != x.size()) throw ShapeError("KmProblem: samples and weights differ in length");
  check(anyq_kmeans_problems(x.data(), w.data(), 1, n, k, &c, mode, &key, &ctr, cen.data(),
                             asg.empty() ? nullptr : asg.data(), &loss, &it));
  rng_set(rng, ctr);
  iters = it;
}

}  // namespace

void KmProblem::validate() const {
  if (samples.size() != weights.size())
    throw ShapeError("KmProblem: samples and weights differ in length");
  if (samples.empty()) throw ShapeError("KmProblem: empty problem");
  const bool all_ok = std::all_of(weights.begin(), weights.end(),
                                   [](Real w) { return w >= 0 && std::isfinite(w); });
  if (!all_ok) throw StatsError("KmProblem: weights must be >= 0");
  if (std::none_of(weights.begin(), weights.end(), [](Real w) { return w > 0; }))
    throw StatsError("KmProblem: all sample weights are zero");
  if (!std::all_of(samples.begin(), samples.end(), [](Real x) { return std::isfinite(x); }))
    throw NonFiniteError("KmProblem: non-finite sample");
}

Vecf build_sample_weights(const ScaleSet& s, Index row, const Vecf* stats, Weighting mode) {
  const anyq_config c = group_cfg(s);
  Vecf out(s.cols);
  check(anyq_build_sample_weights(&c, s.rows, s.cols, s.alphas.data(), s.num_groups(), row,
                                  stats ? stats->data() : nullptr, stats ? stats->size() : 0,
                                  static_cast<int32_t>(mode), out.data()));
  return out;
}

std::vector<double> kmeans_pp_init(const KmProblem& p, int k, Rng& rng) {
  p.validate();
  if (k < 1) throw ConfigError("k must be >= 1");
  std::vector<double> cen;
  std::vector<uint8_t> asg;
  double loss = 0;
  int iters = 0;
  run_problem(p.samples, p.weights, k, LearnerConfig{}, rng, 2, cen, asg, loss, iters);
  return cen;
}

KmResult weighted_kmeans(const KmProblem& p, int k, const LearnerConfig& cfg, Rng& rng) {
  p.validate();
  if (k < 1) throw ConfigError("k must be >= 1");
  if (k > 256) throw ConfigError("k must fit an 8-bit code");
  KmResult r;
  run_problem(p.samples, p.weights, k, cfg, rng, 1, r.centroids, r.assignments, r.loss, r.iters);
  return r;
}

RowQuant learn_row_lut(std::span<const Real> ws_row, std::span<const Real> weights,
                       const LearnerConfig& cfg, int bits, Rng& rng) {
  if (ws_row.size() != weights.size())
    throw ShapeError("learn_row_lut: row and weights differ in length");
  KmProblem p;
  p.samples.assign(ws_row.begin(), ws_row.end());
  p.weights.assign(weights.begin(), weights.end());
  p.validate();
  const int k = 1 << bits;
  if (k > 256) throw ConfigError("k must fit an 8-bit code");
  std::vector<double> lut;
  RowQuant rq;
  int iters = 0;
  // mode 0: the GPU sorts the table and rank-remaps the codes (learner.cpp:355-367)
  run_problem(p.samples, p.weights, k, cfg, rng, 0, lut, rq.codes, rq.loss, iters);
  rq.lut.values.assign(lut.begin(), lut.end());
  return rq;
}

// ---------------------------------------------------------------------------
// Front door (quantize.hpp:17-45)
// ---------------------------------------------------------------------------
QuantizedTensor quantize(const Eigen::Ref<const Matf>& w, const QuantConfig& cfg,
                         const ActivationStats* stats, const std::string& module_name,
                         int threads) {
  if (cfg.codebook != CodebookKind::AnyN) return quantize_fixed(w, cfg);
  const Vecf* exj = stats ? &stats->for_module(module_name, w.cols()) : nullptr;
  return quantize_any(w, cfg, exj, threads);
}

namespace {

template <typename E>
struct Named {
  const char* name;
  E value;
};

constexpr Named<Granularity> kGranularities[] = {
    {"tensorwise", Granularity::Tensorwise}, {"rowwise", Granularity::Rowwise},
    {"columnwise", Granularity::Columnwise}, {"groupwise", Granularity::Groupwise},
    {"blockwise", Granularity::Blockwise}};
constexpr Named<Weighting> kWeightings[] = {
    {"weights", Weighting::WeightsOnly},
    {"weights-activations", Weighting::WeightsTimesActivations},
    {"full", Weighting::WeightsTimesActivationsTimesScales}};
constexpr Named<LutInit> kInits[] = {{"kmeans++", LutInit::KMeansPlusPlus},
                                     {"random", LutInit::Random},
                                     {"int-grid", LutInit::IntGridSeed},
                                     {"nf4", LutInit::Nf4Seed}};
constexpr Named<Store16> kStores[] = {
    {"fp16", Store16::Fp16}, {"bf16", Store16::Bf16}, {"fp32", Store16::Fp32}};

template <typename E, size_t N>
E parse_named(const Named<E> (&table)[N], const std::string& name, const char* what) {
  for (const auto& e : table)
    if (name == e.name) return e.value;
  throw ConfigError(std::string("unknown ") + what + " '" + name + "'");
}

template <typename E, size_t N>
std::string name_of(const Named<E> (&table)[N], E value) {
  for (const auto& e : table)
    if (e.value == value) return e.name;
  return "?";
}

// format names (quantize.cpp:34-54): a codebook kind and a bit width each
struct Format {
  const char* name;
  CodebookKind kind;
  int bits;
};
constexpr Format kFormats[] = {
    {"int2", CodebookKind::IntGrid, 2}, {"int3", CodebookKind::IntGrid, 3},
    {"int4", CodebookKind::IntGrid, 4}, {"int8", CodebookKind::IntGrid, 8},
    {"fp4", CodebookKind::Fp4, 4},      {"nf4", CodebookKind::Nf4, 4},
    {"any2", CodebookKind::AnyN, 2},    {"any3", CodebookKind::AnyN, 3},
    {"any4", CodebookKind::AnyN, 4},    {"any8", CodebookKind::AnyN, 8}};

}  // namespace

void apply_format(QuantConfig& cfg, const std::string& format) {
  for (const auto& f : kFormats) {
    if (format == f.name) {
      cfg.codebook = f.kind;
      cfg.bits = f.bits;
      return;
    }
  }
  throw ConfigError("unknown format '" + format + "'");
}

std::string format_name(const QuantConfig& cfg) {
  switch (cfg.codebook) {
    case CodebookKind::IntGrid: return "int" + std::to_string(cfg.bits);
    case CodebookKind::AnyN: return "any" + std::to_string(cfg.bits);
    case CodebookKind::Fp4: return "fp4";
    case CodebookKind::Nf4: return "nf4";
  }
  return "?";
}

Granularity parse_granularity(const std::string& name) {
  return parse_named(kGranularities, name, "granularity");
}
std::string granularity_name(Granularity g) { return name_of(kGranularities, g); }
Weighting parse_weighting(const std::string& name) {
  return parse_named(kWeightings, name, "weighting");
}
std::string weighting_name(Weighting w) { return name_of(kWeightings, w); }
LutInit parse_init(const std::string& name) { return parse_named(kInits, name, "init"); }
std::string init_name(LutInit init) { return name_of(kInits, init); }
Store16 parse_store(const std::string& name) {
  return parse_named(kStores, name, "storage precision");
}
std::string store_name(Store16 s) { return name_of(kStores, s); }

// ---------------------------------------------------------------------------
// GEMM plan and the benchmark (qgemm.hpp:24, 55-59)
// ---------------------------------------------------------------------------
GemmPlan make_plan(const Eigen::Ref<const Matf>& x, const QuantizedTensor& qt) {
  GemmPlan plan;
  plan.m = x.rows();
  plan.n = qt.rows;
  plan.k = qt.cols;
  plan.layout = qt.layout;
  plan.tile_k = qt.tile_k;
  return plan;
}

namespace {

// Linear-interpolated percentile of a sample (qgemm.cpp bench semantics).
double quantile(std::vector<double> v, double p) {
  std::sort(v.begin(), v.end());
  const double pos = p * static_cast<double>(v.size() - 1);
  const size_t lo = static_cast<size_t>(pos);
  const size_t hi = std::min(lo + 1, v.size() - 1);
  const double t = pos - static_cast<double>(lo);
  return v[lo] + (v[hi] - v[lo]) * t;
}

}  // namespace

// The reference times its CPU gemm_fused per (shape, format) next to a dense
// fp32 row. Here every timing is a device run with HBM-resident operands
// (CUDA events): "dense" = fp32 gemm_dense, "rowmajor" = the bit-exact
// gemm_fused kernel, "b200" = the A16W4 LUT GEMM on the prepacked tensor (the
// AUTO kernel for m; formats it does not take — 8-bit codes, groups that are
// not multiples of 128 — get no such row). Inputs are generated as the
// reference generates them (rng_for_row(seed, row index) Gaussians).
std::vector<BenchRow> bench(const std::vector<BenchShape>& shapes,
                            const std::vector<std::string>& formats, int repeats, uint64_t seed) {
  if (repeats < 1) throw ConfigError("bench: repeats must be >= 1");
  std::vector<BenchRow> rows;
  auto gaussian = [](Index r, Index c, Rng& rng) {
    Matf m(r, c);
    for (Index i = 0; i < r; ++i)
      for (Index j = 0; j < c; ++j) m(i, j) = static_cast<Real>(rng.next_gaussian());
    return m;
  };
  for (const BenchShape& shape : shapes) {
    Rng rng = rng_for_row(seed, static_cast<Index>(rows.size()));
    const Matf w = gaussian(shape.n, shape.k, rng);
    const Matf x = gaussian(shape.m, shape.k, rng);
    std::vector<double> ns(static_cast<size_t>(repeats));
    auto push = [&](const std::string& fmt, const std::string& layout, double bpw) {
      BenchRow r;
      r.shape = shape;
      r.format = fmt;
      r.layout = layout;
      r.median_ns = quantile(ns, 0.5);
      r.p10_ns = quantile(ns, 0.1);
      r.p90_ns = quantile(ns, 0.9);
      r.bytes_per_weight = bpw;
      rows.push_back(r);
    };
    check(anyq_bench_gemm(0, nullptr, w.data(), shape.n, shape.k, x.data(), shape.m, repeats,
                          ns.data()));
    push("fp32", "dense", 4.0);
    for (const std::string& fmt : formats) {
      QuantConfig cfg;
      cfg.granularity = Granularity::Groupwise;
      cfg.group_size = static_cast<int>(std::min<Index>(128, shape.k));
      cfg.seed = seed;
      apply_format(cfg, fmt);
      const QuantizedTensor qt = quantize(w, cfg);
      const double bpw = storage_bits_per_entry(cfg, shape.n, shape.k) / 8.0;
      CView v(qt);
      check(anyq_bench_gemm(1, &v.t, nullptr, shape.n, shape.k, x.data(), shape.m, repeats,
                            ns.data()));
      push(fmt, "rowmajor", bpw);
      if (anyq_bench_gemm(2, &v.t, nullptr, shape.n, shape.k, x.data(), shape.m, repeats,
                          ns.data()) == ANYQ_OK)
        push(fmt, "b200", bpw);
    }
  }
  return rows;
}

std::string bench_csv(const std::vector<BenchRow>& rows) {
  std::ostringstream os;
  os << "shape,format,layout,median_ns,p10_ns,p90_ns,bytes_per_weight\n";
  for (const BenchRow& r : rows)
    os << r.shape.m << 'x' << r.shape.n << 'x' << r.shape.k << ',' << r.format << ',' << r.layout
       << ',' << static_cast<uint64_t>(r.median_ns) << ',' << static_cast<uint64_t>(r.p10_ns)
       << ',' << static_cast<uint64_t>(r.p90_ns) << ',' << r.bytes_per_weight << '\n';
  return os.str();
}

}  // namespace anyq
