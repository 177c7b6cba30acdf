// ANYQ v1 tensor files (pack.cpp:240-471) <-> anyq_qtensor, and straight into
// the prepacked device layout.
//
// Host code: a file is a 120-byte little-endian header followed by the packed
// codes, the alphas then betas, and the LUTs, each 16-bit stored value
// narrowed with the same RNE conversions as narrowed() (common.cuh). The
// writer is byte-identical to write_file; the reader performs every check of
// read_file in the same order and raises the same error classes
// (MagicError, VersionError, TruncatedError, InvariantError, CodeRangeError).
// anyq_dev_tensor_load then prepacks on the GPU (lutgemm_create).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "common.cuh"
#include "lutgemm.cuh"

namespace anyq_b200 {

void validate_config(const anyq_config& c, int64_t rows, int64_t cols);  // capi.cu
void set_last_error(const std::string& msg);                                // capi.cu

namespace {

constexpr char kMagic[4] = {'A', 'N', 'Y', 'Q'};
constexpr uint32_t kVersion = 1;
constexpr uint64_t kHeaderSize = 120;

template <typename F>
anyq_status host_guard(F&& f) {  // file IO needs no device
  try {
    f();
    set_last_error("");
    return ANYQ_OK;
  } catch (const Failure& e) {
    set_last_error(e.msg);
    return e.status;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return ANYQ_ERR_INTERNAL;
  }
}

size_t store_width(int s) { return s == ANYQ_STORE_FP32 ? 4 : 2; }

void put_u16(std::string& o, uint16_t v) {
  o.push_back((char)(v & 0xff));
  o.push_back((char)(v >> 8));
}
void put_u32(std::string& o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back((char)((v >> (8 * i)) & 0xff));
}
void put_u64(std::string& o, uint64_t v) {
  for (int i = 0; i < 8; ++i) o.push_back((char)((v >> (8 * i)) & 0xff));
}
void put_f32(std::string& o, float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  put_u32(o, u);
}
uint16_t get_u16(const std::string& b, size_t off) {
  return (uint16_t)((uint8_t)b[off] | ((uint16_t)(uint8_t)b[off + 1] << 8));
}
uint32_t get_u32(const std::string& b, size_t off) {
  uint32_t v = 0;
  for (int i = 3; i >= 0; --i) v = (v << 8) | (uint8_t)b[off + i];
  return v;
}
uint64_t get_u64(const std::string& b, size_t off) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | (uint8_t)b[off + i];
  return v;
}
float get_f32(const std::string& b, size_t off) {
  uint32_t u = get_u32(b, off);
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// put_stored / get_stored (pack.cpp:252-268)
void put_stored(std::string& o, float v, int s) {
  int st = ANYQ_OK;
  if (s == ANYQ_STORE_FP16) {
    const uint16_t h = f32_to_f16_exact(v, &st);
    if (st != ANYQ_OK) fail((anyq_status)st, st == ANYQ_ERR_IO ? "value overflows fp16" : "non-finite value");
    put_u16(o, h);
  } else if (s == ANYQ_STORE_BF16) {
    const uint16_t h = f32_to_bf16_exact(v, &st);
    if (st != ANYQ_OK) fail((anyq_status)st, st == ANYQ_ERR_IO ? "value overflows bf16" : "non-finite value");
    put_u16(o, h);
  } else if (s == ANYQ_STORE_FP32) {
    put_f32(o, v);
  } else {
    fail(ANYQ_ERR_CONFIG, "unknown storage precision");
  }
}
float get_stored(const std::string& b, size_t off, int s) {
  if (s == ANYQ_STORE_FP16) return f16_to_f32_exact(get_u16(b, off));
  if (s == ANYQ_STORE_BF16) return bf16_to_f32_exact(get_u16(b, off));
  return get_f32(b, off);
}

void need(const std::string& buf, uint64_t off, uint64_t len, const char* what) {
  if (off > buf.size() || len > buf.size() - off)
    fail(ANYQ_ERR_TRUNCATED, std::string("ANYQ file truncated reading ") + what + " at offset " +
                                 std::to_string(off));
}

int checked_enum(uint8_t raw, uint8_t max, const char* what) {
  if (raw > max) fail(ANYQ_ERR_INVARIANT, std::string("ANYQ file has invalid ") + what);
  return raw;
}

std::string slurp(const char* path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) fail(ANYQ_ERR_IO, std::string("cannot open ANYQ file '") + path + "'");
  const std::streamoff n = in.tellg();
  std::string buf(n > 0 ? (size_t)n : 0, '\0');
  in.seekg(0);
  if (n > 0 && !in.read(&buf[0], n)) fail(ANYQ_ERR_IO, std::string("cannot read ANYQ file '") + path + "'");
  return buf;
}

// temp file + rename (io_util.hpp:62-79): no partial output survives an error
void atomic_write(const char* path, const std::string& bytes) {
  const std::string tmp = std::string(path) + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    if (!out) fail(ANYQ_ERR_IO, "cannot open '" + tmp + "' for writing");
    out.write(bytes.data(), (std::streamsize)bytes.size());
    if (!out) fail(ANYQ_ERR_IO, "short write to '" + tmp + "'");
  }
  if (std::rename(tmp.c_str(), path) != 0) {
    std::remove(tmp.c_str());
    fail(ANYQ_ERR_IO, std::string("cannot rename '") + tmp + "' to '" + path + "'");
  }
}

// Header + section table of a file already in memory (read_file, pack.cpp:347-401).
struct Parsed {
  anyq_qtensor h{};
  uint32_t lut_entries = 0;
  uint64_t codes_off = 0, codes_len = 0, scales_off = 0, luts_off = 0;
};

Parsed parse_header(const std::string& buf) {
  need(buf, 0, kHeaderSize, "header");
  if (std::memcmp(buf.data(), kMagic, 4) != 0) fail(ANYQ_ERR_MAGIC, "not an ANYQ file");
  const uint32_t version = get_u32(buf, 4);
  if (version != kVersion) fail(ANYQ_ERR_VERSION, "unsupported ANYQ version " + std::to_string(version));
  Parsed P;
  anyq_qtensor& q = P.h;
  anyq_config_default(&q.cfg);
  q.rows = get_u32(buf, 8);
  q.cols = get_u32(buf, 12);
  q.cfg.bits = (uint8_t)buf[16];
  q.cfg.codebook = checked_enum((uint8_t)buf[17], 3, "codebook kind");
  q.cfg.granularity = checked_enum((uint8_t)buf[18], 4, "granularity");
  q.cfg.symmetric = buf[19] != 0;
  q.layout = checked_enum((uint8_t)buf[20], 1, "layout");
  q.lut_store = checked_enum((uint8_t)buf[21], 2, "LUT storage");
  q.scale_store = checked_enum((uint8_t)buf[22], 2, "scale storage");
  q.cfg.int_range_shifted = buf[23] != 0;
  q.cfg.group_size = (int32_t)get_u32(buf, 24);
  q.cfg.block_size = (int32_t)get_u32(buf, 28);
  q.tile_k = (int32_t)get_u32(buf, 32);
  q.cfg.seed = get_u64(buf, 36);
  q.cfg.init = checked_enum((uint8_t)buf[44], 3, "learner init");
  q.cfg.weighting = checked_enum((uint8_t)buf[45], 2, "learner weighting");
  q.cfg.max_iters = (int32_t)get_u32(buf, 48);
  q.cfg.rel_tol = get_f32(buf, 52);
  q.cfg.restarts = (int32_t)get_u32(buf, 56);
  const uint32_t num_groups = get_u32(buf, 60);
  P.lut_entries = get_u32(buf, 64);
  try {
    validate_config(q.cfg, q.rows, q.cols);
  } catch (const Failure& e) {
    fail(ANYQ_ERR_INVARIANT, "ANYQ file header invalid: " + e.msg);
  }
  if (q.layout == ANYQ_LAYOUT_KTILED && q.tile_k < 1) fail(ANYQ_ERR_INVARIANT, "ANYQ file has invalid tile_k");
  const uint32_t expect_lut = q.cfg.codebook == ANYQ_CB_ANY ? (1u << q.cfg.bits) : 0u;
  if (P.lut_entries != expect_lut) fail(ANYQ_ERR_INVARIANT, "ANYQ file LUT entry count mismatch");
  P.codes_off = get_u64(buf, 72);
  P.codes_len = get_u64(buf, 80);
  P.scales_off = get_u64(buf, 88);
  const uint64_t scales_len = get_u64(buf, 96);
  P.luts_off = get_u64(buf, 104);
  const uint64_t luts_len = get_u64(buf, 112);
  const uint64_t expect_codes = (uint64_t)q.rows * (uint64_t)packed_bpr(q.cols, q.cfg.bits);
  const uint64_t expect_scales = 2ull * num_groups * store_width(q.scale_store);
  const uint64_t expect_luts = (uint64_t)q.rows * P.lut_entries * store_width(q.lut_store);
  if (P.codes_len != expect_codes || scales_len != expect_scales || luts_len != expect_luts)
    fail(ANYQ_ERR_INVARIANT, "ANYQ file section lengths do not match its shape");
  need(buf, P.codes_off, P.codes_len, "codes");
  need(buf, P.scales_off, scales_len, "scales");
  need(buf, P.luts_off, luts_len, "LUTs");
  if (buf.size() != P.luts_off + luts_len)
    fail(ANYQ_ERR_INVARIANT, "ANYQ file size does not match declared sections");
  q.num_groups = num_groups;
  return P;
}

// Section contents into the caller's arrays, with read_file's value checks
// (pack.cpp:403-470) in its order. The scales are checked from the file
// bytes first: the header's group count is only trusted (and compared with
// the caller's capacity `cap_groups`) once it matched the granularity, so a
// corrupt count can never write past the caller's alpha/beta arrays.
void read_body(const std::string& buf, const Parsed& P, anyq_qtensor* q, int64_t cap_groups) {
  const anyq_qtensor& h = P.h;
  std::memcpy(q->codes, buf.data() + P.codes_off, P.codes_len);
  const size_t w = store_width(h.scale_store);
  const int64_t ng = h.num_groups;
  for (int64_t g = 0; g < ng; ++g) {
    const float a = get_stored(buf, P.scales_off + w * g, h.scale_store);
    const float b = get_stored(buf, P.scales_off + w * (ng + g), h.scale_store);
    if (!(a > 0) || !std::isfinite(a)) fail(ANYQ_ERR_INVARIANT, "ANYQ file scale alpha must be positive and finite");
    if (!std::isfinite(b)) fail(ANYQ_ERR_INVARIANT, "ANYQ file scale beta must be finite");
    if (h.cfg.symmetric && b != 0) fail(ANYQ_ERR_INVARIANT, "ANYQ file symmetric tensor has nonzero beta");
  }
  if (ng != group_count(h.cfg, h.rows, h.cols))
    fail(ANYQ_ERR_INVARIANT, "ANYQ file group count does not match granularity");
  if (ng > cap_groups) fail(ANYQ_ERR_SHAPE, "read_file: caller scale arrays are too small");
  for (int64_t g = 0; g < ng; ++g) {
    q->alphas[g] = get_stored(buf, P.scales_off + w * g, h.scale_store);
    q->betas[g] = get_stored(buf, P.scales_off + w * (ng + g), h.scale_store);
  }
  const size_t lw = store_width(h.lut_store);
  const int64_t nl = h.rows * (int64_t)P.lut_entries;
  for (int64_t i = 0; i < nl; ++i) {
    q->luts[i] = get_stored(buf, P.luts_off + lw * i, h.lut_store);
    if (!std::isfinite(q->luts[i])) fail(ANYQ_ERR_INVARIANT, "ANYQ file LUT value must be finite");
  }
  for (int64_t i = 0; i < h.rows && P.lut_entries > 0; ++i)
    for (uint32_t e = 1; e < P.lut_entries; ++e)
      if (q->luts[i * P.lut_entries + e] < q->luts[i * P.lut_entries + e - 1])
        fail(ANYQ_ERR_INVARIANT, "ANYQ file row LUT is not sorted");
  // every code must index inside its value table (only tables shorter than
  // 2^bits can be violated: fp4's 15 entries)
  const int table = h.cfg.codebook == ANYQ_CB_ANY ? (int)P.lut_entries : fixed_table(h.cfg).n;
  if (table < (1 << h.cfg.bits)) {
    const int64_t bpr = packed_bpr(h.cols, h.cfg.bits);
    const int bits = h.cfg.bits;
    for (int64_t i = 0; i < h.rows; ++i) {
      const uint8_t* row = q->codes + i * bpr;
      for (int64_t j = 0; j < h.cols; ++j) {  // little-end-first bit packing (pack.cpp:15-33)
        const int64_t bit = j * bits;
        uint32_t v = row[bit >> 3] | (((bit >> 3) + 1 < bpr ? (uint32_t)row[(bit >> 3) + 1] : 0u) << 8);
        const int code = (int)((v >> (bit & 7)) & ((1u << bits) - 1));
        if (code >= table)
          fail(ANYQ_ERR_CODE_RANGE, "ANYQ file code " + std::to_string(code) + " exceeds table size " +
                                        std::to_string(table));
      }
    }
  }
}

}  // namespace
}  // namespace anyq_b200

using namespace anyq_b200;

extern "C" {

anyq_status anyq_write_file(const anyq_qtensor* qt, const char* path) {
  return host_guard([&] {
    if (!qt || !path) fail(ANYQ_ERR_SHAPE, "null tensor or path");
    validate_config(qt->cfg, qt->rows, qt->cols);
    if (!qt->codes || !qt->alphas || !qt->betas || (qt->cfg.codebook == ANYQ_CB_ANY && !qt->luts))
      fail(ANYQ_ERR_SHAPE, "write_file: tensor arrays missing");
    if (qt->num_groups != group_count(qt->cfg, qt->rows, qt->cols))
      fail(ANYQ_ERR_SHAPE, "write_file: group count does not match the granularity");
    const int64_t ng = qt->num_groups;
    const uint64_t codes = (uint64_t)qt->rows * (uint64_t)packed_bpr(qt->cols, qt->cfg.bits);
    const uint64_t lut_entries = qt->cfg.codebook == ANYQ_CB_ANY ? (1ull << qt->cfg.bits) : 0ull;
    const uint64_t scales = 2ull * (uint64_t)ng * store_width(qt->scale_store);
    const uint64_t luts = (uint64_t)qt->rows * lut_entries * store_width(qt->lut_store);
    std::string b;
    b.reserve(kHeaderSize + codes + scales + luts);
    b.append(kMagic, 4);
    put_u32(b, kVersion);
    put_u32(b, (uint32_t)qt->rows);
    put_u32(b, (uint32_t)qt->cols);
    b.push_back((char)qt->cfg.bits);
    b.push_back((char)qt->cfg.codebook);
    b.push_back((char)qt->cfg.granularity);
    b.push_back((char)(qt->cfg.symmetric ? 1 : 0));
    b.push_back((char)qt->layout);
    b.push_back((char)qt->lut_store);
    b.push_back((char)qt->scale_store);
    b.push_back((char)(qt->cfg.int_range_shifted ? 1 : 0));
    put_u32(b, (uint32_t)qt->cfg.group_size);
    put_u32(b, (uint32_t)qt->cfg.block_size);
    put_u32(b, (uint32_t)qt->tile_k);
    put_u64(b, qt->cfg.seed);
    b.push_back((char)qt->cfg.init);
    b.push_back((char)qt->cfg.weighting);
    put_u16(b, 0);
    put_u32(b, (uint32_t)qt->cfg.max_iters);
    put_f32(b, qt->cfg.rel_tol);
    put_u32(b, (uint32_t)qt->cfg.restarts);
    put_u32(b, (uint32_t)ng);
    put_u32(b, (uint32_t)lut_entries);
    put_u32(b, 0);
    put_u64(b, kHeaderSize);
    put_u64(b, codes);
    put_u64(b, kHeaderSize + codes);
    put_u64(b, scales);
    put_u64(b, kHeaderSize + codes + scales);
    put_u64(b, luts);
    if (b.size() != kHeaderSize) fail(ANYQ_ERR_INTERNAL, "internal: ANYQ header size drift");
    b.append(reinterpret_cast<const char*>(qt->codes), codes);
    for (int64_t g = 0; g < ng; ++g) put_stored(b, qt->alphas[g], qt->scale_store);
    for (int64_t g = 0; g < ng; ++g) put_stored(b, qt->betas[g], qt->scale_store);
    for (uint64_t i = 0; i < (uint64_t)qt->rows * lut_entries; ++i) put_stored(b, qt->luts[i], qt->lut_store);
    atomic_write(path, b);
  });
}

anyq_status anyq_read_file_header(const char* path, anyq_qtensor* hdr) {
  return host_guard([&] {
    const std::string buf = slurp(path);
    const Parsed P = parse_header(buf);
    const anyq_qtensor keep = *hdr;
    *hdr = P.h;
    hdr->codes = keep.codes;
    hdr->luts = keep.luts;
    hdr->alphas = keep.alphas;
    hdr->betas = keep.betas;
  });
}

anyq_status anyq_read_file(const char* path, anyq_qtensor* qt) {
  return host_guard([&] {
    const std::string buf = slurp(path);
    const Parsed P = parse_header(buf);
    if (!qt->codes || !qt->alphas || !qt->betas || (P.lut_entries && !qt->luts))
      fail(ANYQ_ERR_SHAPE, "read_file: caller arrays not allocated");
    // codes / LUT sizes follow from rows, cols and cfg, which the caller took
    // from the header; the scale capacity is the caller's num_groups
    if (qt->rows != P.h.rows || qt->cols != P.h.cols || qt->cfg.bits != P.h.cfg.bits ||
        qt->cfg.codebook != P.h.cfg.codebook)
      fail(ANYQ_ERR_SHAPE, "read_file: caller arrays were sized for a different header");
    read_body(buf, P, qt, qt->num_groups);
    uint8_t* codes = qt->codes;
    float *luts = qt->luts, *alphas = qt->alphas, *betas = qt->betas;
    *qt = P.h;
    qt->codes = codes;
    qt->luts = P.lut_entries ? luts : nullptr;
    qt->alphas = alphas;
    qt->betas = betas;
  });
}

}  // extern "C"

namespace anyq_b200 {
// read_file straight into the prepacked device layout (lutgemm_create).
LutTensor* load_device_tensor(const char* path) {
  const std::string buf = slurp(path);
  const Parsed P = parse_header(buf);
  anyq_qtensor q = P.h;
  std::vector<uint8_t> codes(P.codes_len);
  std::vector<float> luts(q.rows * (int64_t)P.lut_entries), alphas(q.num_groups), betas(q.num_groups);
  q.codes = codes.data();
  q.luts = P.lut_entries ? luts.data() : nullptr;
  q.alphas = alphas.data();
  q.betas = betas.data();
  read_body(buf, P, &q, (int64_t)alphas.size());
  return lutgemm_create(&q);
}
}  // namespace anyq_b200
