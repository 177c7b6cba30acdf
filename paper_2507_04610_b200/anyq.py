"""Python mirror of the reference `anyq::` hot-path API, backed by the B200
C-ABI library (include/anyq_b200.h, paper_2507_04610_b200/_lib/libanyq_b200.so).

Names, argument meaning and error classes follow proj/include/anyq/*.hpp:

  quantize_any      learner.hpp:74          quantize / quantize_fixed  quantize.hpp:17-23
  pack_codes        pack.hpp:50             unpack_codes               pack.hpp:51
  to_ktiled         pack.hpp:86             from_ktiled                pack.hpp:87
  narrowed          pack.hpp:68             dequantize                 pack.hpp:98
  make_plan         qgemm.hpp:24            gemm_dense                 qgemm.hpp:28
  gemm_reference    qgemm.hpp:31            gemm_fused                 qgemm.hpp:36
  apply_format      quantize.hpp:33         storage_bits_per_entry     codebooks.hpp:53

Every call runs on the GPU. When the CUDA library or a device is missing the
calls raise (CudaError / OSError) — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._abi import (  # noqa: F401  (re-exported vocabulary)
    CB_ANY, CB_FP4, CB_INT, CB_NF4, G_BLOCK, G_COLUMN, G_GROUP, G_ROW, G_TENSOR,
    INIT_GRID, INIT_KMPP, INIT_NF4, INIT_RANDOM, LAYOUT_KTILED, LAYOUT_ROWMAJOR,
    STORE_BF16, STORE_FP16, STORE_FP32, W_ACTS, W_FULL, W_WEIGHTS, Config, default_config,
)
from .qtensor import QuantizedTensor

LIB_PATH = os.environ.get("ANYQ_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                     "libanyq_b200.so")


# ---------------------------------------------------------------------------
# errors (core.hpp:27-74)
# ---------------------------------------------------------------------------
class Error(RuntimeError):
    status = 11


class ShapeError(Error):
    status = 1


class ConfigError(Error):
    status = 2


class CodeRangeError(Error):
    status = 3


class NonFiniteError(Error):
    status = 4


class StatsError(Error):
    status = 5


class IoError(Error):
    status = 6


class MagicError(IoError):
    status = 7


class VersionError(IoError):
    status = 8


class TruncatedError(IoError):
    status = 9


class InvariantError(IoError):
    status = 10


class CudaError(Error):
    status = 12


_BY_STATUS = {
    c.status: c
    for c in (ShapeError, ConfigError, CodeRangeError, NonFiniteError, StatsError, IoError,
              MagicError, VersionError, TruncatedError, InvariantError, Error, CudaError)
}

_lib_handle = None


def lib() -> C.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib_handle
    if _lib_handle is not None:
        return _lib_handle
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} not built; run __graft_entry__.build() or make -C "
                      "paper_2507_04610_b200/csrc")
    L = C.CDLL(LIB_PATH)
    i64, i32, st = C.c_int64, C.c_int32, C.c_int
    fptr, u8 = C.POINTER(C.c_float), C.POINTER(C.c_uint8)
    cfg, qt = C.POINTER(_abi.Config), C.POINTER(_abi.QTensor)
    vp = C.c_void_p
    sigs = {
        "anyq_last_error": (C.c_char_p, []),
        "anyq_launch_count": (C.c_uint64, []),
        "anyq_config_default": (None, [cfg]),
        "anyq_packed_bytes_per_row": (i64, [i64, i32]),
        "anyq_num_groups": (i64, [cfg, i64, i64]),
        "anyq_lut_entries": (i64, [cfg]),
        "anyq_quantize_any": (st, [fptr, i64, i64, cfg, fptr, i64, qt]),
        "anyq_quantize_fixed": (st, [fptr, i64, i64, cfg, qt]),
        "anyq_pack_codes": (st, [u8, i64, i64, i32, u8]),
        "anyq_unpack_codes": (st, [u8, i64, i64, i32, u8]),
        "anyq_ktile_codes": (st, [u8, i64, i64, i32, i32, i32, u8]),
        "anyq_narrow_inplace": (st, [qt]),
        "anyq_dequantize": (st, [qt, fptr]),
        "anyq_gemm_fused": (st, [fptr, i64, qt, i32, i32, fptr]),
        "anyq_gemm_dense": (st, [fptr, i64, fptr, i64, i64, fptr]),
        "anyq_dev_tensor_create": (st, [qt, C.POINTER(vp)]),
        "anyq_dev_tensor_destroy": (None, [vp]),
        "anyq_dev_tensor_export": (st, [vp, qt]),
        "anyq_dev_tensor_config": (None, [vp, cfg]),
        "anyq_dev_tensor_weight_bytes": (i64, [vp]),
        "anyq_dev_tensor_rows": (i64, [vp]),
        "anyq_dev_tensor_cols": (i64, [vp]),
        "anyq_dev_gemm_bf16": (st, [vp, vp, i64, vp, vp, vp]),
        "anyq_dev_gemm_bf16_path": (st, [vp, vp, i64, vp, vp, i32, vp]),
        "anyq_dev_gemm_auto_path": (i32, [vp, i64]),
        "anyq_dev_gemm_chain": (st, [i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                     C.POINTER(vp), C.POINTER(i32), i64, vp]),
        "anyq_dev_gemm_chain_deps": (st, [i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                          C.POINTER(vp), C.POINTER(i32), i64, vp]),
        "anyq_dev_gemm_chain_path": (st, [i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                          C.POINTER(vp), C.POINTER(i32), i64, i32, vp]),
        "anyq_dev_quantize_any": (st, [vp, i64, i64, cfg, vp, i64, vp, vp, vp, vp, vp]),
        "anyq_dev_gemm_allgather": (st, [vp, vp, i64, C.POINTER(_abi.TpPeers), vp]),
        "anyq_dev_tp_wait": (st, [vp, C.POINTER(_abi.TpPeers), i32, vp]),
        "anyq_ipc_handle": (st, [vp, C.POINTER(C.c_uint8)]),
        "anyq_ipc_open": (st, [C.POINTER(C.c_uint8), C.POINTER(vp)]),
        "anyq_ipc_close": (st, [vp]),
        "anyq_column_mean_abs": (st, [fptr, i64, i64, fptr]),
        "anyq_write_file": (st, [qt, C.c_char_p]),
        "anyq_read_file_header": (st, [C.c_char_p, qt]),
        "anyq_read_file": (st, [C.c_char_p, qt]),
        "anyq_dev_tensor_load": (st, [C.c_char_p, C.POINTER(vp)]),
        "anyq_weight_error": (st, [fptr, i64, i64, qt, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "anyq_output_error": (st, [fptr, i64, i64, qt, fptr, i64, i64, C.POINTER(C.c_double)]),
        "anyq_dev_column_mean_abs": (st, [vp, i64, i64, vp, vp]),
        "anyq_dev_stream_status": (st, [vp]),
        "anyq_kmeans_problems": (st, [fptr, fptr, i64, i64, i32, cfg, i32, vp, vp,
                                      C.POINTER(C.c_double), u8, C.POINTER(C.c_double),
                                      C.POINTER(i32)]),
        "anyq_build_sample_weights": (st, [cfg, i64, i64, fptr, i64, i64, fptr, i64, i32, fptr]),
        "anyq_round_to_table": (st, [fptr, i64, i64, fptr, i32, u8]),
        "anyq_scaled_values": (st, [qt, fptr]),
        "anyq_fixed_table": (st, [i32, i32, i32, fptr, C.POINTER(i32)]),
        "anyq_f32_to_f16": (st, [C.c_float, C.POINTER(C.c_uint16)]),
        "anyq_f16_to_f32": (C.c_float, [C.c_uint16]),
        "anyq_f32_to_bf16": (st, [C.c_float, C.POINTER(C.c_uint16)]),
        "anyq_bf16_to_f32": (C.c_float, [C.c_uint16]),
        "anyq_storage_bits_per_entry": (st, [cfg, i64, i64, C.POINTER(C.c_double)]),
        "anyq_bench_gemm": (st, [i32, qt, fptr, i64, i64, fptr, i64, i32, C.POINTER(C.c_double)]),
        "anyq_eval_activations": (st, [i64, i64, fptr, C.c_uint64, fptr]),
        "anyq_compare_formats": (st, [fptr, i64, i64, C.c_char_p, cfg, fptr, i64, C.c_uint64,
                                      C.POINTER(C.c_double), C.POINTER(i32)]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib_handle = L
    return L


# Symbols include/anyq_b200.h declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = (
    "anyq_last_error", "anyq_config_default", "anyq_packed_bytes_per_row", "anyq_num_groups",
    "anyq_lut_entries", "anyq_quantize_any", "anyq_quantize_fixed", "anyq_pack_codes",
    "anyq_unpack_codes", "anyq_ktile_codes", "anyq_narrow_inplace", "anyq_dequantize",
    "anyq_gemm_fused", "anyq_gemm_dense", "anyq_dev_tensor_create", "anyq_dev_tensor_destroy",
    "anyq_dev_tensor_weight_bytes", "anyq_dev_tensor_export", "anyq_dev_tensor_config", "anyq_dev_tensor_rows", "anyq_dev_tensor_cols",
    "anyq_dev_gemm_bf16", "anyq_dev_gemm_bf16_path", "anyq_dev_gemm_chain",
    "anyq_dev_gemm_chain_deps", "anyq_dev_gemm_chain_path", "anyq_dev_gemm_auto_path",
    "anyq_dev_quantize_any", "anyq_eval_activations", "anyq_compare_formats",
    "anyq_dev_gemm_allgather", "anyq_dev_tp_wait", "anyq_ipc_handle", "anyq_ipc_open", "anyq_ipc_close",
    "anyq_launch_count",
    "anyq_compute_scales", "anyq_scale_weights", "anyq_dequantize_values",
    "anyq_column_mean_abs", "anyq_dev_column_mean_abs", "anyq_weight_error", "anyq_output_error",
    "anyq_write_file", "anyq_read_file_header", "anyq_read_file", "anyq_dev_tensor_load",
    "anyq_dev_stream_status", "anyq_kmeans_problems", "anyq_build_sample_weights",
    "anyq_round_to_table", "anyq_scaled_values", "anyq_fixed_table", "anyq_f32_to_f16",
    "anyq_f16_to_f32", "anyq_f32_to_bf16", "anyq_bf16_to_f32", "anyq_storage_bits_per_entry",
    "anyq_bench_gemm",
)


def _check(status: int):
    if status != 0:
        msg = lib().anyq_last_error().decode()
        raise _BY_STATUS.get(status, Error)(msg)


def launch_count() -> int:
    return int(lib().anyq_launch_count())


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------------------
# formats (quantize.cpp:34-64)
# ---------------------------------------------------------------------------
def apply_format(cfg: Config, fmt: str) -> Config:
    table = {
        "int2": (CB_INT, 2), "int3": (CB_INT, 3), "int4": (CB_INT, 4), "int8": (CB_INT, 8),
        "fp4": (CB_FP4, 4), "nf4": (CB_NF4, 4),
        "any2": (CB_ANY, 2), "any3": (CB_ANY, 3), "any4": (CB_ANY, 4), "any8": (CB_ANY, 8),
    }
    if fmt not in table:
        raise ConfigError(f"unknown format '{fmt}'")
    cfg.codebook, cfg.bits = table[fmt]
    return cfg


def format_name(cfg: Config) -> str:
    return {CB_INT: f"int{cfg.bits}", CB_FP4: "fp4", CB_NF4: "nf4", CB_ANY: f"any{cfg.bits}"}[
        cfg.codebook]


def storage_bits_per_entry(cfg: Config, rows: int, cols: int) -> float:
    """codebooks.cpp:99-121 storage_bits_per_entry (anyq_storage_bits_per_entry)."""
    out = C.c_double()
    _check(lib().anyq_storage_bits_per_entry(C.byref(cfg), rows, cols, C.byref(out)))
    return out.value


def fixed_table(codebook: int, bits: int = 4, shifted: bool = False) -> np.ndarray:
    """codebooks.cpp:8-55 int_grid / fp4_table / nf4_table (nominal values)."""
    v = np.empty(256, np.float32)
    n = C.c_int32()
    _check(lib().anyq_fixed_table(codebook, bits, int(shifted), _abi.fp(v), C.byref(n)))
    return v[: n.value].copy()


def round_to_codebook(ws, table) -> np.ndarray:
    """codebooks.cpp:75-97 round_to_codebook on the GPU (ties to the lower index)."""
    ws = _f32(ws)
    t = _f32(table).ravel()
    codes = np.empty(ws.shape, np.uint8)
    _check(lib().anyq_round_to_table(_abi.fp(ws), ws.shape[0], ws.shape[1], _abi.fp(t), t.size,
                                     _abi.u8p(codes)))
    return codes


def f32_to_f16(f: float) -> int:
    """pack.cpp:61-101 RNE narrowing (NonFiniteError / IoError on overflow)."""
    h = C.c_uint16()
    _check(lib().anyq_f32_to_f16(C.c_float(f), C.byref(h)))
    return h.value


def f32_to_bf16(f: float) -> int:
    h = C.c_uint16()
    _check(lib().anyq_f32_to_bf16(C.c_float(f), C.byref(h)))
    return h.value


def f16_to_f32(h: int) -> float:
    return lib().anyq_f16_to_f32(h)


def bf16_to_f32(h: int) -> float:
    return lib().anyq_bf16_to_f32(h)


# ---------------------------------------------------------------------------
# the per-row learner (learner.hpp:30-68) on the GPU
# ---------------------------------------------------------------------------
_M64 = (1 << 64) - 1


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def rng_for_row(seed: int, row: int) -> list:
    """core.hpp:196-200: the Rng state [key, counter] of stream (seed, row)."""
    return [_splitmix64(seed) ^ _splitmix64((0x9E3779B97F4A7C15 * (row + 1)) & _M64), 0]


def _km(x, w, k, cfg: Config | None, mode: int, rng):
    x = np.ascontiguousarray(x, np.float32).ravel()
    w = np.ascontiguousarray(w, np.float32).ravel()
    if x.size != w.size:
        raise ShapeError("KmProblem: samples and weights differ in length")
    c = cfg if cfg is not None else _abi.default_config(codebook=CB_ANY)
    key = np.array([rng[0]], np.uint64)
    ctr = np.array([rng[1]], np.uint64)
    cen = np.empty(max(k, 1), np.float64)
    asg = np.empty(max(x.size, 1), np.uint8)
    loss = C.c_double()
    iters = C.c_int32()
    _check(lib().anyq_kmeans_problems(
        _abi.fp(x), _abi.fp(w), 1, x.size, k, C.byref(c), mode,
        key.ctypes.data_as(C.c_void_p), ctr.ctypes.data_as(C.c_void_p), _abi.f64p(cen),
        _abi.u8p(asg), C.byref(loss), C.byref(iters)))
    rng[1] = int(ctr[0])
    return cen[:k], asg[:x.size], loss.value, iters.value


def kmeans_pp_init(x, w, k: int, rng) -> np.ndarray:
    """learner.hpp:55 kmeans_pp_init; `rng` = [key, counter] (advanced in place)."""
    return _km(x, w, k, None, 2, rng)[0]


def weighted_kmeans(x, w, k: int, cfg: Config, rng):
    """learner.hpp:61 weighted_kmeans -> (centroids f64, assignments, loss, iters)."""
    return _km(x, w, k, cfg, 1, rng)


def learn_row_lut(x, w, bits: int, cfg: Config, rng):
    """learner.hpp:66 learn_row_lut -> (sorted LUT f32, codes, loss)."""
    cen, codes, loss, _ = _km(x, w, 1 << bits, cfg, 0, rng)
    return cen.astype(np.float32), codes, loss


def build_sample_weights(cfg: Config, rows: int, cols: int, alphas, row: int, stats=None,
                         weighting: int | None = None) -> np.ndarray:
    """learner.hpp:45 build_sample_weights for the scale set (cfg's group map)."""
    a = _f32(alphas).ravel()
    st = None if stats is None else _f32(stats).ravel()
    out = np.empty(cols, np.float32)
    mode = cfg.weighting if weighting is None else weighting
    _check(lib().anyq_build_sample_weights(
        C.byref(cfg), rows, cols, _abi.fp(a), a.size, row, None if st is None else _abi.fp(st),
        0 if st is None else st.size, mode, _abi.fp(out)))
    return out


# ---------------------------------------------------------------------------
# quantization
# ---------------------------------------------------------------------------
def quantize_any(w, cfg: Config, exj=None, row_offset: int = 0) -> QuantizedTensor:
    w = _f32(w)
    rows, cols = w.shape
    qt = QuantizedTensor.empty(rows, cols, cfg)
    c = qt.as_c()
    e = None if exj is None else _f32(exj)
    if e is not None and e.size != cols:
        raise StatsError(f"sample weights: stats length {e.size} does not match row length {cols}")
    _check(lib().anyq_quantize_any(_abi.fp(w), rows, cols, C.byref(qt.cfg),
                                   None if e is None else _abi.fp(e), row_offset, C.byref(c)))
    return qt


def quantize_fixed(w, cfg: Config) -> QuantizedTensor:
    w = _f32(w)
    rows, cols = w.shape
    qt = QuantizedTensor.empty(rows, cols, cfg)
    c = qt.as_c()
    _check(lib().anyq_quantize_fixed(_abi.fp(w), rows, cols, C.byref(qt.cfg), C.byref(c)))
    return qt


def quantize(w, cfg: Config, stats: dict | None = None, module_name: str = "",
             threads: int = 1) -> QuantizedTensor:
    """quantize.cpp:25-32; `stats` maps module name -> E|x_j| (ActivationStats)."""
    if cfg.codebook != CB_ANY:
        return quantize_fixed(w, cfg)
    exj = None
    if stats is not None:
        if module_name not in stats:
            raise StatsError(f"no activation stats for module '{module_name}'")
        exj = _f32(stats[module_name])
        if exj.size != np.shape(w)[1]:
            raise StatsError("activation stats channel count mismatch")
    return quantize_any(w, cfg, exj)


# ---------------------------------------------------------------------------
# packing / layout / dequant
# ---------------------------------------------------------------------------
def pack_codes(codes, bits: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, np.uint8)
    rows, cols = codes.shape
    out = np.zeros(rows * _abi.packed_bytes_per_row(cols, bits), np.uint8)
    _check(lib().anyq_pack_codes(_abi.u8p(codes), rows, cols, bits, _abi.u8p(out)))
    return out


def unpack_codes(packed, rows: int, cols: int, bits: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, np.uint8)
    if packed.size != rows * _abi.packed_bytes_per_row(cols, bits):
        raise ShapeError("unpack_codes: packed size does not match shape")
    out = np.zeros((rows, cols), np.uint8)
    _check(lib().anyq_unpack_codes(_abi.u8p(packed), rows, cols, bits, _abi.u8p(out)))
    return out


def _retile(qt: QuantizedTensor, tile_k: int, inverse: int) -> np.ndarray:
    out = np.empty_like(qt.codes)
    _check(lib().anyq_ktile_codes(_abi.u8p(qt.codes), qt.rows, qt.cols, qt.cfg.bits, tile_k,
                                  inverse, _abi.u8p(out)))
    return out


def from_ktiled(qt: QuantizedTensor) -> QuantizedTensor:
    if qt.layout == LAYOUT_ROWMAJOR:
        return qt
    out = qt.clone()
    out.codes = _retile(qt, qt.tile_k, 1)
    out.layout, out.tile_k = LAYOUT_ROWMAJOR, 1
    return out


def to_ktiled(qt: QuantizedTensor, tile_k: int) -> QuantizedTensor:
    if tile_k < 1:
        raise ConfigError("tile_k must be >= 1")
    src = from_ktiled(qt) if qt.layout == LAYOUT_KTILED else qt
    out = src.clone()
    out.codes = _retile(src, tile_k, 0)
    out.layout, out.tile_k = LAYOUT_KTILED, tile_k
    return out


def narrowed(qt: QuantizedTensor) -> QuantizedTensor:
    out = qt.clone()
    c = out.as_c()
    _check(lib().anyq_narrow_inplace(C.byref(c)))
    return out


def scaled_values(qt: QuantizedTensor) -> np.ndarray:
    """pack.cpp:205-236: the table value of every code (before alpha / beta)."""
    out = np.empty((qt.rows, qt.cols), np.float32)
    c = qt.as_c()
    _check(lib().anyq_scaled_values(C.byref(c), _abi.fp(out)))
    return out


def bench_gemm(kind: int, qt: QuantizedTensor | None, w, x, repeats: int) -> np.ndarray:
    """qgemm.cpp bench's timing loop on the device (anyq_bench_gemm): per-run ns.
    kind 0: fp32 gemm_dense(x, w); 1: exact gemm_fused on qt; 2: A16W4 LUT GEMM."""
    x = _f32(x)
    ns = np.empty(repeats, np.float64)
    if kind == 0:
        w = _f32(w)
        n, k = w.shape
        _check(lib().anyq_bench_gemm(0, None, _abi.fp(w), n, k, _abi.fp(x), x.shape[0], repeats,
                                     _abi.f64p(ns)))
    else:
        c = qt.as_c()
        _check(lib().anyq_bench_gemm(kind, C.byref(c), None, qt.rows, qt.cols, _abi.fp(x),
                                     x.shape[0], repeats, _abi.f64p(ns)))
    return ns


def dequantize(qt: QuantizedTensor) -> np.ndarray:
    out = np.empty((qt.rows, qt.cols), np.float32)
    c = qt.as_c()
    _check(lib().anyq_dequantize(C.byref(c), _abi.fp(out)))
    return out


def write_file(qt: QuantizedTensor, path) -> None:
    """pack.cpp:293-345 write_file: byte-identical ANYQ v1 file (lut_store / scale_store of qt)."""
    c = qt.as_c()
    _check(lib().anyq_write_file(C.byref(c), os.fsencode(path)))


def read_file(path) -> QuantizedTensor:
    """pack.cpp:347-471 read_file, with every check of the reference in its order."""
    p = os.fsencode(path)
    h = _abi.QTensor()
    _check(lib().anyq_read_file_header(p, C.byref(h)))
    qt = QuantizedTensor.empty(int(h.rows), int(h.cols), h.cfg)
    qt.layout, qt.tile_k, qt.lut_store, qt.scale_store = h.layout, h.tile_k, h.lut_store, h.scale_store
    c = qt.as_c()
    _check(lib().anyq_read_file(p, C.byref(c)))
    qt.cfg = _abi.Config.from_buffer_copy(bytes(c.cfg))
    return qt


def weight_error(w, qt: QuantizedTensor):
    """eval.cpp:11-29: (mse, relative Frobenius error) of dequantize(qt) against w."""
    w = _f32(w)
    mse, rel = C.c_double(), C.c_double()
    c = qt.as_c()
    _check(lib().anyq_weight_error(_abi.fp(w), w.shape[0], w.shape[1], C.byref(c), C.byref(mse),
                                   C.byref(rel)))
    return mse.value, rel.value


def output_error(w, qt: QuantizedTensor, x) -> float:
    """eval.cpp:31-46: mean squared error of gemm_reference(x, qt) against gemm_dense(x, w)."""
    w, x = _f32(w), _f32(x)
    mse = C.c_double()
    c = qt.as_c()
    _check(lib().anyq_output_error(_abi.fp(w), w.shape[0], w.shape[1], C.byref(c), _abi.fp(x),
                                   x.shape[0], x.shape[1], C.byref(mse)))
    return mse.value


# ---------------------------------------------------------------------------
# GEMM
# ---------------------------------------------------------------------------
@dataclass
class GemmPlan:
    """qgemm.hpp:16-22."""

    m: int
    n: int
    k: int
    layout: int = LAYOUT_ROWMAJOR
    tile_k: int = 1


def make_plan(x, qt: QuantizedTensor) -> GemmPlan:
    x = np.asarray(x)
    return GemmPlan(m=x.shape[0], n=qt.rows, k=qt.cols, layout=qt.layout, tile_k=qt.tile_k)


def gemm_dense(x, w) -> np.ndarray:
    x, w = _f32(x), _f32(w)
    if x.shape[1] != w.shape[1]:
        raise ShapeError("gemm: reduction dimensions differ")
    y = np.empty((x.shape[0], w.shape[0]), np.float32)
    _check(lib().anyq_gemm_dense(_abi.fp(x), x.shape[0], _abi.fp(w), w.shape[0], w.shape[1],
                                 _abi.fp(y)))
    return y


def gemm_reference(x, qt: QuantizedTensor) -> np.ndarray:
    x = _f32(x)
    if x.shape[1] != qt.cols:
        raise ShapeError("gemm_reference: reduction dimensions differ")
    return gemm_dense(x, dequantize(qt))


def gemm_fused(x, qt: QuantizedTensor, plan: GemmPlan | None = None) -> np.ndarray:
    """Bit-exact LUT GEMM on the GPU (same k-ascending fp32 order as qgemm.cpp)."""
    x = _f32(x)
    if x.shape[1] != qt.cols:
        raise ShapeError("gemm_fused: reduction dimensions differ")
    plan = plan or make_plan(x, qt)
    if plan.m != x.shape[0] or plan.n != qt.rows or plan.k != qt.cols:
        raise ShapeError("gemm_fused: plan does not match operands")
    y = np.empty((x.shape[0], qt.rows), np.float32)
    c = qt.as_c()
    _check(lib().anyq_gemm_fused(_abi.fp(x), x.shape[0], C.byref(c), plan.layout, plan.tile_k,
                                 _abi.fp(y)))
    return y


# ---------------------------------------------------------------------------
# device-resident fast path (LUT GEMV / tensor-core LUT GEMM)
PATH_AUTO, PATH_GEMV, PATH_TC, PATH_DEQUANT, PATH_MMA, PATH_GEMV_TC, PATH_K2 = 0, 1, 2, 3, 4, 5, 6
# ---------------------------------------------------------------------------
class DeviceTensor:
    """A prepacked any4/int4/nf4/fp4 weight resident in HBM.

    `gemm(x, y, y32=None, stream=None)` takes torch CUDA tensors (bf16 x of
    shape [m, cols], bf16 y of shape [m, rows]) and launches the tcgen05 LUT
    GEMM on `stream` (default: torch's current stream).
    """

    def __init__(self, qt: QuantizedTensor):
        self._h = C.c_void_p()
        c = qt.as_c()
        _check(lib().anyq_dev_tensor_create(C.byref(c), C.byref(self._h)))
        self.rows, self.cols = qt.rows, qt.cols
        self.weight_bytes = int(lib().anyq_dev_tensor_weight_bytes(self._h))

    @classmethod
    def load(cls, path) -> "DeviceTensor":
        """An ANYQ v1 file straight into the prepacked device layout (read_file's checks)."""
        self = cls.__new__(cls)
        self._h = C.c_void_p()
        _check(lib().anyq_dev_tensor_load(os.fsencode(path), C.byref(self._h)))
        self.rows = int(lib().anyq_dev_tensor_rows(self._h))
        self.cols = int(lib().anyq_dev_tensor_cols(self._h))
        self.weight_bytes = int(lib().anyq_dev_tensor_weight_bytes(self._h))
        return self

    def close(self):
        if self._h:
            lib().anyq_dev_tensor_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self) -> QuantizedTensor:
        """prepack^-1: the tensor back in the reference layout (narrowed values)."""
        cfg = _abi.Config()
        lib().anyq_dev_tensor_config(self._h, C.byref(cfg))
        out = QuantizedTensor.empty(self.rows, self.cols, cfg)
        c = out.as_c()
        _check(lib().anyq_dev_tensor_export(self._h, C.byref(c)))
        out.cfg = c.cfg
        out.lut_store, out.scale_store, out.layout = c.lut_store, c.scale_store, c.layout
        return out

    def auto_path(self, m: int) -> int:
        """The kernel PATH_AUTO runs at m rows of x (PATH_GEMV / PATH_TC / PATH_DEQUANT)."""
        return int(lib().anyq_dev_gemm_auto_path(self._h, m))

    def gemm_ptr(self, x_ptr: int, m: int, y_ptr: int, y32_ptr: int | None, stream: int,
                 path: int = 0):
        _check(lib().anyq_dev_gemm_bf16_path(self._h, C.c_void_p(x_ptr), m, C.c_void_p(y_ptr),
                                             C.c_void_p(y32_ptr) if y32_ptr else None, path,
                                             C.c_void_p(stream)))

    def gemm(self, x, y=None, y32=None, stream=None, path: int = 0):
        import torch

        assert x.is_cuda and x.dtype == torch.bfloat16 and x.is_contiguous()
        m = x.shape[0]
        if x.shape[1] != self.cols:
            raise ShapeError("gemm: reduction dimensions differ")
        if y is None:
            y = torch.empty((m, self.rows), dtype=torch.bfloat16, device=x.device)
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        self.gemm_ptr(x.data_ptr(), m, y.data_ptr(), y32.data_ptr() if y32 is not None else None,
                      s.cuda_stream, path)
        return y


def gemm_chain_ptrs(tensors, x_ptrs, y_ptrs, m: int, stream: int, wait_prev=None, y32_ptrs=None,
                    deps=None, path=None):
    """One launch of y_i = x_i W_i^T for a list of DeviceTensors.

    deps[i] = j (< i) makes problem i read x_i only after problem j completed
    (x_i is y_j); -1 = no dependency (anyq_dev_gemm_chain_deps). The older
    wait_prev[i] = 1 waits for every earlier problem (anyq_dev_gemm_chain).
    Pointers are raw device addresses. path (PATH_GEMV / PATH_GEMV_TC /
    PATH_AUTO) picks the chain engine (anyq_dev_gemm_chain_path).
    """
    n = len(tensors)
    VP = C.c_void_p * n
    t = VP(*[d._h.value for d in tensors])
    xs = VP(*x_ptrs)
    ys = VP(*y_ptrs)
    y32 = VP(*[p or 0 for p in y32_ptrs]) if y32_ptrs is not None else None
    if path is not None:
        if deps is None:
            deps = [i - 1 if (wait_prev and i > 0 and wait_prev[i]) else -1 for i in range(n)]
        d = (C.c_int32 * n)(*deps)
        _check(lib().anyq_dev_gemm_chain_path(n, t, xs, ys, y32, d, m, path, C.c_void_p(stream)))
        return
    if deps is not None:
        d = (C.c_int32 * n)(*deps)
        _check(lib().anyq_dev_gemm_chain_deps(n, t, xs, ys, y32, d, m, C.c_void_p(stream)))
        return
    w = (C.c_int32 * n)(*(wait_prev or [0] * n))
    _check(lib().anyq_dev_gemm_chain(n, t, xs, ys, y32, w, m, C.c_void_p(stream)))


def gemm_chain(tensors, xs, ys=None, wait_prev=None, y32s=None, stream=None, deps=None,
               path=None):
    """gemm_chain_ptrs on torch CUDA tensors; returns the list of y (bf16)."""
    import torch

    m = xs[0].shape[0]
    if ys is None:
        ys = [torch.empty((m, d.rows), dtype=torch.bfloat16, device=xs[0].device) for d in tensors]
    s = stream if stream is not None else torch.cuda.current_stream(xs[0].device)
    gemm_chain_ptrs(tensors, [x.data_ptr() for x in xs], [y.data_ptr() for y in ys], m,
                    s.cuda_stream, wait_prev,
                    [y.data_ptr() for y in y32s] if y32s is not None else None, deps, path)
    return ys


def eval_activations(rows: int, cols: int, exj=None, seed: int = 1) -> np.ndarray:
    """eval_activations (eval.cpp:48-61): N(0, E|x_j| sqrt(pi/2)) per channel."""
    out = np.empty((rows, cols), np.float32)
    e = _abi.fp(_f32(exj)) if exj is not None else None
    _check(lib().anyq_eval_activations(rows, cols, e, seed, _abi.fp(out)))
    return out


def compare_formats(w, formats, base, exj=None, eval_rows: int = 64, eval_seed: int = 1,
                    module: str = "w"):
    """compare_formats (eval.cpp:62-86) on the GPU: one row per format with
    weight_mse, weight_rel_frobenius, output_mse, bits_per_entry; returns
    (rows as a list of dicts, the report CSV of EvalReport::to_csv)."""
    w = _f32(w)
    out = np.zeros((len(formats), 4), np.float64)
    n = C.c_int32(0)
    e = _abi.fp(_f32(exj)) if exj is not None else None
    _check(lib().anyq_compare_formats(_abi.fp(w), w.shape[0], w.shape[1], ",".join(formats).encode(),
                                      C.byref(base), e, eval_rows, eval_seed,
                                      out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n)))
    rows = [dict(module=module, format=f, weight_mse=o[0], weight_rel_frobenius=o[1], output_mse=o[2],
                 bits_per_entry=o[3]) for f, o in zip(formats, out)]
    lines = ["schema_version,module,format,weight_mse,weight_rel_frobenius,output_mse,bits_per_entry"]
    lines += [f"v1,{r['module']},{r['format']},{r['weight_mse']:.9g},{r['weight_rel_frobenius']:.9g},"
              f"{r['output_mse']:.9g},{r['bits_per_entry']:.9g}" for r in rows]
    return rows, "\n".join(lines) + "\n"


def tp_peers(world: int, rank: int, rows_total: int, row0: int, y_ptrs, flag_ptrs) -> "_abi.TpPeers":
    """anyq_tp_peers of this rank (device pointers valid on this device)."""
    p = _abi.TpPeers()
    p.world, p.rank, p.rows_total, p.row0 = world, rank, rows_total, row0
    for r in range(world):
        p.y[r] = y_ptrs[r]
        p.flags[r] = flag_ptrs[r]
    return p


def gemm_allgather(shard: "DeviceTensor", x, peers, stream=None):
    """y_r = x W_r^T of this rank's row shard, stored into every rank's y (fused gather)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    _check(lib().anyq_dev_gemm_allgather(shard._h, C.c_void_p(x.data_ptr()), x.shape[0], C.byref(peers),
                                         C.c_void_p(s.cuda_stream)))


def tp_wait(shard: "DeviceTensor", peers, epoch: int, stream=None):
    """Make the stream wait until every rank's contribution of call `epoch` landed."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().anyq_dev_tp_wait(shard._h, C.byref(peers), epoch, C.c_void_p(s.cuda_stream)))


def ipc_handle(ptr: int) -> bytes:
    h = (C.c_uint8 * 64)()
    _check(lib().anyq_ipc_handle(C.c_void_p(ptr), h))
    return bytes(h)


def ipc_open(handle: bytes) -> int:
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    _check(lib().anyq_ipc_open(h, C.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(lib().anyq_ipc_close(C.c_void_p(ptr)))


def column_mean_abs(x) -> np.ndarray:
    """E|x_j| over M x K activations: the per-layer statistic of collect_stats
    (calibration.cpp:62-67), computed on the GPU, bit-identical to the reference."""
    x = _f32(x)
    if x.ndim != 2:
        raise ShapeError("activations must be a 2-D (samples x channels) array")
    out = np.empty(x.shape[1], np.float32)
    _check(lib().anyq_column_mean_abs(_abi.fp(x), x.shape[0], x.shape[1], _abi.fp(out)))
    return out


def dev_stream_status(stream=None):
    """Synchronise the stream and raise the first data error the stream-ordered
    entries recorded on the device (anyq_dev_stream_status)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().anyq_dev_stream_status(C.c_void_p(s.cuda_stream)))


def dev_column_mean_abs(x, out=None, stream=None, check=True):
    """column_mean_abs on a contiguous fp32 CUDA tensor; returns the (K,) fp32 tensor.
    Stream ordered; check=True synchronises and raises a recorded data error."""
    import torch

    assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.dim() == 2
    if out is None:
        out = torch.empty(x.shape[1], dtype=torch.float32, device=x.device)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    _check(lib().anyq_dev_column_mean_abs(C.c_void_p(x.data_ptr()), x.shape[0], x.shape[1],
                                          C.c_void_p(out.data_ptr()), C.c_void_p(s.cuda_stream)))
    if check:
        dev_stream_status(s)
    return out


def dev_quantize_any(w, cfg: Config, exj=None, row_offset: int = 0, stream=None, check=True):
    """Device-resident quantize_any on torch CUDA tensors.

    Returns (codes uint8 [rows, bpr], luts f32 [rows, 2^bits], alphas, betas)
    as torch tensors in the reference layout. Stream ordered (capturable);
    check=True synchronises and raises a data error recorded on the device.
    """
    import torch

    assert w.is_cuda and w.dtype == torch.float32 and w.is_contiguous()
    rows, cols = w.shape
    dev = w.device
    ng = _abi.num_groups(cfg, rows, cols)
    codes = torch.empty((rows, _abi.packed_bytes_per_row(cols, cfg.bits)), dtype=torch.uint8,
                        device=dev)
    luts = torch.empty((rows, 1 << cfg.bits), dtype=torch.float32, device=dev)
    alphas = torch.empty(ng, dtype=torch.float32, device=dev)
    betas = torch.empty(ng, dtype=torch.float32, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    _check(lib().anyq_dev_quantize_any(
        C.c_void_p(w.data_ptr()), rows, cols, C.byref(cfg),
        C.c_void_p(exj.data_ptr()) if exj is not None else None, row_offset,
        C.c_void_p(codes.data_ptr()), C.c_void_p(luts.data_ptr()), C.c_void_p(alphas.data_ptr()),
        C.c_void_p(betas.data_ptr()), C.c_void_p(s.cuda_stream)))
    if check:
        dev_stream_status(s)
    return codes, luts, alphas, betas
