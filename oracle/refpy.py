"""TEST INFRASTRUCTURE ONLY — numpy front end over the two CPU oracles.

* ``Ref``    : the unmodified reference (oracle/_ref/libanyq_ref.so, built by
               oracle/Makefile from /root/reference/proj/src in place).
* ``Oracle`` : the C restatement (oracle/_build/liboracle.so, anyq_oracle.c).

Both expose the same methods with the same signatures so tests can pin one
against the other. Only tests/, __graft_entry__.smoke() and bench.py's CPU
legs may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

from paper_2507_04610_b200 import _abi
from paper_2507_04610_b200.qtensor import QuantizedTensor

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libanyq_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")


class OracleError(Exception):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.kind = _abi.STATUS_NAMES.get(status, "Error")
        super().__init__(f"{self.kind}: {msg}")


def fnv1a64(data: bytes) -> str:
    """FNV-1a-64 fingerprint used in SURVEY.md §8(c)."""
    h = 0xCBF29CE484222325
    arr = np.frombuffer(data, np.uint8)
    # vectorised in chunks would change semantics; FNV is sequential.
    for b in arr.tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle`")
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        i64, i32, u64 = C.c_int64, C.c_int, C.c_uint64
        fptr = C.POINTER(C.c_float)
        dptr = C.POINTER(C.c_double)
        u8 = C.POINTER(C.c_uint8)
        qt = C.POINTER(_abi.QTensor)
        cfg = C.POINTER(_abi.Config)
        sig = {
            "last_error": (C.c_char_p, []),
            "quantize": (i32, [fptr, i64, i64, cfg, fptr, i32, qt]),
            "narrowed": (i32, [qt]),
            "dequantize": (i32, [qt, fptr]),
            "gemm_reference": (i32, [fptr, i64, qt, fptr]),
            "gemm_fused": (i32, [fptr, i64, i64, qt, i32, i32, fptr]),
            "gemm_dense": (i32, [fptr, i64, fptr, i64, i64, fptr]),
            "column_mean_abs": (i32, [fptr, i64, i64, fptr]),
            "write_file": (i32, [qt, C.c_char_p]),
            "read_file": (i32, [C.c_char_p, qt]),
            "weight_error": (i32, [fptr, qt, dptr, dptr]),
            "output_error": (i32, [fptr, qt, fptr, i64, dptr]),
            "pack_codes": (i32, [u8, i64, i64, i32, u8]),
            "unpack_codes": (i32, [u8, i64, i64, i32, u8]),
            "to_ktiled": (i32, [qt, i32, u8]),
            "from_ktiled": (i32, [qt, u8]),
            "f32_to_f16": (i32, [C.c_float, C.POINTER(C.c_uint16)]),
            "f16_to_f32": (C.c_float, [C.c_uint16]),
            "f32_to_bf16": (i32, [C.c_float, C.POINTER(C.c_uint16)]),
            "bf16_to_f32": (C.c_float, [C.c_uint16]),
            "storage_bits_per_entry": (C.c_double, [cfg, i64, i64]),
            "kmeans_pp_init": (i32, [fptr, fptr, i64, i32, u64, i64, dptr]),
            "weighted_kmeans": (
                i32,
                [fptr, fptr, i64, i32, cfg, u64, i64, dptr, u8, dptr, C.POINTER(C.c_int)],
            ),
            "learn_row_lut": (i32, [fptr, fptr, i64, i32, cfg, u64, i64, fptr, u8, dptr]),
            "gaussian": (None, [i64, i64, u64, C.c_float, fptr]),
            "uniform": (None, [i64, i64, u64, C.c_float, C.c_float, fptr]),
            "dyadic": (None, [i64, i64, u64, i32, C.c_float, fptr]),
            "heavy_tailed": (None, [i64, i64, u64, C.c_float, C.c_float, fptr]),
            "synthetic_stats": (None, [i64, u64, fptr]),
            "rng_u64": (None, [u64, i64, i64, C.POINTER(C.c_uint64)]),
            "rng_double": (None, [u64, i64, i64, dptr]),
            "collect_stats": (i32, [fptr, i64, i64, fptr]),
            "bench": (i32, [i32, C.POINTER(C.c_int64), C.c_char_p, i32, u64, dptr, C.POINTER(C.c_int),
                            C.POINTER(C.c_int)]),
            "eval_activations": (i32, [i64, i64, fptr, u64, fptr]),
            "compare_formats": (i32, [fptr, i64, i64, C.c_char_p, cfg, fptr, i64, u64, i32, dptr,
                                      C.c_char_p, i64]),
        }
        self.fn = {}
        for name, (res, args) in sig.items():
            f = getattr(L, p + name, None)
            if f is None:
                continue
            f.restype = res
            f.argtypes = args
            self.fn[name] = f
        if hasattr(L, p + "time_quantize"):
            f = getattr(L, p + "time_quantize")
            f.restype = i32
            f.argtypes = [fptr, i64, i64, cfg, fptr, i32, dptr]
            self.fn["time_quantize"] = f
        if hasattr(L, p + "time_gemm_fused"):
            f = getattr(L, p + "time_gemm_fused")
            f.restype = i32
            f.argtypes = [fptr, i64, qt, i32, dptr]
            self.fn["time_gemm_fused"] = f

    # -- helpers -----------------------------------------------------------
    def _check(self, st: int):
        if st != 0:
            raise OracleError(st, self.fn["last_error"]().decode())

    # -- generators (helpers.hpp) -------------------------------------------
    def gaussian(self, rows, cols, seed, scale=1.0):
        out = np.empty((rows, cols), np.float32)
        self.fn["gaussian"](rows, cols, seed, scale, _abi.fp(out))
        return out

    def uniform(self, rows, cols, seed, lo, hi):
        out = np.empty((rows, cols), np.float32)
        self.fn["uniform"](rows, cols, seed, lo, hi, _abi.fp(out))
        return out

    def dyadic(self, rows, cols, seed, span=1024, step=1.0 / 1024.0):
        out = np.empty((rows, cols), np.float32)
        self.fn["dyadic"](rows, cols, seed, span, step, _abi.fp(out))
        return out

    def heavy_tailed(self, rows, cols, seed, rate=0.01, gain=8.0):
        out = np.empty((rows, cols), np.float32)
        self.fn["heavy_tailed"](rows, cols, seed, rate, gain, _abi.fp(out))
        return out

    def synthetic_stats(self, cols, seed):
        out = np.empty(cols, np.float32)
        self.fn["synthetic_stats"](cols, seed, _abi.fp(out))
        return out

    def rng_u64(self, seed, row, n):
        out = np.empty(n, np.uint64)
        self.fn["rng_u64"](seed, row, n, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return out

    def rng_double(self, seed, row, n):
        out = np.empty(n, np.float64)
        self.fn["rng_double"](seed, row, n, _abi.f64p(out))
        return out

    # -- quantization -------------------------------------------------------
    def quantize(self, w, cfg, exj=None, threads=1) -> QuantizedTensor:
        w = np.ascontiguousarray(w, np.float32)
        rows, cols = w.shape
        qt = QuantizedTensor.empty(rows, cols, cfg)
        c = qt.as_c()
        e = None if exj is None else np.ascontiguousarray(exj, np.float32)
        self._check(
            self.fn["quantize"](
                _abi.fp(w), rows, cols, C.byref(qt.cfg), None if e is None else _abi.fp(e),
                threads, C.byref(c)
            )
        )
        return qt

    def time_quantize(self, w, cfg, exj=None, threads=1) -> float:
        w = np.ascontiguousarray(w, np.float32)
        secs = C.c_double()
        e = None if exj is None else np.ascontiguousarray(exj, np.float32)
        self._check(
            self.fn["time_quantize"](
                _abi.fp(w), w.shape[0], w.shape[1], C.byref(cfg),
                None if e is None else _abi.fp(e), threads, C.byref(secs)
            )
        )
        return secs.value

    def narrowed(self, qt: QuantizedTensor) -> QuantizedTensor:
        out = qt.clone()
        c = out.as_c()
        self._check(self.fn["narrowed"](C.byref(c)))
        return out

    def dequantize(self, qt: QuantizedTensor) -> np.ndarray:
        out = np.empty((qt.rows, qt.cols), np.float32)
        c = qt.as_c()
        self._check(self.fn["dequantize"](C.byref(c), _abi.fp(out)))
        return out

    def gemm_reference(self, x, qt: QuantizedTensor) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty((x.shape[0], qt.rows), np.float32)
        c = qt.as_c()
        self._check(self.fn["gemm_reference"](_abi.fp(x), x.shape[0], C.byref(c), _abi.fp(y)))
        return y

    def gemm_fused(self, x, qt: QuantizedTensor, layout=None, tile_k=None) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty((x.shape[0], qt.rows), np.float32)
        c = qt.as_c()
        layout = qt.layout if layout is None else layout
        tile_k = qt.tile_k if tile_k is None else tile_k
        self._check(
            self.fn["gemm_fused"](
                _abi.fp(x), x.shape[0], x.shape[1], C.byref(c), layout, tile_k, _abi.fp(y)
            )
        )
        return y

    def time_gemm_fused(self, x, qt: QuantizedTensor, repeats=5) -> float:
        x = np.ascontiguousarray(x, np.float32)
        secs = C.c_double()
        c = qt.as_c()
        self._check(
            self.fn["time_gemm_fused"](_abi.fp(x), x.shape[0], C.byref(c), repeats, C.byref(secs))
        )
        return secs.value

    def gemm_dense(self, x, w) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        y = np.empty((x.shape[0], w.shape[0]), np.float32)
        self._check(
            self.fn["gemm_dense"](_abi.fp(x), x.shape[0], _abi.fp(w), w.shape[0], w.shape[1],
                                  _abi.fp(y))
        )
        return y

    def column_mean_abs(self, x) -> np.ndarray:
        """E|x_j| of collect_stats (calibration.cpp:62-67) over M x K activations."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(x.shape[1], np.float32)
        self._check(self.fn["column_mean_abs"](_abi.fp(x), x.shape[0], x.shape[1], _abi.fp(out)))
        return out

    def write_file(self, qt: QuantizedTensor, path) -> None:
        """pack.cpp:293-345 (reference build only)."""
        c = qt.as_c()
        self._check(self.fn["write_file"](C.byref(c), os.fsencode(path)))

    def read_file(self, path, like: QuantizedTensor) -> QuantizedTensor:
        """pack.cpp:347-471 (reference build only); `like` supplies the array sizes."""
        out = like.clone()
        c = out.as_c()
        self._check(self.fn["read_file"](os.fsencode(path), C.byref(c)))
        out.layout, out.tile_k, out.lut_store, out.scale_store = c.layout, c.tile_k, c.lut_store, c.scale_store
        return out

    def bench(self, shapes, formats, repeats=3, seed=1):
        """qgemm.cpp bench(): [(shape, format, layout, median, p10, p90, bytes_per_weight)]."""
        mnk = (C.c_int64 * (3 * len(shapes)))(*[v for s in shapes for v in s])
        nmax = len(shapes) * (len(formats) + 1)
        out = np.zeros((nmax, 4), np.float64)
        lay = (C.c_int * nmax)()
        n = C.c_int(0)
        self._check(self.fn["bench"](len(shapes), mnk, ",".join(formats).encode(), repeats, seed,
                                     out.ctypes.data_as(C.POINTER(C.c_double)), lay, C.byref(n)))
        rows, i = [], 0
        for s in shapes:
            for f in ["fp32"] + list(formats):
                rows.append((s, f, "dense" if lay[i] == 0 else "rowmajor", *out[i]))
                i += 1
        return rows[: n.value]

    def collect_stats(self, x) -> np.ndarray:
        """collect_stats (calibration.cpp:50-75) of a one-layer identity toy model."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(x.shape[1], np.float32)
        self._check(self.fn["collect_stats"](_abi.fp(x), x.shape[0], x.shape[1], _abi.fp(out)))
        return out

    def eval_activations(self, rows, cols, exj=None, seed=1) -> np.ndarray:
        out = np.empty((rows, cols), np.float32)
        e = _abi.fp(np.ascontiguousarray(exj, np.float32)) if exj is not None else None
        self._check(self.fn["eval_activations"](rows, cols, e, seed, _abi.fp(out)))
        return out

    def compare_formats(self, w, formats, cfg, exj=None, eval_rows=64, eval_seed=1, threads=1):
        """compare_formats (eval.cpp:62-86): [n, 4] weight_mse, rel, output_mse, bits."""
        w = np.ascontiguousarray(w, np.float32)
        out = np.zeros((len(formats), 4), np.float64)
        e = _abi.fp(np.ascontiguousarray(exj, np.float32)) if exj is not None else None
        # (EvalReport::to_csv is not called through ctypes: its iostream
        # formatting faults inside the Python process; the reference's own
        # test_eval.cpp pins the CSV/JSON schema against the drop-in instead)
        self._check(self.fn["compare_formats"](_abi.fp(w), w.shape[0], w.shape[1],
                                               ",".join(formats).encode(), C.byref(cfg), e,
                                               eval_rows, eval_seed, threads,
                                               out.ctypes.data_as(C.POINTER(C.c_double)), None, 0))
        return out

    def weight_error(self, w, qt: QuantizedTensor):
        """eval.cpp:11-29 -> (mse, rel)."""
        w = np.ascontiguousarray(w, np.float32)
        mse, rel = C.c_double(), C.c_double()
        c = qt.as_c()
        self._check(self.fn["weight_error"](_abi.fp(w), C.byref(c), C.byref(mse), C.byref(rel)))
        return mse.value, rel.value

    def output_error(self, w, qt: QuantizedTensor, x) -> float:
        """eval.cpp:31-46."""
        w = np.ascontiguousarray(w, np.float32)
        x = np.ascontiguousarray(x, np.float32)
        mse = C.c_double()
        c = qt.as_c()
        self._check(self.fn["output_error"](_abi.fp(w), C.byref(c), _abi.fp(x), x.shape[0], C.byref(mse)))
        return mse.value

    def pack_codes(self, codes, bits) -> np.ndarray:
        codes = np.ascontiguousarray(codes, np.uint8)
        rows, cols = codes.shape
        out = np.zeros(rows * _abi.packed_bytes_per_row(cols, bits), np.uint8)
        self._check(self.fn["pack_codes"](_abi.u8p(codes), rows, cols, bits, _abi.u8p(out)))
        return out

    def unpack_codes(self, packed, rows, cols, bits) -> np.ndarray:
        packed = np.ascontiguousarray(packed, np.uint8)
        out = np.zeros((rows, cols), np.uint8)
        self._check(self.fn["unpack_codes"](_abi.u8p(packed), rows, cols, bits, _abi.u8p(out)))
        return out

    def to_ktiled(self, qt: QuantizedTensor, tile_k: int) -> QuantizedTensor:
        out = qt.clone()
        c = qt.as_c()
        self._check(self.fn["to_ktiled"](C.byref(c), tile_k, _abi.u8p(out.codes)))
        out.layout = _abi.LAYOUT_KTILED
        out.tile_k = tile_k
        return out

    def from_ktiled(self, qt: QuantizedTensor) -> QuantizedTensor:
        out = qt.clone()
        c = qt.as_c()
        self._check(self.fn["from_ktiled"](C.byref(c), _abi.u8p(out.codes)))
        out.layout = _abi.LAYOUT_ROWMAJOR
        out.tile_k = 1
        return out

    def f32_to_f16(self, f: float) -> int:
        o = C.c_uint16()
        self._check(self.fn["f32_to_f16"](f, C.byref(o)))
        return o.value

    def f16_to_f32(self, h: int) -> float:
        return self.fn["f16_to_f32"](h)

    def f32_to_bf16(self, f: float) -> int:
        o = C.c_uint16()
        self._check(self.fn["f32_to_bf16"](f, C.byref(o)))
        return o.value

    def bf16_to_f32(self, h: int) -> float:
        return self.fn["bf16_to_f32"](h)

    def storage_bits_per_entry(self, cfg, rows, cols) -> float:
        return self.fn["storage_bits_per_entry"](C.byref(cfg), rows, cols)

    # -- learner pieces ----------------------------------------------------
    def kmeans_pp_init(self, x, w, k, seed, row) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        out = np.empty(k, np.float64)
        self._check(
            self.fn["kmeans_pp_init"](_abi.fp(x), _abi.fp(w), x.size, k, seed, row, _abi.f64p(out))
        )
        return out

    def weighted_kmeans(self, x, w, k, cfg, seed, row):
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        cen = np.empty(k, np.float64)
        asg = np.empty(x.size, np.uint8)
        loss = C.c_double()
        iters = C.c_int()
        self._check(
            self.fn["weighted_kmeans"](
                _abi.fp(x), _abi.fp(w), x.size, k, C.byref(cfg), seed, row, _abi.f64p(cen),
                _abi.u8p(asg), C.byref(loss), C.byref(iters)
            )
        )
        return cen, asg, loss.value, iters.value

    def learn_row_lut(self, x, w, bits, cfg, seed, row):
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        lut = np.empty(1 << bits, np.float32)
        codes = np.empty(x.size, np.uint8)
        loss = C.c_double()
        self._check(
            self.fn["learn_row_lut"](
                _abi.fp(x), _abi.fp(w), x.size, bits, C.byref(cfg), seed, row, _abi.fp(lut),
                _abi.u8p(codes), C.byref(loss)
            )
        )
        return lut, codes, loss.value


class Ref(_Lib):
    """The unmodified reference, compiled in place."""

    prefix = "ref_"

    def __init__(self):
        super().__init__(REF_SO)


class Oracle(_Lib):
    """The C restatement (anyq_oracle.c)."""

    prefix = "orc_"

    def __init__(self):
        super().__init__(ORACLE_SO)


_ref = None
_orc = None


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def oracle() -> Oracle:
    global _orc
    if _orc is None:
        _orc = Oracle()
    return _orc


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 -> fp32, RNE (pack.cpp:121-128 semantics)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)
