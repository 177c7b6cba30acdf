"""ctypes mirror of include/anyq_b200.h (structs, enums, status codes).

Shared by the product binding (paper_2507_04610_b200.anyq) and the test-only
oracle wrappers, so both sides marshal exactly the same memory layout.
"""
from __future__ import annotations

import ctypes as C

# Status codes (anyq_status) -> reference exception class names (core.hpp:27-74).
OK = 0
STATUS_NAMES = {
    1: "ShapeError",
    2: "ConfigError",
    3: "CodeRangeError",
    4: "NonFiniteError",
    5: "StatsError",
    6: "IoError",
    7: "MagicError",
    8: "VersionError",
    9: "TruncatedError",
    10: "InvariantError",
    11: "Error",
    12: "CudaError",
}

CB_INT, CB_FP4, CB_NF4, CB_ANY = 0, 1, 2, 3
G_TENSOR, G_ROW, G_COLUMN, G_GROUP, G_BLOCK = 0, 1, 2, 3, 4
INIT_KMPP, INIT_RANDOM, INIT_GRID, INIT_NF4 = 0, 1, 2, 3
W_WEIGHTS, W_ACTS, W_FULL = 0, 1, 2
LAYOUT_ROWMAJOR, LAYOUT_KTILED = 0, 1
STORE_FP16, STORE_BF16, STORE_FP32 = 0, 1, 2


class Config(C.Structure):
    """anyq_config == QuantConfig + LearnerConfig (core.hpp:98-121)."""

    _fields_ = [
        ("bits", C.c_int32),
        ("codebook", C.c_int32),
        ("granularity", C.c_int32),
        ("group_size", C.c_int32),
        ("block_size", C.c_int32),
        ("symmetric", C.c_int32),
        ("int_range_shifted", C.c_int32),
        ("init", C.c_int32),
        ("max_iters", C.c_int32),
        ("rel_tol", C.c_float),
        ("restarts", C.c_int32),
        ("weighting", C.c_int32),
        ("check_invariants", C.c_int32),
        ("reserved", C.c_int32),
        ("seed", C.c_uint64),
    ]


def default_config(**kw) -> Config:
    """QuantConfig{} defaults (core.hpp:98-121), optionally overridden."""
    c = Config(
        bits=4,
        codebook=CB_INT,
        granularity=G_GROUP,
        group_size=128,
        block_size=1,
        symmetric=0,
        int_range_shifted=0,
        init=INIT_KMPP,
        max_iters=100,
        rel_tol=1e-6,
        restarts=1,
        weighting=W_FULL,
        check_invariants=0,
        reserved=0,
        seed=0,
    )
    for k, v in kw.items():
        setattr(c, k, int(v) if not isinstance(v, float) else v)
    return c


class QTensor(C.Structure):
    """anyq_qtensor == QuantizedTensor (pack.hpp:21-39) as flat arrays."""

    _fields_ = [
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("cfg", Config),
        ("layout", C.c_int32),
        ("tile_k", C.c_int32),
        ("lut_store", C.c_int32),
        ("scale_store", C.c_int32),
        ("codes", C.POINTER(C.c_uint8)),
        ("luts", C.POINTER(C.c_float)),
        ("alphas", C.POINTER(C.c_float)),
        ("betas", C.POINTER(C.c_float)),
        ("num_groups", C.c_int64),
    ]


def packed_bytes_per_row(cols: int, bits: int) -> int:
    """pack.hpp:45."""
    return (cols * bits + 7) // 8


def num_groups(cfg: Config, rows: int, cols: int) -> int:
    """Group count of scaling.cpp:8-24."""
    g = cfg.granularity
    if g == G_TENSOR:
        return 1
    if g == G_ROW:
        return rows
    if g == G_COLUMN:
        return cols
    if g == G_GROUP:
        return rows * ((cols + cfg.group_size - 1) // cfg.group_size)
    if g == G_BLOCK:
        b = cfg.block_size
        return ((rows + b - 1) // b) * ((cols + b - 1) // b)
    raise ValueError("unknown granularity")


def group_of(cfg: Config, rows: int, cols: int, i, j):
    """ScaleSet::group_of (scaling.hpp:36-45), vectorised over numpy arrays."""
    g = cfg.granularity
    if g == G_TENSOR:
        return 0 * (i + j)
    if g == G_ROW:
        return i + 0 * j
    if g == G_COLUMN:
        return j + 0 * i
    if g == G_GROUP:
        gpr = (cols + cfg.group_size - 1) // cfg.group_size
        return i * gpr + j // cfg.group_size
    b = cfg.block_size
    bpr = (cols + b - 1) // b
    return (i // b) * bpr + j // b


def fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def f64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class TpPeers(C.Structure):
    """anyq_tp_peers (include/anyq_b200.h): the fused tensor-parallel gather."""
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("rows_total", C.c_int64), ("row0", C.c_int64),
                ("y", C.c_void_p * 8), ("flags", C.c_void_p * 8)]
