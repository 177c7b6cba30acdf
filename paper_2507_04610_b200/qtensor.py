"""Host-side QuantizedTensor (pack.hpp:21-39) backed by numpy arrays."""
from __future__ import annotations

import copy
from dataclasses import dataclass, field

import numpy as np

from . import _abi


@dataclass
class QuantizedTensor:
    rows: int
    cols: int
    cfg: _abi.Config
    codes: np.ndarray  # uint8, rows * packed_bytes_per_row
    alphas: np.ndarray  # float32, num_groups
    betas: np.ndarray  # float32, num_groups
    luts: np.ndarray | None = None  # float32, rows * 2^bits (AnyN only)
    layout: int = _abi.LAYOUT_ROWMAJOR
    tile_k: int = 1
    lut_store: int = _abi.STORE_FP16
    scale_store: int = _abi.STORE_FP16
    _keep: list = field(default_factory=list, repr=False)

    @classmethod
    def empty(cls, rows: int, cols: int, cfg: _abi.Config) -> "QuantizedTensor":
        ng = _abi.num_groups(cfg, rows, cols)
        nbytes = rows * _abi.packed_bytes_per_row(cols, cfg.bits)
        luts = (
            np.zeros(rows * (1 << cfg.bits), np.float32)
            if cfg.codebook == _abi.CB_ANY
            else None
        )
        return cls(
            rows=rows,
            cols=cols,
            cfg=_abi.Config.from_buffer_copy(bytes(cfg)),
            codes=np.zeros(nbytes, np.uint8),
            alphas=np.zeros(ng, np.float32),
            betas=np.zeros(ng, np.float32),
            luts=luts,
        )

    @property
    def num_groups(self) -> int:
        return int(self.alphas.size)

    @property
    def lut_entries(self) -> int:
        return (1 << self.cfg.bits) if self.cfg.codebook == _abi.CB_ANY else 0

    def row_lut(self, i: int) -> np.ndarray:
        k = self.lut_entries
        return self.luts[i * k : (i + 1) * k]

    def clone(self) -> "QuantizedTensor":
        out = copy.copy(self)
        out.cfg = _abi.Config.from_buffer_copy(bytes(self.cfg))
        out.codes = self.codes.copy()
        out.alphas = self.alphas.copy()
        out.betas = self.betas.copy()
        out.luts = None if self.luts is None else self.luts.copy()
        out._keep = []
        return out

    def as_c(self) -> _abi.QTensor:
        """A C view over the arrays (arrays must stay alive while it is used)."""
        for name in ("codes", "alphas", "betas"):
            a = getattr(self, name)
            if not a.flags["C_CONTIGUOUS"]:
                setattr(self, name, np.ascontiguousarray(a))
        q = _abi.QTensor()
        q.rows = self.rows
        q.cols = self.cols
        q.cfg = self.cfg
        q.layout = self.layout
        q.tile_k = self.tile_k
        q.lut_store = self.lut_store
        q.scale_store = self.scale_store
        q.codes = _abi.u8p(self.codes)
        q.luts = _abi.fp(self.luts) if self.luts is not None else None
        q.alphas = _abi.fp(self.alphas)
        q.betas = _abi.fp(self.betas)
        q.num_groups = self.num_groups
        return q

    def same_as(self, other: "QuantizedTensor") -> bool:
        """Bit-identity of codes, LUTs and scales."""
        if (self.luts is None) != (other.luts is None):
            return False
        return (
            np.array_equal(self.codes, other.codes)
            and np.array_equal(self.alphas.view(np.uint32), other.alphas.view(np.uint32))
            and np.array_equal(self.betas.view(np.uint32), other.betas.view(np.uint32))
            and (
                self.luts is None
                or np.array_equal(self.luts.view(np.uint32), other.luts.view(np.uint32))
            )
        )
