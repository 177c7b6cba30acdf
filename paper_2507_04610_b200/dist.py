"""Multi-GPU partitioning of the any4 hot path.

* Quantization shards by rows with NO collective: rank r quantizes rows
  [row_range(N, P, r)) with `row_offset` = its first global row, which keys the
  per-row RNG exactly as the reference keys matrix row i (learner.cpp:381,
  core.hpp:196-200). The result is bit-identical for every P; gathering the
  shards (optional) is plain concatenation.
* The A16W4 GEMM shards W by output rows (tensor parallel): every rank owns
  rows [row_range(N, P, r)) with their LUTs and alpha/beta rows (all row-local),
  x is replicated, and the y slices are all-gathered — the one real exchange
  step, NCCL over NVLink on GPUs (gloo in the CPU tests).

The process-group plumbing is torch.distributed; compute goes through the CUDA
library (anyq.py). Only rowwise / groupwise scale granularities shard by rows
(learned LUTs require them, core.hpp:124-142).
"""
from __future__ import annotations

import numpy as np

from . import _abi
from .qtensor import QuantizedTensor


def row_range(n: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous, balanced row range of `rank`; boundaries are multiples of
    `align` (32 = one GEMV row block) except the last."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    units = (n + align - 1) // align
    u0, u1 = units * rank // world, units * (rank + 1) // world
    return min(n, u0 * align), min(n, u1 * align)


def groups_per_row(cfg: _abi.Config, cols: int) -> int:
    if cfg.granularity == _abi.G_ROW:
        return 1
    if cfg.granularity == _abi.G_GROUP:
        return (cols + cfg.group_size - 1) // cfg.group_size
    raise ValueError("row sharding needs rowwise or groupwise scales")


def shard_rows(qt: QuantizedTensor, r0: int, r1: int) -> QuantizedTensor:
    """Rows [r0, r1) of a QuantizedTensor (codes, LUT and alpha/beta rows)."""
    gpr = groups_per_row(qt.cfg, qt.cols)
    bpr = _abi.packed_bytes_per_row(qt.cols, qt.cfg.bits)
    out = QuantizedTensor.empty(r1 - r0, qt.cols, qt.cfg)
    out.layout, out.tile_k = qt.layout, qt.tile_k
    out.lut_store, out.scale_store = qt.lut_store, qt.scale_store
    out.codes = qt.codes[r0 * bpr:r1 * bpr].copy()
    out.alphas = qt.alphas[r0 * gpr:r1 * gpr].copy()
    out.betas = qt.betas[r0 * gpr:r1 * gpr].copy()
    if qt.luts is not None:
        k = 1 << qt.cfg.bits
        out.luts = qt.luts[r0 * k:r1 * k].copy()
    return out


def concat_rows(shards: list[QuantizedTensor]) -> QuantizedTensor:
    """Inverse of shard_rows over a full partition (rank order)."""
    first = shards[0]
    rows = sum(s.rows for s in shards)
    out = QuantizedTensor.empty(rows, first.cols, first.cfg)
    out.codes = np.concatenate([s.codes for s in shards])
    out.alphas = np.concatenate([s.alphas for s in shards])
    out.betas = np.concatenate([s.betas for s in shards])
    if first.luts is not None:
        out.luts = np.concatenate([s.luts for s in shards])
    return out


def quantize_any_rows(w_local, cfg: _abi.Config, exj=None, row_offset: int = 0, quantizer=None):
    """Quantize this rank's rows; `row_offset` is their first global row.

    `quantizer(w, cfg, exj, row_offset)` defaults to the CUDA library's
    anyq.quantize_any (host buffers)."""
    if quantizer is None:
        from . import anyq

        quantizer = anyq.quantize_any
    return quantizer(w_local, cfg, exj, row_offset)


def gather_rows(local: QuantizedTensor, group=None) -> QuantizedTensor:
    """All-gather the row shards of a quantized matrix (object collective)."""
    import torch.distributed as dist

    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, local, group=group)
    return concat_rows(parts)


def all_gather_rows_y(y_local, group=None):
    """y slices [M, N_r] of the row-sharded GEMM -> full y [M, sum N_r] in rank
    order (torch tensors; NCCL on GPUs). Slices may differ in width."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    widths = [None] * world
    dist.all_gather_object(widths, int(y_local.shape[1]), group=group)
    m = y_local.shape[0]
    if len(set(widths)) == 1:
        out = torch.empty((world * m, widths[0]), dtype=y_local.dtype, device=y_local.device)
        dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
        return out.view(world, m, widths[0]).permute(1, 0, 2).reshape(m, -1)
    # uneven shards: pad to the widest slice, gather, trim
    wmax = max(widths)
    pad = torch.zeros((y_local.shape[0], wmax), dtype=y_local.dtype, device=y_local.device)
    pad[:, :y_local.shape[1]] = y_local
    out = torch.empty((world * m, wmax), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    out = out.view(world, m, wmax)
    return torch.cat([out[r, :, :widths[r]] for r in range(world)], dim=1)


class RowShardedLinear:
    """Tensor-parallel A16W4 linear: this rank's row shard of W in HBM,
    y = all_gather(x W_r^T) over the process group."""

    def __init__(self, qt: QuantizedTensor, group=None, align: int = 32):
        import torch.distributed as dist

        from . import anyq

        self.group = group
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self.r0, self.r1 = row_range(qt.rows, world, rank, align)
        self.rows = qt.rows
        self.dt = anyq.DeviceTensor(shard_rows(qt, self.r0, self.r1))

    def __call__(self, x):
        y_local = self.dt.gemm(x)
        return all_gather_rows_y(y_local, self.group)

    def close(self):
        self.dt.close()


class FusedRowShardedLinear:
    """Tensor-parallel A16W4 linear with the all-gather fused into the GEMV
    writer (anyq_dev_gemm_allgather): every rank's kernel stores its y slice
    straight into every rank's full-width y buffer over NVLink (CUDA IPC
    mappings exchanged once through the process group) and signals a flag per
    CTA; `__call__` returns this rank's full y after the flags of the call are
    in (no NCCL call on the hot path). M <= 4 (the GEMV).

    y buffers alternate between two slots by call parity, so the output of
    call e stays valid until call e + 2 is issued; a decode loop's own data
    dependency (every rank consumes y before the next layer's call) keeps the
    ranks within that distance."""

    def __init__(self, qt: QuantizedTensor, group=None, m_max: int = 4, align: int = 32):
        import torch
        import torch.distributed as dist

        from . import anyq

        self.group = group
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if world > 8:
            raise ValueError("the fused gather supports up to 8 ranks")
        self.world, self.rank, self.rows = world, rank, qt.rows
        self.r0, self.r1 = row_range(qt.rows, world, rank, align)
        self.dt = anyq.DeviceTensor(shard_rows(qt, self.r0, self.r1))
        self.m_max = m_max
        self.y = [torch.empty(m_max, qt.rows, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
        self.flags = [torch.zeros(world, dtype=torch.int32, device="cuda") for _ in range(2)]
        mine = [(anyq.ipc_handle(self.y[s].data_ptr()), anyq.ipc_handle(self.flags[s].data_ptr())) for s in range(2)]
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        self.peers = []
        for s in range(2):
            yp, fp = [], []
            for r in range(world):
                if r == rank:
                    yp.append(self.y[s].data_ptr())
                    fp.append(self.flags[s].data_ptr())
                else:
                    a, b = anyq.ipc_open(allh[r][s][0]), anyq.ipc_open(allh[r][s][1])
                    self._opened += [a, b]
                    yp.append(a)
                    fp.append(b)
            self.peers.append(anyq.tp_peers(world, rank, qt.rows, self.r0, yp, fp))
        self.calls = 0
        dist.barrier(group=group)

    def __call__(self, x):
        from . import anyq

        m = x.shape[0]
        if m > self.m_max:
            raise ValueError(f"at most {self.m_max} rows of x")
        s = self.calls & 1
        self.calls += 1
        anyq.gemm_allgather(self.dt, x, self.peers[s])
        anyq.tp_wait(self.dt, self.peers[s], (self.calls + 1) // 2)
        return self.y[s][:m]

    def close(self):
        from . import anyq

        for p in self._opened:
            anyq.ipc_close(p)
        self._opened = []
        self.dt.close()
