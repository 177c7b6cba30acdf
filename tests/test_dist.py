"""Multi-process (gloo, world_size 2, CPU) tests of the row partitioning:

* quantization shards by rows with no collective and is bit-identical for any
  world size (the oracle stands in for the device quantizer here; it keys the
  RNG by matrix-local row, so each rank quantizes the global matrix's rows the
  way the reference does and the shard is sliced out);
* the tensor-parallel GEMM: per-rank row shards (codes, LUT, alpha/beta rows)
  computed locally, y slices all-gathered in rank order == the full GEMM,
  bit for bit (rows are independent).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from anyq_testutil import bits_equal, cfg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return out


def test_row_range_partition():
    from paper_2507_04610_b200.dist import row_range

    for n in (1, 31, 32, 1000, 4096, 14336):
        for world in (1, 2, 3, 4, 8):
            for align in (1, 32):
                rs = [row_range(n, world, r, align) for r in range(world)]
                assert rs[0][0] == 0 and rs[-1][1] == n
                assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
                assert all(a % align == 0 for a, _ in rs)


def test_shard_concat_roundtrip(orc):
    from paper_2507_04610_b200.dist import concat_rows, row_range, shard_rows

    qt = orc.quantize(orc.gaussian(37, 40, 1), cfg(codebook=3, group_size=16, max_iters=5))
    for world in (1, 2, 3):
        parts = [shard_rows(qt, *row_range(37, world, r)) for r in range(world)]
        assert concat_rows(parts).same_as(qt)


def _tp_gemm(rank, world):
    import torch
    import torch.distributed as dist

    from oracle.refpy import oracle
    from paper_2507_04610_b200.dist import all_gather_rows_y, row_range, shard_rows

    orc = oracle()
    qt = orc.quantize(orc.gaussian(70, 96, 3), cfg(codebook=3, group_size=32, max_iters=6))
    x = orc.gaussian(3, 96, 4)
    r0, r1 = row_range(70, world, rank, align=32)
    y_local = orc.gemm_fused(x, shard_rows(qt, r0, r1))  # the rank's shard (oracle as device)
    y = all_gather_rows_y(torch.from_numpy(y_local)).numpy()
    ok = bits_equal(y, orc.gemm_fused(x, qt))
    dist.barrier()
    return ok


def _dist_quantize(rank, world):
    import torch.distributed as dist

    from oracle.refpy import oracle
    from paper_2507_04610_b200.dist import gather_rows, quantize_any_rows, row_range, shard_rows

    orc = oracle()
    w = orc.gaussian(23, 48, 7)
    c = cfg(codebook=3, group_size=16, seed=5, max_iters=8)
    r0, r1 = row_range(23, world, rank)

    def oracle_quantizer(w_rows, cfg_, exj, row_offset):
        # the reference keys row i's RNG by (seed, i): quantizing the rows at
        # their global index = the global matrix's rows, sliced
        full = np.zeros((row_offset + w_rows.shape[0], w_rows.shape[1]), np.float32)
        full[row_offset:] = w_rows
        full[:row_offset] = 1.0  # placeholder rows (row-local: do not affect the shard)
        return shard_rows(orc.quantize(full, cfg_, exj), row_offset, row_offset + w_rows.shape[0])

    local = quantize_any_rows(w[r0:r1], c, None, r0, quantizer=oracle_quantizer)
    full = gather_rows(local)
    ok = full.same_as(orc.quantize(w, c))
    dist.barrier()
    return ok


def test_tp_gemm_gloo_world2():
    out = run_ranks(_tp_gemm, 2)
    assert out == {0: True, 1: True}, out


def test_row_partitioned_quantize_gloo_world2():
    out = run_ranks(_dist_quantize, 2)
    assert out == {0: True, 1: True}, out


@pytest.mark.gpu
def test_device_row_offset_matches_full_quantize(aq, orc, cuda):
    """On the device: quantizing row slices with row_offset and concatenating
    is bit-identical to quantizing the whole matrix (any P)."""
    from paper_2507_04610_b200.dist import concat_rows, row_range

    w = orc.gaussian(300, 256, 9)
    c = cfg(codebook=3, group_size=128, seed=2)
    full = aq.quantize_any(w, c)
    assert full.same_as(orc.quantize(w, c))
    for world in (2, 3, 8):
        parts = []
        for r in range(world):
            r0, r1 = row_range(300, world, r)
            parts.append(aq.quantize_any(w[r0:r1], c, None, r0))
        assert concat_rows(parts).same_as(full), world


@pytest.mark.gpu
def test_device_row_sharded_gemm_matches_full(aq, orc, cuda):
    import torch

    from paper_2507_04610_b200.dist import row_range, shard_rows

    qt = aq.quantize_any(orc.gaussian(5000, 512, 3), cfg(codebook=3, max_iters=4))
    x = torch.from_numpy(orc.gaussian(1, 512, 4)).cuda().to(torch.bfloat16)
    full = aq.DeviceTensor(qt)
    yf = torch.empty(1, 5000, device="cuda")
    full.gemm(x, None, yf)
    for world in (2, 4, 8):
        parts = []
        for r in range(world):
            r0, r1 = row_range(5000, world, r, align=32)
            d = aq.DeviceTensor(shard_rows(qt, r0, r1))
            y = torch.empty(1, r1 - r0, device="cuda")
            d.gemm(x, None, y)
            parts.append(y)
            d.close()
        torch.cuda.synchronize()
        assert torch.equal(torch.cat(parts, dim=1), yf), world
    full.close()
