"""Tensor-parallel GEMM with the all-gather fused into the GEMV writer
(anyq_dev_gemm_allgather / anyq_dev_tp_wait).

Each rank's kernel stores its row shard's y straight into EVERY rank's
full-width y and bumps a system-scope flag per CTA on every rank; the wait
kernel holds the stream until all ranks' flags of the call are in. With one
GPU per box here, W ranks are simulated in one process on one device (the
peer buffers are plain local pointers instead of IPC mappings): every rank's
y must equal the unsharded GEMV bit for bit (an item is one 32-row block, so
32-aligned shards compute every row the same way)."""
import numpy as np
import pytest

from anyq_testutil import cfg
from test_gpu_gemm import bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("m", [1, 2, 4])
def test_fused_allgather_equals_unsharded(aq, orc, cuda, world, m):
    import torch

    from paper_2507_04610_b200.dist import row_range, shard_rows

    N, K = 1000, 512
    qt = aq.quantize_any(orc.gaussian(N, K, 61), cfg(codebook=3, max_iters=3, seed=5))
    full = aq.DeviceTensor(qt)
    shards = []
    for r in range(world):
        r0, r1 = row_range(N, world, r, 32)
        shards.append((r0, aq.DeviceTensor(shard_rows(qt, r0, r1))))
    x = torch.from_numpy(bf16(orc.gaussian(m, K, 62))).cuda().to(torch.bfloat16)
    want = torch.empty(m, N, device="cuda", dtype=torch.bfloat16)
    full.gemm(x, want, path=aq.PATH_GEMV)
    ys = [torch.full((m, N), float("nan"), device="cuda", dtype=torch.bfloat16) for _ in range(world)]
    flags = [torch.zeros(world, device="cuda", dtype=torch.int32) for _ in range(world)]
    peers = [aq.tp_peers(world, r, N, shards[r][0], [y.data_ptr() for y in ys], [f.data_ptr() for f in flags])
             for r in range(world)]
    for epoch in (1, 2, 3):  # flags count calls; buffers are rewritten each call
        for r in range(world):
            aq.gemm_allgather(shards[r][1], x, peers[r])
        for r in range(world):
            aq.tp_wait(shards[r][1], peers[r], epoch)
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(ys[r], want), (epoch, r)
        for f in flags:
            assert f.cpu().tolist() == [epoch * 148] * world or f.cpu().min().item() >= epoch
    for _, d in shards:
        d.close()
    full.close()


def test_tp_argument_errors(aq, orc, cuda):
    import torch

    qt = aq.quantize_any(orc.gaussian(64, 256, 63), cfg(codebook=3, max_iters=2))
    d = aq.DeviceTensor(qt)
    x = torch.zeros(1, 256, device="cuda", dtype=torch.bfloat16)
    y = torch.zeros(1, 64, device="cuda", dtype=torch.bfloat16)
    f = torch.zeros(2, device="cuda", dtype=torch.int32)
    with pytest.raises(aq.ShapeError):  # shard outside y
        aq.gemm_allgather(d, x, aq.tp_peers(1, 0, 64, 32, [y.data_ptr()], [f.data_ptr()]))
    with pytest.raises(aq.ShapeError):  # rank out of range
        aq.gemm_allgather(d, x, aq.tp_peers(2, 2, 64, 0, [y.data_ptr()] * 2, [f.data_ptr()] * 2))
    with pytest.raises(aq.ShapeError):  # the fused gather runs on the GEMV (m <= 4)
        aq.gemm_allgather(d, torch.zeros(5, 256, device="cuda", dtype=torch.bfloat16),
                          aq.tp_peers(1, 0, 64, 0, [y.data_ptr()], [f.data_ptr()]))
    d.close()
