"""Stream semantics of the device API.

* A DeviceTensor may be used from several streams at once: the GEMV's release
  counters live per stream and the tcgen05 path's workspace is allocated per
  call (stream ordered), so concurrent launches cannot corrupt each other.
* anyq_dev_quantize_any is fully stream ordered (no host synchronisation): it
  captures into a CUDA graph, and its data errors (require_finite, the stats
  and KmProblem weight checks, learner.cpp:10-51) surface through
  anyq_dev_stream_status in the reference's order.
"""
import numpy as np
import pytest

from anyq_testutil import cfg

pytestmark = pytest.mark.gpu


def _bf16(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda().to(torch.bfloat16)


@pytest.mark.parametrize("path", [1, 2])  # GEMV chain kernel, tcgen05 kernel
def test_shared_tensor_on_two_streams(aq, orc, cuda, path):
    import torch

    qt = aq.quantize_any(orc.gaussian(1024, 2048, 3), cfg(codebook=3, max_iters=3))
    dt = aq.DeviceTensor(qt)
    xa = _bf16(orc.gaussian(2, 2048, 4))
    xb = _bf16(orc.gaussian(2, 2048, 5))
    ra = torch.empty(2, 1024, device="cuda", dtype=torch.float32)
    rb = torch.empty_like(ra)
    dt.gemm(xa, None, ra, path=path)
    dt.gemm(xb, None, rb, path=path)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    ya = [torch.empty_like(ra) for _ in range(20)]
    yb = [torch.empty_like(rb) for _ in range(20)]
    for i in range(20):  # interleaved issue: both streams in flight together
        with torch.cuda.stream(sa):
            dt.gemm(xa, None, ya[i], path=path)
        with torch.cuda.stream(sb):
            dt.gemm(xb, None, yb[i], path=path)
    torch.cuda.synchronize()
    for i in range(20):
        assert torch.equal(ya[i], ra), i
        assert torch.equal(yb[i], rb), i
    dt.close()


def test_dev_quantize_any_graph_capture(aq, orc, cuda):
    import torch

    from paper_2507_04610_b200 import _abi

    w = torch.from_numpy(orc.gaussian(256, 512, 7)).cuda()
    c = _abi.default_config(codebook=_abi.CB_ANY, max_iters=20)
    eager = aq.dev_quantize_any(w, c)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up on the capture stream (attributes, pools)
        aq.dev_quantize_any(w, c, stream=s, check=False)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        out = aq.dev_quantize_any(w, c, stream=s, check=False)
    for _ in range(2):
        for t in out:
            t.zero_()
        g.replay()
        torch.cuda.synchronize()
        for a, b in zip(out, eager):
            assert torch.equal(a, b)
    aq.dev_stream_status(s)


def test_dev_quantize_any_errors_are_stream_ordered(aq, orc, cuda):
    import torch

    from paper_2507_04610_b200 import _abi

    c = _abi.default_config(codebook=_abi.CB_ANY, max_iters=5)
    w = torch.from_numpy(orc.gaussian(64, 256, 9)).cuda()
    bad = w.clone()
    bad[3, 7] = float("nan")
    neg = torch.ones(256, device="cuda")
    neg[5] = -1.0
    # NonFiniteError (require_finite) precedes the stats check, as in the reference
    aq.dev_quantize_any(bad, c, exj=neg, check=False)
    with pytest.raises(aq.NonFiniteError):
        aq.dev_stream_status()
    aq.dev_quantize_any(w, c, exj=neg, check=False)
    with pytest.raises(aq.StatsError):
        aq.dev_stream_status()
    aq.dev_quantize_any(w, c)  # cleared: a clean call reports nothing
    aq.dev_stream_status()
