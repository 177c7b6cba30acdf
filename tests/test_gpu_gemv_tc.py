"""K1t — the persistent LUT GEMV chain with its products on tcgen05
(ANYQ_PATH_GEMV_TC, gemv.cu) — against the oracle.

Products are exact (fp16 pair-table values x fp16 x scaled by 2^e per chunk)
and accumulate in fp32 in TMEM, so the bound is the CUDA-core GEMV's:
|dy| <= 1e-5 * sum_j |x_j| (|alpha T[c]| + |beta|) of
gemm_reference(bf16(x), narrowed(qt)) (qgemm.cpp:36-40), stated in
tests/test_gpu_gemm.py::tc_tolerance.
"""
import numpy as np
import pytest

from anyq_testutil import cfg
from test_gpu_gemm import bf16, tc_gemm, tc_tolerance

pytestmark = pytest.mark.gpu
TC = 5


@pytest.mark.parametrize("fmt", ["any4", "int4", "nf4", "fp4", "any3", "any2"])
@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8, 9, 16])
def test_formats_and_m(aq, orc, cuda, fmt, m):
    n, k = 200, 384  # ragged rows, 3 chunks (a partial chunk group), 3 groups
    w = orc.gaussian(n, k, 31)
    c = cfg(granularity=3, group_size=128, seed=2)
    aq.apply_format(c, fmt)
    qt = orc.quantize(w, c)
    x = bf16(orc.gaussian(m, k, 33))
    y32, ybf = tc_gemm(aq, cuda, qt, x, TC)
    ref = orc.gemm_reference(x, orc.narrowed(qt))
    tol = tc_tolerance(orc, x, qt)
    err = np.abs(y32 - ref)
    assert np.all(err <= tol), f"max err {err.max()} tol {tol.min()}"
    assert np.all(np.abs(ybf - bf16(ref)) <= np.abs(ref) * 2 ** -7 + tol)


@pytest.mark.parametrize("m", [1, 4, 16])
@pytest.mark.parametrize("n,k,g", [(4096, 4096, 128), (1024, 4096, 128), (4096, 1024, 256),
                                   (96, 1280, 1280), (33, 128, 128), (151 * 32 - 5, 512, 128),
                                   (70, 200, 128), (300, 1000, 128)])
def test_shapes(aq, orc, cuda, m, n, k, g):
    """m * k beyond one x image in shared memory (M = 16 at K = 4096) runs as
    K-slices chained through the fp32 running sum."""
    w = orc.gaussian(n, k, 41)
    gran = 1 if g == k else 3
    c = cfg(codebook=3, granularity=gran, group_size=g, seed=1, max_iters=8)
    qt = aq.quantize_any(w, c)
    x = bf16(orc.gaussian(m, k, 43))
    y32, _ = tc_gemm(aq, cuda, qt, x, TC)
    ref = orc.gemm_reference(x, orc.narrowed(qt))
    tol = tc_tolerance(orc, x, qt)
    assert np.all(np.abs(y32 - ref) <= tol)


def test_deterministic_and_rowwise_consistent(aq, orc, cuda):
    w = orc.gaussian(512, 1024, 5)
    qt = aq.quantize_any(w, cfg(codebook=3, max_iters=5))
    x1 = bf16(orc.gaussian(1, 1024, 6))
    a, _ = tc_gemm(aq, cuda, qt, x1, TC)
    b, _ = tc_gemm(aq, cuda, qt, x1, TC)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    for mm in (2, 3, 7, 16):
        c, _ = tc_gemm(aq, cuda, qt, np.repeat(x1, mm, axis=0), TC)
        for r in range(mm):  # every x row is computed the same way: bit-identical
            assert np.array_equal(c[r].view(np.uint32), a[0].view(np.uint32)), (mm, r)


def test_wide_dynamic_range_x(aq, orc, cuda):
    """x entries spanning 2^-30..2^10 inside one chunk: the per-chunk 2^e
    scaling puts the largest in [2^14, 2^15); entries ~2^-25 below it become
    fp16 subnormals (their products stay well inside the 1e-5 bound)."""
    n, k = 256, 512
    w = orc.gaussian(n, k, 7)
    qt = aq.quantize_any(w, cfg(codebook=3, max_iters=5))
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, k)).astype(np.float32) * np.exp2(rng.integers(-30, 11, (2, k))).astype(np.float32)
    x = bf16(x)
    for path in (1, TC):
        y32, _ = tc_gemm(aq, cuda, qt, x, path)
        ref = orc.gemm_reference(x, orc.narrowed(qt))
        assert np.all(np.abs(y32 - ref) <= tc_tolerance(orc, x, qt)), path


@pytest.mark.parametrize("m", [1, 2, 4, 8, 16])
def test_chain_decoder_pattern(aq, orc, cuda, m):
    """q, k, v <- x; o <- q; gate, up <- o; down <- up in ONE K1t launch equals
    K1t single launches bit for bit, and the oracle within the bound."""
    import torch

    K0 = 256
    shapes = [(256, K0), (64, K0), (64, K0), (K0, 256), (640, K0), (640, K0), (K0, 640)]
    deps = [-1, -1, -1, 0, 3, 3, 5]
    dts, qts = [], []
    for i, (n, k) in enumerate(shapes):
        qt = aq.quantize_any(orc.gaussian(n, k, 110 + i), cfg(codebook=3, max_iters=4, seed=i))
        qts.append(qt)
        dts.append(aq.DeviceTensor(qt))
    x0 = torch.from_numpy(bf16(orc.gaussian(m, K0, 120 + m))).cuda().to(torch.bfloat16)
    ys = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for n, _ in shapes]
    y32 = [torch.empty(m, n, device="cuda", dtype=torch.float32) for n, _ in shapes]
    xs = [x0 if d < 0 else ys[d] for d in deps]
    for _ in range(3):  # repeated launches reuse the self-resetting counters
        aq.gemm_chain(dts, xs, ys, y32s=y32, deps=deps, path=TC)
    torch.cuda.synchronize()
    for i, d in enumerate(dts):
        xi = (x0 if deps[i] < 0 else ys[deps[i]]).clone()
        r = torch.empty(m, shapes[i][0], device="cuda", dtype=torch.float32)
        d.gemm(xi, None, r, path=TC)
        torch.cuda.synchronize()
        assert torch.equal(r, y32[i]), i
        xn = xi.float().cpu().numpy()
        ref = orc.gemm_reference(xn, orc.narrowed(qts[i]))
        assert np.all(np.abs(r.cpu().numpy() - ref) <= tc_tolerance(orc, xn, qts[i])), i
    for d in dts:
        d.close()


def test_chain_edge_cases(aq, orc, cuda):
    """8 problems, a repeated tensor, 1- and 31-row tensors, ragged K, a
    dependency reaching back 7 problems, a K = 1 tensor."""
    import torch

    shapes = [(1, 256), (31, 256), (256, 256), (96, 256), (256, 200), (256, 256), (40, 256), (256, 256)]
    deps = [-1, -1, -1, 2, -1, 2, -1, 0]
    base = []
    for i, (n, k) in enumerate(shapes):
        qt = aq.quantize_any(orc.gaussian(n, k, 130 + i), cfg(codebook=3, max_iters=3, seed=i))
        base.append(aq.DeviceTensor(qt))
    dts = list(base)
    dts[5] = dts[2]
    qt7 = aq.quantize_any(orc.gaussian(256, 1, 140), cfg(codebook=3, max_iters=3, seed=7))
    dts[7] = aq.DeviceTensor(qt7)
    for m in (1, 3, 16):
        xin = {256: torch.from_numpy(bf16(orc.gaussian(m, 256, 150 + m))).cuda().to(torch.bfloat16),
               200: torch.from_numpy(bf16(orc.gaussian(m, 200, 160 + m))).cuda().to(torch.bfloat16)}
        ys = [torch.empty(m, d.rows, device="cuda", dtype=torch.bfloat16) for d in dts]
        y32 = [torch.empty(m, d.rows, device="cuda", dtype=torch.float32) for d in dts]
        xs = [ys[d] if d >= 0 else xin[dts[i].cols] for i, d in enumerate(deps)]
        for _ in range(2):
            aq.gemm_chain(dts, xs, ys, y32s=y32, deps=deps, path=TC)
        torch.cuda.synchronize()
        for i, d in enumerate(dts):
            r = torch.empty(m, d.rows, device="cuda", dtype=torch.float32)
            d.gemm(xs[i].clone(), None, r, path=TC)
            torch.cuda.synchronize()
            assert torch.equal(r, y32[i]), (m, i)
    for d in base + [dts[7]]:
        d.close()


@pytest.mark.parametrize("m,k,g", [(3, 14336, 128), (4, 14336, 128), (8, 14336, 512), (16, 4096, 256),
                                   (12, 6144, 128)])
def test_k_slices(aq, orc, cuda, m, k, g):
    """x images beyond shared memory: the GEMM runs as up to 8 K-slices (whole
    chunk groups and scale groups) in one launch, slice s waiting for s - 1 and
    adding to its fp32 partial; with and without a caller y32 (the running sum
    then lives in stream scratch); deterministic."""
    import torch

    n = 300
    w = orc.gaussian(n, k, 51)
    qt = aq.quantize_any(w, cfg(codebook=3, granularity=3, group_size=g, seed=1, max_iters=3))
    dt = aq.DeviceTensor(qt)
    x = bf16(orc.gaussian(m, k, 52))
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16).contiguous()
    y = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    y32 = torch.empty((m, n), dtype=torch.float32, device="cuda")
    dt.gemm(xt, y, y32, path=TC)
    y2 = torch.empty_like(y)
    dt.gemm(xt, y2, None, path=TC)
    y3 = torch.empty_like(y)
    dt.gemm(xt, y3, None, path=TC)
    torch.cuda.synchronize()
    ref = orc.gemm_reference(x, orc.narrowed(qt))
    tol = tc_tolerance(orc, x, qt)
    assert np.all(np.abs(y32.cpu().numpy() - ref) <= tol)
    assert torch.equal(y, y2) and torch.equal(y2, y3)
    dt.close()
