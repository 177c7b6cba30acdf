"""GEMM on the GPU vs the oracle.

* anyq_gemm_fused (exact path): bit-identical to the reference gemm_fused /
  gemm_reference for every format, layout and M (test_qgemm.cpp:53-160).
* device LUT GEMM paths (bf16 x, exact fp16 x fp16 products, fp32
  accumulation): the CUDA-core GEMV (m <= 4, gemv.cu) and the tcgen05 LUT GEMM
  (m <= 16, lutgemm.cu), each within
  |dy| <= 1e-5 * sum_j |x_j| * (|alpha*T| + |beta|) of
  gemm_reference(bf16(x), narrowed(qt)) computed by the oracle in fp32.
"""
import numpy as np
import pytest

from anyq_testutil import bits_equal, cfg

pytestmark = pytest.mark.gpu


def quantize_format(aq, orc, w, fmt, seed, group_size):
    c = cfg(granularity=3, group_size=group_size, seed=seed)
    aq.apply_format(c, fmt)
    return orc.quantize(w, c)


def test_hand_case(aq):
    from paper_2507_04610_b200.qtensor import QuantizedTensor

    c = cfg(codebook=0, bits=4, granularity=1, symmetric=1)
    qt = QuantizedTensor.empty(4, 4, c)
    codes = np.array([[8, 9, 10, 11], [12, 13, 14, 15], [0, 2, 4, 6], [7, 8, 9, 15]], np.uint8)
    qt.codes = aq.pack_codes(codes, 4)
    qt.alphas[:] = 0.2
    qt.betas[:] = 0
    y = aq.gemm_reference(np.array([[1, 2, 3, 4]], np.float32), qt)
    exp = 0.2 * np.array([0 + 2 + 6 + 12, 4 + 10 + 18 + 28, -8 - 12 - 12 - 8, -1 + 0 + 3 + 28])
    assert np.allclose(y[0], exp, rtol=1e-6)
    assert np.abs(aq.gemm_fused(np.zeros((2, 4), np.float32), qt)).max() == 0


@pytest.mark.parametrize("fmt", ["int4", "fp4", "nf4", "any4", "any2", "any3", "int8"])
@pytest.mark.parametrize("m", [1, 5, 16])
def test_fused_bit_exact_vs_reference(aq, orc, fmt, m):
    w = orc.gaussian(24, 56, 11)
    qt = quantize_format(aq, orc, w, fmt, 5, 8)
    x = orc.gaussian(m, 56, 13 + m)
    y = aq.gemm_fused(x, qt)
    assert bits_equal(y, orc.gemm_fused(x, qt))
    assert bits_equal(y, orc.gemm_reference(x, qt))
    assert bits_equal(aq.gemm_reference(x, qt), orc.gemm_reference(x, qt))


@pytest.mark.parametrize("tile_k", [2, 8, 32])
def test_ktiled_equals_rowmajor(aq, orc, tile_k):
    w = orc.gaussian(17, 40, 17)
    qt = quantize_format(aq, orc, w, "any4", 9, 8)
    tiled = aq.to_ktiled(qt, tile_k)
    x = orc.gaussian(4, 40, 19)
    assert bits_equal(aq.gemm_fused(x, tiled), aq.gemm_fused(x, qt))
    assert bits_equal(aq.gemm_fused(x, tiled), orc.gemm_fused(x, tiled))


def test_plan_mismatch_rejected(aq, orc):
    w = orc.gaussian(6, 16, 53)
    qt = quantize_format(aq, orc, w, "int4", 1, 8)
    x = orc.gaussian(2, 16, 59)
    plan = aq.make_plan(x, qt)
    plan.layout, plan.tile_k = 1, 4
    with pytest.raises(aq.ConfigError):
        aq.gemm_fused(x, qt, plan)
    with pytest.raises(aq.ShapeError):
        aq.gemm_reference(orc.gaussian(2, 17, 61), qt)


def test_fp4_code_15_raises(aq, orc):
    w = orc.gaussian(4, 32, 3)
    qt = quantize_format(aq, orc, w, "fp4", 1, 16)
    qt.codes[0] = 0xFF
    with pytest.raises(aq.CodeRangeError):
        aq.gemm_fused(orc.gaussian(1, 32, 2), qt)


@pytest.mark.slow
def test_property_sweep_1000_cases(aq, orc):
    """acceptance.cpp:415-453: M in 1..16, K,N in 8..256, 4 formats, both layouts."""
    r = orc.rng_double(4242, 0, 6000)
    fmts = ["int4", "fp4", "nf4", "any4"]
    for t in range(200):
        m = 1 + int(r[6 * t] * 16)
        n = 8 + int(r[6 * t + 1] * 249)
        k = 8 + int(r[6 * t + 2] * 249)
        fmt = fmts[int(r[6 * t + 3] * 4)]
        tile = [1, 2, 8, 32][int(r[6 * t + 4] * 4)]
        w = orc.gaussian(n, k, 7000 + t)
        qt = quantize_format(aq, orc, w, fmt, t, min(128, k) if k >= 2 else 2)
        if r[6 * t + 5] < 0.5:
            qt = orc.to_ktiled(qt, tile)
        x = orc.gaussian(m, k, 9000 + t)
        assert bits_equal(aq.gemm_fused(x, qt), orc.gemm_fused(x, qt)), (m, n, k, fmt)


# ---------------------------------------------------------------------------
# tensor-core path
# ---------------------------------------------------------------------------
def bf16(x):
    from oracle.refpy import bf16_round

    return bf16_round(x)


PATHS = {"gemv": 1, "tc": 2, "dequant": 3, "mma": 4}


def tc_gemm(aq, cuda, qt, x, path=2):
    import torch

    dt = aq.DeviceTensor(qt)
    xt = torch.from_numpy(bf16(x)).to("cuda", torch.bfloat16).contiguous()
    y = torch.empty((x.shape[0], qt.rows), dtype=torch.bfloat16, device="cuda")
    y32 = torch.empty((x.shape[0], qt.rows), dtype=torch.float32, device="cuda")
    dt.gemm(xt, y, y32, path=path)
    torch.cuda.synchronize()
    out = y32.cpu().numpy(), y.float().cpu().numpy()
    dt.close()
    return out


def tc_tolerance(orc, x, qt):
    """1e-5 * sum_j |x_j| (|alpha T[c]| + |beta|) per output element.

    Fixed tables are not narrowed by the reference (pack.cpp:159-169 narrows
    only learned LUTs) while the tensor-core path holds every table in fp16:
    for nf4 (the only fixed table with values that are not fp16-exact) the
    bound adds the table rounding, sum_j |x_j| * alpha * 2^-11 |T[c]|.
    """
    n = orc.narrowed(qt)
    nq = n.clone()
    nq.betas[:] = 0
    aT = np.abs(orc.dequantize(nq))
    b = np.abs(orc.dequantize(n) - orc.dequantize(nq))
    tol = 1e-5 * (np.abs(x) @ (aT + b).T)
    if qt.cfg.codebook == 2:  # nf4
        tol = tol + 2.0 ** -11 * (np.abs(x) @ aT.T)
    return tol + 1e-30


@pytest.mark.parametrize("path", ["gemv", "tc"])
@pytest.mark.parametrize("fmt", ["any4", "int4", "nf4", "fp4", "any3", "any2"])
@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8, 9, 16])
def test_tc_gemm_matches_reference(aq, orc, cuda, fmt, m, path):
    """any3 / any2 run on the 4-bit device layout (2^bits-entry LUT padded to 16)."""
    if path == "gemv" and m > 4:
        pytest.skip("the GEMV serves m <= 4")
    n, k = 200, 384  # ragged rows (not a multiple of 32), 3 chunks, 3 groups
    w = orc.gaussian(n, k, 31)
    c = cfg(granularity=3, group_size=128, seed=2)
    aq.apply_format(c, fmt)
    qt = orc.quantize(w, c)
    x = bf16(orc.gaussian(m, k, 33))
    y32, ybf = tc_gemm(aq, cuda, qt, x, PATHS[path])
    ref = orc.gemm_reference(x, orc.narrowed(qt))
    tol = tc_tolerance(orc, x, qt)
    err = np.abs(y32 - ref)
    assert np.all(err <= tol), f"max err {err.max()} tol {tol.min()}"
    assert np.all(np.abs(ybf - bf16(ref)) <= np.abs(ref) * 2 ** -7 + tol)


@pytest.mark.parametrize("path", ["gemv", "tc"])
@pytest.mark.parametrize("n,k,g", [(4096, 4096, 128), (1024, 4096, 128), (4096, 1024, 256),
                                   (96, 1280, 1280), (33, 128, 128),
                                   # GEMV work split: 151 row blocks (one full wave +
                                   # 3 split over 148 CTAs, some with empty ranges)
                                   (151 * 32 - 5, 512, 128)])
def test_tc_gemm_shapes(aq, orc, cuda, n, k, g, path):
    w = orc.gaussian(n, k, 41)
    gran = 1 if g == k else 3
    c = cfg(codebook=3, granularity=gran, group_size=g, seed=1, max_iters=8)
    qt = aq.quantize_any(w, c)
    x = bf16(orc.gaussian(3, k, 43))
    y32, _ = tc_gemm(aq, cuda, qt, x, PATHS[path])
    ref = orc.gemm_reference(x, orc.narrowed(qt))
    tol = tc_tolerance(orc, x, qt)
    assert np.all(np.abs(y32 - ref) <= tol)


@pytest.mark.parametrize("path", ["gemv", "tc"])
def test_tc_gemm_is_deterministic_and_rowwise_consistent(aq, orc, cuda, path):
    w = orc.gaussian(512, 1024, 5)
    qt = aq.quantize_any(w, cfg(codebook=3, max_iters=5))
    x1 = bf16(orc.gaussian(1, 1024, 6))
    mm = 4 if path == "gemv" else 16
    xm = np.repeat(x1, mm, axis=0)
    a, _ = tc_gemm(aq, cuda, qt, x1, PATHS[path])
    b, _ = tc_gemm(aq, cuda, qt, x1, PATHS[path])
    c, _ = tc_gemm(aq, cuda, qt, xm, PATHS[path])
    assert bits_equal(a, b)
    for r in range(mm):
        assert np.allclose(c[r], a[0], rtol=0, atol=1e-5 * np.abs(a[0]).max())


def test_gemv_rejects_unsupported_group(aq, orc, cuda):
    """group_size 384 is not 128 * 2^j: the GEMV refuses, AUTO falls back to tcgen05."""
    w = orc.gaussian(64, 768, 3)
    qt = aq.quantize_any(w, cfg(codebook=3, group_size=384, max_iters=3))
    x = bf16(orc.gaussian(1, 768, 4))
    with pytest.raises(aq.ConfigError):
        tc_gemm(aq, cuda, qt, x, PATHS["gemv"])
    y32, _ = tc_gemm(aq, cuda, qt, x, 0)
    ref = orc.gemm_reference(x, orc.narrowed(qt))
    assert np.all(np.abs(y32 - ref) <= tc_tolerance(orc, x, qt))


def test_gemm_chain_matches_single_launches(aq, orc, cuda):
    """anyq_dev_gemm_chain: one launch of a dependent chain equals the single
    launches bit for bit (x of problem i may be the y of problem i-1)."""
    import torch

    shapes = [(256, 384), (192, 384), (5000, 256), (384, 5000)]  # phase A + B + sparse split
    dts, qts = [], []
    for i, (n, k) in enumerate(shapes):
        qt = aq.quantize_any(orc.gaussian(n, k, 70 + i), cfg(codebook=3, max_iters=4, seed=i))
        qts.append(qt)
        dts.append(aq.DeviceTensor(qt))
    for m in (1, 2, 4):
        x0 = torch.from_numpy(bf16(orc.gaussian(m, 384, 80 + m))).cuda().to(torch.bfloat16)
        x2 = torch.from_numpy(bf16(orc.gaussian(m, 256, 90 + m))).cuda().to(torch.bfloat16)
        # chain: y0 = x0 W0, y1 = x0 W1 (independent), y2 = x2 W2, y3 = y2 W3 (waits on y2)
        ys = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for n, _ in shapes]
        y32 = [torch.empty(m, n, device="cuda", dtype=torch.float32) for n, _ in shapes]
        aq.gemm_chain(dts, [x0, x0, x2, ys[2]], ys, wait_prev=[0, 0, 1, 1], y32s=y32, path=aq.PATH_GEMV)
        torch.cuda.synchronize()
        xs = [x0, x0, x2, ys[2].clone()]
        for i, d in enumerate(dts):
            r = torch.empty(m, shapes[i][0], device="cuda", dtype=torch.float32)
            d.gemm(xs[i], None, r, path=1)
            torch.cuda.synchronize()
            assert torch.equal(r, y32[i]), i
            ref = orc.gemm_reference(xs[i].float().cpu().numpy(), orc.narrowed(qts[i]))
            assert np.all(np.abs(r.cpu().numpy() - ref) <= tc_tolerance(orc, xs[i].float().cpu().numpy(), qts[i]))
        # repeated launches reuse the self-resetting counters
        for _ in range(3):
            aq.gemm_chain(dts, [x0, x0, x2, ys[2]], ys, wait_prev=[0, 0, 1, 1], path=aq.PATH_GEMV)
        torch.cuda.synchronize()
    for d in dts:
        d.close()


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("n,k", [(70, 200), (33, 130), (300, 1000)])
def test_gemv_ragged_k(aq, orc, cuda, m, n, k):
    """K not a multiple of 128: the GEMV loads x directly (no bulk copy) and the
    zero-padded tail chunk contributes nothing; within the exact-product
    tolerance of gemm_reference(bf16(x), narrowed(qt))."""
    w = orc.gaussian(n, k, 71)
    qt = aq.quantize_any(w, cfg(codebook=3, granularity=1, seed=3, max_iters=5))
    x = bf16(orc.gaussian(m, k, 72))
    y32, _ = tc_gemm(aq, cuda, qt, x, PATHS["gemv"])
    ref = orc.gemm_reference(x, orc.narrowed(qt))
    assert np.all(np.abs(y32 - ref) <= tc_tolerance(orc, x, qt))


@pytest.mark.parametrize("m", [1, 3, 8, 16, 33, 64])
@pytest.mark.parametrize("n,k,g", [(200, 384, 128), (4096, 1024, 256), (96, 1280, 1280), (70, 200, 128),
                                   (1024, 4096, 128)])
def test_fused_mma_path(aq, orc, cuda, m, n, k, g):
    """Fused dequant-to-shared-memory + mma.sync path (lutmma.cu): bf16 weights
    as the dequant path, within 2^-8 * sum|x*w| of gemm_reference(bf16(x),
    narrowed(qt)), deterministic (fixed-order split-K combine)."""
    w = orc.gaussian(n, k, 61)
    gran = 1 if g == k else 3
    qt = aq.quantize_any(w, cfg(codebook=3, granularity=gran, group_size=g, seed=1, max_iters=6))
    x = bf16(orc.gaussian(m, k, 62))
    y32, ybf = tc_gemm(aq, cuda, qt, x, PATHS["mma"])
    y32b, _ = tc_gemm(aq, cuda, qt, x, PATHS["mma"])
    assert bits_equal(y32, y32b)
    nq = orc.narrowed(qt)
    ref = orc.gemm_reference(x, nq)
    tol = 2.0 ** -8 * (np.abs(x) @ np.abs(orc.dequantize(nq)).T) + 1e-30
    assert np.all(np.abs(y32 - ref) <= tol), float(np.max(np.abs(y32 - ref) / tol))
    # same bf16 weights and fp32 accumulation as the dequant + cuBLAS path
    yd, _ = tc_gemm(aq, cuda, qt, x, PATHS["dequant"])
    assert np.all(np.abs(y32 - yd) <= tol)


def test_auto_path_choice_and_agreement(aq, orc, cuda):
    """AUTO on a small tensor (3 row blocks): GEMV at m <= 2, K1t (tcgen05
    GEMV) at 3 <= m <= 4, the fused mma kernel for 5 <= m <= 32 (few row
    blocks), dequant + cuBLAS above; a long-K tensor leaves the GEMV at m = 3
    for the tcgen05 LUT GEMM; a tall tensor takes K1t from m = 2 to 16. AUTO's
    output equals the explicit path's output bit for bit."""
    import torch

    qt = aq.quantize_any(orc.gaussian(96, 512, 7), cfg(codebook=3, max_iters=4))
    dt = aq.DeviceTensor(qt)
    expect = {1: aq.PATH_GEMV, 2: aq.PATH_GEMV, 3: aq.PATH_GEMV_TC, 4: aq.PATH_GEMV_TC,
              5: aq.PATH_MMA, 8: aq.PATH_MMA, 32: aq.PATH_MMA, 33: aq.PATH_DEQUANT,
              64: aq.PATH_DEQUANT}
    for m, path in expect.items():
        assert dt.auto_path(m) == path, m
        x = torch.from_numpy(bf16(orc.gaussian(m, 512, 8 + m))).cuda().to(torch.bfloat16)
        ya = torch.empty(m, 96, device="cuda", dtype=torch.float32)
        ye = torch.empty(m, 96, device="cuda", dtype=torch.float32)
        dt.gemm(x, None, ya)
        dt.gemm(x, None, ye, path=path)
        torch.cuda.synchronize()
        assert torch.equal(ya, ye), m
    dt.close()
    # K = 14336 at m = 3: the x image (3 x 14336 bf16 -> fp16) no longer fits next to the table
    # and the weight ring, so AUTO hands it to the tcgen05 kernel
    long_k = aq.DeviceTensor(aq.quantize_any(orc.gaussian(64, 14336, 9), cfg(codebook=3, max_iters=2)))
    assert long_k.auto_path(1) == aq.PATH_GEMV
    assert long_k.auto_path(3) == aq.PATH_TC
    long_k.close()
    tall = aq.DeviceTensor(aq.quantize_any(orc.gaussian(300 * 32, 256, 10), cfg(codebook=3, max_iters=2)))
    assert [tall.auto_path(m) for m in (1, 2, 8, 16, 17, 128, 129)] == \
        [aq.PATH_GEMV] + [aq.PATH_GEMV_TC] * 3 + [aq.PATH_K2] * 2 + [aq.PATH_DEQUANT]
    tall.close()
    # down-shaped (32 row tiles, K = 14336): K2 split stream-K over every SM from m = 16
    down = aq.DeviceTensor(aq.quantize_any(orc.gaussian(4096, 14336, 11), cfg(codebook=3, max_iters=1)))
    assert [down.auto_path(m) for m in (16, 64, 128, 129)] == [aq.PATH_K2] * 3 + [aq.PATH_DEQUANT]
    down.close()


def test_gemm_chain_deps_decoder_pattern(aq, orc, cuda):
    """anyq_dev_gemm_chain_deps: a decoder-layer pattern (q, k, v, o <- q,
    gate <- o, up <- o, down <- up) in one launch, each problem waiting only for
    the problem its x comes from, equals the single launches bit for bit."""
    import torch

    K0 = 256
    shapes = [(256, K0), (64, K0), (64, K0), (K0, 256), (640, K0), (640, K0), (K0, 640)]
    deps = [-1, -1, -1, 0, 3, 3, 5]
    dts, qts = [], []
    for i, (n, k) in enumerate(shapes):
        qt = aq.quantize_any(orc.gaussian(n, k, 110 + i), cfg(codebook=3, max_iters=4, seed=i))
        qts.append(qt)
        dts.append(aq.DeviceTensor(qt))
    for m in (1, 2, 3):
        x0 = torch.from_numpy(bf16(orc.gaussian(m, K0, 120 + m))).cuda().to(torch.bfloat16)
        ys = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for n, _ in shapes]
        y32 = [torch.empty(m, n, device="cuda", dtype=torch.float32) for n, _ in shapes]
        xs = [x0 if d < 0 else ys[d] for d in deps]
        for _ in range(3):  # repeated launches reuse the self-resetting counters
            aq.gemm_chain(dts, xs, ys, y32s=y32, deps=deps, path=aq.PATH_GEMV)
        torch.cuda.synchronize()
        for i, d in enumerate(dts):
            xi = (x0 if deps[i] < 0 else ys[deps[i]]).clone()
            r = torch.empty(m, shapes[i][0], device="cuda", dtype=torch.float32)
            d.gemm(xi, None, r, path=1)
            torch.cuda.synchronize()
            assert torch.equal(r, y32[i]), i
    with pytest.raises(aq.ShapeError):  # a dependency must point backwards
        aq.gemm_chain(dts[:2], [x0, x0], ys[:2], deps=[-1, 1])
    for d in dts:
        d.close()


def test_gemm_chain_edge_cases(aq, orc, cuda):
    """The chain at its limits: 8 problems (the maximum), the same DeviceTensor
    in two problems, a 1-row and a 31-row tensor (a partial row block), a ragged
    K, a dependency reaching back 7 problems and two reading the same earlier
    output; equals the single launches bit for bit. 9 problems are refused."""
    import torch

    shapes = [(1, 256), (31, 256), (256, 256), (96, 256), (256, 200), (256, 256), (40, 256), (256, 256)]
    deps = [-1, -1, -1, 2, -1, 2, -1, 0]
    base = []
    for i, (n, k) in enumerate(shapes):
        qt = aq.quantize_any(orc.gaussian(n, k, 130 + i), cfg(codebook=3, max_iters=3, seed=i))
        base.append(aq.DeviceTensor(qt))
    dts = list(base)
    dts[5] = dts[2]  # same weights twice
    # problem 7 reads y0, which has 1 column: it needs a K = 1 tensor
    qt7 = aq.quantize_any(orc.gaussian(256, 1, 140), cfg(codebook=3, max_iters=3, seed=7))
    dts[7] = aq.DeviceTensor(qt7)
    for m in (1, 2, 4):
        xin = {256: torch.from_numpy(bf16(orc.gaussian(m, 256, 150 + m))).cuda().to(torch.bfloat16),
               200: torch.from_numpy(bf16(orc.gaussian(m, 200, 160 + m))).cuda().to(torch.bfloat16)}
        ns = [d.rows for d in dts]
        ys = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for n in ns]
        y32 = [torch.empty(m, n, device="cuda", dtype=torch.float32) for n in ns]
        xs = []
        for i, d in enumerate(deps):
            xs.append(ys[d] if d >= 0 else xin[dts[i].cols])
        for _ in range(2):
            aq.gemm_chain(dts, xs, ys, y32s=y32, deps=deps, path=aq.PATH_GEMV)
        torch.cuda.synchronize()
        for i, d in enumerate(dts):
            xi = xs[i].clone()
            r = torch.empty(m, d.rows, device="cuda", dtype=torch.float32)
            d.gemm(xi, None, r, path=1)
            torch.cuda.synchronize()
            assert torch.equal(r, y32[i]), (m, i)
    with pytest.raises(aq.ShapeError):
        x = torch.zeros(1, 256, device="cuda", dtype=torch.bfloat16)
        aq.gemm_chain([base[2]] * 9, [x] * 9, deps=[-1] * 9)
    for d in base + [dts[7]]:
        d.close()


@pytest.mark.parametrize("m", [1, 17, 64, 300])
@pytest.mark.parametrize("n,k,g", [(200, 384, 128), (4096, 1024, 256), (96, 1280, 1280), (70, 200, 128)])
def test_dequant_gemm_large_m(aq, orc, cuda, m, n, k, g):
    """Large-M path: bf16 dequantization + cuBLAS (fp32 accumulation), within
    2^-8 * sum|x*w| of gemm_reference(bf16(x), narrowed(qt))."""
    w = orc.gaussian(n, k, 51)
    gran = 1 if g == k else 3
    qt = aq.quantize_any(w, cfg(codebook=3, granularity=gran, group_size=g, seed=1, max_iters=6))
    x = bf16(orc.gaussian(m, k, 52))
    y32, ybf = tc_gemm(aq, cuda, qt, x, PATHS["dequant"])
    nq = orc.narrowed(qt)
    ref = orc.gemm_reference(x, nq)
    tol = 2.0 ** -8 * (np.abs(x) @ np.abs(orc.dequantize(nq)).T) + 1e-30
    assert np.all(np.abs(y32 - ref) <= tol)
    if m > 32:  # AUTO picks this path above m = 32
        y32a, _ = tc_gemm(aq, cuda, qt, x, 0)
        assert bits_equal(y32a, y32)
