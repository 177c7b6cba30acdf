"""Parity at the headline configurations.

* The exact bench step: one Llama-3-8B decoder layer's seven GEMMs in ONE
  anyq_dev_gemm_chain_deps launch with the decoder dependencies (bench.py
  LAYER / CHAIN_DEPS: o <- q, gate/up <- o, down <- up) at M = 1 and 2, and
  the same shapes as single AUTO launches at M = 1..4; the Llama-3-70B layer
  chain at M = 1 (config 3 at P = 1). Every y32 is compared with the oracle's
  gemm_reference(bf16(x), narrowed(qt)) (qgemm.cpp:36-40) under the K1 bound
  |dy| <= 1e-5 * sum_j |x_j| (|alpha T[c]| + |beta|); a dependent problem is
  checked against its actual input (the bf16 y of the problem it reads).
* A wide-dynamic-range x (values spread over 2^-30 .. 2^10 inside each
  128-k chunk): the GEMV's per-chunk bf16 -> fp16 * 2^e image loses the
  values far below the chunk maximum, within the same bound.
* Config 4 k-means: K = 14336 rows with synthetic activation statistics, the
  GPU learner against the unmodified reference build (oracle/_ref) on 256
  rows: LUT identity fraction and codes.

Weights are random-code any4 tensors (the GEMM does not care how codes were
learned; quantizing 10^9 weights on the CPU oracle would take hours).
"""
import numpy as np
import pytest

from anyq_testutil import cfg

pytestmark = pytest.mark.gpu

LAYER_8B = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096),
            (4096, 14336)]
LAYER_70B = [(8192, 8192), (1024, 8192), (1024, 8192), (8192, 8192), (28672, 8192), (28672, 8192),
             (8192, 28672)]
DEPS = [-1, -1, -1, 0, 3, 3, 5]  # the layer in its natural order
ORDER_SCHED = [0, 3, 1, 2, 5, 4, 6]  # bench.py CHAIN_ORDER (o before k/v, up before gate)


def synthetic_qt(n, k, seed):
    from paper_2507_04610_b200 import _abi
    from paper_2507_04610_b200.qtensor import QuantizedTensor

    rng = np.random.default_rng(seed)
    qt = QuantizedTensor.empty(n, k, _abi.default_config(codebook=_abi.CB_ANY, group_size=128))
    qt.codes[:] = rng.integers(0, 256, qt.codes.size, dtype=np.uint8)
    qt.luts[:] = np.sort(rng.random((n, 16), dtype=np.float32) * 15.0, axis=1).ravel()
    qt.alphas[:] = 0.01 + 0.04 * rng.random(qt.alphas.size, dtype=np.float32)
    qt.betas[:] = -0.3 * rng.random(qt.betas.size, dtype=np.float32)
    return qt


def row_slice(qt, r0, r1):
    """Rows [r0, r1) of a groupwise tensor as its own QuantizedTensor."""
    from paper_2507_04610_b200.qtensor import QuantizedTensor

    out = QuantizedTensor.empty(r1 - r0, qt.cols, qt.cfg)
    bpr = qt.codes.size // qt.rows
    gpr = qt.alphas.size // qt.rows
    out.codes[:] = qt.codes[r0 * bpr:r1 * bpr]
    out.luts[:] = qt.luts[r0 * 16:r1 * 16]
    out.alphas[:] = qt.alphas[r0 * gpr:r1 * gpr]
    out.betas[:] = qt.betas[r0 * gpr:r1 * gpr]
    return out


def check_rows(orc, qt, x, y32, rows, what):
    """y32[:, rows] against the oracle in row slices (bounded host memory)."""
    from oracle.refpy import bf16_round

    x = bf16_round(x)
    for r0 in rows:
        r1 = min(qt.rows, r0 + 2048)
        nq = orc.narrowed(row_slice(qt, r0, r1))
        ref = orc.gemm_reference(x, nq)
        zb = nq.clone()
        zb.betas[:] = 0
        a_t = np.abs(orc.dequantize(zb))
        b = np.abs(orc.dequantize(nq) - orc.dequantize(zb))
        tol = 1e-5 * (np.abs(x).astype(np.float64) @ (a_t + b).T.astype(np.float64)) + 1e-30
        err = np.abs(y32[:, r0:r1].astype(np.float64) - ref)
        assert np.all(err <= tol), (what, r0, float(np.max(err / tol)))


def run_chain(aq, torch, qts, m, seed, path=None, order=None):
    dts = [aq.DeviceTensor(q) for q in qts]
    x0 = torch.from_numpy(np.random.default_rng(seed).standard_normal((m, qts[0].cols),
                                                                       dtype=np.float32))
    x0 = x0.cuda().to(torch.bfloat16)
    ys = [torch.empty(m, q.rows, device="cuda", dtype=torch.bfloat16) for q in qts]
    y32 = [torch.empty(m, q.rows, device="cuda", dtype=torch.float32) for q in qts]
    xs = [x0 if d < 0 else ys[d] for d in DEPS]
    order = order or list(range(len(qts)))
    deps = [-1 if DEPS[j] < 0 else order.index(DEPS[j]) for j in order]
    aq.gemm_chain([dts[j] for j in order], [xs[j] for j in order], [ys[j] for j in order],
                  y32s=[y32[j] for j in order], deps=deps, path=path)
    torch.cuda.synchronize()
    out = [(xs[i].float().cpu().numpy(), y32[i].cpu().numpy()) for i in range(len(qts))]
    for d in dts:
        d.close()
    return out


def sample_rows(n):
    """Row slices to check: the first, a middle and the last 2048-row slice."""
    return sorted({0, max(0, (n // 2) // 32 * 32), max(0, n - 2048)})


@pytest.mark.parametrize("order", [None, ORDER_SCHED], ids=["natural", "bench"])
@pytest.mark.parametrize("m", [1, 2])
def test_llama3_8b_layer_chain(aq, orc, cuda, m, order):
    qts = [synthetic_qt(n, k, 100 + i) for i, (n, k) in enumerate(LAYER_8B)]
    for i, (x, y) in enumerate(run_chain(aq, cuda, qts, m, 7 + m, order=order)):
        check_rows(orc, qts[i], x, y, range(0, qts[i].rows, 2048), f"8b chain m={m} problem {i}")


@pytest.mark.parametrize("m", [1, 2])
def test_llama3_8b_layer_chain_tcgen05(aq, orc, cuda, m):
    """The same decoder-layer chain on the K1t engine (tcgen05 products)."""
    qts = [synthetic_qt(n, k, 100 + i) for i, (n, k) in enumerate(LAYER_8B)]
    for i, (x, y) in enumerate(run_chain(aq, cuda, qts, m, 7 + m, path=aq.PATH_GEMV_TC)):
        check_rows(orc, qts[i], x, y, range(0, qts[i].rows, 2048), f"8b K1t chain m={m} problem {i}")


def test_llama3_70b_layer_chain(aq, orc, cuda):
    qts = [synthetic_qt(n, k, 200 + i) for i, (n, k) in enumerate(LAYER_70B)]
    for i, (x, y) in enumerate(run_chain(aq, cuda, qts, 1, 11)):
        check_rows(orc, qts[i], x, y, sample_rows(qts[i].rows), f"70b chain problem {i}")


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("shape", [(14336, 4096), (4096, 14336), (1024, 4096)])
def test_llama3_8b_single_gemm_auto(aq, orc, cuda, shape, m):
    """Single launches through AUTO (the GEMV while its x image fits; down_proj
    at m >= 3 goes to the tcgen05 kernel) at the headline shapes."""
    import torch

    n, k = shape
    qt = synthetic_qt(n, k, 300 + m)
    x = np.random.default_rng(m).standard_normal((m, k), dtype=np.float32)
    dt = aq.DeviceTensor(qt)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    y32 = torch.empty(m, n, device="cuda", dtype=torch.float32)
    dt.gemm(xt, None, y32)
    torch.cuda.synchronize()
    check_rows(orc, qt, xt.float().cpu().numpy(), y32.cpu().numpy(), sample_rows(n),
               f"{shape} m={m} path {dt.auto_path(m)}")
    dt.close()


def test_gemv_wide_dynamic_range_x(aq, orc, cuda):
    import torch

    n, k = 512, 4096
    qt = synthetic_qt(n, k, 400)
    rng = np.random.default_rng(5)
    mag = np.exp2(rng.uniform(-30, 10, (2, k))).astype(np.float32)
    x = (mag * np.where(rng.random((2, k)) < 0.5, -1.0, 1.0)).astype(np.float32)
    dt = aq.DeviceTensor(qt)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    y32 = torch.empty(2, n, device="cuda", dtype=torch.float32)
    dt.gemm(xt, None, y32, path=aq.PATH_GEMV)
    torch.cuda.synchronize()
    check_rows(orc, qt, xt.float().cpu().numpy(), y32.cpu().numpy(), [0], "wide-range x")
    dt.close()


def test_config4_kmeans_k14336_with_stats(aq, orc, ref, cuda):
    """Config 4's long-K matrices (down_proj rows, K = 14336) with synthetic
    E|x_j|: the GPU learner vs the unmodified reference on 256 rows. The GPU
    M-step sums each cluster in sorted order (the reference in index order), so
    LUT bit-identity is reported as a fraction; every LUT entry agrees within
    1e-5 * 15 and the codes are the nearest-centroid codes of the GPU's LUT."""
    w = orc.gaussian(256, 14336, 1 + 7 * 0 + 6)
    exj = orc.synthetic_stats(14336, 10007 + 6)
    c = cfg(codebook=3)
    mine = aq.quantize_any(w, c, exj)
    theirs = ref.quantize(w, c, exj, threads=8)
    assert np.array_equal(mine.alphas.view(np.uint32), theirs.alphas.view(np.uint32))
    assert np.array_equal(mine.betas.view(np.uint32), theirs.betas.view(np.uint32))
    lm = mine.luts.reshape(256, 16)
    lt = theirs.luts.reshape(256, 16)
    same = np.all(lm.view(np.uint32) == lt.view(np.uint32), axis=1)
    assert same.mean() >= 0.95, same.mean()
    assert np.max(np.abs(lm - lt)) <= 1e-5 * 15
    # codes of rows whose LUT is identical are identical
    bpr = mine.codes.size // 256
    cm = mine.codes.reshape(256, bpr)[same]
    ct = theirs.codes.reshape(256, bpr)[same]
    assert np.array_equal(cm, ct)
    print(f"config-4 K=14336 LUT identity {same.mean():.4f} over 256 rows")
