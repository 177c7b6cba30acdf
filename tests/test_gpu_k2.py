"""K2 — the large-M tcgen05 LUT GEMM (ANYQ_PATH_K2, lutgemm2.cu): weights
dequantised to bf16 in shared memory (alpha * T[c] + beta in fp32, rounded
once), x by TMA (SWIZZLE_128B), tcgen05.mma with fp32 accumulation in TMEM.
Bound: |dy| <= 2^-8 * sum_j |x_j w_j| against gemm_reference(bf16(x),
narrowed(qt)) (qgemm.cpp:36-40), the tensor-core tolerance of
tests/test_gpu_gemm.py."""
import numpy as np
import pytest

from anyq_testutil import cfg
from test_gpu_gemm import bf16, tc_gemm

pytestmark = pytest.mark.gpu
K2 = 6


def check(aq, orc, cuda, qt, x):
    y32, ybf = tc_gemm(aq, cuda, qt, x, K2)
    nq = orc.narrowed(qt)
    ref = orc.gemm_reference(x, nq)
    w = orc.dequantize(nq)
    tol = 2.0 ** -8 * (np.abs(x).astype(np.float64) @ np.abs(w).T.astype(np.float64)) + 1e-30
    err = np.abs(y32.astype(np.float64) - ref)
    assert np.all(err <= tol), float(np.max(err / tol))
    assert np.all(np.isfinite(ybf))


@pytest.mark.parametrize("m", [1, 17, 64, 65, 128, 200, 256, 300, 513])
def test_k2_m_sweep(aq, orc, cuda, m):
    w = orc.gaussian(256, 512, 3)
    qt = aq.quantize_any(w, cfg(codebook=3, max_iters=4, seed=1))
    check(aq, orc, cuda, qt, bf16(orc.gaussian(m, 512, 4)))


@pytest.mark.parametrize("fmt", ["any4", "int4", "nf4", "fp4", "any3", "any2"])
def test_k2_formats(aq, orc, cuda, fmt):
    c = cfg(granularity=3, group_size=128, seed=2)
    aq.apply_format(c, fmt)
    qt = orc.quantize(orc.gaussian(200, 384, 31), c)  # ragged rows (not a multiple of 128), 3 chunks
    check(aq, orc, cuda, qt, bf16(orc.gaussian(96, 384, 33)))


@pytest.mark.parametrize("n,k,g", [(4096, 1024, 256), (96, 1280, 1280), (33, 136, 128), (1000, 4096, 128),
                                   (4096, 4096, 128)])
def test_k2_shapes(aq, orc, cuda, n, k, g):
    gran = 1 if g == k else 3
    qt = aq.quantize_any(orc.gaussian(n, k, 41), cfg(codebook=3, granularity=gran, group_size=g, seed=1, max_iters=3))
    check(aq, orc, cuda, qt, bf16(orc.gaussian(130, k, 43)))


def test_k2_deterministic(aq, orc, cuda):
    qt = aq.quantize_any(orc.gaussian(512, 1024, 5), cfg(codebook=3, max_iters=3))
    x = bf16(orc.gaussian(300, 1024, 6))
    a, _ = tc_gemm(aq, cuda, qt, x, K2)
    b, _ = tc_gemm(aq, cuda, qt, x, K2)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


# stream-K (one token tile, tiles not a whole number of waves): a tile split
# over CTAs is finished by the CTA holding its step 0, adding the later CTAs'
# fp32 partials in k order. (512, 14336): 4 tiles x 56 steps on 148 CTAs, every
# tile split over ~37 CTAs; (14336, 4096): the gate shape, 112 tiles x 16 steps.
@pytest.mark.parametrize("n,k,m", [(4096, 4096, 16), (4096, 4096, 128), (512, 14336, 64), (14336, 4096, 33),
                                   (4224, 1024, 100)])
def test_k2_stream_k(aq, orc, cuda, n, k, m):
    qt = aq.quantize_any(orc.gaussian(n, k, 51), cfg(codebook=3, granularity=3, group_size=128, seed=1, max_iters=2))
    check(aq, orc, cuda, qt, bf16(orc.gaussian(m, k, 53)))


def test_k2_stream_k_deterministic(aq, orc, cuda):
    qt = aq.quantize_any(orc.gaussian(512, 14336, 7), cfg(codebook=3, granularity=3, group_size=128, max_iters=2))
    x = bf16(orc.gaussian(64, 14336, 8))
    a, _ = tc_gemm(aq, cuda, qt, x, K2)
    for _ in range(3):
        b, _ = tc_gemm(aq, cuda, qt, x, K2)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
