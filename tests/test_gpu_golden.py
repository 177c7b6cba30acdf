"""GPU: the CUDA library reproduces the reference-generated golden fixtures
(tests/golden/, made by tests/golden/make_golden.py from the unmodified
reference) bit for bit — quantization (codes, LUTs, alpha/beta), narrowing,
dequantization and the exact gemm_fused path — plus the full config-1
fingerprints of SURVEY.md §8(c) (4096x4096 any4 g128, with and without stats).
"""
import json
import os

import numpy as np
import pytest

from anyq_testutil import bits_equal

from test_oracle import CASES, GOLD, case_cfg, sha  # noqa: F401

pytestmark = pytest.mark.gpu


def gpu_quantize(aq, orc, c):
    w = orc.gaussian(c["rows"], c["cols"], c["w_seed"])
    exj = orc.synthetic_stats(c["cols"], c["stats_seed"]) if c["stats"] else None
    k = case_cfg(c)
    if k.codebook == 3:
        return aq.quantize_any(w, k, exj)
    return aq.quantize_fixed(w, k)


@pytest.mark.parametrize("c", GOLD["quant_cases"], ids=lambda c: c["name"])
def test_gpu_quantize_matches_golden(aq, orc, cuda, c):
    qt = gpu_quantize(aq, orc, c)
    n = c["name"]
    assert bits_equal(qt.codes, CASES[f"{n}.codes"])
    assert bits_equal(qt.alphas, CASES[f"{n}.alphas"])
    assert bits_equal(qt.betas, CASES[f"{n}.betas"])
    if qt.luts is not None:
        assert bits_equal(qt.luts, CASES[f"{n}.luts"])
    nq = aq.narrowed(qt)
    assert bits_equal(nq.alphas, CASES[f"{n}.narrowed_alphas"])
    if nq.luts is not None:
        assert bits_equal(nq.luts, CASES[f"{n}.narrowed_luts"])
    assert bits_equal(aq.dequantize(qt), CASES[f"{n}.dequant"])
    for m, xs in c["x_seed"].items():
        x = orc.gaussian(int(m), c["cols"], xs)
        assert bits_equal(aq.gemm_fused(x, qt), CASES[f"{n}.y_fused_m{m}"])


@pytest.mark.parametrize("tag", ["nostats", "stats"])
def test_gpu_config1_fingerprints(aq, orc, cuda, tag):
    g = GOLD["config1"][tag]
    from anyq_testutil import cfg

    w = orc.gaussian(4096, 4096, 1)
    exj = orc.synthetic_stats(4096, 3) if tag == "stats" else None
    qt = aq.quantize_any(w, cfg(codebook=3), exj)
    assert sha(qt.codes) == g["codes"]
    assert sha(qt.luts) == g["luts"]
    assert sha(qt.alphas) == g["alphas"]
    assert sha(qt.betas) == g["betas"]
    if tag == "nostats":
        y = aq.gemm_fused(orc.gaussian(1, 4096, 2), qt)
        assert sha(y) == g["y"]
        assert np.array_equal(y[0, :3], np.array(g["y_first3"], np.float32))
