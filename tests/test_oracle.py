"""CPU: the oracle (oracle/anyq_oracle.c, a C restatement of the reference) is
pinned against the golden fixtures generated from the UNMODIFIED reference
(tests/golden/make_golden.py) and, where the reference build is present
(oracle/_ref), against the reference itself on fresh random cases.

Covers the hot-path known-answer tests of the reference's own suite:
  pack 0x21 / 2-bit 0b11100100 / round trips   test_pack.cpp:53-88
  fp16 / bf16 KATs                              test_pack.cpp:96-118
  hand GEMM                                     test_qgemm.cpp:53-65
  sample weights [6,2,4,1]                      test_learner.cpp:60-97
  weighted mean 0.25, separable clusters        test_learner.cpp:137-158
  bits per weight 4.3125 / 4.25                 test_codebooks.cpp:179-201
  fused == reference bit-exact                  test_qgemm.cpp:83-95
"""
import json
import os

import numpy as np
import pytest

from anyq_testutil import bits_equal, cfg

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))
CASES = np.load(os.path.join(HERE, "golden", "cases.npz"))


def sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case_cfg(c):
    from paper_2507_04610_b200 import _abi

    cb, bits = {"int4": (0, 4), "fp4": (1, 4), "nf4": (2, 4), "any4": (3, 4), "any3": (3, 3),
                "any2": (3, 2), "int8": (0, 8), "int3": (0, 3)}[c["fmt"]]
    k = _abi.default_config(codebook=cb, bits=bits, granularity=c["granularity"],
                            symmetric=c["symmetric"], seed=c["seed"])
    if c["granularity"] == 3:
        k.group_size = c["group_size"]
    return k


def quantize_case(lib, c):
    w = lib.gaussian(c["rows"], c["cols"], c["w_seed"])
    exj = lib.synthetic_stats(c["cols"], c["stats_seed"]) if c["stats"] else None
    return lib.quantize(w, case_cfg(c), exj)


# ---------------------------------------------------------------------------
# golden (reference-generated) cases
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("c", GOLD["quant_cases"], ids=lambda c: c["name"])
def test_oracle_quantize_matches_golden(orc, c):
    qt = quantize_case(orc, c)
    n = c["name"]
    assert bits_equal(qt.codes, CASES[f"{n}.codes"])
    assert bits_equal(qt.alphas, CASES[f"{n}.alphas"])
    assert bits_equal(qt.betas, CASES[f"{n}.betas"])
    if qt.luts is not None:
        assert bits_equal(qt.luts, CASES[f"{n}.luts"])
    nq = orc.narrowed(qt)
    assert bits_equal(nq.alphas, CASES[f"{n}.narrowed_alphas"])
    if nq.luts is not None:
        assert bits_equal(nq.luts, CASES[f"{n}.narrowed_luts"])
    assert bits_equal(orc.dequantize(qt), CASES[f"{n}.dequant"])


@pytest.mark.parametrize("c", GOLD["quant_cases"], ids=lambda c: c["name"])
def test_oracle_gemm_matches_golden(orc, c):
    qt = quantize_case(orc, c)
    n = c["name"]
    for m, xs in c["x_seed"].items():
        x = orc.gaussian(int(m), c["cols"], xs)
        yf = orc.gemm_fused(x, qt)
        assert bits_equal(yf, CASES[f"{n}.y_fused_m{m}"])
        assert bits_equal(orc.gemm_reference(x, qt), CASES[f"{n}.y_ref_m{m}"])
        assert bits_equal(yf, CASES[f"{n}.y_ref_m{m}"])  # fused == reference (qgemm.hpp:6)


@pytest.mark.parametrize("i", range(3))
def test_oracle_kmeans_matches_golden(orc, i):
    c = GOLD["kmeans_cases"][i]
    x, w = CASES[f"km{i}.x"], CASES[f"km{i}.w"]
    k = cfg(codebook=3)
    init = orc.kmeans_pp_init(x, w, c["k"], c["seed"], c["row"])
    assert bits_equal(init.view(np.uint64), CASES[f"km{i}.init"].view(np.uint64))
    cen, asg, loss, iters = orc.weighted_kmeans(x, w, c["k"], k, c["seed"], c["row"])
    assert bits_equal(cen.view(np.uint64), CASES[f"km{i}.centroids"].view(np.uint64))
    assert bits_equal(asg, CASES[f"km{i}.assign"])
    assert loss == c["loss"] and iters == c["iters"]


def test_oracle_rng_stream(orc):
    assert np.array_equal(orc.rng_u64(7, 3, 16), CASES["rng_u64_seed7_row3"])
    assert bits_equal(orc.rng_double(7, 3, 16).view(np.uint64),
                      CASES["rng_double_seed7_row3"].view(np.uint64))


def test_config1_first_256_rows(orc):
    """the RNG is keyed by row, so the first 256 rows
    of the 4096x4096 quantization are reproducible on their own."""
    g = GOLD["config1"]["nostats"]
    w = orc.gaussian(4096, 4096, 1)[:256]
    qt = orc.quantize(w, cfg(codebook=3))
    assert sha(qt.codes) == g["codes_rows256"]
    assert sha(qt.luts) == g["luts_rows256"]
    assert sha(qt.alphas) == g["alphas_rows256"]
    assert sha(qt.betas) == g["betas_rows256"]
    assert qt.codes[:8].tobytes().hex() == g["row0_code_bytes"]
    assert np.float32(g["alpha0"]) == qt.alphas[0] and np.float32(g["beta0"]) == qt.betas[0]
    assert np.array_equal(qt.luts[:16], np.array(g["row0_lut"], np.float32))
    # the SURVEY's spot values (§8(c)) — identical to the reference build
    assert abs(qt.alphas[0] - 0.308991164) < 1e-8 and abs(qt.betas[0] + 2.30097008) < 1e-7
    s = GOLD["config1"]["stats"]
    qs = orc.quantize(w, cfg(codebook=3), orc.synthetic_stats(4096, 3))
    assert sha(qs.codes) == s["codes_rows256"] and sha(qs.luts) == s["luts_rows256"]


# ---------------------------------------------------------------------------
# known answers from the reference test-suite
# ---------------------------------------------------------------------------
def test_pack_kats(orc):
    assert orc.pack_codes(np.array([[1, 2]], np.uint8), 4).tolist() == [0x21]
    assert orc.pack_codes(np.array([[0, 1, 2, 3]], np.uint8), 2).tolist() == [0b11100100]
    rng = np.random.default_rng(0)
    for bits in (2, 3, 4, 8):
        codes = rng.integers(0, 1 << bits, (5, 13), dtype=np.uint8)
        p = orc.pack_codes(codes, bits)
        assert p.size == 5 * ((13 * bits + 7) // 8)  # rows byte-aligned (pack.hpp:45)
        assert np.array_equal(orc.unpack_codes(p, 5, 13, bits), codes)


def test_half_kats(orc):
    for v, h in GOLD["f16_kat"]:
        if isinstance(h, str):
            with pytest.raises(Exception):
                orc.f32_to_f16(v)
        else:
            assert orc.f32_to_f16(v) == h, v
    for v, h in GOLD["bf16_kat"]:
        assert orc.f32_to_bf16(v) == h, v
    # exhaustive fp16 round trip (test_pack.cpp:120-131)
    for h in range(0, 65536, 7):
        f = orc.f16_to_f32(h)
        if np.isfinite(f):
            assert orc.f32_to_f16(f) == h or (f == 0 and (h & 0x7FFF) == 0)


def test_bits_per_weight(orc):
    assert GOLD["bits_per_weight_4096"] == {"any4": 4.3125, "int4": 4.25, "nf4": 4.25}
    for fmt, cb in (("any4", 3), ("int4", 0), ("nf4", 2)):
        assert orc.storage_bits_per_entry(cfg(codebook=cb), 4096, 4096) == \
            GOLD["bits_per_weight_4096"][fmt]


def test_weighted_mean_and_separable(orc):
    k = cfg(codebook=3)
    cen, asg, _, _ = orc.weighted_kmeans(np.array([0, 1], np.float32),
                                         np.array([3, 1], np.float32), 1, k, 0, 0)
    assert cen[0] == 0.25
    x = np.array([0, 0, 0, 10, 10, 10], np.float32)
    cen, asg, loss, _ = orc.weighted_kmeans(x, np.ones(6, np.float32), 2, k, 0, 0)
    assert sorted(cen.tolist()) == [0.0, 10.0] and loss == 0.0


def test_hand_gemm(orc):
    from paper_2507_04610_b200.qtensor import QuantizedTensor

    c = cfg(codebook=0, bits=4, granularity=1, symmetric=1)
    qt = QuantizedTensor.empty(4, 4, c)
    codes = np.array([[8, 9, 10, 11], [12, 13, 14, 15], [0, 2, 4, 6], [7, 8, 9, 15]], np.uint8)
    qt.codes = orc.pack_codes(codes, 4)
    qt.alphas[:] = 0.2
    y = orc.gemm_fused(np.array([[1, 2, 3, 4]], np.float32), qt)
    exp = 0.2 * np.array([0 + 2 + 6 + 12, 4 + 10 + 18 + 28, -8 - 12 - 12 - 8, -1 + 0 + 3 + 28])
    assert np.allclose(y[0], exp, rtol=1e-6)


# ---------------------------------------------------------------------------
# oracle == unmodified reference on fresh random cases (skipped without _ref)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("fmt", ["any4", "any3", "int4", "nf4", "fp4"])
@pytest.mark.parametrize("trial", range(3))
def test_oracle_equals_reference(orc, ref, fmt, trial):
    from paper_2507_04610_b200 import anyq

    r = orc.rng_double(99, trial, 8)
    n = 3 + int(r[0] * 40)
    k = 8 + int(r[1] * 120)
    c = cfg(granularity=3, group_size=[8, 16, 32][int(r[2] * 3)], seed=trial)
    anyq.apply_format(c, fmt)
    w = orc.heavy_tailed(n, k, 600 + trial) if r[3] < 0.5 else orc.gaussian(n, k, 600 + trial)
    exj = orc.synthetic_stats(k, 700 + trial) if r[4] < 0.5 else None
    a, b = orc.quantize(w, c, exj), ref.quantize(w, c, exj)
    assert bits_equal(a.codes, b.codes) and bits_equal(a.alphas, b.alphas)
    assert bits_equal(a.betas, b.betas)
    if a.luts is not None:
        assert bits_equal(a.luts, b.luts)
    x = orc.gaussian(1 + int(r[5] * 9), k, 800 + trial)
    assert bits_equal(orc.gemm_fused(x, a), ref.gemm_fused(x, b))


def _seq_mean_abs(x):
    """collect_stats' statistic in numpy: the double sum runs over samples in order."""
    acc = np.zeros(x.shape[1], np.float64)
    for r in range(x.shape[0]):
        acc += np.abs(x[r].astype(np.float64))
    return (acc / x.shape[0]).astype(np.float32)


def test_column_mean_abs_oracle(orc):
    """E|x_j| of collect_stats (calibration.cpp:62-67): the reference's own hand
    case (test_calibration.cpp:30-40), zeros, order/duplication invariance
    (test_calibration.cpp:64-84, 1e-6) and the sequential double sum."""
    from oracle.refpy import OracleError

    assert orc.column_mean_abs(np.array([[1, -1], [3, -3]], np.float32)).tolist() == [2.0, 2.0]
    assert not orc.column_mean_abs(np.zeros((5, 4), np.float32)).any()
    x = orc.gaussian(32, 16, 77)
    base = orc.column_mean_abs(x)
    assert np.allclose(orc.column_mean_abs(x[::-1]), base, rtol=1e-6, atol=0)
    assert np.allclose(orc.column_mean_abs(np.vstack([x, x])), base, rtol=1e-6, atol=0)
    for shape, seed in [((1, 7), 1), ((300, 33), 2), ((1000, 5), 3)]:
        x = orc.heavy_tailed(*shape, seed, 0.05, 40.0)
        assert np.array_equal(orc.column_mean_abs(x), _seq_mean_abs(x))
    bad = np.ones((3, 3), np.float32)
    bad[1, 2] = np.inf
    with pytest.raises(OracleError):
        orc.column_mean_abs(bad)
    with pytest.raises(OracleError):
        orc.column_mean_abs(np.zeros((0, 3), np.float32))


def test_eval_metrics_oracle(orc):
    """weight_error / output_error restated from eval.cpp:11-46, against numpy."""
    w = orc.gaussian(40, 200, 5)
    qt = orc.quantize(w, cfg(codebook=3, granularity=3, group_size=64, max_iters=5, seed=1))
    d = orc.dequantize(qt).astype(np.float64)
    mse, rel = orc.weight_error(w, qt)
    e = w.astype(np.float64) - d
    assert np.isclose(mse, (e * e).sum() / w.size, rtol=1e-12)
    assert np.isclose(rel, np.sqrt((e * e).sum()) / np.sqrt((w.astype(np.float64) ** 2).sum()), rtol=1e-12)
    x = orc.gaussian(6, 200, 6)
    y = orc.gemm_dense(x, w).astype(np.float64)
    yq = orc.gemm_reference(x, qt).astype(np.float64)
    assert np.isclose(orc.output_error(w, qt, x), ((yq - y) ** 2).mean(), rtol=1e-12)
