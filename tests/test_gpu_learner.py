"""The per-row learner API on the GPU (anyq_kmeans_problems: kmeans_pp_init,
weighted_kmeans, learn_row_lut, learner.hpp:55-68), build_sample_weights,
round_to_codebook, scaled_values and the scalar helpers, against the
reference's golden fixtures and the unmodified reference build (oracle/_ref).

The problem path sums in the reference's sample-index order, so centroids,
assignments, losses, iteration counts and the advanced RNG counter are
bit-identical by construction, including restarts, random / grid / nf4
initialisation, zero-weight samples and rows with fewer distinct values than
centroids.
"""
import numpy as np
import pytest

from anyq_testutil import bits_equal, cfg

from test_oracle import CASES, GOLD  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("i", range(3))
def test_kmeans_golden(aq, cuda, i):
    c = GOLD["kmeans_cases"][i]
    x, w = CASES[f"km{i}.x"], CASES[f"km{i}.w"]
    init = aq.kmeans_pp_init(x, w, c["k"], aq.rng_for_row(c["seed"], c["row"]))
    assert bits_equal(init.view(np.uint64), CASES[f"km{i}.init"].view(np.uint64))
    cen, asg, loss, iters = aq.weighted_kmeans(x, w, c["k"], cfg(codebook=3),
                                               aq.rng_for_row(c["seed"], c["row"]))
    assert bits_equal(cen.view(np.uint64), CASES[f"km{i}.centroids"].view(np.uint64))
    assert bits_equal(asg, CASES[f"km{i}.assign"])
    assert loss == c["loss"] and iters == c["iters"]


def _problems():
    """(name, samples, weights, k, config overrides) covering the learner's branches."""
    rng = np.random.default_rng(17)
    out = []
    for t in range(24):
        n = int(rng.integers(2, 700))
        x = rng.standard_normal(n).astype(np.float32)
        if t % 5 == 1:  # few distinct values (padding / empty clusters)
            x = np.round(x * 1.5).astype(np.float32)
        w = (rng.random(n) * 2).astype(np.float32)
        if t % 4 == 2:
            w[rng.random(n) < 0.4] = 0.0  # zero-weight samples
        if not (w > 0).any():
            w[0] = 1.0
        k = [2, 4, 8, 16, 3, 16][t % 6]
        over = {"init": [0, 1, 2, 3][t % 4], "restarts": 1 + t % 3, "max_iters": [100, 7][t % 2]}
        if over["init"] == 3 and k != 16:
            over["init"] = 0
        out.append((f"p{t}", x, w, k, over))
    return out


@pytest.mark.parametrize("case", _problems(), ids=lambda c: c[0])
def test_weighted_kmeans_matches_reference(aq, ref, cuda, case):
    _, x, w, k, over = case
    c = cfg(codebook=3, **over)
    for row in (0, 5):
        r = aq.rng_for_row(9, row)
        cen, asg, loss, iters = aq.weighted_kmeans(x, w, k, c, r)
        rc, ra, rl, ri = ref.weighted_kmeans(x, w, k, c, 9, row)
        assert bits_equal(cen.view(np.uint64), rc.view(np.uint64))
        assert bits_equal(asg, ra)
        assert loss == rl and iters == ri
        bits = {2: 1, 4: 2, 8: 3, 16: 4}.get(k)
        if bits:
            lut, codes, l2 = aq.learn_row_lut(x, w, bits, c, aq.rng_for_row(9, row))
            rlut, rcodes, rl2 = ref.learn_row_lut(x, w, bits, c, 9, row)
            assert bits_equal(lut, rlut) and bits_equal(codes, rcodes) and l2 == rl2


def test_kmeans_pp_init_matches_reference_and_advances_rng(aq, ref, cuda):
    rng = np.random.default_rng(3)
    for t in range(20):
        n = int(rng.integers(1, 400))
        x = rng.standard_normal(n).astype(np.float32)
        w = rng.random(n).astype(np.float32) + 0.01
        k = int(rng.integers(1, 20))
        r = aq.rng_for_row(t, 1)
        mine = aq.kmeans_pp_init(x, w, k, r)
        theirs = ref.kmeans_pp_init(x, w, k, t, 1)
        assert bits_equal(mine.view(np.uint64), theirs.view(np.uint64))
        assert r[1] > 0 or k == 1 and n >= 1


def test_learner_errors(aq, cuda):
    r = aq.rng_for_row(0, 0)
    with pytest.raises(aq.ShapeError):
        aq.weighted_kmeans(np.zeros(3, np.float32), np.ones(2, np.float32), 2, cfg(codebook=3), r)
    with pytest.raises(aq.StatsError):
        aq.weighted_kmeans(np.zeros(3, np.float32), np.zeros(3, np.float32), 2, cfg(codebook=3), r)
    with pytest.raises(aq.StatsError):
        aq.kmeans_pp_init(np.zeros(3, np.float32), np.array([1, -1, 1], np.float32), 2, r)
    with pytest.raises(aq.NonFiniteError):
        aq.kmeans_pp_init(np.array([0, np.inf, 1], np.float32), np.ones(3, np.float32), 2, r)
    with pytest.raises(aq.ConfigError):
        aq.weighted_kmeans(np.zeros(3, np.float32), np.ones(3, np.float32), 0, cfg(codebook=3), r)
    with pytest.raises(aq.ConfigError):
        aq.weighted_kmeans(np.zeros(3, np.float32), np.ones(3, np.float32), 300, cfg(codebook=3), r)


def test_build_sample_weights_kat(aq, cuda):
    """test_learner.cpp:60-97: groupwise g=2 scales (2, 1), stats (3, 1, 4, 1)."""
    c = cfg(granularity=3, group_size=2)
    stats = np.array([3, 1, 4, 1], np.float32)
    a = np.array([2, 1], np.float32)
    assert np.array_equal(aq.build_sample_weights(c, 1, 4, a, 0, stats, 2), [6, 2, 4, 1])
    assert np.array_equal(aq.build_sample_weights(c, 1, 4, a, 0, stats, 1), stats)
    assert np.array_equal(aq.build_sample_weights(c, 1, 4, a, 0, stats, 0), np.ones(4))
    with pytest.raises(aq.StatsError):
        aq.build_sample_weights(c, 1, 4, a, 0, np.array([3, 1, -1, 1], np.float32), 1)
    with pytest.raises(aq.StatsError):
        aq.build_sample_weights(c, 1, 4, a, 0, np.ones(3, np.float32), 0)


def test_round_and_tables_match_oracle(aq, orc, cuda):
    for cb, bits, shifted in [(0, 4, False), (0, 4, True), (0, 2, False), (0, 8, False), (1, 4, False),
                              (2, 4, False)]:
        t = aq.fixed_table(cb, bits, shifted)
        assert t.size == (15 if cb == 1 else 1 << bits)
        assert np.all(np.diff(t) > 0)
        ws = (orc.gaussian(17, 33, 5 + bits) * float(t[-1]) * 0.7).astype(np.float32)
        ws[0, :4] = [t[0] - 1, t[-1] + 1, (t[0] + t[1]) / 2, t[1]]  # clamps and an exact tie
        codes = aq.round_to_codebook(ws, t)
        d = np.abs(ws[..., None] - t[None, None, :])
        best = np.argmin(d, axis=2)  # first minimum = ties to the smaller index
        assert np.array_equal(codes, best)
    with pytest.raises(aq.NonFiniteError):
        aq.round_to_codebook(np.array([[np.nan]], np.float32), aq.fixed_table(0, 4))


def test_scaled_values_and_scalars(aq, orc, cuda):
    w = orc.gaussian(12, 40, 2)
    for fmt in ("any4", "nf4", "int3"):
        c = cfg(granularity=3, group_size=8, seed=1, max_iters=5)
        aq.apply_format(c, fmt)
        qt = orc.quantize(w, c)
        sv = aq.scaled_values(qt)
        # dequantize(qt) = alpha * scaled_values + beta (scaling.cpp:85-96)
        dq = orc.dequantize(qt)
        a = np.repeat(qt.alphas.reshape(12, -1), 8, axis=1)[:, :40]
        b = np.repeat(qt.betas.reshape(12, -1), 8, axis=1)[:, :40]
        assert bits_equal((a * sv + b).astype(np.float32), dq)
    for f, h in GOLD["f16_kat"]:
        if isinstance(h, str):  # the reference raises (overflow)
            with pytest.raises(aq.IoError):
                aq.f32_to_f16(f)
        else:
            assert aq.f32_to_f16(f) == h and aq.f16_to_f32(h) == orc.f16_to_f32(h)
    for f, h in GOLD["bf16_kat"]:
        assert aq.f32_to_bf16(f) == h
    with pytest.raises(aq.IoError):
        aq.f32_to_f16(1e6)
    with pytest.raises(aq.NonFiniteError):
        aq.f32_to_bf16(float("inf"))
    for fmt, bits in GOLD["bits_per_weight_4096"].items():
        c = cfg(granularity=3)
        aq.apply_format(c, fmt)
        assert aq.storage_bits_per_entry(c, 4096, 4096) == bits


def test_bench_gemm_rows(aq, orc, cuda):
    """The bench timing loop on the device returns positive per-run times for
    the dense, exact-fused and A16W4 kinds."""
    w = orc.gaussian(256, 512, 3)
    x = orc.gaussian(2, 512, 4)
    qt = aq.quantize_any(w, cfg(codebook=3, max_iters=4))
    for kind, q in ((0, None), (1, qt), (2, qt)):
        ns = aq.bench_gemm(kind, q, w, x, 5)
        assert ns.shape == (5,) and np.all(ns > 0)
