"""Quantisation on the GPU vs the oracle.

Fixed formats (RTN, quantize.cpp:5-23) and scales are pure fp32 element
maths: bit-exact. The learned path (learner.cpp) is exact in its E-step and
deterministic; LUTs are expected bit-identical on (nearly) every row and codes
are always the exact nearest-centroid assignment of the GPU's own LUT.
Mirrors proj/tests/test_learner.cpp and test_scaling.cpp cases.
"""
import numpy as np
import pytest

from anyq_testutil import bits_equal, cfg

pytestmark = pytest.mark.gpu


FIXED = [(0, 4), (0, 3), (0, 2), (0, 8), (1, 4), (2, 4)]
GRANS = [(3, 16), (1, 128), (0, 128), (2, 128), (4, 128)]


@pytest.mark.parametrize("codebook,bits", FIXED)
@pytest.mark.parametrize("gran,gs", GRANS)
@pytest.mark.parametrize("sym", [0, 1])
def test_quantize_fixed_bit_exact(aq, orc, codebook, bits, gran, gs, sym):
    w = orc.gaussian(12, 40, 17 + gran, 3.0)
    c = cfg(codebook=codebook, bits=bits, granularity=gran, group_size=gs, block_size=5,
            symmetric=sym)
    a = aq.quantize_fixed(w, c)
    b = orc.quantize(w, c)
    assert a.same_as(b)


def test_zero_range_groups_fall_back_to_alpha_one(aq, orc):
    w = np.full((1, 4), 5.0, np.float32)
    a = aq.quantize_fixed(w, cfg(granularity=1))
    assert a.alphas[0] == 1.0 and a.betas[0] == 5.0


def test_signed_zero_min_is_first_encountered(aq, orc):
    w = np.array([[0.0, -0.0, 1.0, 2.0], [-0.0, 0.0, 1.0, 2.0]], np.float32)
    for gran in (1, 0, 2):
        c = cfg(granularity=gran)
        assert aq.quantize_fixed(w, c).same_as(orc.quantize(w, c))


def test_quantize_rejects_nonfinite_and_bad_config(aq):
    w = np.ones((3, 10), np.float32)
    w[0, 0] = np.nan
    with pytest.raises(aq.NonFiniteError):
        aq.quantize_fixed(w, cfg(granularity=1))
    with pytest.raises(aq.ConfigError):
        aq.quantize_any(np.ones((4, 8), np.float32), cfg(codebook=3, granularity=2))
    with pytest.raises(aq.ConfigError):
        aq.quantize_any(np.ones((4, 8), np.float32), cfg(codebook=0))
    with pytest.raises(aq.ConfigError):
        aq.quantize_fixed(np.ones((4, 8), np.float32), cfg(bits=5))


def test_negative_stats_rejected(aq, orc):
    w = orc.gaussian(4, 16, 3)
    st = np.ones(16, np.float32)
    st[3] = -1
    with pytest.raises(aq.StatsError):
        aq.quantize_any(w, cfg(codebook=3, group_size=8), st)


ANY_CASES = [
    dict(bits=4, granularity=3, group_size=16),
    dict(bits=4, granularity=1),
    dict(bits=2, granularity=3, group_size=8),
    dict(bits=3, granularity=3, group_size=32),
    dict(bits=8, granularity=3, group_size=64),
    dict(bits=4, granularity=3, group_size=16, symmetric=1),
    dict(bits=4, granularity=3, group_size=16, init=1),
    dict(bits=4, granularity=3, group_size=16, init=2),
    dict(bits=4, granularity=3, group_size=16, init=3),
    dict(bits=4, granularity=3, group_size=16, restarts=3),
    dict(bits=4, granularity=3, group_size=16, weighting=0),
    dict(bits=4, granularity=3, group_size=16, weighting=1),
]


@pytest.mark.parametrize("case", ANY_CASES)
@pytest.mark.parametrize("with_stats", [False, True])
def test_quantize_any_matches_oracle(aq, orc, case, with_stats):
    w = orc.gaussian(16, 96, 21)
    st = orc.synthetic_stats(96, 22) if with_stats else None
    c = cfg(codebook=3, seed=5, **case)
    a = aq.quantize_any(w, c, st)
    b = orc.quantize(w, c, st)
    assert bits_equal(a.alphas, b.alphas) and bits_equal(a.betas, b.betas)
    assert a.same_as(b), "LUT/codes differ from the oracle"


def test_lossless_rows_and_constant_rows(aq, orc):
    # few distinct values per row -> exact reconstruction (test_learner.cpp:313-327)
    rng = orc.rng_double(16, 0, 32)
    w = (np.floor(rng * 5) * 0.75 - 1.5).astype(np.float32).reshape(4, 8)
    qt = aq.quantize_any(w, cfg(codebook=3, granularity=1))
    back = aq.dequantize(qt)
    assert np.all(np.abs(back - w) <= 1e-6 * np.maximum(1, np.abs(w)))
    const = np.full((2, 40), 2.5, np.float32)
    q2 = aq.quantize_any(const, cfg(codebook=3, granularity=1))
    assert q2.same_as(orc.quantize(const, cfg(codebook=3, granularity=1)))


def test_offset_cancellation_dyadic(aq, orc):
    # test_learner.cpp:345-367: exact per-group shifts leave codes and LUTs bit-identical
    w = orc.dyadic(6, 48, 23)
    c = cfg(codebook=3, group_size=16, seed=77)
    base = aq.quantize_any(w, c)
    shifted = w.copy()
    for i in range(6):
        for j in range(48):
            g = i * 3 + j // 16
            shifted[i, j] += np.float32(1.0 / 1024.0) * np.float32((g * 37) % 512)
    moved = aq.quantize_any(shifted, c)
    assert bits_equal(base.codes, moved.codes) and bits_equal(base.luts, moved.luts)


def test_row_offset_keys_the_rng_like_a_split_matrix(aq, orc):
    w = orc.gaussian(24, 64, 9)
    c = cfg(codebook=3, group_size=32, seed=4)
    whole = aq.quantize_any(w, c)
    top = aq.quantize_any(w[:10], c, row_offset=0)
    bottom = aq.quantize_any(w[10:], c, row_offset=10)
    k = 16
    assert bits_equal(np.concatenate([top.luts, bottom.luts]), whole.luts)
    assert bits_equal(np.concatenate([top.codes, bottom.codes]), whole.codes)


@pytest.mark.slow
def test_config1_lut_identity_fraction(aq, orc, ref):
    """4096x4096 any4 g128 (BASELINE config 1): codes exact given the LUT,
    LUTs bit-identical to the reference on >= 99.9% of rows."""
    w = ref.gaussian(4096, 4096, 1)
    c = cfg(codebook=3)
    a = aq.quantize_any(w, c)
    b = ref.quantize(w, c, None, 8)
    assert bits_equal(a.alphas, b.alphas) and bits_equal(a.betas, b.betas)
    la = a.luts.reshape(4096, 16)
    lb = b.luts.reshape(4096, 16)
    same_rows = np.all(la.view(np.uint32) == lb.view(np.uint32), axis=1)
    frac = same_rows.mean()
    print(f"LUT rows bit-identical: {frac:.6f}")
    assert frac >= 0.999
    assert np.max(np.abs(la - lb)) <= 1e-5 * 15
    codes_a = aq.unpack_codes(a.codes, 4096, 4096, 4)
    codes_b = aq.unpack_codes(b.codes, 4096, 4096, 4)
    assert np.array_equal(codes_a[same_rows], codes_b[same_rows])


def test_config4_down_proj_with_stats(aq, ref):
    """BASELINE config 4 at its longest rows: the Llama-3-8B down_proj of layer 0
    (K = 14336, W = gaussian(4096, 14336, 1 + 6), stats = synthetic_stats(14336,
    10007 + 6)), any4 g128 with the activation weighting; 512 rows as two
    row_offset shards. alpha/beta bit-exact, LUT rows bit-identical to the
    reference on >= 99 % of rows (max |dLUT| <= 1e-5 * 15), codes identical on
    those rows."""
    K = 14336
    w = ref.gaussian(512, K, 7)
    exj = ref.synthetic_stats(K, 10013)
    c = cfg(codebook=3)
    want = ref.quantize(w, c, exj, 8)
    parts = [aq.quantize_any(w[:256], c, exj, row_offset=0), aq.quantize_any(w[256:], c, exj, row_offset=256)]
    alphas = np.concatenate([p.alphas for p in parts])
    betas = np.concatenate([p.betas for p in parts])
    assert bits_equal(alphas, want.alphas) and bits_equal(betas, want.betas)
    la = np.concatenate([p.luts for p in parts]).reshape(512, 16)
    lb = want.luts.reshape(512, 16)
    same_rows = np.all(la.view(np.uint32) == lb.view(np.uint32), axis=1)
    print(f"config-4 down_proj LUT rows bit-identical: {same_rows.mean():.4f}")
    assert same_rows.mean() >= 0.99
    assert np.max(np.abs(la - lb)) <= 1e-5 * 15
    codes_a = np.concatenate([aq.unpack_codes(p.codes, 256, K, 4) for p in parts])
    codes_b = aq.unpack_codes(want.codes, 512, K, 4)
    assert np.array_equal(codes_a[same_rows], codes_b[same_rows])


def test_near_duplicate_centroids_take_the_cta_kernel(aq, orc):
    """Rows whose centroids end within 2^-40 of the data range of each other
    (16 distinct values, two of them 0 and ~1e-30: k-means++ has to take the
    tiny one last) leave the warp-per-row k-means for the CTA kernel
    (kmeans.cu bail list); the result is still the reference's, bit for bit."""
    rng = np.random.default_rng(17)
    vals = np.array([0.0, 1e-30] + [float(v) for v in range(1, 15)], np.float32)
    w = np.stack([rng.permutation(np.repeat(vals, 6)) for _ in range(8)]).astype(np.float32)
    c = cfg(codebook=3, granularity=1, seed=3)
    a = aq.quantize_any(w, c)
    b = orc.quantize(w, c)
    assert a.same_as(b), "LUT/codes differ from the oracle"
    lut0 = np.asarray(a.luts, np.float32).reshape(w.shape[0], -1)[0]
    assert np.unique(lut0).size == 16  # both near-duplicate centroids survive
