"""§8(f) rows 3-4 pinned to the reference build: calibration.cpp and eval.cpp
are compiled unmodified into oracle/_ref (oracle/Makefile), so

* the C restatement's E|x_j| (orc_column_mean_abs) equals collect_stats
  (calibration.cpp:50-75) bit for bit, and its weight_error / output_error
  (anyq_oracle.c) equal eval.cpp:11-46 bit for bit;
* the product's eval_activations (host Box-Muller, capi.cu) equals
  eval.cpp:48-61 bit for bit (CPU);
* on the GPU, column_mean_abs equals collect_stats bit for bit and
  compare_formats (quantize + weight/output error per format, eval.cpp:62-86)
  matches the reference's report: the quantizations are bit-identical, the
  error sums differ only by summation order (rel 1e-12), bits exactly.
"""
import numpy as np
import pytest

from anyq_testutil import cfg


@pytest.mark.parametrize("shape,seed", [((1, 7), 1), ((300, 33), 2), ((1000, 5), 3), ((64, 4096), 4)])
def test_stats_restatement_equals_collect_stats(orc, ref, shape, seed):
    x = ref.heavy_tailed(*shape, seed, 0.05, 40.0)
    assert np.array_equal(orc.column_mean_abs(x), ref.collect_stats(x))


@pytest.mark.parametrize("fmt_cfg", [dict(codebook=3, granularity=3, group_size=64, max_iters=5, seed=1),
                                     dict(codebook=0, granularity=1),
                                     dict(codebook=2, granularity=3, group_size=32, symmetric=1)])
def test_eval_restatement_equals_reference(orc, ref, fmt_cfg):
    w = ref.gaussian(40, 200, 5)
    qt = ref.quantize(w, cfg(**fmt_cfg))
    assert orc.weight_error(w, qt) == ref.weight_error(w, qt)
    x = ref.gaussian(6, 200, 6)
    assert orc.output_error(w, qt, x) == ref.output_error(w, qt, x)


@pytest.mark.parametrize("rows,cols,seed,stats", [(5, 7, 3, False), (64, 128, 1, True), (3, 4096, 9, True)])
def test_eval_activations_equal_reference(aq, ref, rows, cols, seed, stats):
    exj = ref.synthetic_stats(cols, seed + 10) if stats else None
    assert np.array_equal(aq.eval_activations(rows, cols, exj, seed), ref.eval_activations(rows, cols, exj, seed))


def _compare(aq, ref, w, formats, base, exj, eval_rows):
    rows, csv = aq.compare_formats(w, formats, base, exj, eval_rows=eval_rows)
    want = ref.compare_formats(w, formats, base, exj, eval_rows=eval_rows)
    for r, (mse, rel, omse, bits) in zip(rows, want):
        assert np.isclose(r["weight_mse"], mse, rtol=1e-12, atol=0), r
        assert np.isclose(r["weight_rel_frobenius"], rel, rtol=1e-12, atol=0), r
        assert np.isclose(r["output_mse"], omse, rtol=1e-12, atol=0), r
        assert r["bits_per_entry"] == bits
    assert csv.startswith("schema_version,module,format,")
    return rows


@pytest.mark.gpu
def test_compare_formats_reference_case(aq, ref, cuda):
    """test_eval.cpp:155-183's case: 16 x 128, g64, seed 9, synthetic stats."""
    w = ref.gaussian(16, 128, 17)
    base = cfg(granularity=3, group_size=64, seed=9)
    rows = _compare(aq, ref, w, ["int4", "fp4", "nf4", "any4"], base, ref.synthetic_stats(128, 18), 16)
    assert rows[3]["bits_per_entry"] > rows[0]["bits_per_entry"] > 4.0


@pytest.mark.gpu
@pytest.mark.parametrize("stats", [False, True])
def test_compare_formats_larger(aq, ref, cuda, stats):
    w = ref.gaussian(256, 1024, 23)
    exj = ref.synthetic_stats(1024, 24) if stats else None
    base = cfg(granularity=3, group_size=128, seed=5)
    _compare(aq, ref, w, ["int4", "nf4", "any3", "any4"], base, exj, 64)


@pytest.mark.gpu
def test_column_mean_abs_equals_collect_stats(aq, ref, cuda):
    for shape, seed in [((4096, 4096), 1), ((333, 1000), 2)]:
        x = ref.heavy_tailed(*shape, seed, 0.05, 40.0)
        assert np.array_equal(aq.column_mean_abs(x), ref.collect_stats(x))
