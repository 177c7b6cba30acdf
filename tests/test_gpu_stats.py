"""The statistics around the path on the GPU: E|x_j| of
collect_stats (calibration.cpp:62-67, bit-exact) and weight_error / output_error
(eval.cpp:11-46), against the oracle restatement."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,seed", [(1, 1, 1), (1, 4096, 2), (2, 5, 3), (255, 33, 4), (256, 32, 5),
                                      (257, 31, 6), (1000, 100, 7), (4096, 1024, 8), (513, 4097, 9)])
def test_column_mean_abs_bit_exact(aq, orc, cuda, m, k, seed):
    x = orc.heavy_tailed(m, k, seed, 0.02, 60.0)
    x[::7, ::3] *= -1.0
    if m > 3 and k > 3:
        x[1, 1] = -0.0
        x[2, 2] = 1e-42  # subnormal
        x[3, 3] = 3.0e38
    exp = orc.column_mean_abs(x)
    got = aq.column_mean_abs(x)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    xd = cuda.from_numpy(x).cuda()
    dev = aq.dev_column_mean_abs(xd)
    cuda.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), exp.view(np.uint32))


def test_column_mean_abs_reference_cases(aq, orc, cuda):
    """test_calibration.cpp:30-48: the hand case and all-zero inputs."""
    assert aq.column_mean_abs(np.array([[1, -1], [3, -3]], np.float32)).tolist() == [2.0, 2.0]
    assert not aq.column_mean_abs(np.zeros((5, 4), np.float32)).any()


def test_column_mean_abs_errors(aq, cuda):
    bad = np.ones((4, 3), np.float32)
    bad[2, 1] = np.nan
    with pytest.raises(aq.NonFiniteError):
        aq.column_mean_abs(bad)
    with pytest.raises(aq.ShapeError):
        aq.column_mean_abs(np.zeros((0, 3), np.float32))


@pytest.mark.parametrize("fmt", ["any4", "int4", "fp4", "nf4", "any3"])
def test_eval_metrics_match_oracle(aq, orc, cuda, fmt):
    """weight_error / output_error (eval.cpp:11-46): dequantisation and both GEMMs are the
    bit-identical device paths; the double sums differ from the reference's sequential
    order only by reassociation (rtol 1e-12)."""
    from anyq_testutil import cfg

    codebook, bits = {"any4": (3, 4), "int4": (0, 4), "fp4": (1, 4), "nf4": (2, 4), "any3": (3, 3)}[fmt]
    w = orc.heavy_tailed(300, 520, 11, 0.02, 20.0)
    qt = orc.quantize(w, cfg(codebook=codebook, bits=bits, granularity=3, group_size=128,
                             max_iters=6, seed=2))
    mse, rel = aq.weight_error(w, qt)
    omse, orel = orc.weight_error(w, qt)
    assert np.isclose(mse, omse, rtol=1e-12, atol=0) and np.isclose(rel, orel, rtol=1e-12, atol=0)
    for m in (1, 7, 64):
        x = orc.gaussian(m, 520, 20 + m)
        assert np.isclose(aq.output_error(w, qt, x), orc.output_error(w, qt, x), rtol=1e-12, atol=0)


def test_eval_metrics_edges(aq, orc, cuda):
    from anyq_testutil import cfg

    w = np.zeros((8, 64), np.float32)  # zero reference energy: rel = sqrt(sq) (eval.cpp:27)
    qt = orc.quantize(orc.gaussian(8, 64, 1), cfg(codebook=3, granularity=3, group_size=64, max_iters=3))
    assert np.isclose(aq.weight_error(w, qt)[1], orc.weight_error(w, qt)[1], rtol=1e-12)
    with pytest.raises(aq.ShapeError):
        aq.weight_error(np.zeros((8, 63), np.float32), qt)
    with pytest.raises(aq.ShapeError):
        aq.output_error(np.zeros((8, 64), np.float32), qt, np.zeros((2, 63), np.float32))
