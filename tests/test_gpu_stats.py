"""E|x_j| activation statistics on the GPU (collect_stats, calibration.cpp:62-67;
SURVEY.md §8(f) row 4) against the oracle restatement: bit-exact."""
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
