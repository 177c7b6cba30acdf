"""The reference's OWN hot-path unit tests (proj/tests/test_{core,scaling,
codebooks,pack,learner,qgemm}.cpp, 76 doctest cases compiled unmodified by
tests/reftests/Makefile) run against:

* the unmodified reference build (CPU) — validates the doctest subset harness;
* the B200 drop-in (paper_2507_04610_b200/host/anyq_host.cpp over the C-ABI):
  on a B200 every case must pass; on a host without a GPU the hot-path cases
  must fail with the library's "no usable CUDA device" error (the drop-in never
  falls back to the CPU).

The binaries are built where /root/reference exists and travel prebuilt.
"""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "reftests", "_build")
REF_BIN = os.path.join(BUILD, "anyq_tests_ref")
B200_BIN = os.path.join(BUILD, "anyq_tests_b200")


def _run(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C tests/reftests)")
    return subprocess.run([path], capture_output=True, text=True, timeout=900)


def test_reference_suite_on_reference_build():
    r = _run(REF_BIN)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "76 passed | 0 failed" in r.stdout


def test_drop_in_has_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    r = _run(B200_BIN)
    assert r.returncode != 0
    assert "no usable CUDA device" in r.stderr


@pytest.mark.gpu
def test_reference_suite_on_b200(cuda):
    r = _run(B200_BIN)
    assert r.returncode == 0, (r.stdout[-500:], r.stderr[-4000:])
    assert "76 passed | 0 failed" in r.stdout
