"""The reference's OWN hot-path unit tests (proj/tests/test_{core,scaling,
codebooks,pack,learner,qgemm}.cpp, 85 doctest cases compiled unmodified by
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
    assert "85 passed | 0 failed" in r.stdout


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
    assert "85 passed | 0 failed" in r.stdout


def _defined(path, demangle=True):
    """Defined (text, weak, data) symbol names of an object or shared library."""
    args = ["nm", "--defined-only"] + (["-C"] if demangle else []) + ([] if path.endswith(".o") else ["-D"])
    out = subprocess.run(args + [path], capture_output=True, text=True, check=True).stdout
    syms = set()
    for line in out.splitlines():
        parts = line.split(" ", 2)
        if len(parts) == 3 and parts[1] in "TWVBDR":
            syms.add(parts[2])
    return syms


def test_drop_in_links_no_reference_code():
    """libanyq_host.so and the B200 test binary are anyq_host.o + libanyq_b200.so
    only: the Makefile has no rule that pulls (or weakens) reference objects
    into them, every anyq:: function the .so defines is defined by anyq_host.o,
    and it exports none of the oracle shim's ref_* entry points."""
    mk = open(os.path.join(HERE, "reftests", "Makefile")).read()
    assert "objcopy" not in mk and "weak/" not in mk
    b200_rule = mk[mk.index("$(B)/anyq_tests_b200:"):mk.index("$(LIBDIR)/libanyq_host.so:")]
    host_rule = mk[mk.index("$(LIBDIR)/libanyq_host.so:"):mk.index("clean:")]
    for rule in (b200_rule, host_rule):
        assert "oracle/_ref" not in rule and "REF_LINK_OBJS" not in rule
    so = os.path.join(HERE, "..", "paper_2507_04610_b200", "_lib", "libanyq_host.so")
    obj = os.path.join(BUILD, "anyq_host.o")
    if not (os.path.exists(so) and os.path.exists(obj)):
        pytest.skip("drop-in not built (make -C tests/reftests)")
    lib_syms = {s for s in _defined(so) if s.startswith("anyq::")}
    obj_syms = {s for s in _defined(obj) if s.startswith("anyq::")}
    assert lib_syms and lib_syms <= obj_syms, sorted(lib_syms - obj_syms)[:10]
    assert not any(s.startswith("ref_") for s in _defined(so, demangle=False))
    needed = subprocess.run(["readelf", "-d", so], capture_output=True, text=True).stdout
    assert "anyq_ref" not in needed
