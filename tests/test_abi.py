"""CPU: the C-ABI boundary (include/anyq_b200.h) and the host-side mirror.

* the CUDA library loads without a GPU and exports every function the header
  declares (no compute calls here);
* on a host without a device every compute entry fails loudly with
  ANYQ_ERR_CUDA (there is no CPU fallback);
* host logic that needs no device: defaults (core.hpp:98-121), sizes
  (pack.hpp:45, scaling.hpp:36-45), format names (quantize.cpp:34-64), bits
  accounting (codebooks.cpp:99-121), error classes (core.hpp:27-74).
"""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "anyq_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(anyq_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for must in ("anyq_quantize_any", "anyq_quantize_fixed", "anyq_pack_codes", "anyq_unpack_codes",
                 "anyq_dequantize", "anyq_gemm_fused", "anyq_gemm_dense", "anyq_narrow_inplace",
                 "anyq_ktile_codes", "anyq_dev_gemm_bf16", "anyq_dev_quantize_any"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2507_04610_b200 import anyq

    assert os.path.exists(anyq.LIB_PATH), "build the CUDA library first (__graft_entry__.build())"
    lib = ctypes.CDLL(anyq.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(anyq.EXPORTED_SYMBOLS) <= set(declared_functions())


def test_defaults_match_reference_core_hpp():
    from paper_2507_04610_b200 import _abi, anyq

    L = anyq.lib()
    c = _abi.Config()
    L.anyq_config_default(c)
    ref = _abi.default_config()
    assert bytes(c) == bytes(ref)
    assert (c.bits, c.codebook, c.granularity, c.group_size, c.max_iters, c.restarts) == \
        (4, _abi.CB_INT, _abi.G_GROUP, 128, 100, 1)
    assert abs(c.rel_tol - 1e-6) < 1e-12


def test_sizes():
    from paper_2507_04610_b200 import _abi, anyq

    L = anyq.lib()
    for cols, bits in ((4096, 4), (33, 3), (7, 2), (5, 8), (1, 3)):
        assert L.anyq_packed_bytes_per_row(cols, bits) == (cols * bits + 7) // 8
    c = _abi.default_config(codebook=_abi.CB_ANY)
    assert L.anyq_num_groups(c, 4096, 4096) == 4096 * 32
    c.group_size = 100
    assert L.anyq_num_groups(c, 10, 250) == 30  # ceil(250 / 100) groups per row
    assert L.anyq_lut_entries(c) == 16


def test_formats_and_bits():
    from paper_2507_04610_b200 import _abi, anyq

    for name in ("int2", "int3", "int4", "int8", "fp4", "nf4", "any2", "any3", "any4", "any8"):
        c = anyq.apply_format(_abi.default_config(), name)
        assert anyq.format_name(c) == name
    with pytest.raises(anyq.ConfigError):
        anyq.apply_format(_abi.default_config(), "any5")
    c = anyq.apply_format(_abi.default_config(), "any4")
    assert anyq.storage_bits_per_entry(c, 4096, 4096) == 4.3125
    assert anyq.storage_bits_per_entry(anyq.apply_format(c, "int4"), 4096, 4096) == 4.25


def test_error_classes_mirror_core_hpp():
    from paper_2507_04610_b200 import anyq

    assert issubclass(anyq.MagicError, anyq.IoError)
    assert issubclass(anyq.TruncatedError, anyq.IoError)
    assert issubclass(anyq.ShapeError, anyq.Error)
    assert anyq.ConfigError.status == 2 and anyq.CudaError.status == 12


def test_no_cpu_fallback_without_device():
    """Every compute entry reports ANYQ_ERR_CUDA when no GPU is visible."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2507_04610_b200 import _abi, anyq

    w = np.ones((4, 8), np.float32)
    with pytest.raises(anyq.CudaError):
        anyq.quantize_any(w, _abi.default_config(codebook=_abi.CB_ANY, group_size=4))
    with pytest.raises(anyq.CudaError):
        anyq.pack_codes(np.zeros((2, 4), np.uint8), 4)
