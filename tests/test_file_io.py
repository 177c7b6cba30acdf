"""ANYQ v1 files (pack.cpp:293-471): the writer is
byte-identical to the reference's write_file, the reader matches read_file's
arrays and error classes, on files either side wrote. Host-only (no device);
the device load (read_file straight into the prepacked layout) is a gpu test."""

import numpy as np
import pytest

from anyq_testutil import cfg


def _cases(orc):
    w = orc.gaussian(37, 300, 3)
    out = []
    for name, kw, stores, layout in [
        ("any4_g128", dict(codebook=3, granularity=3, group_size=128), (0, 0), (0, 1)),
        ("any4_row_bf16", dict(codebook=3, granularity=1), (1, 1), (0, 1)),
        ("any4_fp32", dict(codebook=3, granularity=3, group_size=64), (2, 2), (0, 1)),
        ("any4_ktiled", dict(codebook=3, granularity=3, group_size=128), (0, 0), (1, 4)),
        ("any3", dict(codebook=3, bits=3, granularity=3, group_size=128), (0, 0), (0, 1)),
        ("any2", dict(codebook=3, bits=2, granularity=1), (0, 0), (0, 1)),
        ("int4_sym_tensor", dict(codebook=0, granularity=0, symmetric=1), (0, 0), (0, 1)),
        ("int8_col", dict(codebook=0, bits=8, granularity=2), (0, 1), (0, 1)),
        ("nf4_block", dict(codebook=2, granularity=4, block_size=16), (0, 0), (0, 1)),
        ("fp4_g64", dict(codebook=1, granularity=3, group_size=64), (0, 0), (0, 1)),
    ]:
        qt = orc.quantize(w, cfg(max_iters=4, seed=5, **kw))
        qt.lut_store, qt.scale_store = stores
        if layout[0] == 1:
            qt = orc.to_ktiled(qt, layout[1])
        out.append((name, qt))
    return out


def _same(a, b):
    assert (a.rows, a.cols, a.layout, a.tile_k, a.lut_store, a.scale_store) == (
        b.rows, b.cols, b.layout, b.tile_k, b.lut_store, b.scale_store)
    assert np.array_equal(a.codes, b.codes)
    for x, y in ((a.alphas, b.alphas), (a.betas, b.betas), (a.luts, b.luts)):
        assert (x is None) == (y is None)
        if x is not None:
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def test_write_is_byte_identical_and_reads_match(aq, orc, ref, tmp_path):
    for name, qt in _cases(orc):
        mine, theirs = tmp_path / f"{name}.mine.anyq", tmp_path / f"{name}.ref.anyq"
        aq.write_file(qt, mine)
        ref.write_file(qt, theirs)
        assert mine.read_bytes() == theirs.read_bytes(), name
        got = aq.read_file(theirs)
        _same(got, ref.read_file(theirs, got))
        for f in ("bits", "codebook", "granularity", "group_size", "block_size", "symmetric",
                  "int_range_shifted", "init", "max_iters", "restarts", "weighting", "seed"):
            assert getattr(got.cfg, f) == getattr(qt.cfg, f), (name, f)
        assert got.cfg.rel_tol == qt.cfg.rel_tol
        # what a read returns writes back to the same bytes
        again = tmp_path / f"{name}.again.anyq"
        aq.write_file(got, again)
        assert again.read_bytes() == theirs.read_bytes(), name


def _err_kind(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        return getattr(e, "kind", type(e).__name__)
    return None


def test_reader_errors_match_reference(aq, orc, ref, tmp_path):
    """Corrupted files raise the reference's error class (pack.cpp:347-470)."""
    qts = dict(_cases(orc))
    good = tmp_path / "good.anyq"
    aq.write_file(qts["any4_g128"], good)
    data = bytearray(good.read_bytes())
    fp4 = tmp_path / "fp4.anyq"
    aq.write_file(qts["fp4_g64"], fp4)
    fp4_data = bytearray(fp4.read_bytes())

    def patched(b, off, val):
        c = bytearray(b)
        c[off:off + len(val)] = val
        return c

    ng = qts["any4_g128"].num_groups
    codes_len = len(qts["any4_g128"].codes)
    alpha0 = 120 + codes_len
    lut0 = 120 + codes_len + 4 * ng
    cases = {
        "magic": patched(data, 0, b"ANYX"),
        "version": patched(data, 4, (2).to_bytes(4, "little")),
        "truncated_header": data[:100],
        "truncated_body": data[:-3],
        "bad_enum": patched(data, 17, b"\x07"),
        "bad_config": patched(data, 16, b"\x05"),
        "lut_entries": patched(data, 64, (8).to_bytes(4, "little")),
        "trailing_byte": data + b"\x00",
        "negative_alpha": patched(data, alpha0, (0xBC00).to_bytes(2, "little")),
        "unsorted_lut": patched(data, lut0, (0x7BFF).to_bytes(2, "little")),
        "fp4_code_15": patched(fp4_data, 120, b"\xff"),
        # header group_size 64 -> 128: the declared group count (consistent with the
        # section lengths) is twice what the granularity gives, so a reader that
        # sizes its arrays from the granularity must not write the scales first
        "fp4_group_count": patched(fp4_data, 24, (128).to_bytes(4, "little")),
    }
    for name, blob in cases.items():
        p = tmp_path / f"{name}.anyq"
        p.write_bytes(bytes(blob))
        mine = _err_kind(lambda: aq.read_file(p))
        like = qts["fp4_g64"] if name.startswith("fp4") else qts["any4_g128"]
        theirs = _err_kind(lambda: ref.read_file(p, like))
        assert mine is not None and mine == theirs, (name, mine, theirs)
    assert _err_kind(lambda: aq.read_file(tmp_path / "missing.anyq")) == "IoError"


@pytest.mark.gpu
def test_device_load_matches_host_tensor(aq, orc, cuda, tmp_path):
    """DeviceTensor.load(path) == DeviceTensor(read_file(path)) on the GEMM."""
    import torch

    for name, qt in _cases(orc):
        if name not in ("any4_g128", "any4_row_bf16", "any4_ktiled", "any3", "any2"):
            continue
        if qt.lut_store != 0 or qt.scale_store != 0:
            continue  # the device GEMM stores LUT and scales as fp16
        p = tmp_path / f"{name}.anyq"
        aq.write_file(qt, p)
        a = aq.DeviceTensor.load(p)
        b = aq.DeviceTensor(aq.read_file(p))
        x = torch.randn(3, qt.cols, device="cuda").to(torch.bfloat16)
        ya = torch.empty(3, qt.rows, device="cuda", dtype=torch.float32)
        yb = torch.empty_like(ya)
        a.gemm(x, None, ya)
        b.gemm(x, None, yb)
        torch.cuda.synchronize()
        assert torch.equal(ya, yb), name
        a.close()
        b.close()
    with pytest.raises(aq.MagicError):
        bad = tmp_path / "bad.anyq"
        bad.write_bytes(b"NOPE" + bytes(200))
        aq.DeviceTensor.load(bad)
