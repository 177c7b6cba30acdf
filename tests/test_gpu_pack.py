"""Packing, k-tiling, narrowing and dequantisation on the GPU vs the oracle.

Mirrors proj/tests/test_pack.cpp (KATs at :53-67, round trips :69-88,
range errors :90-94, k-tiling :158-172, narrowing :140-156).
"""
import numpy as np
import pytest

from anyq_testutil import bits_equal, cfg

pytestmark = pytest.mark.gpu


def random_codes(orc, rows, cols, bits, seed):
    u = orc.rng_double(seed, 0, rows * cols)
    return np.floor(u * (1 << bits)).astype(np.uint8).reshape(rows, cols)


def test_nibble_packing_puts_first_code_low(aq):
    assert aq.pack_codes(np.array([[1, 2]], np.uint8), 4).tolist() == [0x21]


def test_two_bit_packing_little_end_first(aq):
    assert aq.pack_codes(np.array([[0, 1, 2, 3]], np.uint8), 2).tolist() == [0b11100100]


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("cols", [1, 5, 8, 31, 257])
def test_pack_round_trip_matches_oracle(aq, orc, bits, cols):
    codes = random_codes(orc, 5, cols, bits, 100 + bits + cols)
    packed = aq.pack_codes(codes, bits)
    assert bits_equal(packed, orc.pack_codes(codes, bits))
    assert packed.size == 5 * ((cols * bits + 7) // 8)
    assert np.array_equal(aq.unpack_codes(packed, 5, cols, bits), codes)


def test_three_bit_rows_are_byte_aligned(aq, orc):
    codes = random_codes(orc, 3, 7, 3, 7)
    packed = aq.pack_codes(codes, 3)
    assert packed.size == 9
    assert np.array_equal(aq.pack_codes(codes[1:2], 3), packed[3:6])


def test_out_of_range_codes_rejected(aq):
    with pytest.raises(aq.CodeRangeError):
        aq.pack_codes(np.array([[3, 16]], np.uint8), 4)
    with pytest.raises(aq.ConfigError):
        aq.pack_codes(np.array([[1]], np.uint8), 5)


def sample_tensor(aq, orc, seed, codebook=3, bits=4, rows=8, cols=48):
    w = orc.gaussian(rows, cols, seed)
    c = cfg(codebook=codebook, bits=bits, group_size=16, seed=seed)
    return orc.quantize(w, c), w


@pytest.mark.parametrize("tile_k", [1, 2, 8, 32])
def test_ktiling_is_invertible_and_matches_oracle(aq, orc, tile_k):
    for seed in (21, 22):
        qt, _ = sample_tensor(aq, orc, seed)
        tiled = aq.to_ktiled(qt, tile_k)
        assert bits_equal(tiled.codes, orc.to_ktiled(qt, tile_k).codes)
        back = aq.from_ktiled(tiled)
        assert bits_equal(back.codes, qt.codes)
        assert bits_equal(aq.dequantize(tiled), aq.dequantize(qt))


def test_tile_one_is_identity(aq, orc):
    qt, _ = sample_tensor(aq, orc, 13)
    assert bits_equal(aq.to_ktiled(qt, 1).codes, qt.codes)


@pytest.mark.parametrize("codebook,bits", [(3, 4), (3, 2), (3, 3), (0, 4), (1, 4), (2, 4), (0, 8)])
def test_narrowed_and_dequantize_bit_exact(aq, orc, codebook, bits):
    qt, _ = sample_tensor(aq, orc, 31 + codebook + bits, codebook, bits)
    a = aq.narrowed(qt)
    b = orc.narrowed(qt)
    assert a.same_as(b)
    assert bits_equal(aq.dequantize(qt), orc.dequantize(qt))
    assert bits_equal(aq.dequantize(a), orc.dequantize(b))


def test_narrowed_rejects_underflowing_scale(aq, orc):
    qt, _ = sample_tensor(aq, orc, 11)
    qt.alphas[0] = 1e-9
    with pytest.raises(aq.InvariantError):
        aq.narrowed(qt)


def test_dequantize_rejects_fp4_code_15(aq, orc):
    qt, _ = sample_tensor(aq, orc, 43, codebook=1)
    qt.codes[0] = 0xFF
    with pytest.raises(aq.CodeRangeError):
        aq.dequantize(qt)


@pytest.mark.parametrize("fmt", ["any4", "any3", "any2", "int4", "nf4", "fp4"])
@pytest.mark.parametrize("shape,gran,g", [((200, 384), 3, 128), ((33, 130), 1, 128), ((64, 1024), 3, 256),
                                          ((5, 17), 1, 128)])
def test_prepack_inverse_round_trip(aq, orc, cuda, fmt, shape, gran, g):
    """unpack(prepack^-1(prepack(codes))) == codes bit for bit:
    the device layout [RB][C][4 slabs][32 rows][16 B] exported back
    (anyq_dev_tensor_export) equals narrowed(qt) — codes, LUT and alpha/beta."""
    c = cfg(granularity=gran, group_size=g, seed=3)
    aq.apply_format(c, fmt)
    qt = orc.quantize(orc.gaussian(*shape, 11), c)
    dt = aq.DeviceTensor(qt)
    back = dt.export()
    dt.close()
    want = orc.narrowed(qt)
    assert np.array_equal(back.codes, want.codes)
    assert np.array_equal(aq.unpack_codes(back.codes, *shape, c.bits), aq.unpack_codes(qt.codes, *shape, c.bits))
    assert bits_equal(back.alphas, want.alphas) and bits_equal(back.betas, want.betas)
    if want.luts is not None:
        assert bits_equal(back.luts, want.luts)


def test_prepack_inverse_of_ktiled_tensor(aq, orc, cuda):
    """A k-tiled tensor prepacks in logical order; its export is row-major."""
    qt = orc.quantize(orc.gaussian(64, 512, 12), cfg(codebook=3, max_iters=3, seed=4))
    kt = orc.to_ktiled(qt, 32)
    dt = aq.DeviceTensor(kt)
    back = dt.export()
    dt.close()
    assert np.array_equal(back.codes, orc.narrowed(qt).codes)
