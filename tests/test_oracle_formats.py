"""Pins for oracle/formats.py against the format definitions and independent
library conversions (torch dtypes), not against the oracle itself."""
import numpy as np
import pytest
import torch

from oracle import formats as F


def test_e2m1_table_matches_golden(golden):
    (row,) = [r for r in golden("e4m3_e2m1_tables.txt") if r[0] == "e2m1"]
    mags = [float(t) for t in row[1].split()]
    assert list(F.e2m1_decode(np.arange(8))) == mags
    assert list(F.e2m1_decode(np.arange(8, 16))) == [-m for m in mags]
    assert max(mags) == F.E2M1_QMAX == 6.0


def test_e4m3_table_matches_golden(golden):
    for r in golden("e4m3_e2m1_tables.txt"):
        if r[0] != "e4m3":
            continue
        code, val = r[1].split()
        assert F.e4m3_decode(int(code, 16)) == float(val)


def test_e4m3_decode_matches_torch_all_codes():
    codes = np.arange(0, 0x7F, dtype=np.uint8)
    ref = torch.from_numpy(codes).view(torch.float8_e4m3fn).float().numpy()
    np.testing.assert_array_equal(F.e4m3_decode(codes).astype(np.float32), ref)


def test_e4m3_encode_matches_torch_in_range():
    # torch's fp32 -> float8_e4m3fn cast is RNE (library routine); inside [0, 448]
    # satfinite changes nothing, so the two must agree bit for bit.
    rng = np.random.default_rng(0)
    v = np.concatenate([
        rng.uniform(0, 448, 200000),
        np.exp(rng.uniform(np.log(1e-4), np.log(448), 200000)),
        F.E4M3_VALUES,                                             # lattice points
        (F.E4M3_VALUES[:-1] + F.E4M3_VALUES[1:]) / 2,             # exact midpoints (ties)
        [2.0 ** -10, 2.0 ** -10 * 1.0000001, 2.0 ** -11, 0.0],
    ]).astype(np.float32)
    v = v[v <= 448]
    ref = torch.from_numpy(v).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    np.testing.assert_array_equal(F.e4m3_encode(v), ref)


def test_e4m3_satfinite():
    v = np.array([448.0, 449.0, 463.9, 464.0, 1e6, 3e38], dtype=np.float32)
    assert np.all(F.e4m3_encode(v) == 0x7E)


def test_e2m1_brute_force_nearest():
    """Brute force: the encoder picks a lattice point at minimal distance; on
    exact ties the code is even (Q5); beyond 6 it saturates (Q13)."""
    rng = np.random.default_rng(1)
    v = np.concatenate([rng.uniform(-8, 8, 100000),
                        np.arange(-7, 7.01, 0.25)]).astype(np.float32)
    codes = F.e2m1_encode(v)
    lattice = F.E2M1_MAG
    for x, c in zip(v[:5000].tolist() + v[100000:].tolist(), np.concatenate([codes[:5000], codes[100000:]])):
        a = min(abs(x), 6.0)
        d = np.abs(lattice - a)
        best = np.flatnonzero(d == d.min())
        assert (c & 7) in best
        if len(best) == 2:
            assert (c & 7) % 2 == 0
        assert bool(c & 8) == bool(np.signbit(np.float32(x)))
    # vectorised: distance optimality everywhere
    dec = np.abs(F.e2m1_decode(codes))
    a = np.minimum(np.abs(v.astype(np.float64)), 6.0)
    dist = np.abs(dec - a)
    best = np.min(np.abs(lattice[None, :] - a[:, None]), axis=1)
    np.testing.assert_array_equal(dist, best)


def test_e2m1_negative_zero():
    assert F.e2m1_encode(np.float32(-0.0)) == 0x8
    assert F.e2m1_encode(np.float32(-0.1)) == 0x8
    assert F.e2m1_encode(np.float32(0.1)) == 0x0


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
def test_16bit_rounding_matches_torch(dt):
    rng = np.random.default_rng(2)
    v = np.concatenate([rng.standard_normal(100000) * 10.0 ** rng.integers(-6, 4, 100000),
                        [0.0, -0.0, 1.0, 65504.0, 1e-8]]).astype(np.float32)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float16
    ref = torch.from_numpy(v).to(tdt).float().numpy()
    np.testing.assert_array_equal(F.round16(v, dt), ref)


def test_bf16_from_fp64_no_double_rounding():
    """fp64 -> bf16 must round once.  A value just above a bf16 midpoint but
    whose fp32 rounding lands exactly on the midpoint exposes double rounding."""
    mid = 1.0 + 2.0 ** -8            # midpoint between 1 and 1 + 2^-7
    v = mid + 2.0 ** -40             # fp32(v) == mid -> double rounding would go to 1.0
    assert np.float32(v) == np.float32(mid)
    assert F.bf16_round(np.float64(v)) == np.float32(1.0 + 2.0 ** -7)
    assert F.bf16_round(np.float64(mid)) == np.float32(1.0)     # tie -> even
    # brute force against the two bf16 neighbours on random fp64 values
    rng = np.random.default_rng(3)
    x = rng.standard_normal(20000) * 10.0 ** rng.integers(-3, 3, 20000)
    r = F.bf16_round(x).astype(np.float64)
    bits = F.bf16_bits(x).astype(np.int64)
    up = F.bf16_from_bits((bits + 1).astype(np.uint16)).astype(np.float64)
    dn = F.bf16_from_bits((bits - 1).astype(np.uint16)).astype(np.float64)
    assert np.all(np.abs(r - x) <= np.abs(up - x))
    assert np.all(np.abs(r - x) <= np.abs(dn - x))


def test_pack_low_nibble_is_even_index():
    """low nibble = even flat index."""
    codes = np.array([[1, 2, 3, 4, 15, 0]], dtype=np.uint8)
    p = F.pack_nibbles(codes)
    assert p.tolist() == [[0x21, 0x43, 0x0F]]
    np.testing.assert_array_equal(F.unpack_nibbles(p), codes)
    rng = np.random.default_rng(4)
    c = rng.integers(0, 16, (7, 64)).astype(np.uint8)
    np.testing.assert_array_equal(F.unpack_nibbles(F.pack_nibbles(c)), c)
    q = np.arange(-8, 8)
    np.testing.assert_array_equal(F.nibble_to_int4(F.int4_to_nibble(q)), q)


def test_sf_layout_is_bijection_with_zero_padding():
    rows, k = 200, 192
    rng = np.random.default_rng(5)
    sf = rng.integers(1, 255, (rows, k // 16)).astype(np.uint8)
    buf = F.sf_to_layout(sf, k)
    assert buf.size == 256 * 12
    np.testing.assert_array_equal(F.sf_from_layout(buf, rows, k), sf)
    # every byte is written at most once; padding rows are zero (Q22)
    r, c = np.meshgrid(np.arange(rows), np.arange(k // 16), indexing="ij")
    offs = F.sf_offset(r, c, k).ravel()
    assert len(np.unique(offs)) == offs.size
    mask = np.ones(buf.size, bool)
    mask[offs] = False
    assert np.all(buf[mask] == 0)
    # the 4 scale factors of one 64-wide K block of one row are contiguous bytes
    assert list(F.sf_offset(37, np.arange(4, 8), k) - F.sf_offset(37, 4, k)) == [0, 1, 2, 3]
