"""Pins for oracle/quant.py: worked examples (golden), Eq. (1) invariants,
and Prop. 4.2 as a Monte-Carlo theorem check."""
import numpy as np
import pytest

from oracle import diagnostics as D
from oracle import formats as F
from oracle import quant as Q


def test_nvfp4_golden(golden):
    for name, gs, vals, sf, codes in golden("nvfp4_worked_examples.txt"):
        v = np.array([float(t) for t in vals.split()], dtype=np.float32)[None]
        c, s = Q.quantize_nvfp4(v, np.float32(gs))
        assert s[0, 0] == int(sf, 16), name
        assert c[0].tolist() == [int(t, 16) for t in codes.split()], name


def test_nvfp4_s224_dequant_is_09375():
    v = np.zeros((1, 16), np.float32)
    v[0, 0] = 0.9
    c, s = Q.quantize_nvfp4(v, 1.0)
    assert Q.dequantize_nvfp4(c, s, 1.0)[0, 0] == 0.9375   # SURVEY §8(c.3), corrects S:224


def test_int4_golden(golden):
    for name, dt, vals, scale, codes in golden("int4_worked_examples.txt"):
        lead = [float(t) for t in vals.split()]
        v = np.zeros((1, 64), np.float32)
        v[0, :len(lead)] = lead
        q, s = Q.quantize_int4(v, dt)
        assert F.from_bits16(s, dt)[0, 0] == float(scale), name
        assert q[0, :len(lead)].tolist() == [int(t) for t in codes.split()], name
        assert np.all(q[0, len(lead):] == 0)


def _nvfp4_lattice_tensor(rng, rows, k, gs):
    """Inputs exactly representable: v = e2m1 * sf * gs with group amax = 6 sf."""
    codes = rng.integers(0, 16, (rows, k)).astype(np.uint8)
    codes[:, ::16] = rng.choice([7, 15], size=(rows, k // 16))          # amax hits 6
    sf = rng.integers(0x20, 0x60, (rows, k // 16)).astype(np.uint8)     # normal scales
    v = (F.e2m1_decode(codes).reshape(rows, k // 16, 16)
         * F.e4m3_decode(sf)[..., None] * gs).reshape(rows, k).astype(np.float32)
    return v, codes, sf


@pytest.mark.parametrize("gs", [1.0, 0.25, 2.0 ** -7])
def test_nvfp4_quant_dequant_identity_on_lattice(gs):
    rng = np.random.default_rng(10)
    v, codes, sf = _nvfp4_lattice_tensor(rng, 64, 256, gs)
    c2, s2 = Q.quantize_nvfp4(v, gs)
    np.testing.assert_array_equal(s2, sf)
    deq = Q.dequantize_nvfp4(c2, s2, gs)
    np.testing.assert_array_equal(deq, v.astype(np.float64))
    # codes equal except that +0 / -0 may differ only where the value is 0
    same = (c2 == codes) | ((c2 & 7) == 0) & ((codes & 7) == 0)
    assert np.all(same)


def test_int4_quant_dequant_identity_on_lattice():
    rng = np.random.default_rng(11)
    for dt in ("bf16", "fp16"):
        q = rng.integers(-7, 8, (32, 256))
        q[:, ::64] = rng.choice([-7, 7], size=(32, 4))
        s = F.round16(2.0 ** rng.uniform(-8, 4, (32, 4)), dt)
        v = (q.reshape(32, 4, 64) * s[..., None]).reshape(32, 256).astype(np.float32)
        q2, s2 = Q.quantize_int4(v, dt)
        np.testing.assert_array_equal(q2, q)
        np.testing.assert_array_equal(F.from_bits16(s2, dt), s)
        np.testing.assert_array_equal(Q.dequantize_int4(q2, s2, dt), v.astype(np.float64))


def test_power_of_two_equivariance():
    """Eq. (1): scaling X by 2^j (within normal range) leaves codes unchanged
    and scales every scale by exactly 2^j."""
    rng = np.random.default_rng(12)
    x = (rng.standard_normal((16, 128)) * 3).astype(np.float32)
    c0, s0 = Q.quantize_nvfp4(x, 1.0)
    for j in (-3, 2):
        c1, s1 = Q.quantize_nvfp4((x * 2.0 ** j).astype(np.float32), 1.0)
        np.testing.assert_array_equal(c1, c0)
        np.testing.assert_array_equal(F.e4m3_decode(s1), F.e4m3_decode(s0) * 2.0 ** j)
        q0, t0 = Q.quantize_int4(x, "bf16")
        q1, t1 = Q.quantize_int4((x * 2.0 ** j).astype(np.float32), "bf16")
        np.testing.assert_array_equal(q1, q0)
        np.testing.assert_array_equal(F.bf16_from_bits(t1), F.bf16_from_bits(t0) * np.float32(2.0 ** j))


def test_codes_in_range_and_error_bound():
    """Every code is a valid lattice point; per element |x - Q(x)| is at most
    half the local lattice spacing times the stored scale (rounding to nearest)."""
    rng = np.random.default_rng(13)
    x = (rng.standard_normal((64, 512)) * np.exp(rng.standard_normal((64, 1)))).astype(np.float32)
    q, s = Q.quantize_int4(x, "fp16")
    assert q.min() >= -7 and q.max() <= 7
    deq = Q.dequantize_int4(q, s, "fp16")
    sd = np.repeat(F.fp16_from_bits(s).astype(np.float64), 64, axis=1)
    inside = np.abs(x) <= 7 * sd          # not clipped by scale rounding
    assert np.all(np.abs(x - deq)[inside] <= 0.5 * sd[inside] * (1 + 1e-6))
    c, sf = Q.quantize_nvfp4(x, 1.0)
    deq = Q.dequantize_nvfp4(c, sf, 1.0)
    sfd = np.repeat(F.e4m3_decode(sf), 16, axis=1)
    # E2M1 spacing is at most 2 (between 4 and 6) -> error <= 1 * sf unless saturated
    sat = np.abs(x) > 6 * sfd
    assert np.all(np.abs(x - deq)[~sat] <= 1.0 * sfd[~sat] * (1 + 1e-6))


def test_nonfinite_rejected():
    x = np.zeros((1, 64), np.float32)
    x[0, 3] = np.nan
    with pytest.raises(ValueError):
        Q.quantize_nvfp4(x, 1.0)
    with pytest.raises(ValueError):
        Q.quantize_int4(x, "bf16")


@pytest.mark.parametrize("size", [256, 1024, 4096])
@pytest.mark.parametrize("quantizer", ["int4_g64", "int8_per_tensor"])
def test_prop42_monte_carlo(size, quantizer):
    """Prop. 4.2 through the ORACLE's own quantizers:
    E||R - Q(R)||_F <= c sqrt(size(R)) / q_max * E||R||_F with the Gaussian
    c = sqrt(log(size) pi / size), R ~ N(0, 1) of `size` elements.
      * int4_g64: oracle.quant.quantize_int4 (Eq. 1 per group of 64 with 16-bit scales, q_max 7);
        every element's error is at most half its group's step, and a group step never exceeds
        the per-tensor one (up to the 16-bit scale rounding), so the per-tensor bound applies.
      * int8_per_tensor: oracle.quant.quantize_int8_rows on the tensor as ONE row -- exactly the
        proposition's per-tensor Eq. (1) quantizer, q_max 127, fp32 scale."""
    rng = np.random.default_rng(size)
    trials = 200
    lhs, fr = [], []
    for _ in range(trials):
        r = rng.standard_normal((1, size)).astype(np.float32)
        if quantizer == "int4_g64":
            q, sb = Q.quantize_int4(r, "bf16")
            deq, qmax = Q.dequantize_int4(q, sb, "bf16"), 7.0
        else:
            q, sc = Q.quantize_int8_rows(r)
            deq, qmax = Q.dequantize_int8_rows(q, sc), 127.0
        # the proof's per-element step: |r - Q(r)| <= s / 2 (round to nearest; the max element
        # is clamped at q_max but its overshoot is only the scale's storage rounding)
        step = (F.from_bits16(sb, "bf16").astype(np.float64).repeat(64, axis=1) if quantizer == "int4_g64"
                else np.asarray(sc, np.float64)[:, None])
        assert np.all(np.abs(r.astype(np.float64) - deq) <= 0.5 * step * (1 + 1e-5))
        lhs.append(np.linalg.norm(r.astype(np.float64) - deq))
        fr.append(np.linalg.norm(r.astype(np.float64)))
    rhs = D.prop42_rhs(size, qmax, np.mean(fr))
    se = np.std(lhs) / np.sqrt(trials)
    assert np.mean(lhs) <= rhs + 3 * se


def test_prop42_regularity_condition_gaussian():
    """The proposition's regularity condition with its Gaussian constant:
    E max|R| <= c E||R||_F, c = sqrt(log(size) pi / size)."""
    rng = np.random.default_rng(0)
    for size in (256, 1024, 4096):
        r = rng.standard_normal((400, size))
        assert np.mean(np.abs(r).max(axis=1)) <= D.prop42_gaussian_c(size) * np.mean(np.linalg.norm(r, axis=1))
