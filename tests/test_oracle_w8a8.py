"""Oracle pins for the 8-bit setting of App. D: "per-token dynamic activation
quantization and per-channel weight quantization with a low-rank branch of rank 16" --
Eq. (1) with q_max = 127, one fp32 scale per token / output channel (reading W1)."""
import itertools

import numpy as np
import pytest

import synth
from oracle import formats as F
from oracle import quant as Q
from oracle import svdquant as S


def test_int8_worked_example_ties_to_even():
    """Hand-derived: amax 254 -> s = 2 exactly, qinv = 0.5; x / s = [127, 63.5, -31.5, 0.75,
    -0.25] -> round half to even (reading Q6 applied to 8 bits) -> [127, 64, -32, 1, 0]."""
    v = np.array([[254.0, 127.0, -63.0, 1.5, -0.5]], np.float32)
    q, s = Q.quantize_int8_rows(v)
    assert s[0] == np.float32(2.0)
    np.testing.assert_array_equal(q[0], [127, 64, -32, 1, 0])


def test_int8_zero_row_and_saturation():
    q, s = Q.quantize_int8_rows(np.zeros((1, 8), np.float32))
    assert s[0] == 0 and np.all(q == 0)
    # the amax element maps to +-127 exactly; nothing exceeds the range
    rng = np.random.default_rng(0)
    v = (rng.standard_normal((64, 96)) * 10 ** rng.uniform(-3, 3, (64, 1))).astype(np.float32)
    q, s = Q.quantize_int8_rows(v)
    assert q.min() >= -127 and q.max() <= 127
    assert np.all(np.abs(q).max(axis=1) == 127)
    # per-element error bound |v - q s| <= s / 2 (+ fp32 slack)
    err = np.abs(v.astype(np.float64) - Q.dequantize_int8_rows(q, s))
    assert np.all(err <= s[:, None].astype(np.float64) * (0.5 + 1e-5))


def test_int8_quant_dequant_identity_on_lattice():
    rng = np.random.default_rng(1)
    s = (2.0 ** rng.integers(-8, 8, 32)).astype(np.float32)
    c = rng.integers(-127, 128, (32, 64))
    c[:, 0] = 127                                  # amax = 127 s -> the scale is recovered exactly
    v = (c * s[:, None]).astype(np.float32)
    q, s2 = Q.quantize_int8_rows(v)
    np.testing.assert_array_equal(s2, s)
    np.testing.assert_array_equal(q, c)
    np.testing.assert_array_equal(Q.dequantize_int8_rows(q, s2), v.astype(np.float64))


def test_int8_power_of_two_equivariance():
    rng = np.random.default_rng(2)
    v = rng.standard_normal((16, 128)).astype(np.float32)
    q1, s1 = Q.quantize_int8_rows(v)
    q2, s2 = Q.quantize_int8_rows((v * np.float32(8.0)).astype(np.float32))
    np.testing.assert_array_equal(q1, q2)
    np.testing.assert_array_equal(s2, (s1 * np.float32(8.0)).astype(np.float32))


def _w8a8_layer(M=6, K=96, N=20, r=16, seed=3):
    x = F.bf16_round(synth.gen_x(M, K, synth.rng(60, seed, 0)))
    w = synth.gen_w(K, N, synth.rng(60, seed, 1))
    lam = S.compute_smoothing(synth.gen_x(64, K, synth.rng(60, seed, 2)), w, 0.5)
    bias = F.bf16_round(synth.gen_bias(N, synth.rng(60, seed, 3)))
    ops = S.prepare_operands(w, lam, r, "w8a8", bias=bias)
    return x, w, ops


def test_w8a8_forward_matches_brute_force():
    """Triple loop: Y = sum_k qa qb * sx[m] * sw[n] + xl1 L2s^T + bias (alpha = 1)."""
    x, w, ops = _w8a8_layer()
    y_ref, y64, qa = S.forward(x, ops)
    M, K = qa.codes.shape
    xl1 = F.bf16_from_bits(qa.xl1_bits).astype(np.float64)
    bf = np.zeros((M, ops.N))
    for m, n in itertools.product(range(M), range(ops.N)):
        acc = sum(int(qa.codes[m, k]) * int(ops.w_codes[n, k]) for k in range(K))
        y = acc * float(qa.scales[m]) * float(ops.w_scales[n])
        y += sum(xl1[m, t] * float(ops.L2s[n, t]) for t in range(ops.rank))
        bf[m, n] = y + float(ops.bias[n])
    np.testing.assert_allclose(y64, bf, rtol=1e-12, atol=1e-12 * np.abs(bf).max())
    # the integer accumulator of the main product is exact
    acc = qa.codes.astype(np.int64) @ ops.w_codes.astype(np.int64).T
    main = S.main_product(qa.codes, qa.scales, ops)
    np.testing.assert_array_equal(np.rint(main / (qa.scales[:, None] * ops.w_scales[None, :].astype(np.float64))),
                                  acc.astype(np.float64))


def test_w8a8_eq5_error_equality():
    """Eq. (5): ||X_hat W_hat - (X_hat L1 L2 + Q(X_hat) Q(R))|| = E(X_hat, R)."""
    x, w, ops = _w8a8_layer(M=12, K=128, N=24, r=16, seed=4)
    lam_inv = ops.lam_inv32.astype(np.float64)
    xh = x.astype(np.float64) * lam_inv
    d = S.decompose(w, (1.0 / ops.lam_inv32).astype(np.float32), 16)
    qa_c, qa_s = Q.quantize_int8_rows(Q.smooth_activation(x, ops.lam_inv32))
    qx = Q.dequantize_int8_rows(qa_c, qa_s)
    qr = Q.dequantize_int8_rows(ops.w_codes, ops.w_scales).T          # [K, N]
    lhs = np.linalg.norm(xh @ d.w_hat - (xh @ d.L1 @ d.L2 + qx @ qr))
    rhs = np.linalg.norm(xh @ d.R - qx @ qr)
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, rhs)


def test_w8a8_more_accurate_than_int4():
    """The 8-bit setting is the higher-fidelity one (Table 1: W8A8 rows vs W4A4 rows)."""
    M, K, N = 64, 512, 128
    x = F.bf16_round(synth.gen_x(M, K, synth.rng(61, 0, 0)))
    w = synth.gen_w(K, N, synth.rng(61, 0, 1))
    lam = S.compute_smoothing(synth.gen_x(128, K, synth.rng(61, 0, 2)), w, 0.5)
    ref = x.astype(np.float64) @ w
    e = {}
    for fmt, r in (("w8a8", 16), ("int4", 32)):
        ops = S.prepare_operands(w, lam, r, fmt)
        e[fmt] = np.linalg.norm(S.forward(x, ops)[1] - ref) / np.linalg.norm(ref)
    assert e["w8a8"] < 0.25 * e["int4"], e
