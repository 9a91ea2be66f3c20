"""Oracle pins for the iterative low-rank refinement (reading Q3).

What fixes the refinement independently of its own code:
* a planted fixed point: W_hat = D + L with D on the residual quantizer's lattice and L of exact
  rank r -- re-decomposing W_hat - Q(R) with Q(R) = D must return L1 L2 = L and R = D, and
  re-quantizing R must give D back (catches a wrong target W vs W_hat, a sign, a transpose);
* Eckart-Young on every step: the re-decomposed split is the best rank-r approximation of
  W_hat - Q(R_{t-1}), so its error is sqrt(sum_{i>r} sigma_i^2) of that matrix and never exceeds
  the previous iterate's weight-space error ||W_hat - L1 L2 - Q(R)||_F;
* the quantizer round trip: Q(dequantize(Q(R))) == Q(R) for each format;
* degenerate cases: iters = 0 is the plain split, rank 0 leaves every iterate identical;
* the selection rule of P:158 ("picking the result with the smallest error").
"""
import numpy as np
import pytest

import synth
from oracle import formats as F
from oracle import quant as Q
from oracle import svdquant as S


def _cal(K=128, N=96, M=64, seed=0):
    x = F.bf16_round(synth.gen_x(M, K, synth.rng(73, seed, 0)))
    w = synth.gen_w(K, N, synth.rng(73, seed, 1))
    return x, w


def _int4_lattice(K, N, rng):
    """D [K, N] exactly on the INT4 residual lattice: per (n, 64-group) a bf16 scale s and codes in
    [-7, 7] with a +-7 in every group, so quantize_int4(D^T) reproduces (codes, s) exactly."""
    G = K // 64
    codes = rng.integers(-7, 8, size=(N, K))
    codes[:, ::64] = 7 * rng.choice([-1, 1], size=(N, G))
    s = F.bf16_round(rng.uniform(0.01, 0.05, size=(N, G)))
    return (codes.reshape(N, G, 64) * s[:, :, None]).reshape(N, K).T.copy(), codes


def test_planted_fixed_point_int4():
    """Q(R_{t-1}) = D for W_hat = D + L: the step returns exactly (L, D) -- in the smoothed space."""
    rng = np.random.default_rng(5)
    K, N, r = 128, 64, 4
    D, codes = _int4_lattice(K, N, rng)
    L = rng.standard_normal((K, r)) @ rng.standard_normal((r, N))
    lam = rng.uniform(0.5, 2.0, size=K).astype(np.float32)
    w = (D + L) / lam.astype(np.float64)[:, None]          # so that W_hat = diag(lambda) W = D + L
    w_hat = S.smooth_weight(w, lam)
    d = S.redecompose(w_hat, D, r)
    np.testing.assert_allclose(d.L1 @ d.L2, L, rtol=0, atol=1e-9 * np.abs(L).max())
    np.testing.assert_allclose(d.R, D, rtol=0, atol=1e-9 * np.abs(D).max())
    ops = S.prepare_operands(w, lam, r, "int4", decomp=d)
    np.testing.assert_array_equal(ops.w_codes, codes)
    np.testing.assert_array_equal(S.dequantize_residual(ops), D)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
def test_dequantize_round_trip(fmt):
    """Q(deq(Q(R))) == Q(R): the dequantized residual sits on the lattice the quantizer maps to itself
    (pins the scale indexing and the [N, K] -> [K, N] transpose of dequantize_residual)."""
    x, w = _cal(seed=2)
    lam = S.compute_smoothing(x, w, 0.5)
    ops = S.prepare_operands(w, lam, 8, fmt)
    deq = S.dequantize_residual(ops)
    assert deq.shape == (ops.K, ops.N)
    codes, scales, gs = S.quantize_residual(deq.astype(np.float32), fmt, ops.scale_dtype if fmt == "int4" else "bf16")
    np.testing.assert_array_equal(codes, ops.w_codes)
    np.testing.assert_array_equal(scales, ops.w_scales)
    assert gs == ops.gs_w
    # and it is Q(R) within the quantizer's error: |R - deq| <= half a step of each group
    d = S.decompose(w, lam, 8)
    err = np.abs(d.R.astype(np.float32).astype(np.float64) - deq).T        # [N, K]
    if fmt == "int4":
        step = np.repeat(F.from_bits16(ops.w_scales, "bf16").astype(np.float64), 64, axis=1)
        assert np.all(err <= 0.5 * step * (1 + 1e-6))
    elif fmt == "w8a8":
        assert np.all(err <= 0.5 * ops.w_scales.astype(np.float64)[:, None] * (1 + 1e-6))


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
def test_every_step_is_the_optimal_redecomposition(fmt):
    """Eckart-Young on W_hat - Q(R_{t-1}): residual norm = sqrt(sum_{i>r} sigma_i^2), which is <= the
    previous iterate's weight-space error ||W_hat - L1 L2 - Q(R)||_F; L1 L2 + R = W_hat at every iterate."""
    x, w = _cal(seed=3)
    lam = S.compute_smoothing(x, w, 0.5)
    r = 8
    best, ops, errs, decs = S.refine_lowrank(x, w, lam, r, fmt, 3)
    prev_ops = S.prepare_operands(w, lam, r, fmt, decomp=decs[0])
    for t in range(1, len(decs)):
        d = decs[t]
        np.testing.assert_allclose(d.L1 @ d.L2 + d.R, d.w_hat, rtol=0, atol=1e-9 * np.abs(d.w_hat).max())
        T = d.w_hat - S.dequantize_residual(prev_ops)
        tail = np.sqrt(np.sum(np.linalg.svd(T, compute_uv=False)[r:] ** 2))
        np.testing.assert_allclose(np.linalg.norm(T - d.L1 @ d.L2), tail, rtol=1e-8)
        prev_err = np.linalg.norm(decs[t - 1].w_hat - decs[t - 1].L1 @ decs[t - 1].L2 - S.dequantize_residual(prev_ops))
        assert tail <= prev_err * (1 + 1e-12)
        prev_ops = S.prepare_operands(w, lam, r, fmt, decomp=d)


def test_iters_zero_is_the_plain_split():
    x, w = _cal(seed=4)
    lam = S.compute_smoothing(x, w, 0.5)
    best, ops, errs, _ = S.refine_lowrank(x, w, lam, 8, "nvfp4", 0)
    ref = S.prepare_operands(w, lam, 8, "nvfp4")
    assert best == 0 and len(errs) == 1
    np.testing.assert_array_equal(ops.w_codes, ref.w_codes)
    np.testing.assert_array_equal(ops.L2s_bits, ref.L2s_bits)


def test_rank_zero_iterates_are_identical():
    """With r = 0 there is no branch to update: R_t = W_hat for all t, best = 0 (ties -> earliest)."""
    x, w = _cal(seed=5)
    lam = S.compute_smoothing(x, w, 0.5)
    best, ops, errs, _ = S.refine_lowrank(x, w, lam, 0, "int4", 3)
    assert best == 0 and len(set(errs)) == 1


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_selection_and_improvement(fmt):
    """The returned iterate has the smallest objective and, on the synthetic workload, the
    refinement lowers the 4-bit layer's calibration error below the plain split in every seed."""
    for seed in range(3):
        x, w = _cal(seed=10 + seed)
        lam = S.compute_smoothing(x, w, 0.5)
        best, ops, errs, _ = S.refine_lowrank(x, w, lam, 8, fmt, 3)
        assert errs[best] == min(errs) and best == errs.index(min(errs))
        assert errs[best] < errs[0]
        assert S.calibration_error(x, w, ops) == errs[best]


def test_refine_with_gptq_iterate0_is_gptq_split():
    """gptq=True: iterate 0 is the plain split with the GPTQ residual, and the selection holds."""
    x, w = _cal(seed=20)
    lam = S.compute_smoothing(x, w, 0.5)
    best, ops, errs, decs = S.refine_lowrank(x, w, lam, 8, "int4", 2, gptq=True)
    ref = S.prepare_operands(w, lam, 8, "int4", gptq_x=x)
    assert errs[0] == S.calibration_error(x, w, ref)
    assert errs[best] == min(errs)
