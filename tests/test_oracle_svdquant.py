"""Pins for oracle/svdquant.py + oracle/linalg.py against closed forms,
algebraic identities, the paper's propositions and brute force."""
import itertools

import numpy as np
import pytest
import torch

import synth
from oracle import diagnostics as D
from oracle import formats as F
from oracle import linalg as LA
from oracle import quant as Q
from oracle import svdquant as S


# ---------------------------------------------------------------- smoothing
def test_smoothing_examples():
    """col absmax(X)=4, row absmax(W)=1, alpha=.5 -> 2; alpha=1 -> max|X|;
    alpha=0, row absmax(W)=5 -> 1/5 (P:467 formula)."""
    x = np.array([[4.0, -2.0], [1.0, 3.0]])
    w = np.array([[1.0, -0.5], [5.0, 2.0]])
    lam = S.compute_smoothing(x, w, 0.5)
    assert lam[0] == np.float32(2.0)
    assert np.allclose(S.compute_smoothing(x, w, 1.0), [4.0, 3.0])
    assert np.allclose(S.compute_smoothing(x, w, 0.0), [1.0, 1 / 5.0])


def test_smoothing_identity():
    """X W = X_hat W_hat (reading Q1) to 1e-12 relative."""
    rng = synth.rng(9, 0, 0)
    x = synth.gen_x(64, 128, rng).astype(np.float64)
    w = synth.gen_w(128, 96, synth.rng(9, 0, 1)).astype(np.float64)
    lam = S.compute_smoothing(synth.gen_x(64, 128, synth.rng(9, 0, 2)), w, 0.5)
    xh = x / lam.astype(np.float64)[None, :]
    wh = S.smooth_weight(w, lam)
    assert D.rel_fro(xh @ wh, x @ w) <= 1e-12


# ---------------------------------------------------------------- SVD split
def _spiked(K, N, seed):
    return synth.gen_w(K, N, synth.rng(7, seed, 1)).astype(np.float64)


@pytest.mark.parametrize("r", [0, 4, 16])
def test_residual_norm_closed_form(r):
    """||R||_F = sqrt(sum_{i>r} sigma_i^2) to 1e-8 relative."""
    w = _spiked(96, 80, r)
    lam = np.ones(96, np.float32)
    d = S.decompose(w, lam, r)
    assert abs(D.fro(d.R) - D.residual_norm_closed_form(d.sigma, r)) <= 1e-8 * D.fro(d.w_hat)
    assert D.rel_fro(d.L1 @ d.L2 + d.R, d.w_hat) <= 1e-12


def test_full_rank_residual_vanishes():
    w = _spiked(40, 24, 1)
    d = S.decompose(w, np.full(40, 1.5, np.float32), 24)
    assert D.fro(d.R) <= 1e-12 * D.fro(d.w_hat)


def test_eckart_young_on_6x6():
    """The truncated SVD beats 1000 random rank-r competitors."""
    rng = np.random.default_rng(21)
    w = rng.standard_normal((6, 6))
    r = 2
    d = S.decompose(w, np.ones(6, np.float32), r, svd=LA.jacobi_svd)
    best = D.fro(d.R)
    for _ in range(1000):
        a = rng.standard_normal((6, r))
        b = rng.standard_normal((r, 6))
        # best rank-r approximation within the column space of a: least squares
        coef, *_ = np.linalg.lstsq(a, w, rcond=None)
        assert D.fro(w - a @ coef) >= best - 1e-12
        assert D.fro(w - a @ b) >= best - 1e-12


def test_jacobi_svd_matches_lapack():
    rng = np.random.default_rng(22)
    for shape in [(6, 6), (9, 5), (5, 9), (16, 12)]:
        a = rng.standard_normal(shape)
        U, s, Vt = LA.jacobi_svd(a)
        s_ref = np.linalg.svd(a, compute_uv=False)
        np.testing.assert_allclose(s, s_ref, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(U @ np.diag(s) @ Vt, a, atol=1e-12)
        np.testing.assert_allclose(U.T @ U, np.eye(len(s)), atol=1e-12)


def test_lowrank_cost_fraction():
    """(mr + nr)/mn = 2.08 % for m = n = 3072, r = 32."""
    assert abs(D.lowrank_cost_fraction(3072, 3072, 32) - 0.0208333) < 1e-6


# ---------------------------------------------------------------- Eq. 5 / props
def _small_layer(fmt, M=48, K=128, N=80, r=16, seed=3, dt="bf16"):
    x = F.round16(synth.gen_x(M, K, synth.rng(5, seed, 0)), dt)
    w = synth.gen_w(K, N, synth.rng(5, seed, 1))
    lam = S.compute_smoothing(synth.gen_x(M, K, synth.rng(5, seed, 2)), w, 0.5)
    bias = F.round16(synth.gen_bias(N, synth.rng(5, seed, 3)), dt)
    ops = S.prepare_operands(w, lam, r, fmt, gs_x=1.0, scale_dtype=dt, bias=bias)
    return x, w, lam, ops


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_eq5_error_equality_and_prop41(fmt):
    """||X_hat W_hat - (X_hat L1 L2 + Q(X_hat) Q(R))|| = E(X_hat, R),
    and Prop. 4.1 holds for (X_hat, R)."""
    x, w, lam, ops = _small_layer(fmt)
    d = S.decompose(w, lam, ops.rank)
    xh = Q.smooth_activation(x, ops.lam_inv32).astype(np.float64)
    qa = S.quantize_activation(x, ops)
    if fmt == "nvfp4":
        deq_x = Q.dequantize_nvfp4(qa.codes, qa.scales, ops.gs_x)
        deq_r = Q.dequantize_nvfp4(ops.w_codes, ops.w_scales, ops.gs_w).T
    else:
        deq_x = Q.dequantize_int4(qa.codes, qa.scales, ops.scale_dtype)
        deq_r = Q.dequantize_int4(ops.w_codes, ops.w_scales, ops.scale_dtype).T
    R32 = d.R.astype(np.float32).astype(np.float64)
    w_hat = d.L1 @ d.L2 + R32
    lhs = D.fro(xh @ w_hat - (xh @ d.L1 @ d.L2 + deq_x @ deq_r))
    e = D.quant_error(xh, R32, deq_x, deq_r)
    assert abs(lhs - e) <= 1e-9 * max(1.0, e)
    assert e <= D.prop41_bound(xh, R32, deq_x, deq_r)
    # the full layer (original X, W) obeys Prop 4.1 too, with Q(W) := L1L2 + Q(R)
    lam64 = lam.astype(np.float64)
    qw = (d.L1 @ d.L2 + deq_r) / lam64[:, None]
    qx = deq_x * lam64[None, :]
    assert D.quant_error(x, w, qx, qw) <= D.prop41_bound(x, w, qx, qw) * (1 + 1e-12)


def test_svdquant_beats_ablations_on_synthetic():
    """Ablation ordering: SVDQuant's layer error is below
    naive W4A4, smoothing-only and SVD-only on outlier-heavy synthetic layers."""
    for seed in range(3):
        M, K, N, r = 128, 256, 192, 16
        x = F.bf16_round(synth.gen_x(M, K, synth.rng(6, seed, 0))).astype(np.float64)
        w = synth.gen_w(K, N, synth.rng(6, seed, 1)).astype(np.float64)
        lam = S.compute_smoothing(synth.gen_x(M, K, synth.rng(6, seed, 2)), w, 0.5)
        ref = x @ w

        def err(lam_, r_):
            ops = S.prepare_operands(w, lam_, r_, "int4", scale_dtype="bf16")
            _, y64, _ = S.forward(x.astype(np.float32), ops)
            return D.rel_fro(y64, ref)

        ones = np.ones(K, np.float32)
        e_svdq = err(lam, r)
        assert e_svdq < err(ones, 0)        # naive
        assert e_svdq < err(lam, 0)         # smoothing only
        assert e_svdq < err(ones, r)        # SVD only


# ---------------------------------------------------------------- forward
def _brute_force_nvfp4(qa_codes, qa_sf, ops, xl1_bits, alpha, bias):
    M, K = qa_codes.shape
    N = ops.N
    y = np.zeros((M, N))
    xl1 = F.bf16_from_bits(xl1_bits).astype(np.float64)
    L2s = ops.L2s.astype(np.float64)
    for m, n in itertools.product(range(M), range(N)):
        acc = 0.0
        for k in range(K):
            a = float(F.e2m1_decode(qa_codes[m, k])) * float(F.e4m3_decode(qa_sf[m, k // 16]))
            b = float(F.e2m1_decode(ops.w_codes[n, k])) * float(F.e4m3_decode(ops.w_scales[n, k // 16]))
            acc += a * b
        for t in range(ops.rank):
            acc += xl1[m, t] * L2s[n, t]
        y[m, n] = float(alpha) * acc + (0.0 if bias is None else float(bias[n]))
    return y


def _brute_force_int4(qa_codes, qa_s, ops, xl1_bits, bias):
    M, K = qa_codes.shape
    N = ops.N
    sdt = ops.scale_dtype
    y = np.zeros((M, N))
    xl1 = F.bf16_from_bits(xl1_bits).astype(np.float64)
    L2s = ops.L2s.astype(np.float64)
    sx = F.from_bits16(qa_s, sdt).astype(np.float64)
    sw = F.from_bits16(ops.w_scales, sdt).astype(np.float64)
    for m, n in itertools.product(range(M), range(N)):
        acc = 0.0
        for g in range(K // 64):
            ig = sum(int(qa_codes[m, k]) * int(ops.w_codes[n, k]) for k in range(64 * g, 64 * g + 64))
            acc += ig * sx[m, g] * sw[n, g]
        for t in range(ops.rank):
            acc += xl1[m, t] * L2s[n, t]
        y[m, n] = acc + (0.0 if bias is None else float(bias[n]))
    return y


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_forward_matches_brute_force(fmt):
    x, w, lam, ops = _small_layer(fmt, M=5, K=128, N=18, r=16, seed=8)
    y_ref, y64, qa = S.forward(x, ops)
    if fmt == "nvfp4":
        bf = _brute_force_nvfp4(qa.codes, qa.scales, ops, qa.xl1_bits, ops.alpha, ops.bias)
    else:
        bf = _brute_force_int4(qa.codes, qa.scales, ops, qa.xl1_bits, ops.bias)
    np.testing.assert_allclose(y64, bf, rtol=1e-12, atol=1e-12 * np.abs(bf).max())
    # int4 accumulators exact
    if fmt == "int4":
        acc = S.int4_group_accum(qa.codes, ops.w_codes)
        for g in range(2):
            ref = qa.codes[:, 64 * g:64 * g + 64] @ ops.w_codes[:, 64 * g:64 * g + 64].T
            np.testing.assert_array_equal(acc[g], ref)


def test_lossless_case_forward_equals_xw():
    """lambda = 1, r = 0, residual and activations on the lattice ->
    forward = X W exactly (NVFP4 with gs = 1)."""
    rng = np.random.default_rng(30)
    M, K, N = 8, 64, 16
    qx = rng.integers(0, 16, (M, K)).astype(np.uint8)
    qx[:, ::16] = 7
    qw = rng.integers(0, 16, (N, K)).astype(np.uint8)
    qw[:, ::16] = 7
    x = F.e2m1_decode(qx).astype(np.float32)          # sf = e4m3(1.0) when amax 6
    w = F.e2m1_decode(qw).T.astype(np.float32)        # [K, N]
    ops = S.prepare_operands(w, np.ones(K, np.float32), 0, "nvfp4", gs_x=1.0)
    # gs_w = 6/2688 is not a power of two, so re-quantize R with gs_w = 1 (the
    # boundary lets the caller fix gs_w, svdq_quantize_residual's "in: > 0")
    codes, sf, gs = S.quantize_residual(w, "nvfp4", gs_w=1.0)
    ops.w_codes, ops.w_scales, ops.gs_w = codes, sf, np.float32(1.0)
    y_ref, y64, _ = S.forward(x, ops, out_dtype="fp32")
    np.testing.assert_array_equal(y64, x.astype(np.float64) @ w.astype(np.float64))


def test_lowrank_only_matches_matmul():
    """R codes all zero -> Y = alpha xl1 L2s^T + bias (library matmul)."""
    x, w, lam, ops = _small_layer("nvfp4", M=32, K=128, N=64, r=16, seed=4)
    ops.w_codes = np.zeros_like(ops.w_codes)
    _, y64, qa = S.forward(x, ops)
    xl1 = torch.from_numpy(F.bf16_from_bits(qa.xl1_bits).astype(np.float64))
    l2 = torch.from_numpy(ops.L2s.astype(np.float64))
    ref = float(ops.alpha) * (xl1 @ l2.T) + torch.from_numpy(ops.bias.astype(np.float64))
    np.testing.assert_allclose(y64, ref.numpy(), rtol=1e-13, atol=1e-13)


def test_zero_input_gives_bias():
    x, w, lam, ops = _small_layer("nvfp4", M=4, K=64, N=32, r=16, seed=5)
    y_ref, y64, qa = S.forward(np.zeros_like(x), ops)
    np.testing.assert_array_equal(y64, np.broadcast_to(ops.bias.astype(np.float64), y64.shape))
    assert np.all(qa.scales == 0)


# ---------------------------------------------------------------- LoRA
@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_lora_fuse_identity(fmt):
    """fused branch = original branch + scale X A B, to
    1e-9 relative in fp64 with storage-exact factors; R untouched."""
    x, w, lam, ops = _small_layer(fmt, M=40, K=128, N=64, r=16, seed=6)
    if fmt == "nvfp4":
        ops.gs_w = np.float32(2.0 ** -6)          # alpha a power of two: B / alpha exact
    a, b = synth.gen_lora(128, 64, 16, synth.rng(5, 6, 4), synth.rng(5, 6, 5))
    a = F.bf16_round(a)
    b = F.bf16_round(b)
    fused = S.lora_fuse(ops, a, b, 0.5)
    assert fused.rank == 32
    np.testing.assert_array_equal(fused.w_codes, ops.w_codes)
    y0 = S.lowrank_branch_exact(x, ops.L1s, ops.L2s, ops.alpha)
    y1 = S.lowrank_branch_exact(x, fused.L1s, fused.L2s, fused.alpha)
    delta = 0.5 * x.astype(np.float64) @ a.astype(np.float64) @ b.astype(np.float64)
    assert D.rel_fro(y1 - y0, delta) <= 1e-9
    # zero LoRA leaves the layer output unchanged
    z = S.lora_fuse(ops, np.zeros_like(a), b, 1.0)
    _, y_a, _ = S.forward(x, ops)
    _, y_b, _ = S.forward(x, z)
    np.testing.assert_allclose(y_a, y_b, rtol=0, atol=1e-12 * np.abs(y_a).max())


def test_lora_shape_mismatch():
    x, w, lam, ops = _small_layer("int4", M=4, K=64, N=32, r=16)
    with pytest.raises(ValueError):
        S.lora_fuse(ops, np.zeros((32, 16), np.float32), np.zeros((16, 32), np.float32), 1.0)
