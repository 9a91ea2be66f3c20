"""Oracle pins for GPTQ residual quantization (App. D).

* diagonal Hessian (orthogonal calibration columns): no error propagation, so GPTQ == RTN
  (svdquant.quantize_residual) code for code, scale for scale, in every format;
* lattice-exact residual: every quantization error is zero, so codes round-trip exactly;
* the Cholesky row update equals the Optimal-Brain-Surgeon update written with the explicit
  inverse of the remaining sub-Hessian (the identity GPTQ rests on), recomputed per column;
* GPTQ lowers the proxy loss ||X_hat R - X_hat Q(R)||^2 below RTN on random instances (paired);
* dead calibration channels quantize to zero codes.
"""
import numpy as np
import pytest

import synth
from oracle import formats as F
from oracle import gptq as G
from oracle import quant as Q
from oracle import svdquant as S

GROUP = {"nvfp4": 16, "int4": 64, "w8a8": None}


def _deq(codes, scales, gs, fmt, K, N, sdt="bf16"):
    ops = S.Operands(fmt, K, N, 0, codes, scales, {"nvfp4": "e4m3", "w8a8": "fp32"}.get(fmt, sdt), gs,
                     np.float32(1), np.ones(K, np.float32), np.zeros((0, K), np.uint16),
                     np.zeros((N, 0), np.uint16), None)
    return S.dequantize_residual(ops)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
def test_diagonal_hessian_is_rtn(fmt):
    rng = np.random.default_rng(1)
    K, N = 128, 48
    R = (rng.standard_normal((K, N)) * 0.1).astype(np.float32)
    xh = np.zeros((2 * K, K), np.float32)
    xh[np.arange(2 * K), np.arange(2 * K) % K] = rng.uniform(0.5, 2.0, 2 * K)
    codes, scales, gs = G.gptq_quantize_residual(R, xh, fmt)
    rc, rs, rgs = S.quantize_residual(R, fmt)
    np.testing.assert_array_equal(codes, rc)
    np.testing.assert_array_equal(scales, rs)
    assert gs == rgs


def test_lattice_residual_round_trips():
    rng = np.random.default_rng(2)
    K, N, G64 = 128, 32, 2
    codes = rng.integers(-7, 8, size=(N, K))
    codes[:, ::64] = 7
    s = F.bf16_round(rng.uniform(0.01, 0.05, size=(N, G64)))
    R = (codes.reshape(N, G64, 64) * s[:, :, None]).reshape(N, K).T.astype(np.float32)
    xh = rng.standard_normal((256, K)).astype(np.float32)
    c, sc, _ = G.gptq_quantize_residual(R, xh, "int4")
    np.testing.assert_array_equal(c, codes)
    np.testing.assert_array_equal(_deq(c, sc, np.float32(1), "int4", K, N), R.astype(np.float64))


def _obs_explicit(R32, xh, fmt, damp=G.DAMP):
    """Column-by-column OBS with the explicit inverse of the not-yet-quantized sub-Hessian:
    delta_F = -(w_k - q_k) / [H_F^-1]_{kk} * [H_F^-1]_{k, F} (Frantar et al., Eq. 3 / Algorithm 1)."""
    Wt = np.asarray(R32, np.float32).T.astype(np.float64)
    N, K = Wt.shape
    H = xh.astype(np.float64).T @ xh.astype(np.float64)
    H[np.diag_indices_from(H)] += damp * np.mean(np.diag(H))
    g = GROUP[fmt] or K
    gs = Q.nvfp4_global_scale(Wt.astype(np.float32)) if fmt == "nvfp4" else np.float32(1)
    codes = np.zeros((N, K), np.int64)
    w8_s = Q.quantize_int8_rows(Wt.astype(np.float32))[1] if fmt == "w8a8" else None
    for k in range(K):
        if k % g == 0 and fmt != "w8a8":
            slab = Wt[:, k:k + g].astype(np.float32)
            col_s = (Q.quantize_nvfp4(slab, gs) if fmt == "nvfp4" else Q.quantize_int4(slab, "bf16"))[1][:, 0]
        q, deq = G._encode_col(Wt[:, k].astype(np.float32), fmt, w8_s if fmt == "w8a8" else col_s, "bf16", gs)
        codes[:, k] = q
        Hi = np.linalg.inv(H[k:, k:])
        Wt[:, k:] -= ((Wt[:, k] - deq) / Hi[0, 0])[:, None] * Hi[0][None, :]
    return codes


@pytest.mark.parametrize("fmt,K", [("nvfp4", 48), ("int4", 64), ("w8a8", 32)])
def test_cholesky_update_equals_explicit_obs(fmt, K):
    rng = np.random.default_rng(3)
    N = 24
    R = (rng.standard_normal((K, N)) * 0.1).astype(np.float32)
    A = rng.standard_normal((K, K)) * 0.3 + np.eye(K)          # correlated calibration channels
    xh = (rng.standard_normal((3 * K, K)) @ A).astype(np.float32)
    codes, _, _ = G.gptq_quantize_residual(R, xh, fmt)
    np.testing.assert_array_equal(np.asarray(codes, np.int64), _obs_explicit(R, xh, fmt))


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
def test_gptq_beats_rtn_on_proxy_loss(fmt):
    wins = 0
    for seed in range(10):
        M, K, N = 256, 128, 48
        x = F.bf16_round(synth.gen_x(M, K, synth.rng(76, seed, 0)))
        w = synth.gen_w(K, N, synth.rng(76, seed, 1))
        lam = S.compute_smoothing(x, w, 0.5)
        R = S.decompose(w, lam, 16).R.astype(np.float32)
        xh = Q.smooth_activation(x, S.lambda_inverse(lam))
        c, s, gs = G.gptq_quantize_residual(R, xh, fmt)
        rc, rs, rgs = S.quantize_residual(R, fmt)
        sdt = "bf16"
        lg = G.proxy_loss(R, xh, _deq(c, s, gs, fmt, K, N, sdt))
        lr = G.proxy_loss(R, xh, _deq(rc, rs, rgs, fmt, K, N, sdt))
        wins += lg < lr
    assert wins >= 9


def test_dead_channels_quantize_to_zero():
    rng = np.random.default_rng(4)
    K, N = 64, 16
    R = (rng.standard_normal((K, N)) * 0.1).astype(np.float32)
    xh = rng.standard_normal((128, K)).astype(np.float32)
    xh[:, [3, 40]] = 0
    codes, _, _ = G.gptq_quantize_residual(R, xh, "int4")
    assert np.all(codes[:, [3, 40]] == 0)
