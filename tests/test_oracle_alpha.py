"""Oracle pins for the migration-strength search (App. D): lambda(alpha) end points,
singleton grid, and an independent re-evaluation of every objective."""
import numpy as np
import pytest

import synth
from oracle import formats as F
from oracle import svdquant as S


def _cal(K=128, N=64, M=96, seed=0):
    x = F.bf16_round(synth.gen_x(M, K, synth.rng(70, seed, 0)))
    w = synth.gen_w(K, N, synth.rng(70, seed, 1))
    return x, w


def test_lambda_end_points():
    """alpha = 1: lambda = max|X_:,i| (all migration to W); alpha = 0: lambda = 1 / max|W_i,:|."""
    x, w = _cal()
    np.testing.assert_allclose(S.compute_smoothing(x, w, 1.0), np.max(np.abs(x), 0).astype(np.float32), rtol=0)
    np.testing.assert_allclose(S.compute_smoothing(x, w, 0.0), (1.0 / np.max(np.abs(w), 1)).astype(np.float32),
                               rtol=1e-7)


def test_singleton_grid_returns_it():
    x, w = _cal()
    a, lam, errs = S.search_alpha(x, w, 16, "nvfp4", [0.35])
    assert a == 0.35 and len(errs) == 1
    np.testing.assert_array_equal(lam, S.compute_smoothing(x, w, 0.35))


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_objective_is_the_deployed_output_error(fmt):
    """Each objective equals ||XW - Y||^2 recomputed from an independent fake-quant GEMM:
    dequantized activation codes times dequantized residual plus the fp64 low-rank branch."""
    x, w = _cal(seed=1)
    grid = [0.0, 0.5, 1.0]
    a, lam, errs = S.search_alpha(x, w, 16, fmt, grid)
    for alpha, e in zip(grid, errs):
        lam_a = S.compute_smoothing(x, w, alpha)
        ops = S.prepare_operands(w, lam_a, 16, fmt)
        xh = (x.astype(np.float32) * ops.lam_inv32).astype(np.float32)
        from oracle import quant as Q
        if fmt == "nvfp4":
            c, sf = Q.quantize_nvfp4(xh, ops.gs_x)
            qx = Q.dequantize_nvfp4(c, sf, ops.gs_x)
            qr = Q.dequantize_nvfp4(ops.w_codes, ops.w_scales, ops.gs_w)
        else:
            c, sb = Q.quantize_int4(xh, ops.scale_dtype)
            qx = Q.dequantize_int4(c, sb, ops.scale_dtype)
            qr = Q.dequantize_int4(ops.w_codes, ops.w_scales, ops.scale_dtype)
        xl1 = F.bf16_round(x.astype(np.float64) @ ops.L1s.astype(np.float64).T).astype(np.float64)
        low = float(ops.alpha) * (xl1 @ ops.L2s.astype(np.float64).T)
        y = qx @ qr.T + low
        ref = x.astype(np.float64) @ w
        np.testing.assert_allclose(e, np.sum((y - ref) ** 2), rtol=1e-9)
    assert errs[grid.index(a)] == min(errs)


def test_search_prefers_migration_on_outliers():
    """Activations with x50 outlier channels (Fig. 3): some migration beats none (alpha = 0 keeps
    all outliers in X) -- the reason SmoothQuant-style smoothing precedes the SVD."""
    x, w = _cal(K=256, N=128, M=128, seed=2)
    a, lam, errs = S.search_alpha(x, w, 16, "int4", [0.0, 0.25, 0.5, 0.75])
    assert a > 0.0 and min(errs) < errs[0]
