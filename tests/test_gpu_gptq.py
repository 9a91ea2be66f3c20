"""GPTQ residual quantization (App. D) through the C ABI against
oracle/gptq.py.  Given the same residual and calibration batch, codes and scales match the oracle
(the GPU applies the trailing updates as blocked DGEMMs, a different fp64 summation order than the
oracle's rank-1 updates, so a code at an exact rounding boundary may flip: <= 0.2 % of codes, proxy
loss within 0.1 %); orthogonal calibration channels reduce GPTQ to RTN bit for bit; dead channels
give zero codes; the full weight preparation with GPTQ matches the oracle's calibration error and
beats round-to-nearest."""
from types import SimpleNamespace

import numpy as np
import pytest

import synth
from helpers import need_cuda
from oracle import formats as F
from oracle import gptq as G
from oracle import quant as Q
from oracle import svdquant as S

pytestmark = pytest.mark.gpu


def _unpack(fmt, codes, scales, K, N, sdt="bf16"):
    c = codes.cpu().numpy()
    s = scales.cpu().numpy()
    if fmt == "nvfp4":
        return F.unpack_nibbles(c.reshape(N, K // 2)), F.sf_from_layout(s, N, K)
    if fmt == "int4":
        return F.nibble_to_int4(F.unpack_nibbles(c.reshape(N, K // 2))), s.view(np.uint16).reshape(N, K // 64)
    return c.view(np.int8).reshape(N, K).astype(np.int64), s.view(np.float32)[:N]


def _deq(fmt, codes, scales, gs, K, N):
    ops = SimpleNamespace(fmt=fmt, w_codes=codes, w_scales=scales, gs_w=np.float32(gs), scale_dtype="bf16")
    return S.dequantize_residual(ops)


def _inputs(seed, M, K, N):
    x = F.bf16_round(synth.gen_x(M, K, synth.rng(77, seed, 0)))
    w = synth.gen_w(K, N, synth.rng(77, seed, 1)).astype(np.float32)
    lam = S.compute_smoothing(x, w, 0.5)
    R = S.decompose(w, lam, 16).R.astype(np.float32)
    return x, w, lam, R


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
@pytest.mark.parametrize("M,K,N", [(300, 256, 208), (64, 192, 128)])
def test_gptq_residual_matches_oracle(fmt, M, K, N):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    dev = torch.device("cuda")
    x, w, lam, R = _inputs(K + N, M, K, N)
    lam_inv = S.lambda_inverse(lam)
    X = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    codes, scales, gs = P.svdq_quantize_residual_gptq(torch.from_numpy(R).to(dev), X,
                                                      torch.from_numpy(lam_inv).to(dev), fmt)
    gc, gsc = _unpack(fmt, codes, scales, K, N)
    xh = Q.smooth_activation(x, lam_inv)
    rc, rs, rgs = G.gptq_quantize_residual(R, xh, fmt)
    assert np.float32(gs) == rgs
    assert np.mean(gc != rc) <= 2e-3
    assert np.mean(gsc != rs) <= 2e-3
    lg = G.proxy_loss(R, xh, _deq(fmt, gc, gsc, gs, K, N))
    lr = G.proxy_loss(R, xh, _deq(fmt, rc, rs, rgs, K, N))
    assert abs(lg - lr) <= 1e-3 * lr


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
def test_gptq_orthogonal_calibration_is_rtn(fmt):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    dev = torch.device("cuda")
    rng = np.random.default_rng(9)
    K, N, M = 256, 128, 512
    R = (rng.standard_normal((K, N)) * 0.1).astype(np.float32)
    x = np.zeros((M, K), np.float32)
    x[np.arange(M), np.arange(M) % K] = F.bf16_round(rng.uniform(0.5, 2.0, M))
    Rd = torch.from_numpy(R).to(dev)
    codes, scales, gs = P.svdq_quantize_residual_gptq(Rd, torch.from_numpy(x).to(dev).to(torch.bfloat16),
                                                      torch.ones(K, device=dev), fmt)
    c2, s2, gs2 = P.svdq_quantize_residual(Rd, fmt)
    assert torch.equal(codes, c2) and gs == gs2
    assert torch.equal(scales[: s2.numel()], s2)


def test_gptq_dead_channels_zero():
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    dev = torch.device("cuda")
    x, w, lam, R = _inputs(3, 128, 128, 64)
    x[:, [5, 77]] = 0
    codes, scales, gs = P.svdq_quantize_residual_gptq(torch.from_numpy(R).to(dev),
                                                      torch.from_numpy(x).to(dev).to(torch.bfloat16),
                                                      torch.from_numpy(S.lambda_inverse(lam)).to(dev), "int4")
    gc, _ = _unpack("int4", codes, scales, 128, 64)
    assert np.all(gc[:, [5, 77]] == 0)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
def test_weights_gptq_pipeline(fmt):
    """svdq_quantize_weights_gptq vs oracle prepare_operands(gptq_x=...): calibration error within 3 %
    (independent SVDs), and below the round-to-nearest layer's on the same data."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    dev = torch.device("cuda")
    M, K, N, r = 256, 256, 128, 16
    x, w, lam, _ = _inputs(11, M, K, N)
    X = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    W = torch.from_numpy(w).to(dev)
    L = torch.from_numpy(lam).to(dev)
    lay_g = P.svdq_quantize_weights_gptq(W, L, r, fmt, X)
    lay_r = P.svdq_quantize_weights(W, L, r, fmt)

    def obj(layer):
        xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, X)
        Y = torch.empty(M, N, dtype=torch.float32, device=dev)
        P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, Y=Y)
        return float(np.sum((Y.double().cpu().numpy() - x.astype(np.float64) @ w.astype(np.float64)) ** 2))

    e_g, e_r = obj(lay_g), obj(lay_r)
    ref = S.calibration_error(x, w, S.prepare_operands(w, lam, r, fmt, gptq_x=x))
    np.testing.assert_allclose(e_g, ref, rtol=3e-2)
    assert e_g < e_r
