"""Offline weight path through the C ABI: residual quantization bit-exact
against the oracle; full weight preparation (GPU fp64 Gram + eigensolver SVD)
against the oracle's LAPACK SVD (products, not factors: reading Q2); LoRA
fusion bit-exact; and the end-to-end K1 -> K2 forward."""
import numpy as np
import pytest

import synth
from helpers import layer_from_ops, make_case, need_cuda, pack_weight, rel_fro, to_dev
from oracle import formats as F
from oracle import svdquant as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt,sdt", [("nvfp4", "bf16"), ("int4", "bf16"), ("int4", "fp16")])
@pytest.mark.parametrize("K,N", [(512, 512), (256, 144), (1152, 3456)])
def test_quantize_residual_bit_exact(fmt, sdt, K, N):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    R32 = (synth.gen_w(K, N, synth.rng(13, K + N, 1)) * 0.3).astype(np.float32)
    codes, scales, gs = P.svdq_quantize_residual(torch.from_numpy(R32).cuda(), fmt, sdt)
    torch.cuda.synchronize()
    rc, rs, rgs = S.quantize_residual(R32, fmt, sdt)
    assert np.float32(gs) == rgs
    ops = S.Operands(fmt, K, N, 0, rc, rs, sdt if fmt == "int4" else "e4m3", rgs, np.float32(1),
                     None, None, None, None)
    ref_c, ref_s = pack_weight(ops)
    np.testing.assert_array_equal(codes.cpu().numpy(), ref_c.reshape(-1))
    np.testing.assert_array_equal(scales.cpu().numpy(), ref_s.reshape(-1))


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("K,N,r", [(512, 512, 16), (256, 768, 32), (1152, 384, 32)])
def test_quantize_weights_svd(fmt, K, N, r):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    w = synth.gen_w(K, N, synth.rng(14, K, 1))
    lam = S.compute_smoothing(synth.gen_x(128, K, synth.rng(14, K, 2)), w, 0.5)
    layer = P.svdq_quantize_weights(torch.from_numpy(w).cuda(), torch.from_numpy(lam).cuda(), r, fmt,
                                    "bf16", 1.0)
    torch.cuda.synchronize()
    d = S.decompose(w, lam, r)
    # lambda_inv bit-exact
    np.testing.assert_array_equal(layer.lambda_inv.cpu().numpy(), S.lambda_inverse(lam))
    # the low-rank product, reconstructed from the stored bf16 operands, vs the oracle's
    alpha = np.float32(layer.gs_x * layer.gs_w) if fmt == "nvfp4" else np.float32(1)
    l1s = F.bf16_from_bits(layer.l1s.cpu().numpy().view(np.uint16).reshape(r, K)).astype(np.float64)
    l2s = F.bf16_from_bits(layer.l2s.cpu().numpy().view(np.uint16).reshape(N, r)).astype(np.float64)
    prod = (l1s.T * lam.astype(np.float64)[:, None]) @ (l2s.T * float(alpha))
    assert rel_fro(prod, d.L1 @ d.L2) <= 2e-2        # bf16 storage of both factors dominates
    # residual codes: compare against the oracle's quantizer on the oracle's R
    ops = S.prepare_operands(w, lam, r, fmt, scale_dtype="bf16")
    ref_c, ref_s = pack_weight(ops)
    got = layer.w_codes.cpu().numpy()
    mismatch = np.mean(got != ref_c.reshape(-1))
    assert mismatch <= 2e-3, mismatch
    if fmt == "nvfp4":
        assert abs(layer.gs_w - float(ops.gs_w)) <= 1e-5 * float(ops.gs_w)


def test_quantize_weights_given_factors_exact():
    """With L1 / L2 supplied, R = W_hat - L1 L2 is formed in fp64 on the device;
    the stored operands then follow the fp32 recipe bit for bit."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    K, N, r = 256, 192, 16
    w = synth.gen_w(K, N, synth.rng(15, 0, 1))
    lam = S.compute_smoothing(synth.gen_x(64, K, synth.rng(15, 0, 2)), w, 0.5)
    d = S.decompose(w, lam, r)
    L1 = d.L1.astype(np.float32)
    L2 = d.L2.astype(np.float32)
    layer = P.svdq_quantize_weights(torch.from_numpy(w).cuda(), torch.from_numpy(lam).cuda(), r, "nvfp4",
                                    "bf16", 1.0, L1=torch.from_numpy(L1).cuda(), L2=torch.from_numpy(L2).cuda())
    torch.cuda.synchronize()
    R = S.smooth_weight(w, lam) - L1.astype(np.float64) @ L2.astype(np.float64)
    rc, rs, gs = S.quantize_residual(R.astype(np.float32), "nvfp4")
    assert np.float32(layer.gs_w) == gs
    np.testing.assert_array_equal(layer.w_codes.cpu().numpy(), F.pack_nibbles(rc).reshape(-1))
    lam_inv = S.lambda_inverse(lam)
    ref_l1s = F.bf16_bits((lam_inv[:, None] * L1).astype(np.float32)).T
    np.testing.assert_array_equal(layer.l1s.cpu().numpy().view(np.uint16).reshape(r, K), ref_l1s)
    alpha = np.float32(np.float32(1.0) * gs)
    ref_l2s = F.bf16_bits((L2 / alpha).astype(np.float32)).T
    np.testing.assert_array_equal(layer.l2s.cpu().numpy().view(np.uint16).reshape(N, r), ref_l2s)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("ab", ["bf16", "fp32"])
def test_lora_fuse_bit_exact(fmt, ab):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    x, w, lam, ops = make_case(fmt, 64, 640, 320, 32, dt="fp16", seed=2)
    dev = torch.device("cuda")
    layer = layer_from_ops(P, ops, dev, bias_dtype="fp16")
    a, b = synth.gen_lora(640, 320, 16, synth.rng(16, 0, 4), synth.rng(16, 0, 5))
    if ab == "bf16":
        a, b = F.bf16_round(a), F.bf16_round(b)
    tdt = P.TORCH_DTYPE[ab]
    fused = P.svdq_lora_fuse(layer, torch.from_numpy(a).to(dev).to(tdt), torch.from_numpy(b).to(dev).to(tdt), 0.75)
    torch.cuda.synchronize()
    ref = S.lora_fuse(ops, a, b, 0.75)
    assert fused.rank == ref.rank == 48
    np.testing.assert_array_equal(fused.l1s.cpu().numpy().view(np.uint16).reshape(48, 640), ref.L1s_bits)
    np.testing.assert_array_equal(fused.l2s.cpu().numpy().view(np.uint16).reshape(320, 48), ref.L2s_bits)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("dt", ["bf16", "fp16"])
def test_end_to_end_forward(fmt, dt):
    """svdq_linear_forward (K1 -> K2) vs the oracle's forward, 1e-3 relative Frobenius."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    M, K, N, r = 384, 1152, 640, 32
    x, w, lam, ops = make_case(fmt, M, K, N, r, dt=dt, seed=21)
    dev = torch.device("cuda")
    layer = layer_from_ops(P, ops, dev, bias_dtype=dt)
    X = torch.from_numpy(x).to(dev).to(P.TORCH_DTYPE[dt])
    try:
        Y = layer(X)
    except P.SvdqError as e:
        if e.status == 5 and fmt == "int4":
            pytest.skip("INT4 GEMM not built")
        raise
    torch.cuda.synchronize()
    y_ref, y64, _ = S.forward(x, ops, out_dtype=dt)
    assert rel_fro(Y.float().cpu().numpy(), y_ref) <= 1e-3
