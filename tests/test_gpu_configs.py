"""Full-size parity on the BASELINE.json configurations: one K1 -> K2 pass
through the C ABI at the real PixArt-Sigma (C2), SDXL + LoRA (C3) and FLUX.1 (C4) layer
shapes, in the launch configuration bench.py times.  The oracle recomputes sampled rows
one by one (quantization, xl1 and Y are row-local), so the comparison is:
  * codes / scale bytes of sampled rows: bit-exact;
  * xl1 of sampled rows: <= 1e-3 relative Frobenius vs the oracle's bf16 xl1;
  * Y of sampled rows given the GPU's own operands: <= 1e-3 vs oracle Y rounded to the
    output dtype (reading Q17), and end to end with the oracle's operands: <= 1e-3.
Plus the library pins of SURVEY §8(c.3): K2 at r = 0 against cuBLASLt's NVFP4 GEMM
(torch._scaled_mm) on identical operands, INT4 with unit scales against an exact integer
GEMM (torch._int_mm), and the low-rank-only case against torch.matmul."""
import numpy as np
import pytest

import synth
from helpers import layer_from_ops, make_case, need_cuda, rel_fro, to_dev
from oracle import formats as F
from oracle import svdquant as S

pytestmark = pytest.mark.gpu

BY_NAME = {L.name: L for L in synth.C2 + synth.C3 + synth.C4}


def _rows(M, n, seed):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([rng.choice(M, min(n, M), replace=False), [0, M - 1]]))


def _act_rows(fmt, xq, xs, M, K, rows):
    """Device K1 outputs -> (codes bytes [rows, K/2], scale bytes / bits [rows, K/16 | K/64])."""
    xq = xq.cpu().numpy().reshape(-1)[: M * K // 2].reshape(M, K // 2)[rows]
    xs = xs.cpu().numpy()
    if fmt == "nvfp4":
        sf = F.sf_from_layout(xs, M, K)[rows]
    else:
        sf = xs.view(np.uint16).reshape(-1)[: M * K // 64].reshape(M, K // 64)[rows]
    return xq, sf


@pytest.mark.parametrize("name,fmt", [
    ("pixart_qkv", "nvfp4"), ("pixart_fc2", "int4"), ("pixart_attn_out", "nvfp4"),
    ("sdxl640_geglu", "nvfp4"), ("sdxl1280_ffout", "int4"), ("sdxl640_out", "nvfp4"),
    ("flux_mlp_down", "nvfp4"), ("flux_single_linear2", "nvfp4"), ("flux_attn_out", "int4"),
])
def test_config_layer_full_size(name, fmt):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    L = BY_NAME[name]
    M, K, N, r, dt = L.M, L.K, L.N, L.r, L.dtype
    x, w, lam, ops = make_case(fmt, M, K, N, r, dt=dt, seed=sum(name.encode()) % 1000, cfg=40)
    dev = torch.device("cuda")
    layer = layer_from_ops(P, ops, dev, bias_dtype=dt)
    if L.lora:                                         # C3: r = 32 + LoRA 16 by concatenation
        a, b = synth.gen_lora(K, N, L.lora, synth.rng(40, 1, 4), synth.rng(40, 1, 5))
        layer = P.svdq_lora_fuse(layer, torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), 1.0)
        ops = S.lora_fuse(ops, a, b, 1.0)
        assert layer.rank == ops.rank == r + L.lora
    X = torch.from_numpy(x).to(dev).to(P.TORCH_DTYPE[dt])
    xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, X)
    Y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, out_dtype=P.TORCH_DTYPE[dt])
    torch.cuda.synchronize()
    rows = _rows(M, 24, M + K)
    qa = S.quantize_activation(x[rows], ops)
    gq, gs = _act_rows(fmt, xq, xs, M, K, rows)
    ref_q = F.pack_nibbles(qa.codes if fmt == "nvfp4" else F.int4_to_nibble(qa.codes))
    np.testing.assert_array_equal(gq, ref_q)
    np.testing.assert_array_equal(gs, np.asarray(qa.scales).astype(gs.dtype))
    g_xl1 = xl1.cpu().numpy().view(np.uint16).reshape(M, ops.rank)[rows]
    assert rel_fro(F.bf16_from_bits(g_xl1), F.bf16_from_bits(qa.xl1_bits)) <= 1e-3
    y = Y.float().cpu().numpy()[rows]
    # given identical operands (the GPU's xl1)
    qg = S.QuantAct(qa.codes, qa.scales, g_xl1, qa.xl1_exact)
    err_k2 = rel_fro(y, S.round_output(S.gemm_reference(qg, ops), dt))
    # end to end against the oracle's own K1
    err_e2e = rel_fro(y, S.round_output(S.gemm_reference(qa, ops), dt))
    assert err_k2 <= 1e-3, err_k2
    assert err_e2e <= 1e-3, err_e2e


def _random_nvfp4_layer(P, torch, M, K, N, dev, gen, rank=0):
    layer = P.QuantizedLinear.empty("nvfp4", K, N, rank, device=dev)
    layer.w_codes.random_(0, 256, generator=gen)
    layer.w_scales.random_(0x28, 0x40, generator=gen)
    layer.lambda_inv.fill_(1.0)
    layer.gs_w = 1.0
    layer._sync_view()
    return layer


@pytest.mark.parametrize("M,K,N", [(256, 512, 512), (4096, 3072, 9216), (4608, 15360, 3072), (512, 12288, 3072)])
def test_k2_rank0_matches_cublas_nvfp4(M, K, N):
    """SURVEY §8(c.3) 'Main GEMM with r=0, lambda=1': K2 vs cuBLASLt block-scaled NVFP4
    (torch._scaled_mm, float4_e2m1fn_x2 x float4_e2m1fn_x2, e4m3 128x4-swizzled scales) on
    the very same code / scale-factor bytes.  Both accumulate exact e2m1 products in fp32."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    if not hasattr(torch, "float4_e2m1fn_x2"):
        pytest.skip("torch without float4_e2m1fn_x2")
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(M + N)
    layer = _random_nvfp4_layer(P, torch, M, K, N, dev, gen)
    x = torch.randn(M, K, device=dev, generator=gen).to(torch.bfloat16)
    xq, xs, _ = P.svdq_quantize_act_lowrank_down(layer, x)
    Y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, None, M)
    fa = xq.reshape(M, K // 2).view(torch.float4_e2m1fn_x2)
    fb = layer.w_codes.reshape(N, K // 2).view(torch.float4_e2m1fn_x2)
    try:
        yl = torch._scaled_mm(fa, fb.t(), xs.view(torch.float8_e4m3fn), layer.w_scales.view(torch.float8_e4m3fn),
                              out_dtype=torch.bfloat16)
    except (RuntimeError, NotImplementedError) as e:
        pytest.skip(f"library NVFP4 GEMM unavailable: {e}")
    torch.cuda.synchronize()
    err = float((Y.float() - yl.float()).norm() / yl.float().norm())
    assert err <= 1e-3, err
    # accumulation order differs at most by fp32 rounding; bf16 outputs then agree almost everywhere
    assert float((Y == yl).float().mean()) >= 0.99


def test_int4_unit_scales_match_int_mm():
    """INT4 K2 with unit scales and r = 0: Y = bf16(sum_k qa qb) exactly (|sum| < 2^24),
    checked against torch._int_mm on the int8-widened codes (an exact integer GEMM)."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    M, K, N = 320, 1024, 384
    rng = np.random.default_rng(5)
    qa = rng.integers(-7, 8, (M, K))
    qb = rng.integers(-7, 8, (N, K))
    dev = torch.device("cuda")
    one = np.full((N, K // 64), F.bf16_bits(np.float32(1.0)), dtype=np.uint16)
    z = torch.zeros(8, dtype=torch.int16, device=dev)
    layer = P.QuantizedLinear("int4", K, N, 0, to_dev(F.pack_nibbles(F.int4_to_nibble(qb)).reshape(-1), dev),
                              to_dev(one.view(np.uint8).reshape(-1), dev),
                              torch.ones(K, dtype=torch.float32, device=dev), z, z, None, "bf16", 1.0, 1.0)
    xs = np.full((M, K // 64), F.bf16_bits(np.float32(1.0)), dtype=np.uint16)
    Y = P.svdq_gemm_w4a4_lowrank_up(layer, to_dev(F.pack_nibbles(F.int4_to_nibble(qa)).reshape(-1), dev),
                                    to_dev(xs.view(np.uint8).reshape(-1), dev), None, M, out_dtype=torch.float32)
    ref = torch._int_mm(torch.from_numpy(qa).to(dev).to(torch.int8),
                        torch.from_numpy(qb).to(dev).to(torch.int8).t())
    torch.cuda.synchronize()
    assert torch.equal(Y, ref.float())


def test_lowrank_only_matches_matmul():
    """All residual codes zero: Y = alpha * xl1 L2s^T + bias, vs torch.matmul in fp32."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    M, K, N, r = 640, 1024, 768, 32
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(11)
    bias = (torch.randn(N, device=dev, generator=gen) * 0.1).to(torch.bfloat16)
    layer = P.QuantizedLinear.empty("nvfp4", K, N, r, device=dev, bias=bias)
    layer.w_codes.zero_()
    layer.w_scales.fill_(0x38)
    layer.lambda_inv.fill_(1.0)
    l2 = (torch.randn(N, r, device=dev, generator=gen) * 0.05).to(torch.bfloat16)
    layer.l2s.copy_(l2.view(torch.int16).reshape(-1))
    layer.gs_w = 0.75
    layer._sync_view()
    xl1 = torch.randn(M, r, device=dev, generator=gen).to(torch.bfloat16)
    xq = torch.zeros(M * K // 2, dtype=torch.uint8, device=dev)
    _, xs_b, _ = P.svdq_act_buffer_sizes("nvfp4", M, K, r)
    xs = torch.full((xs_b,), 0x38, dtype=torch.uint8, device=dev)
    Y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1.view(torch.int16).reshape(-1), M, out_dtype=torch.float32)
    ref = 0.75 * (xl1.float() @ l2.float().t()) + bias.float()
    torch.cuda.synchronize()
    err = float((Y - ref).norm() / ref.norm())
    assert err <= 1e-6, err
