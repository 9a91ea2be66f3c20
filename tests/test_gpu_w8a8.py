"""W8A8 (the paper's 8-bit setting) through the C ABI against the oracle:
per-token INT8 codes and fp32 scales bit-exact, per-channel weight codes / scales bit-exact
from svdq_quantize_residual, Y within 1e-3 relative Frobenius (reading Q17), the whole-K int32
accumulation exact (unit scales vs torch._int_mm), and end to end at FLUX / PixArt shapes."""
import numpy as np
import pytest

import synth
from helpers import layer_from_ops, make_case, need_cuda, pack_act, rel_fro, to_dev
from oracle import formats as F
from oracle import svdquant as S

pytestmark = pytest.mark.gpu


def _k1(P, torch, layer, x, dt, dev):
    X = torch.from_numpy(x).to(dev).to(P.TORCH_DTYPE[dt])
    xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, X)
    torch.cuda.synchronize()
    return X, xq, xs, xl1


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
# rank 0: the INT8 kernel takes its own amax pass; rank > 0: the amax comes from the row-tile
# kernel's down-projection pass (one encode pass), incl. a ragged last stage (K = 6208 = 97 blocks)
@pytest.mark.parametrize("M,K,N,r", [(256, 512, 512, 16), (129, 1152, 208, 16), (1, 64, 16, 0), (300, 3072, 384, 32),
                                     (300, 1152, 208, 0), (129, 6208, 64, 16)])
def test_w8a8_k1_k2_parity(dt, M, K, N, r):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    x, w, lam, ops = make_case("w8a8", M, K, N, r, dt=dt, seed=M + K)
    dev = torch.device("cuda")
    layer = layer_from_ops(P, ops, dev, bias_dtype=dt)
    X, xq, xs, xl1 = _k1(P, torch, layer, x, dt, dev)
    qa = S.quantize_activation(x, ops)
    ref_q, ref_s = pack_act("w8a8", qa, K)
    np.testing.assert_array_equal(xq.cpu().numpy().reshape(M, K), ref_q)
    np.testing.assert_array_equal(xs.cpu().numpy()[: M * 4], ref_s)
    if r:
        g = xl1.cpu().numpy().view(np.uint16).reshape(M, r)
        assert rel_fro(F.bf16_from_bits(g), F.bf16_from_bits(qa.xl1_bits)) <= 1e-3
        qa = S.QuantAct(qa.codes, qa.scales, g, qa.xl1_exact)
    Y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, out_dtype=P.TORCH_DTYPE[dt])
    torch.cuda.synchronize()
    y_ref = S.round_output(S.gemm_reference(qa, ops), dt)
    err = rel_fro(Y.float().cpu().numpy(), y_ref)
    assert err <= 1e-3, err


@pytest.mark.parametrize("K,N", [(512, 512), (1152, 3456)])
def test_w8a8_residual_quantization_bit_exact(K, N):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    R = (np.random.default_rng(K).standard_normal((K, N)) * 0.05).astype(np.float32)
    R[:, 3] = 0.0                                          # zero channel: s = 0, codes 0
    dev = torch.device("cuda")
    codes, scales, gs = P.svdq_quantize_residual(torch.from_numpy(R).to(dev), "w8a8")
    torch.cuda.synchronize()
    rc, rs, _ = S.quantize_residual(R, "w8a8")
    np.testing.assert_array_equal(codes.cpu().numpy().view(np.int8).reshape(N, K), rc.astype(np.int8))
    np.testing.assert_array_equal(scales.cpu().numpy().view(np.float32), rs)


def test_w8a8_whole_k_int32_accumulation_exact():
    """Unit scales, rank 0, no bias, fp32 Y: Y == f32(sum_k qa qb), the exact int32 sum over
    the whole K (|sum| up to K 127^2 > 2^24, so both sides round it once to fp32)."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    M, K, N = 200, 2048, 256
    rng = np.random.default_rng(9)
    qa = rng.integers(-127, 128, (M, K))
    qb = rng.integers(-127, 128, (N, K))
    qa[0, :] = 127
    qb[0, :] = 127                                         # 2048 * 127^2 = 33 032 192 > 2^24
    dev = torch.device("cuda")
    z = torch.zeros(8, dtype=torch.int16, device=dev)
    one_w = torch.ones(N, dtype=torch.float32, device=dev)
    layer = P.QuantizedLinear("w8a8", K, N, 0, to_dev(qb.astype(np.int8).view(np.uint8).reshape(-1), dev),
                              one_w.view(torch.uint8), torch.ones(K, dtype=torch.float32, device=dev), z, z,
                              None, "bf16", 1.0, 1.0)
    xs = torch.ones(M, dtype=torch.float32, device=dev).view(torch.uint8)
    Y = P.svdq_gemm_w4a4_lowrank_up(layer, to_dev(qa.astype(np.int8).view(np.uint8).reshape(-1), dev), xs, None, M,
                                    out_dtype=torch.float32)
    ref = torch._int_mm(torch.from_numpy(qa).to(dev).to(torch.int8), torch.from_numpy(qb).to(dev).to(torch.int8).t())
    torch.cuda.synchronize()
    assert torch.equal(Y, ref.float())


@pytest.mark.parametrize("name", ["flux_attn_out", "pixart_fc1"])
def test_w8a8_config_layer_sampled(name):
    """Full-size BASELINE-shaped layer at rank 16, sampled rows vs the oracle."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    L = {l.name: l for l in synth.C2 + synth.C4}[name]
    M, K, N, dt = L.M, L.K, L.N, L.dtype
    x, w, lam, ops = make_case("w8a8", M, K, N, 16, dt=dt, seed=7, cfg=41)
    dev = torch.device("cuda")
    layer = layer_from_ops(P, ops, dev, bias_dtype=dt)
    X, xq, xs, xl1 = _k1(P, torch, layer, x, dt, dev)
    Y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, out_dtype=P.TORCH_DTYPE[dt])
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([np.random.default_rng(1).choice(M, 24, replace=False), [0, M - 1]]))
    qa = S.quantize_activation(x[rows], ops)
    np.testing.assert_array_equal(xq.cpu().numpy().reshape(M, K)[rows], qa.codes.astype(np.int8).view(np.uint8))
    y_ref = S.round_output(S.gemm_reference(qa, ops), dt)
    assert rel_fro(Y.float().cpu().numpy()[rows], y_ref) <= 1e-3


def test_w8a8_pair_kernel_forced():
    """The CTA-pair kind::i8 K2 (256 x 192 tiles, separate fp32 low-rank accumulator) on the
    parity cases above, forced for every M > 128 (SVDQ_K2_PAIR=1 is read once per process)."""
    import os, subprocess, sys
    need_cuda()
    env = dict(os.environ, SVDQ_K2_PAIR="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        f"{__file__}::test_w8a8_k1_k2_parity"], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "12 passed" in r.stdout, r.stdout[-500:]      # every parametrization of the parity test ran
