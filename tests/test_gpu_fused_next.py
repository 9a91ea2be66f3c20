"""Layer-boundary fusion: K2 whose epilogue runs the next layer's K1.
The fused outputs equal K1 of the next layer applied to this layer's stored bf16 output: NVFP4
codes and scale factors (incl. 0x00 padding rows) byte for byte for the identity hand-off; with
GELU (tanh form, reading N1) against K1 of the oracle's bf16(gelu(y)) (fp32 vs fp64 GELU may move
a value across a bf16 rounding boundary: <= 0.1 % of codes); xl1_next within K1's tolerance
(different fp32 summation order); Y itself unchanged; ragged M / N, multi-slot reductions, grouped
problems and the full FLUX MLP-up -> MLP-down shape."""
import numpy as np
import pytest

import synth
from helpers import need_cuda, rel_fro
from oracle import formats as F
from oracle import svdquant as S

pytestmark = pytest.mark.gpu


def _layers(P, torch, K, N, N2, r, r2, seed):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    W = torch.randn(K, N, device=dev, generator=g) / K ** 0.5
    lam = torch.rand(K, device=dev, generator=g) + 0.5
    bias = (torch.randn(N, device=dev, generator=g) * 0.1).to(torch.bfloat16)
    L = P.svdq_quantize_weights(W, lam, r, "nvfp4", bias=bias)
    W2 = torch.randn(N, N2, device=dev, generator=g) / N ** 0.5
    lam2 = torch.rand(N, device=dev, generator=g) * 2 + 0.25
    Nx = P.svdq_quantize_weights(W2, lam2, r2, "nvfp4", gs_x=0.5)
    return L, Nx


def _x(torch, M, K, seed):
    x = F.bf16_round(synth.gen_x(M, K, synth.rng(79, seed, 0)))
    return torch.from_numpy(x).cuda().to(torch.bfloat16)


def _check_case(P, torch, Ls, Nxs, Xs, act, store_y=True, code_tol=0.0):
    ins = [P.svdq_quantize_act_lowrank_down(L, X) for L, X in zip(Ls, Xs)]
    Ms = [X.shape[0] for X in Xs]
    Yref = [P.svdq_gemm_w4a4_lowrank_up(L, *k, M) for L, k, M in zip(Ls, ins, Ms)]
    Ys = [torch.empty_like(y) for y in Yref] if store_y else None
    xq_n, xs_n, xl1_n = P.svdq_gemm_w4a4_lowrank_up_fused_next(
        Ls, [k[0] for k in ins], [k[1] for k in ins], [k[2] for k in ins], Ms, Nxs, act=act, Y=Ys)
    torch.cuda.synchronize()
    for i, (Nx, y, M) in enumerate(zip(Nxs, Yref, Ms)):
        if store_y:
            assert torch.equal(Ys[i], y)
        if act == "none":
            a = y
        else:
            a = torch.from_numpy(S.next_layer_input(y.float().cpu().numpy(), act).astype(np.float32)).cuda().to(torch.bfloat16)
        rq, rs, rl = P.svdq_quantize_act_lowrank_down(Nx, a)
        torch.cuda.synchronize()
        if code_tol == 0.0:
            assert torch.equal(xq_n[i], rq), f"codes differ (problem {i})"
            assert torch.equal(xs_n[i], rs), f"scale factors differ (problem {i})"
        else:
            cq = F.unpack_nibbles(xq_n[i].cpu().numpy().reshape(M, -1))
            cr = F.unpack_nibbles(rq.cpu().numpy().reshape(M, -1))
            assert np.mean(cq != cr) <= code_tol
            assert np.mean(xs_n[i].cpu().numpy() != rs.cpu().numpy()) <= code_tol
        if Nx.rank:
            g = xl1_n[i][: M * Nx.rank].view(torch.bfloat16).float().cpu().numpy()
            ref = rl[: M * Nx.rank].view(torch.bfloat16).float().cpu().numpy()
            assert rel_fro(g, ref) <= 2e-3


@pytest.mark.parametrize("M,K,N,N2,r2", [(300, 256, 320, 128, 32), (64, 128, 192, 64, 16), (1024, 512, 3072, 256, 32),
                                         (2048, 256, 3072, 128, 0), (129, 64, 1024, 192, 32)])
def test_fused_next_identity_bit_exact(M, K, N, N2, r2):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    L, Nx = _layers(P, torch, K, N, N2, 32, r2, seed=M + N)
    _check_case(P, torch, [L], [Nx], [_x(torch, M, K, M)], "none")


def test_fused_next_without_y_store():
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    L, Nx = _layers(P, torch, 256, 384, 128, 32, 32, seed=5)
    _check_case(P, torch, [L], [Nx], [_x(torch, 200, 256, 5)], "none", store_y=False)


def test_fused_next_gelu():
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    L, Nx = _layers(P, torch, 256, 768, 128, 32, 32, seed=6)
    _check_case(P, torch, [L], [Nx], [_x(torch, 384, 256, 6)], "gelu_tanh", code_tol=1e-3)


def test_fused_next_grouped_img_txt():
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    L1, N1 = _layers(P, torch, 256, 768, 128, 32, 32, seed=7)
    L2, N2 = _layers(P, torch, 256, 768, 128, 32, 16, seed=8)
    _check_case(P, torch, [L1, L2], [N1, N2], [_x(torch, 1000, 256, 7), _x(torch, 77, 256, 8)], "none")


def test_fused_next_flux_mlp():
    """FLUX.1 double-block image stream: MLP-up (3072 -> 12288) -> GELU -> MLP-down (12288 -> 3072)."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    L, Nx = _layers(P, torch, 3072, 12288, 3072, 32, 32, seed=9)
    _check_case(P, torch, [L], [Nx], [_x(torch, 4096, 3072, 9)], "gelu_tanh", code_tol=1e-3)


# ---------------------------------------------------------------------------------------------
# Against the ORACLE (VERDICT r1 "next" 1b): oracle operands for both layers, the oracle's K1
# outputs as K2's input, and oracle.fused_next (K1 of next_layer_input(round_output(y64))) as
# the expected hand-off.  The next layer's codes / scale factor of a 16-wide group depend only on
# that group's 16 stored outputs, so they are compared exactly wherever the GPU's stored Y equals
# the oracle's bf16 Y on the whole group (all but rare fp32-vs-fp64 rounding flips); with GELU the
# fp32 (kernel) vs fp64 (oracle) activation may move a value across a bf16 boundary (reading N1):
# <= 0.1 % of those groups may differ.  xl1_next within 2e-3 of the oracle's bf16 X L1s_next^T.
# ---------------------------------------------------------------------------------------------
def _oracle_case(M, K, N, N2, r, r2, seed, gs_x_next):
    from helpers import make_case
    x, w, lam, ops = make_case("nvfp4", M, K, N, r, seed=seed, cfg=31)
    w2 = synth.gen_w(N, N2, synth.rng(31, seed, 6))
    lam2 = S.compute_smoothing(synth.gen_x(256, N, synth.rng(31, seed, 7)), w2, 0.5)
    ops2 = S.prepare_operands(w2, lam2, r2, "nvfp4", gs_x=gs_x_next)
    return x, ops, ops2


@pytest.mark.parametrize("M,K,N,N2,r2,act", [(300, 256, 320, 128, 32, "none"), (129, 128, 1024, 192, 16, "none"),
                                              (384, 256, 768, 128, 32, "gelu_tanh"),
                                              (4096, 3072, 12288, 3072, 32, "gelu_tanh")])
def test_fused_next_vs_oracle(M, K, N, N2, r2, act):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    from helpers import layer_from_ops, pack_act, to_dev
    dev = torch.device("cuda")
    x, ops, ops2 = _oracle_case(M, K, N, N2, 32, r2, seed=M + N2, gs_x_next=0.5)
    L, Nx = layer_from_ops(P, ops, dev), layer_from_ops(P, ops2, dev)
    qa = S.quantize_activation(x, ops)
    q, s = pack_act("nvfp4", qa, K)
    Y = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=dev)
    nq, ns, nl = P.svdq_gemm_w4a4_lowrank_up_fused_next(
        [L], [to_dev(q.reshape(-1), dev)], [to_dev(s.reshape(-1), dev)],
        [to_dev(qa.xl1_bits.view(np.int16).reshape(-1), dev)], [M], [Nx], act=act, Y=[Y])
    torch.cuda.synchronize()
    y64 = S.gemm_reference(qa, ops)
    y_ref = S.round_output(y64, "bf16")
    y = Y.float().cpu().numpy()
    assert rel_fro(y, y_ref) <= 1e-3
    on = S.fused_next(y64, ops2, act)
    same = (y == y_ref).reshape(M, N // 16, 16).all(axis=2)           # [M, groups]
    assert same.mean() > 0.95, f"only {same.mean():.3f} of Y groups bit-equal to the oracle"
    codes = F.unpack_nibbles(nq[0].cpu().numpy().reshape(M, N // 2)).reshape(M, N // 16, 16)
    sf = F.sf_from_layout(ns[0].cpu().numpy(), M, N)
    code_bad = (codes != on.codes.reshape(M, N // 16, 16)).any(axis=2) & same
    sf_bad = (sf != on.scales) & same
    lim = 0 if act == "none" else int(1e-3 * same.sum())
    assert code_bad.sum() <= lim, f"{code_bad.sum()} groups' codes differ"
    assert sf_bad.sum() <= lim, f"{sf_bad.sum()} scale factors differ"
    # padding rows of the 128x4 layout are written 0x00 (reading Q22)
    ref_layout = F.sf_to_layout(on.scales, N).reshape(-1)
    pad = F.sf_to_layout(np.full_like(on.scales, 1), N).reshape(-1) == 0
    assert np.all(ns[0].cpu().numpy()[pad] == ref_layout[pad])
    if r2:
        g = F.bf16_from_bits(nl[0][: M * r2].cpu().numpy().view(np.uint16).reshape(M, r2))
        assert rel_fro(g, F.bf16_from_bits(on.xl1_bits)) <= 2e-3
