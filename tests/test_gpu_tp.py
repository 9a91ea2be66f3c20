"""Single-GPU emulation of the tensor-parallel path: the P column
shards run one after another through the real kernels; concatenated they must equal the
unsharded output bit for bit (every output column depends only on its own operands, and
the per-element K order does not depend on the N tiling)."""
import numpy as np
import pytest

from helpers import layer_from_ops, make_case, need_cuda

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
@pytest.mark.parametrize("P_,N", [(2, 1536), (4, 3072), (8, 3072), (3, 480)])
def test_sharded_equals_unsharded(fmt, P_, N):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    from paper_2411_05007_b200 import tp
    M, K, r = 384, 1024, 32
    x, w, lam, ops = make_case(fmt, M, K, N, r, seed=P_, cfg=23)
    dev = torch.device("cuda")
    full = layer_from_ops(P, ops, dev)
    X = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    y_full = full(X)
    parts = []
    for rank in range(P_):
        shard = tp.shard_layer(full, P_, rank)
        parts.append(shard(X))
    y_cat = torch.cat(parts, dim=1)
    torch.cuda.synchronize()
    assert torch.equal(y_cat.view(torch.int16), y_full.view(torch.int16))


# ---------------------------------------------------------------------------------------------
# Variant 2 (SURVEY 8(e) "quantize, then gather"), single-GPU emulation of P ranks: each rank's
# K1 runs on its K-slice of the input, the packed slices are concatenated (what
# all_gather_into_tensor leaves on every rank), every rank assembles the full K1 outputs and runs
# K2 on its N-shard.  Codes / scales equal the unsharded K1's bit for bit; xl1 (partials summed in
# rank order) within the K1 tolerance; every rank assembles identical bytes; Y vs the oracle.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("P_,M,K,N,r", [(2, 384, 1024, 1536, 32), (4, 300, 3072, 1024, 32), (8, 129, 3072, 512, 16),
                                        (3, 200, 576, 480, 0), (8, 256, 12288, 384, 32)])
def test_variant2_emulated(fmt, P_, M, K, N, r):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    from paper_2411_05007_b200 import tp
    from helpers import pack_act, rel_fro
    from oracle import formats as F
    from oracle import svdquant as S
    x, w, lam, ops = make_case(fmt, M, K, N, r, seed=P_ + K, cfg=24)
    dev = torch.device("cuda")
    full = layer_from_ops(P, ops, dev)
    X = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    ranks = [tp.ColumnParallelSVDQLinear(full, world=P_, rank=p) for p in range(P_)]
    kp = K // P_
    slices = [ranks[p].quantize_slice(X[:, p * kp:(p + 1) * kp].contiguous()).clone() for p in range(P_)]
    gathered = torch.cat(slices)
    outs, ys = [], []
    for p in range(P_):
        xq, xs, xl1 = ranks[p].assemble(gathered, M)
        outs.append((xq.clone(), xs.clone(), xl1.clone()))
        ys.append(P.svdq_gemm_w4a4_lowrank_up(ranks[p].local, xq, xs, xl1 if r else None, M))
    torch.cuda.synchronize()
    for o in outs[1:]:                          # (xl1 is not written at rank 0)
        assert all(torch.equal(a, b) for a, b in zip(o[:3 if r else 2], outs[0])), "ranks assembled different bytes"
    sq, ss, sl = P.svdq_quantize_act_lowrank_down(full, X)
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], sq), "codes differ from the unsharded K1"
    assert torch.equal(outs[0][1], ss), "scales differ from the unsharded K1"
    qa = S.quantize_activation(x, ops)
    ref_q, ref_s = pack_act(fmt, qa, K)
    np.testing.assert_array_equal(outs[0][0].cpu().numpy().reshape(M, K // 2), ref_q)
    if r:
        g = F.bf16_from_bits(outs[0][2][: M * r].cpu().numpy().view(np.uint16).reshape(M, r))
        assert rel_fro(g, F.bf16_from_bits(qa.xl1_bits)) <= 1e-3
    y = torch.cat(ys, dim=1).float().cpu().numpy()
    y_ref = S.round_output(S.gemm_reference(qa, ops), "bf16")
    assert rel_fro(y, y_ref) <= 1e-3


def test_variant2_rejects_w8a8_and_bad_slices():
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    from paper_2411_05007_b200 import tp
    with pytest.raises(ValueError):
        tp.kslice_bounds(3072, 5, 0)
    with pytest.raises(P.SvdqError) as e:
        P.svdq_tp_slice_sizes("w8a8", 64, 384, 16)
    assert e.value.status == 5


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("world,M,K,r", [(4, 200, 3072, 32), (8, 129, 3072, 16), (2, 300, 1152, 0)])
def test_fused_gather_emulated(fmt, world, M, K, r):
    """Fused packed all-gather, P ranks emulated on one GPU: rank p's K-sliced K1
    stores into all P gather buffers (local stand-ins for the symmetric-memory peers); afterwards every
    buffer's xq / xs equal the unsharded K1's bit for bit and the reduced xl1 equals the all-gather
    path's (svdq_tp_assemble_act) bit for bit."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    from paper_2411_05007_b200 import tp
    x, w, lam, ops = make_case(fmt, M, K, 256, r, seed=11 + world, cfg=26)
    dev = torch.device("cuda")
    full = layer_from_ops(P, ops, dev)
    X = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    kp = K // world
    oq, os_, op, nb = P.svdq_tp_gather_sizes(fmt, M, K, r, world)
    bufs = [torch.full((nb,), 0xAB, dtype=torch.uint8, device=dev) for _ in range(world)]
    slices = []
    for p in range(world):
        xsh = X[:, p * kp:(p + 1) * kp].contiguous()
        P.svdq_quantize_act_lowrank_down_kslice_fused(full, p * kp, xsh, world, p, [b.data_ptr() for b in bufs])
        slices.append(P.svdq_quantize_act_lowrank_down_kslice(full, p * kp, xsh).clone())
    sq, ss, sl = P.svdq_quantize_act_lowrank_down(full, X)
    aq, as_, al = P.svdq_tp_assemble_act(fmt, world, M, K, r, torch.cat(slices))
    torch.cuda.synchronize()
    bq, bs, _ = P.svdq_act_buffer_sizes(fmt, M, K, r)
    for b in bufs:
        assert torch.equal(b[oq:oq + bq], sq), "codes differ from the unsharded K1"
        assert torch.equal(b[os_:os_ + bs], ss), "scales differ from the unsharded K1"
        if r:
            xl1 = torch.empty(M * r, dtype=torch.int16, device=dev)
            P.svdq_tp_reduce_partials(world, M, r, b[op:op + world * M * r * 4], xl1)
            torch.cuda.synchronize()
            assert torch.equal(xl1, al[:M * r]), "xl1 differs from the all-gather path's"
