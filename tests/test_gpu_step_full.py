"""The bench's exact step, oracle-checked at full size (VERDICT r1 "next" 1a).

bench.py times one FLUX.1-dev double block (image stream 4096 tokens + text stream 512 tokens:
qkv, proj, MLP up, MLP down) plus one single block (4608 tokens: linear1, linear2), rank 32,
NVFP4, bf16 (BASELINE config C4), as the launch sequence `bench.flux_step_grouped`: one grouped
K1 + one grouped K2 per double-block kind, single launches for the single block.  This test runs
that same function on operands prepared by the ORACLE (oracle.svdquant.prepare_operands: fp64
LAPACK SVD, residual quantization) and compares EVERY row:
  * every activation code byte and every scale-factor byte (incl. the 0x00 padding rows of the
    128x4 layout) bit-exact;
  * xl1 [M, r] within 1e-3 relative Frobenius of the oracle's bf16 xl1;
  * Y [M, N] end to end within 1e-3 relative Frobenius of the oracle's fp64 result rounded to
    bf16 (reading Q17), every row within 5e-3, and no row left unwritten (Y starts as NaN).
"""
import numpy as np
import pytest

import synth
from helpers import layer_from_ops, need_cuda, pack_act, rel_fro
from oracle import formats as F
from oracle import svdquant as S

pytestmark = pytest.mark.gpu


def _oracle_layer(L, i):
    """Layer i of the bench step with the bench's seeds (synth.rng(4, i, t)); lambda(alpha = 0.5)
    from the oracle, operands from the oracle's weight preparation."""
    x = F.bf16_round(synth.gen_x(L.M, L.K, synth.rng(4, i, 0)))
    w = synth.gen_w(L.K, L.N, synth.rng(4, i, 1))
    lam = S.compute_smoothing(F.bf16_round(synth.gen_x(256, L.K, synth.rng(4, i, 2))), w, 0.5)
    bias = F.bf16_round(synth.gen_bias(L.N, synth.rng(4, i, 3)))
    ops = S.prepare_operands(w, lam, L.r, "nvfp4", gs_x=1.0, bias=bias)
    return x, ops


def test_bench_step_full_size_every_row():
    need_cuda()
    import torch
    import bench
    import paper_2411_05007_b200 as P

    dev = torch.device("cuda")
    layers = bench.flux_block_layers(1)
    built, host = [], []
    for i, L in enumerate(layers):
        x, ops = _oracle_layer(L, i)
        layer = layer_from_ops(P, ops, dev)
        bq, bs, bl = P.svdq_act_buffer_sizes("nvfp4", L.M, L.K, L.r)
        bufs = dict(x=torch.from_numpy(x).to(dev).to(torch.bfloat16),
                    xq=torch.full((bq,), 0xEE, dtype=torch.uint8, device=dev),
                    xs=torch.full((bs,), 0xEE, dtype=torch.uint8, device=dev),
                    xl1=torch.zeros(max(bl // 2, 8), dtype=torch.int16, device=dev),
                    y=torch.full((L.M, L.N), float("nan"), dtype=torch.bfloat16, device=dev))
        built.append((L, layer, bufs))
        host.append((x, ops))
    stream = torch.cuda.Stream(device=dev)
    groups = []
    with torch.cuda.stream(stream):
        bench.flux_step_grouped(P, built, stream, launch_groups=groups)
    torch.cuda.synchronize()
    assert len(groups) == 6 and sum(len(g) for g in groups) == len(layers)   # the bench's 6 + 6 launches

    for (L, layer, b), (x, ops) in zip(built, host):
        qa = S.quantize_activation(x, ops)
        ref_q, ref_s = pack_act("nvfp4", qa, L.K)
        got_q = b["xq"].cpu().numpy().reshape(L.M, L.K // 2)
        bad = np.argwhere(got_q != ref_q)
        assert bad.size == 0, f"{L.name}: {len(bad)} code bytes differ, first at {bad[0]}"
        got_s = b["xs"].cpu().numpy()
        bad = np.flatnonzero(got_s != ref_s.reshape(-1))
        assert bad.size == 0, f"{L.name}: {bad.size} scale bytes differ, first at {bad[0]}"
        xl1 = F.bf16_from_bits(b["xl1"][: L.M * L.r].cpu().numpy().view(np.uint16).reshape(L.M, L.r))
        assert rel_fro(xl1, F.bf16_from_bits(qa.xl1_bits)) <= 1e-3, L.name
        y = b["y"].float().cpu().numpy()
        assert np.all(np.isfinite(y)), f"{L.name}: rows left unwritten"
        y_ref = S.round_output(S.gemm_reference(qa, ops), "bf16")
        err = rel_fro(y, y_ref)
        d = np.linalg.norm((y - y_ref).astype(np.float64), axis=1)
        row_err = d / np.maximum(np.linalg.norm(y_ref.astype(np.float64), axis=1), 1e-30)
        assert err <= 1e-3, f"{L.name}: rel fro {err:.3e}"
        assert row_err.max() <= 5e-3, f"{L.name}: row {int(row_err.argmax())} rel err {row_err.max():.3e}"
        del qa, y, y_ref
