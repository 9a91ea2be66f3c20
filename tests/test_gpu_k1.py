"""K1 parity (svdq_quantize_act_lowrank_down through the C ABI) against the
oracle: codes and scales bit-exact (including the 0x00 padding rows of the
NVFP4 128x4 layout), xl1 within 1e-3 relative Frobenius of the oracle's fp64
X L1s^T rounded to bf16."""
import numpy as np
import pytest

from helpers import layer_from_ops, make_case, need_cuda, pack_act, rel_fro
from oracle import formats as F
from oracle import svdquant as S

pytestmark = pytest.mark.gpu


def run_k1(fmt, M, K, N, r, dt="bf16", seed=0, ldx_pad=0, gs_x=1.0):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    x, w, lam, ops = make_case(fmt, M, K, N, r, dt=dt, seed=seed, gs_x=gs_x)
    dev = torch.device("cuda")
    layer = layer_from_ops(P, ops, dev)
    tdt = P.TORCH_DTYPE[dt]
    Xfull = torch.zeros(M, K + ldx_pad, dtype=tdt, device=dev)
    Xfull[:, :K] = torch.from_numpy(x).to(dev).to(tdt)
    X = Xfull[:, :K]
    xs_size = P.svdq_act_buffer_sizes(fmt, M, K, r)[1]
    xs = torch.full((xs_size,), 0xEE, dtype=torch.uint8, device=dev)     # poison: padding must be written
    xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, X, xs=xs)
    torch.cuda.synchronize()
    qa = S.quantize_activation(x, ops)
    ref_xq, ref_xs = pack_act(fmt, qa, K)
    got_xq = xq.cpu().numpy().reshape(M, K // 2)
    got_xs = xs.cpu().numpy()
    bad = np.argwhere(got_xq != ref_xq)
    assert bad.size == 0, f"{len(bad)} code bytes differ, first at {bad[0]}"
    bad = np.flatnonzero(got_xs != ref_xs.reshape(-1))
    assert bad.size == 0, f"{bad.size} scale bytes differ, first at {bad[0]}"
    if r:
        got = F.bf16_from_bits(xl1.cpu().numpy().view(np.uint16).reshape(M, r))
        ref = F.bf16_from_bits(qa.xl1_bits)
        err = rel_fro(got, ref)
        assert err <= 1e-3, err
        assert rel_fro(got, qa.xl1_exact) <= 5e-3      # bf16 storage rounding only
    return ops, qa


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_k1_c1(fmt):
    run_k1(fmt, 256, 512, 512, 16)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("M", [1, 127, 129, 300])
def test_k1_ragged_rows(fmt, M):
    run_k1(fmt, M, 256, 64, 16, seed=M)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("r", [0, 32, 48, 64, 80, 128])
def test_k1_ranks(fmt, r):
    run_k1(fmt, 160, 1152, 128 if r <= 128 else r, r, seed=r)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_k1_fp16_and_pitch(fmt):
    run_k1(fmt, 200, 640, 128, 32, dt="fp16", ldx_pad=64, seed=3)


def test_k1_k64_minimal():
    run_k1("nvfp4", 33, 64, 16, 16)


def test_k1_nvfp4_static_gs():
    run_k1("nvfp4", 128, 512, 64, 16, gs_x=0.125, seed=9)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_k1_flux_qkv_full(fmt):
    """BASELINE config C4 activation shape (M=4608, K=3072, r=32), bit-exact at full size."""
    run_k1(fmt, 4608, 3072, 64, 32, seed=4)


@pytest.mark.parametrize("fmt,dt,shapes", [
    ("nvfp4", "bf16", [(300, 1152, 32), (64, 1152, 32), (129, 3072, 32)]),
    ("int4", "bf16", [(300, 1152, 32), (64, 1152, 32), (129, 3072, 32)]),
    ("nvfp4", "fp16", [(300, 640, 48), (64, 640, 48)]),
    ("nvfp4", "bf16", [(4096, 1152, 32), (512, 1152, 32)]),     # row tile differs from the single launches
])
def test_k1_grouped_equals_single(fmt, dt, shapes):
    """svdq_quantize_act_lowrank_down_grouped: every problem's codes and scales are bit-identical
    to its own single launch and to the oracle; xl1 bit-identical when the row tile matches, else
    within 1e-3 (fp32 summation order follows the launch's row tile)."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    dev = torch.device("cuda")
    layers, X, outs, refs = [], [], [], []
    for i, (M, K, r) in enumerate(shapes):
        x, w, lam, ops = make_case(fmt, M, K, 128, r, dt=dt, seed=90 + i)
        layers.append(layer_from_ops(P, ops, dev))
        X.append(torch.from_numpy(x).to(dev).to(P.TORCH_DTYPE[dt]))
        bq, bs, bl = P.svdq_act_buffer_sizes(fmt, M, K, r)
        outs.append((torch.zeros(bq, dtype=torch.uint8, device=dev), torch.zeros(bs, dtype=torch.uint8, device=dev),
                     torch.zeros(bl // 2, dtype=torch.int16, device=dev)))
        refs.append((ops, x))
    P.svdq_quantize_act_lowrank_down_grouped(layers, X, [o[0] for o in outs], [o[1] for o in outs],
                                             [o[2] for o in outs])
    torch.cuda.synchronize()
    for i, (M, K, r) in enumerate(shapes):
        sq, ss, sl = P.svdq_quantize_act_lowrank_down(layers[i], X[i])
        torch.cuda.synchronize()
        assert torch.equal(outs[i][0], sq) and torch.equal(outs[i][1], ss)
        same_tile = P.svdq_k1_row_tile(sum((m + 127) // 128 * 128 for m, _, _ in shapes), r) == \
            P.svdq_k1_row_tile((M + 127) // 128 * 128, r)
        if same_tile:
            assert torch.equal(outs[i][2], sl)
        else:
            g = F.bf16_from_bits(outs[i][2].cpu().numpy().view(np.uint16))
            assert rel_fro(g, F.bf16_from_bits(sl.cpu().numpy().view(np.uint16))) <= 1e-3
        ops, x = refs[i]
        qa = S.quantize_activation(x, ops)
        ref_q = F.pack_nibbles(qa.codes if fmt == "nvfp4" else F.int4_to_nibble(qa.codes))
        np.testing.assert_array_equal(sq.cpu().numpy().reshape(M, K // 2), ref_q)


# Every row tile of the row-tile kernel (RT = 16 / 32 / 64 / 128, i.e. Q = 8 / 4 / 2 / 1 K-blocks per
# block-major stage, quantizer rows m and m + RT/2 of one block) -- the tile is the smallest whose
# CTA count fits one wave, so M selects it; ragged M (a partial last tile) and fp16 X included.
@pytest.mark.parametrize("M,dt", [(1000, "bf16"), (2500, "fp16"), (9000, "bf16"), (9700, "fp16")])
def test_k1_every_row_tile(M, dt):
    need_cuda()
    import paper_2411_05007_b200 as P
    rt = P.svdq_k1_row_tile((M + 127) // 128 * 128, 32)
    assert rt in (16, 32, 64, 128)
    run_k1("nvfp4", M, 576, 64, 32, dt=dt, seed=M)


def test_k1_row_tiles_all_reached():
    need_cuda()
    import paper_2411_05007_b200 as P
    got = {P.svdq_k1_row_tile((M + 127) // 128 * 128, 32) for M in (1000, 2500, 9000, 9700)}
    assert got == {16, 32, 64, 128}, got
