"""K2 parity (svdq_gemm_w4a4_lowrank_up through the C ABI) given the
oracle's quantized operands: Y within 1e-3 relative Frobenius of the oracle's
fp64 result rounded to the output dtype (reading Q17).
Full-size shapes compare sampled rows the oracle computes one by one."""
import numpy as np
import pytest

from helpers import layer_from_ops, make_case, need_cuda, pack_act, rel_fro, to_dev
from oracle import svdquant as S

pytestmark = pytest.mark.gpu


def _subset(qa, rows):
    return S.QuantAct(qa.codes[rows], qa.scales[rows], qa.xl1_bits[rows], qa.xl1_exact[rows])


def run_k2(fmt, M, K, N, r, dt="bf16", out="bf16", seed=0, with_bias=True, sample=None, tol=1e-3):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    x, w, lam, ops = make_case(fmt, M, K, N, r, dt=dt, seed=seed, with_bias=with_bias)
    dev = torch.device("cuda")
    layer = layer_from_ops(P, ops, dev, bias_dtype=dt)
    qa = S.quantize_activation(x, ops)
    xq, xs = pack_act(fmt, qa, K)
    xl1 = to_dev(qa.xl1_bits.view(np.int16).reshape(-1), dev) if r else None
    try:
        Y = P.svdq_gemm_w4a4_lowrank_up(layer, to_dev(xq.reshape(-1), dev), to_dev(xs.reshape(-1), dev),
                                        xl1, M, out_dtype=P.TORCH_DTYPE[out])
    except P.SvdqError as e:
        if e.status == 5 and fmt == "int4":
            pytest.skip("INT4 GEMM not built")
        raise
    torch.cuda.synchronize()
    y = Y.float().cpu().numpy()
    assert np.all(np.isfinite(y))
    rows = np.arange(M) if sample is None else np.unique(np.concatenate(
        [np.random.default_rng(seed).choice(M, sample, replace=False), [0, M - 1]]))
    y_ref = S.round_output(S.gemm_reference(_subset(qa, rows), ops), out)
    err = rel_fro(y[rows], y_ref)
    assert err <= tol, f"rel fro err {err:.3e}"
    exact = np.mean(y[rows] == y_ref)
    return err, exact


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_k2_c1(fmt):
    err, exact = run_k2(fmt, 256, 512, 512, 16)
    assert exact > 0.9         # fp32 accumulation order only flips rare output roundings


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("M,N", [(1, 64), (129, 144), (300, 400), (127, 16)])
def test_k2_ragged(fmt, M, N):
    run_k2(fmt, M, 256, N, 16, seed=M + N)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("r", [0, 48, 64, 128])
def test_k2_ranks(fmt, r):
    run_k2(fmt, 200, 512, 256, r, seed=r)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("K", [64, 192, 1152])
def test_k2_k_tails(fmt, K):
    run_k2(fmt, 130, K, 128 if K > 64 else 64, 16, seed=K)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("out", ["fp16", "fp32"])
def test_k2_out_dtypes(fmt, out):
    run_k2(fmt, 256, 640, 192, 32, dt="fp16", out=out, seed=5)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_k2_no_bias(fmt):
    run_k2(fmt, 96, 256, 128, 16, with_bias=False, seed=6)


def test_k2_nvfp4_wide_tiles():
    """Enough 128x256 tiles to select the BN = 256 kernel."""
    run_k2("nvfp4", 2048, 512, 2560, 32, seed=7, sample=96)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_k2_flux_qkv_full(fmt):
    """BASELINE config C4, FLUX.1 qkv: M=4608, K=3072, N=9216, r=32 (sampled rows)."""
    run_k2(fmt, 4608, 3072, 9216, 32, seed=8, sample=48)


def test_int4_group_accumulators_bit_exact():
    """svdq_debug_int4_group_accum (same kind::i8 path as K2) vs the oracle's exact int64."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    from oracle import formats as F
    rng = np.random.default_rng(3)
    M, N, K = 200, 144, 384
    qa = rng.integers(-7, 8, (M, K))
    qb = rng.integers(-7, 8, (N, K))
    qa[0, :] = 7
    qb[0, :] = 7                # extreme group sums: 64 * 49
    qb[1, :] = -7
    dev = torch.device("cuda")
    try:
        acc = P.svdq_debug_int4_group_accum(to_dev(F.pack_nibbles(F.int4_to_nibble(qa)).reshape(-1), dev),
                                            to_dev(F.pack_nibbles(F.int4_to_nibble(qb)).reshape(-1), dev),
                                            M, N, K)
    except P.SvdqError as e:
        if e.status == 5:
            pytest.skip("INT4 GEMM not built")
        raise
    ref = S.int4_group_accum(qa, qb)
    np.testing.assert_array_equal(acc.cpu().numpy(), ref)


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
@pytest.mark.parametrize("M,K,N,r", [(300, 6208, 400, 48), (257, 6144, 192, 0), (1000, 8192, 3072, 128),
                                     (129, 6400, 208, 16)])
def test_k2_long_k_pair_kernel(fmt, M, K, N, r):
    """K >= 6144 selects the CTA-pair (cta_group::2) NVFP4 kernel: ragged M / N (N not a
    multiple of the 192 tile, second SF atom absent), K tails (K % 256 = 64), ranks 0..128."""
    run_k2(fmt, M, K, N, r, seed=M + K, sample=64 if M > 512 else None)


@pytest.mark.parametrize("shapes", [
    [(4096 // 8, 3072, 9216 // 8, 32), (512 // 8, 3072, 9216 // 8, 32)],          # img / txt stream pair
    [(300, 1152, 400, 48), (129, 640, 208, 16), (1, 256, 64, 0), (513, 6208, 192, 32)],
])
def test_k2_grouped_equals_single(shapes):
    """svdq_gemm_w4a4_lowrank_up_grouped: problem i of one grouped launch is bit-identical to
    its own single launch (same tiles, same per-element K order), and within 1e-3 of the oracle."""
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    dev = torch.device("cuda")
    layers, xq, xs, xl1, Ms, refs, Ys = [], [], [], [], [], [], []
    for i, (M, K, N, r) in enumerate(shapes):
        x, w, lam, ops = make_case("nvfp4", M, K, N, r, seed=70 + i)
        layer = layer_from_ops(P, ops, dev)
        qa = S.quantize_activation(x, ops)
        q, sc = pack_act("nvfp4", qa, K)
        layers.append(layer)
        xq.append(to_dev(q.reshape(-1), dev))
        xs.append(to_dev(sc.reshape(-1), dev))
        xl1.append(to_dev(qa.xl1_bits.view(np.int16).reshape(-1), dev) if r else None)
        Ms.append(M)
        refs.append(S.round_output(S.gemm_reference(qa, ops), "bf16"))
        Ys.append(torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=dev))
    P.svdq_gemm_w4a4_lowrank_up_grouped(layers, xq, xs, xl1, Ms, Ys)
    torch.cuda.synchronize()
    for i in range(len(shapes)):
        single = P.svdq_gemm_w4a4_lowrank_up(layers[i], xq[i], xs[i], xl1[i], Ms[i])
        torch.cuda.synchronize()
        assert torch.equal(Ys[i], single), f"problem {i} differs from its single launch"
        assert rel_fro(Ys[i].float().cpu().numpy(), refs[i]) <= 1e-3


# ---- the opt-in 384-wide CTA-pair tile (SVDQ_K2_BN=384: the launcher reads it once per process)
_BN384_CASES = [(1000, 1536, 768, 32, "bf16"), (300, 6144, 384, 0, "bf16"), (513, 3072, 1152, 48, "fp32")]


@pytest.mark.parametrize("M,K,N,r,out", _BN384_CASES)
def test_k2_bn384_cases(M, K, N, r, out):
    import os
    if os.environ.get("SVDQ_RUN_BN384") != "1":
        pytest.skip("runs in the subprocess of test_k2_bn384_opt_in")
    run_k2("nvfp4", M, K, N, r, out=out, seed=M)


def test_k2_bn384_opt_in():
    import os, subprocess, sys
    need_cuda()
    env = dict(os.environ, SVDQ_K2_BN="384", SVDQ_K2_PAIR="1", SVDQ_RUN_BN384="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        f"{__file__}::test_k2_bn384_cases"], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"{len(_BN384_CASES)} passed" in r.stdout, r.stdout[-500:]
