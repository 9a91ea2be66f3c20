"""K2's L2-banded tile order (large M) covers every output tile exactly once: the same launch with
banding forced on (SVDQ_K2_BAND_MB tiny, so a few 256-row tiles per band, ragged last band,
ragged M / N) and off (SVDQ_K2_BAND_MB=0) gives bit-identical Y, single, grouped and W8A8.  The
unbanded path is itself oracle-checked (test_gpu_k2.py, test_gpu_step_full.py); tile order cannot
change a tile's arithmetic, so equality is the whole contract.  The knob is read once per process,
hence one subprocess per setting."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2411_05007_b200 as P
dev = torch.device("cuda")
out = {}
shapes = [(3000, 1024, 528), (1800, 2048, 768)]      # ragged M (11.7 / 7.0 row tiles), ragged N
layers, xqs, xss, xl1s = [], [], [], []
for i, (M, K, N) in enumerate(shapes):
    g = torch.Generator(device=dev).manual_seed(10 + i)
    layer = P.QuantizedLinear.empty("nvfp4", K, N, 32, device=dev)
    layer.w_codes.random_(0, 256, generator=g)
    layer.w_scales.random_(0x28, 0x38, generator=g)
    layer.l1s.random_(-3000, 3000, generator=g)
    layer.l2s.random_(-3000, 3000, generator=g)
    layer.lambda_inv.uniform_(0.5, 2.0, generator=g)
    layer._sync_view()
    x = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, x)
    y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M)
    out[f"single{i}"] = y.view(torch.int16).cpu().numpy()
    layers.append(layer); xqs.append(xq); xss.append(xs); xl1s.append(xl1)
# W8A8 (kind::i8 pair tiles, 1-byte operands: bands of fewer row tiles)
g = torch.Generator(device=dev).manual_seed(7)
M8, K8, N8 = 2600, 1024, 576
w8 = P.QuantizedLinear.empty("w8a8", K8, N8, 16, device=dev)
w8.w_codes.random_(0, 256, generator=g)
w8.w_scales.view(torch.float32).uniform_(0.001, 0.01, generator=g)
w8.l1s.random_(-3000, 3000, generator=g)
w8.l2s.random_(-3000, 3000, generator=g)
w8.lambda_inv.uniform_(0.5, 2.0, generator=g)
w8._sync_view()
x8 = torch.randn(M8, K8, device=dev, generator=g).to(torch.bfloat16)
q8, s8, l8 = P.svdq_quantize_act_lowrank_down(w8, x8)
out["w8a8"] = P.svdq_gemm_w4a4_lowrank_up(w8, q8, s8, l8, M8).view(torch.int16).cpu().numpy()
ys = [torch.empty(M, N, dtype=torch.bfloat16, device=dev) for (M, K, N) in shapes]
P.svdq_gemm_w4a4_lowrank_up_grouped(layers, xqs, xss, xl1s, [s[0] for s in shapes], ys)
torch.cuda.synchronize()
for i, y in enumerate(ys):
    out[f"grouped{i}"] = y.view(torch.int16).cpu().numpy()
np.savez(sys.argv[2], **out)
'''


def _run(tmp_path, band_mb, name):
    path = tmp_path / f"{name}.npz"
    env = dict(os.environ, SVDQ_K2_BAND_MB=str(band_mb), SVDQ_K2_PAIR="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(path)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


@pytest.mark.gpu
def test_banded_tile_order_bit_identical(tmp_path):
    off = _run(tmp_path, 0, "off")
    on = _run(tmp_path, 0.4, "on")         # 0.4 MB of A per band: 3 / 1 row tiles per band
    assert set(off.files) == set(on.files)
    for k in off.files:
        assert np.array_equal(off[k], on[k]), k
        assert np.any(off[k] != 0), k      # the launch wrote something
