"""Run K1 and K2 of one synthetic layer a few times (for ncu / compute-sanitizer).

    python tools/profile_layer.py --M 4096 --K 3072 --N 9216 --r 32 --fmt nvfp4 --iters 3
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05007_b200 as P  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=4096)
ap.add_argument("--K", type=int, default=3072)
ap.add_argument("--N", type=int, default=9216)
ap.add_argument("--r", type=int, default=32)
ap.add_argument("--fmt", default="nvfp4")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda")
w = synth.gen_w(a.K, a.N, synth.rng(9, 0, 1))
xcal = synth.gen_x(256, a.K, synth.rng(9, 0, 2))
lam = (np.max(np.abs(xcal), 0) ** 0.5 / np.max(np.abs(w), 1) ** 0.5).clip(1e-5, 1e5).astype(np.float32)
tdt = P.TORCH_DTYPE[a.dtype]
layer = P.svdq_quantize_weights(torch.from_numpy(w).to(dev), torch.from_numpy(lam).to(dev), a.r, a.fmt,
                                a.dtype, 1.0, bias=torch.zeros(a.N, dtype=tdt, device=dev))
x = torch.from_numpy(synth.gen_x(a.M, a.K, synth.rng(9, 0, 0))).to(dev).to(tdt)
for _ in range(a.iters):
    xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, x)
    y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, a.M, out_dtype=tdt)
torch.cuda.synchronize()
print("ok", y.shape)
