"""Time K2 alone on one FLUX shape (CUDA-graph replay of 20 launches); for A/B experiments.
    SVDQ_LIB=... SVDQ_K2_PAIR=0|1 python tools/time_k2.py M K N"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05007_b200 as P
M, K, N = (int(a) for a in sys.argv[1:4])
dev = torch.device("cuda")
fmt = os.environ.get("SVDQ_FMT", "nvfp4")
layer = P.QuantizedLinear.empty(fmt, K, N, 32, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
layer.w_codes.random_(0, 256, generator=g)
if fmt == "w8a8":
    layer.w_scales.view(torch.float32).fill_(0.01)
else:
    layer.w_scales.fill_(0x30 if fmt == "nvfp4" else 0x3c)
layer.l1s.zero_(); layer.l2s.zero_(); layer.lambda_inv.fill_(1.0)
layer.gs_w = 1.0
layer._sync_view()
x = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, x)
y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, Y=y, stream=s)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    for _ in range(20):
        P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, Y=y, stream=s)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    gr.replay()
    a.record(s)
    gr.replay()
    b.record(s)
torch.cuda.synchronize()
us = a.elapsed_time(b) / 20 * 1e3
print(f"{fmt} M={M} K={K} N={N} pair={os.environ.get('SVDQ_K2_PAIR', '1')} lib={os.path.basename(os.environ.get('SVDQ_LIB', 'libsvdq.so'))}: {us:.2f} us  {2*M*N*K/us/1e6:.1f} TFLOP/s")
