"""Time K1 alone on one shape: a CUDA graph of 10 launches cycling over distinct DRAM-cold
inputs (back to back), and single launches with an L2 flush (512 MiB write + 256 MiB read)
before each (the bench's condition).
    SVDQ_LIB=... python tools/time_k1.py M K [r]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05007_b200 as P
M, K = int(sys.argv[1]), int(sys.argv[2])
r = int(sys.argv[3]) if len(sys.argv) > 3 else 32
dev = torch.device("cuda")
fmt = os.environ.get("SVDQ_FMT", "nvfp4")
layer = P.QuantizedLinear.empty(fmt, K, 64, r, device=dev)
layer.lambda_inv.fill_(1.0); layer.l1s.zero_(); layer._sync_view()
nb = max(3, int(400e6 // (M * K * 2)) + 1)
xs = [torch.randn(M, K, device=dev).to(torch.bfloat16) for _ in range(nb)]
outs = [P.svdq_quantize_act_lowrank_down(layer, x) for x in xs[:1]]
xq, xsc, xl1 = outs[0]
s = torch.cuda.Stream()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(10):
        P.svdq_quantize_act_lowrank_down(layer, xs[i % nb], xq, xsc, xl1, stream=s)
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1, stream=s):
    P.svdq_quantize_act_lowrank_down(layer, xs[0], xq, xsc, xl1, stream=s)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    g.replay()
    a.record(s); g.replay(); b.record(s)
torch.cuda.synchronize()
us = a.elapsed_time(b) / 10 * 1e3
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
sink = torch.empty((), dtype=torch.int64, device=dev)
tf, tw = [], []
for i in range(10):
    with torch.cuda.stream(s):
        flush.zero_(); sink.copy_(flush[: 256 << 20].view(torch.int64).sum())
        a.record(s); g1.replay(); b.record(s)
    torch.cuda.synchronize()
    tf.append(a.elapsed_time(b) * 1e3)
    with torch.cuda.stream(s):
        a.record(s); g1.replay(); b.record(s)
    torch.cuda.synchronize()
    tw.append(a.elapsed_time(b) * 1e3)
tf = sum(tf) / len(tf); tw = sum(tw) / len(tw)
B = M * K * 2.5625 + 2 * M * r
print(f"K1 {fmt} M={M} K={K} r={r} lib={os.path.basename(os.environ.get('SVDQ_LIB', 'libsvdq.so'))}: "
      f"back-to-back cold {us:.2f} us ({B/us/1e3:.2f} TB/s) | single after flush {tf:.2f} us ({B/tf/1e3:.2f} TB/s) "
      f"| single L2-warm {tw:.2f} us")
