"""Timeline of CTA 0 of the row-tile K1 (needs SVDQ_LIB=_build_trace/libsvdq.so):
    python tools/trace_k1r.py M K [r]      (COLD=1: L2 flushed before the launch)"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05007_b200 as P
import synth
M, K = int(sys.argv[1]), int(sys.argv[2]); r = int(sys.argv[3]) if len(sys.argv) > 3 else 32
dev = torch.device("cuda")
layer = P.QuantizedLinear.empty("nvfp4", K, 64, r, device=dev)
layer.lambda_inv.fill_(1.0); layer.l1s.zero_(); layer._sync_view()
x = torch.from_numpy(synth.gen_x(M, K, synth.rng(9, 0, 0))).to(dev).to(torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    P.svdq_quantize_act_lowrank_down(layer, x)
torch.cuda.synchronize()
if os.environ.get("COLD", "0") == "1":
    flush.zero_(); flush[: 256 << 20].view(torch.int64).sum()
P.svdq_quantize_act_lowrank_down(layer, x)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 512)()
P.abi.lib().svdq_k1r_trace_read(buf)
t = np.array(buf[:], dtype=np.int64)
rel = lambda i: (t[i] - t[0]) / 1000.0
print("cold" if os.environ.get("COLD") == "1" else "warm", f"M={M} K={K}: setup done {rel(1):.2f} us")
print("stage issue times:", " ".join(f"{rel(2 + i):.2f}" for i in range(64) if t[2 + i] > 0 and t[2 + i] >= t[0]))
print("stage seen by quantizer warp 0:", " ".join(f"{rel(110 + i):.2f}" for i in range(64) if t[110 + i] >= t[0]))
print("L1s issue times:", " ".join(f"{rel(200 + i):.2f}" for i in range(64) if t[200 + i] >= t[0]))
print("MMA passes waits:", " ".join(f"{rel(300 + i):.2f}" for i in range(64) if t[300 + i] >= t[0]))
print("quantizer warps at stage nsteps/2:", " ".join(f"{rel(420 + i):.2f}" for i in range(16)))
print("quantizer warps done:", " ".join(f"{rel(400 + i):.2f}" for i in range(16)))
print(f"tail: sync1 {rel(102):.2f}  dfull {rel(103):.2f}  drained {rel(104):.2f}  sync2 {rel(105):.2f}  stored {rel(101):.2f}")
print(f"quantizer 0 done {rel(100):.2f}  xl1 stored {rel(101):.2f}")
print(f"tail in SM cycles: sync1 -> dfull {t[501] - t[500]}  dfull -> tmem loads done {t[503] - t[501]}  -> drained {t[502] - t[503]}")
