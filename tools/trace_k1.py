"""Dump the K1 timeline of CTA (0,0) (needs SVDQ_LIB=_build_trace/libsvdq.so)."""
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
cold = os.environ.get("COLD", "0") == "1"
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    P.svdq_quantize_act_lowrank_down(layer, x)
torch.cuda.synchronize()
if cold:
    flush.zero_()
    flush[: 256 << 20].view(torch.int64).sum()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
P.svdq_quantize_act_lowrank_down(layer, x)
e1.record()
torch.cuda.synchronize()
print("cold" if cold else "warm", "event time %.2f us" % (e0.elapsed_time(e1) * 1e3))
buf = (ctypes.c_ulonglong * 256)()
P.abi.lib().svdq_k1_trace_read(buf)
t = np.array(buf[:], dtype=np.int64)
t0 = t[0]
rel = lambda i: (t[i] - t0) / 1000.0
print("setup done %.2f us" % rel(1))
for i in range(64):
    if t[2 + i] == 0: break
    print("stage %2d: issue %.2f  seen %.2f  released %.2f" % (i, rel(2 + i), rel(66 + i), rel(130 + i)))
print("quant done %.2f  drained %.2f  cl1 %.2f  reduced %.2f  cl2 %.2f" % tuple(rel(i) for i in (194, 195, 196, 197, 198)))
cta = (ctypes.c_ulonglong * (1024 * 3))()
P.abi.lib().svdq_k1_cta_read(cta)
c = np.array(cta[:], dtype=np.int64).reshape(1024, 3)
n = 1024
c = c[(c[:, 0] > 0) & (c[:, 1] > 0)]
s0 = c[:, 0].min()
st = (c[:, 0] - s0) / 1000.0
en = (c[:, 1] - s0) / 1000.0
print("CTA start: min %.2f med %.2f max %.2f | quant-done: min %.2f med %.2f max %.2f" % (st.min(), np.median(st), st.max(), en.min(), np.median(en), en.max()))
print("start histogram (us):", np.histogram(st, bins=8)[0], np.histogram(st, bins=8)[1].round(1))
print("duration (us): min %.2f med %.2f max %.2f" % ((en - st).min(), np.median(en - st), (en - st).max()))
print("distinct SMs:", len(set(c[:, 2].tolist())))
