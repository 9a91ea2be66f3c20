"""Per-CTA wait-time breakdown of the 1-CTA NVFP4 GEMM (needs SVDQ_LIB=_build_trace/libsvdq.so,
SVDQ_K2_PAIR=0).  Columns: producer waits on free stages, MMA waits on accumulator release,
on SF-slot reuse, on stage data; totals in cycles."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SVDQ_K2_PAIR", "0")
import paper_2411_05007_b200 as P
M, K, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda")
layer = P.QuantizedLinear.empty("nvfp4", K, N, 32, device=dev)
for t in (layer.w_codes, layer.w_scales, layer.l1s, layer.l2s):
    t.zero_()
layer.w_scales.fill_(0x38)
layer.gs_w = 1.0
layer._sync_view()
x = torch.randn(M, K, device=dev).to(torch.bfloat16)
for _ in range(3):
    xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, x)
    y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (148 * 8))()
pair = os.environ.get("SVDQ_K2_PAIR") == "1"
(P.abi.lib().svdq_k2p_trace_read if pair else P.abi.lib().svdq_k2_trace_read)(buf)
if pair:
    t = np.array(buf[:], dtype=np.int64).reshape(148, 8)[:74]
    for i, n in enumerate(["mma_acc_wait", "mma_full_wait", "mma_total", "epi_accfull_wait", "epi_drain",
                           "epi_total", "prod_empty_wait"]):
        print("%-16s median %9.0f  min %9.0f  max %9.0f" % (n, np.median(t[:, i]), t[:, i].min(), t[:, i].max()))
    sys.exit(0)
t = np.array(buf[:], dtype=np.int64).reshape(148, 8)
names = ["prod_empty_wait", "prod_total", "mma_acc_wait", "mma_slot_wait", "mma_full_wait", "mma_total"]
for i, n in enumerate(names):
    print("%-16s median %9.0f  min %9.0f  max %9.0f" % (n, np.median(t[:, i]), t[:, i].min(), t[:, i].max()))
