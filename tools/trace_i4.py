"""Per-CTA wait breakdown of the INT4 K2 (needs SVDQ_LIB=_build_trace/libsvdq.so)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05007_b200 as P
M, K, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda")
layer = P.QuantizedLinear.empty("int4", K, N, 32, device=dev)
layer.w_codes.random_(0, 256); layer.w_scales.fill_(0x3c); layer.l1s.zero_(); layer.l2s.zero_()
layer.lambda_inv.fill_(1.0); layer._sync_view()
x = torch.randn(M, K, device=dev).to(torch.bfloat16)
for _ in range(3):
    xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, x)
    y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (148 * 8))()
P.abi.lib().svdq_i4_trace_read(buf)
t = np.array(buf[:], dtype=np.int64).reshape(148, 8)
for i, n in enumerate(["mma_ufull_wait", "mma_gempty_wait", "mma_total", "unp_pfull_wait", "unp_uempty_wait",
                       "unp_total", "epi_gfull_wait", "epi_total"]):
    print("%-16s median %10.0f  min %10.0f  max %10.0f" % (n, np.median(t[:, i]), t[:, i].min(), t[:, i].max()))
