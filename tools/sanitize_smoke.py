"""Small K1 / K2 / grouped / INT4 / weight-prep calls for compute-sanitizer (memcheck, racecheck).
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05007_b200 as P
import synth
dev = torch.device("cuda")
for fmt in ("nvfp4", "int4"):
    for (M, K, N, r, dt) in [(200, 640, 208, 32, "bf16"), (129, 6208, 400, 48, "bf16"), (300, 1152, 384, 16, "fp16")]:
        w = synth.gen_w(K, N, synth.rng(5, M, 1))
        lam = np.ones(K, np.float32)
        layer = P.svdq_quantize_weights(torch.from_numpy(w).to(dev), torch.from_numpy(lam).to(dev), r, fmt, dt, 1.0)
        X = torch.randn(M, K, device=dev).to(P.TORCH_DTYPE[dt])
        xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, X)
        Y = P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, out_dtype=P.TORCH_DTYPE[dt])
        torch.cuda.synchronize()
        print(fmt, M, K, N, r, dt, "ok", float(Y.float().abs().mean()))
# grouped
ls, Xs, outs = [], [], []
for i, (M, K, N) in enumerate([(300, 1152, 400), (64, 1152, 208)]):
    w = synth.gen_w(K, N, synth.rng(6, i, 1))
    l = P.svdq_quantize_weights(torch.from_numpy(w).to(dev), torch.ones(K, device=dev), 32, "nvfp4", "bf16", 1.0)
    ls.append(l); Xs.append(torch.randn(M, K, device=dev).to(torch.bfloat16))
    bq, bs, bl = P.svdq_act_buffer_sizes("nvfp4", M, K, 32)
    outs.append((torch.empty(bq, dtype=torch.uint8, device=dev), torch.empty(bs, dtype=torch.uint8, device=dev),
                 torch.empty(bl // 2, dtype=torch.int16, device=dev), torch.empty(M, N, dtype=torch.bfloat16, device=dev)))
P.svdq_quantize_act_lowrank_down_grouped(ls, Xs, [o[0] for o in outs], [o[1] for o in outs], [o[2] for o in outs])
P.svdq_gemm_w4a4_lowrank_up_grouped(ls, [o[0] for o in outs], [o[1] for o in outs], [o[2] for o in outs],
                                    [x.shape[0] for x in Xs], [o[3] for o in outs])
torch.cuda.synchronize()
print("grouped ok")
# layer-boundary fusion (ragged M and N, GELU, grouped), GPTQ, refinement, alpha search
ups, downs, Xs = [], [], []
for i, (M, K, N, N2, r2) in enumerate([(300, 256, 320, 128, 32), (77, 256, 320, 64, 16)]):
    W = torch.randn(K, N, device=dev) / K ** 0.5
    ups.append(P.svdq_quantize_weights(W, torch.rand(K, device=dev) + 0.5, 32, "nvfp4"))
    W2 = torch.randn(N, N2, device=dev) / N ** 0.5
    downs.append(P.svdq_quantize_weights(W2, torch.rand(N, device=dev) + 0.5, r2, "nvfp4"))
    Xs.append(torch.randn(M, K, device=dev).to(torch.bfloat16))
ins = [P.svdq_quantize_act_lowrank_down(L, X) for L, X in zip(ups, Xs)]
Ms = [X.shape[0] for X in Xs]
Ys = [torch.empty(M, L.N, dtype=torch.bfloat16, device=dev) for M, L in zip(Ms, ups)]
P.svdq_gemm_w4a4_lowrank_up_fused_next(ups, [k[0] for k in ins], [k[1] for k in ins], [k[2] for k in ins], Ms, downs,
                                       act="gelu_tanh", Y=Ys)
torch.cuda.synchronize()
print("fused next ok")
Xc = torch.randn(128, 256, device=dev).to(torch.bfloat16)
Wc = torch.randn(256, 192, device=dev) / 16
lam = torch.rand(256, device=dev) + 0.5
for fmt in ("nvfp4", "int4", "w8a8"):
    P.svdq_quantize_weights_gptq(Wc, lam, 16, fmt, Xc)
    P.svdq_refine_lowrank(Xc, Wc, lam, 16, fmt, 2, gptq=fmt != "w8a8")
P.svdq_search_alpha(Xc, Wc, 16, "nvfp4", [0.25, 0.75])
torch.cuda.synchronize()
print("offline ok")
