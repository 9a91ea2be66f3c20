"""Layer-boundary fusion timing on the FLUX.1 double block's MLP:
MLP-up (3072 -> 12288) -> GELU -> MLP-down (12288 -> 3072), image (4096 tokens) and text (512)
streams grouped, NVFP4, rank 32.  Compared, each as one CUDA graph with L2 flushed before it:
  unfused : grouped K2(mlp_up) -> Y -> grouped K1(mlp_down)   (GELU itself excluded, as in bench.py)
  fused   : grouped K2(mlp_up) with the next layer's K1 in its epilogue (+ the xl1 reduce), Y stored
  fused_noY: the same without storing Y
and then + grouped K2(mlp_down) for the whole MLP.  Device time from CUDA events.

    python tools/time_fused_next.py [--out profiles/r01/fused_next.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2411_05007_b200 as P  # noqa: E402
from bench_configs import Flusher  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "fused_next.json"))
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--r2", type=int, default=32, help="MLP-down rank (0 drops the fused xl1 work)")
    ap.add_argument("--act", default="gelu_tanh")
    a = ap.parse_args()
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    Ms = [4096, 512]
    ups, downs, X = [], [], []
    for M in Ms:
        W = torch.randn(3072, 12288, device=dev, generator=g) / 3072 ** 0.5
        ups.append(P.svdq_quantize_weights(W, torch.rand(3072, device=dev, generator=g) + 0.5, 32, "nvfp4"))
        W2 = torch.randn(12288, 3072, device=dev, generator=g) / 12288 ** 0.5
        downs.append(P.svdq_quantize_weights(W2, torch.rand(12288, device=dev, generator=g) + 0.5, a.r2, "nvfp4"))
        X.append(torch.randn(M, 3072, device=dev, generator=g).to(torch.bfloat16))
    s = torch.cuda.Stream()
    flush = Flusher()
    k1 = [P.svdq_quantize_act_lowrank_down(L, x) for L, x in zip(ups, X)]
    Y = [torch.empty(M, 12288, dtype=torch.bfloat16, device=dev) for M in Ms]
    bufs = [P.svdq_act_buffer_sizes("nvfp4", M, 12288, a.r2) for M in Ms]
    xq2 = [torch.empty(b[0], dtype=torch.uint8, device=dev) for b in bufs]
    xs2 = [torch.empty(b[1], dtype=torch.uint8, device=dev) for b in bufs]
    xl2 = [torch.empty(max(b[2] // 2, 8), dtype=torch.int16, device=dev) for b in bufs]
    Y2 = [torch.empty(M, 3072, dtype=torch.bfloat16, device=dev) for M in Ms]
    ws = torch.empty(P.svdq_gemm_fused_next_workspace(ups, Ms, downs) + 16, dtype=torch.uint8, device=dev)

    def k2_up():
        P.svdq_gemm_w4a4_lowrank_up_grouped(ups, [k[0] for k in k1], [k[1] for k in k1], [k[2] for k in k1], Ms, Y)

    def k1_down():
        P.svdq_quantize_act_lowrank_down_grouped(downs, Y, xq2, xs2, xl2)

    def fused(store):
        out = P.svdq_gemm_w4a4_lowrank_up_fused_next(ups, [k[0] for k in k1], [k[1] for k in k1], [k[2] for k in k1],
                                                     Ms, downs, act=a.act, Y=Y if store else None, ws=ws,
                                                     out=(xq2, xs2, xl2))
        return out

    fused_out = {}

    def k2_down(src):
        xq, xs, xl = src
        P.svdq_gemm_w4a4_lowrank_up_grouped(downs, xq, xs, xl, Ms, Y2)

    variants = {
        "unfused_k2up_k1down": lambda: (k2_up(), k1_down()),
        "fused_k2up_with_y": lambda: fused(True),
        "fused_k2up_no_y": lambda: fused(False),
        "k2up_only": lambda: k2_up(),
        "k1down_only": lambda: k1_down(),
    }
    res = {}
    for name, fn in variants.items():
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            fn()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                flush()
                e0.record(s)
                gr.replay()
                e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res[name] = {"median_us": round(1e3 * ts[len(ts) // 2], 2), "min_us": round(1e3 * ts[0], 2)}
        print(name, res[name], flush=True)
    out = {"workload": "FLUX.1 double block MLP-up -> GELU -> MLP-down, img 4096 + txt 512 tokens, NVFP4 r32",
           "method": "one CUDA graph per variant, L2 flushed before each replay, CUDA events; median of reps",
           "results": res,
           "saving_us_with_y": round(res["unfused_k2up_k1down"]["median_us"] - res["fused_k2up_with_y"]["median_us"], 2),
           "saving_us_no_y": round(res["unfused_k2up_k1down"]["median_us"] - res["fused_k2up_no_y"]["median_us"], 2)}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
