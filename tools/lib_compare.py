"""Our K2 (NVFP4, rank r and rank 0) against the library NVFP4 GEMM (cuBLASLt through
torch._scaled_mm with float4_e2m1fn_x2 operands and e4m3 128x4-swizzled block scales) and
bf16 cuBLAS, on FLUX.1 shapes and 8192^3.  Also checks that K2 at r = 0 agrees with the
library GEMM on the same codes/scales ("Main GEMM with r=0, lambda=1").

    python tools/lib_compare.py [--shapes flux|square|all] [--iters 50]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05007_b200 as P  # noqa: E402

FLUX = [("img_qkv", 4096, 3072, 9216), ("img_proj", 4096, 3072, 3072), ("img_mlp_up", 4096, 3072, 12288),
        ("img_mlp_down", 4096, 12288, 3072), ("txt_qkv", 512, 3072, 9216), ("txt_mlp_down", 512, 12288, 3072),
        ("single_linear1", 4608, 3072, 21504), ("single_linear2", 4608, 15360, 3072)]
SQUARE = [("sq8192", 8192, 8192, 8192), ("sq16384", 16384, 16384, 16384)]


def time_graph(fn, iters, stream):
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(iters):
            fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        g.replay()
        a.record(stream)
        g.replay()
        b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3   # us (L2-warm weights when they fit)


def layer_random(M, K, N, r, dev, gen):
    layer = P.QuantizedLinear.empty("nvfp4", K, N, r, device=dev)
    layer.w_codes.random_(0, 256, generator=gen)
    # scale bytes 0x30..0x3f (e4m3 0.5 .. 0.94), padding included (never read by either GEMM)
    layer.w_scales.random_(0x30, 0x40, generator=gen)
    if r:
        layer.l1s.copy_((torch.randn(r * K, device=dev, generator=gen) * 0.02).to(torch.bfloat16).view(torch.int16))
        layer.l2s.copy_((torch.randn(N * r, device=dev, generator=gen) * 0.02).to(torch.bfloat16).view(torch.int16))
    layer.lambda_inv.fill_(1.0)
    layer.gs_w = 1.0
    layer._sync_view()
    return layer


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="all")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--r", type=int, default=32)
    a = ap.parse_args()
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(0)
    stream = torch.cuda.Stream()
    shapes = {"flux": FLUX, "square": SQUARE, "all": FLUX + SQUARE}[a.shapes]
    out = []
    for name, M, K, N in shapes:
        row = {"shape": name, "M": M, "K": K, "N": N}
        x = torch.randn(M, K, device=dev, generator=gen).to(torch.bfloat16)
        for r in (a.r, 0):
            layer = layer_random(M, K, N, r, dev, gen)
            xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, x)
            y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
            us = time_graph(lambda: P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, Y=y, stream=stream),
                            a.iters, stream)
            row[f"k2_r{r}_us"] = round(us, 2)
            row[f"k2_r{r}_tflops"] = round(2 * M * N * K / us / 1e6, 1)
            us1 = time_graph(lambda: P.svdq_quantize_act_lowrank_down(layer, x, xq, xs, xl1, stream=stream),
                             a.iters, stream)
            row[f"k1_r{r}_us"] = round(us1, 2)
        # library NVFP4 on the rank-0 operands (same codes and scales)
        try:
            fa = xq.view(torch.uint8).reshape(M, K // 2).view(torch.float4_e2m1fn_x2)
            fb = layer.w_codes.view(torch.uint8).reshape(N, K // 2).view(torch.float4_e2m1fn_x2)
            sa = xs.view(torch.float8_e4m3fn)
            sb = layer.w_scales.view(torch.float8_e4m3fn)
            yl = torch._scaled_mm(fa, fb.t(), sa, sb, out_dtype=torch.bfloat16)
            us = time_graph(lambda: torch._scaled_mm(fa, fb.t(), sa, sb, out_dtype=torch.bfloat16), a.iters, stream)
            row["cublas_nvfp4_us"] = round(us, 2)
            row["cublas_nvfp4_tflops"] = round(2 * M * N * K / us / 1e6, 1)
            P.svdq_gemm_w4a4_lowrank_up(layer, xq, xs, xl1, M, Y=y)
            torch.cuda.synchronize()
            d = (y.float() - yl.float()).norm() / yl.float().norm()
            row["k2_r0_vs_cublas_rel_fro"] = float(d)
        except Exception as e:  # noqa: BLE001
            row["cublas_nvfp4_error"] = f"{type(e).__name__}: {str(e)[:200]}"
        xb = torch.randn(M, K, device=dev, generator=gen).to(torch.bfloat16)
        wb = torch.randn(K, N, device=dev, generator=gen).to(torch.bfloat16)
        us = time_graph(lambda: torch.matmul(xb, wb), max(5, a.iters // 5), stream)
        row["cublas_bf16_tflops"] = round(2 * M * N * K / us / 1e6, 1)
        if r == 0 and f"k2_r{a.r}_us" in row and "k1_r0_us" in row:
            row["lowrank_overhead"] = round((row[f"k1_r{a.r}_us"] + row[f"k2_r{a.r}_us"] - row["k1_r0_us"]
                                             - row["k2_r0_us"]) / row["k2_r0_us"], 4)
        print(json.dumps(row), flush=True)
        out.append(row)
        del x, xb, wb
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
