"""Per-layer performance on every BASELINE.json configuration:
C2 PixArt-Sigma (fp16, r 32), C3 SDXL (fp16, r 32 + LoRA 16 = 48), C4 FLUX.1 (bf16, r 32),
NVFP4 and INT4, plus the C5 57-block FLUX stack latency at batch 1..8 (19 double + 38
single blocks, measured one block pair per batch as a CUDA graph and scaled by the block
counts -- attention / norms / GELU are not on the linear's hot path and are excluded).

Each layer: K1 -> K2 captured as a CUDA graph, L2 flushed (512 MiB write + 256 MiB read)
before every replay, CUDA events around K1 and K2 separately.  Timing does not depend on the
values, so the stored operands are random valid codes / scales (parity is the tests' job).

    python tools/bench_configs.py [--out profiles/r01/configs_perf.json] [--reps 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_05007_b200 as P  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
TD = {"bf16": torch.bfloat16, "fp16": torch.float16}


def random_layer(fmt, K, N, r, dt, gen):
    bias = (torch.randn(N, device=dev, generator=gen) * 0.1).to(TD[dt])
    L = P.QuantizedLinear.empty(fmt, K, N, r, device=dev, scale_dtype=dt, bias=bias)
    L.w_codes.random_(0, 256, generator=gen)
    if fmt == "nvfp4":
        L.w_scales.random_(0x30, 0x40, generator=gen)
        L.gs_w = 0.01
    elif fmt == "w8a8":
        L.w_scales.view(torch.float32).copy_(torch.rand(N, device=dev, generator=gen) * 0.01 + 0.005)
    else:
        s = (torch.rand(L.w_scales.numel() // 2, device=dev, generator=gen) * 0.01 + 0.005).to(TD[dt])
        L.w_scales.copy_(s.view(torch.uint8))
    if r:
        L.l1s.copy_((torch.randn(L.l1s.numel(), device=dev, generator=gen) * 0.02).to(torch.bfloat16).view(torch.int16))
        L.l2s.copy_((torch.randn(L.l2s.numel(), device=dev, generator=gen) * 0.02).to(torch.bfloat16).view(torch.int16))
    L.lambda_inv.copy_(torch.rand(K, device=dev, generator=gen) + 0.5)
    L._sync_view()
    return L


class Flusher:
    def __init__(self):
        self.buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        self.sink = torch.empty((), dtype=torch.int64, device=dev)

    def __call__(self):
        self.buf.zero_()
        self.sink.copy_(self.buf[: 256 << 20].view(torch.int64).sum())


def time_layers(items, reps, stream, flush):
    """items: list of (layer, X, bufs, M).  Returns per-item (k1_s, k2_s) averaged over reps."""
    ext = lambda: torch.cuda.Event(enable_timing=True, external=True)
    evs = [(ext(), ext(), ext()) for _ in items]

    def run(with_ev):
        for j, (L, X, b, M) in enumerate(items):
            if with_ev:
                evs[j][0].record(stream)
            P.svdq_quantize_act_lowrank_down(L, X, b["xq"], b["xs"], b["xl1"], stream=stream)
            if with_ev:
                evs[j][1].record(stream)
            P.svdq_gemm_w4a4_lowrank_up(L, b["xq"], b["xs"], b["xl1"], M, Y=b["y"], stream=stream)
            if with_ev:
                evs[j][2].record(stream)
    with torch.cuda.stream(stream):
        for _ in range(3):
            run(False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        run(True)
    gp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gp, stream=stream):
        run(False)
    rows = []
    for _ in range(reps):
        with torch.cuda.stream(stream):
            flush()
            g.replay()
        torch.cuda.synchronize()
        rows.append([(a.elapsed_time(b) / 1e3, b.elapsed_time(c) / 1e3) for a, b, c in evs])
    tot = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush()
            a.record(stream)
            gp.replay()
            b.record(stream)
        torch.cuda.synchronize()
        tot.append(a.elapsed_time(b) / 1e3)
    return np.array(rows).mean(axis=0), float(np.mean(tot))


def make_items(layers, fmt, gen, rank_override=None):
    items = []
    for Ly in layers:
        r = Ly.r + Ly.lora if rank_override is None else rank_override
        L = random_layer(fmt, Ly.K, Ly.N, r, Ly.dtype, gen)
        X = torch.randn(Ly.M, Ly.K, device=dev, generator=gen).to(TD[Ly.dtype])
        bq, bs, bl = P.svdq_act_buffer_sizes(fmt, Ly.M, Ly.K, r)
        b = {"xq": torch.empty(bq, dtype=torch.uint8, device=dev), "xs": torch.empty(bs, dtype=torch.uint8, device=dev),
             "xl1": torch.empty(max(bl // 2, 8), dtype=torch.int16, device=dev),
             "y": torch.empty(Ly.M, Ly.N, dtype=TD[Ly.dtype], device=dev)}
        items.append((L, X, b, Ly.M))
    return items


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "configs_perf.json"))
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops_sustained": 1400.0}
    fp4_peak = 4.0 * pk["bf16_tflops_sustained"]
    hbm = pk["hbm_gbs"]
    gen = torch.Generator(device=dev).manual_seed(1)
    stream = torch.cuda.Stream()
    flush = Flusher()
    out = {"peaks": {"fp4_tflops": fp4_peak, "hbm_gbs": hbm, "source": "MEASURED_PEAKS.json (fp4 = 4 x sustained bf16)"},
           "method": "per layer K1 -> K2 CUDA graph, L2 flushed before each replay, CUDA events; random valid operands",
           "configs": {}}
    cfgs = {"C2_pixart_sigma": synth.C2, "C3_sdxl_lora": synth.C3, "C4_flux": synth.C4}
    for cname, layers in cfgs.items():
        for fmt in ("nvfp4", "int4", "w8a8"):
            items = make_items(layers, fmt, gen, rank_override=16 if fmt == "w8a8" else None)
            t, _ = time_layers(items, a.reps, stream, flush)
            items0 = make_items(layers, fmt, gen, rank_override=0)
            t0, _ = time_layers(items0, a.reps, stream, flush)
            rows = {}
            for j, Ly in enumerate(layers):
                M, K, N, r = Ly.M, Ly.K, Ly.N, (16 if fmt == "w8a8" else Ly.r + Ly.lora)
                k1, k2 = t[j]
                k1z, k2z = t0[j]
                fl = 2.0 * M * N * K
                cb = {"nvfp4": 0.5625, "int4": 0.53125, "w8a8": 1.0}[fmt]
                k2_bytes = cb * (M + N) * K + 2 * (M + N) * r + 2 * N + 2 * M * N
                k1_bytes = 2 * M * K + cb * M * K + 2 * M * r
                rows[Ly.name] = {
                    "M": M, "K": K, "N": N, "rank": r, "dtype": Ly.dtype,
                    "k1_us": round(k1 * 1e6, 2), "k2_us": round(k2 * 1e6, 2),
                    "k2_tflops": round(fl / k2 / 1e12, 1), "k2_pct_fp4": round(100 * fl / k2 / 1e12 / fp4_peak, 1),
                    "k2_gbs": round(k2_bytes / k2 / 1e9, 1), "k2_pct_hbm": round(100 * k2_bytes / k2 / 1e9 / hbm, 1),
                    "k2_flop_per_byte": round(fl / k2_bytes, 1),
                    "k1_gbs": round(k1_bytes / k1 / 1e9, 1), "k1_pct_hbm": round(100 * k1_bytes / k1 / 1e9 / hbm, 1),
                    "lowrank_overhead": round((k1 + k2 - k1z - k2z) / k2z, 4),
                    "layer_tflops": round(fl / (k1 + k2) / 1e12, 1),
                }
            out["configs"][f"{cname}/{fmt}"] = rows
            print(cname, fmt, json.dumps(rows), flush=True)
            del items, items0
            torch.cuda.empty_cache()
    # C5: FLUX 57-block stack (19 double + 38 single), batch 1..8, NVFP4
    stack = {}
    for B in (1, 2, 4, 8):
        dbl = make_items(synth.flux_double_block(B), "nvfp4", gen)
        sgl = make_items(synth.flux_single_block(B), "nvfp4", gen)
        _, td = time_layers(dbl, a.reps, stream, flush)
        _, ts = time_layers(sgl, a.reps, stream, flush)
        fl = sum(2.0 * L.M * L.N * L.K for L in synth.flux_double_block(B)) * 19 + \
            sum(2.0 * L.M * L.N * L.K for L in synth.flux_single_block(B)) * 38
        lat = 19 * td + 38 * ts
        stack[f"batch{B}"] = {"double_block_ms": round(td * 1e3, 4), "single_block_ms": round(ts * 1e3, 4),
                              "stack_ms": round(lat * 1e3, 3), "stack_tflops": round(fl / lat / 1e12, 1)}
        print("C5", B, stack[f"batch{B}"], flush=True)
        del dbl, sgl
        torch.cuda.empty_cache()
    out["C5_flux_stack_1gpu"] = {"note": "57 W4A4 block-linear sets (19 double + 38 single); one block of each kind "
                                         "timed as a CUDA graph (K1+K2 per linear, L2 flushed before the block), "
                                         "stack = 19 x double + 38 x single", **stack}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
