"""Benchmark of the fused W4A4 + low-rank linear (BASELINE.json metric:
"fused W4A4+low-rank linear TFLOPS (% FP4 peak); FLUX.1 block latency").

A step = the W4A4 linears of one FLUX.1-dev double block (image stream at
4096 tokens, text stream at 512 tokens: qkv, proj, MLP up, MLP down) and one
single block (4608 tokens: linear1 3072->21504, linear2 15360->3072), rank
32, NVFP4, bf16 activations -- BASELINE config C4.  Each linear is K1
(svdq_quantize_act_lowrank_down) followed by K2 (svdq_gemm_w4a4_lowrank_up).
TFLOPS counts 2*M*N*K per linear (the low-rank FLOPs are overhead).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl svdq|reference]

N > 1 (torchrun, NCCL): by default the step runs TENSOR PARALLEL over the ranks
(BASELINE config C5; column-parallel over N, Variant 2 packed
all-gathers where a layer's input is the previous column-parallel output;
strong scaling, value = the step's FLOPs / max-over-ranks time); --mode
replicas runs an independent copy of the step per GPU instead (weak scaling).
Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "fused W4A4+low-rank linear TFLOPS (% FP4 peak); FLUX.1 block latency"
UNIT = "TFLOP/s"


def flux_block_layers(batch=1):
    return synth.flux_double_block(batch) + synth.flux_single_block(batch)


def config_layers(args):
    """The step's linears: FLUX.1 block pair (C4, default), a PixArt-Sigma block's linears (C2,
    fp16, 4096 tokens per image) or an SDXL attention/FF set (C3, fp16, CFG batch 2, rank 32 + LoRA
    16), token counts scaled by --batch."""
    import dataclasses
    if args.config == "flux":
        return flux_block_layers(args.batch)
    base = synth.C2 if args.config == "pixart" else synth.C3
    return [dataclasses.replace(L, M=L.M * args.batch) for L in base]


def eff_rank(L):
    """Rank of the deployed low-rank branch: r, plus the LoRA rank concatenated into it."""
    return L.r + L.lora


WORKLOADS = {
    "flux": "flux1-dev block linears: 1 double block (img 4096 tok + txt 512 tok: qkv, proj, mlp_up, mlp_down) "
            "+ 1 single block (4608 tok: linear1, linear2)",
    "pixart": "pixart-sigma 1024px block linears (4096 tok: qkv, attn_out, cross_q, cross_out, fc1, fc2), fp16",
    "sdxl": "sdxl 1024px attention/FF linears, CFG batch 2 (8192 tok at 640 ch, 2048 tok at 1280 ch), fp16, "
            "rank 32 + LoRA 16",
}


def bench_config(args, world):
    """The workload description shared by both arms (svdq and --impl reference)."""
    dims = {"flux": (3072, 12288), "pixart": (1152, 4608), "sdxl": (640, 5120)}[args.config]
    rank = 16 if args.fmt == "w8a8" else (48 if args.config == "sdxl" else 32)
    return {"workload": WORKLOADS[args.config], "config": args.config,
            "batch": args.batch, "hidden": dims[0], "mlp": dims[1], "rank": rank, "format": args.fmt,
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
            "l2": "flushed between steps outside the per-step events (512 MiB write, then a 256 MiB read "
                  "so the flush's dirty lines are written back before the step starts)"}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return p, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


KINDS = ["qkv", "proj", "mlp_up", "mlp_down", "single_linear1", "single_linear2"]


def flux_step_grouped(P, bl, st, ev1=None, ev2=None, launch_groups=None):
    """The timed step's launch sequence (also run by tests/test_gpu_step_full.py): the double
    block's image- and text-stream linears of the same kind (qkv, proj, MLP up, MLP down) as ONE
    grouped K1 and ONE grouped K2 launch each (independent problems; a FLUX double block's two
    streams share no linear); the single block's linears alone.  `bl` = [(Layer, QuantizedLinear,
    buffers dict with x / xq / xs / xl1 / y)]; ev1 / ev2 = per-launch (start, end) event pairs."""
    by = {L.name: (L, layer, b) for (L, layer, b) in bl}
    for kind in ("qkv", "proj", "mlp_up", "mlp_down"):
        grp = [by[f"double_{s_}_{kind}"] for s_ in ("img", "txt") if f"double_{s_}_{kind}" in by]
        if not grp:
            continue
        if ev1 is not None:
            ev1[KINDS.index(kind)][0].record(st)
        P.svdq_quantize_act_lowrank_down_grouped([g_[1] for g_ in grp], [g_[2]["x"] for g_ in grp],
                                                 [g_[2]["xq"] for g_ in grp], [g_[2]["xs"] for g_ in grp],
                                                 [g_[2]["xl1"] for g_ in grp], stream=st)
        if ev1 is not None:
            ev1[KINDS.index(kind)][1].record(st)
            ev2[KINDS.index(kind)][0].record(st)
        P.svdq_gemm_w4a4_lowrank_up_grouped([g_[1] for g_ in grp], [g_[2]["xq"] for g_ in grp],
                                            [g_[2]["xs"] for g_ in grp], [g_[2]["xl1"] for g_ in grp],
                                            [g_[0].M for g_ in grp], [g_[2]["y"] for g_ in grp], stream=st)
        if ev2 is not None:
            ev2[KINDS.index(kind)][1].record(st)
        if launch_groups is not None:
            launch_groups.append([g_[0] for g_ in grp])
    for (L, layer, b) in bl:
        if L.name.startswith("single"):
            if ev1 is not None:
                ev1[KINDS.index(L.name)][0].record(st)
            P.svdq_quantize_act_lowrank_down(layer, b["x"], b["xq"], b["xs"], b["xl1"], stream=st)
            if ev1 is not None:
                ev1[KINDS.index(L.name)][1].record(st)
                ev2[KINDS.index(L.name)][0].record(st)
            P.svdq_gemm_w4a4_lowrank_up(layer, b["xq"], b["xs"], b["xl1"], L.M, Y=b["y"], stream=st)
            if ev2 is not None:
                ev2[KINDS.index(L.name)][1].record(st)
            if launch_groups is not None:
                launch_groups.append([L])


def _nbytes(t):
    return 0 if t is None else t.numel() * t.element_size()


def b2b_slope(torch, stream, l2_flush, nrep, launch, copies):
    """Seconds per launch of `launch(j)` (j = copy index): CUDA events on `stream` around graphs of
    R and 2R back-to-back launches cycling over the copies, L2 flushed before each replay;
    (median t_2R - median t_R) / R."""
    ev = lambda: torch.cuda.Event(enable_timing=True)
    R = max(8, copies)
    graphs = []
    for n in (R, 2 * R):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            for j in range(n):
                launch(j % copies)
        graphs.append(gr)
    t = [[], []]
    for _ in range(nrep):
        for k, gr in enumerate(graphs):
            a, b = ev(), ev()
            with torch.cuda.stream(stream):
                l2_flush()
                a.record(stream)
                gr.replay()
                b.record(stream)
            torch.cuda.synchronize()
            t[k].append(a.elapsed_time(b))
    return (float(np.median(t[1])) - float(np.median(t[0]))) / R / 1e3


def b2b_cold_durations(P, torch, units, stream, l2_flush, nrep, l2_bytes=126 << 20):
    """Per-launch durations of each unit's K1 and K2 launch, back to back and DRAM-cold.

    A unit is the list of (Layer, QuantizedLinear, buffers) one launch covers (a grouped launch or a
    single linear).  For each kernel: C copies of everything the launch reads (K1: X; K2: codes,
    scale factors, L2s, xq / xs / xl1), C chosen so the copies span >= 3x the 126 MB L2, so every
    launch reads its operands from DRAM as in the flushed step.  Two CUDA graphs of R and 2R
    launches cycling over the copies are timed with CUDA events on the launch stream (L2 flushed
    before each replay); duration = (t_2R - t_R) / R, which removes the graph-launch and event
    overhead of a replay and keeps what the step keeps: launches queued back to back (PDL lets a
    launch's prologue overlap its predecessor's tail, as between K1 and K2 in the step)."""
    import math

    def slope(launch, copies):
        return b2b_slope(torch, stream, l2_flush, nrep, launch, copies)

    out = []
    for unit in units:
        grouped = len(unit) > 1
        # ---- K1: copies of X
        xin = sum(_nbytes(b["x"]) for (_, _, b) in unit)
        c1 = int(min(16, max(2, math.ceil(3 * l2_bytes / xin))))
        xc = [[b["x"].clone() for (_, _, b) in unit] for _ in range(c1)]

        def k1(j):
            if grouped:
                P.svdq_quantize_act_lowrank_down_grouped([u[1] for u in unit], xc[j], [u[2]["xq"] for u in unit],
                                                         [u[2]["xs"] for u in unit], [u[2]["xl1"] for u in unit],
                                                         stream=stream)
            else:
                (L, layer, b), = unit
                P.svdq_quantize_act_lowrank_down(layer, xc[j][0], b["xq"], b["xs"], b["xl1"], stream=stream)
        with torch.cuda.stream(stream):
            k1(0)
        torch.cuda.synchronize()
        t1 = slope(k1, c1)
        del xc
        # ---- K2: copies of the weights and of K1's outputs
        win = sum(_nbytes(l.w_codes) + _nbytes(l.w_scales) + _nbytes(l.l2s) + _nbytes(b["xq"]) + _nbytes(b["xs"])
                  + _nbytes(b["xl1"]) for (_, l, b) in unit)
        c2 = int(min(16, max(2, math.ceil(3 * l2_bytes / win))))
        cp = []
        for _ in range(c2):
            cp.append([(P.QuantizedLinear(l.fmt, l.K, l.N, l.rank, l.w_codes.clone(), l.w_scales.clone(),
                                          l.lambda_inv, l.l1s, l.l2s.clone(), l.bias, l.scale_dtype, l.gs_w, l.gs_x),
                        b["xq"].clone(), b["xs"].clone(), b["xl1"].clone()) for (_, l, b) in unit])

        def k2(j):
            c = cp[j]
            if grouped:
                P.svdq_gemm_w4a4_lowrank_up_grouped([e[0] for e in c], [e[1] for e in c], [e[2] for e in c],
                                                    [e[3] for e in c], [u[0].M for u in unit],
                                                    [u[2]["y"] for u in unit], stream=stream)
            else:
                (L, _, b), = unit
                P.svdq_gemm_w4a4_lowrank_up(c[0][0], c[0][1], c[0][2], c[0][3], L.M, Y=b["y"], stream=stream)
        with torch.cuda.stream(stream):
            k2(0)
        torch.cuda.synchronize()
        t2 = slope(k2, c2)
        del cp
        torch.cuda.empty_cache()
        out.append((t1, t2))
    return out


# ------------------------------------------------------------------ svdq arm
def build_layers(P, torch, layers, fmt, dev, quality=None, seed_index=None):
    """Synthetic FLUX-shaped layers (DESIGN.md input recipe), weights prepared on the GPU
    by svdq_quantize_weights (fp64 Gram + eigensolver SVD, residual quantization).  Layer i draws
    from synth.rng(4, i, t); `seed_index` overrides i for a one-layer list."""
    out = []
    for i, L in enumerate(layers):
        if seed_index is not None:
            i = seed_index
        g = torch.Generator(device="cpu").manual_seed(4000 + i)
        td = torch.float16 if L.dtype == "fp16" else torch.bfloat16
        w = synth.gen_w(L.K, L.N, synth.rng(4, i, 1))
        xcal = torch.from_numpy(synth.gen_x(256, L.K, synth.rng(4, i, 2))).to(dev).to(td)
        w_d = torch.from_numpy(w).to(dev)
        # lambda(alpha = 0.5) (App. D) from the library's offline alpha search on a one-point grid
        _, lam, _ = P.svdq_search_alpha(xcal, w_d, L.r, fmt, [0.5], scale_dtype=L.dtype)
        bias = torch.from_numpy(synth.gen_bias(L.N, synth.rng(4, i, 3))).to(dev).to(td)
        layer = P.svdq_quantize_weights(w_d, lam, L.r, fmt, L.dtype, 1.0, bias=bias)
        if L.lora:                                   # LoRA by concatenation into L1 / L2
            a, b_ = synth.gen_lora(L.K, L.N, L.lora, synth.rng(4, i, 4), synth.rng(4, i, 5))
            layer = P.svdq_lora_fuse(layer, torch.from_numpy(a).to(dev), torch.from_numpy(b_).to(dev))
        x = torch.from_numpy(synth.gen_x(L.M, L.K, synth.rng(4, i, 0))).to(dev).to(td)
        if quality is not None:
            # unscored sanity metric: ||XW + b - Y|| / ||XW + b|| on 64 rows, fp64 reference
            rows = torch.arange(0, L.M, max(1, L.M // 64), device=dev)[:64]
            y_s = P.svdq_linear_forward(layer, x[rows].contiguous()).double()
            ref = x[rows].double() @ torch.from_numpy(w).to(dev).double() + bias.double()
            if L.lora:
                ref = ref + x[rows].double() @ (torch.from_numpy(a).to(dev).double() @ torch.from_numpy(b_).to(dev).double())
            quality[L.name] = round(float((y_s - ref).norm() / ref.norm()), 5)
        bq, bs, bl = P.svdq_act_buffer_sizes(fmt, L.M, L.K, layer.rank)
        bufs = dict(
            x=x,
            xq=torch.empty(bq, dtype=torch.uint8, device=dev),
            xs=torch.empty(bs, dtype=torch.uint8, device=dev),
            xl1=torch.empty(max(bl // 2, 8), dtype=torch.int16, device=dev),
            y=torch.empty(L.M, L.N, dtype=td, device=dev),
        )
        out.append((L, layer, bufs))
        del w, g
    torch.cuda.synchronize()
    return out


def run_svdq(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2411_05007_b200 as P

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    layers = config_layers(args)
    if args.fmt == "w8a8":                      # the paper's 8-bit setting uses rank 16
        import dataclasses
        layers = [dataclasses.replace(L, r=16, lora=0) for L in layers]
    quality = {}
    built = build_layers(P, torch, layers, args.fmt, dev, quality)
    flops = sum(2.0 * L.M * L.N * L.K for L in layers)
    cbytes = {"nvfp4": 0.5625, "int4": 0.53125, "w8a8": 1.0}[args.fmt]
    k1_bytes = sum(L.M * L.K * (2 + cbytes) + L.M * eff_rank(L) * 2 for L in layers)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush_sink = torch.empty((), dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def l2_flush():
        flush.zero_()
        flush_sink.copy_(flush[: 256 << 20].view(torch.int64).sum())

    def step(bl, st, k1_events=None, k2_events=None, only=None):
        for j, (L, layer, b) in enumerate(bl):
            if only != "k2":
                if k1_events is not None:
                    k1_events[j][0].record(st)
                P.svdq_quantize_act_lowrank_down(layer, b["x"], b["xq"], b["xs"], b["xl1"], stream=st)
                if k1_events is not None:
                    k1_events[j][1].record(st)
            if only != "k1":
                if k2_events is not None:
                    k2_events[j][0].record(st)
                P.svdq_gemm_w4a4_lowrank_up(layer, b["xq"], b["xs"], b["xl1"], L.M, Y=b["y"], stream=st)
                if k2_events is not None:
                    k2_events[j][1].record(st)

    ext = lambda: torch.cuda.Event(enable_timing=True, external=True)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    side = torch.cuda.Stream(device=dev)

    def step_dag(bl, st):
        """The block's dependency structure: a FLUX double block's image and text streams
        share no linear until the joint attention (not on this path), so their W4A4 linears
        run concurrently on two streams; the single block follows the join."""
        fork, join = torch.cuda.Event(), torch.cuda.Event()
        fork.record(st)
        side.wait_event(fork)
        for (L, layer, b) in bl:
            s_ = side if L.name.startswith("double_txt") else st
            if L.name.startswith("single"):
                continue
            P.svdq_quantize_act_lowrank_down(layer, b["x"], b["xq"], b["xs"], b["xl1"], stream=s_)
            P.svdq_gemm_w4a4_lowrank_up(layer, b["xq"], b["xs"], b["xl1"], L.M, Y=b["y"], stream=s_)
        join.record(side)
        st.wait_event(join)
        for (L, layer, b) in bl:
            if L.name.startswith("single"):
                P.svdq_quantize_act_lowrank_down(layer, b["x"], b["xq"], b["xs"], b["xl1"], stream=st)
                P.svdq_gemm_w4a4_lowrank_up(layer, b["xq"], b["xs"], b["xl1"], L.M, Y=b["y"], stream=st)

    def step_grouped(bl, st, ev1=None, ev2=None):
        flux_step_grouped(P, bl, st, ev1, ev2, launch_groups if ev1 is None else None)

    kinds = KINDS
    launch_groups = []                  # layers covered by each launch of the grouped step

    def capture(bl):
        """CUDA graphs of one step: plain (timed region), with external timing events around
        every launch (per-kernel durations), K1-only and K2-only."""
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                step(bl, stream)
        torch.cuda.synchronize()
        g = {"k1_ev": [(ext(), ext()) for _ in bl], "k2_ev": [(ext(), ext()) for _ in bl]}
        for name in ("plain", "ev", "k1", "k2"):
            g[name] = torch.cuda.CUDAGraph()
        n0 = P.svdq_launch_count()
        with torch.cuda.graph(g["plain"], stream=stream):
            step(bl, stream)
        g["launches"] = P.svdq_launch_count() - n0
        g["dag"] = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g["dag"], stream=stream):
            step_dag(bl, stream)
        g["grouped"] = None
        if args.fmt == "nvfp4" and args.config == "flux":
            with torch.cuda.stream(stream):
                step_grouped(bl, stream)
            torch.cuda.synchronize()
            n1 = P.svdq_launch_count()
            g["grouped"] = torch.cuda.CUDAGraph()
            launch_groups.clear()
            with torch.cuda.graph(g["grouped"], stream=stream):
                step_grouped(bl, stream)
            g["launches_grouped"] = P.svdq_launch_count() - n1
            g["gk1_ev"] = [(ext(), ext()) for _ in kinds]
            g["gk2_ev"] = [(ext(), ext()) for _ in kinds]
            g["grouped_ev"] = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g["grouped_ev"], stream=stream):
                step_grouped(bl, stream, g["gk1_ev"], g["gk2_ev"])
        with torch.cuda.graph(g["ev"], stream=stream):
            step(bl, stream, g["k1_ev"], g["k2_ev"])
        with torch.cuda.graph(g["k1"], stream=stream):
            step(bl, stream, only="k1")
        with torch.cuda.graph(g["k2"], stream=stream):
            step(bl, stream, only="k2")
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                g["plain"].replay()
        torch.cuda.synchronize()
        return g

    def time_graph(gr, n):
        tot = []
        for _ in range(n):
            a, b = ev(), ev()
            with torch.cuda.stream(stream):
                l2_flush()
                a.record(stream)
                gr.replay()
                b.record(stream)
            torch.cuda.synchronize()
            tot.append(a.elapsed_time(b))
        return float(np.mean(tot))

    def per_kernel(g, n):
        k1_rows, k2_rows = [], []
        for _ in range(n):
            with torch.cuda.stream(stream):
                l2_flush()
                g["ev"].replay()
            torch.cuda.synchronize()
            k1_rows.append([a.elapsed_time(b) for a, b in g["k1_ev"]])
            k2_rows.append([a.elapsed_time(b) for a, b in g["k2_ev"]])
        return np.array(k1_rows).mean(axis=0) / 1e3, np.array(k2_rows).mean(axis=0) / 1e3   # seconds

    g = capture(built)
    step_ev = [(ev(), ev()) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        with torch.cuda.stream(stream):
            for s in range(args.steps):
                l2_flush()                          # L2 flush (outside the per-step events)
                step_ev[s][0].record(stream)
                (g["grouped"] or g["dag"]).replay()
                step_ev[s][1].record(stream)
        torch.cuda.synchronize()
    launches = (g["launches_grouped"] if g["grouped"] is not None else g["launches"]) * args.steps
    if world > 1:
        dist.barrier()
    total_ms = float(sum(a.elapsed_time(b) for a, b in step_ev))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    nrep = max(3, min(args.steps, 20))
    k1_avg_s, k2_avg_s = per_kernel(g, nrep)
    # the step's own launches (grouped): roofline `achieved` is measured on these
    launch_k1_s = launch_k2_s = None
    if g["grouped"] is not None:
        r1, r2 = [], []
        for _ in range(nrep):
            with torch.cuda.stream(stream):
                l2_flush()
                g["grouped_ev"].replay()
            torch.cuda.synchronize()
            r1.append([a.elapsed_time(b) for a, b in g["gk1_ev"]])
            r2.append([a.elapsed_time(b) for a, b in g["gk2_ev"]])
        launch_k1_s = np.array(r1).mean(axis=0) / 1e3
        launch_k2_s = np.array(r2).mean(axis=0) / 1e3
    # back-to-back DRAM-cold durations of the step's own launches (the roofline's denominators)
    by_name = {L.name: (L, layer, b) for (L, layer, b) in built}
    units = ([[by_name[L.name] for L in grp] for grp in launch_groups] if g["grouped"] is not None
             else [[e] for e in built])
    b2b = b2b_cold_durations(P, torch, units, stream, l2_flush, nrep)
    only_ms = {"k1": time_graph(g["k1"], nrep), "k2": time_graph(g["k2"], nrep),
               "serial": time_graph(g["plain"], nrep), "dag": time_graph(g["dag"], nrep),
               "grouped": time_graph(g["grouped"], nrep) if g["grouped"] is not None else None}

    # ---------------- low-rank overhead: the same step at rank 0
    lowrank = None
    if rank == 0 and not args.no_extras:
        layers0 = [synth.Layer(L.name, L.M, L.K, L.N, 0, L.dtype, 0) for L in layers]
        built0 = build_layers(P, torch, layers0, args.fmt, dev)
        g0 = capture(built0)
        step0_ms = time_graph(g0["plain"], nrep)
        step_r_ms = time_graph(g["plain"], nrep)
        k1_0, k2_0 = per_kernel(g0, nrep)
        lowrank = {
            "value": round((step_r_ms - step0_ms) / (time_graph(g0["k2"], nrep)), 4),
            "def": "[t_step(r=32) - t_step(r=0)] / t_K2-only(r=0), CUDA-graph replays, L2 flushed "
                   "(SURVEY 8(d): [t_K1(r)+t_K2(r)-t_K1(0)-t_K2(0)] / t_K2(0))",
            "step_ms_r32": round(step_r_ms, 4), "step_ms_r0": round(step0_ms, 4),
            "per_layer_isolated": {L.name: round(float((k1_avg_s[j] + k2_avg_s[j] - k1_0[j] - k2_0[j]) / k2_0[j]), 4)
                                   for j, L in enumerate(layers)},
        }
        # per launch of the step, from back-to-back DRAM-cold durations (b2b_cold_durations)
        by0 = {L.name: (L, layer, b) for (L, layer, b) in built0}
        b2b0 = b2b_cold_durations(P, torch, [[by0[u[0].name] for u in unit] for unit in units], stream, l2_flush, nrep)
        lowrank["per_launch"] = {"+".join(u[0].name for u in unit): round((t1 + t2 - z1 - z2) / z2, 4)
                                 for unit, (t1, t2), (z1, z2) in zip(units, b2b, b2b0)}
        lowrank["per_launch_def"] = ("[t_K1(r) + t_K2(r) - t_K1(0) - t_K2(0)] / t_K2(0) per launch of the step, "
                                     "back-to-back DRAM-cold durations")
        # ---------------- library context: cuBLASLt NVFP4 GEMM alone on the rank-0 operands
        library = None
        if args.fmt == "nvfp4" and hasattr(torch, "float4_e2m1fn_x2"):
            try:
                mm = []
                for (L, layer, b) in built0:
                    fa = b["xq"].reshape(L.M, L.K // 2).view(torch.float4_e2m1fn_x2)
                    fb = layer.w_codes.reshape(L.N, L.K // 2).view(torch.float4_e2m1fn_x2)
                    mm.append((fa, fb.t(), b["xs"].view(torch.float8_e4m3fn),
                               layer.w_scales.view(torch.float8_e4m3fn), b["y"]))
                lev = [(ext(), ext()) for _ in mm]

                def lib_step(events=None):
                    for j, (fa, fbt, sa, sb, y) in enumerate(mm):
                        if events is not None:
                            events[j][0].record(stream)
                        torch._scaled_mm(fa, fbt, sa, sb, out_dtype=torch.bfloat16)
                        if events is not None:
                            events[j][1].record(stream)
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        lib_step()
                torch.cuda.synchronize()
                gl = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gl, stream=stream):
                    lib_step(lev)
                rows = []
                for _ in range(nrep):
                    with torch.cuda.stream(stream):
                        l2_flush()
                        gl.replay()
                    torch.cuda.synchronize()
                    rows.append([a.elapsed_time(b) for a, b in lev])
                lib_s = np.array(rows).mean(axis=0) / 1e3
                k2f = np.array([2.0 * L.M * L.N * L.K for L in layers])
                # the same back-to-back DRAM-cold method as K2's roofline durations, per layer
                import math
                lib_b2b = []
                for (fa, fbt, sa, sb, y) in mm:
                    nb = _nbytes(fa) + _nbytes(fbt) + _nbytes(sa) + _nbytes(sb)
                    c = int(min(16, max(2, math.ceil(3 * (126 << 20) / nb))))
                    cps = [(fa.clone(), fbt.t().clone().t(), sa.clone(), sb.clone()) for _ in range(c)]
                    lib_b2b.append(b2b_slope(torch, stream, l2_flush, nrep,
                                             lambda j, cps=cps, y=y: torch._scaled_mm(*cps[j], out_dtype=torch.bfloat16),
                                             c))
                    del cps
                lib_b2b = np.array(lib_b2b)
                library = {
                    "kernel": "cuBLASLt block-scaled NVFP4 GEMM (torch._scaled_mm), plain Q(X)Q(W) only: "
                              "no smoothing, quantization, low-rank branch or bias",
                    "tflops": round(float(k2f.sum() / lib_b2b.sum() / 1e12), 1),
                    "tflops_def": "per-layer back-to-back DRAM-cold durations (bench.b2b_slope), as K2's roofline",
                    "per_layer_tflops": {L.name: round(float(k2f[j] / lib_b2b[j] / 1e12), 1)
                                         for j, L in enumerate(layers)},
                    "tflops_isolated": round(float(k2f.sum() / lib_s.sum() / 1e12), 1),
                    "k2_r0_tflops_isolated": round(float(k2f.sum() / k2_0.sum() / 1e12), 1),
                }
            except Exception as e:  # noqa: BLE001  (context only; never part of the product path)
                library = {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}
        lowrank["library_context"] = library
        # ---------------- unfused pipeline (the paper's Fig. 5(a)): K1(r=0) + K2(r=0) + the
        # low-rank branch as two separate cuBLAS bf16 GEMMs and an add, vs the fused step
        try:
            lr = []
            for (L, l32, b32), (_, l0, b0) in zip(built, built0):
                td = b32["x"].dtype
                l1 = l32.l1s.view(torch.bfloat16).reshape(l32.rank, L.K).to(td)
                l2 = l32.l2s.view(torch.bfloat16).reshape(L.N, l32.rank).to(td)
                lr.append((L, l0, b0, l1, l2, torch.empty(L.M, l32.rank, dtype=td, device=dev)))

            def unfused_step():
                for (L, l0, b0, l1, l2, xl1u) in lr:
                    P.svdq_quantize_act_lowrank_down(l0, b0["x"], b0["xq"], b0["xs"], b0["xl1"], stream=stream)
                    P.svdq_gemm_w4a4_lowrank_up(l0, b0["xq"], b0["xs"], b0["xl1"], L.M, Y=b0["y"], stream=stream)
                    torch.matmul(b0["x"], l1.t(), out=xl1u)                # X L1s^T   (re-reads X)
                    b0["y"].addmm_(xl1u, l2.t(), alpha=l0.gs_x * l0.gs_w)   # + xl1 L2s^T (re-reads / writes Y)
            with torch.cuda.stream(stream):
                unfused_step()
            torch.cuda.synchronize()
            gu = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gu, stream=stream):
                unfused_step()
            t_unf = time_graph(gu, nrep)
            lowrank["unfused_fig5a"] = {
                "step_ms_unfused": round(t_unf, 4), "step_ms_fused": round(step_r_ms, 4),
                "fused_speedup": round(t_unf / step_r_ms, 3),
                "lowrank_overhead_unfused": round((t_unf - step0_ms) / step0_ms, 4),
                "lowrank_overhead_fused": round((step_r_ms - step0_ms) / step0_ms, 4),
                "paper": "57 % for the naive rank-32 branch (Fig. 5(a) caption, P:165); ~50 % of the 4-bit "
                         "branch latency (P:173)",
                "def": "K1(r=0) + K2(r=0) + cuBLAS bf16 X.L1s^T + cuBLAS addmm xl1.L2s^T into Y, per linear, serial graph"}
        except Exception as e:  # noqa: BLE001  (context only)
            lowrank["unfused_fig5a"] = {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}
        del built0, g0
        torch.cuda.empty_cache()

    # ---------------- end to end through the public API with host buffers
    hx = [b["x"].cpu().pin_memory() for (_, _, b) in built]
    hy = [torch.empty(b["y"].shape, dtype=b["y"].dtype, pin_memory=True) for (_, _, b) in built]
    ws = [torch.empty(P.abi.forward_workspace_bytes(layer, L.M), dtype=torch.uint8, device=dev)
          for (L, layer, _) in built]
    h2d = sum(x.numel() * x.element_size() for x in hx)
    d2h = sum(y.numel() * y.element_size() for y in hy)

    # host <-> device copies on their own streams (PCIe is full duplex): layer j+1's input upload
    # and layer j-1's result download overlap layer j's compute
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    e_in = [torch.cuda.Event() for _ in built]
    e_cmp = [torch.cuda.Event() for _ in built]

    def e2e_step():
        for j, (L, layer, b) in enumerate(built):
            with torch.cuda.stream(s_in):
                b["x"].copy_(hx[j], non_blocking=True)
                e_in[j].record(s_in)
            stream.wait_event(e_in[j])
            P.svdq_linear_forward(layer, b["x"], Y=b["y"], ws=ws[j], stream=stream)
            e_cmp[j].record(stream)
            s_out.wait_event(e_cmp[j])
            with torch.cuda.stream(s_out):
                hy[j].copy_(b["y"], non_blocking=True)
        s_out.synchronize()
        stream.synchronize()

    for _ in range(max(1, args.warmup)):
        e2e_step()
    if world > 1:
        dist.barrier()
    e0, e1 = ev(), ev()
    e0.record(stream)
    s_in.wait_event(e0)                     # the first upload starts inside the timed interval
    n_e2e = max(3, min(args.steps, 20))
    for _ in range(n_e2e):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    if rank != 0:
        return None
    pk, pk_kind = peaks()
    # guide nominal ratios: fp4 = 4 x bf16 (9 : 2.25 PF), int8 / fp8 = 2 x bf16 (4.5 : 2.25)
    ratio = 4.0 if args.fmt == "nvfp4" else 2.0
    fp4_sus = ratio * pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    fp4_burst = ratio * pk["bf16_tflops"]
    k2_flops = np.array([2.0 * L.M * L.N * L.K for L in layers])
    k2_t = float(sum(t2 for _, t2 in b2b))
    k1_t = float(sum(t1 for t1, _ in b2b))
    k2_achieved = float(k2_flops.sum() / k2_t / 1e12)
    k1_gbs = float(k1_bytes / k1_t / 1e9)
    iso_k2 = launch_k2_s.sum() if launch_k2_s is not None else k2_avg_s.sum()
    iso_k1 = launch_k1_s.sum() if launch_k1_s is not None else k1_avg_s.sum()
    per_launch = []
    iso = (list(zip(launch_k1_s, launch_k2_s)) if launch_k2_s is not None
           else list(zip(k1_avg_s, k2_avg_s)))
    for unit, (t1, t2), (i1, i2) in zip(units, b2b, iso):
        fl = sum(2.0 * u[0].M * u[0].N * u[0].K for u in unit)
        by = sum(u[0].M * u[0].K * (2 + cbytes) + 2 * u[0].M * eff_rank(u[0]) for u in unit)
        per_launch.append({"layers": [u[0].name for u in unit], "k1_us": round(t1 * 1e6, 2),
                           "k2_us": round(t2 * 1e6, 2), "k2_tflops": round(fl / t2 / 1e12, 1),
                           "k1_gbs": round(by / t1 / 1e9, 1),
                           "k1_us_isolated": round(float(i1 * 1e6), 2), "k2_us_isolated": round(float(i2 * 1e6), 2)})
    value = world * flops * args.steps / (total_ms / 1e3) / 1e12
    per_layer = {L.name: {"M": L.M, "K": L.K, "N": L.N,
                          "k1_us": round(float(k1_avg_s[j] * 1e6), 2),
                          "k2_us": round(float(k2_avg_s[j] * 1e6), 2),
                          "k2_tflops": round(float(k2_flops[j] / k2_avg_s[j] / 1e12), 1),
                          "k1_gbs": round(float((L.M * L.K * (2 + cbytes)
                                                 + 2 * L.M * eff_rank(L)) / k1_avg_s[j] / 1e9), 1)}
                 for j, L in enumerate(layers)}
    traffic = None                     # ncu DRAM bytes per K2 launch: captured for the NVFP4 FLUX step only
    tpath = os.path.join(ROOT, "profiles", "k2_traffic.json")
    if os.path.exists(tpath) and args.fmt == "nvfp4" and args.config == "flux" and args.batch == 1:
        traffic = json.load(open(tpath)).get("bytes_per_launch")
    clocks = clk.summary()
    f_sm = (clocks.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)) * 1e6
    cfg = bench_config(args, world)
    cfg["block_latency_ms"] = round(total_ms / args.steps, 4)
    return {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": {
            "nvfp4": "e2m1 x e2m1 -> f32 (NVFP4 g16 e4m3 scales) + bf16 low-rank",
            "int4": "int4 x int4 -> int32 (kind::i8) -> f32 (g64 16-bit scales) + bf16 low-rank",
            "w8a8": "int8 x int8 -> int32 (kind::i8, per-token / per-channel fp32 scales) + bf16 low-rank r16"}[args.fmt],
        "data": "synthetic (seeded; DESIGN.md input recipe), weights prepared on GPU by svdq_quantize_weights",
        "config": cfg,
        "roofline": {"bound": "tensor", "achieved": round(k2_achieved, 1), "peak": round(fp4_burst, 1),
                     "unit": "TFLOP/s", "frac": round(k2_achieved / fp4_burst, 4), "traffic": traffic,
                     "kernel": f"svdq_gemm_w4a4_lowrank_up (K2, {args.fmt.upper()})",
                     "peak_source": (f"4 x {pk_kind} BURST bf16 (MEASURED_PEAKS.json), guide fp4:bf16 = 9:2.25; "
                                     "burst because each K2 launch is timed alone in a sub-ms graph replay"
                                     if args.fmt == "nvfp4" else
                                     f"2 x {pk_kind} BURST bf16 (MEASURED_PEAKS.json): the kind::i8 dense "
                                     "rate, guide int8:bf16 = 4.5:2.25"),
                     "frac_vs_sustained": round(k2_achieved / fp4_sus, 4),
                     "frac_vs_clock_peak": round(k2_achieved * 1e12 / (148 * 8192 * ratio * f_sm), 4),
                     "clock_peak_def": f"148 SMs x {int(8192 * ratio)} dense FLOP/clk ({args.fmt}) x median SM clock "
                                       "of the timed region",
                     "achieved_def": "sum 2*M*N*K over the step's linears / sum of the step's K2 launch durations; "
                                     "each duration = CUDA events (launch stream) around graphs of R and 2R "
                                     "back-to-back launches of that launch on DRAM-cold operand copies, "
                                     "(t_2R - t_R) / R (bench.b2b_cold_durations)",
                     "achieved_isolated": round(float(k2_flops.sum() / iso_k2 / 1e12), 1),
                     "isolated_def": "same FLOPs / durations from events around each single launch of the step "
                                     "sequence (includes each launch's event + launch gap)"},
        "k1": {"bound": "hbm", "achieved": round(k1_gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
               "frac": round(k1_gbs / pk["hbm_gbs"], 4),
               "achieved_def": "sum (2MK + c MK + 2Mr) / sum of K1 launch durations (back-to-back DRAM-cold, "
                               "as for K2)",
               "achieved_isolated": round(float(k1_bytes / iso_k1 / 1e9), 1)},
        "kernel_sum_ms": {"k1": round(k1_t * 1e3, 4), "k2": round(k2_t * 1e3, 4),
                          "total": round((k1_t + k2_t) * 1e3, 4),
                          "note": "sum of the back-to-back per-launch durations; compare with ms_per_step"},
        "lowrank_overhead": lowrank,
        "quality_rel_err_vs_fp64_XW": {"note": "unscored sanity metric: ||XW + b - Y|| / ||XW + b||, 64 rows per "
                                               "linear, synthetic outlier activations (SURVEY 8(d))", **quality},
        "per_launch": per_launch,
        "per_layer": per_layer,
        "e2e": {"value": round(world * flops * n_e2e / (e2e_ms / 1e3) / 1e12, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": round(e2e_ms / n_e2e, 3),
                "path": "svdq_linear_forward (C ABI) per linear; pinned host X in, Y out on separate copy "
                        "streams (uploads / downloads overlap other linears' compute)"},
        "graph_only_ms": {"k1_all_layers": round(only_ms["k1"], 4), "k2_all_layers": round(only_ms["k2"], 4),
                          "step_serial": round(only_ms["serial"], 4), "step_img_txt_concurrent": round(only_ms["dag"], 4),
                          "step_img_txt_grouped": round(only_ms["grouped"], 4) if only_ms["grouped"] else None,
                          "note": "each kernel's launches replayed back to back as one graph (L2 flushed before)"},
        "gpu_launches": int(launches),
        "timing": ("step captured once as a CUDA graph and replayed per step: the double block's image- and "
                   "text-stream linears of each kind run as one grouped K1 + one grouped K2 launch (12 launches "
                   "per step; INT4: two graph branches, 20 launches); per-kernel times from a second, serial "
                   "graph of single launches with external timing events around each launch") if args.config == "flux"
                  else ("step captured once as a CUDA graph of K1 -> K2 per linear in model order; per-kernel times "
                        "from a second graph with external timing events around each launch"),
        "clocks": clocks,
    }


# ------------------------------------------------------------------ tensor-parallel arm (C5)
# Layers whose input is the output of a column-parallel predecessor (attention-out input, MLP-down
# input after GELU, single-block linear2 input): the rank holds only its K-shard of the input and
# the layer runs SURVEY 8(e) Variant 2 (K1 on the slice, one packed all-gather, assemble, K2 on the
# N-shard).  The other inputs (qkv, MLP-up, linear1: from the norm of the replicated residual
# stream; attention / norms / GELU are pre-generated inputs) are replicated, so
# their K1 runs on every rank and K2 on the shard.  Outputs stay N-sharded.
SHARDED_INPUT = ("proj", "mlp_down", "linear2")


def run_tp(args, rank, world, local_rank, backend):
    import torch
    import torch.distributed as dist
    import paper_2411_05007_b200 as P
    from paper_2411_05007_b200 import tp

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    layers = flux_block_layers(args.batch)
    # --tp-emulate P (one GPU): rank 0's share of a P-way TP step -- its shards, K-slices and the
    # assembly of P slices -- with the gather replaced by a local copy of this rank's slice; the
    # NVLink transfer is MODELED below (a projection, labelled as such)
    emulate = args.tp_emulate if world == 1 and args.tp_emulate > 1 else 0
    shard_world, shard_rank = (emulate, 0) if emulate else (world, rank)
    net = []
    for i, L in enumerate(layers):
        (_, full, b), = build_layers(P, torch, [L], args.fmt, dev, seed_index=i)
        cp = tp.ColumnParallelSVDQLinear(full, world=shard_world, rank=shard_rank)
        sharded = L.name.endswith(SHARDED_INPUT)
        n = cp.local.N
        e = dict(L=L, cp=cp, sharded=sharded, y=torch.empty(L.M, n, dtype=torch.bfloat16, device=dev))
        if sharded:
            k0, kp = tp.kslice_bounds(L.K, shard_world, shard_rank)
            e["x"] = b["x"][:, k0:k0 + kp].contiguous()
            nb = P.svdq_tp_slice_sizes(args.fmt, L.M, kp, L.r)[3]
            e["slice"] = torch.empty(nb, dtype=torch.uint8, device=dev)
            e["k0"] = k0
        else:
            e["x"] = b["x"]
        e["xq"], e["xs"], e["xl1"] = b["xq"], b["xs"], b["xl1"]
        del full, b
        net.append(e)
    torch.cuda.synchronize()
    by = {e["L"].name: e for e in net}
    groups = [[by[f"double_{s_}_{k}"] for s_ in ("img", "txt")] for k in ("qkv", "proj", "mlp_up", "mlp_down")]
    groups += [[by["single_linear1"]], [by["single_linear2"]]]
    # one packed all-gather per sharded group: the img and txt slices travel together.  --tp-gather
    # fused: no collective -- K1 stores each slice into every rank's symmetric-memory buffer
    # (SURVEY 8(f) row 2), then one device-side barrier (CUDA IPC + host barrier for gloo tests)
    gbuf, sgs = {}, {}
    fused = args.tp_gather == "fused" and (world > 1 or emulate)
    for gi, grp in enumerate(groups):
        if grp[0]["sharded"]:
            if fused:
                specs = [(args.fmt, e["L"].M, e["L"].K, e["L"].r) for e in grp]
                if emulate:
                    sgs[gi] = tp.EmulatedGather(specs, dev, world=shard_world)
                else:
                    sgs[gi] = (tp.IpcGather if backend == "gloo" else tp.SymmetricGather)(specs, dev)
                gbuf[gi] = (None, sgs[gi].buf)
            else:
                tot = sum(e["slice"].numel() for e in grp)
                gbuf[gi] = (torch.empty(tot, dtype=torch.uint8, device=dev),
                            torch.zeros(shard_world * tot, dtype=torch.uint8, device=dev))
    stream = torch.cuda.Stream(device=dev)
    comm_ev = []

    def step(st, record=None):
        for gi, grp in enumerate(groups):
            if grp[0]["sharded"] and fused:
                if record is not None:
                    record[gi][0].record(st)
                for j, e in enumerate(grp):         # K1 stores straight into every rank's buffer
                    sgs[gi].fill(j, e["cp"].local, e["k0"], e["x"], stream=st)
                sgs[gi].sync()
                if record is not None:
                    record[gi][1].record(st)
                for j, e in enumerate(grp):
                    e["xq"], e["xs"], e["xl1"] = sgs[gi].outputs(j, stream=st)
            elif grp[0]["sharded"]:
                send, recv = gbuf[gi]
                tot = recv.numel() // shard_world
                off = 0
                for e in grp:
                    nb = e["slice"].numel()
                    P.svdq_quantize_act_lowrank_down_kslice(e["cp"].local, e["k0"], e["x"], send[off:off + nb],
                                                            stream=st)
                    off += nb
                if record is not None:
                    record[gi][0].record(st)
                if world > 1:
                    tp.all_gather(recv, send)
                else:                            # P = 1, or emulation: this rank's slice only
                    recv[:tot].copy_(send)
                if record is not None:
                    record[gi][1].record(st)
                off = 0
                for e in grp:                    # rank p's slice of this layer at recv[p * tot + off]
                    P.svdq_tp_assemble_act(args.fmt, shard_world, e["L"].M, e["L"].K, e["L"].r, recv[off:], e["xq"], e["xs"],
                                           e["xl1"], slice_stride=tot, stream=st)
                    off += e["slice"].numel()
            elif len(grp) > 1:
                P.svdq_quantize_act_lowrank_down_grouped([e["cp"].local for e in grp], [e["x"] for e in grp],
                                                         [e["xq"] for e in grp], [e["xs"] for e in grp],
                                                         [e["xl1"] for e in grp], stream=st)
            else:
                e = grp[0]
                P.svdq_quantize_act_lowrank_down(e["cp"].local, e["x"], e["xq"], e["xs"], e["xl1"], stream=st)
            P.svdq_gemm_w4a4_lowrank_up_grouped([e["cp"].local for e in grp], [e["xq"] for e in grp],
                                                [e["xs"] for e in grp], [e["xl1"] for e in grp],
                                                [e["L"].M for e in grp], [e["y"] for e in grp], stream=st)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(stream)
    torch.cuda.synchronize()
    graph, graph_err = None, None
    if backend == "nccl" or world == 1:
        try:                                     # NCCL collectives inside CUDA-graph capture
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step(stream)
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001  (capture unsupported here: eager launches instead)
            graph, graph_err = None, f"{type(ex).__name__}: {str(ex)[:120]}"
            torch.cuda.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)
    step_ev = [(ev(), ev()) for _ in range(args.steps)]
    barrier = dist.barrier if world > 1 else (lambda: None)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        with torch.cuda.stream(stream):
            for s in range(args.steps):
                step_ev[s][0].record(stream)
                if graph is not None:
                    graph.replay()
                else:
                    step(stream)
                step_ev[s][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    total_ms = float(sum(a.elapsed_time(b) for a, b in step_ev))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # communication share: eager step with events around every all-gather
    rec = {gi: (ev(), ev()) for gi in gbuf}
    nrep = max(3, min(args.steps, 10))
    comm = []
    for _ in range(nrep):
        barrier()
        with torch.cuda.stream(stream):
            a, b = ev(), ev()
            a.record(stream)
            step(stream, rec)
            b.record(stream)
        torch.cuda.synchronize()
        comm.append((sum(x.elapsed_time(y) for x, y in rec.values()), a.elapsed_time(b)))
    comm_ms, eager_ms = (float(np.mean([c[0] for c in comm])), float(np.mean([c[1] for c in comm])))
    if rank != 0:
        return None
    flops = sum(2.0 * L.M * L.N * L.K for L in layers)
    gathered_bytes = sum(gbuf[gi][1].numel() for gi in gbuf)
    cfg = bench_config(args, world)
    cfg["parallelism"] = f"tp{world} (column-parallel over N; SURVEY 8(e) Variant 2 packed all-gathers)"
    cfg["block_latency_ms"] = round(total_ms / args.steps, 4)
    projection = None
    if emulate:
        # one rank's measured compute + the modeled packed all-gathers (bytes each rank receives at an
        # assumed all-gather bus bandwidth + a per-collective latency); overlapped = max per gather
        # bytes each rank receives: (P-1)/P of the packed slices (all-gather) or of the full K1 outputs
        # written by the peers (fused)
        recv_bytes = [gbuf[gi][1].numel() * (emulate - 1) / emulate for gi in gbuf]
        comm_model_ms = sum(b_ / (args.tp_bw_gbs * 1e9) * 1e3 + args.tp_lat_us * 1e-3 for b_ in recv_bytes)
        step_ms = total_ms / args.steps
        projection = {"P": emulate, "per_rank_compute_ms": round(step_ms, 4),
                      "modeled_comm_ms": round(comm_model_ms, 4),
                      "projected_step_ms_serial": round(step_ms + comm_model_ms, 4),
                      "projected_tflops_serial": round(flops / ((step_ms + comm_model_ms) / 1e3) / 1e12, 1),
                      "assumptions": {"allgather_bus_GBps": args.tp_bw_gbs, "per_collective_latency_us": args.tp_lat_us},
                      "note": "MEASURED: rank 0's kernels of a P-way TP step on one B200 (its N-shards, K-slice K1, "
                              "assembly of P slices); MODELED: the NVLink all-gathers.  Not a multi-GPU run."}
        cfg["parallelism"] = f"tp{emulate} emulated on one GPU (rank 0's work; gathers modeled)"
    return {
        "metric": METRIC, "value": round(flops * args.steps / (total_ms / 1e3) / 1e12, 2), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "e2m1 x e2m1 -> f32 (NVFP4 g16 e4m3 scales) + bf16 low-rank" if args.fmt == "nvfp4" else args.fmt,
        "data": "synthetic (seeded; DESIGN.md input recipe), weights prepared on GPU by svdq_quantize_weights, "
                "column-sharded", "config": cfg,
        "tp": {"backend": backend, "gather": "fused K1 peer stores (symmetric memory)" if fused else "all_gather_into_tensor",
               "graph": graph is not None, "graph_error": graph_err,
               "comm_ms_per_step": round(comm_ms, 4), "eager_step_ms": round(eager_ms, 4),
               "comm_def": "fused: the K1 launches that store into every rank's buffer + the barrier; else the "
                           "all-gathers",
               "comm_fraction_eager": round(comm_ms / eager_ms, 4) if eager_ms else None,
               "gathered_bytes_per_rank_per_step": int(gathered_bytes),
               "sharded_input_layers": [L.name for L in layers if L.name.endswith(SHARDED_INPUT)],
               "note": "value = the full block-pair FLOPs (sum 2MNK over all linears) / max-over-ranks step time "
                       "(strong scaling: the total work is fixed); comm from events around each all-gather in an "
                       "eager replay of the step"},
        "tp_projection": projection,
        "clocks": clk.summary(),
    }


# ------------------------------------------------------------------ oracle timings
def oracle_operands(L, i, fmt):
    """Valid stored operands of the layer's shape for TIMING the oracle forward: random
    E2M1 / INT4 codes and scale bytes, bf16 L1s / L2s, lambda from the input recipe.  The
    oracle's forward cost does not depend on the values; its weight preparation (SVD,
    residual quantization) is offline on both arms and untimed."""
    from oracle import formats as F
    from oracle import svdquant as S
    g = np.random.default_rng(7000 + i)
    if fmt == "nvfp4":
        codes = g.integers(0, 16, (L.N, L.K), dtype=np.uint8)
        scales = g.integers(0x30, 0x40, (L.N, L.K // 16), dtype=np.uint8)
        sdt, gs_w = "e4m3", np.float32(0.01)
    else:
        codes = g.integers(-7, 8, (L.N, L.K), dtype=np.int8)
        scales = F.bf16_bits(g.uniform(0.005, 0.02, (L.N, L.K // 64)))
        sdt, gs_w = "bf16", np.float32(1.0)
    lam_inv = np.float32(1.0) / np.abs(g.standard_normal(L.K)).astype(np.float32).clip(0.1, 10)
    l1s = F.bf16_bits(g.standard_normal((L.r, L.K)) * 0.02)
    l2s = F.bf16_bits(g.standard_normal((L.N, L.r)) * 0.02)
    bias = F.bf16_round(synth.gen_bias(L.N, synth.rng(4, i, 3)))
    return S.Operands(fmt, L.K, L.N, L.r, codes, scales, sdt, gs_w, np.float32(1.0),
                      lam_inv.astype(np.float32), l1s, l2s, bias)


def oracle_forward_time(layers, rows, fmt, idx=None):
    """Seconds and algorithmic FLOPs of the oracle forward (K1 + K2 semantics) on `rows`
    tokens of each layer (the layers' own synthetic activations, first `rows` rows)."""
    from oracle import formats as F
    from oracle import svdquant as S
    t_total, flops = 0.0, 0.0
    for i, L in enumerate(layers):
        if idx is not None and i not in idx:
            continue
        ops = oracle_operands(L, i, fmt)
        x = F.bf16_round(synth.gen_x(rows, L.K, synth.rng(4, i, 0)))
        t0 = time.perf_counter()
        S.forward(x, ops)
        t_total += time.perf_counter() - t0
        flops += 2.0 * rows * L.N * L.K
    return t_total, flops


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def host_info():
    """What the oracle's CPU time ran on: logical CPUs, the affinity mask, the
    NumPy BLAS vendor and its thread count."""
    info = {"os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "blas_threads": blas_threads(), "blas": None}
    try:
        from threadpoolctl import threadpool_info
        libs = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if libs:
            info["blas"] = f"{libs[0].get('internal_api')} {libs[0].get('version')}"
    except Exception:
        pass
    return info


def oracle_cores():
    """Threads the oracle actually used: its fp64 GEMMs run on the BLAS pool (bounded by the
    affinity mask); the fp32 quantizer steps are single-threaded NumPy."""
    return min(blas_threads(), len(os.sched_getaffinity(0)))


def run_reference(args):
    """The reference arm of this tier: the CPU oracle, as it stands, on the same workload.
    Step s = the oracle forward of `--ref-rows` tokens of linear (s mod 10) of the step, so
    every step is a bounded sample and the run ends within a few minutes."""
    layers = config_layers(args)
    rows = args.ref_rows
    for w in range(args.warmup):
        oracle_forward_time(layers, 8, args.fmt, idx={w % len(layers)})
    t_all, f_all, ts = 0.0, 0.0, []
    for s in range(args.steps):
        t, f = oracle_forward_time(layers, rows, args.fmt, idx={s % len(layers)})
        t_all += t
        f_all += f
        ts.append(t)
    value = f_all / t_all / 1e12
    cores = oracle_cores()
    sample = (f"{rows} tokens of one of the step's {len(layers)} linears per step (rotating; oracle "
              f"forward in fp64 with NumPy/BLAS)")
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * float(np.mean(ts)), 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)",
        "data": "synthetic (seeded)",
        "config": bench_config(args, 1),
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample, "host": host_info()},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="svdq", choices=["svdq", "reference"])
    ap.add_argument("--fmt", default="nvfp4", choices=["nvfp4", "int4", "w8a8"])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ref-rows", type=int, default=512)   # per-step sample of the reference arm (oracle)
    ap.add_argument("--cpu-rows", type=int, default=1024)   # ~10-30 s of oracle CPU work (weight prep is ~6 s of it)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the rank-0 overhead / library legs")
    ap.add_argument("--config", default="flux", choices=["flux", "pixart", "sdxl"],
                    help="BASELINE config: C4 FLUX.1 block pair (default), C2 PixArt-Sigma block, C3 SDXL + LoRA")
    ap.add_argument("--mode", default="auto", choices=["auto", "tp", "replicas"],
                    help="N > 1: tensor parallel over N (C5, default) or independent replicas")
    ap.add_argument("--tp-gather", default="nccl", choices=["nccl", "fused"],
                    help="TP packed-slice gather: one all_gather_into_tensor, or K1 storing into every rank's "
                         "symmetric-memory buffer (SURVEY 8(f) row 2)")
    ap.add_argument("--tp-emulate", type=int, default=0,
                    help="one GPU, --mode tp: time rank 0's share of a P-way TP step, model the gathers")
    ap.add_argument("--tp-bw-gbs", type=float, default=750.0, help="modeled all-gather bus bandwidth (emulation)")
    ap.add_argument("--tp-lat-us", type=float, default=10.0, help="modeled per-collective latency (emulation)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: multi-process tests on one GPU (NCCL refuses two ranks per device)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "svdq":
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)))
        return

    mode = ("tp" if world > 1 else "single") if args.mode == "auto" else args.mode
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.backend == "gloo":                 # test mode: ranks may share the box's one GPU
            local_rank %= max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    if mode == "tp":                           # world 1: the TP code path with P = 1 (functional check)
        if args.fmt == "w8a8":
            raise SystemExit("TP mode: W8A8's per-token scales need the whole row (use --mode replicas)")
        out = run_tp(args, rank, world, local_rank, args.backend if world > 1 else "none")
        if rank == 0:
            print(json.dumps(out))
        if world > 1:
            dist.destroy_process_group()
        return
    out = run_svdq(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            t, f = oracle_forward_time(config_layers(args), args.cpu_rows, args.fmt)
            out["cpu_baseline"] = {"value": round(f / t / 1e12, 6), "unit": UNIT, "cores": oracle_cores(),
                                   "kind": "oracle", "host": host_info(),
                                   "sample": f"{args.cpu_rows} tokens of each of the step's {len(config_layers(args))} linears "
                                             f"(oracle forward, fp64 NumPy/BLAS; {t:.1f} s of CPU time)"}
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
