"""C5 (FLUX.1 57-block linear stack, tensor-parallel at P = 2/4/8) -- a PROJECTION from one GPU.

gpurun grants one B200, so the P-rank run cannot be executed here.  What is measured: one
rank's compute for column-parallel sharding (paper_2411_05007_b200/tp.py) --
K1 on the replicated activation (identical on every rank) + K2 on its N/P output columns --
for every W4A4 linear of a double and a single block at batch B, as CUDA graphs with L2
flushed before each.  What is modeled: the bf16 all-gathers where the next consumer needs the
full feature dimension (attention-out input 3072, MLP-down input 12288, single-block linear2
input 15360; qkv / linear1 outputs feed head-aligned attention locally): per-rank bytes
2 * M * width * (P-1)/P at an assumed NVLink-5 all-gather bus bandwidth (--bw GB/s), plus a
fixed per-collective latency.  Reported: compute-only, serial compute + comm, and the
comm-overlapped bound max(compute, comm) per block.

    python tools/tp_projection.py [--bw 750] [--lat-us 8] [--out profiles/r01/tp_projection.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import synth  # noqa: E402
from bench_configs import Flusher, make_items, time_layers  # noqa: E402

dev = torch.device("cuda")
GATHER_WIDTH = {"proj": 3072, "mlp_down": 12288, "linear2": 15360}   # inputs that need the full features


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bw", type=float, default=750.0, help="all-gather bus bandwidth per GPU, GB/s")
    ap.add_argument("--lat-us", type=float, default=8.0, help="per all-gather fixed latency, us")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "tp_projection.json"))
    a = ap.parse_args()
    gen = torch.Generator(device=dev).manual_seed(3)
    stream = torch.cuda.Stream()
    flush = Flusher()
    out = {"assumptions": {"allgather_bus_GBps": a.bw, "per_collective_latency_us": a.lat_us,
                           "note": "per-rank compute MEASURED on one B200; communication MODELED; not a multi-GPU run"},
           "results": {}}
    for B in (1, 2, 4, 8):
        for P in (1, 2, 4, 8):
            layers = synth.flux_double_block(B) + synth.flux_single_block(B)
            shard = [synth.Layer(L.name, L.M, L.K, L.N // P, L.r) for L in layers]
            items = make_items(shard, "nvfp4", gen)
            t, _ = time_layers(items, a.reps, stream, flush)
            del items
            torch.cuda.empty_cache()
            comp_d = sum(t[j][0] + t[j][1] for j, L in enumerate(layers) if L.name.startswith("double"))
            comp_s = sum(t[j][0] + t[j][1] for j, L in enumerate(layers) if L.name.startswith("single"))
            comm_d = comm_s = 0.0
            if P > 1:
                for L in layers:
                    kind = L.name.split("_", 2)[-1]
                    for key, width in GATHER_WIDTH.items():
                        if kind.endswith(key) and not (key == "proj" and L.name.startswith("single")):
                            # the gather feeding this linear: its input of `width` features, M tokens
                            sec = 2.0 * L.M * width * (P - 1) / P / (a.bw * 1e9) + a.lat_us * 1e-6
                            if L.name.startswith("double"):
                                comm_d += sec
                            else:
                                comm_s += sec
            stack_comp = 19 * comp_d + 38 * comp_s
            stack_serial = 19 * (comp_d + comm_d) + 38 * (comp_s + comm_s)
            stack_overlap = 19 * max(comp_d, comm_d) + 38 * max(comp_s, comm_s)
            r = {"per_rank_compute_ms": round(stack_comp * 1e3, 3), "comm_ms": round((19 * comm_d + 38 * comm_s) * 1e3, 3),
                 "stack_ms_serial": round(stack_serial * 1e3, 3), "stack_ms_overlapped": round(stack_overlap * 1e3, 3)}
            out["results"][f"batch{B}_P{P}"] = r
            print(B, P, r, flush=True)
    for B in (1, 2, 4, 8):
        base = out["results"][f"batch{B}_P1"]["stack_ms_serial"]
        for P in (2, 4, 8):
            r = out["results"][f"batch{B}_P{P}"]
            r["speedup_serial"] = round(base / r["stack_ms_serial"], 3)
            r["speedup_overlapped"] = round(base / r["stack_ms_overlapped"], 3)
            r["efficiency_overlapped"] = round(base / r["stack_ms_overlapped"] / P, 3)
    json.dump(out, open(a.out, "w"), indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
