"""C5 on one GPU: the FLUX.1-dev 57-block linear stack (19 double + 38 single blocks) at batch
1..8, with the bench's launch sequence (bench.flux_step_grouped: a double block's img + txt linears
of each kind as one grouped K1 + one grouped K2 launch; the single block's linears alone).  One
double block and one single block are each captured as a CUDA graph and timed with CUDA events,
L2 flushed before every replay; stack = 19 x double + 38 x single (every block of a kind has the
same shapes).  This is the P = 1 point of the north star's tensor-parallel C5 configuration.
    python tools/c5_stack.py [--out profiles/r02/c5_stack_1gpu.json]"""
import argparse, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2411_05007_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(bench.ROOT, "profiles", "r02", "c5_stack_1gpu.json"))
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--batches", default="1,2,4,8")
a = ap.parse_args()
dev = torch.device("cuda")
st = torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
sink = torch.empty((), dtype=torch.int64, device=dev)


def time_block(built):
    with torch.cuda.stream(st):
        for _ in range(3):
            bench.flux_step_grouped(P, built, st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        bench.flux_step_grouped(P, built, st)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            flush.zero_()
            sink.copy_(flush[: 256 << 20].view(torch.int64).sum())
            e0.record(st)
            g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


out = {"note": __doc__.split("\n    python")[0], "batches": {}}
for B in (int(b) for b in a.batches.split(",")):
    dl, sl = synth.flux_double_block(B), synth.flux_single_block(B)
    td = time_block(bench.build_layers(P, torch, dl, "nvfp4", dev))
    torch.cuda.empty_cache()
    ts = time_block(bench.build_layers(P, torch, sl, "nvfp4", dev))
    torch.cuda.empty_cache()
    fl = 19 * sum(2.0 * L.M * L.N * L.K for L in dl) + 38 * sum(2.0 * L.M * L.N * L.K for L in sl)
    lat = 19 * td + 38 * ts
    row = {"double_block_ms": round(td, 4), "single_block_ms": round(ts, 4), "stack_ms": round(lat, 3),
           "stack_tflops": round(fl / (lat * 1e-3) / 1e12, 1)}
    out["batches"][f"batch{B}"] = row
    print("C5", B, row, flush=True)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(out, open(a.out, "w"), indent=1)
print("wrote", a.out)
