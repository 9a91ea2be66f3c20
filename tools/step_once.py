"""Run the bench's grouped FLUX step (bench.flux_step_grouped) WARM times, then once more: the
target for `ncu --set full` / launch lists of exactly the step's 12 launches.
    python tools/step_once.py [--warm 2]      (under ncu: --profile-from-start off)"""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2411_05007_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warm", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda")
built = bench.build_layers(P, torch, synth.flux_double_block(1) + synth.flux_single_block(1), "nvfp4", dev)
st = torch.cuda.current_stream()
for _ in range(a.warm):
    bench.flux_step_grouped(P, built, st)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()          # ncu --profile-from-start off: only this step
bench.flux_step_grouped(P, built, st)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
