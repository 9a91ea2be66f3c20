"""Run one bench step WARM times, then once more between cudaProfilerStart/Stop: the target for
`ncu --set full` / launch lists of exactly the step's launches.
  --config flux (default): bench.flux_step_grouped, 6 K1 + 6 K2 launches;
  --config pixart | sdxl, or --fmt int4 | w8a8: the serial step (K1 -> K2 per linear).
    python tools/step_once.py [--warm 2] [--config flux|pixart|sdxl]   (under ncu: --profile-from-start off)"""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2411_05007_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--config", default="flux", choices=["flux", "pixart", "sdxl"])
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--fmt", default="nvfp4", choices=["nvfp4", "int4", "w8a8"])
a = ap.parse_args()
dev = torch.device("cuda")
built = bench.build_layers(P, torch, bench.config_layers(a), a.fmt, dev)
st = torch.cuda.current_stream()


def step():
    if a.config == "flux" and a.fmt == "nvfp4":
        bench.flux_step_grouped(P, built, st)
        return
    for (L, layer, b) in built:
        P.svdq_quantize_act_lowrank_down(layer, b["x"], b["xq"], b["xs"], b["xl1"], stream=st)
        P.svdq_gemm_w4a4_lowrank_up(layer, b["xq"], b["xs"], b["xl1"], L.M, Y=b["y"], stream=st)


for _ in range(a.warm):
    step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()          # ncu --profile-from-start off: only this step
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
