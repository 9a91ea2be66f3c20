"""Wall time of the offline weight pipeline on one B200 at FLUX.1 linear shapes:
svdq_quantize_weights (RTN), svdq_quantize_weights_gptq, svdq_search_alpha (5-point grid) and
svdq_refine_lowrank (3 iterations), NVFP4, rank 32, M_cal calibration tokens.  Offline steps:
host wall clock around synchronizing calls (they synchronize internally).

    python tools/time_offline.py [--out profiles/r01/offline_times.json]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_05007_b200 as P  # noqa: E402


def wall(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "offline_times.json"))
    ap.add_argument("--m-cal", type=int, default=1024)
    a = ap.parse_args()
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    out = {"method": "host wall clock around synchronizing offline calls, mean of 2 after 1 warm-up",
           "fmt": "nvfp4", "rank": 32, "M_cal": a.m_cal, "shapes": {}}
    for name, K, N in (("qkv_3072x9216", 3072, 9216), ("mlp_down_12288x3072", 12288, 3072)):
        W = torch.randn(K, N, device=dev, generator=g) / K ** 0.5
        X = torch.randn(a.m_cal, K, device=dev, generator=g).to(torch.bfloat16)
        lam = torch.rand(K, device=dev, generator=g) + 0.5
        r = {
            "quantize_weights_s": wall(lambda: P.svdq_quantize_weights(W, lam, 32, "nvfp4")),
            "quantize_weights_gptq_s": wall(lambda: P.svdq_quantize_weights_gptq(W, lam, 32, "nvfp4", X)),
            "search_alpha_5pt_s": wall(lambda: P.svdq_search_alpha(X, W, 32, "nvfp4", [0.0, 0.25, 0.5, 0.75, 1.0]), 1),
            "refine_3iter_s": wall(lambda: P.svdq_refine_lowrank(X, W, lam, 32, "nvfp4", 3), 1),
        }
        out["shapes"][name] = {k: round(v, 3) for k, v in r.items()}
        print(name, out["shapes"][name], flush=True)
        del W, X
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
