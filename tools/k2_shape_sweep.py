"""K2 per-launch duration (back to back, DRAM-cold, bench.b2b_slope) on the small-layer shapes of
C2 (PixArt-Sigma) and C3 (SDXL) under the tile-shape knobs in the environment (SVDQ_K2_PAIR,
SVDQ_K2_BN, SVDQ_K2_BN1).     python tools/k2_shape_sweep.py [tag]"""
import json, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2411_05007_b200 as P  # noqa: E402

SHAPES = [(4096, 1152, 3456), (4096, 1152, 1152), (4096, 1152, 4608), (4096, 4608, 1152),
          (8192, 640, 1920), (8192, 640, 640), (8192, 640, 5120), (8192, 2560, 640),
          (2048, 1280, 3840), (2048, 1280, 1280), (2048, 1280, 10240), (2048, 5120, 1280),
          (512, 3072, 3072), (512, 3072, 9216), (512, 12288, 3072), (512, 3072, 12288),
          (4096, 3072, 3072), (4608, 15360, 3072)]
tag = sys.argv[1] if len(sys.argv) > 1 else "default"
dev = torch.device("cuda")
st = torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
sink = torch.empty((), dtype=torch.int64, device=dev)


def l2_flush():
    flush.zero_()
    sink.copy_(flush[: 256 << 20].view(torch.int64).sum())


res = {}
for (M, K, N) in SHAPES:
    layer = P.QuantizedLinear.empty("nvfp4", K, N, 32, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    layer.w_codes.random_(0, 256, generator=g)
    layer.w_scales.fill_(0x30)
    layer.l1s.random_(-2000, 2000, generator=g)
    layer.l2s.random_(-2000, 2000, generator=g)
    layer.lambda_inv.fill_(1.0)
    layer._sync_view()
    x = torch.randn(M, K, device=dev).to(torch.bfloat16)
    xq, xs, xl1 = P.svdq_quantize_act_lowrank_down(layer, x)
    y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    wb = layer.w_codes.numel() + layer.w_scales.numel() + xq.numel() + xs.numel()
    c = int(min(16, max(2, math.ceil(3 * (126 << 20) / wb))))
    cps = [(P.QuantizedLinear("nvfp4", K, N, 32, layer.w_codes.clone(), layer.w_scales.clone(), layer.lambda_inv,
                              layer.l1s, layer.l2s.clone(), None, "bf16", 1.0, 1.0),
            xq.clone(), xs.clone(), xl1.clone()) for _ in range(c)]
    t = bench.b2b_slope(torch, st, l2_flush, 5,
                        lambda j: P.svdq_gemm_w4a4_lowrank_up(cps[j][0], cps[j][1], cps[j][2], cps[j][3], M, Y=y,
                                                              stream=st), c)
    res[f"{M}x{K}x{N}"] = round(t * 1e6, 2)
    del cps
    torch.cuda.empty_cache()
print(json.dumps({"tag": tag, "k2_us": res}))
