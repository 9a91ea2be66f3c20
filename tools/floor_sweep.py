"""Small-layer floor: per-launch K1 / K2 durations (back to back, DRAM-cold, bench.b2b_slope) over
M at one (K, N), plus the per-node cost of a trivial kernel in the same graph form.  The intercept
of time vs M is the fixed cost per launch (prologue, first DRAM latency, drain).
    python tools/floor_sweep.py [K N [dtype]]      (defaults: PixArt attn_out 1152 1152 fp16)"""
import json, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2411_05007_b200 as P  # noqa: E402
from paper_2411_05007_b200 import abi  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1152
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1152
xdt = {"fp16": torch.float16, "bf16": torch.bfloat16}[sys.argv[3] if len(sys.argv) > 3 else "fp16"]
dev = torch.device("cuda")
st = torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
sink = torch.empty((), dtype=torch.int64, device=dev)


def l2_flush():
    flush.zero_()
    sink.copy_(flush[: 256 << 20].view(torch.int64).sum())


def make_layer():
    layer = P.QuantizedLinear.empty("nvfp4", K, N, 32, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    layer.w_codes.random_(0, 256, generator=g)
    layer.w_scales.fill_(0x30)
    layer.l1s.random_(-2000, 2000, generator=g)
    layer.l2s.random_(-2000, 2000, generator=g)
    layer.lambda_inv.fill_(1.0)
    layer._sync_view()
    return layer


out = {"K": K, "N": N, "x_dtype": str(xdt), "rows": []}
tiny = torch.zeros(1, device=dev)
with torch.cuda.stream(st):
    tiny.add_(1)
torch.cuda.synchronize()
out["trivial_kernel_us"] = bench.b2b_slope(torch, st, l2_flush, 5, lambda j: tiny.add_(1), 1) * 1e6
layer = make_layer()
for M in (256, 512, 1024, 2048, 4096, 8192, 16384):
    c = int(min(16, max(2, math.ceil(3 * (126 << 20) / (M * K * 2)))))
    xs = [torch.randn(M, K, device=dev).to(xdt) for _ in range(c)]
    xq, xsc, xl1 = P.svdq_quantize_act_lowrank_down(layer, xs[0])
    y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    t1 = bench.b2b_slope(torch, st, l2_flush, 5,
                         lambda j: P.svdq_quantize_act_lowrank_down(layer, xs[j], xq, xsc, xl1, stream=st), c)
    wb = layer.w_codes.numel() + layer.w_scales.numel() + xq.numel() + xsc.numel()
    c2 = int(min(16, max(2, math.ceil(3 * (126 << 20) / wb))))
    cps = [(P.QuantizedLinear(layer.fmt, K, N, 32, layer.w_codes.clone(), layer.w_scales.clone(), layer.lambda_inv,
                              layer.l1s, layer.l2s.clone(), None, "bf16", 1.0, 1.0),
            xq.clone(), xsc.clone(), xl1.clone()) for _ in range(c2)]
    t2 = bench.b2b_slope(torch, st, l2_flush, 5,
                         lambda j: P.svdq_gemm_w4a4_lowrank_up(cps[j][0], cps[j][1], cps[j][2], cps[j][3], M, Y=y,
                                                               stream=st), c2)
    b1 = M * K * (xs[0].element_size() + 0.5625) + 2 * M * 32
    f2 = 2.0 * M * N * K
    row = {"M": M, "k1_us": t1 * 1e6, "k1_tbs": b1 / t1 / 1e12, "k2_us": t2 * 1e6, "k2_tflops": f2 / t2 / 1e12,
           "k1_rt": abi._lib.svdq_k1_row_tile(M, 32)}
    out["rows"].append(row)
    print(json.dumps(row), flush=True)
    del xs, cps
    torch.cuda.empty_cache()
print(json.dumps(out))
