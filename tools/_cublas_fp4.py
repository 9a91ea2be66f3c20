import torch, sys
M, K, N = (int(a) for a in sys.argv[1:4])
dev = torch.device("cuda")
a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
sa = torch.full(((M + 127) // 128 * 128 * K // 16,), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
sb = torch.full(((N + 127) // 128 * 128 * K // 16,), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
for _ in range(3):
    y = torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
print("ok", y.shape)
