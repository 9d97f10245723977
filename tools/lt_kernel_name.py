"""Name of the cuBLASLt NVFP4 kernel torch._scaled_mm launches (tile/cluster shape in the name)."""
import torch
from torch.profiler import profile, ProfilerActivity
M, N, K = 16384, 2048, 11264
dev = "cuda"
a = torch.randint(0, 255, (M, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
b = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
sa = torch.randint(0x30, 0x48, (M * K // 16,), dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
sb = torch.randint(0x30, 0x48, (N * K // 16,), dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
for shape in ((16384, 2048, 11264), (16384, 11264, 2048)):
    M, N, K = shape
    a = torch.randint(0, 255, (M, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
    b = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
    sa = torch.randint(0x30, 0x48, (M * K // 16,), dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
    sb = torch.randint(0x30, 0x48, (N * K // 16,), dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
    torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
    for e in p.key_averages():
        print(shape, e.key[:300])
