"""Our tcgen05 NVFP4 GEMM vs cuBLASLt NVFP4 (torch._scaled_mm) vs BF16 cuBLAS at the c3 shapes."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2601_22813_b200 as q2

dev = torch.device("cuda:0")
T = bench.TOKENS
for name, din, dout in bench.PROJECTIONS:
    for gname, M, N, K in (("fprop", T, dout, din), ("dgrad", T, din, dout), ("wgrad", dout, din, T)):
        qa, qb = bench._random_nvfp4(q2, M, K, dev), bench._random_nvfp4(q2, N, K, dev)
        od = torch.float32 if gname == "wgrad" else torch.bfloat16
        fl = 2.0 * M * N * K
        ours = bench._time_ms(lambda: q2.gemm(qa, qb, od), iters=10, warmup=3)
        A = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
        B = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
        bf = bench._time_ms(lambda: A @ B.t(), iters=10, warmup=3)
        lt = bench._cublaslt_nvfp4(qa, qb, fl)
        print(f"{name:7s} {gname}: M={M} N={N} K={K}  ours {fl / ours / 1e9:6.0f} TF/s ({ours * 1e3:6.1f} us)  "
              f"cuBLASLt nvfp4 {lt.get('cublaslt_nvfp4_TFLOP/s', 0):6.0f}  bf16 {fl / bf / 1e9:6.0f}")
