"""Time q2.gemm at one shape (env knobs are read once per process): M N K [f32]."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_22813_b200 as q2  # noqa: E402

dev = torch.device("cuda:0")
for spec in sys.argv[1:]:
    M, N, K = (int(v) for v in spec.split("x"))
    qa, qb = bench._random_nvfp4(q2, M, K, dev), bench._random_nvfp4(q2, N, K, dev)
    if os.environ.get("ZERO"):               # data-dependence probe: all-zero codes
        qa.codes.zero_()
        qb.codes.zero_()
    od = torch.bfloat16
    it = int(os.environ.get("ITERS", "20"))
    if os.environ.get("LT"):                 # cuBLASLt NVFP4 (torch._scaled_mm), scales random as in bench.py
        a = qa.codes.view(torch.float4_e2m1fn_x2)
        b = qb.codes.view(torch.float4_e2m1fn_x2)
        sa = torch.randint(0x30, 0x48, (((M + 127) // 128) * 128 * ((K // 16 + 3) // 4) * 4,), dtype=torch.uint8,
                           device=dev).view(torch.float8_e4m3fn)
        sb = torch.randint(0x30, 0x48, (((N + 127) // 128) * 128 * ((K // 16 + 3) // 4) * 4,), dtype=torch.uint8,
                           device=dev).view(torch.float8_e4m3fn)
        ms = bench._time_ms(lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16), iters=it, warmup=int(os.environ.get("WARM", "5")))
    else:
        ms = bench._time_ms(lambda: q2.gemm(qa, qb, od), iters=it, warmup=int(os.environ.get("WARM", "5")))
    print(f"{spec:>20s} {ms * 1e3:7.1f} us {2.0 * M * N * K / ms / 1e9:6.0f} TF/s  [{os.environ.get('TAG', '')}]")
