"""Per-tile GEMM timeline (Q2_GEMM_TRACE=1): fprop, dgrad-like and wgrad-like shapes.

    Q2_GEMM_TRACE=1 python tools/gemm_trace_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for name, (m, n, k) in (("fprop K=2048", (16384, 11264, 2048)), ("dgrad K=11264", (16384, 2048, 11264))):
    A = torch.randn(m, k, device="cuda", generator=g).bfloat16()
    B = (torch.randn(n, k, device="cuda", generator=g) / 45).bfloat16()
    qa, qb = q2.quantize_rtn_46(A), q2.quantize_rtn_46(B)
    print(name, flush=True)
    for _ in range(2):
        y = q2.gemm(qa, qb, torch.bfloat16)
    torch.cuda.synchronize()
