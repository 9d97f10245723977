"""One launch of each hot kernel at the c3 UpGate shapes (for ncu --set full).

    ncu --set full -k regex:<kernel> -s 1 -c 1 python tools/prof_targets.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402

q2.set_error_mode("deferred")
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(16384, 2048, device="cuda", generator=g).bfloat16()
W = (torch.randn(11264, 2048, device="cuda", generator=g) / 45).bfloat16()
E = (1e-3 * torch.randn(16384, 11264, device="cuda", generator=g)).bfloat16()
S = q2.SeedPair(1, 2)
for _ in range(2):
    qx, qw = q2.quantize_rtn_46(X), q2.quantize_rtn_46(W)
    y = q2.gemm(qx, qw, torch.bfloat16)                                  # fprop
    qe = q2.msed(E, S, 6.0, 1, 2, "posthoc", "rows")                     # MS(E)
    qet = q2.msed(E, S, 6.0, 3, 4, "posthoc", "cols")                    # MS(E^T)
    qxt = q2.msed(qx, S, 6.0, 5, 4, "posthoc", "tape")                   # MS(X^T) from the tape
    dw = q2.gemm(qet, qxt, torch.float32)                                # wgrad
    qwt = q2.msed(qw, S, 6.0, 6, 2, "posthoc", "tape")                   # MS(W^T) from the tape
    dx = q2.gemm(qe, qwt, torch.bfloat16)                                # dgrad
    torch.cuda.synchronize()
q2.check_errors()
