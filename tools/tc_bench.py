"""Tensor-core MS-EDEN: literal-path rate per parity family and timing at c3 shapes
(dual E, tape X^T / W^T) against the literal float64 kernels (Q2_MSED_LITERAL=1 run)."""
import os
import sys
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from tests.families import FAMILIES, make

dev = torch.device("cuda:0")
q2.set_msed_engine(os.environ.get("Q2_ENGINE", "auto"))
if "--rates" in sys.argv:
    for fam in FAMILIES:
        e = torch.from_numpy(make(fam, (1024, 1024), seed=3)).to(dev).to(torch.bfloat16)
        for mode in ("exact", "posthoc"):
            q2.msed_stats(reset=True)
            q2.msed_dual(e, q2.SeedPair(1, 2), 1, 2, 3, 4, 6.0, mode)
            tot, lit = q2.msed_stats()
            w = q2.quantize_rtn_46(e)
            q2.msed_stats(reset=True)
            q2.msed(w, q2.SeedPair(1, 2), 6.0, 5, 6, mode, "tape")
            tt, tl = q2.msed_stats()
            print(f"{fam:15s} {mode:8s} dual literal {lit}/{tot} = {lit / max(tot, 1):.2e}   tape {tl}/{tt} = {tl / max(tt, 1):.2e}")


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(iters):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / iters


T = 16384
for (inp, out) in ((2048, 6144), (2048, 2048), (2048, 11264), (5632, 2048)):
    E = torch.randn(T, out, device=dev).mul_(1e-3).to(torch.bfloat16)
    X = torch.randn(T, inp, device=dev).to(torch.bfloat16)
    W = (torch.randn(out, inp, device=dev) / inp ** 0.5).to(torch.bfloat16)
    qX, qW = q2.quantize_rtn_46(X), q2.quantize_rtn_46(W)
    sp = q2.SeedPair(1, 2)
    for mode in ("posthoc", "exact"):
        q2.msed_stats(reset=True)
        td = timeit(lambda: q2.msed_dual(E, sp, 1, 2, 3, 4, 6.0, mode))
        tot, lit = q2.msed_stats()
        tx = timeit(lambda: q2.msed(qX, sp, 6.0, 5, 6, mode, "tape"))
        tw = timeit(lambda: q2.msed(qW, sp, 6.0, 7, 8, mode, "tape"))
        ne = T * out
        gbs = ne * 3.125 / td / 1e6
        print(f"E {T}x{out} {mode:8s}: dual {td * 1e3:7.1f} us ({gbs:6.0f} GB/s credited, {gbs / 6500.3:.2f} of HBM)"
              f"  X^T tape {tx * 1e3:6.1f} us ({T * inp / tx / 1e6:5.2f} Gelem/s)  W^T tape {tw * 1e3:6.1f} us"
              f"  literal {lit}/{tot}")
