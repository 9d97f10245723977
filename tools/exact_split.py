"""Per-kernel device time of the MS-EDEN calls at one c3 shape (torch.profiler / CUPTI),
both modes: splits the exact mode into its absmax and quantize passes."""
import os
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2

dev = torch.device("cuda:0")
q2.set_error_mode("deferred")
T, inp, out = 16384, int(os.environ.get("IN", "2048")), int(os.environ.get("OUT", "11264"))
E = torch.randn(T, out, device=dev).mul_(1e-3).to(torch.bfloat16)
X = torch.randn(T, inp, device=dev).to(torch.bfloat16)
qX = q2.quantize_rtn_46(X)
sp = q2.SeedPair(1, 2)
REPS = 5
for mode in ("posthoc", "exact"):
    for name, fn in (("dual E", lambda: q2.msed_dual(E, sp, 1, 2, 3, 4, 6.0, mode)),
                     ("tape X^T", lambda: q2.msed(qX, sp, 6.0, 5, 6, mode, "tape"))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(REPS):
                fn()
            torch.cuda.synchronize()
        acc = defaultdict(float)
        for ev in prof.events():
            if ev.device_type == torch.autograd.DeviceType.CUDA:
                acc[ev.name] += ev.device_time / REPS
        tot = sum(acc.values())
        print(f"{mode:8s} {name:9s} total {tot:8.1f} us: " +
              ", ".join(f"{k[:40]} {v:.1f}" for k, v in sorted(acc.items(), key=lambda kv: -kv[1])))
