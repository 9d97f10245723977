"""Time msed_dual (posthoc/exact) and the tape source at the c3 UpGate shape under the
current Q2_TC_DBG setting (1: epilogue drains only, 2: + no split work, 3: no small MMA,
4: no MMA) -- locates the tensor-core MS-EDEN bottleneck."""
import os
import sys
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2

dev = torch.device("cuda:0")
T, out = 16384, int(os.environ.get("PROF_OUT", "11264"))
E = torch.randn(T, out, device=dev).mul_(1e-3).to(torch.bfloat16)
X = torch.randn(T, 2048, device=dev).to(torch.bfloat16)
qX = q2.quantize_rtn_46(X)
sp = q2.SeedPair(1, 2)
q2.set_msed_engine(os.environ.get("Q2_ENGINE", "tc"))


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(iters):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / iters * 1e3


q2.set_error_mode("deferred")
r = {}
for mode in ("posthoc", "exact"):
    r["dual_" + mode] = timeit(lambda: q2.msed_dual(E, sp, 1, 2, 3, 4, 6.0, mode))
    r["tape_" + mode] = timeit(lambda: q2.msed(qX, sp, 6.0, 5, 6, mode, "tape"))
print("DBG", os.environ.get("Q2_TC_DBG", "0"), " ".join(f"{k}={v:.1f}us" for k, v in r.items()))
