"""Tensor-core MS-EDEN timing probe: per-source time and literal-chunk rate at one c3 shape.
Run with Q2_TC_DBG=1..4 to time the pipeline with parts of the work removed."""
import os
import sys
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2

dev = torch.device("cuda:0")
q2.set_msed_engine(os.environ.get("Q2_ENGINE", "tc"))
T, inp, out = 16384, int(os.environ.get("IN", "2048")), int(os.environ.get("OUT", "11264"))


q2.set_error_mode("deferred")


def timeit(fn, iters=10):
    """Device time per call: iters calls captured in one CUDA graph (no host overhead)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / iters * 1e3


E = torch.randn(T, out, device=dev).mul_(1e-3).to(torch.bfloat16)
X = torch.randn(T, inp, device=dev).to(torch.bfloat16)
qX = q2.quantize_rtn_46(X)
sp = q2.SeedPair(1, 2)
for mode in ("posthoc", "exact"):
    for name, fn in (("dual E", lambda: q2.msed_dual(E, sp, 1, 2, 3, 4, 6.0, mode)),
                     ("tape X^T", lambda: q2.msed(qX, sp, 6.0, 5, 6, mode, "tape"))):
        q2.msed_stats(reset=True)
        t = timeit(fn)
        tot, lit = q2.msed_stats()
        print(f"dbg={os.environ.get('Q2_TC_DBG', '0')} {mode:8s} {name:9s} {t:8.1f} us  literal {lit / max(tot, 1):.4%}")
