"""One tensor-core MS-EDEN launch per kind at a c3 shape, for ncu (-k regex:msed_tc)."""
import os
import sys
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2

dev = torch.device("cuda:0")
T, inp, out = 16384, 2048, int(os.environ.get("PROF_OUT", "11264"))
mode = os.environ.get("PROF_MODE", "posthoc")
E = torch.randn(T, out, device=dev).mul_(1e-3).to(torch.bfloat16)
X = torch.randn(T, inp, device=dev).to(torch.bfloat16)
qX = q2.quantize_rtn_46(X)
sp = q2.SeedPair(1, 2)
q2.set_msed_engine(os.environ.get("PROF_ENGINE", "auto"))
for _ in range(2):
    q2.msed_dual(E, sp, 1, 2, 3, 4, 6.0, mode)
    q2.msed(qX, sp, 6.0, 5, 6, mode, "tape")
torch.cuda.synchronize()
