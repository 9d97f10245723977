import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2601_22813_b200 as q2
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(16384, 2048, device="cuda", generator=g).bfloat16()
b = torch.randn(11264, 2048, device="cuda", generator=g).bfloat16()
qa, qb = q2.quantize_rtn_46(a), q2.quantize_rtn_46(b)
out = torch.empty(16384, 11264, device="cuda", dtype=torch.bfloat16)
for _ in range(3): q2.gemm(qa, qb, out=out)
torch.cuda.synchronize()
os.environ["Q2_GEMM_TRACE"] = "1"
q2.gemm(qa, qb, out=out)
torch.cuda.synchronize()
