import os, sys, torch
sys.path.insert(0, '/root/repo')
import paper_2601_22813_b200 as q2
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(16384, 2048, device="cuda", generator=g).bfloat16()
W = (torch.randn(11264, 2048, device="cuda", generator=g) / 45).bfloat16()
qx, qw = q2.quantize_rtn_46(X), q2.quantize_rtn_46(W)
for _ in range(3):
    y = q2.gemm(qx, qw, torch.bfloat16)
torch.cuda.synchronize()
