"""Scale-replica probe: GEMM output with Q2_GEMM_DBG variants vs the normal path."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2601_22813_b200 as q2
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(512, 1024, device="cuda", generator=g).bfloat16()
b = torch.randn(512, 1024, device="cuda", generator=g).bfloat16()
qa, qb = q2.quantize_rtn_46(a), q2.quantize_rtn_46(b)
y = q2.gemm(qa, qb, torch.float32)
p = "gpurun_out/gemm_ref.pt"
if os.environ.get("Q2_GEMM_DBG", "0") == "0":
    torch.save(y.cpu(), p)
else:
    r = torch.load(p)
    print(os.environ.get("Q2_GEMM_DBG"), "max abs diff", float((y.cpu() - r).abs().max()), "ref max", float(r.abs().max()))
