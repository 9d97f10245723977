"""One launch of each hot kernel at c3 shapes (for ncu --set full)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
q2.set_error_mode("deferred")
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(16384, 2048, device="cuda", generator=g).bfloat16()
W = (torch.randn(11264, 2048, device="cuda", generator=g) / 45).bfloat16()
E = (1e-3 * torch.randn(16384, 11264, device="cuda", generator=g)).bfloat16()
S = q2.SeedPair(1, 2)
for _ in range(2):
    qx, qw = q2.quantize_rtn_46(X), q2.quantize_rtn_46(W)
    y = q2.gemm(qx, qw, torch.bfloat16)
    qe = q2.msed(E, S, 6.0, 1, 2, "posthoc", "rows")
    qet = q2.msed(E, S, 6.0, 3, 4, "posthoc", "cols")
    qxt = q2.msed(qx, S, 6.0, 5, 4, "posthoc", "tape")
    torch.cuda.synchronize()
q2.check_errors()
