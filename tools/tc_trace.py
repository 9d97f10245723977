import os, sys, torch
sys.path.insert(0, '.')
import paper_2601_22813_b200 as q2
E = torch.randn(16384, 11264, device='cuda').mul_(1e-3).to(torch.bfloat16)
q2.msed_dual(E, q2.SeedPair(1, 2), 1, 2, 3, 4, 6.0, "posthoc")
torch.cuda.synchronize()
