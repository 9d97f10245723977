"""One dual MS-EDEN (posthoc) call at c3 UpGate for ncu: E 16384 x 11264 bf16."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402
q2.set_error_mode("deferred")
E = torch.randn(16384, int(os.environ.get("OUT", "11264")), device="cuda").mul_(1e-3).to(torch.bfloat16)
X = torch.randn(16384, 2048, device="cuda").to(torch.bfloat16)
W = (torch.randn(int(os.environ.get("OUT", "11264")), 2048, device="cuda") / 45).to(torch.bfloat16)
cfg = q2.LayerConfig(posthoc=True)
y, tape = q2.forward(X, W, cfg, out_dtype=torch.bfloat16)
for _ in range(2):
    q2.backward(tape, E, q2.SeedPair(3, 4), dx_dtype=torch.bfloat16)
torch.cuda.synchronize()
