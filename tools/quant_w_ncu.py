"""Forward quantizer at weight shapes for ncu (kernel durations: amax vs quant)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402
g = torch.Generator(device="cuda").manual_seed(0)
for R, K in ((2048, 2048), (11264, 2048), (16384, 2048)):
    x = (torch.randn(R, K, device="cuda", generator=g) * K ** -0.5).bfloat16()
    for _ in range(2):
        q2.quantize_rtn_46(x)
torch.cuda.synchronize()
