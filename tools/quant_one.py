"""One forward 4/6 quantization of a c3 activation (16384 x 5632 bf16) for ncu."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
K = int(os.environ.get("QK", "5632"))
x = torch.randn(16384, K, device="cuda").bfloat16()
for _ in range(2):
    q2.quantize_rtn_46(x)
torch.cuda.synchronize()
