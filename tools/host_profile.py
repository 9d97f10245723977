"""cProfile of eager forward/backward calls (host-side overhead per projection).

    python tools/host_profile.py
"""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402

q2.set_error_mode("deferred")
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(16384, 2048, device="cuda", generator=g).bfloat16()
W = (torch.randn(2048, 2048, device="cuda", generator=g) / 45).bfloat16()
E = (1e-3 * torch.randn(16384, 2048, device="cuda", generator=g)).bfloat16()
cfg = q2.LayerConfig(posthoc=True)


def step():
    for _ in range(10):
        y, tape = q2.forward(X, W, cfg, out_dtype=torch.bfloat16)
        q2.backward(tape, E, q2.SeedPair(1, 2), dx_dtype=torch.bfloat16)


step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
