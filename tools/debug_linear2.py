import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from oracle import nvfp4_oracle as O
from tests.families import make, to_bf16
x = make("normal", (256, 384), seed=1); w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
dev = lambda a: torch.from_numpy(a).cuda().bfloat16()
for posthoc in (False, True, True, True):
    y, tape = q2.forward(dev(x), dev(w), q2.LayerConfig(posthoc=posthoc))
    g = q2.backward(tape, dev(e), q2.SeedPair(7, 9))
    ry, rt = O.forward(x, w); rdx, rdw = O.backward(rt, e, O.SeedPair(7, 9), posthoc=posthoc)
    rel = lambda a, b: np.linalg.norm(a.double().cpu().numpy() - b) / np.linalg.norm(b)
    print(posthoc, "y", rel(y, ry), "dx", rel(g.dX, rdx), "dw", rel(g.dW, rdw))
    # recompute gemm from quantized operands
