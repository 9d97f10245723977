import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from tests.families import make, to_bf16
dev = lambda a: torch.from_numpy(a).cuda().bfloat16()
x = make("normal", (256, 384), seed=1); w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
e = dev(to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32)))
y, tape = q2.forward(dev(x), dev(w), q2.LayerConfig(posthoc=True))
S = q2.SeedPair(7, 9)
def bwd(sync):
    outs = []
    def s():
        if sync: torch.cuda.synchronize()
    qe = q2.msed(e, S, 6.0, q2.derive_stream(q2.PAIR_DX, 0), q2.PAIR_DX, "posthoc", "rows", err=torch.zeros(1, dtype=torch.int32, device="cuda")); s()
    qwt = q2.msed(tape.qW, S, 6.0, q2.derive_stream(q2.PAIR_DX, 1), q2.PAIR_DX, "posthoc", "tape", err=torch.zeros(1, dtype=torch.int32, device="cuda")); s()
    dx = q2.gemm(qe, qwt); s()
    qet = q2.msed(e, S, 6.0, q2.derive_stream(q2.PAIR_DW, 0), q2.PAIR_DW, "posthoc", "cols", err=torch.zeros(1, dtype=torch.int32, device="cuda")); s()
    qxt = q2.msed(tape.qX, S, 6.0, q2.derive_stream(q2.PAIR_DW, 1), q2.PAIR_DW, "posthoc", "tape", err=torch.zeros(1, dtype=torch.int32, device="cuda")); s()
    dw = q2.gemm(qet, qxt); s()
    torch.cuda.synchronize()
    return [t.to_reference() for t in (qe, qwt, qet, qxt)], dx, dw
for sync in (True, False):
    base = bwd(sync)
    for rep in range(4):
        r = bwd(sync)
        d = [(int(np.sum(a[0] != b[0])), int(np.sum(a[1] != b[1]))) for a, b in zip(r[0], base[0])]
        print("sync", sync, "rep", rep, "operand (codes,s8) diffs", d, "dx", (r[1] - base[1]).abs().max().item(), "dw", (r[2] - base[2]).abs().max().item())
