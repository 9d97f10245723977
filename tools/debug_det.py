import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from tests.families import make, to_bf16
dev = lambda a: torch.from_numpy(a).cuda().bfloat16()
for (m, n, k) in [(256, 384, 256), (1024, 768, 2048), (2048, 2048, 4096)]:
    a, b = make("normal", (m, k), 1), make("normal", (n, k), 2)
    qa, qb = q2.quantize_rtn_46(dev(a)), q2.quantize_rtn_46(dev(b))
    outs = [q2.gemm(qa, qb).clone() for _ in range(20)]
    torch.cuda.synchronize()
    print("gemm", (m, n, k), "max diff across runs", max((o - outs[0]).abs().max().item() for o in outs))
x = make("normal", (256, 384), seed=1); w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
for posthoc in (False, True):
    y, tape = q2.forward(dev(x), dev(w), q2.LayerConfig(posthoc=posthoc))
    res = []
    for _ in range(5):
        g = q2.backward(tape, dev(e), q2.SeedPair(7, 9))
        res.append((g.dX.clone(), g.dW.clone()))
    torch.cuda.synchronize()
    print("posthoc", posthoc, "dx diffs", [ (r[0] - res[0][0]).abs().max().item() for r in res], "dw", [(r[1] - res[0][1]).abs().max().item() for r in res])
    # operand determinism in layer order
    mode = "posthoc" if posthoc else "exact"
    qs = []
    for _ in range(5):
        qe = q2.msed(dev(e), q2.SeedPair(7, 9), 6.0, 5, q2.PAIR_DX, mode, "rows")
        qwt = q2.msed(tape.qW, q2.SeedPair(7, 9), 6.0, 6, q2.PAIR_DX, mode, "tape")
        qs.append((qe.to_reference(), qwt.to_reference()))
    for i in range(1, 5):
        print(" rep", i, "E codes diff", np.sum(qs[i][0][0] != qs[0][0][0]), "E s8 diff", np.sum(qs[i][0][1] != qs[0][0][1]), "Wt codes", np.sum(qs[i][1][0] != qs[0][1][0]), "Wt s8", np.sum(qs[i][1][1] != qs[0][1][1]))
