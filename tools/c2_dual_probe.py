"""c2-shaped MS-EDEN timing ([N/4096, 4096] bf16, N(0,1) x LogNormal(0,1) per row), graph-timed."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from tools.tc_probe import timeit
for lg in (24, 28):
    n = 1 << lg
    x = (torch.randn(n // 4096, 4096, device="cuda") * torch.randn(n // 4096, 1, device="cuda").exp()).bfloat16()
    sp = q2.SeedPair(1, 2)
    for mode in ("posthoc",):
        for tag, fn in (("rows", lambda: q2.msed(x, sp, 6.0, 1, 2, mode, "rows")), ("dual", lambda: q2.msed_dual(x, sp, 1, 2, 3, 4, 6.0, mode))):
            q2.msed_stats(reset=True)
            t = timeit(fn)
            tot, lit = q2.msed_stats()
            print(f"2^{lg} {mode} {tag}: {t:8.1f} us  literal {lit / max(tot, 1):.3%}")
