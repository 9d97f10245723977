"""Deferral reasons of the tensor-core MS-EDEN epilogue (needs a library built with the
g_tc_why counters: tools/libq2_why.so via Q2_LIB_OVERRIDE)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from paper_2601_22813_b200 import _lib
L = _lib.lib()
E = torch.randn(16384, 11264, device="cuda").mul_(1e-3).to(torch.bfloat16)
q2.msed_stats(reset=True)
q2.msed_dual(E, q2.SeedPair(1, 2), 1, 2, 3, 4, 6.0, "posthoc")
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
L.q2_tc_why(buf)
tot, lit = q2.msed_stats()
v = list(buf)
print("chunks", tot, "literal", lit)
print("scale-uncertain groups", v[0], "sign-check groups exact/nonexact", v[1] & 0xFFFFFFFF, v[1] >> 32,
      "code-mismatch groups (non-exact)", v[2], "S degenerate chunks", v[3], "SR-uncertain groups", v[4])
