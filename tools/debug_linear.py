import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from oracle import nvfp4_oracle as O
from tests.families import make, to_bf16
x = make("normal", (256, 384), seed=1); w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
dev = lambda a: torch.from_numpy(a).cuda().bfloat16()
S = q2.SeedPair(7, 9); RS = O.SeedPair(7, 9)
qx, qw = q2.quantize_rtn_46(dev(x)), q2.quantize_rtn_46(dev(w))
rqx, rqw = O.quantize_rtn_46(x), O.quantize_rtn_46(w)
def cmp(name, got, ref):
    f, s8, s32 = got.to_reference()
    print(f"{name:10s} scale32 {'ok' if s32 == ref.scale32 else 'BAD'}  codes bad {np.sum(f != ref.fp4)}  scales bad {np.sum(s8 != ref.scales8)}")
for mode in ("exact", "posthoc"):
    rq = O.posthoc_quantize if mode == "posthoc" else O.ms_eden_quantize
    print("mode", mode)
    cmp("E rows", q2.msed(dev(e), S, 6.0, q2.derive_stream(q2.PAIR_DX, 0), q2.PAIR_DX, mode, "rows"), rq(e, RS, 6.0, O.derive_stream(O.PAIR_DX, 0), O.PAIR_DX))
    cmp("W^T tape", q2.msed(qw, S, 6.0, q2.derive_stream(q2.PAIR_DX, 1), q2.PAIR_DX, mode, "tape"), rq(np.ascontiguousarray(O.dequantize(rqw).T), RS, 6.0, O.derive_stream(O.PAIR_DX, 1), O.PAIR_DX))
    cmp("E^T cols", q2.msed(dev(e), S, 6.0, q2.derive_stream(q2.PAIR_DW, 0), q2.PAIR_DW, mode, "cols"), rq(np.ascontiguousarray(e.T), RS, 6.0, O.derive_stream(O.PAIR_DW, 0), O.PAIR_DW))
    cmp("X^T tape", q2.msed(qx, S, 6.0, q2.derive_stream(q2.PAIR_DW, 1), q2.PAIR_DW, mode, "tape"), rq(np.ascontiguousarray(O.dequantize(rqx).T), RS, 6.0, O.derive_stream(O.PAIR_DW, 1), O.PAIR_DW))
