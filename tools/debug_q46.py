"""Diagnose 4/6 forward-quantizer scale mismatches against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402
from oracle import nvfp4_oracle as O  # noqa: E402
from tests.families import make  # noqa: E402

x = make("normal", (192, 512), seed=11)
t = q2.quantize_rtn_46(torch.from_numpy(x).cuda().bfloat16())
fp4, s8, s32 = t.to_reference()
ref = O.quantize_rtn_46(x)
bad = np.argwhere(s8 != ref.scales8)
print("scale32", s32, ref.scale32, "bad groups", len(bad))
thr = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])
for r, j in bad[:6]:
    g = x[r, 16 * j:16 * j + 16].astype(np.float64)
    gm = np.abs(g).max()
    for c in (6.0, 4.0):
        y = gm / (float(ref.scale32) * c)
        k = O.e4m3_rtn(y)
        d = O.E4M3_VALUES[k] * float(ref.scale32)
        codes, err = O.rtn_codes(g, np.array([d]), want_err=True)
        rho = np.abs(g) / d
        print(f"  ({r},{j}) cap {c}: y={y!r} s8={int(k)} err={err[0]!r} ties={int(np.isin(rho, thr).sum())}")
    print(f"  gpu s8={s8[r, j]} ref s8={ref.scales8[r, j]} gpu codes==ref: {np.array_equal(fp4[r,16*j:16*j+16], ref.fp4[r,16*j:16*j+16])}")
