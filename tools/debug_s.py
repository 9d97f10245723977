import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_22813_b200 import _lib
_lib._LIB = _lib.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libq2_debug.so"))
import paper_2601_22813_b200 as q2
from oracle import nvfp4_oracle as O
from tests.families import make
x = make("normal", (64, 256), seed=5)
L = q2._lib.lib(); R, K = x.shape
ws = torch.zeros(L.q2_msed_ws_bytes(R, K), dtype=torch.uint8, device="cuda")
try:
    q2.msed(torch.from_numpy(x).cuda().bfloat16(), q2.SeedPair(123, 456), 6.0, 77, 99, "posthoc", "rows", ws=ws)
except Exception as e: print("exc", e)
torch.cuda.synchronize()
al = lambda v: (v + 255) // 256 * 256
g, ch = R * K // 16, R * K // 128
b = ws.cpu().numpy(); c0 = 256 + al(g * 2); corr = b[c0:c0 + ch * 8].view(np.float64); d0 = c0 + al(ch * 8); dS = b[d0:d0 + ch * 4].view(np.float32)
xr = O.rht_apply(x, 123, 99); er, rd = O.pass1(x, 123, tensor_id=77, rotation_id=99)
deq = (O.FP4_VALUES[er.fp4].reshape(-1, 16) * er.pseudo_scales.reshape(-1, 1)).reshape(x.shape)
c = 128 ** -0.5
num_ref = (xr.reshape(-1, 128) ** 2).sum(-1) / c**2
den_ref = (xr.reshape(-1, 128) * deq.reshape(-1, 128)).sum(-1) / c
print("num got", dS[:4], "ref", num_ref[:4]); print("den got", corr[:4], "ref", den_ref[:4])
