import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from oracle import nvfp4_oracle as O
from tests.families import make
x = make("normal", (64, 256), seed=5)
L = q2._lib.lib()
R, K = x.shape
ws = torch.zeros(L.q2_msed_ws_bytes(R, K), dtype=torch.uint8, device="cuda")
t = q2.msed(torch.from_numpy(x).cuda().bfloat16(), q2.SeedPair(123, 456), 6.0, 77, 99, "posthoc", "rows", ws=ws)
torch.cuda.synchronize()
al = lambda v: (v + 255) // 256 * 256
g, ch = R * K // 16, R * K // 128
b = ws.cpu().numpy()
red = b[:16].view(np.float64); cnt = b[16:24].view(np.uint32)
p0 = 256; pseudo = b[p0:p0 + g * 2].view(np.uint16)
c0 = p0 + al(g * 2); corr = b[c0:c0 + ch * 8].view(np.float64)
d0 = c0 + al(ch * 8); dS = b[d0:d0 + ch * 4].view(np.float32)
er, rd = O.pass1(x, 123, tensor_id=77, rotation_id=99)
ps_ref = er.pseudo_scales.reshape(-1).astype(np.float32).view(np.uint32) >> 16
print("red", red, "counts", cnt, "pmax ref", er.pseudo_scales.max())
print("pseudo equal", np.mean(pseudo == ps_ref))
print("corr ref", rd.corrections.reshape(-1)[:6]); print("corr got", corr[:6]); print("dS", dS[:6])
print("codes equal", np.mean(t.fp4 == er.fp4))
rel = np.abs(corr - rd.corrections.reshape(-1)) / np.abs(rd.corrections.reshape(-1))
print("max rel corr err", rel.max(), "max dS", dS.max(), "violations", np.sum(rel > dS))
