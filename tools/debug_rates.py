import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2
from paper_2601_22813_b200 import _lib
import ctypes
L = _lib.lib()
g = torch.Generator(device="cuda").manual_seed(0)
E = (1e-3 * torch.randn(16384, 11264, device="cuda", generator=g)).bfloat16()
T, N = E.shape
qr, qc = q2.NVFP4Tensor.empty((T, N), "cuda"), q2.NVFP4Tensor.empty((N, T), "cuda")
wr = torch.zeros(L.q2_msed_ws_bytes(T, N), dtype=torch.uint8, device="cuda"); wc = torch.zeros(L.q2_msed_ws_bytes(N, T), dtype=torch.uint8, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
a, b = qr.c(), qc.c()
S = q2.SeedPair(1, 2)
rc = L.q2_msed_dual_posthoc(E.data_ptr(), T, N, N, _lib._U32x4(*q2.sign_mask(1, 3)), _lib._U32x4(*q2.sign_mask(1, 4)), 6.0, 128 ** -0.5, 2, 5, 6, ctypes.byref(a), ctypes.byref(b), wr.data_ptr(), wc.data_ptr(), err.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
for name, w, R, K in (("rows", wr, T, N), ("cols", wc, N, T)):
    cnt = w[16:24].cpu().numpy().view(np.uint32)
    print(name, "chunks", R * K // 128, "listA (uncertain pass1)", cnt[0], f"{cnt[0] / (R*K/128) * 100:.2f}%", "listB (uncertain SR)", cnt[1], f"{cnt[1]/(R*K/16)*100:.3f}% of groups")
