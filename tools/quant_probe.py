"""Forward-quantizer timing at the bench shapes: amax + quantize pass vs the amax
pass alone (CUDA events, L2 flushed).

    python tools/quant_probe.py
"""

import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402
from paper_2601_22813_b200 import _lib  # noqa: E402
from paper_2601_22813_b200.quantizers import NVFP4Tensor, stream_handle  # noqa: E402


def main():
    L = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, R, K, sc in (("X 16384x2048", 16384, 2048, 1.0), ("X 16384x5632", 16384, 5632, 1.0),
                           ("W 11264x2048", 11264, 2048, 2048 ** -0.5), ("W 2048x2048", 2048, 2048, 2048 ** -0.5),
                           ("W 2048x5632", 2048, 5632, 5632 ** -0.5)):
        x = (torch.randn(R, K, device="cuda", generator=g) * sc).bfloat16()
        out = NVFP4Tensor.empty((R, K), "cuda")
        t = out.c()
        ws = torch.zeros(L.q2_quant_fwd_ws_bytes(R, K), dtype=torch.uint8, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        run = lambda: L.q2_quant_fwd(x.data_ptr(), 0, R, K, K, 2, 6.0, 4.0, 6.0 * 448.0, ctypes.byref(t),
                                     ws.data_ptr(), err.data_ptr(), stream_handle())
        amax = lambda: L.q2_amax(x.data_ptr(), 0, R, K, K, ws.data_ptr(), err.data_ptr(), stream_handle())
        for fn, lab in ((run, "quant_fwd total"), (amax, "amax only")):
            for _ in range(3):
                fn()
            tot = 0.0
            for _ in range(20):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                fn()
                e.record()
                torch.cuda.synchronize()
                tot += s.elapsed_time(e)
            us = tot / 20 * 1e3
            gb = R * K * (2.5625 if lab.startswith("quant") else 2) / us / 1e3
            print(f"{name:16s} {lab:16s} {us:8.1f} us  {gb:7.0f} GB/s credited (2.5625 B/elem, amax incl.)"
                  if lab.startswith("quant") else f"{name:16s} {lab:16s} {us:8.1f} us  {gb:7.0f} GB/s")


if __name__ == "__main__":
    main()
