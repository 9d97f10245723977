"""Per-kernel timing at the c3 shapes (CUDA events, warm, L2-cold inputs).

    python tools/microbench.py [--only quant,msed,gemm]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="quant,msed,gemm")
    ap.add_argument("--T", type=int, default=16384)
    args = ap.parse_args()
    only = set(args.only.split(","))
    q2.set_error_mode("deferred")
    T = args.T
    g = torch.Generator(device="cuda").manual_seed(0)
    res = {}
    X = torch.randn(T, 2048, device="cuda", generator=g).bfloat16()
    E = (1e-3 * torch.randn(T, 11264, device="cuda", generator=g)).bfloat16()
    W = (torch.randn(11264, 2048, device="cuda", generator=g) / 45).bfloat16()
    seeds = q2.SeedPair(1, 2)
    if "quant" in only:
        for name, t in (("X 16384x2048", X), ("E 16384x11264", E)):
            ms = timeit(lambda: q2.quantize_rtn_46(t))
            res[f"quant46 {name}"] = {"ms": ms, "GB/s": t.numel() * 2.5625 / ms / 1e6}
        amax = torch.zeros(1, dtype=torch.int32, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        L = q2._lib.lib()
        ms = timeit(lambda: L.q2_amax(E.data_ptr(), 0, E.shape[0], E.shape[1], E.shape[1], amax.data_ptr(),
                                      err.data_ptr(), torch.cuda.current_stream().cuda_stream))
        res["amax E"] = {"ms": ms, "GB/s": E.numel() * 2 / ms / 1e6}
    if "msed" in only:
        for mode in ("posthoc", "exact"):
            ms = timeit(lambda: q2.msed(E, seeds, 6.0, 1, 2, mode, "rows"))
            res[f"msed rows {mode} E"] = {"ms": ms, "GB/s": E.numel() * 2.5625 / ms / 1e6}
            ms = timeit(lambda: q2.msed(E, seeds, 6.0, 1, 2, mode, "cols"))
            res[f"msed cols {mode} E"] = {"ms": ms, "GB/s": E.numel() * 2.5625 / ms / 1e6}
            if mode == "posthoc":
                ms = timeit(lambda: q2.msed_dual_posthoc(E, seeds, 1, 2, 3, 4))
                res["msed dual posthoc E (rows+cols)"] = {"ms": ms, "GB/s": E.numel() * 3.125 / ms / 1e6}
            qw = q2.quantize_rtn_46(W)
            ms = timeit(lambda: q2.msed(qw, seeds, 6.0, 1, 2, mode, "tape"))
            res[f"msed tape {mode} W"] = {"ms": ms, "GB/s": W.numel() * 1.125 / ms / 1e6}
            qx = q2.quantize_rtn_46(X)
            ms = timeit(lambda: q2.msed(qx, seeds, 6.0, 1, 2, mode, "tape"))
            res[f"msed tape {mode} X"] = {"ms": ms, "GB/s": X.numel() * 1.125 / ms / 1e6}
    if "gemm" in only:
        for name, (m, n, k) in (("fprop upgate", (T, 11264, 2048)), ("dgrad upgate", (T, 2048, 11264)),
                                ("wgrad upgate", (11264, 2048, T)), ("fprop o", (T, 2048, 2048)),
                                ("square 8192", (8192, 8192, 8192))):
            a = torch.randn(m, k, device="cuda", generator=g).bfloat16()
            b = torch.randn(n, k, device="cuda", generator=g).bfloat16()
            qa, qb = q2.quantize_rtn_46(a), q2.quantize_rtn_46(b)
            out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            ms = timeit(lambda: q2.gemm(qa, qb, out=out))
            msb = timeit(lambda: torch.matmul(a, b.t(), out=out))
            res[f"gemm {name} {m}x{n}x{k}"] = {"ms": ms, "TFLOP/s": 2 * m * n * k / ms / 1e9,
                                               "bf16_TFLOP/s": 2 * m * n * k / msb / 1e9}
            del a, b, qa, qb, out
    q2.check_errors()
    for k, v in res.items():
        print(f"{k:40s} " + "  ".join(f"{a}={b:.3f}" for a, b in v.items()))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
