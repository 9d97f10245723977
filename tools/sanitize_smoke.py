"""One small call of every kernel family, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
    compute-sanitizer --tool synccheck python tools/sanitize_smoke.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22813_b200 as q2  # noqa: E402


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    T, DIN, DOUT = 256, 256, 384
    X = torch.randn(T, DIN, device="cuda", generator=g).bfloat16()
    W = (torch.randn(DOUT, DIN, device="cuda", generator=g) / 16).bfloat16()
    E = (1e-2 * torch.randn(T, DOUT, device="cuda", generator=g)).bfloat16()
    for name in ("quartet2", "tetrajet_v2", "nvidia", "four_over_six", "four_over_six_backward"):
        for posthoc in (False, True):
            cfg = q2.baseline_config(name)
            cfg = q2.LayerConfig(cfg.forward_scheme, cfg.backward_scheme, posthoc=posthoc,
                                 reuse_forward_weights=cfg.reuse_forward_weights)
            y, tape = q2.forward(X, W, cfg, out_dtype=torch.bfloat16)
            gr = q2.backward(tape, E, q2.SeedPair(3, 4), dx_dtype=torch.bfloat16)
            torch.cuda.synchronize()
            print(name, posthoc, float(y.float().norm()), float(gr.dX.float().norm()), float(gr.dW.norm()))
    # exact-mode MS-EDEN on fp32 input, pow2, dual posthoc, serialization round trip
    xf = torch.randn(256, 512, device="cuda", generator=g)
    q2.ms_eden_quantize(xf, q2.SeedPair(1, 2), tensor_id=5)
    q2.ms_eden_quantize(xf, q2.SeedPair(1, 2), tensor_id=5, pow2_scale=True)
    t = q2.quantize_rtn_46(xf)
    assert q2.deserialize_nvfp4(q2.serialize_nvfp4(t)).to_reference()[2] == t.to_reference()[2]
    # standalone ops: rotations, formats, EDEN factors, ablation masks
    r = q2.rht_apply(xf, 3, 4, chunk=256)
    q2.rht_inverse(r, 3, 4, chunk=256)
    q2.hadamard_128(xf[:, :128])
    from paper_2601_22813_b200 import formats as F
    F.encode_fp4_rtn(xf), F.encode_fp4_sr(xf.clamp(-6, 6), torch.rand_like(xf))
    F.encode_fp8_rtn(xf.abs()), F.encode_fp8_sr(xf.abs().clamp(max=448), torch.rand_like(xf))
    F.round_e8m3_rtn(xf.abs()), F.decode_fp4(torch.arange(16)), F.decode_fp8(torch.arange(256))
    q2.ms_eden.chunk_correction_factors(r, r * 0.5)
    for abl in ("a", "b", "c", "d"):
        cfg = q2.LayerConfig("rtn_1x16", "sr_rht", ablation=abl)
        y, tape = q2.forward(X, W, cfg)
        q2.backward(tape, E, q2.SeedPair(3, 4))
    m = q2.Quartet2Linear(256, 128, bias=True, device="cuda")
    m(X).float().sum().backward()
    torch.cuda.synchronize()
    q2.check_errors()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
