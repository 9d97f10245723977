"""Generate golden vectors by running the REFERENCE (nvfp4emu) in this container.

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  The reference lives at /root/reference and
does not travel to the GPU box, so its outputs are frozen here; the oracle is
pinned against them by tests/test_oracle_pin.py.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

import nvfp4emu as R  # noqa: E402
from nvfp4emu import linear_graph as LG, ms_eden as ME, posthoc as PH, quantizers as Q, rht as RH  # noqa: E402

from tests.families import FAMILIES, make  # noqa: E402


ABLATION_CASES = [("ms_a", "rtn_1x16_46", "ms_eden", "a", False), ("ms_c", "rtn_1x16_46", "ms_eden", "c", False),
                  ("ms_e", "rtn_1x16_46", "ms_eden", "e", False), ("rht_b", "rtn_1x16", "sr_rht", "b", False),
                  ("rht_d", "rtn_1x16", "sr_rht", "d", False), ("sr46_a", "rtn_1x16_46", "sr_46", "a", False),
                  ("nv_b", "rtn_16x16", "sr_rht", "b", True), ("nv_c", "rtn_16x16", "sr_rht", "c", True),
                  ("nv_a", "rtn_16x16", "sr_rht", "a", True)]


def pack(prefix, t, out):
    out[prefix + "fp4"] = t.fp4
    out[prefix + "s8"] = t.scales8
    out[prefix + "s32"] = np.float32(t.scale32)


def main():
    out = {}
    seeds = RH.SeedPair(123, 456)
    for fam in FAMILIES:
        for bf16 in (True, False):
            x = make(fam, (64, 256), seed=31, bf16=bf16)
            key = f"{fam}_{'bf16' if bf16 else 'f32'}_"
            out[key + "x"] = x
            pack(key + "q46_", R.quantize_rtn_46(x), out)
            pack(key + "rtn_", R.quantize_rtn(x), out)
            pack(key + "msed_", ME.ms_eden_quantize(x, seeds, tensor_id=77, rotation_id=99), out)
            pack(key + "pow2_", ME.ms_eden_quantize(x, seeds, tensor_id=77, rotation_id=99, pow2_scale=True), out)
            er, red = PH.pass1(x, seeds.rht, tensor_id=77, rotation_id=99)
            pack(key + "posthoc_", PH.pass2(er, red, seeds.sr, tensor_id=77), out)
            # stochastic-rounding baselines (quantizers.py:139-161, :237-262); the
            # non-clipping AssertionError is recorded as a flag
            for tag, u46 in (("sq_", False), ("sq46_", True)):
                pack(key + tag, R.quantize_square_block(x, use_46=u46), out)
            for tag, fn in (("sr_", lambda v: R.quantize_sr(v, 123, 7)), ("sr46_", lambda v: R.quantize_sr_46(v, 123, 7)),
                            ("srrht_", lambda v: R.quantize_sr(RH.rht_apply(v, 11, 3), 5, 9))):
                try:
                    pack(key + tag, fn(x), out)
                except AssertionError:
                    out[key + tag + "assert"] = np.ones(1, dtype=np.uint8)
    # end-to-end digest case of SURVEY.md §8(c)
    rng = np.random.default_rng(2026)
    X = rng.standard_normal((128, 256)).astype(np.float32)
    W = (rng.standard_normal((256, 256)) / 16).astype(np.float32)
    E = (1e-2 * rng.standard_normal((128, 256))).astype(np.float32)
    y, tape = LG.forward(X, W, LG.baseline_config("quartet2"))
    g = LG.backward(tape, E, RH.SeedPair(7, 9))
    out.update(e2e_X=X, e2e_W=W, e2e_E=E, e2e_Y=y, e2e_dX=g.dX, e2e_dW=g.dW)
    pack("e2e_qX_", tape.qX, out)
    pack("e2e_qW_", tape.qW, out)
    # tetrajet_v2 baseline (rtn_1x16 forward, sr_rht backward) on the same data
    y, tape = LG.forward(X, W, LG.baseline_config("tetrajet_v2"))
    g = LG.backward(tape, E, RH.SeedPair(7, 9))
    out.update(tj_Y=y, tj_dX=g.dX, tj_dW=g.dW)
    for name, tag in (("nvidia", "nv"), ("four_over_six", "fos"), ("four_over_six_backward", "fosb")):
        y, tape = LG.forward(X, W, LG.baseline_config(name))
        g = LG.backward(tape, E, RH.SeedPair(7, 9))
        out.update({f"{tag}_Y": y, f"{tag}_dX": g.dX, f"{tag}_dW": g.dW})
    # ablation masks (linear_graph.py:59-70, :296): (forward, backward, ablation, reuse)
    for tag, fwd, bwd, abl, reuse in ABLATION_CASES:
        y, tape = LG.forward(X, W, LG.LayerConfig(fwd, bwd, ablation=abl, reuse_forward_weights=reuse))
        g = LG.backward(tape, E, RH.SeedPair(7, 9))
        out.update({f"abl_{tag}_dX": g.dX, f"abl_{tag}_dW": g.dW})
    # rotations (rht.py:121-163) on wide-range fp32 rows
    rx = (rng.standard_normal((6, 512)) * np.exp(rng.normal(0, 4, (6, 512)))).astype(np.float32)
    out.update(rot_x=rx, rot_apply128=RH.rht_apply(rx, 11, RH.derive_stream(1)),
               rot_apply32=RH.rht_apply(rx, 11, 5, chunk=32), rot_apply512=RH.rht_apply(rx, 3, 0, chunk=512),
               rot_inv128=RH.rht_inverse(rx, 11, RH.derive_stream(1)), rot_h128=RH.hadamard_128(rx.reshape(-1, 128)))
    # element formats (formats.py:76-229) on grid points, exact midpoints/ties and random values
    from nvfp4emu import formats as F
    g4 = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    x4 = np.concatenate([g4, -g4, (g4[:-1] + g4[1:]) / 2, -(g4[:-1] + g4[1:]) / 2, [-0.0, 6.0000000001, 7.5, np.inf],
                         rng.standard_normal(300) * 2.5]).astype(np.float64)
    x4sr = np.clip(x4, -6.0, 6.0)
    u4 = rng.random(x4.size)
    p8 = F.E4M3_VALUES[:127]
    x8 = np.concatenate([p8, (p8[:-1] + p8[1:]) / 2, [0.0, 2.0 ** -10, 2.0 ** -6 * 0.99, 440.0, 448.0, 500.0, np.inf],
                         np.exp(rng.normal(-2, 3, 300))]).astype(np.float64)
    x8sr = np.minimum(x8, 448.0)
    u8 = rng.random(x8.size)
    xe = np.concatenate([[0.0, 2.0 ** -126, 2.0 ** -127, 2.0 ** -127 * 1.01, 1.0625, 1.1875, 3.0e38],
                         np.exp(rng.normal(0, 20, 300))]).astype(np.float64)
    out.update(fmt_x4=x4, fmt_x4sr=x4sr, fmt_u4=u4, fmt_fp4_rtn=F.encode_fp4_rtn(x4),
               fmt_fp4_sr=F.encode_fp4_sr(x4sr, u4), fmt_x8=x8, fmt_x8sr=x8sr, fmt_u8=u8,
               fmt_fp8_rtn=F.encode_fp8_rtn(x8), fmt_fp8_sr=F.encode_fp8_sr(x8sr, u8), fmt_xe=xe,
               fmt_e8m3=F.round_e8m3_rtn(xe), fmt_dec_fp4=F.decode_fp4(np.arange(16)),
               fmt_dec_fp8=F.decode_fp8(np.arange(256)))
    # EDEN correction factors (ms_eden.py:57-83) on a rotated wide-range tensor, with
    # an all-zero chunk and a chunk whose quantization is zero (degenerate den)
    xf = (rng.standard_normal((8, 512)) * np.exp(rng.normal(0, 3, (8, 1)))).astype(np.float32).astype(np.float64)
    xf[2, 128:256] = 0.0
    xr = RH.rht_apply(xf, 5, 9)
    xr[5, 256:384] = xr[5, 256:384] * 1e-30
    xq = Q.dequantize(Q.quantize_rtn(xr))
    out.update(eden_xrot=xr, eden_xrtn=xq, eden_S=ME.chunk_correction_factors(xr, xq),
               eden_S1=np.array([ME.correction_factor(xr[0, :128], xq[0, :128])]))
    # NV4T container bytes (quantizers.py:330-348), dequantize (quantizers.py:315-323) and the
    # MS-EDEN GEMM-operand pair (ms_eden.py:156-180) on a normal and a wide-range input
    for tag, fam in (("n", "normal"), ("w", "lognormal_rows")):
        xs = make(fam, (96, 256), seed=41)
        t46 = R.quantize_rtn_46(xs)
        out[f"nv4t_{tag}_x"] = xs
        out[f"nv4t_{tag}_bytes"] = np.frombuffer(Q.serialize_nvfp4(t46), dtype=np.uint8)
        out[f"nv4t_{tag}_msed_bytes"] = np.frombuffer(
            Q.serialize_nvfp4(ME.ms_eden_quantize(xs, seeds, tensor_id=5, rotation_id=6)), dtype=np.uint8)
        out[f"deq_{tag}"] = Q.dequantize(t46)
        pa, pb = ME.ms_eden_estimate_pair(xs[:64], xs[32:], seeds, pair_id=RH.derive_stream(1))
        pack(f"pair_{tag}_a_", pa, out)
        pack(f"pair_{tag}_b_", pb, out)
    # PRNG known answers
    out["kat_bits"] = np.array([int(RH._bits(0, 0, 0)), int(RH._bits(123, 456, 789))], dtype=np.uint64)
    out["kat_uniform"] = RH.prng_uniform(0, 0, np.arange(4, dtype=np.uint64))
    out["kat_signs_pair_dx"] = RH._sign_vector(0, RH.derive_stream(1), 128)
    out["kat_streams"] = np.array([RH.derive_stream(1), RH.derive_stream(2), RH.derive_stream("mse-data", 0)],
                                  dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
