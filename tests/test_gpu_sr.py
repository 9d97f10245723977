"""GPU parity of the stochastic-rounding baselines against the oracle.

quantize_sr / quantize_sr_46 (quantizers.py:139-161, :237-262), the rotated
sr_rht operand quantizer from every source (linear_graph.py:259-274), and the
tetrajet_v2 linear pass (rtn_1x16 forward, sr_rht backward).  Codes, scales
and scale32 bit-exact; GEMM outputs within the tolerance of test_gpu_parity.
"""

import os

import numpy as np
import pytest

from oracle import nvfp4_oracle as O
from tests.families import FAMILIES, make, to_bf16
from tests.test_gpu_parity import _dev, _q2, assert_same

pytestmark = pytest.mark.gpu


def _raises_or_same(gpu_fn, ref_fn, what):
    try:
        ref = ref_fn()
    except AssertionError:
        with pytest.raises(AssertionError, match="encoder bug"):
            gpu_fn()
        return
    assert_same(gpu_fn(), ref, what)


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("bf16", [True, False])
def test_quantize_sr(cuda, family, bf16):
    q2 = _q2()
    x = make(family, (192, 512), seed=13, bf16=bf16)
    _raises_or_same(lambda: q2.quantize_sr(_dev(x, bf16), 123, 7), lambda: O.quantize_sr(x, 123, 7), f"sr[{family}]")


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("bf16", [True, False])
def test_quantize_sr_46(cuda, family, bf16):
    q2 = _q2()
    x = make(family, (192, 512), seed=14, bf16=bf16)
    assert_same(q2.quantize_sr_46(_dev(x, bf16), 321, 5), O.quantize_sr_46(x, 321, 5), f"sr46[{family}]")


def test_quantize_sr_zero(cuda):
    q2 = _q2()
    z = np.zeros((64, 256), np.float32)
    assert_same(q2.quantize_sr(_dev(z), 1, 2), O.quantize_sr(z, 1, 2), "sr zero")
    assert_same(q2.quantize_sr_46(_dev(z), 1, 2), O.quantize_sr_46(z, 1, 2), "sr46 zero")


@pytest.mark.parametrize("family", ["normal", "t2", "zero_rows", "outliers", "tie_grid"])
@pytest.mark.parametrize("source", ["rows", "cols", "tape"])
def test_rht_sr(cuda, family, source):
    """quantize_sr(rht_apply(x)) without materialising the rotation or the transpose."""
    q2 = _q2()
    seeds = q2.SeedPair(11, 17)
    x = make(family, (256, 384), seed=15)                       # rows: [R=256, K=384]
    if source == "rows":
        gpu_fn = lambda: q2.rht_sr(_dev(x), seeds, 99, 7, "rows")        # noqa: E731
        logical = x
    elif source == "cols":
        gpu_fn = lambda: q2.rht_sr(_dev(x), seeds, 99, 7, "cols")        # noqa: E731  logical x^T [384, 256]
        logical = np.ascontiguousarray(x.T)
    else:
        qx = q2.quantize_rtn_46(_dev(x), caps=(6.0,))
        gpu_fn = lambda: q2.rht_sr(qx, seeds, 99, 7, "tape")             # noqa: E731  logical dequant(x)^T
        logical = np.ascontiguousarray(O.dequantize(O.quantize_rtn_46(x, caps=(6.0,))).T)
    ref_fn = lambda: O.quantize_sr(O.rht_apply(logical, 11, 7), 17, 99)   # noqa: E731
    _raises_or_same(gpu_fn, ref_fn, f"rht_sr {source} [{family}]")


def test_tetrajet_v2_linear(cuda):
    """rtn_1x16 forward + sr_rht backward (linear_graph.py:119-140 'tetrajet_v2')."""
    q2 = _q2()
    x = make("normal", (256, 384), seed=1)
    w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
    e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
    cfg = q2.baseline_config("tetrajet_v2")
    y, tape = q2.forward(_dev(x), _dev(w), cfg)
    g = q2.backward(tape, _dev(e), q2.SeedPair(7, 9))
    ry, rtape = O.forward(x, w, forward_scheme="rtn_1x16")
    assert_same(tape.qX, rtape[0], "qX")
    assert_same(tape.qW, rtape[1], "qW")
    rdx, rdw = O.backward(rtape, e, O.SeedPair(7, 9), backward_scheme="sr_rht")
    for got, ref in ((y, ry), (g.dX, rdx), (g.dW, rdw)):
        got = got.double().cpu().numpy()
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-5, rel


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("use_46", [False, True])
def test_quantize_square_block(cuda, family, use_46):
    """16x16 blocks (quantizers.py:265-312): codes, block scales, scale32; the transposed
    copy holds the same codes and the same (expanded) block scales."""
    q2 = _q2()
    x = make(family, (96, 160), seed=16)
    t = q2.quantize_square_block(_dev(x), use_46)
    ref = O.quantize_square_block(x, use_46)
    fp4, s8, s32 = t.to_reference()
    assert np.float32(s32).tobytes() == np.float32(ref.scale32).tobytes()
    np.testing.assert_array_equal(s8, ref.scales8)
    np.testing.assert_array_equal(fp4, ref.fp4)
    tf, ts, _ = t.t.to_reference()
    np.testing.assert_array_equal(tf, ref.fp4.T)
    np.testing.assert_array_equal(ts, np.repeat(ref.scales8.T, 16, axis=0))
    one_col = make(family, (64, 16), seed=17)                           # single block column: flat sum order
    got = q2.quantize_square_block(_dev(one_col), use_46).to_reference()
    ref = O.quantize_square_block(one_col, use_46)
    np.testing.assert_array_equal(got[0], ref.fp4)
    np.testing.assert_array_equal(got[1], ref.scales8)


@pytest.mark.parametrize("name,fwd", [("nvidia", "rtn_16x16"), ("four_over_six", "rtn_16x16_46")])
def test_square_block_recipes_linear(cuda, name, fwd):
    """nvidia / four_over_six: square-block W, reused W^T in dX, sr_rht dW (linear_graph.py:119-140, :308-326)."""
    q2 = _q2()
    x = make("normal", (256, 384), seed=1)
    w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
    e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
    cfg = q2.baseline_config(name)
    y, tape = q2.forward(_dev(x), _dev(w), cfg)
    g = q2.backward(tape, _dev(e), q2.SeedPair(7, 9))
    ry, rtape = O.forward(x, w, forward_scheme=fwd)
    assert_same(tape.qX, rtape[0], "qX")
    np.testing.assert_array_equal(tape.qW.to_reference()[0], rtape[1].fp4)
    rdx, rdw = O.backward(rtape, e, O.SeedPair(7, 9), backward_scheme="sr_rht", reuse_forward_weights=True)
    for got, ref in ((y, ry), (g.dX, rdx), (g.dW, rdw)):
        got = got.double().cpu().numpy()
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-5, rel


@pytest.mark.parametrize("rotate,use_46", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("source", ["rows", "cols", "tape"])
def test_sr_operand(cuda, source, rotate, use_46):
    """The general _sr_pair operand: plain / rotated, quantize_sr / quantize_sr_46, every source."""
    q2 = _q2()
    seeds = q2.SeedPair(21, 23)
    x = make("normal", (256, 384), seed=18)
    if source == "tape":
        qx = q2.quantize_rtn_46(_dev(x), caps=(6.0,))
        gpu_fn = lambda: q2.sr_operand(qx, seeds, 55, 8, "tape", rotate, use_46)     # noqa: E731
        logical = np.ascontiguousarray(O.dequantize(O.quantize_rtn_46(x, caps=(6.0,))).T)
    else:
        gpu_fn = lambda: q2.sr_operand(_dev(x), seeds, 55, 8, source, rotate, use_46)  # noqa: E731
        logical = x if source == "rows" else np.ascontiguousarray(x.T)
    src = O.rht_apply(logical, 21, 8) if rotate else logical
    quant = O.quantize_sr_46 if use_46 else O.quantize_sr
    _raises_or_same(gpu_fn, lambda: quant(src, 23, 55), f"sr_operand {source} rot={rotate} 46={use_46}")


@pytest.mark.parametrize("cfg_args,reuse", [(("rtn_1x16", "sr"), False), (("rtn_1x16", "sr_46"), False),
                                            (("rtn_1x16_46", "sr_rht_46"), False),
                                            (("rtn_16x16_46", "sr_46"), True)])
def test_sr_schemes_linear(cuda, cfg_args, reuse):
    """Every SR backward scheme of linear_graph.backward (:290-326), incl. four_over_six_backward."""
    q2 = _q2()
    x = make("normal", (256, 384), seed=1)
    w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
    e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
    cfg = q2.LayerConfig(*cfg_args, reuse_forward_weights=reuse)
    y, tape = q2.forward(_dev(x), _dev(w), cfg)
    g = q2.backward(tape, _dev(e), q2.SeedPair(7, 9))
    ry, rtape = O.forward(x, w, forward_scheme=cfg_args[0])
    rdx, rdw = O.backward(rtape, e, O.SeedPair(7, 9), backward_scheme=cfg_args[1], reuse_forward_weights=reuse)
    for got, ref in ((y, ry), (g.dX, rdx), (g.dW, rdw)):
        got = got.double().cpu().numpy()
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-5, rel


@pytest.mark.parametrize("cfg_args", [("identity", "identity"), ("identity", "ms_eden"), ("rtn_1x16_46", "identity")])
def test_identity_schemes_linear(cuda, cfg_args):
    """The unquantized control (linear_graph.py:136-140 'identity') and its mixes: dense FP32
    GEMMs (cuBLAS, no TF32) where nothing is quantized, dense X/W sources for a quantized backward."""
    q2 = _q2()
    x = make("normal", (256, 384), seed=1)
    w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
    e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
    cfg = q2.LayerConfig(*cfg_args)
    y, tape = q2.forward(_dev(x), _dev(w), cfg)
    g = q2.backward(tape, _dev(e), q2.SeedPair(7, 9))
    ry, rtape = O.forward(x, w, forward_scheme=cfg_args[0])
    rdx, rdw = O.backward(rtape, e, O.SeedPair(7, 9), backward_scheme=cfg_args[1])
    for got, ref in ((y, ry), (g.dX, rdx), (g.dW, rdw)):
        got = got.double().cpu().numpy()
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-5, rel


@pytest.mark.parametrize("fwd,bwd,abl,reuse,posthoc", [
    ("rtn_1x16_46", "ms_eden", "a", False, False), ("rtn_1x16_46", "ms_eden", "c", False, True),
    ("rtn_1x16_46", "ms_eden", "e", False, False), ("rtn_1x16", "sr_rht", "b", False, False),
    ("rtn_1x16", "sr_rht", "d", False, False), ("rtn_1x16", "sr_rht", "a", False, False),
    ("rtn_1x16_46", "sr_46", "b", False, False), ("rtn_1x16_46", "sr_rht_46", "c", False, False),
    ("rtn_16x16", "sr_rht", "b", True, False), ("rtn_16x16", "sr_rht", "a", True, False),
    ("rtn_16x16_46", "sr_46", "d", True, False), ("identity", "sr_rht", "d", False, False)])
def test_ablation_masks_linear(cuda, fwd, bwd, abl, reuse, posthoc):
    """Ablations a-e (linear_graph.py:59-70, :296): quantized operands bit-exact through the
    oracle (pinned to the reference in test_oracle_pin), dense ones as fp32 products."""
    q2 = _q2()
    x = make("normal", (256, 384), seed=1)
    w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
    e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
    cfg = q2.LayerConfig(fwd, bwd, ablation=abl, reuse_forward_weights=reuse, posthoc=posthoc)
    y, tape = q2.forward(_dev(x), _dev(w), cfg)
    g = q2.backward(tape, _dev(e), q2.SeedPair(7, 9))
    ry, rtape = O.forward(x, w, forward_scheme=fwd)
    rdx, rdw = O.backward(rtape, e, O.SeedPair(7, 9), backward_scheme=bwd, reuse_forward_weights=reuse,
                          ablation=abl, posthoc=posthoc)
    for got, ref in ((y, ry), (g.dX, rdx), (g.dW, rdw)):
        got = got.double().cpu().numpy()
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-5, rel


def test_ablation_golden_case(cuda):
    """One ablation straight against the reference's own frozen output (tests/golden)."""
    q2 = _q2()
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    cfg = q2.LayerConfig("rtn_1x16_46", "ms_eden", ablation="a")
    _, tape = q2.forward(_dev(gold["e2e_X"], False), _dev(gold["e2e_W"], False), cfg)   # fp32, as generated
    g = q2.backward(tape, _dev(gold["e2e_E"], False), q2.SeedPair(7, 9))
    for got, ref in ((g.dX, gold["abl_ms_a_dX"]), (g.dW, gold["abl_ms_a_dW"])):
        got = got.double().cpu().numpy()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5


def test_baseline_quantizer_errors(cuda):
    """The reference's input checks (quantizers.py:114-120, :276-280) on the baseline quantizers."""
    import torch
    q2 = _q2()
    bad = np.ones((32, 64), np.float32)
    bad[3, 5] = np.inf
    for fn in (lambda v: q2.quantize_sr(v, 1, 2), lambda v: q2.quantize_sr_46(v, 1, 2),
               lambda v: q2.quantize_square_block(v)):
        with pytest.raises(ValueError, match="finite"):
            fn(_dev(bad, False))
    with pytest.raises(ValueError, match="multiple of 16"):
        q2.quantize_sr(torch.ones(4, 24, device="cuda"), 1)
    with pytest.raises(ValueError, match="2D with both dims multiples of 16"):
        q2.quantize_square_block(torch.ones(24, 32, device="cuda"))
    with pytest.raises(ValueError, match="multiple of 128"):
        q2.rht_sr(torch.ones(32, 64, device="cuda"), q2.SeedPair(1, 2), 3, 4)
    z = q2.quantize_sr(torch.zeros(0, 64, device="cuda"), 1, 2)
    assert z.shape == (0, 64) and float(z.scale32) == 0.0


@pytest.mark.parametrize("fwd,bwd,abl,reuse", [("rtn_1x16_46", "ms_eden", "full", False),
                                               ("rtn_1x16", "sr_rht", "b", False),
                                               ("rtn_16x16", "sr_rht", "full", True),
                                               ("identity", "identity", "full", False)])
def test_accumulate_f64(cuda, fwd, bwd, abl, reuse):
    """accumulate="f64" (linear_graph.py:190-205): float64 products of the same quantized
    operands; only the DGEMM summation order differs from the reference's."""
    q2 = _q2()
    import torch
    x = make("normal", (256, 384), seed=1)
    w = to_bf16((make("normal", (256, 384), seed=2) / 16).astype(np.float32))
    e = to_bf16((1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32))
    cfg = q2.LayerConfig(fwd, bwd, ablation=abl, reuse_forward_weights=reuse)
    y, tape = q2.forward(_dev(x), _dev(w), cfg, accumulate="f64")
    g = q2.backward(tape, _dev(e), q2.SeedPair(7, 9), accumulate="f64")
    ry, rtape = O.forward(x, w, accumulate="f64", forward_scheme=fwd)
    rdx, rdw = O.backward(rtape, e, O.SeedPair(7, 9), accumulate="f64", backward_scheme=bwd,
                          reuse_forward_weights=reuse, ablation=abl)
    for got, ref in ((y, ry), (g.dX, rdx), (g.dW, rdw)):
        assert got.dtype == torch.float64
        got = got.cpu().numpy()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12


def test_gemm_emulated_operands(cuda):
    q2 = _q2()
    a = _dev(make("normal", (128, 256), seed=4), bf16=False)
    b = _dev(make("normal", (64, 256), seed=5), bf16=False)
    qa = q2.quantize_rtn_46(a)
    ref = O.gemm_emulated(O.quantize_rtn_46(a.cpu().numpy()), b.cpu().numpy())
    got = q2.gemm_emulated(qa, b).double().cpu().numpy()          # NVFP4 x dense: FP32 product
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-6
    with pytest.raises(ValueError, match="inner dimensions disagree"):
        q2.gemm_emulated(qa, b[:, :128])
    with pytest.raises(ValueError, match="unknown accumulate precision"):
        q2.gemm_emulated(qa, qa, "f16")
