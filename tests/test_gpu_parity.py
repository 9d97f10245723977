"""GPU parity: the CUDA path against the CPU oracle on identical inputs.

Bit-exact for codes, scales and scale32 (integer/byte outputs); GEMM outputs
within the stated tolerances (SURVEY.md §8(c) calibration):
  FP32 out:  |D - D_ref| <= 1e-5 * (|deq A| . |deq B|^T) elementwise
  BF16 out:  relative Frobenius <= 4e-3 and |D - D_ref| <= 2^-8 |D_ref| + 1e-5 * bound
"""

import numpy as np
import pytest
import torch

from oracle import nvfp4_oracle as O
from tests.families import FAMILIES, make

pytestmark = pytest.mark.gpu


def _q2():
    import paper_2601_22813_b200 as q2
    return q2


def _dev(x, bf16=True):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(torch.bfloat16) if bf16 else t


def assert_same(gpu_t, ref_t, what=""):
    fp4, s8, s32 = gpu_t.to_reference()
    assert np.float32(s32).tobytes() == np.float32(ref_t.scale32).tobytes(), f"{what} scale32 {s32!r} vs {ref_t.scale32!r}"
    bad_s = np.argwhere(s8 != ref_t.scales8)
    assert bad_s.size == 0, f"{what} scales differ at {bad_s[:5].tolist()} ({len(bad_s)} groups)"
    bad_c = np.argwhere(fp4 != ref_t.fp4)
    assert bad_c.size == 0, f"{what} codes differ at {bad_c[:5].tolist()} ({len(bad_c)} elements)"


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("bf16", [True, False])
def test_quantize_rtn_46(cuda, family, bf16):
    q2 = _q2()
    x = make(family, (192, 512), seed=11, bf16=bf16)
    assert_same(q2.quantize_rtn_46(_dev(x, bf16)), O.quantize_rtn_46(x), f"q46[{family}]")


def test_quantize_rtn_46_single_cap_and_rtn(cuda):
    q2 = _q2()
    x = make("lognormal_rows", (64, 256), seed=3)
    assert_same(q2.quantize_rtn_46(_dev(x), caps=(6.0,)), O.quantize_rtn_46(x, caps=(6.0,)), "q46 one cap")
    for s in (6.0, 4.0, 5.5):
        assert_same(q2.quantize_rtn(_dev(x), s), O.quantize_rtn(x, s), f"rtn s={s}")


def test_quantize_zero_and_errors(cuda):
    q2 = _q2()
    z = np.zeros((128, 256), np.float32)
    assert_same(q2.quantize_rtn_46(_dev(z)), O.quantize_rtn_46(z), "zero")
    x = make("normal", (128, 256), seed=1, bf16=False)
    x[5, 7] = np.inf
    with pytest.raises(ValueError, match="finite"):
        q2.quantize_rtn_46(_dev(x, False))
    with pytest.raises(ValueError, match="multiple of 16"):
        q2.quantize_rtn_46(torch.ones(4, 24, device="cuda"))


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("mode", ["exact", "pow2", "posthoc"])
def test_ms_eden_rows(cuda, family, mode):
    q2 = _q2()
    x = make(family, (192, 512), seed=5)
    seeds = q2.SeedPair(123, 456)
    ref_seeds = O.SeedPair(123, 456)
    if mode == "posthoc":
        got = q2.posthoc_quantize(_dev(x), seeds, tensor_id=77, rotation_id=99)
        ref = O.posthoc_quantize(x, ref_seeds, tensor_id=77, rotation_id=99)
    else:
        got = q2.ms_eden_quantize(_dev(x), seeds, tensor_id=77, rotation_id=99, pow2_scale=mode == "pow2")
        ref = O.ms_eden_quantize(x, ref_seeds, tensor_id=77, rotation_id=99, pow2_scale=mode == "pow2")
    assert_same(got, ref, f"msed[{mode},{family}]")


@pytest.mark.parametrize("mode", ["exact", "posthoc"])
def test_ms_eden_fp32_rows(cuda, mode):
    q2 = _q2()
    x = make("t2", (128, 384), seed=8, bf16=False)
    got = q2.msed(_dev(x, False), q2.SeedPair(1, 2), 6.0, 5, 6, mode, "rows")
    ref = (O.posthoc_quantize if mode == "posthoc" else O.ms_eden_quantize)(x, O.SeedPair(1, 2), 6.0, 5, 6)
    assert_same(got, ref, f"msed fp32 {mode}")


@pytest.mark.parametrize("mode", ["exact", "posthoc"])
@pytest.mark.parametrize("family", ["normal", "lognormal_rows", "zero_rows"])
def test_ms_eden_cols(cuda, mode, family):
    """E^T quantized straight from E (source='cols')."""
    q2 = _q2()
    e = make(family, (384, 192), seed=21)          # [K=tokens, R=out]
    got = q2.msed(_dev(e), q2.SeedPair(3, 4), 6.0, 10, 20, mode, "cols")
    quant = O.posthoc_quantize if mode == "posthoc" else O.ms_eden_quantize
    ref = quant(np.ascontiguousarray(e.T), O.SeedPair(3, 4), 6.0, 10, 20)
    assert_same(got, ref, f"msed cols {mode}")


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("mode", ["exact", "posthoc"])
def test_ms_eden_tape(cuda, mode, family):
    """W^T / X^T re-quantized from the saved NVFP4 tape (source='tape'); narrow-range
    families take the exact fp32 transform, wide-range ones the float64 one."""
    q2 = _q2()
    w = make(family, (256, 192), seed=9)                # tape logical [K=256, R=192]
    qw = q2.quantize_rtn_46(_dev(w))
    got = q2.msed(qw, q2.SeedPair(5, 6), 6.0, 30, 40, mode, "tape")
    deq = O.dequantize(O.quantize_rtn_46(w))
    quant = O.posthoc_quantize if mode == "posthoc" else O.ms_eden_quantize
    ref = quant(np.ascontiguousarray(deq.T), O.SeedPair(5, 6), 6.0, 30, 40)
    assert_same(got, ref, f"msed tape {mode}")


def test_posthoc_pass1_pass2_api(cuda):
    q2 = _q2()
    x = make("normal", (128, 256), seed=2)
    er, red = q2.pass1(_dev(x), 7, tensor_id=3, rotation_id=4)
    ref_er, ref_red = O.pass1(x, 7, tensor_id=3, rotation_id=4)
    np.testing.assert_array_equal(er.pseudo_scales.cpu().numpy(), ref_er.pseudo_scales)
    np.testing.assert_array_equal(red.corrections.cpu().numpy(), ref_red.corrections)
    assert red.global_absmax == ref_red.global_absmax
    assert_same(q2.pass2(er, red, 8, tensor_id=3), O.pass2(ref_er, ref_red, 8, tensor_id=3), "pass2")


def _gemm_check(d, qa_ref, qb_ref, bf16):
    a, b = O.dequantize(qa_ref), O.dequantize(qb_ref)
    ref = O.gemm_emulated(qa_ref, qb_ref)
    bound = np.abs(a) @ np.abs(b).T
    d = d.double().cpu().numpy()
    if bf16:
        rel = np.linalg.norm(d - ref) / max(np.linalg.norm(ref), 1e-300)
        assert rel <= 4e-3, rel
        assert np.all(np.abs(d - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-5 * bound)
    else:
        worst = np.max(np.abs(d - ref) - 1e-5 * bound)
        assert worst <= 0, f"fp32 gemm exceeds 1e-5*|A||B|^T by {worst}"


@pytest.mark.parametrize("mnk", [(128, 256, 256), (256, 512, 1024), (384, 640, 320), (200, 136, 192),
                                 (1024, 768, 2048), (1280, 768, 512), (768, 1280, 512), (2048, 1792, 256)])
@pytest.mark.parametrize("bf16_out", [False, True])
def test_gemm(cuda, mnk, bf16_out):
    q2 = _q2()
    m, n, k = mnk
    a = make("lognormal_rows", (m, k), seed=m + k)
    b = make("normal", (n, k), seed=n)
    qa, qb = q2.quantize_rtn_46(_dev(a)), q2.quantize_rtn_46(_dev(b))
    d = q2.gemm(qa, qb, torch.bfloat16 if bf16_out else torch.float32)
    torch.cuda.synchronize()
    _gemm_check(d, O.quantize_rtn_46(a), O.quantize_rtn_46(b), bf16_out)


def test_gemm_accumulate(cuda):
    q2 = _q2()
    a, b = make("normal", (256, 512), 1), make("normal", (256, 512), 2)
    qa, qb = q2.quantize_rtn_46(_dev(a)), q2.quantize_rtn_46(_dev(b))
    d = q2.gemm(qa, qb)
    d2 = d.clone()
    q2.gemm(qa, qb, out=d2, accumulate=True)
    torch.testing.assert_close(d2, 2 * d, rtol=1e-6, atol=0)


@pytest.mark.parametrize("posthoc", [False, True])
def test_linear_fwd_bwd(cuda, posthoc):
    q2 = _q2()
    x = make("normal", (256, 384), seed=1)
    w = (make("normal", (256, 384), seed=2) / 16).astype(np.float32)
    e = (1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32)
    from tests.families import to_bf16
    w, e = to_bf16(w), to_bf16(e)
    cfg = q2.LayerConfig(posthoc=posthoc)
    y, tape = q2.forward(_dev(x), _dev(w), cfg)
    g = q2.backward(tape, _dev(e), q2.SeedPair(7, 9))
    ry, rtape = O.forward(x, w)
    assert_same(tape.qX, rtape[0], "qX")
    assert_same(tape.qW, rtape[1], "qW")
    _gemm_check(y, rtape[0], rtape[1], False)
    rdx, rdw = O.backward(rtape, e, O.SeedPair(7, 9), posthoc=posthoc)
    for got, ref in ((g.dX, rdx), (g.dW, rdw)):
        got = got.double().cpu().numpy()
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-5, rel


@pytest.mark.parametrize("posthoc", [False, True])
def test_backward_deterministic(cuda, posthoc):
    """Same inputs and seeds -> bit-identical gradients (SPEC linear_graph determinism);
    also guards every scale-factor replica the GEMM reads being written."""
    q2 = _q2()
    x, w = make("normal", (256, 384), seed=1), make("normal", (256, 384), seed=2)
    e = (1e-2 * make("normal", (256, 256), seed=3)).astype(np.float32)
    y, tape = q2.forward(_dev(x), _dev(w), q2.LayerConfig(posthoc=posthoc))
    ref = q2.backward(tape, _dev(e), q2.SeedPair(7, 9))
    for _ in range(3):
        junk = torch.full((1 << 22,), 0x7F, dtype=torch.uint8, device="cuda")   # dirty the allocator cache
        del junk
        g = q2.backward(tape, _dev(e), q2.SeedPair(7, 9))
        assert torch.equal(g.dX, ref.dX) and torch.equal(g.dW, ref.dW)


@pytest.mark.parametrize("family", FAMILIES)
def test_ms_eden_rows_cols_dual(cuda, family):
    """Post-hoc MS(E) and MS(E^T) of one bf16 E (dims % 128), singly and through the dual entry."""
    q2 = _q2()
    e = make(family, (256, 384), seed=41)                 # [T, N]
    s, rs = q2.SeedPair(11, 12), O.SeedPair(11, 12)
    assert_same(q2.msed(_dev(e), s, 6.0, 3, 4, "posthoc", "rows"), O.posthoc_quantize(e, rs, 6.0, 3, 4), "rows")
    et = np.ascontiguousarray(e.T)
    assert_same(q2.msed(_dev(e), s, 6.0, 5, 6, "posthoc", "cols"), O.posthoc_quantize(et, rs, 6.0, 5, 6), "cols")
    qr, qc = q2.msed_dual_posthoc(_dev(e), s, 3, 4, 5, 6)
    assert_same(qr, O.posthoc_quantize(e, rs, 6.0, 3, 4), "dual rows")
    assert_same(qc, O.posthoc_quantize(et, rs, 6.0, 5, 6), "dual cols")


@pytest.mark.parametrize("family", ["normal", "zero_rows", "tiny_chunk"])
def test_nv4t_container(cuda, family):
    """serialize_nvfp4 / deserialize_nvfp4 (quantizers.py:326-372): byte-identical
    to the reference container of the same quantization, and a lossless round trip."""
    q2 = _q2()
    x = make(family, (192, 256), seed=21)
    t = q2.quantize_rtn_46(_dev(x))
    blob = q2.serialize_nvfp4(t)
    assert blob == O.serialize_nvfp4(O.quantize_rtn_46(x))
    back = q2.deserialize_nvfp4(blob)
    for a, b in zip(back.to_reference(), t.to_reference()):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    assert torch.equal(back.codes, t.codes)
    with pytest.raises(ValueError, match="magic"):
        q2.deserialize_nvfp4(b"XXXX" + blob[4:])


@pytest.mark.parametrize("family", ["normal", "tie_grid", "lognormal_rows"])
def test_quantize_rtn_46_producer_amax(cuda, family):
    """The amax supplied by the producer (q2_quant_fwd_amax) gives the same tensor."""
    q2 = _q2()
    x = _dev(make(family, (192, 512), seed=19))
    am = q2.absmax(x)
    assert float(am.item()) == float(x.float().abs().max().item())
    a, b = q2.quantize_rtn_46(x), q2.quantize_rtn_46(x, amax=am)
    for u, v in zip(a.to_reference(), b.to_reference()):       # (sf padding rows are unspecified)
        assert np.array_equal(np.asarray(u), np.asarray(v))


def test_empty_inputs(cuda):
    """Zero-row tensors quantize to the zero tensor (quantizers.py:174-176, 219-220; ms_eden.py:135-137)."""
    q2 = _q2()
    e = torch.zeros(0, 256, device="cuda", dtype=torch.bfloat16)
    for t in (q2.quantize_rtn_46(e), q2.quantize_rtn(e), q2.ms_eden_quantize(e, q2.SeedPair(1, 2)),
              q2.posthoc_quantize(e, q2.SeedPair(1, 2)), q2.quantize_sr_46(e, 1, 2)):
        assert t.shape == (0, 256) and float(t.scale32) == 0.0
