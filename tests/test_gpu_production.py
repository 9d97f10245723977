"""Bit-exact parity at BASELINE.json's production shapes, both MS-EDEN modes.

c1 (2048 tokens, 1024 -> 1024, the CPU oracle shape): the whole layer fwd+bwd.  The six
quantized tensors the three GEMMs consume -- Q46(X), Q46(W), MS(E), MS(W^T), MS(E^T),
MS(X^T), taken from ``backward(..., operands=...)`` -- equal the oracle's bit for bit;
Y, dX and dW meet the fp32 GEMM tolerance against the oracle's GEMMs of the same
operands (|D - D_ref| <= 1e-5 |A||B|^T elementwise).

c3 (16,384 tokens, all four Llama-1.9B projections): the same six tensors on sampled
rows.  Forward: rows of X and W.  MS(E): rows of E; MS(E^T): columns of E; MS(W^T) and
MS(X^T): columns of the dequantized tape.  The sample always holds the row with the
tensor's (rotated) absmax, so scale32 and the post-hoc shift are the full tensor's;
given those, rows are independent, and the oracle draws the SR uniforms with the full
tensor's group index (``row_ids``).  This exercises the index paths only large shapes
reach: 32-bit tile division, K = 11264 and 16384 column tiles, the R % 256 scale
padding of the last row block.
"""

import numpy as np
import pytest
import torch

from oracle import nvfp4_oracle as O

pytestmark = pytest.mark.gpu

SEEDS = (7, 9)
MODES = ["exact", "posthoc"]
C3 = [("qkv", 2048, 6144), ("o", 2048, 2048), ("upgate", 2048, 11264), ("down", 5632, 2048)]


def _q2():
    import paper_2601_22813_b200 as q2
    return q2


def _layer(T, din, dout, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = torch.randn(T, din, device="cuda", generator=g).bfloat16()
    W = (torch.randn(dout, din, device="cuda", generator=g) / din ** 0.5).bfloat16()
    E = (1e-3 * torch.randn(T, dout, device="cuda", generator=g)).bfloat16()
    return X, W, E


def _ms_ref(mode):
    if mode == "posthoc":
        return lambda x, tid, rot, rows=None: O.posthoc_quantize(x, O.SeedPair(*SEEDS), 6.0, tid, rot, row_ids=rows)
    return lambda x, tid, rot, rows=None: O.ms_eden_quantize(x, O.SeedPair(*SEEDS), 6.0, tid, rot, row_ids=rows)


def _rows(q, rows):
    """(fp4, scales8, scale32) of the given rows of a device NVFP4 tensor."""
    fp4, s8 = q.unpacked()
    idx = torch.as_tensor(rows, device=fp4.device)
    return fp4[idx].cpu().numpy(), s8[idx].cpu().numpy(), q.scale32


def _same(got, ref, what):
    fp4, s8, s32 = got
    assert np.float32(s32).tobytes() == np.float32(ref.scale32).tobytes(), f"{what}: scale32 {s32!r} vs {ref.scale32!r}"
    bad = np.argwhere(s8 != ref.scales8)
    assert bad.size == 0, f"{what}: scales differ at {bad[:5].tolist()} ({len(bad)} groups)"
    bad = np.argwhere(fp4 != ref.fp4)
    assert bad.size == 0, f"{what}: codes differ at {bad[:5].tolist()} ({len(bad)} elements)"


def _gemm_ok(got, qa, qb, what):
    """fp32-output GEMM tolerance against the oracle's GEMM of the same operands."""
    a, b = O.dequantize(qa), O.dequantize(qb)
    ref = a @ b.T
    bound = np.abs(a) @ np.abs(b).T
    err = np.abs(got.double().cpu().numpy() - ref)
    assert (err <= 1e-5 * bound + 1e-30).all(), f"{what}: max excess {np.max(err - 1e-5 * bound)}"


# ------------------------------------------------------------------------- c1 --
@pytest.mark.parametrize("mode", MODES)
def test_c1_layer_bit_exact(cuda, mode):
    q2 = _q2()
    X, W, E = _layer(2048, 1024, 1024, seed=11)
    y, tape = q2.forward(X, W, q2.LayerConfig(posthoc=mode == "posthoc"))
    ops = {}
    g = q2.backward(tape, E, q2.SeedPair(*SEEDS), operands=ops)
    torch.cuda.synchronize()
    x64, w64, e64 = (t.double().cpu().numpy() for t in (X, W, E))
    _, (qx, qw) = O.forward(x64, w64)
    _same(tape.qX.to_reference(), qx, "Q46(X)")
    _same(tape.qW.to_reference(), qw, "Q46(W)")
    ms = _ms_ref(mode)
    xd, wd = O.dequantize(qx), O.dequantize(qw)
    ref = {"E": ms(e64, q2.derive_stream(q2.PAIR_DX, 0), q2.PAIR_DX),
           "Wt": ms(np.ascontiguousarray(wd.T), q2.derive_stream(q2.PAIR_DX, 1), q2.PAIR_DX),
           "Et": ms(np.ascontiguousarray(e64.T), q2.derive_stream(q2.PAIR_DW, 0), q2.PAIR_DW),
           "Xt": ms(np.ascontiguousarray(xd.T), q2.derive_stream(q2.PAIR_DW, 1), q2.PAIR_DW)}
    for k, r in ref.items():
        _same(ops[k].to_reference(), r, f"MS({k}) {mode}")
    _gemm_ok(y, qx, qw, "Y")
    _gemm_ok(g.dX, ref["E"], ref["Wt"], "dX")
    _gemm_ok(g.dW, ref["Et"], ref["Xt"], "dW")
    # the oracle's own backward agrees with the GEMMs of those operands
    rdx, rdw = O.backward((qx, qw), e64, O.SeedPair(*SEEDS), posthoc=mode == "posthoc")
    assert np.allclose(rdx, O.gemm_emulated(ref["E"], ref["Wt"])) and np.allclose(rdw, O.gemm_emulated(ref["Et"], ref["Xt"]))


# ------------------------------------------------------------------------- c3 --
def _sample(n, seed, must=()):
    rng = np.random.default_rng(seed)
    rows = set(rng.integers(0, n, 12).tolist()) | {0, n - 1, n - 129} | set(int(m) for m in must)
    return sorted(r for r in rows if 0 <= r < n)


def _rot_argmax(m64, rot):
    """Row of the float64 device matrix m64 holding max |rht_apply(m64)| (rotated in blocks)."""
    q2 = _q2()
    best, arg = -1.0, 0
    for r0 in range(0, m64.shape[0], 2048):
        y = q2.rht_apply(m64[r0:r0 + 2048], SEEDS[0], rot).abs().amax(dim=1)
        v, i = torch.max(y, dim=0)
        if float(v) > best:
            best, arg = float(v), r0 + int(i)
        del y
    return arg


@pytest.fixture(scope="module", params=C3, ids=[c[0] for c in C3])
def c3_layer(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    q2 = _q2()
    name, din, dout = request.param
    X, W, E = _layer(16384, din, dout, seed=100 + din + dout)
    out = {}
    for mode in MODES:
        y, tape = q2.forward(X, W, q2.LayerConfig(posthoc=mode == "posthoc"))
        ops = {}
        q2.backward(tape, E, q2.SeedPair(*SEEDS), operands=ops)
        out[mode] = (tape, ops)
    torch.cuda.synchronize()
    return X, W, E, out


def test_c3_forward_sampled_rows(cuda, c3_layer):
    X, W, E, out = c3_layer
    tape, _ = out["exact"]
    for src, q in ((X, tape.qX), (W, tape.qW)):
        flat = int(src.float().abs().argmax())
        rows = _sample(src.shape[0], 5, [flat // src.shape[1]])
        ref = O.quantize_rtn_46(src[rows].double().cpu().numpy())
        _same(_rows(q, rows), ref, f"Q46 {tuple(src.shape)}")


@pytest.mark.parametrize("mode", MODES)
def test_c3_msed_sampled_rows(cuda, c3_layer, mode):
    q2 = _q2()
    X, W, E, out = c3_layer
    tape, ops = out[mode]
    ms = _ms_ref(mode)
    srcs = {"E": (E.double(), q2.PAIR_DX, 0),                          # rows of E
            "Et": (E.double().t().contiguous(), q2.PAIR_DW, 0),        # columns of E
            "Wt": (q2.dequantize(tape.qW).t().contiguous(), q2.PAIR_DX, 1),
            "Xt": (q2.dequantize(tape.qX).t().contiguous(), q2.PAIR_DW, 1)}
    for k, (m64, pair, operand) in srcs.items():
        rows = _sample(m64.shape[0], 17 + operand, [_rot_argmax(m64, pair)])
        ref = ms(m64[rows].cpu().numpy(), q2.derive_stream(pair, operand), pair, np.array(rows))
        _same(_rows(ops[k], rows), ref, f"MS({k}) {mode} {tuple(m64.shape)}")
        del m64
    torch.cuda.empty_cache()
