"""Tensor-core MS-EDEN (msed_tc.cuh) against the oracle: bit-exact codes, scales
and scale32 for every source kind (rows, cols, dual rows+cols from one read,
NVFP4 tape), every mode (exact, pow2, posthoc) and every parity family, at
shapes that take the tensor-core path (both dims multiples of 128)."""

import numpy as np
import pytest
import torch

from oracle import nvfp4_oracle as O
from tests.families import FAMILIES, make
from tests.test_gpu_parity import assert_same, _dev

pytestmark = pytest.mark.gpu

MODES = ["exact", "pow2", "posthoc"]


def _q2():
    import paper_2601_22813_b200 as q2
    return q2


@pytest.fixture(autouse=True)
def _tc_engine(cuda):
    """Single-operand sources take the tensor-core kernel in these tests."""
    q2 = _q2()
    q2.set_msed_engine("tc")
    yield
    q2.set_msed_engine("auto")


def _ref(mode):
    if mode == "posthoc":
        return lambda x, seeds, s, tid, rid: O.posthoc_quantize(x, seeds, s, tid, rid)
    return lambda x, seeds, s, tid, rid: O.ms_eden_quantize(x, seeds, s, tid, rid, pow2_scale=mode == "pow2")


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("mode", MODES)
def test_tc_rows(cuda, family, mode):
    q2 = _q2()
    x = make(family, (256, 512), seed=5)
    got = q2.msed(_dev(x), q2.SeedPair(123, 456), 6.0, 77, 99, mode, "rows")
    assert_same(got, _ref(mode)(x, O.SeedPair(123, 456), 6.0, 77, 99), f"tc rows {mode} {family}")


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("mode", MODES)
def test_tc_cols(cuda, family, mode):
    q2 = _q2()
    e = make(family, (384, 256), seed=21)          # [K=tokens, R=out]
    got = q2.msed(_dev(e), q2.SeedPair(3, 4), 6.0, 10, 20, mode, "cols")
    assert_same(got, _ref(mode)(np.ascontiguousarray(e.T), O.SeedPair(3, 4), 6.0, 10, 20), f"tc cols {mode} {family}")


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("mode", MODES)
def test_tc_dual(cuda, family, mode):
    q2 = _q2()
    e = make(family, (256, 384), seed=31)          # E [T, N]
    qr, qc = q2.msed_dual(_dev(e), q2.SeedPair(8, 9), 101, 102, 201, 202, 6.0, mode)
    ref = _ref(mode)
    assert_same(qr, ref(e, O.SeedPair(8, 9), 6.0, 101, 102), f"tc dual rows {mode} {family}")
    assert_same(qc, ref(np.ascontiguousarray(e.T), O.SeedPair(8, 9), 6.0, 201, 202), f"tc dual cols {mode} {family}")


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("mode", MODES)
def test_tc_tape(cuda, family, mode):
    q2 = _q2()
    w = make(family, (256, 384), seed=9)           # tape logical [K=256, R=384]
    qw = q2.quantize_rtn_46(_dev(w))
    got = q2.msed(qw, q2.SeedPair(5, 6), 6.0, 30, 40, mode, "tape")
    deq = O.dequantize(O.quantize_rtn_46(w))
    assert_same(got, _ref(mode)(np.ascontiguousarray(deq.T), O.SeedPair(5, 6), 6.0, 30, 40), f"tc tape {mode} {family}")


def test_tc_literal_rate(cuda):
    """On N(0,1) data the certified fast path decides (almost) every chunk."""
    q2 = _q2()
    e = torch.randn(2048, 2048, device="cuda").to(torch.bfloat16)
    q2.msed_stats(reset=True)
    q2.msed_dual(e, q2.SeedPair(1, 2), 1, 2, 3, 4, 6.0, "posthoc")
    q2.msed_dual(e, q2.SeedPair(1, 2), 1, 2, 3, 4, 6.0, "exact")
    total, literal = q2.msed_stats()
    assert total > 0
    assert literal <= 0.01 * total, (literal, total)
