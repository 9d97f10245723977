"""Element formats on the GPU (formats.py:76-229) against the reference's frozen
outputs (tests/golden/make_golden.py): grid points, exact midpoints (ties), the
subnormal and saturation edges, and the reference's errors."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def _F():
    from paper_2601_22813_b200 import formats as F
    return F


def _np(t):
    return t.cpu().numpy()


def test_encoders_golden(cuda):
    F = _F()
    np.testing.assert_array_equal(_np(F.encode_fp4_rtn(GOLD["fmt_x4"])), GOLD["fmt_fp4_rtn"])
    np.testing.assert_array_equal(_np(F.encode_fp4_sr(GOLD["fmt_x4sr"], GOLD["fmt_u4"])), GOLD["fmt_fp4_sr"])
    np.testing.assert_array_equal(_np(F.encode_fp8_rtn(GOLD["fmt_x8"])), GOLD["fmt_fp8_rtn"])
    np.testing.assert_array_equal(_np(F.encode_fp8_sr(GOLD["fmt_x8sr"], GOLD["fmt_u8"])), GOLD["fmt_fp8_sr"])
    np.testing.assert_array_equal(_np(F.round_e8m3_rtn(GOLD["fmt_xe"])), GOLD["fmt_e8m3"])


def test_decoders_golden(cuda):
    F = _F()
    np.testing.assert_array_equal(_np(F.decode_fp4(np.arange(16))), GOLD["fmt_dec_fp4"])
    got = _np(F.decode_fp8(torch.arange(256, dtype=torch.uint8)))
    np.testing.assert_array_equal(got, GOLD["fmt_dec_fp8"])               # NaN == NaN here
    assert np.array_equal(np.signbit(got), np.signbit(GOLD["fmt_dec_fp8"]))  # -0.0 for code 0x80
    assert not np.signbit(_np(F.decode_fp4([8]))[0])                       # both zero codes give +0.0


def test_round_trips(cuda):
    F = _F()
    codes = torch.arange(127, dtype=torch.uint8)
    assert torch.equal(F.encode_fp8_rtn(F.decode_fp8(codes)), codes.cuda())
    c4 = torch.tensor([c for c in range(16) if c != 8], dtype=torch.uint8)
    assert torch.equal(F.encode_fp4_rtn(F.decode_fp4(c4)), c4.cuda())
    assert F.round_e8m3_rtn(1.1875) == 1.25 and isinstance(F.round_e8m3_rtn(3.0), float)


def test_format_errors(cuda):
    F = _F()
    with pytest.raises(ValueError, match="NaN input to encode_fp4_rtn"):
        F.encode_fp4_rtn([1.0, float("nan")])
    with pytest.raises(ValueError, match="encode_fp4_sr input 7.0 exceeds the FP4 grid max 6.0"):
        F.encode_fp4_sr([7.0], [0.5])
    with pytest.raises(ValueError, match="negative input to encode_fp8_rtn"):
        F.encode_fp8_rtn([-1.0])
    with pytest.raises(ValueError, match="encode_fp8_sr input 500.0 exceeds 448; EDEN-corrected"):
        F.encode_fp8_sr([500.0], [0.1])
    with pytest.raises(OverflowError, match="round_e8m3_rtn overflow"):
        F.round_e8m3_rtn([1e300])
    with pytest.raises(IndexError):
        F.decode_fp4([16])
    assert F.encode_fp8_rtn(np.zeros(0)).numel() == 0


def test_eden_correction_factors_golden(cuda):
    """chunk_correction_factors (ms_eden.py:75-83) bit-exact incl. degenerate chunks;
    correction_factor (:57-72, a BLAS dot in the reference) to rounding."""
    import paper_2601_22813_b200 as q2
    S = q2.ms_eden.chunk_correction_factors(GOLD["eden_xrot"], GOLD["eden_xrtn"])
    assert S.shape == (8, 4) and S.dtype == torch.float64
    np.testing.assert_array_equal(_np(S), GOLD["eden_S"])
    s1 = q2.ms_eden.correction_factor(GOLD["eden_xrot"][0, :128], GOLD["eden_xrtn"][0, :128])
    assert abs(s1 - GOLD["eden_S1"][0]) <= 1e-14 * abs(GOLD["eden_S1"][0])
    with pytest.raises(ValueError, match="correction_factor expects matching length-128 chunks"):
        q2.ms_eden.correction_factor(np.ones(64), np.ones(64))
    with pytest.raises(ValueError, match="chunk_correction_factors expects matching shapes"):
        q2.ms_eden.chunk_correction_factors(np.ones((2, 256)), np.ones((2, 128)))
