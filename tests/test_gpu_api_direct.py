"""Direct GPU parity of three public functions against the reference's own outputs
(tests/golden, written by make_golden.py importing nvfp4emu):
  * dequantize             quantizers.py:315-323   (float64, exact)
  * serialize_nvfp4        quantizers.py:330-348   (NV4T bytes)
  * ms_eden_estimate_pair  ms_eden.py:156-180      (both operands of a GEMM pair)
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def _q2():
    import paper_2601_22813_b200 as q2
    return q2


def _same(t, prefix):
    fp4, s8, s32 = t.to_reference()
    np.testing.assert_array_equal(fp4, GOLD[prefix + "fp4"])
    np.testing.assert_array_equal(s8, GOLD[prefix + "s8"])
    assert np.float32(s32).tobytes() == GOLD[prefix + "s32"].tobytes()


@pytest.mark.parametrize("tag", ["n", "w"])
def test_dequantize_golden(cuda, tag):
    q2 = _q2()
    x = torch.from_numpy(GOLD[f"nv4t_{tag}_x"]).cuda()
    got = q2.dequantize(q2.quantize_rtn_46(x)).cpu().numpy()
    np.testing.assert_array_equal(got, GOLD[f"deq_{tag}"])


@pytest.mark.parametrize("tag", ["n", "w"])
def test_serialize_golden_bytes(cuda, tag):
    q2 = _q2()
    x = torch.from_numpy(GOLD[f"nv4t_{tag}_x"]).cuda()
    assert q2.serialize_nvfp4(q2.quantize_rtn_46(x)) == GOLD[f"nv4t_{tag}_bytes"].tobytes()
    t = q2.ms_eden_quantize(x, q2.SeedPair(123, 456), tensor_id=5, rotation_id=6)
    assert q2.serialize_nvfp4(t) == GOLD[f"nv4t_{tag}_msed_bytes"].tobytes()
    back = q2.deserialize_nvfp4(GOLD[f"nv4t_{tag}_bytes"].tobytes())
    assert q2.serialize_nvfp4(back) == GOLD[f"nv4t_{tag}_bytes"].tobytes()


@pytest.mark.parametrize("tag", ["n", "w"])
def test_ms_eden_estimate_pair_golden(cuda, tag):
    q2 = _q2()
    x = torch.from_numpy(GOLD[f"nv4t_{tag}_x"]).cuda()
    pa, pb = q2.ms_eden_estimate_pair(x[:64], x[32:], q2.SeedPair(123, 456), pair_id=q2.derive_stream(1))
    _same(pa, f"pair_{tag}_a_")
    _same(pb, f"pair_{tag}_b_")
