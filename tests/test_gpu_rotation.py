"""rht_apply / rht_inverse / hadamard_128 on the GPU (q2_rht): bit-exact against the
reference's frozen outputs (tests/golden) and the oracle, for bf16/fp32/fp64 inputs
and every chunk size; the reference's errors."""

import os

import numpy as np
import pytest
import torch

from oracle import nvfp4_oracle as O
from tests.families import make

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def _q2():
    import paper_2601_22813_b200 as q2
    return q2


def test_rotations_golden(cuda):
    q2 = _q2()
    x = torch.from_numpy(GOLD["rot_x"]).cuda()
    for got, key in ((q2.rht_apply(x, 11, q2.derive_stream(1)), "rot_apply128"),
                     (q2.rht_apply(x, 11, 5, chunk=32), "rot_apply32"),
                     (q2.rht_apply(x, 3, 0, chunk=512), "rot_apply512"),
                     (q2.rht_inverse(x, 11, q2.derive_stream(1)), "rot_inv128"),
                     (q2.hadamard_128(x.reshape(-1, 128)), "rot_h128")):
        assert got.dtype == torch.float64
        np.testing.assert_array_equal(got.cpu().numpy(), GOLD[key], err_msg=key)


@pytest.mark.parametrize("chunk", [16, 64, 128, 256, 1024, 2048])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
def test_rht_apply_inverse(cuda, chunk, dtype):
    q2 = _q2()
    x = torch.from_numpy(make("lognormal_rows", (12, 4096), seed=chunk)).to(dtype).cuda()
    x64 = x.double().cpu().numpy()
    y = q2.rht_apply(x, 9, 77, chunk=chunk)
    np.testing.assert_array_equal(y.cpu().numpy(), O.rht_apply(x64, 9, 77, chunk=chunk))
    z = q2.rht_inverse(y, 9, 77, chunk=chunk)
    np.testing.assert_array_equal(z.cpu().numpy(), O.rht_inverse(O.rht_apply(x64, 9, 77, chunk=chunk), 9, 77,
                                                                 chunk=chunk))
    assert float((z.cpu() - torch.from_numpy(x64)).abs().max()) <= 1e-12 * float(np.abs(x64).max())


def test_rotation_shapes_and_errors(cuda):
    q2 = _q2()
    x = torch.randn(3, 2, 256, device="cuda")
    assert q2.rht_apply(x, 1).shape == (3, 2, 256)
    assert q2.rht_apply(torch.empty(0, 128, device="cuda"), 1).shape == (0, 128)
    np.testing.assert_array_equal(q2.rht_apply(x.cpu().numpy(), 1).cpu().numpy(),
                                  O.rht_apply(x.cpu().numpy(), 1, 0))
    with pytest.raises(ValueError, match="must be a power of two and a multiple of 16"):
        q2.rht_apply(x, 1, chunk=48)
    with pytest.raises(ValueError, match=r"rotation requires the last dimension \(256\) to be a multiple of 512"):
        q2.rht_apply(x, 1, chunk=512)
    with pytest.raises(ValueError, match="hadamard_128 requires length 128, got 256"):
        q2.hadamard_128(x)
