"""The GPU statistical harness (harness.py:132-293) on B200 ops."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_normal_samples_match_reference_draws():
    from paper_2601_22813_b200 import harness as H
    from oracle import nvfp4_oracle as O
    idx = np.arange(8, dtype=np.uint64)
    u1 = O.prng_uniform(3, 77, 2 * idx) + 2.0 ** -53
    u2 = O.prng_uniform(3, 77, 2 * idx + 1)
    np.testing.assert_array_equal(H.normal_samples(3, 77, 8), np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2))


def test_mse_bench_table(cuda):
    """Each method within 6% of the paper's table (harness.py:53-61) on 2^19 samples."""
    from paper_2601_22813_b200 import harness as H
    for r in H.mse_bench(n_samples=1 << 19, seed=1):
        tol = 0.06 * H.TABLE_TARGETS_E3[r.method] + 3 * r.stderr * 1e3
        assert abs(r.mse_e3 - H.TABLE_TARGETS_E3[r.method]) <= tol, r.to_dict()


def test_concentration_unbiased_vs_biased(cuda):
    """quartet2 decays like 1/B; the four_over_six_backward negative control flattens."""
    from paper_2601_22813_b200 import harness as H
    good = H.concentration("quartet2", b_max=256, trials=1, seed=3)
    assert -1.2 <= good.slope <= -0.8, good.to_dict()
    bad = H.concentration("four_over_six_backward", b_max=256, trials=1, seed=3)
    assert bad.tail_slope > -0.6, bad.to_dict()


def test_grad_check_identity(cuda):
    from paper_2601_22813_b200 import harness as H
    r = H.grad_check("identity", seed=0, n_probes=16)
    assert r.max_rel_err < 1e-3, r.to_dict()          # float64 central differences of a ~1e4 loss


def test_train_demo_quartet2_learns(cuda):
    """QAT demo (harness.py:375-458) on the B200 layers: quartet2 tracks the unquantized run."""
    from paper_2601_22813_b200 import harness as H
    runs = H.train_demo(("identity", "quartet2"), steps=300, n_seeds=1)
    ident, q = runs
    assert q.losses[-1] < 0.5 * q.losses[0], q.losses[[0, -1]]
    assert q.final_loss < 3.0 * ident.final_loss, (q.final_loss, ident.final_loss)
