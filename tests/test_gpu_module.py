"""Quartet2Linear / Quartet2LinearFunction: the autograd op returns exactly what
linear_graph.forward/backward return for the same seeds, handles batch
dimensions and bias, and trains."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _q2():
    import paper_2601_22813_b200 as q2
    return q2


def test_module_matches_graph_calls(cuda):
    q2 = _q2()
    torch.manual_seed(0)
    m = q2.Quartet2Linear(256, 384, seed=11, device="cuda")
    x = torch.randn(512, 256, device="cuda").bfloat16().requires_grad_()
    y = m(x)
    gy = (1e-2 * torch.randn_like(y.float())).bfloat16()
    y.backward(gy)
    y_ref, tape = q2.forward(x.detach(), m.weight.detach(), m.cfg, out_dtype=torch.bfloat16)
    g = q2.backward(tape, gy, m.seeds_for(0), dx_dtype=torch.bfloat16)
    assert torch.equal(y, y_ref)
    assert torch.equal(x.grad, g.dX)
    assert torch.equal(m.weight.grad, g.dW.to(m.weight.dtype))
    assert m.calls == 1 and m.seeds_for(1) != m.seeds_for(0)


def test_batch_dims_and_bias(cuda):
    q2 = _q2()
    torch.manual_seed(1)
    m = q2.Quartet2Linear(256, 128, bias=True, device="cuda", dtype=torch.float32)
    x = torch.randn(2, 64, 256, device="cuda", requires_grad=True)
    y = m(x)
    assert y.shape == (2, 64, 128) and y.dtype == torch.float32
    gy = torch.randn_like(y)
    y.backward(gy)
    assert x.grad.shape == x.shape and m.weight.grad.shape == m.weight.shape
    torch.testing.assert_close(m.bias.grad, gy.reshape(-1, 128).sum(0))
    # same call on the flattened input gives the same numbers
    y2 = q2.quartet2_linear(x.detach().reshape(128, 256), m.weight.detach(), m.bias.detach(), m.cfg,
                            m.seeds_for(0))
    assert torch.equal(y.detach().reshape(128, 128), y2)


def test_no_grad_inputs_and_fp32_grads(cuda):
    q2 = _q2()
    m = q2.Quartet2Linear(128, 128, device="cuda")
    x = torch.randn(128, 128, device="cuda").bfloat16()       # no grad for x
    m(x).float().square().mean().backward()
    assert m.weight.grad is not None and torch.isfinite(m.weight.grad.float()).all()


def test_trains_a_linear_map(cuda):
    """Recover a random linear map from noiseless data through the NVFP4 layer."""
    q2 = _q2()
    torch.manual_seed(3)
    target = torch.randn(128, 256, device="cuda") / 16
    m = q2.Quartet2Linear(256, 128, device="cuda", dtype=torch.float32)
    opt = torch.optim.Adam(m.parameters(), lr=3e-3)
    losses = []
    for step in range(150):
        x = torch.randn(256, 256, device="cuda")
        loss = (m(x) - x @ target.t()).square().mean()
        opt.zero_grad()
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    assert losses[-1] < 0.1 * losses[0], (losses[0], losses[-1])


def test_default_is_reference_quartet2_and_retain_graph(cuda):
    """The module's default config is baseline_config("quartet2") (exact MS-EDEN), and a
    second backward through a retained graph gives the same gradients."""
    q2 = _q2()
    m = q2.Quartet2Linear(256, 128, device="cuda")
    assert m.cfg == q2.baseline_config("quartet2")
    x = torch.randn(128, 256, device="cuda").bfloat16()
    y = m(x)
    gy = (1e-2 * torch.randn_like(y.float())).bfloat16()
    y.backward(gy, retain_graph=True)
    g1 = m.weight.grad.clone()
    m.weight.grad = None
    y.backward(gy)
    assert torch.equal(m.weight.grad, g1)


def test_deferred_errors_no_sync(cuda):
    """Non-finite input is recorded on the device without raising at the call; the
    layer's check_errors() raises the reference's ValueError."""
    q2 = _q2()
    m = q2.Quartet2Linear(128, 128, device="cuda", check_every=0)
    x = torch.randn(128, 128, device="cuda").bfloat16()
    x[3, 5] = float("inf")
    m(x)                                             # no exception: no host sync in the call
    with pytest.raises(ValueError, match="finite"):
        m.check_errors()
    m.check_errors()                                 # cleared
