"""torch.ops.quartet2.* on the GPU: the custom-op form of the layer returns exactly
what forward()/backward() return, and each op passes torch.library.opcheck
(schema, fake kernel and dispatcher registration consistent with the real kernel)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _q2():
    import paper_2601_22813_b200 as q2
    return q2


@pytest.mark.parametrize("mode", ["exact", "posthoc"])
def test_ops_layer_equals_graph(cuda, mode):
    q2 = _q2()
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(256, 512, device="cuda", generator=g).bfloat16()
    w = (torch.randn(384, 512, device="cuda", generator=g) / 16).bfloat16()
    e = (1e-2 * torch.randn(256, 384, device="cuda", generator=g)).bfloat16()
    seeds = q2.SeedPair(2 ** 63 + 5, 17)                   # unsigned 64-bit seed through the int64 schema
    y, dx, dw = q2.ops.linear_fwd_bwd(x, w, e, seeds, mode)
    y_ref, tape = q2.forward(x, w, q2.LayerConfig(posthoc=mode == "posthoc"), out_dtype=torch.bfloat16)
    ref = q2.backward(tape, e, seeds)
    assert torch.equal(y, y_ref) and torch.equal(dx, ref.dX) and torch.equal(dw, ref.dW)


def test_opcheck(cuda):
    q2 = _q2()
    x = torch.randn(128, 256, device="cuda").bfloat16()
    torch.library.opcheck(torch.ops.quartet2.quantize_rtn_46.default, (x,))
    torch.library.opcheck(torch.ops.quartet2.msed.default, (x, 1, 2, 3, 4, "exact", "cols"))
    qx = torch.ops.quartet2.quantize_rtn_46(x)
    torch.library.opcheck(torch.ops.quartet2.msed_tape.default, (*qx, 128, 256, 1, 2, 3, 4, "posthoc"))
    qw = torch.ops.quartet2.quantize_rtn_46(torch.randn(192, 256, device="cuda").bfloat16())
    torch.library.opcheck(torch.ops.quartet2.gemm.default, (*qx, *qw, 256, True))
