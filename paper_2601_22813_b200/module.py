"""Training-framework entry point: the Quartet II linear as a torch autograd op.

``Quartet2Linear`` is the layer a user drops into a model in place of
``torch.nn.Linear``: the forward pass is ``linear_graph.forward`` (Q46(X)·Q46(W)ᵀ
on the tcgen05 NVFP4 GEMM) and autograd's backward is ``linear_graph.backward``
(MS-EDEN dX / dW GEMMs), the pair the reference wires up in
``linear_graph.py:243-333``.  Leading batch dimensions are flattened into tokens
(the reference's ``X [tokens, in]``).  Each forward call draws a fresh
``SeedPair`` from the module's seed and call counter with ``derive_stream``
(rht.py:78-86), so every backward uses independent rotations and rounding,
which the unbiasedness argument requires.

Defaults: the layer computes ``baseline_config("quartet2")`` (linear_graph.py:133),
i.e. the exact ``ms_eden_quantize`` backward of the reference; pass
``cfg=LayerConfig(posthoc=True)`` for the single-read post-hoc schedule (faster, the
paper's kernel schedule, statistically equivalent but not bit-identical gradients).
Data-dependent errors (non-finite input, scale overflow) accumulate in the module's
device error word without a host sync; ``check_errors()`` raises them with the
reference's messages, and the module does so by itself every ``check_every`` calls.
"""

from __future__ import annotations

import math

import torch

from .linear_graph import LayerConfig, backward, forward
from .quantizers import _raise_bits
from .rht import SeedPair, derive_stream


class Quartet2LinearFunction(torch.autograd.Function):
    """y = x·Wᵀ (+ b) with the quantized forward and the quantized backward.

    ``seeds`` are the backward's (rht, sr) pair.  dX comes back in x's dtype,
    dW in W's dtype (accumulated in fp32 by the wgrad GEMM), db = Σ_tokens dY.
    """

    @staticmethod
    def forward(ctx, x, weight, bias, cfg: LayerConfig, seeds: SeedPair, err=None):
        lead, din = x.shape[:-1], x.shape[-1]
        x2 = x.reshape(-1, din)
        y, tape = forward(x2, weight, cfg, out_dtype=x.dtype, err=err)
        if bias is not None:
            y = y + bias.to(y.dtype)
        ctx.tape, ctx.seeds, ctx.err = tape, seeds, err
        ctx.x_dtype, ctx.w_dtype, ctx.lead = x.dtype, weight.dtype, lead
        ctx.has_bias = bias is not None
        return y.reshape(*lead, weight.shape[0])

    @staticmethod
    def backward(ctx, gy):
        e = gy.reshape(-1, gy.shape[-1])
        if e.dtype not in (torch.bfloat16, torch.float32):
            e = e.float()
        g = backward(ctx.tape, e, ctx.seeds, dx_dtype=ctx.x_dtype, err=ctx.err)
        dx = g.dX.reshape(*ctx.lead, g.dX.shape[-1]) if ctx.needs_input_grad[0] else None
        dw = g.dW.to(ctx.w_dtype) if ctx.needs_input_grad[1] else None
        db = e.float().sum(0).to(ctx.w_dtype) if ctx.has_bias and ctx.needs_input_grad[2] else None
        # the tape stays with ctx (freed with the graph), so retain_graph backward works
        return dx, dw, db, None, None, None


def quartet2_linear(x, weight, bias=None, cfg: LayerConfig = LayerConfig(), seeds: SeedPair = SeedPair(1, 2)):
    """Functional form of ``Quartet2Linear`` (explicit backward seeds)."""
    return Quartet2LinearFunction.apply(x, weight, bias, cfg, seeds)


class Quartet2Linear(torch.nn.Module):
    """Drop-in replacement for ``torch.nn.Linear`` computed in NVFP4 on B200.

    ``in_features`` must be a multiple of 128 and ``out_features`` of 128 for
    the MS-EDEN backward, and the tokens of each call a multiple of 128
    (``linear_graph._check_dims``).  ``seed`` fixes the stream of per-call
    ``SeedPair``s; ``seeds_for(call)`` reproduces the pair of any call.
    """

    def __init__(self, in_features: int, out_features: int, bias: bool = False, cfg: LayerConfig = None,
                 seed: int = 0, device=None, dtype=torch.bfloat16, check_every: int = 64):
        super().__init__()
        self.in_features, self.out_features = in_features, out_features
        self.cfg = cfg if cfg is not None else LayerConfig()        # baseline_config("quartet2")
        self.seed = seed
        self.calls = 0
        self.check_every = check_every
        self._err = None
        self.weight = torch.nn.Parameter(torch.empty(out_features, in_features, device=device, dtype=dtype))
        self.bias = torch.nn.Parameter(torch.empty(out_features, device=device, dtype=dtype)) if bias else None
        self.reset_parameters()

    def reset_parameters(self) -> None:
        torch.nn.init.kaiming_uniform_(self.weight, a=math.sqrt(5))      # torch.nn.Linear's init
        if self.bias is not None:
            bound = 1 / math.sqrt(self.in_features)
            torch.nn.init.uniform_(self.bias, -bound, bound)

    def seeds_for(self, call: int) -> SeedPair:
        return SeedPair(derive_stream(self.seed, 1, call), derive_stream(self.seed, 2, call))

    def check_errors(self) -> None:
        """Raise the first data-dependent error of this layer's calls so far (host sync)."""
        if self._err is not None:
            bits = int(self._err.item())
            self._err.zero_()
            _raise_bits(bits)

    def forward(self, x):
        if self._err is None or self._err.device != self.weight.device:
            self._err = torch.zeros(1, dtype=torch.int32, device=self.weight.device)
        if self.check_every and self.calls and self.calls % self.check_every == 0:
            self.check_errors()
        seeds = self.seeds_for(self.calls)
        self.calls += 1
        return Quartet2LinearFunction.apply(x, self.weight, self.bias, self.cfg, seeds, self._err)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, "
                f"bias={self.bias is not None}, forward={self.cfg.forward_scheme}, "
                f"backward={self.cfg.backward_scheme}, posthoc={self.cfg.posthoc}")
