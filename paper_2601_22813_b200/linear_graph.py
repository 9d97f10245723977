"""Quartet II linear-layer graph on B200 (host mirror of linear_graph.py).

forward:  Y  = Q46(X) . Q46(W)^T                         linear_graph.py:243-256
backward: dX = MS(E) . MS(W^T)^T     pair derive_stream(1)  linear_graph.py:300-307
          dW = MS(E^T) . MS(X^T)^T   pair derive_stream(2)  linear_graph.py:322-326
W^T and X^T are re-quantized straight from the saved NVFP4 tape and E^T
straight from E (no transposed copies are materialised); the three GEMMs run
on the tcgen05 NVFP4 kernel.  ``LayerConfig.posthoc`` selects the
single-read post-hoc MS-EDEN schedule (posthoc.py) for the four backward
quantizations; the default mirrors the reference exactly.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .ms_eden import msed
from .quantizers import NVFP4Tensor, _err_word, _finish, as_device_matrix, quantize_rtn_46, stream_handle
from .rht import CHUNK, SeedPair, derive_stream

FORWARD_SCHEMES = ("rtn_1x16_46",)
BACKWARD_SCHEMES = ("ms_eden",)
PAIR_DX = derive_stream(1)   # linear_graph.py:300
PAIR_DW = derive_stream(2)   # linear_graph.py:301

# The two independent chains of each pass (Q(X) | Q(W); dX chain | dW chain)
# run on the caller's stream and one side stream per device, forked and joined
# with events (captured as parallel branches under CUDA-graph capture), so one
# chain's small kernels and tails fill the SMs the other leaves idle.
_SIDE_STREAMS = {}


def _side_stream(device) -> torch.cuda.Stream:
    key = torch.device(device).index
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = torch.cuda.Stream(device=device)
    return _SIDE_STREAMS[key]


def _keep(main: torch.cuda.Stream, *tensors) -> None:
    """Memory made on the side stream is later used on ``main``."""
    for t in tensors:
        if isinstance(t, NVFP4Tensor):
            for u in (t.codes, t.sf, t.scale):
                u.record_stream(main)
        elif isinstance(t, torch.Tensor):
            t.record_stream(main)


@dataclass(frozen=True)
class LayerConfig:
    """linear_graph.py:73-99, restricted to the Quartet II recipe this build accelerates."""

    forward_scheme: str = "rtn_1x16_46"
    backward_scheme: str = "ms_eden"
    ablation: str = "full"
    reuse_forward_weights: bool = False
    posthoc: bool = False

    def __post_init__(self):
        if self.forward_scheme not in FORWARD_SCHEMES:
            raise ValueError(f"unknown forward scheme {self.forward_scheme!r}")
        if self.backward_scheme not in BACKWARD_SCHEMES:
            raise ValueError(f"unknown backward scheme {self.backward_scheme!r}")
        if self.ablation != "full":
            raise ValueError(f"unknown ablation {self.ablation!r}")
        if self.reuse_forward_weights:
            raise ValueError("ms_eden requires weight re-quantization")


def baseline_config(name: str) -> LayerConfig:
    """linear_graph.py:143-150 (the accelerated recipe: quartet2)."""
    if name == "quartet2":
        return LayerConfig()
    raise ValueError(f"unknown baseline {name!r}; known: ['quartet2']")


@dataclass
class LinearTape:
    """Quantized forward operands saved for the backward pass (linear_graph.py:102-110)."""

    qX: NVFP4Tensor
    qW: NVFP4Tensor
    x_shape: tuple
    w_shape: tuple
    config: LayerConfig


@dataclass
class GradPair:
    dX: torch.Tensor
    dW: torch.Tensor


def gemm(qa: NVFP4Tensor, qb: NVFP4Tensor, out_dtype=torch.float32, out: torch.Tensor = None,
         accumulate: bool = False) -> torch.Tensor:
    """D = dequant(qa) . dequant(qb)^T on the tcgen05 NVFP4 kernel (FP32 accumulation)."""
    if qa.K != qb.K:
        raise ValueError(f"inner dimensions disagree: {qa.shape} vs {qb.shape}")
    M, N = qa.R, qb.R
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=qa.device)
    dt = _lib.Q2_F32 if out.dtype == torch.float32 else _lib.Q2_BF16
    if out.dtype not in (torch.float32, torch.bfloat16) or out.stride(-1) != 1:
        raise ValueError("output must be float32/bfloat16 with unit column stride")
    a, b = qa.c(), qb.c()
    _lib.check(_lib.lib().q2_gemm_tn(ctypes.byref(a), ctypes.byref(b), out.data_ptr(), dt, out.stride(0),
                                     int(accumulate), stream_handle()), "gemm")
    return out


def gemm_emulated(qa, qb, accumulate: str = "f32") -> torch.Tensor:
    """Name-compatible entry for linear_graph.gemm_emulated: FP32-accumulated NVFP4 GEMM."""
    if accumulate != "f32":
        raise ValueError(f"unknown accumulate precision {accumulate!r}")
    return gemm(qa, qb, torch.float32)


def _check_dims(x_shape, w_shape) -> None:
    """linear_graph.py:224-240 for quartet2 (ms_eden: all rotated dims % 128)."""
    tokens, in_dim = x_shape
    out_dim, w_in = w_shape
    if w_in != in_dim:
        raise ValueError(f"X is {x_shape} but W is {w_shape}")
    if in_dim % CHUNK or out_dim % CHUNK or tokens % CHUNK:
        raise ValueError(
            f"dims (tokens={tokens}, in={in_dim}, out={out_dim}) are not compatible with backward scheme "
            f"ms_eden; the rotated inner dimensions must be multiples of {CHUNK}")


def forward(x, w, cfg: LayerConfig = LayerConfig(), accumulate: str = "f32", out_dtype=torch.float32,
            err=None):
    """Quantized forward pass; returns (Y, tape) (linear_graph.py:243-256)."""
    x2, xs, _ = as_device_matrix(x, "X")
    w2, ws, _ = as_device_matrix(w, "W")
    _check_dims(xs, ws)
    own = err is None
    if own:
        err = _err_word(x2.device)
    main = torch.cuda.current_stream(x2.device)
    side = _side_stream(x2.device)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        qw = quantize_rtn_46(w2, _err=err)
    qx = quantize_rtn_46(x2, _err=err)
    main.wait_stream(side)
    _keep(main, qw)
    y = gemm(qx, qw, out_dtype)
    if own:
        _finish(err)
    return y, LinearTape(qx, qw, xs, ws, cfg)


def backward(tape: LinearTape, e, seeds: SeedPair, accumulate: str = "f32", dx_dtype=torch.float32,
             err=None) -> GradPair:
    """Backward from the tape and the output gradient (linear_graph.py:277-333)."""
    cfg = tape.config
    tokens, in_dim = tape.x_shape
    out_dim = tape.w_shape[0]
    e2, es, _ = as_device_matrix(e, "E")
    if es != (tokens, out_dim):
        raise ValueError(f"E has shape {es}, expected {(tokens, out_dim)}")
    mode = "posthoc" if cfg.posthoc else "exact"
    own = err is None
    if own:
        err = _err_word(e2.device)
    main = torch.cuda.current_stream(e2.device)
    side = _side_stream(e2.device)
    side.wait_stream(main)
    # dW = Q(E^T) Q(X^T)^T, inner dimension = tokens (side stream)
    with torch.cuda.stream(side):
        qet = msed(e2, seeds, 6.0, derive_stream(PAIR_DW, 0), PAIR_DW, mode, "cols", err)
        qxt = msed(tape.qX, seeds, 6.0, derive_stream(PAIR_DW, 1), PAIR_DW, mode, "tape", err)
        dw = gemm(qet, qxt, torch.float32)
    # dX = Q(E) Q(W^T)^T, inner dimension = out features
    qe = msed(e2, seeds, 6.0, derive_stream(PAIR_DX, 0), PAIR_DX, mode, "rows", err)
    qwt = msed(tape.qW, seeds, 6.0, derive_stream(PAIR_DX, 1), PAIR_DX, mode, "tape", err)
    dx = gemm(qe, qwt, dx_dtype)
    main.wait_stream(side)
    _keep(main, dw)
    e2.record_stream(side)
    for t in (tape.qX,):
        _keep(side, t)
    if own:
        _finish(err)
    return GradPair(dx, dw)
