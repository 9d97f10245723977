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
from .ms_eden import msed, msed_dual
from .quantizers import (NVFP4Tensor, _err_word, _finish, api, as_device_matrix, dequantize, quantize_rtn_46,
                         stream_handle)
from .rht import CHUNK, SeedPair, derive_stream
from .sr import SquareBlockTensor, quantize_sr, quantize_sr_46, quantize_square_block, sr_operand

FORWARD_SCHEMES = ("rtn_1x16_46", "rtn_1x16", "rtn_16x16", "rtn_16x16_46", "identity")
BACKWARD_SCHEMES = ("ms_eden", "sr_rht", "sr", "sr_46", "sr_rht_46", "identity")
ABLATIONS = ("a", "b", "c", "d", "e", "full")
# Operands each ablation quantizes: (E in dX, W^T in dX, E^T in dW, X^T in dW), linear_graph.py:59-70
ABLATION_MASK = {"a": (False, False, True, True), "b": (True, False, False, False),
                 "c": (True, True, False, False), "d": (True, False, True, True),
                 "e": (True, True, True, True), "full": (True, True, True, True)}
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
    """linear_graph.py:73-99.  ``posthoc`` (not in the reference) selects the
    single-read post-hoc MS-EDEN schedule for the four backward quantizations."""

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
        if self.ablation not in ABLATIONS:
            raise ValueError(f"unknown ablation {self.ablation!r}")
        if self.backward_scheme == "ms_eden":
            if self.ablation in ("b", "d"):
                raise ValueError("ms_eden cannot quantize a single GEMM operand; "
                                 f"ablation {self.ablation!r} is incompatible")
            if self.reuse_forward_weights:
                raise ValueError("ms_eden requires weight re-quantization")
        if self.reuse_forward_weights and not self.forward_scheme.startswith("rtn_16x16"):
            raise ValueError("weight reuse requires a square-block forward scheme")


def format_config(cfg: LayerConfig) -> str:
    """The key = value text form (linear_graph.py:153-159); ``posthoc`` is written only when set."""
    text = (f"forward_scheme = {cfg.forward_scheme}\n"
            f"backward_scheme = {cfg.backward_scheme}\n"
            f"ablation = {cfg.ablation}\n"
            f"reuse_forward_weights = {str(cfg.reuse_forward_weights).lower()}\n")
    return text + ("posthoc = true\n" if cfg.posthoc else "")


def parse_config(text: str) -> LayerConfig:
    """Parse ``format_config`` text (linear_graph.py:162-182): '#' comments, blank lines,
    unset keys default to the identity recipe; errors name the line."""
    fields = {}
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"config line {lineno}: expected key = value")
        key, val = (part.strip() for part in line.split("=", 1))
        if key in ("reuse_forward_weights", "posthoc"):
            if val not in ("true", "false"):
                raise ValueError(f"config line {lineno}: expected true/false")
            fields[key] = val == "true"
        elif key in ("forward_scheme", "backward_scheme", "ablation"):
            fields[key] = val
        else:
            raise ValueError(f"config line {lineno}: unknown key {key!r}")
    base = {"forward_scheme": "identity", "backward_scheme": "identity"}
    base.update(fields)
    return LayerConfig(**base)


def baseline_config(name: str) -> LayerConfig:
    """linear_graph.py:119-150 for the accelerated recipes."""
    if name == "quartet2":
        return LayerConfig()
    if name == "tetrajet_v2":
        return LayerConfig("rtn_1x16", "sr_rht")
    if name == "nvidia":
        return LayerConfig("rtn_16x16", "sr_rht", reuse_forward_weights=True)
    if name == "four_over_six":
        return LayerConfig("rtn_16x16_46", "sr_rht", reuse_forward_weights=True)
    if name == "four_over_six_backward":
        return LayerConfig("rtn_16x16_46", "sr_46", reuse_forward_weights=True)
    if name == "identity":
        return LayerConfig("identity", "identity")
    known = sorted(["quartet2", "tetrajet_v2", "nvidia", "four_over_six", "four_over_six_backward", "identity"])
    raise ValueError(f"unknown baseline {name!r}; known: {known}")


@dataclass
class LinearTape:
    """Quantized forward operands saved for the backward pass (linear_graph.py:102-110)."""

    qX: NVFP4Tensor
    qW: "NVFP4Tensor | SquareBlockTensor"
    x_shape: tuple
    w_shape: tuple
    config: LayerConfig


@dataclass
class GradPair:
    dX: torch.Tensor
    dW: torch.Tensor


_ACC_MODES = {False: _lib.Q2_ACC_STORE, True: _lib.Q2_ACC_ADD, "store": _lib.Q2_ACC_STORE,
              "add": _lib.Q2_ACC_ADD, "red": _lib.Q2_ACC_RED, "multimem": _lib.Q2_ACC_MULTIMEM}


def gemm(qa: NVFP4Tensor, qb: NVFP4Tensor, out_dtype=torch.float32, out: torch.Tensor = None,
         accumulate=False, multicast_ptr: int = 0) -> torch.Tensor:
    """D = dequant(qa) . dequant(qb)^T on the tcgen05 NVFP4 kernel (FP32 accumulation).

    ``accumulate``: False / "store" (D = A.B^T), True / "add" (D += A.B^T, this call is the
    only writer), "red" (D += A.B^T by atomic reductions: concurrent writers allowed) or
    "multimem" (the epilogue adds the tile into every rank's replica of ``out`` through the
    NVLS multicast address ``multicast_ptr`` of ``out``'s symmetric buffer: the dW
    all-reduce fused into the wgrad GEMM; see ``parallel.MulticastReducer``)."""
    if accumulate not in _ACC_MODES:
        raise ValueError(f"unknown accumulate mode {accumulate!r}")
    acc = _ACC_MODES[accumulate]
    if acc != _lib.Q2_ACC_STORE and (out is None or out.dtype != torch.float32):
        raise ValueError("accumulating GEMMs need a float32 `out`")
    if (acc == _lib.Q2_ACC_MULTIMEM) != bool(multicast_ptr):
        raise ValueError("multicast_ptr is required by, and only by, accumulate='multimem'")
    if qa.K != qb.K:
        raise ValueError(f"inner dimensions disagree: {qa.shape} vs {qb.shape}")
    M, N = qa.R, qb.R
    if qa.device != qb.device:
        raise ValueError(f"operands on different devices: {qa.device} vs {qb.device}")
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=qa.device)
    if out.dtype not in (torch.float32, torch.bfloat16) or out.dim() != 2 or out.stride(-1) != 1:
        raise ValueError("output must be a 2-D float32/bfloat16 tensor with unit column stride")
    if tuple(out.shape) != (M, N) or out.device != qa.device or out.stride(0) < N:
        raise ValueError(f"output must be ({M}, {N}) on {qa.device} with row stride >= {N}, "
                         f"got {tuple(out.shape)} on {out.device} (stride {out.stride(0)})")
    dt = _lib.Q2_F32 if out.dtype == torch.float32 else _lib.Q2_BF16
    a, b = qa.c(), qb.c()
    with torch.cuda.device(qa.device), torch.cuda.nvtx.range("q2.gemm"):
        dst = multicast_ptr if acc == _lib.Q2_ACC_MULTIMEM else out.data_ptr()
        _lib.check(_lib.lib().q2_gemm_tn(ctypes.byref(a), ctypes.byref(b), dst, dt, out.stride(0),
                                         acc, stream_handle()), "gemm")
    return out


def _dense64(t) -> torch.Tensor:
    if isinstance(t, (NVFP4Tensor, SquareBlockTensor)):
        return dequantize(t)
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    return (t if t.is_cuda else t.cuda()).to(torch.float64)


def gemm_emulated(qa, qb, accumulate: str = "f32") -> torch.Tensor:
    """linear_graph.gemm_emulated (linear_graph.py:190-205): ``"f32"`` runs the tcgen05
    NVFP4 GEMM when both operands are NVFP4 (an FP32 product of the dequantized values
    when one is a plain tensor); ``"f64"`` is the float64 product of the dequantized
    operands (cuBLAS DGEMM), the reference's oracle mode."""
    if accumulate not in ("f32", "f64"):
        raise ValueError(f"unknown accumulate precision {accumulate!r}")
    quantized = isinstance(qa, NVFP4Tensor) and isinstance(qb, NVFP4Tensor)
    if accumulate == "f32" and quantized:
        return gemm(qa, qb, torch.float32)
    a, b = _dense64(qa), _dense64(qb)
    if a.shape[-1] != b.shape[-1]:
        raise ValueError(f"inner dimensions disagree: {tuple(a.shape)} vs {tuple(b.shape)}")
    if accumulate == "f64":
        return a @ b.t()
    return a.float() @ b.float().t()


def _check_dims(x_shape, w_shape, cfg: LayerConfig) -> None:
    """linear_graph.py:224-240: the rotated inner dimensions (out, tokens) are
    multiples of 128; in must be too for ms_eden (a multiple of 16 otherwise,
    and of 64 for this build's transposed-tape source)."""
    tokens, in_dim = x_shape
    out_dim, w_in = w_shape
    if w_in != in_dim:
        raise ValueError(f"X is {x_shape} but W is {w_shape}")
    if cfg.forward_scheme != "identity" and in_dim % 16:
        raise ValueError("in dimension must be a multiple of 16")
    if cfg.backward_scheme == "identity":
        return
    in_div = CHUNK if cfg.backward_scheme == "ms_eden" else 16
    if in_dim % in_div or out_dim % CHUNK or tokens % CHUNK:
        raise ValueError(
            f"dims (tokens={tokens}, in={in_dim}, out={out_dim}) are not compatible with backward scheme "
            f"{cfg.backward_scheme}; the rotated inner dimensions must be multiples of {CHUNK}")
    if in_dim % 64:
        raise ValueError(f"in dimension {in_dim}: the B200 transposed-tape quantizer needs a multiple of 64")


@api
def forward(x, w, cfg: LayerConfig = LayerConfig(), accumulate: str = "f32", out_dtype=torch.float32,
            err=None):
    """Quantized forward pass; returns (Y, tape) (linear_graph.py:243-256)."""
    x2, xs, _ = as_device_matrix(x, "X")
    w2, ws, _ = as_device_matrix(w, "W")
    _check_dims(xs, ws, cfg)
    caps = (6.0, 4.0) if cfg.forward_scheme.endswith("_46") else (6.0,)   # linear_graph.py:208-221
    if accumulate not in ("f32", "f64"):
        raise ValueError(f"unknown accumulate precision {accumulate!r}")
    if cfg.forward_scheme == "identity":              # unquantized: plain FP32 GEMM (cuBLAS), linear_graph.py:208-210
        y = gemm_emulated(x2, w2, accumulate)
        y = y.to(out_dtype) if accumulate == "f32" else y
        return y, LinearTape(x2, w2, xs, ws, cfg)
    own = err is None
    if own:
        err = _err_word(x2.device)
    main = torch.cuda.current_stream(x2.device)
    side = _side_stream(x2.device)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        if cfg.forward_scheme.startswith("rtn_16x16"):                     # linear_graph.py:214-221
            qw = quantize_square_block(w2, len(caps) == 2, _err=err)
        else:
            qw = quantize_rtn_46(w2, caps, _err=err)
    qx = quantize_rtn_46(x2, caps, _err=err)
    main.wait_stream(side)
    wop = qw.rows if isinstance(qw, SquareBlockTensor) else qw
    for t in ((qw.rows, qw.t) if isinstance(qw, SquareBlockTensor) else (qw,)):
        _keep(main, t)
    y = gemm(qx, wop, out_dtype) if accumulate == "f32" else gemm_emulated(qx, wop, accumulate)
    if own:
        _finish(err)
    return y, LinearTape(qx, qw, xs, ws, cfg)


@api
def backward(tape: LinearTape, e, seeds: SeedPair, accumulate: str = "f32", dx_dtype=torch.float32,
             err=None, operands: dict | None = None, dw_out: torch.Tensor | None = None,
             dw_accumulate="store", dw_multicast_ptr: int = 0) -> GradPair:
    """Backward from the tape and the output gradient (linear_graph.py:277-333).

    ``dw_out`` / ``dw_accumulate`` / ``dw_multicast_ptr``: the wgrad GEMM writes into a
    caller-owned fp32 [out, in] buffer with ``gemm``'s accumulate modes ("store", "add",
    "red", or "multimem": dW summed over the data-parallel ranks inside the GEMM epilogue
    through the buffer's NVLS multicast address, ``parallel.MulticastReducer``).  The
    returned ``dW`` is then ``dw_out`` (complete only after the caller's cross-rank barrier
    in the "multimem" case).
    ``operands``: optional dict that receives the four quantized GEMM operands the call
    computed ("E", "Wt" for dX; "Et", "Xt" for dW; None where an operand stays dense),
    for parity checks of the exact tensors the GEMMs consumed."""
    cfg = tape.config
    tokens, in_dim = tape.x_shape
    out_dim = tape.w_shape[0]
    e2, es, _ = as_device_matrix(e, "E")
    if es != (tokens, out_dim):
        raise ValueError(f"E has shape {es}, expected {(tokens, out_dim)}")
    mode = "posthoc" if cfg.posthoc else "exact"
    if dw_out is not None and (dw_out.dtype != torch.float32 or tuple(dw_out.shape) != (out_dim, in_dim)):
        raise ValueError(f"dw_out must be a float32 {(out_dim, in_dim)} tensor")
    if dw_accumulate not in ("store", "add", "red", "multimem") or (dw_accumulate != "store" and dw_out is None):
        raise ValueError(f"dw_accumulate={dw_accumulate!r} needs dw_out (store/add/red/multimem)")
    if accumulate not in ("f32", "f64"):
        raise ValueError(f"unknown accumulate precision {accumulate!r}")
    f64 = accumulate == "f64"                         # float64 products (the reference's oracle mode)
    wide = torch.float64 if f64 else torch.float32
    dx_dtype = torch.float64 if f64 else dx_dtype
    dense = lambda t: _dense64(t).to(wide)            # noqa: E731
    if cfg.backward_scheme == "identity":             # no backward quantization (linear_graph.py:286-288)
        ef = e2.to(wide)
        dw = torch.matmul(ef.t(), dense(tape.qX))
        if dw_out is not None:
            if dw_accumulate == "multimem":
                raise ValueError("the multicast dW reduction needs both wgrad operands in NVFP4 (f32 accumulate)")
            dw = dw_out.add_(dw) if dw_accumulate in ("add", "red") else dw_out.copy_(dw)
        return GradPair(torch.matmul(ef, dense(tape.qW)).to(dx_dtype), dw)
    own = err is None
    if own:
        err = _err_word(e2.device)
    main = torch.cuda.current_stream(e2.device)
    side = _side_stream(e2.device)
    side.wait_stream(main)
    # Ablation masks (linear_graph.py:296): operands outside the mask stay dense, and a
    # GEMM with a dense operand runs as the reference's fp32 product of the dequantized
    # values (cuBLAS); ms_eden needs both operands of a GEMM, SR rotates only when both
    # are quantized (_sr_pair, linear_graph.py:259-274).
    q_e, q_w, q_et, q_xt = ABLATION_MASK[cfg.ablation]
    sr_scheme = cfg.backward_scheme != "ms_eden"
    sr_46 = cfg.backward_scheme in ("sr_46", "sr_rht_46")
    rht = cfg.backward_scheme in ("sr_rht", "sr_rht_46")

    def quant(x, pair, operand, source, both):
        if sr_scheme:                                   # _sr_pair via linear_graph.py:310-331
            return sr_operand(x, seeds, derive_stream(pair, operand), pair, source, rht and both, sr_46, err)
        return msed(x, seeds, 6.0, derive_stream(pair, operand), pair, mode, source, err)   # :304-307, :322-326

    def product(qa, qb, a_dense, b_dense, out_dtype):
        """gemm_emulated(qa, qb): the NVFP4 GEMM when both operands are quantized, else
        fp32 of the (dequantized) operands; a_dense/b_dense give the dense [M,K]/[N,K]."""
        if qa is not None and qb is not None and not f64:
            return gemm(qa, qb, out_dtype)
        a = dense(qa) if qa is not None else a_dense()
        b = dense(qb) if qb is not None else b_dense()
        return torch.matmul(a, b.t()).to(out_dtype)

    def wprod(qa, qb, a_dense, b_dense):
        """The wgrad product, into ``dw_out`` with its accumulate mode when one is given."""
        if dw_out is None:
            return product(qa, qb, a_dense, b_dense, wide)
        if qa is not None and qb is not None and not f64:
            return gemm(qa, qb, torch.float32, out=dw_out, accumulate=dw_accumulate,
                        multicast_ptr=dw_multicast_ptr)
        if dw_accumulate == "multimem":
            raise ValueError("the multicast dW reduction needs both wgrad operands in NVFP4 (f32 accumulate)")
        a = dense(qa) if qa is not None else a_dense()
        b = dense(qb) if qb is not None else b_dense()
        r = torch.matmul(a.float(), b.float().t())
        return dw_out.add_(r) if dw_accumulate in ("add", "red") else dw_out.copy_(r)

    # MS-EDEN of E for both GEMMs from one read of E (tensor-core dual kernel) when E is a
    # bf16 [tokens, out] with both dims multiples of 128; identical results to two msed calls
    dual = (not sr_scheme and q_e and q_w and q_et and q_xt and e2.dtype == torch.bfloat16
            and tokens % CHUNK == 0 and out_dim % CHUNK == 0)
    if dual:
        qe_d, qet_d = msed_dual(e2, seeds, derive_stream(PAIR_DX, 0), PAIR_DX, derive_stream(PAIR_DW, 0), PAIR_DW,
                                6.0, mode, err)
        e_done = torch.cuda.Event()
        e_done.record(main)
    with torch.cuda.stream(side):
        # dW = Q(E^T) Q(X^T)^T, inner dimension = tokens (side stream)
        if dual:
            qxt = quant(tape.qX, PAIR_DW, 1, "cols" if isinstance(tape.qX, torch.Tensor) else "tape", True)
            side.wait_event(e_done)
            qet = qet_d
            dw = wprod(qet, qxt, None, None)
            _keep(side, qet_d)                           # made on the caller's stream, read here
        elif (q_et or q_xt) if sr_scheme else (q_et and q_xt):
            both = q_et and q_xt
            qet = quant(e2, PAIR_DW, 0, "cols", both) if q_et else None
            qxt = quant(tape.qX, PAIR_DW, 1, "cols" if isinstance(tape.qX, torch.Tensor) else "tape",
                        both) if q_xt else None
        else:
            qet = qxt = None
        if dual:
            pass
        else:
            dw = wprod(qet, qxt, lambda: e2.to(wide).t(), lambda: dense(tape.qX).t())
    # dX = Q(E) Q(W^T)^T, inner dimension = out features
    qw = tape.qW.rows if isinstance(tape.qW, SquareBlockTensor) else tape.qW
    qe = qwt = None
    if cfg.reuse_forward_weights and q_w and sr_scheme:
        # saved square-block W^T goes in as is; E alone, SR without rotation (linear_graph.py:308-314)
        qe = (quantize_sr_46 if sr_46 else quantize_sr)(e2, seeds.sr, derive_stream(PAIR_DX, 0), _err=err) \
            if q_e else None
        qwt = tape.qW.t
    elif dual:
        qe = qe_d
        qwt = quant(qw, PAIR_DX, 1, "cols" if isinstance(qw, torch.Tensor) else "tape", True)
    elif (q_e or q_w) if sr_scheme else (q_e and q_w):
        both = q_e and q_w
        qe = quant(e2, PAIR_DX, 0, "rows", both) if q_e else None
        qwt = quant(qw, PAIR_DX, 1, "cols" if isinstance(qw, torch.Tensor) else "tape", both) if q_w else None
    if qe is None and qwt is None:
        dx = torch.matmul(e2.to(wide), dense(tape.qW)).to(dx_dtype)
    else:
        dx = product(qe, qwt, lambda: e2.to(wide), lambda: dense(tape.qW).t(), dx_dtype)
    main.wait_stream(side)
    if operands is not None:
        operands.update(E=qe, Wt=qwt, Et=qet, Xt=qxt)
    _keep(main, dw)
    e2.record_stream(side)
    for t in (tape.qX,):
        _keep(side, t)
    if own:
        _finish(err)
    return GradPair(dx, dw)
