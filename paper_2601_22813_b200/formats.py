"""Element formats on the GPU (host mirror of formats.py): E2M1 / E4M3 encoders
(round-to-nearest and stochastic), the E8M3 pseudo-scale rounding and the two
decoders, with the reference's input checks and messages.  The arithmetic is
the device helpers the fused quantizers use (``q2_formats``, csrc/helpers.cu);
results are CUDA tensors (uint8 codes or float64 values)."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .quantizers import stream_handle

FP4_ABS_MAX = 6.0
E4M3_MAX = 448.0
E4M3_MIN_NORMAL = 2.0 ** -6
_GRID_EPS = 1e-9                                     # formats.py:47-50
_OP = {"fp4_rtn": 0, "fp4_sr": 1, "fp8_rtn": 2, "fp8_sr": 3, "e8m3": 4, "dec_fp4": 5, "dec_fp8": 6}


def _f64(x) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x, dtype=np.float64))
    if not x.is_cuda:
        x = x.cuda()
    return x.to(torch.float64).contiguous()


def _run(op: str, x=None, u=None, codes=None):
    src = x if x is not None else codes
    n = src.numel()
    out = torch.empty(src.shape, dtype=torch.float64 if op in ("e8m3", "dec_fp4", "dec_fp8") else torch.uint8,
                      device=src.device)
    err = torch.zeros(1, dtype=torch.int32, device=src.device) if op == "e8m3" else None
    if u is not None:
        u = torch.broadcast_to(_f64(u), src.shape).contiguous()
    ptr = lambda t: t.data_ptr() if t is not None and n else None   # noqa: E731
    rc = _lib.lib().q2_formats(_OP[op], ptr(x), ptr(u), ptr(codes), n,
                               ptr(out) if out.dtype == torch.uint8 else None,
                               ptr(out) if out.dtype == torch.float64 else None, ptr(err), stream_handle())
    _lib.check(rc, "q2_formats")
    if err is not None and int(err.item()) & _lib.Q2_ERR_E8M3_OVF:
        raise OverflowError("round_e8m3_rtn overflow beyond the bf16 carrier range")
    return out


def _checks(x: torch.Tensor, name: str, nonneg: bool) -> None:
    if x.numel() and bool(torch.isnan(x).any()):
        raise ValueError(f"NaN input to {name}")
    if nonneg and x.numel() and bool((x < 0).any()):
        raise ValueError(f"negative input to {name}")


def encode_fp4_rtn(x) -> torch.Tensor:
    """Round-to-nearest E2M1 codes, ties to even mantissa, saturating at +-6 (formats.py:116-124)."""
    x = _f64(x)
    _checks(x, "encode_fp4_rtn", False)
    return _run("fp4_rtn", x)


def encode_fp4_sr(x, u) -> torch.Tensor:
    """Stochastic E2M1 codes with draws u; inputs beyond +-6 raise (formats.py:127-157)."""
    x = _f64(x)
    _checks(x, "encode_fp4_sr", False)
    amax = float(x.abs().max()) if x.numel() else 0.0
    if amax > FP4_ABS_MAX * (1.0 + _GRID_EPS):
        raise ValueError(f"encode_fp4_sr input {amax} exceeds the FP4 grid max 6.0; "
                         "would clip; unbiasedness broken")
    return _run("fp4_sr", x, u)


def encode_fp8_rtn(x) -> torch.Tensor:
    """Nearest E4M3 code of non-negative x, ties to even, saturating at 448 (formats.py:160-171)."""
    x = _f64(x)
    _checks(x, "encode_fp8_rtn", True)
    return _run("fp8_rtn", x)


def encode_fp8_sr(x, u) -> torch.Tensor:
    """Stochastic E4M3 codes of non-negative x <= 448, RTN below 2^-6 (formats.py:174-201)."""
    x = _f64(x)
    _checks(x, "encode_fp8_sr", True)
    amax = float(x.max()) if x.numel() else 0.0
    if amax > E4M3_MAX * (1.0 + _GRID_EPS):
        raise ValueError(f"encode_fp8_sr input {amax} exceeds 448; "
                         "EDEN-corrected scale overflowed FP8; check grid cap")
    return _run("fp8_sr", x, u)


def round_e8m3_rtn(x):
    """Round non-negative x to 4 significant bits in the bf16 exponent range (formats.py:204-229);
    a Python float for a scalar input, else a float64 CUDA tensor."""
    scalar = np.ndim(x) == 0 if not isinstance(x, torch.Tensor) else x.dim() == 0
    x = _f64(x)
    _checks(x, "round_e8m3_rtn", True)
    out = _run("e8m3", x)
    return float(out) if scalar else out


def _codes(codes, limit: int) -> torch.Tensor:
    if not isinstance(codes, torch.Tensor):
        codes = torch.as_tensor(np.asarray(codes, dtype=np.uint8))
    codes = (codes.cuda() if not codes.is_cuda else codes).to(torch.uint8).contiguous()
    if codes.numel() and int(codes.max()) >= limit:
        raise IndexError(f"index {int(codes.max())} is out of bounds for axis 0 with size {limit}")
    return codes


def decode_fp4(codes) -> torch.Tensor:
    """E2M1 code(s) 0..15 to values; both zero codes give +0.0 (formats.py:76-78)."""
    return _run("dec_fp4", codes=_codes(codes, 16))


def decode_fp8(codes) -> torch.Tensor:
    """E4M3 code(s) 0..255 to values; the two NaN codes give NaN (formats.py:81-83)."""
    return _run("dec_fp8", codes=_codes(codes, 256))
