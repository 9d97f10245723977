"""MS-EDEN backward quantizer (host mirror of ms_eden.py and posthoc.py).

``ms_eden_quantize`` / ``ms_eden_estimate_pair`` keep the reference's
signatures (ms_eden.py:116-180).  ``pass1`` / ``pass2`` mirror the post-hoc
range-alignment pipeline (posthoc.py:74-125); ``posthoc_quantize`` is
pass2(pass1(.)) in one call — the single-HBM-read schedule of PAPER.md:422-427.

Internal entry ``msed(...)`` additionally quantizes transposed views without
materialising them: a bf16/fp32 [K, R] tensor (E^T for the wgrad GEMM) or a
saved NVFP4 tape tensor (W^T, X^T of linear_graph.py:293-294, 304, 322-323).
"""

from __future__ import annotations

import ctypes

import numpy as np
from dataclasses import dataclass

import torch

from . import _lib
from .quantizers import (GROUP, NVFP4Tensor, _err_word, _finish, api, as_device_matrix, stream_handle)
from .rht import CHUNK, INV_SQRT_CHUNK, SeedPair, derive_stream, sign_mask, sr_stream

_MODES = {"exact": _lib.Q2_MSED_EXACT, "pow2": _lib.Q2_MSED_POW2, "posthoc": _lib.Q2_MSED_POSTHOC}


def _grid_s(s) -> float:
    s = float(getattr(s, "s", s))
    if not 0.0 < s <= 6.0:
        raise ValueError(f"grid max must be in (0, 6], got {s}")
    return s


@api
def msed(x, seeds: SeedPair, s=6.0, tensor_id: int = 0, rotation_id=None, mode: str = "exact",
         source: str = "rows", err=None, ws=None) -> NVFP4Tensor:
    """Quantize a logical [R, K] tensor along K with MS-EDEN.

    source="rows":  x is [R, K] (bf16/fp32)
    source="cols":  x is [K, R] (bf16/fp32); quantizes x^T
    source="tape":  x is an NVFP4Tensor of shape [K, R]; quantizes dequant(x)^T
    """
    s = _grid_s(s)
    if rotation_id is None:
        rotation_id = tensor_id
    L = _lib.lib()
    tape_c = None
    if source == "tape":
        if not isinstance(x, NVFP4Tensor) or len(x.shape) != 2:
            raise TypeError("tape source must be a 2-D NVFP4Tensor")
        K, R = x.shape
        dev = x.device
        src, xp, dt, ld = _lib.Q2_SRC_TAPE_COLS, None, _lib.Q2_BF16, 0
        tape_c = x.c()
    else:
        x2, shape, dt = as_device_matrix(x)
        dev = x2.device
        if source == "rows":
            R, K = x2.shape
            src = _lib.Q2_SRC_ROWS
            if shape[-1] % GROUP:
                raise ValueError(f"last dimension must be a multiple of {GROUP}")
        elif source == "cols":
            K, R = x2.shape
            src = _lib.Q2_SRC_COLS
        else:
            raise ValueError(f"unknown source {source!r}")
        xp, ld = x2.data_ptr(), x2.shape[1]
    if K % CHUNK:
        raise ValueError(f"last dimension must be a multiple of {CHUNK}")     # ms_eden.py:133-134
    out_shape = shape if source == "rows" else (R, K)
    out = NVFP4Tensor.empty(out_shape, dev)
    own = err is None
    if own:
        err = _err_word(dev)
    if ws is None:
        ws = torch.empty(L.q2_msed_ws_bytes(R, K), dtype=torch.uint8, device=dev)
    oc = out.c()
    mask = _lib._U32x4(*sign_mask(int(seeds.rht), int(rotation_id)))
    rc = L.q2_msed_quant(xp, dt, ctypes.byref(tape_c) if tape_c is not None else None, src, R, K, ld, mask, s,
                         INV_SQRT_CHUNK, int(seeds.sr) & (2**64 - 1), sr_stream(int(tensor_id)), _MODES[mode],
                         ctypes.byref(oc), ws.data_ptr(), err.data_ptr(), stream_handle())
    _lib.check(rc, "ms_eden")
    if own:
        _finish(err)
    return out


@api
def msed_dual(e, seeds: SeedPair, id_rows: int, rot_rows: int, id_cols: int, rot_cols: int, s=6.0,
              mode: str = "exact", err=None):
    """(MS(E), MS(E^T)) from ONE read of a bf16 E [T, N]: the dgrad and wgrad operands
    that read E (linear_graph.py:306, :325), each equal to ``msed`` with its own tensor /
    rotation ids.  Every 128x128 tile of E is rotated along its rows and its columns by
    two tensor-core MMAs from the same shared-memory copy (q2_msed_dual)."""
    s = _grid_s(s)
    e2, shape, dt = as_device_matrix(e, "E")
    T, N = e2.shape
    if dt != _lib.Q2_BF16 or T % CHUNK or N % CHUNK:
        raise ValueError("msed_dual needs a bfloat16 E with both dims multiples of 128")
    L = _lib.lib()
    dev = e2.device
    qr, qc = NVFP4Tensor.empty((T, N), dev), NVFP4Tensor.empty((N, T), dev)
    ws = torch.empty(L.q2_msed_dual_ws_bytes(T, N), dtype=torch.uint8, device=dev)
    own = err is None
    if own:
        err = _err_word(dev)
    a, b = qr.c(), qc.c()
    rc = L.q2_msed_dual(e2.data_ptr(), T, N, e2.stride(0), _lib._U32x4(*sign_mask(int(seeds.rht), int(rot_rows))),
                        _lib._U32x4(*sign_mask(int(seeds.rht), int(rot_cols))), s, INV_SQRT_CHUNK,
                        int(seeds.sr) & (2**64 - 1), sr_stream(int(id_rows)), sr_stream(int(id_cols)), _MODES[mode],
                        ctypes.byref(a), ctypes.byref(b), ws.data_ptr(), err.data_ptr(), stream_handle())
    _lib.check(rc, "msed_dual")
    if own:
        _finish(err)
    return qr, qc


def msed_dual_posthoc(e, seeds: SeedPair, id_rows: int, rot_rows: int, id_cols: int, rot_cols: int, s=6.0,
                      err=None):
    """``msed_dual`` in post-hoc mode: (pass2(pass1(E)), pass2(pass1(E^T)))."""
    return msed_dual(e, seeds, id_rows, rot_rows, id_cols, rot_cols, s, "posthoc", err)


def set_msed_engine(engine: str) -> None:
    """``"auto"`` (tensor-core kernel for the dual E source and the NVFP4 tape), ``"tc"`` (tensor-core kernel
    wherever eligible) or ``"literal"`` (literal float64 kernels).  Results are identical."""
    code = {"auto": 0, "tc": 1, "literal": 2}[engine]
    _lib.check(_lib.lib().q2_set_msed_engine(code), "q2_set_msed_engine")


def msed_stats(reset: bool = False):
    """(chunks quantized, chunks recomputed by the literal float64 path) of the
    tensor-core MS-EDEN kernels since load (host-synchronous)."""
    out = (ctypes.c_ulonglong * 2)()
    torch.cuda.synchronize()
    _lib.check(_lib.lib().q2_msed_stats(out, int(reset)), "q2_msed_stats")
    return int(out[0]), int(out[1])


@api
def ms_eden_quantize(x, seeds: SeedPair, s=6.0, tensor_id: int = 0, rotation_id=None,
                     pow2_scale: bool = False) -> NVFP4Tensor:
    """Rotate, RTN with cap 256, EDEN-correct, SR the scales (ms_eden.py:116-153)."""
    return msed(x, seeds, s, tensor_id, rotation_id, "pow2" if pow2_scale else "exact", "rows")


@api
def ms_eden_estimate_pair(a, b, seeds: SeedPair, pair_id: int = 0, s=6.0):
    """Both GEMM operands along their shared inner axis (ms_eden.py:156-180)."""
    if a.shape[-1] != b.shape[-1]:
        raise ValueError("operands must share the inner (last) dimension")
    qa = msed(a, seeds, s, derive_stream(pair_id, 0), pair_id)
    qb = msed(b, seeds, s, derive_stream(pair_id, 1), pair_id)
    return qa, qb


def posthoc_quantize(x, seeds: SeedPair, s=6.0, tensor_id: int = 0, rotation_id=None) -> NVFP4Tensor:
    """pass2(pass1(x)) in one call: the single-read MS-EDEN schedule."""
    return msed(x, seeds, s, tensor_id, rotation_id, "posthoc", "rows")


# ------------------------------------------------------------------ posthoc ---
@dataclass
class ErNvfp4Tensor:
    """Final FP4 codes + E8M3 pseudo-scales carried in bf16 (posthoc.py:51-63)."""

    codes: torch.Tensor          # uint8 [R, K/2] packed
    pseudo: torch.Tensor         # bfloat16-bits int16 [R, K/16]
    shape: tuple

    @property
    def pseudo_scales(self) -> torch.Tensor:
        return self.pseudo.view(torch.bfloat16).to(torch.float64).reshape(*self.shape[:-1], -1)


@dataclass
class Pass1Reductions:
    """posthoc.py:66-71 — red[0] rotated absmax, red[1] pseudo-scale max (float64 bits)."""

    red: torch.Tensor            # int64 [2]
    corrections: torch.Tensor    # float64 [R, K/128]

    @property
    def global_absmax(self) -> float:
        return float(self.red[:1].view(torch.float64).item())


@api
def pass1(x, seed_rht: int, s=6.0, tensor_id: int = 0, rotation_id=None):
    """Rotate, quantize against E8M3 pseudo-scales, reduce (posthoc.py:74-95)."""
    s = _grid_s(s)
    if rotation_id is None:
        rotation_id = tensor_id
    x2, shape, dt = as_device_matrix(x)
    R, K = x2.shape
    if K % CHUNK:
        raise ValueError(f"last dimension must be a multiple of {CHUNK}")
    dev = x2.device
    codes = torch.empty((R, K // 2), dtype=torch.uint8, device=dev)
    pseudo = torch.empty((R, K // GROUP), dtype=torch.int16, device=dev)
    corr = torch.empty((R, K // CHUNK), dtype=torch.float64, device=dev)
    red = torch.zeros(2, dtype=torch.int64, device=dev)
    err = _err_word(dev)
    mask = _lib._U32x4(*sign_mask(int(seed_rht), int(rotation_id)))
    rc = _lib.lib().q2_posthoc_pass1(x2.data_ptr(), dt, None, _lib.Q2_SRC_ROWS, R, K, K, mask, s, INV_SQRT_CHUNK,
                                     codes.data_ptr(), pseudo.data_ptr(), corr.data_ptr(), red.data_ptr(),
                                     err.data_ptr(), stream_handle())
    _lib.check(rc, "posthoc pass1")
    _finish(err)
    return ErNvfp4Tensor(codes, pseudo, shape), Pass1Reductions(red, corr)


@api
def pass2(er: ErNvfp4Tensor, red: Pass1Reductions, seed_sr: int, tensor_id: int = 0) -> NVFP4Tensor:
    """Align pseudo-scales into E4M3: shift, correct, SR (posthoc.py:98-125)."""
    dev = er.codes.device
    out = NVFP4Tensor.empty(er.shape, dev)
    out.codes.copy_(er.codes)
    err = _err_word(dev)
    oc = out.c()
    rc = _lib.lib().q2_posthoc_pass2(er.pseudo.data_ptr(), red.corrections.data_ptr(), red.red.data_ptr(),
                                     out.R, out.K, int(seed_sr) & (2**64 - 1), sr_stream(int(tensor_id)),
                                     ctypes.byref(oc), err.data_ptr(), stream_handle())
    _lib.check(rc, "posthoc pass2")
    _finish(err)
    return out


@dataclass
class CorrectionFactors:
    """Per-128-chunk rescaling factors (ms_eden.py:50-54)."""

    per_chunk: "torch.Tensor"


def _f64_device(x) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x, dtype=np.float64))
    return (x if x.is_cuda else x.cuda()).to(torch.float64).contiguous()


def chunk_correction_factors(x_rot, x_rtn) -> torch.Tensor:
    """EDEN factors S = <x,x>/<x,q> for every 128-chunk of the last axis, 1.0 when
    degenerate (ms_eden.py:75-83), in numpy's summation order: a float64 CUDA
    tensor [..., K/128] equal to the reference bit for bit."""
    xr, xq = _f64_device(x_rot), _f64_device(x_rtn)
    if xr.shape != xq.shape or xr.dim() == 0 or xr.shape[-1] % CHUNK:
        raise ValueError(f"chunk_correction_factors expects matching shapes with the last dimension a multiple of "
                         f"{CHUNK}")
    out = torch.empty(*xr.shape[:-1], xr.shape[-1] // CHUNK, dtype=torch.float64, device=xr.device)
    n = out.numel()
    rc = _lib.lib().q2_eden_factors(xr.data_ptr() if n else None, xq.data_ptr() if n else None, n,
                                    out.data_ptr() if n else None, stream_handle())
    _lib.check(rc, "q2_eden_factors")
    return out


def correction_factor(x_rot, x_rtn) -> float:
    """Factor of one 128-element chunk (ms_eden.py:57-72).  The reference forms the two
    dot products with BLAS (``@``), whose summation order is the BLAS build's; this
    uses numpy's pairwise ``.sum`` order, so results agree to rounding, not bits."""
    xr, xq = _f64_device(x_rot), _f64_device(x_rtn)
    if xr.shape != xq.shape or xr.shape[-1] != CHUNK or xr.dim() != 1:
        raise ValueError(f"correction_factor expects matching length-{CHUNK} chunks")
    return float(chunk_correction_factors(xr, xq)[0])
