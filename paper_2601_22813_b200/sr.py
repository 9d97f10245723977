"""Baseline-recipe quantizers: stochastic rounding (host mirror of
quantizers.py:139-161, :237-262 and linear_graph._sr_pair, linear_graph.py:259-274)
and 16x16 square blocks (quantizers.py:102-111, :265-312).

``quantize_sr`` / ``quantize_sr_46`` keep the reference's signatures.  ``rht_sr``
is one operand of the ``sr_rht`` backward scheme (the tetrajet_v2 recipe):
``quantize_sr(rht_apply(x, seeds.rht, rotation_id), seeds.sr, stream)``, with
the same transposed sources as ``ms_eden.msed`` (E^T from E, W^T / X^T from the
NVFP4 tape) and no materialised rotation.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .quantizers import (FP8_RTN_MARGIN, GROUP, GUARDED_SCALE_CAP, NVFP4Tensor, _err_word, _finish,
                         as_device_matrix, stream_handle)
from .rht import CHUNK, INV_SQRT_CHUNK, SeedPair, derive_stream, sign_mask

FP4_ABS_MAX, E4M3_MAX = 6.0, 448.0
# quantizers.py:151 -- FP4_ABS_MAX * FP8_RTN_MARGIN * E4M3_MAX in the reference's float64 order
_SR_SCALE_DIV = FP4_ABS_MAX * FP8_RTN_MARGIN * E4M3_MAX
_M64 = 2 ** 64 - 1


def _sr(x, seed, streams, caps, scale_div, err) -> NVFP4Tensor:
    x2, shape, dt = as_device_matrix(x)
    if shape[-1] % GROUP:
        raise ValueError(f"last dimension must be a multiple of {GROUP}")
    out = NVFP4Tensor.empty(shape, x2.device)
    own = err is None
    if own:
        err = _err_word(x2.device)
    L = _lib.lib()
    ws = torch.empty(L.q2_quant_sr_ws_bytes(), dtype=torch.uint8, device=x2.device)
    oc = out.c()
    c1 = float(caps[1]) if len(caps) > 1 else 0.0
    s1 = streams[1] if len(streams) > 1 else 0
    _lib.check(L.q2_quant_sr(x2.data_ptr(), dt, x2.shape[0], x2.shape[1], x2.shape[1], len(caps), float(caps[0]), c1,
                             FP8_RTN_MARGIN, float(scale_div), int(seed) & _M64, int(streams[0]) & _M64, int(s1) & _M64,
                             ctypes.byref(oc), ws.data_ptr(), err.data_ptr(), stream_handle()), "quantize_sr")
    if own:
        _finish(err)
    return out


def quantize_sr(x, seed, stream=0, _err=None) -> NVFP4Tensor:
    """Unbiased NVFP4 with stochastic element rounding (quantizers.py:139-161)."""
    return _sr(x, seed, (stream,), (FP4_ABS_MAX,), _SR_SCALE_DIV, _err)


def quantize_sr_46(x, seed, stream=0, caps=(6.0, 4.0), _err=None) -> NVFP4Tensor:
    """SR under both ceilings, per-group lower realised error (quantizers.py:237-262)."""
    caps = tuple(float(c) for c in caps)
    if len(caps) != 2:
        raise ValueError("quantize_sr_46 takes two grid ceilings")
    return _sr(x, seed, (derive_stream(stream, 0), derive_stream(stream, 1)), caps, caps[0] * GUARDED_SCALE_CAP, _err)


def sr_operand(x, seeds: SeedPair, stream: int, rotation_id: int, source: str = "rows", rotate: bool = True,
               use_46: bool = False, err=None) -> NVFP4Tensor:
    """One operand of an SR backward scheme (_sr_pair, linear_graph.py:259-274) of a logical [R, K] tensor:
    quantize_sr / quantize_sr_46 (use_46) of x, or of rht_apply(x, seeds.rht, rotation_id) (rotate).

    source="rows": x is [R, K]; "cols": x is [K, R] (quantizes x^T); "tape": x
    is an NVFP4Tensor [K, R] (quantizes dequant(x)^T).
    """
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
        x2, _, dt = as_device_matrix(x)
        dev = x2.device
        if source == "rows":
            R, K = x2.shape
            src = _lib.Q2_SRC_ROWS
        elif source == "cols":
            K, R = x2.shape
            src = _lib.Q2_SRC_COLS
        else:
            raise ValueError(f"unknown source {source!r}")
        xp, ld = x2.data_ptr(), x2.shape[1]
    if K % CHUNK:
        # rht.py:147-150 for the rotation; this build's transposed sources tile K by 128 as well
        raise ValueError(f"rotation requires the last dimension ({K}) to be a multiple of {CHUNK}")
    out = NVFP4Tensor.empty((R, K), dev)
    own = err is None
    if own:
        err = _err_word(dev)
    ws = torch.empty(L.q2_msed_ws_bytes(R, K), dtype=torch.uint8, device=dev)
    oc = out.c()
    mask = _lib._U32x4(*sign_mask(int(seeds.rht), int(rotation_id)))
    if use_46:                                            # quantizers.py:237-262
        caps, div, streams = (6.0, 4.0), 6.0 * GUARDED_SCALE_CAP, (derive_stream(stream, 0), derive_stream(stream, 1))
    else:                                                 # quantizers.py:139-161
        caps, div, streams = (FP4_ABS_MAX, 0.0), _SR_SCALE_DIV, (stream, 0)
    rc = L.q2_sr_quant_src(xp, dt, ctypes.byref(tape_c) if tape_c is not None else None, src, R, K, ld,
                           int(bool(rotate)), mask, 2 if use_46 else 1, caps[0], caps[1], FP8_RTN_MARGIN, div,
                           INV_SQRT_CHUNK, int(seeds.sr) & _M64, int(streams[0]) & _M64, int(streams[1]) & _M64,
                           ctypes.byref(oc), ws.data_ptr(), err.data_ptr(), stream_handle())
    _lib.check(rc, "sr_operand")
    if own:
        _finish(err)
    return out


def rht_sr(x, seeds: SeedPair, stream: int, rotation_id: int, source: str = "rows", err=None) -> NVFP4Tensor:
    """quantize_sr(rht_apply(x, seeds.rht, rotation_id), seeds.sr, stream): one sr_rht operand."""
    return sr_operand(x, seeds, stream, rotation_id, source, True, False, err)


class SquareBlockTensor:
    """quantizers.py:102-111: codes [R, C], one E4M3 scale per 16x16 block.

    Held in HBM twice for the GEMMs -- ``rows`` ([R, C], the forward weight
    operand) and ``t`` (its transpose [C, R], the reused dX operand) -- each with
    the block scale expanded into the per-16 layout, plus the compact block
    scales ``s8`` [R/16, C/16].  ``to_reference()`` gives (fp4, scales8, scale32).
    """

    def __init__(self, rows: NVFP4Tensor, t: NVFP4Tensor, s8: torch.Tensor):
        self.rows, self.t, self.s8 = rows, t, s8

    @property
    def shape(self):
        return self.rows.shape

    @property
    def device(self):
        return self.rows.device

    @property
    def scale32(self):
        return self.rows.scale32

    def to_reference(self):
        fp4, _, s32 = self.rows.to_reference()
        return fp4, self.s8.cpu().numpy(), s32


def quantize_square_block(x, use_46: bool = False, _err=None) -> SquareBlockTensor:
    """One E4M3 scale per 16x16 block, cap 256; 6/4 per block with use_46 (quantizers.py:265-312)."""
    x2, shape, dt = as_device_matrix(x)
    if len(shape) != 2 or shape[0] % GROUP or shape[1] % GROUP:
        raise ValueError("square-block input must be 2D with both dims multiples of 16")
    R, C = x2.shape
    rows, t = NVFP4Tensor.empty((R, C), x2.device), NVFP4Tensor.empty((C, R), x2.device)
    s8 = torch.empty((R // GROUP, C // GROUP), dtype=torch.uint8, device=x2.device)
    own = _err is None
    err = _err_word(x2.device) if own else _err
    L = _lib.lib()
    ws = torch.empty(16, dtype=torch.uint8, device=x2.device)
    rc_, tc_ = rows.c(), t.c()
    _lib.check(L.q2_quant_square_block(x2.data_ptr(), dt, R, C, int(bool(use_46)), ctypes.byref(rc_), ctypes.byref(tc_),
                                       s8.data_ptr(), ws.data_ptr(), err.data_ptr(), stream_handle()),
               "quantize_square_block")
    if own:
        _finish(err)
    return SquareBlockTensor(rows, t, s8)
