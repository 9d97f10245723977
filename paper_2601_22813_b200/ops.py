"""torch.ops.quartet2.* -- the hot path as PyTorch custom operators.

The compute sits behind the C ABI of libquartet2.so (include/quartet2.h); these
registrations put it in the PyTorch dispatcher so graphs that hold it can be traced
(torch.compile / torch.export see the ops with their fake kernels and keep them as
opaque nodes) and checked with torch.library.opcheck.  Tensors cross the boundary
in the HBM layout of NVFP4Tensor: packed E2M1 codes uint8 [R, K/2], UE4M3 scales in
the tcgen05 block-scale layout uint8 [q2_sf_bytes(R, K)], fp32 tensor scale [1].

    torch.ops.quartet2.quantize_rtn_46(x) -> (codes, sf, scale)        quantizers.py:206-234
    torch.ops.quartet2.msed(x, seed_rht, seed_sr, tensor_id, rotation_id, mode, source)
                                              -> (codes, sf, scale)   ms_eden.py:116-153 / posthoc.py:74-125
    torch.ops.quartet2.msed_tape(codes, sf, scale, rows, cols, seed_rht, seed_sr, tensor_id,
                                 rotation_id, mode) -> (codes, sf, scale)  MS(dequant(tape)^T), linear_graph.py:293-326
    torch.ops.quartet2.gemm(a_codes, a_sf, a_scale, b_codes, b_sf, b_scale, k, out_fp32) -> D
                                                                      linear_graph.py:190-205

Seeds and stream ids are unsigned 64-bit in the reference; they travel as int64 (two's
complement) through the schema.
"""

from __future__ import annotations

from typing import Tuple

import torch

from .linear_graph import gemm as _gemm
from .ms_eden import msed as _msed
from .quantizers import NVFP4Tensor, quantize_rtn_46 as _q46
from .rht import SeedPair

_M64 = (1 << 64) - 1


def _u64(v: int) -> int:
    return int(v) & _M64


def _i64(v: int) -> int:
    v = int(v) & _M64
    return v - (1 << 64) if v >= 1 << 63 else v


def sf_bytes(R: int, K: int) -> int:
    """q2_sf_bytes: one 1 KiB block per (256-row block, 64-element K block)."""
    return ((R + 255) // 256) * ((K + 63) // 64) * 1024


def _parts(t: NVFP4Tensor) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    return t.codes, t.sf, t.scale


def _fake_parts(like: torch.Tensor, R: int, K: int):
    return (like.new_empty((R, K // 2), dtype=torch.uint8), like.new_empty((sf_bytes(R, K),), dtype=torch.uint8),
            like.new_empty((1,), dtype=torch.float32))


def _wrap(codes, sf, scale, R, K) -> NVFP4Tensor:
    return NVFP4Tensor(codes, sf, scale, (int(R), int(K)))


@torch.library.custom_op("quartet2::quantize_rtn_46", mutates_args=())
def quantize_rtn_46(x: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    return _parts(_q46(x))


@quantize_rtn_46.register_fake
def _(x):
    K = x.shape[-1]
    R = x.numel() // K if K else 0
    return _fake_parts(x, R, K)


@torch.library.custom_op("quartet2::msed", mutates_args=())
def msed(x: torch.Tensor, seed_rht: int, seed_sr: int, tensor_id: int, rotation_id: int, mode: str,
         source: str) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    t = _msed(x, SeedPair(_u64(seed_rht), _u64(seed_sr)), 6.0, _u64(tensor_id), _u64(rotation_id), mode, source)
    return _parts(t)


@msed.register_fake
def _(x, seed_rht, seed_sr, tensor_id, rotation_id, mode, source):
    T, N = x.shape[-2], x.shape[-1]
    R, K = (T, N) if source == "rows" else (N, T)
    return _fake_parts(x, R, K)


@torch.library.custom_op("quartet2::msed_tape", mutates_args=())
def msed_tape(codes: torch.Tensor, sf: torch.Tensor, scale: torch.Tensor, rows: int, cols: int, seed_rht: int,
              seed_sr: int, tensor_id: int, rotation_id: int, mode: str) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    t = _msed(_wrap(codes, sf, scale, rows, cols), SeedPair(_u64(seed_rht), _u64(seed_sr)), 6.0, _u64(tensor_id),
              _u64(rotation_id), mode, "tape")
    return _parts(t)


@msed_tape.register_fake
def _(codes, sf, scale, rows, cols, seed_rht, seed_sr, tensor_id, rotation_id, mode):
    return _fake_parts(codes, cols, rows)


@torch.library.custom_op("quartet2::gemm", mutates_args=())
def gemm(a_codes: torch.Tensor, a_sf: torch.Tensor, a_scale: torch.Tensor, b_codes: torch.Tensor,
         b_sf: torch.Tensor, b_scale: torch.Tensor, k: int, out_fp32: bool) -> torch.Tensor:
    qa = _wrap(a_codes, a_sf, a_scale, a_codes.shape[0], k)
    qb = _wrap(b_codes, b_sf, b_scale, b_codes.shape[0], k)
    return _gemm(qa, qb, torch.float32 if out_fp32 else torch.bfloat16)


@gemm.register_fake
def _(a_codes, a_sf, a_scale, b_codes, b_sf, b_scale, k, out_fp32):
    return a_codes.new_empty((a_codes.shape[0], b_codes.shape[0]), dtype=torch.float32 if out_fp32 else torch.bfloat16)


def linear_fwd_bwd(x, w, e, seeds: SeedPair, mode: str = "exact"):
    """The Quartet II layer (linear_graph.py:243-333) written with the custom ops only:
    Y, dX, dW in one traceable function (what torch.compile sees of the hot path)."""
    from .linear_graph import PAIR_DW, PAIR_DX
    from .rht import derive_stream as ds
    T, din = x.shape
    dout = w.shape[0]
    qx = torch.ops.quartet2.quantize_rtn_46(x)
    qw = torch.ops.quartet2.quantize_rtn_46(w)
    y = torch.ops.quartet2.gemm(*qx, *qw, din, False)
    s = (_i64(seeds.rht), _i64(seeds.sr))
    qe = torch.ops.quartet2.msed(e, *s, _i64(ds(PAIR_DX, 0)), _i64(PAIR_DX), mode, "rows")
    qwt = torch.ops.quartet2.msed_tape(*qw, dout, din, *s, _i64(ds(PAIR_DX, 1)), _i64(PAIR_DX), mode)
    dx = torch.ops.quartet2.gemm(*qe, *qwt, dout, True)
    qet = torch.ops.quartet2.msed(e, *s, _i64(ds(PAIR_DW, 0)), _i64(PAIR_DW), mode, "cols")
    qxt = torch.ops.quartet2.msed_tape(*qx, T, din, *s, _i64(ds(PAIR_DW, 1)), _i64(PAIR_DW), mode)
    dw = torch.ops.quartet2.gemm(*qet, *qxt, T, True)
    return y, dx, dw
