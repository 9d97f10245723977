"""Seeds, stream ids and rotation sign vectors (host side).

Integer-exact ports of the reference's counter-based PRNG plumbing
(rht.py:36-106).  Only the per-group scale draws of MS-EDEN run on the device
(common.cuh prng_uniform); the 128-entry sign vector of a rotation is drawn
here once and passed to the kernels as a 128-bit mask.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

CHUNK = 128
_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
DOMAIN_SIGNS = 0x53494748       # rht.py:42
DOMAIN_SCALE_SR = 0x5343414C    # ms_eden.py:47
INV_SQRT_CHUNK = CHUNK ** -0.5  # rht.py:154, the float64 the reference multiplies by


@dataclass(frozen=True)
class SeedPair:
    """Rotation seed and rounding seed of one quantization event (rht.py:45-50)."""

    rht: int
    sr: int


def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _bits(seed: int, stream: int, index: int) -> int:
    """rht.py:63-68"""
    z = _mix64((seed + _GOLDEN) & _M64)
    z = _mix64(z ^ ((stream + _GOLDEN) & _M64))
    return _mix64(z ^ ((index + _GOLDEN) & _M64))


def _fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for byte in data:
        h = ((h ^ byte) * 0x100000001B3) & _M64
    return h


def derive_stream(*parts) -> int:
    """Mix integers (or short string tags) into one 64-bit stream id (rht.py:78-86)."""
    z = 0
    for p in parts:
        if isinstance(p, (str, bytes)):
            p = _fnv1a64(p.encode() if isinstance(p, str) else p)
        z = _mix64(z ^ ((int(p) + _GOLDEN) & _M64))
    return z


def prng_uniform(seed: int, stream: int, index: int) -> float:
    """One uniform [0,1) draw (rht.py:89-96)."""
    return (_bits(seed & _M64, stream & _M64, index & _M64) >> 11) * 2.0 ** -53


def _negative_draws(seed: int, stream: int, n: int) -> np.ndarray:
    """``prng_uniform(seed, stream, i) >= 0.5`` for i < n, i.e. bit 63 of ``_bits``: the
    seed/stream prefix is shared, the n index mixes run as one uint64 vector
    (wrap-around arithmetic, the same integers as rht.py:57-68)."""
    z0 = _mix64(_mix64((seed + _GOLDEN) & _M64) ^ ((stream + _GOLDEN) & _M64))
    z = np.uint64(z0) ^ (np.arange(n, dtype=np.uint64) + np.uint64(_GOLDEN))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return ((z ^ (z >> np.uint64(31))) >> np.uint64(63)).astype(bool)


def prng_signs(seed: int, stream: int, n: int) -> np.ndarray:
    """n deterministic +-1 signs from the stream (rht.py:99-102), float64."""
    return np.where(_negative_draws(seed & _M64, stream & _M64, n), -1.0, 1.0)


@lru_cache(maxsize=1024)
def sign_mask(seed: int, rotation_id: int) -> tuple:
    """The rotation's 128 signs (rht.py:99-106) as four u32 words, bit i = sign i is -1."""
    neg = _negative_draws(seed & _M64, derive_stream(DOMAIN_SIGNS, rotation_id), CHUNK).astype(np.uint64)
    words = (neg.reshape(4, 32) << np.arange(32, dtype=np.uint64)).sum(axis=1)
    return tuple(int(w) for w in words)


def _rotation_call(x, chunk: int, pre, post, scale: float):
    """q2_rht over the last axis of x (CUDA tensor or array-like) -> float64 CUDA tensor."""
    import torch

    from . import _lib
    from .quantizers import stream_handle
    if chunk < 16 or chunk & (chunk - 1) or chunk % 16:        # rht.py:133-135
        raise ValueError("rotation chunk must be a power of two and a multiple of 16")
    if chunk > 2048:
        raise ValueError("this build rotates chunks of at most 2048 elements")
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x))
    if x.dtype not in (torch.bfloat16, torch.float32, torch.float64):
        x = x.to(torch.float64)
    x = x.cuda().contiguous() if not x.is_cuda else x.contiguous()
    if x.dim() == 0 or x.shape[-1] % chunk:                    # rht.py:136-140
        last = x.shape[-1] if x.dim() else 0
        raise ValueError(f"rotation requires the last dimension ({last}) to be a multiple of {chunk}")
    out = torch.empty(x.shape, dtype=torch.float64, device=x.device)
    dt = {torch.bfloat16: _lib.Q2_BF16, torch.float32: _lib.Q2_F32, torch.float64: _lib.Q2_F64}[x.dtype]
    sv = lambda v: None if v is None else torch.as_tensor(v, dtype=torch.float64, device=x.device)  # noqa: E731
    pre_t, post_t = sv(pre), sv(post)
    rc = _lib.lib().q2_rht(x.data_ptr() if x.numel() else None, dt, x.numel(), chunk,
                           None if pre_t is None else pre_t.data_ptr(), None if post_t is None else post_t.data_ptr(),
                           scale, out.data_ptr() if x.numel() else None, stream_handle())
    _lib.check(rc, "q2_rht")
    for t in (pre_t, post_t):
        if t is not None:
            t.record_stream(torch.cuda.current_stream(x.device))
    return out


def hadamard_128(x):
    """Orthonormal Hadamard of length-128 vectors (rht.py:121-130), literal float64 on the GPU."""
    if not hasattr(x, "shape"):
        x = np.asarray(x, dtype=np.float64)
    last = x.shape[-1] if len(x.shape) else 0
    if last != CHUNK:
        raise ValueError(f"hadamard_128 requires length {CHUNK}, got {last}")
    return _rotation_call(x, CHUNK, None, None, CHUNK ** -0.5)


def rht_apply(x, seed: int, rotation_id: int = 0, chunk: int = CHUNK):
    """Seeded sign flip, then the normalized Hadamard, per chunk of the last axis
    (rht.py:144-155); float64 CUDA tensor equal to the reference bit for bit."""
    signs = prng_signs(seed, derive_stream(DOMAIN_SIGNS, rotation_id), chunk)
    return _rotation_call(x, chunk, signs, None, chunk ** -0.5)


def rht_inverse(y, seed: int, rotation_id: int = 0, chunk: int = CHUNK):
    """Exact inverse of rht_apply: Hadamard, then undo the sign flip (rht.py:158-163)."""
    signs = prng_signs(seed, derive_stream(DOMAIN_SIGNS, rotation_id), chunk)
    return _rotation_call(y, chunk, None, signs, chunk ** -0.5)


def sr_stream(tensor_id: int) -> int:
    """Stream of the scale rounding draws of one tensor (ms_eden.py:150)."""
    return derive_stream(DOMAIN_SCALE_SR, tensor_id)
