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


@lru_cache(maxsize=1024)
def sign_mask(seed: int, rotation_id: int) -> tuple:
    """The rotation's 128 signs (rht.py:99-106) as four u32 words, bit i = sign i is -1.

    ``u < 0.5`` is ``(bits >> 11) * 2**-53 < 0.5``, i.e. bit 63 of ``_bits`` is
    clear; the seed/stream prefix of ``_bits`` is shared, so the 128 index mixes
    run as one uint64 vector (wrap-around arithmetic, same integers)."""
    stream = derive_stream(DOMAIN_SIGNS, rotation_id)
    z0 = _mix64(_mix64((seed + _GOLDEN) & _M64) ^ ((stream + _GOLDEN) & _M64))
    z = np.uint64(z0) ^ (np.arange(CHUNK, dtype=np.uint64) + np.uint64(_GOLDEN))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    neg = ((z ^ (z >> np.uint64(31))) >> np.uint64(63)).astype(np.uint64)
    words = (neg.reshape(4, 32) << np.arange(32, dtype=np.uint64)).sum(axis=1)
    return tuple(int(w) for w in words)


def sr_stream(tensor_id: int) -> int:
    """Stream of the scale rounding draws of one tensor (ms_eden.py:150)."""
    return derive_stream(DOMAIN_SCALE_SR, tensor_id)
