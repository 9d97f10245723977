"""Seeded input families for parity tests (SURVEY.md §8(d) parity families)."""

import numpy as np

FAMILIES = ("normal", "lognormal_rows", "coarse_grid", "zero_rows", "outliers", "tiny_chunk", "t2", "tie_grid",
            "signed_zeros")


def make(family: str, shape, seed: int = 0, bf16: bool = True) -> np.ndarray:
    """float32 array (rounded to bf16 precision when bf16=True)."""
    rng = np.random.default_rng(seed)
    r, k = shape
    x = rng.standard_normal((r, k))
    if family == "lognormal_rows":
        x *= np.exp(rng.normal(0.0, 3.0, (r, 1)))
    elif family == "coarse_grid":
        x = np.round(x * 4.0) / 4.0
    elif family == "zero_rows":
        x[::3] = 0.0
        x[:, : min(128, k)] = 0.0 if k >= 256 else x[:, : min(128, k)]
    elif family == "outliers":
        for c in range(0, k, 128):
            rows = rng.integers(0, r, size=2)
            x[rows, c + rng.integers(0, min(128, k - c))] = 1e3
    elif family == "tiny_chunk":
        x[:, :128] *= 1e-7
    elif family == "t2":
        x = rng.standard_t(2.0, (r, k))
    elif family == "tie_grid":
        # absmax 5.25 = 21 * 2^-2 makes scale32 a few-bit number (17 * 2^-13 for
        # the 4/6 quantizer), so values on a 2^-6 grid land exactly on E2M1
        # rounding thresholds and E4M3 midpoints
        x = np.clip(np.round(x * 64.0) / 64.0, -5.25, 5.25)
        x.flat[0] = 5.25
    elif family == "signed_zeros":
        # 60% exact zeros with random signs (-0 included) on a coarse grid: rotated values
        # that cancel to exactly 0 are common, and the sign of such a zero in the
        # reference's butterflies depends on input 0 of the chunk (+0 unless it is -0)
        x = np.round(x * 2.0) / 2.0
        zero = rng.random((r, k)) < 0.6
        x = np.where(zero, np.where(rng.random((r, k)) < 0.5, -0.0, 0.0), x)
        x[::5, ::128] = -0.0
    elif family != "normal":
        raise ValueError(family)
    x = x.astype(np.float32)
    if bf16:
        x = to_bf16(x)
    return x


def to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 to bfloat16 (RNE) and return it as float32."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return b.astype(np.uint32).view(np.float32)
