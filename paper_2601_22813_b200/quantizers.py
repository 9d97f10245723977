"""NVFP4 tensors in HBM and the forward quantizers (host mirror of quantizers.py).

Same names, argument meanings and exceptions as the reference
(quantizers.py:83-98, 164-234, 315-323); the work runs in libquartet2.so.
Inputs are CUDA (or host) tensors of dtype bfloat16 / float32 with groups of
16 along the last axis; float64 inputs are accepted when every value is
exactly representable in float32.
"""

from __future__ import annotations

import ctypes
import functools
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

GROUP = 16
E4M3_MAX = 448.0
FP4_ABS_MAX = 6.0
FP8_RTN_MARGIN = 16.0 / 17.0                         # quantizers.py:64
GUARDED_SCALE_CAP = E4M3_MAX * FP8_RTN_MARGIN        # quantizers.py:67

_ERR_MESSAGES = (
    (_lib.Q2_ERR_NONFINITE, ValueError, "input must be finite"),
    (_lib.Q2_ERR_NAN_SCALE, ValueError, "NaN input to encode_fp8_rtn"),
    (_lib.Q2_ERR_SCALE448, ValueError,
     "corrected group scale exceeds 448; the 448/256 headroom should absorb the correction factor"),
    (_lib.Q2_ERR_E8M3_OVF, OverflowError, "round_e8m3_rtn overflow beyond the bf16 carrier range"),
    (_lib.Q2_ERR_SR_CLIP, AssertionError, "non-clipping construction produced quotient above 6; encoder bug"),
)

# "sync": every public call reads its error word and raises like the reference.
# "deferred": errors accumulate in a device word; call check_errors() to raise.
_ERROR_MODE = {"mode": "sync", "words": {}}


def set_error_mode(mode: str) -> None:
    if mode not in ("sync", "deferred"):
        raise ValueError(f"unknown error mode {mode!r}")
    _ERROR_MODE["mode"] = mode


def _err_word(device) -> torch.Tensor:
    if _ERROR_MODE["mode"] == "sync":
        return torch.zeros(1, dtype=torch.int32, device=device)
    words = _ERROR_MODE["words"]
    if device not in words:
        words[device] = torch.zeros(1, dtype=torch.int32, device=device)
    return words[device]


def _raise_bits(bits: int) -> None:
    for bit, exc, msg in _ERR_MESSAGES:
        if bits & bit:
            raise exc(msg)


def _finish(err: torch.Tensor) -> None:
    if _ERROR_MODE["mode"] == "sync":
        _raise_bits(int(err.item()))


def check_errors() -> None:
    """Raise the first pending deferred error (and clear the words)."""
    for w in _ERROR_MODE["words"].values():
        bits = int(w.item())
        w.zero_()
        _raise_bits(bits)


def _cuda_device_of(args, kw):
    for a in list(args) + list(kw.values()):
        if isinstance(a, torch.Tensor):
            if a.is_cuda:
                return a.device
        else:
            d = getattr(a, "device", None)
            if isinstance(d, torch.device) and d.type == "cuda":
                return d
    return None


def api(fn):
    """Public entry point: an NVTX range named after the reference function, and launches
    on the device that owns the inputs (torch.cuda.device guard when it is not current)."""
    name = "q2." + fn.__name__

    @functools.wraps(fn)
    def wrapper(*args, **kw):
        dev = _cuda_device_of(args, kw)
        with torch.cuda.nvtx.range(name):
            if dev is None or dev.index is None or dev.index == torch.cuda.current_device():
                return fn(*args, **kw)
            with torch.cuda.device(dev):
                return fn(*args, **kw)
    return wrapper


def stream_handle(device=None) -> int:
    """The caller's current stream on ``device`` (default: the current device); entry
    points run under ``torch.cuda.device(tensor.device)`` so launches go to the device
    that owns the data."""
    return torch.cuda.current_stream(device).cuda_stream


@dataclass
class NVFP4Tensor:
    """NVFP4 tensor resident in HBM (quantizers.py:83-98).

    codes   uint8 [R, K/2]  two E2M1 codes per byte, low nibble = even element
    sf      uint8 [q2_sf_bytes]  UE4M3 group scales in the tcgen05 atom layout
    scale   float32 [1]  the fp32 tensor scale, on device
    The reference's attribute names (``fp4``, ``scales8``, ``scale32``) are
    available as host views for parity checks.
    """

    codes: torch.Tensor
    sf: torch.Tensor
    scale: torch.Tensor
    shape: tuple
    group_axis: int = -1

    @property
    def R(self) -> int:
        return int(np.prod(self.shape[:-1])) if len(self.shape) > 1 else 1

    @property
    def K(self) -> int:
        return int(self.shape[-1])

    @property
    def device(self):
        return self.codes.device

    def c(self) -> _lib.Q2Tensor:
        return _lib.Q2Tensor(self.codes.data_ptr(), self.sf.data_ptr(), self.scale.data_ptr(), self.R, self.K)

    @classmethod
    def empty(cls, shape, device) -> "NVFP4Tensor":
        shape = tuple(int(s) for s in shape)
        R = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
        K = shape[-1]
        nsf = _lib.lib().q2_sf_bytes(R, K)
        # Scale padding (rows beyond R in the last 256-row block, K groups beyond K in
        # the last 64-block) only feeds masked GEMM outputs; it is zeroed anyway so the
        # buffer's bytes are a function of the input (deterministic serialization,
        # torch.library.opcheck).  Shapes without padding skip the memset.
        padded = R % 256 != 0 or K % 64 != 0
        return cls(torch.empty((R, K // 2), dtype=torch.uint8, device=device),
                   (torch.zeros if padded else torch.empty)(nsf, dtype=torch.uint8, device=device),
                   torch.empty(1, dtype=torch.float32, device=device), shape)

    # ---- reference-layout views (host numpy) ----
    def unpacked(self):
        fp4 = torch.empty((self.R, self.K), dtype=torch.uint8, device=self.device)
        s8 = torch.empty((self.R, self.K // GROUP), dtype=torch.uint8, device=self.device)
        t = self.c()
        _lib.check(_lib.lib().q2_unpack(ctypes.byref(t), fp4.data_ptr(), s8.data_ptr(), stream_handle()), "unpack")
        return fp4, s8

    @property
    def fp4(self) -> np.ndarray:
        return self.unpacked()[0].cpu().numpy().reshape(self.shape)

    @property
    def scales8(self) -> np.ndarray:
        return self.unpacked()[1].cpu().numpy().reshape(*self.shape[:-1], self.K // GROUP)

    @property
    def scale32(self) -> np.float32:
        return np.float32(self.scale.item())

    def to_reference(self):
        """(fp4, scales8, scale32) in the reference's unpacked layout."""
        fp4, s8 = self.unpacked()
        return (fp4.cpu().numpy().reshape(self.shape),
                s8.cpu().numpy().reshape(*self.shape[:-1], self.K // GROUP), self.scale32)

    @classmethod
    def from_reference(cls, fp4, scales8, scale32, device="cuda") -> "NVFP4Tensor":
        fp4 = torch.from_numpy(np.array(fp4, dtype=np.uint8, order="C")).to(device)
        s8 = torch.from_numpy(np.array(scales8, dtype=np.uint8, order="C")).to(device)
        t = cls.empty(tuple(fp4.shape), device)
        t.scale.fill_(float(np.float32(scale32)))
        tc = t.c()
        _lib.check(_lib.lib().q2_pack(fp4.data_ptr(), s8.data_ptr(), ctypes.byref(tc), stream_handle()), "pack")
        return t


def as_device_matrix(x, what: str = "input"):
    """(2-D contiguous CUDA tensor of bf16/fp32, original shape, dtype code)."""
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    if x.dtype == torch.float64:
        x32 = x.to(torch.float32)
        if not torch.equal(x32.to(torch.float64), x):
            raise TypeError(f"{what}: float64 values must be exactly representable in float32")
        x = x32
    if x.dtype not in (torch.bfloat16, torch.float32):
        raise TypeError(f"{what}: dtype {x.dtype} not supported (bfloat16 / float32)")
    if not x.is_cuda:
        x = x.cuda()
    shape = tuple(x.shape)
    if len(shape) == 0:
        raise ValueError(f"{what}: expected at least one dimension")
    x2 = x.reshape(-1, shape[-1]) if len(shape) != 2 else x
    if not x2.is_contiguous():
        x2 = x2.contiguous()
    if x2.data_ptr() % 32:                  # the vector loads need 32-byte aligned rows (offset views)
        x2 = x2.clone()
    return x2, shape, (_lib.Q2_BF16 if x.dtype == torch.bfloat16 else _lib.Q2_F32)


def _check_group_dim(shape) -> None:
    if shape[-1] % GROUP != 0:
        raise ValueError(f"last dimension must be a multiple of {GROUP}")  # quantizers.py:116-117


def _quant_fwd(x, caps, scale_div, err=None, amax=None) -> NVFP4Tensor:
    x2, shape, dt = as_device_matrix(x)
    _check_group_dim(shape)
    out = NVFP4Tensor.empty(shape, x2.device)
    own = err is None
    if own:
        err = _err_word(x2.device)
    L = _lib.lib()
    ws = torch.empty(L.q2_quant_fwd_ws_bytes(x2.shape[0], x2.shape[1]), dtype=torch.uint8, device=x2.device)
    t = out.c()
    c1 = float(caps[1]) if len(caps) > 1 else 0.0
    args = (x2.data_ptr(), dt, x2.shape[0], x2.shape[1], x2.shape[1], len(caps), float(caps[0]), c1, float(scale_div))
    if amax is None:
        rc = L.q2_quant_fwd(*args, ctypes.byref(t), ws.data_ptr(), err.data_ptr(), stream_handle())
    else:
        if not (isinstance(amax, torch.Tensor) and amax.is_cuda and amax.numel() == 1 and amax.dtype == torch.float32):
            raise TypeError("amax must be a one-element float32 CUDA tensor holding max|x|")
        rc = L.q2_quant_fwd_amax(*args, amax.data_ptr(), ctypes.byref(t), ws.data_ptr(), err.data_ptr(),
                                 stream_handle())
    _lib.check(rc, "quant_fwd")
    if own:
        _finish(err)
    return out


@api
def absmax(x) -> torch.Tensor:
    """max|x| as a one-element float32 CUDA tensor (the value a fused producer would supply)."""
    x2, _, dt = as_device_matrix(x)
    out = torch.zeros(1, dtype=torch.float32, device=x2.device)
    err = _err_word(x2.device)
    _lib.check(_lib.lib().q2_amax(x2.data_ptr(), dt, x2.shape[0], x2.shape[1], x2.shape[1], out.data_ptr(),
                                  err.data_ptr(), stream_handle()), "amax")
    _finish(err)
    return out


@api
def quantize_rtn_46(x, caps=(6.0, 4.0), scale_cap: float = GUARDED_SCALE_CAP, _err=None, amax=None) -> NVFP4Tensor:
    """Forward-pass RTN with per-group Four-over-Six ceiling choice (quantizers.py:206-234).

    ``amax``: optional max|x| from the producer of x (one-element float32 CUDA
    tensor); skips the absmax pass."""
    caps = tuple(float(c) for c in caps)
    if len(caps) not in (1, 2):
        raise ValueError("caps must hold one or two grid ceilings")
    return _quant_fwd(x, caps, caps[0] * scale_cap, _err, amax)


@api
def quantize_rtn(x, s=FP4_ABS_MAX, _err=None) -> NVFP4Tensor:
    """Deterministic NVFP4 quantization with grid ceiling s and cap 256 (quantizers.py:164-181)."""
    s = float(getattr(s, "s", s))
    if not 0.0 < s <= FP4_ABS_MAX:
        raise ValueError(f"grid max must be in (0, 6], got {s}")
    return _quant_fwd(x, (s,), s * 256.0, _err)


@api
def dequantize(t: NVFP4Tensor) -> torch.Tensor:
    """Reconstruct the real-valued tensor, float64 on device (quantizers.py:315-323)."""
    if hasattr(t, "rows") and isinstance(t.rows, NVFP4Tensor):     # SquareBlockTensor: expanded block scales
        t = t.rows
    if not isinstance(t, NVFP4Tensor):
        raise TypeError(f"cannot dequantize {type(t).__name__}")
    out = torch.empty((t.R, t.K), dtype=torch.float64, device=t.device)
    tc = t.c()
    _lib.check(_lib.lib().q2_dequant(ctypes.byref(tc), out.data_ptr(), stream_handle()), "dequant")
    return out.reshape(t.shape)


# ---------------------------------------------------------------- container ---
_MAGIC, _VERSION = b"NV4T", 1


def serialize_nvfp4(t: NVFP4Tensor) -> bytes:
    """The NV4T binary container (quantizers.py:326-349): magic, u16 version,
    u8 ndim, u8 group axis (0xFF = last), ndim x u32 dims, codes packed two per
    byte (low nibble first -- the device layout as is), E4M3 scale bytes
    row-major, fp32 tensor scale, all little-endian."""
    if not isinstance(t, NVFP4Tensor):
        raise TypeError(f"cannot serialize {type(t).__name__}")
    _, s8 = t.unpacked()
    head = struct.pack(f"<4sHBB{len(t.shape)}I", _MAGIC, _VERSION, len(t.shape), 0xFF, *t.shape)
    return (head + t.codes.contiguous().cpu().numpy().tobytes() + s8.cpu().numpy().tobytes()
            + struct.pack("<f", float(t.scale32)))


def deserialize_nvfp4(buf: bytes, device="cuda") -> NVFP4Tensor:
    """Inverse of serialize_nvfp4 (quantizers.py:352-372), onto the device."""
    magic, version, ndim, _axis = struct.unpack_from("<4sHBB", buf, 0)
    if magic != _MAGIC:
        raise ValueError("bad magic in NVFP4 container")
    if version != _VERSION:
        raise ValueError(f"unsupported NVFP4 container version {version}")
    dims = struct.unpack_from(f"<{ndim}I", buf, 8)
    n = int(np.prod(dims))
    off = 8 + 4 * ndim
    packed = np.frombuffer(buf, dtype=np.uint8, count=n // 2, offset=off)
    codes = np.empty(n, dtype=np.uint8)
    codes[0::2] = packed & 0xF
    codes[1::2] = packed >> 4
    off += n // 2
    s8 = np.frombuffer(buf, dtype=np.uint8, count=n // GROUP, offset=off)
    off += n // GROUP
    (scale32,) = struct.unpack_from("<f", buf, off)
    return NVFP4Tensor.from_reference(codes.reshape(dims), s8.reshape(*dims[:-1], dims[-1] // GROUP),
                                      np.float32(scale32), device)
