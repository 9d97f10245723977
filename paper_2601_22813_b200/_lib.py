"""ctypes binding of libquartet2.so (the C ABI declared in include/quartet2.h).

The library is built in-tree by ``build.sh`` / ``__graft_entry__.build()``.
There is no fallback: if the library is missing, importing the compute entry
points raises ImportError.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("Q2_LIB_OVERRIDE") or os.path.join(_HERE, "libquartet2.so")   # override: A/B timing tools only

Q2_OK, Q2_EINVAL, Q2_ECUDA = 0, 1, 2
Q2_BF16, Q2_F32, Q2_F64 = 0, 1, 2
Q2_SRC_ROWS, Q2_SRC_COLS, Q2_SRC_TAPE_COLS = 0, 1, 2
Q2_MSED_EXACT, Q2_MSED_POW2, Q2_MSED_POSTHOC = 0, 1, 2
Q2_ACC_STORE, Q2_ACC_ADD, Q2_ACC_RED, Q2_ACC_MULTIMEM = 0, 1, 2, 3
Q2_ERR_NONFINITE, Q2_ERR_SCALE448, Q2_ERR_NAN_SCALE, Q2_ERR_E8M3_OVF, Q2_ERR_SR_CLIP = 1, 2, 4, 8, 16

# Every symbol include/quartet2.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "q2_sf_bytes", "q2_version", "q2_amax", "q2_quant_fwd_ws_bytes", "q2_quant_fwd",
    "q2_msed_ws_bytes", "q2_msed_quant", "q2_posthoc_pass1", "q2_posthoc_pass2",
    "q2_msed_dual_posthoc", "q2_msed_dual", "q2_msed_dual_ws_bytes", "q2_msed_stats", "q2_set_msed_engine", "q2_gemm_tn", "q2_dequant", "q2_unpack", "q2_pack",
    "q2_quant_sr_ws_bytes", "q2_quant_sr", "q2_rht_sr_quant", "q2_quant_square_block", "q2_sr_quant_src", "q2_quant_fwd_amax",
    "q2_rht", "q2_formats", "q2_eden_factors", "q2_launch_count",
)


class Q2Tensor(ctypes.Structure):
    """q2_nvfp4"""

    _fields_ = [("codes", ctypes.c_void_p), ("sf", ctypes.c_void_p), ("scale32", ctypes.c_void_p),
                ("R", ctypes.c_int64), ("K", ctypes.c_int64)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_U64 = ctypes.c_uint64
_TP = ctypes.POINTER(Q2Tensor)
_U32x4 = ctypes.c_uint32 * 4

_SIGS = {
    "q2_sf_bytes": (ctypes.c_size_t, [_I64, _I64]),
    "q2_version": (ctypes.c_char_p, []),
    "q2_amax": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, _P]),
    "q2_quant_fwd_ws_bytes": (ctypes.c_size_t, [_I64, _I64]),
    "q2_quant_fwd": (_I, [_P, _I, _I64, _I64, _I64, _I, _D, _D, _D, _TP, _P, _P, _P]),
    "q2_quant_fwd_amax": (_I, [_P, _I, _I64, _I64, _I64, _I, _D, _D, _D, _P, _TP, _P, _P, _P]),
    "q2_msed_ws_bytes": (ctypes.c_size_t, [_I64, _I64]),
    "q2_msed_quant": (_I, [_P, _I, _TP, _I, _I64, _I64, _I64, _U32x4, _D, _D, _U64, _U64, _I, _TP, _P, _P, _P]),
    "q2_posthoc_pass1": (_I, [_P, _I, _TP, _I, _I64, _I64, _I64, _U32x4, _D, _D, _P, _P, _P, _P, _P, _P]),
    "q2_posthoc_pass2": (_I, [_P, _P, _P, _I64, _I64, _U64, _U64, _TP, _P, _P]),
    "q2_msed_dual_posthoc": (_I, [_P, _I64, _I64, _I64, _U32x4, _U32x4, _D, _D, _U64, _U64, _U64, _TP, _TP, _P, _P,
                                  _P, _P]),
    "q2_msed_dual": (_I, [_P, _I64, _I64, _I64, _U32x4, _U32x4, _D, _D, _U64, _U64, _U64, _I, _TP, _TP, _P, _P, _P]),
    "q2_msed_dual_ws_bytes": (ctypes.c_size_t, [_I64, _I64]),
    "q2_msed_stats": (_I, [_P, _I]),
    "q2_set_msed_engine": (_I, [_I]),
    "q2_gemm_tn": (_I, [_TP, _TP, _P, _I, _I64, _I, _P]),
    "q2_quant_sr_ws_bytes": (ctypes.c_size_t, []),
    "q2_sr_quant_src": (_I, [_P, _I, _TP, _I, _I64, _I64, _I64, _I, _U32x4, _I, _D, _D, _D, _D, _D, _U64, _U64, _U64,
                             _TP, _P, _P, _P]),
    "q2_quant_square_block": (_I, [_P, _I, _I64, _I64, _I, _TP, _TP, _P, _P, _P, _P]),
    "q2_quant_sr": (_I, [_P, _I, _I64, _I64, _I64, _I, _D, _D, _D, _D, _U64, _U64, _U64, _TP, _P, _P, _P]),
    "q2_rht_sr_quant": (_I, [_P, _I, _TP, _I, _I64, _I64, _I64, _U32x4, _D, _D, _D, _D, _U64, _U64, _TP, _P, _P,
                             _P]),
    "q2_dequant": (_I, [_TP, _P, _P]),
    "q2_unpack": (_I, [_TP, _P, _P, _P]),
    "q2_pack": (_I, [_P, _P, _TP, _P]),
    "q2_rht": (_I, [_P, _I, _I64, _I, _P, _P, _D, _P, _P]),
    "q2_formats": (_I, [_I, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "q2_eden_factors": (_I, [_P, _P, _I64, _P, _P]),
    "q2_launch_count": (ctypes.c_ulonglong, [_I]),
}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run ./build.sh (or __graft_entry__.build()); "
                          "there is no CPU fallback for the Quartet II kernels")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_LIB = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


def check(rc: int, what: str) -> None:
    if rc == Q2_EINVAL:
        raise ValueError(f"{what}: invalid arguments (shape, alignment or dtype)")
    if rc != Q2_OK:
        raise RuntimeError(f"{what}: CUDA launch failed (rc={rc})")
