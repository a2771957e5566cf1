"""ctypes binding of the C ABI (include/qjl_b200.h).

The shared library is built in-tree (`paper_2406_03482_b200/libqjl_b200.so`,
see `__graft_entry__.build`).  There is no CPU fallback: if the library is
missing or no CUDA device is present, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QJL_LIB") or os.path.join(_HERE, "libqjl_b200.so")

QJL_OK, QJL_ERR_ARG, QJL_ERR_UNSUPPORTED, QJL_ERR_CUDA, QJL_ERR_WORKSPACE, QJL_ERR_EMPTY = (
    0, -1, -2, -3, -4, -5)
QJL_F32, QJL_F16, QJL_BF16, QJL_F64 = 0, 1, 2, 3
QJL_VLAYOUT_U8, QJL_VLAYOUT_P2T = 0, 2
QJL_DECODE_CHAINED, QJL_DECODE_DETERMINISTIC = 1, 2
(QJL_REC_BITS_IN, QJL_REC_BITS_OUT, QJL_REC_NORM_IN, QJL_REC_NORM_OUT, QJL_REC_CODES, QJL_REC_ZERO,
 QJL_REC_SCALE) = range(7)

c_i32, c_i64, c_sz, c_vp, c_dbl, c_flt = (ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t,
                                          ctypes.c_void_p, ctypes.c_double, ctypes.c_float)


class KeyCacheDesc(ctypes.Structure):
    _fields_ = [("bits_in", c_vp), ("bits_out", c_vp), ("norm_in", c_vp), ("norm_out", c_vp),
                ("capacity", c_i64), ("units", c_i32), ("d", c_i32), ("m_in", c_i32),
                ("m_out", c_i32), ("tile_stride", c_i64)]


class ValueCacheDesc(ctypes.Structure):
    _fields_ = [("codes", c_vp), ("zero", c_vp), ("scale", c_vp), ("capacity", c_i64),
                ("units", c_i32), ("d", c_i32), ("bits", c_i32), ("group", c_i32),
                ("layout", c_i32), ("pad_", c_i32), ("tile_stride", c_i64)]


class SketchDesc(ctypes.Structure):
    _fields_ = [("s_full", c_vp), ("dtype", c_i32), ("pad_", c_i32), ("unit_stride", c_i64)]


P = ctypes.POINTER
# name -> (restype, argtypes); exactly the functions declared in include/qjl_b200.h
SIGNATURES = {
    "qjl_abi_version": (c_i32, []),
    "qjl_status_string": (ctypes.c_char_p, [c_i32]),
    "qjl_last_error": (ctypes.c_char_p, []),
    "qjl_device_info": (c_i32, [P(c_i32), P(c_i32), P(c_i32)]),
    "qjl_detect_outliers": (c_i32, [c_vp, c_i32, c_i32, c_i64, c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_sz,
                                    c_vp]),
    "qjl_detect_workspace": (c_sz, [c_i32, c_i64, c_i32]),
    "qjl_build_sketch": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "qjl_prefill_profile": (c_i32, [c_vp, c_i32, c_i32, c_i64, c_i32, c_i64, c_i32, c_vp, c_vp, c_i32,
                                    c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "qjl_quantize_keys": (c_i32, [c_vp, c_i32, c_i64, c_i64, P(SketchDesc), c_vp, c_i32,
                                  P(KeyCacheDesc), c_i64, c_vp]),
    "qjl_sketch_query": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, P(SketchDesc), c_i32, c_i32, c_vp, c_vp]),
    "qjl_scores_workspace": (c_sz, [c_i32, c_i32, c_i32]),
    "qjl_scores": (c_i32, [P(KeyCacheDesc), c_i64, c_vp, c_i32, c_i32, P(SketchDesc), c_vp, c_vp,
                           c_sz, ctypes.c_uint, c_vp]),
    "qjl_sign_dot_batch": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_vp, c_i32, c_vp, c_vp]),
    "qjl_softmax_f64": (c_i32, [c_vp, c_i64, c_i64, c_dbl, c_vp, c_vp]),
    "qjl_decode_workspace": (c_sz, [P(KeyCacheDesc), P(ValueCacheDesc), c_i64, c_i32]),
    "qjl_decode": (c_i32, [P(KeyCacheDesc), P(ValueCacheDesc), c_i64, c_vp, c_i32, c_i32,
                           P(SketchDesc), c_flt, c_vp, c_vp, c_vp, c_vp, c_sz, ctypes.c_uint, c_vp]),
    "qjl_decode_step": (c_i32, [P(KeyCacheDesc), P(ValueCacheDesc), c_i64, c_vp, c_i32, c_i32, P(SketchDesc),
                                c_vp, c_i32, c_vp, c_vp, c_flt, c_vp, c_vp, c_vp, c_vp, c_sz, ctypes.c_uint,
                                c_vp]),
    "qjl_bench_decode_kernel": (c_i32, [P(KeyCacheDesc), P(ValueCacheDesc), c_i64, c_vp, c_i32, c_i32,
                                        P(SketchDesc), c_flt, c_vp, c_vp, c_vp, c_sz, ctypes.c_uint, c_i32,
                                        P(c_flt), c_vp]),
    "qjl_tile_record": (c_i64, [c_i32, c_i32, c_i32, c_i32, P(c_i64)]),
    "qjl_tensor_core_path": (c_i32, [P(KeyCacheDesc), P(ValueCacheDesc), c_i32]),
    "qjl_timing_enable": (c_i32, [c_i32]),
    "qjl_timing_read": (c_i32, [P(c_dbl), P(c_i32), c_i32]),
    "qjl_quantize_values": (c_i32, [c_vp, c_i32, c_i64, c_i64, P(ValueCacheDesc), c_i64, c_vp]),
    "qjl_orthogonalize": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "qjl_qjlc_record_bytes": (c_i64, [c_i32, c_i32, c_i32]),
    "qjl_qjlc_export": (c_i32, [P(KeyCacheDesc), P(ValueCacheDesc), c_i32, c_i32, c_i64, c_i64, c_vp,
                                c_i64, c_vp]),
    "qjl_qjlc_import": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_i32, P(KeyCacheDesc), P(ValueCacheDesc),
                                c_i64, c_vp]),
}

_lib = None


class QJLError(RuntimeError):
    """CUDA-side failure of a library call."""


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) the in-tree CUDA library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the QJL device path)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    if lib.qjl_abi_version() != 3:
        raise ImportError("qjl_b200 ABI version mismatch")
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    """Map a C status to the reference's exception types (ValueError for
    argument/shape errors, RuntimeError for CUDA failures)."""
    if status == QJL_OK:
        return
    msg = (_lib.qjl_last_error() or b"").decode() or _lib.qjl_status_string(status).decode()
    if status in (QJL_ERR_ARG, QJL_ERR_EMPTY, QJL_ERR_WORKSPACE):
        raise ValueError(f"{what}: {msg}")
    if status == QJL_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise QJLError(f"{what}: {msg}")
