"""CPU-side checks of the C ABI: the in-tree library loads, exports exactly the
entry points include/qjl_b200.h declares, and rejects bad arguments with the
documented status codes before touching the GPU."""

import ctypes
import os
import re

import pytest

from paper_2406_03482_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "qjl_b200.h")).read()
    return set(re.findall(r"^QJL_API\s+[\w\s\*]+?\b(qjl_\w+)\s*\(", src, flags=re.M))


def test_header_and_binding_agree():
    syms = header_symbols()
    assert len(syms) >= 14
    assert syms == set(_lib.SIGNATURES), syms ^ set(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.qjl_abi_version() == 1
    assert lib.qjl_status_string(-1) == b"invalid argument"


def test_argument_errors_without_gpu():
    lib = _lib.load()
    # empty prompt (kvcache.py:111-112) -> QJL_ERR_ARG, no CUDA call made
    rc = lib.qjl_detect_outliers(None, 0, 1, 0, 128, 0, 1, None, None, None)
    assert rc == _lib.QJL_ERR_ARG
    with pytest.raises(ValueError):
        _lib.check(rc, "detect_outliers")
    # outlier rate check (kvcache.py:219-226): m_out/h < m_in/(d-h)
    rc = lib.qjl_build_sketch(ctypes.c_void_p(8), ctypes.c_void_p(8), 256, 8, 128, 8,
                              ctypes.c_void_p(8), 1, 2, ctypes.c_void_p(8), None)
    assert rc == _lib.QJL_ERR_ARG
    assert b"outlier bit rate" in lib.qjl_last_error()
    # unsupported sketch width (not a multiple of 32)
    kc = _lib.KeyCacheDesc(8, None, 8, None, 16, 1, 128, 100, 0)
    sd = _lib.SketchDesc(8, 2, 0, 0)
    rc = lib.qjl_quantize_keys(ctypes.c_void_p(8), 2, 1, 128, ctypes.byref(sd), None, 0,
                               ctypes.byref(kc), 0, None)
    assert rc == _lib.QJL_ERR_UNSUPPORTED
    # temperature must be positive (kvcache.py:335-336)
    assert lib.qjl_softmax_f64(ctypes.c_void_p(8), 1, 1, 0.0, ctypes.c_void_p(8), None) == _lib.QJL_ERR_ARG
