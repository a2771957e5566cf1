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
    assert lib.qjl_abi_version() == 3
    assert lib.qjl_status_string(-1) == b"invalid argument"


def test_argument_errors_without_gpu():
    lib = _lib.load()
    # empty prompt (kvcache.py:111-112) -> QJL_ERR_ARG, no CUDA call made
    rc = lib.qjl_detect_outliers(None, 0, 1, 0, 128, 0, 1, None, None, None, 0, None)
    assert rc == _lib.QJL_ERR_ARG
    with pytest.raises(ValueError):
        _lib.check(rc, "detect_outliers")
    # outlier rate check (kvcache.py:219-226): m_out/h < m_in/(d-h)
    rc = lib.qjl_build_sketch(ctypes.c_void_p(8), ctypes.c_void_p(8), 256, 8, 128, 8,
                              ctypes.c_void_p(8), 1, 2, ctypes.c_void_p(8), None)
    assert rc == _lib.QJL_ERR_ARG
    assert b"outlier bit rate" in lib.qjl_last_error()
    # unsupported sketch width (not a multiple of 32)
    kc = _lib.KeyCacheDesc(8, None, 8, None, 16, 1, 128, 100, 0, 0)
    sd = _lib.SketchDesc(8, 2, 0, 0)
    rc = lib.qjl_quantize_keys(ctypes.c_void_p(8), 2, 1, 128, ctypes.byref(sd), None, 0,
                               ctypes.byref(kc), 0, None)
    assert rc == _lib.QJL_ERR_UNSUPPORTED
    # qjl_scores flags (ABI 3): QJL_DECODE_CHAINED only
    kc = _lib.KeyCacheDesc(8, None, 8, None, 16, 1, 128, 256, 0, 0)
    rc = lib.qjl_scores(ctypes.byref(kc), 1, ctypes.c_void_p(8), 2, 1, ctypes.byref(sd), ctypes.c_void_p(8),
                        ctypes.c_void_p(8), 1 << 20, _lib.QJL_DECODE_DETERMINISTIC, None)
    assert rc == _lib.QJL_ERR_ARG
    assert b"flags" in lib.qjl_last_error()
    # temperature must be positive (kvcache.py:335-336)
    assert lib.qjl_softmax_f64(ctypes.c_void_p(8), 1, 1, 0.0, ctypes.c_void_p(8), None) == _lib.QJL_ERR_ARG


def test_tile_record_layout():
    """The canonical tile record (qjl_b200.h): C3 shapes give the 11776-byte record the
    tensor-core decode streams with one bulk copy; key fields come first."""
    lib = _lib.load()
    off = (ctypes.c_int64 * 7)()
    assert lib.qjl_tile_record(128, 256, 64, 1, off) == 11776
    assert list(off) == [0, 4096, 5120, 5376, 5632, 9728, 10752]
    assert lib.qjl_tile_record(128, 256, 64, 0, off) == 5632            # keys only
    assert list(off)[4:] == [-1, -1, -1]
    assert lib.qjl_tile_record(128, 256, 0, 1, off) == 128 * 32 + 256 + 4096 + 2048
    assert off[1] == -1 and off[3] == -1
    assert lib.qjl_tile_record(128, 100, 0, 0, off) == -1               # m % 32 != 0
    assert lib.qjl_tile_record(64, 256, 0, 1, off) == -1                # values need d = 128


def test_layout_rules_without_gpu():
    """P2T values live in tile records; U8 values use the rows layout; tiled key arrays
    must sit at their record offsets -- all rejected before any CUDA call."""
    lib = _lib.load()
    sd = _lib.SketchDesc(8, 2, 0, 0)
    base = 1 << 20
    kc = _lib.KeyCacheDesc(base, base + 4096, base + 5120, base + 5376, 256, 1, 128, 256, 64, 11776)
    vc_rows = _lib.ValueCacheDesc(8, 8, 8, 256, 1, 128, 2, 32, _lib.QJL_VLAYOUT_P2T, 0, 0)
    rc = lib.qjl_decode(ctypes.byref(kc), ctypes.byref(vc_rows), 16, ctypes.c_void_p(8), 2, 4, ctypes.byref(sd),
                        1.0, ctypes.c_void_p(8), None, None, ctypes.c_void_p(8), 1 << 30, 0, None)
    assert rc == _lib.QJL_ERR_ARG and b"tile-major" in lib.qjl_last_error()
    vc_u8 = _lib.ValueCacheDesc(8, 8, 8, 256, 1, 128, 2, 128, _lib.QJL_VLAYOUT_U8, 0, 11776)
    rc = lib.qjl_decode(ctypes.byref(kc), ctypes.byref(vc_u8), 16, ctypes.c_void_p(8), 2, 4, ctypes.byref(sd),
                        1.0, ctypes.c_void_p(8), None, None, ctypes.c_void_p(8), 1 << 30, 0, None)
    assert rc == _lib.QJL_ERR_ARG and b"rows layout" in lib.qjl_last_error()
    bad = _lib.KeyCacheDesc(base, base + 4096, base + 5000, base + 5376, 256, 1, 128, 256, 64, 11776)
    rc = lib.qjl_quantize_keys(ctypes.c_void_p(8), 2, 1, 128, ctypes.byref(sd), ctypes.c_void_p(8), 8,
                               ctypes.byref(bad), 0, None)
    assert rc == _lib.QJL_ERR_ARG and b"record offsets" in lib.qjl_last_error()
    odd = _lib.KeyCacheDesc(base, base + 4096, base + 5120, base + 5376, 200, 1, 128, 256, 64, 11776)
    rc = lib.qjl_quantize_keys(ctypes.c_void_p(8), 2, 1, 128, ctypes.byref(sd), ctypes.c_void_p(8), 8,
                               ctypes.byref(odd), 0, None)
    assert rc == _lib.QJL_ERR_ARG and b"128-row tiles" in lib.qjl_last_error()
