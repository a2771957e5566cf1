"""QJLC cache files (kvcache.py:368-520), CPU side: the oracle's restatement of
write_cache/read_cache is pinned byte for byte against files written by the real
reference (tests/golden), and the file header/record arithmetic used by the device
exporter (paper_2406_03482_b200/qjlc.py) agrees with it."""

import struct

import numpy as np
import pytest

from oracle import qjl_oracle as O
from paper_2406_03482_b200 import qjlc as Q
from tests._qjlc import case, oracle_file

CASES = ["c2", "r", "h0"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_writer_reproduces_reference_file(golden, name):
    c = case(golden, name)
    assert oracle_file(c) == c["bytes"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_reader_round_trip(golden, name):
    c = case(golden, name)
    f = O.qjlc_decode(c["bytes"])
    assert (f["d"], f["h"], f["m_in"], f["m_out"], f["seed"], f["orthogonalized"]) == \
        (c["d"], c["h"], c["m_in"], c["m_out"], c["seed"], c["orth"])
    assert tuple(f["channels"].tolist()) == c["channels"]
    again = O.qjlc_encode(d=f["d"], h=f["h"], m_in=f["m_in"], m_out=f["m_out"],
                          value_bits=f["value_bits"], seed=f["seed"],
                          orthogonalized=f["orthogonalized"], channels=f["channels"],
                          magnitudes=f["magnitudes"], bits_in=f["bits_in"], norm_in=f["norm_in"],
                          bits_out=f["bits_out"], norm_out=f["norm_out"], codes=f["codes"],
                          zero=f["zero"], scale=f["scale"])
    assert again == c["bytes"]


def test_header_and_record_sizes_match_reference_layout(golden):
    for name in CASES:
        c = case(golden, name)
        hdr = Q.parse_header(c["bytes"])
        R = Q.record_bytes(c["d"], c["m_in"], c["m_out"])
        assert R == O.qjlc_record_bytes(c["d"], c["m_in"], c["m_out"])
        assert len(c["bytes"]) == Q.HEADER_BYTES + 4 * c["h"] + 8 * c["d"] + hdr.n * R
        assert Q.pack_header(hdr) == c["bytes"][:Q.HEADER_BYTES]


def test_header_errors_are_file_format_errors(golden):
    blob = golden["qjlc_r_bytes"].tobytes()
    with pytest.raises(Q.FileFormatError):
        Q.parse_header(blob[:10])
    with pytest.raises(Q.FileFormatError):
        Q.parse_header(b"XJLC" + blob[4:])
    bad_version = bytearray(blob)
    struct.pack_into("<H", bad_version, 4, 2)
    with pytest.raises(Q.FileFormatError):
        Q.parse_header(bytes(bad_version))
    with pytest.raises(Q.FileFormatError):
        Q.parse_header(blob + b"\0")
    with pytest.raises(ValueError):
        O.qjlc_decode(blob[:-1])


@pytest.mark.parametrize("name", CASES)
def test_golden_cases_have_no_sign_ties(golden, name):
    """Byte equality of device-written files is only a fair test when no projection
    sits within summation-order noise of 0 (bits exact except |Sk| < 1e-6)."""
    c = case(golden, name)
    r = O.append_keys(c["S_in"], c["S_out"], c["channels"], c["keys"])
    for p in (r["proj_in"], r["proj_out"]):
        if p.size:
            assert np.abs(p).min() > 1e-6
