"""QJLC file cases shared by the CPU (oracle) and GPU (device exporter) tests.

Each case rebuilds, from the golden inputs, everything the reference used when
it wrote the golden file in tests/golden/make_golden.py: keys, values, outlier
profile, sketches (drawn by the pinned host sketch module), seed, widths.
"""

from __future__ import annotations

import numpy as np

from oracle import qjl_oracle as O
from paper_2406_03482_b200 import sketch as SK


def _sketches(seed, d, h, m_in, m_out, orth):
    def build(m, dd, stream):
        if dd == 0 or m == 0:
            return None
        s = SK.generate_gaussian(m, dd, SK.derive_seed(seed, stream))
        return (SK.orthogonalize(s) if orth else s).entries
    return build(m_in, d - h, 0), build(m_out, h, 1)


def case(golden, name: str) -> dict:
    if name == "c2":
        c = dict(keys=golden["q2_keys"], values=golden["dec_values"],
                 channels=tuple(int(x) for x in golden["q2_channels"]), mags=golden["q2_mags"],
                 d=128, h=4, m_in=256, m_out=128, seed=22, orth=True, value_bits=2)
    elif name == "r":
        c = dict(keys=golden["qjlc_r_keys"], values=golden["qjlc_r_values"],
                 channels=tuple(int(x) for x in golden["qjlc_r_channels"]), mags=golden["qjlc_r_mags"],
                 d=32, h=4, m_in=96, m_out=40, seed=44, orth=False, value_bits=3)
    elif name == "h0":
        c = dict(keys=golden["qjlc_h0_keys"], values=golden["qjlc_h0_values"], channels=(),
                 mags=golden["qjlc_h0_mags"], d=64, h=0, m_in=64, m_out=0, seed=55, orth=True,
                 value_bits=8)
    else:
        raise KeyError(name)
    c["S_in"], c["S_out"] = _sketches(c["seed"], c["d"], c["h"], c["m_in"], c["m_out"], c["orth"])
    c["bytes"] = golden[f"qjlc_{name}_bytes"].tobytes()
    return c


def oracle_file(c: dict) -> bytes:
    """The oracle's restatement of write_cache on the case's state."""
    r = O.append_keys(c["S_in"], c["S_out"], c["channels"], c["keys"])
    codes, zero, scale = O.quantize_values(c["values"], c["value_bits"], c["d"], const_dtype=None)
    return O.qjlc_encode(d=c["d"], h=c["h"], m_in=c["m_in"], m_out=c["m_out"],
                         value_bits=c["value_bits"], seed=c["seed"], orthogonalized=c["orth"],
                         channels=c["channels"], magnitudes=c["mags"], bits_in=r["bits_in"],
                         norm_in=r["norm_in"], bits_out=r["bits_out"], norm_out=r["norm_out"],
                         codes=codes, zero=zero[:, 0], scale=scale[:, 0])
