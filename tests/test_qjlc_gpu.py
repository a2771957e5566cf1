"""QJLC cache files on the B200: the device record
exporter/importer (qjl_qjlc_export / qjl_qjlc_import) against files written by
the real reference (tests/golden), the oracle's restatement, and round trips at
full C3 size."""

import os

import numpy as np
import pytest
import torch

import paper_2406_03482_b200 as qjl
from oracle import qjl_oracle as O
from paper_2406_03482_b200 import qjlc as Q
from paper_2406_03482_b200.device import DeviceKeyCache
from tests._qjlc import case

pytestmark = pytest.mark.gpu

CASES = ["c2", "r", "h0"]


def _state(c):
    prof = qjl.OutlierProfile(channels=c["channels"], d=c["d"], channel_magnitudes=c["mags"])
    st = qjl.KeyCacheState.create(prof, m_in=c["m_in"], m_out=c["m_out"] if c["h"] else None,
                                  seed=c["seed"], orthogonalize_sketches=c["orth"])
    st.extend(c["keys"])
    toks = [qjl.quantize_value(v, c["value_bits"]) for v in c["values"]]
    return st, toks


@pytest.mark.parametrize("name", CASES)
def test_write_cache_is_byte_identical_to_reference(cuda, golden, tmp_path, name):
    c = case(golden, name)
    st, toks = _state(c)
    p = tmp_path / f"{name}.qjlc"
    qjl.write_cache(p, st, toks)
    got = p.read_bytes()
    assert len(got) == len(c["bytes"])
    assert got == c["bytes"], np.flatnonzero(np.frombuffer(got, np.uint8) != golden[f"qjlc_{name}_bytes"])[:16]


@pytest.mark.parametrize("name", ["r", "h0"])
def test_read_cache_of_reference_file(cuda, golden, tmp_path, name):
    c = case(golden, name)
    p = tmp_path / f"{name}.qjlc"
    p.write_bytes(c["bytes"])
    st, toks, hdr = qjl.read_cache(p)
    assert (hdr.d, hdr.h, hdr.m_in, hdr.m_out, hdr.n, hdr.seed, hdr.orthogonalized) == \
        (c["d"], c["h"], c["m_in"], c["m_out"], len(c["keys"]), c["seed"], c["orth"])
    assert st.n == hdr.n and st.profile.channels == c["channels"]
    f = O.qjlc_decode(c["bytes"])
    for i, (ki, ko) in enumerate(st.entries):       # device rows == file records
        wi = np.ascontiguousarray(ki.bits, "<u8").view(np.uint8) if c["m_in"] else np.zeros(0, np.uint8)
        assert np.array_equal(wi, f["bits_in"][i])
        assert ki.norm == f["norm_in"][i] and ko.norm == f["norm_out"][i]
        if c["m_out"]:
            assert np.array_equal(np.ascontiguousarray(ko.bits, "<u8").view(np.uint8), f["bits_out"][i])
    for i, t in enumerate(toks):
        assert np.array_equal(t.codes, f["codes"][i]) and t.zero == f["zero"][i] and t.scale == f["scale"][i]
    for i, q in enumerate(golden[f"qjlc_{name}_queries"]):
        lg = st.estimate_logits(q)
        ref = golden[f"qjlc_{name}_logits"][i]
        assert np.all(np.abs(lg - ref) <= 1e-3 * np.abs(ref) + 1e-4), np.abs(lg - ref).max()
        out = qjl.quantized_decode(q, st, toks).output
        ref_o = golden[f"qjlc_{name}_out"][i]
        assert np.linalg.norm(out - ref_o) / np.linalg.norm(ref_o) <= 1e-3
    # write it back: the same bytes
    p2 = tmp_path / f"{name}_again.qjlc"
    qjl.write_cache(p2, st, toks)
    assert p2.read_bytes() == c["bytes"]


def test_write_cache_errors(cuda, golden, tmp_path):
    c = case(golden, "r")
    st, toks = _state(c)
    with pytest.raises(ValueError):
        qjl.write_cache(tmp_path / "x", st, toks[:-1])              # kvcache.py:409-412
    bad = toks[:-1] + [qjl.quantize_value(c["values"][0], c["value_bits"] + 1)]
    with pytest.raises(ValueError):
        qjl.write_cache(tmp_path / "x", st, bad)                    # kvcache.py:413-415
    empty = qjl.KeyCacheState.create(st.profile, m_in=96, m_out=40, seed=44, orthogonalize_sketches=False)
    with pytest.raises(ValueError):
        qjl.write_cache(tmp_path / "x", empty, [])                  # kvcache.py:407-408
    blob = bytearray(c["bytes"])
    (tmp_path / "short").write_bytes(bytes(blob[:-3]))
    with pytest.raises(qjl.FileFormatError):
        qjl.read_cache(tmp_path / "short")
    blob[0:4] = b"NOPE"
    (tmp_path / "magic").write_bytes(bytes(blob))
    with pytest.raises(qjl.FileFormatError):
        qjl.read_cache(tmp_path / "magic")


def _u8_cache(units, n, seed=0, h=8, m_in=256, m_out=64, bits=2, cap=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    keys = torch.randn(units, n, 128, device="cuda", generator=g)
    keys[:, :, 5::16] *= 12.0
    keys = keys.to(torch.bfloat16)
    vals = torch.randn(units, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    c = DeviceKeyCache.create(units, 128, m_in, h=h, m_out=m_out, capacity=cap or n, seed=seed + 3,
                              key_dtype=torch.bfloat16, value_layout="u8", value_bits=bits,
                              value_group=128)
    c.detect_outliers(keys)
    c.set_sketches(c.S_in_host, c.S_out_host)
    c.append(keys, vals)
    return c, keys, vals


def _device_arrays(c, n):
    r = dict(bits_in=c.bits_in[:, :n], norm_in=c.norm_in[:, :n], codes=c.v_codes[:, :n],
             zero=c.v_zero[:, :n], scale=c.v_scale[:, :n])
    if c.bits_out is not None:
        r.update(bits_out=c.bits_out[:, :n], norm_out=c.norm_out[:, :n])
    return {k: v.cpu() for k, v in r.items()}


def test_batched_save_matches_oracle_and_load_round_trips(cuda, tmp_path):
    U, n = 5, 1000                                    # ragged last tile
    c, keys, vals = _u8_cache(U, n, seed=7)
    paths = [tmp_path / f"u{u}.qjlc" for u in range(U)]
    Q.save(c, paths)
    dev = _device_arrays(c, n)
    mags = c.magnitudes.cpu().numpy()
    for u, p in enumerate(paths):
        blob = p.read_bytes()
        want = O.qjlc_encode(d=128, h=8, m_in=256, m_out=64, value_bits=2, seed=10, orthogonalized=True,
                             channels=c.channels[u, :8].cpu().numpy(), magnitudes=mags[u],
                             bits_in=dev["bits_in"][u].numpy(),
                             norm_in=dev["norm_in"][u].double().numpy(),
                             bits_out=dev["bits_out"][u].numpy(),
                             norm_out=dev["norm_out"][u].double().numpy(),
                             codes=dev["codes"][u].numpy(), zero=dev["zero"][u, :, 0].double().numpy(),
                             scale=dev["scale"][u, :, 0].double().numpy())
        assert blob == want
    c2 = Q.load(paths, key_dtype=torch.bfloat16)
    assert c2.n == n and c2.n_values == n
    back = _device_arrays(c2, n)
    for k in dev:
        assert torch.equal(dev[k], back[k]), k
    assert torch.equal(c2.channels.cpu(), c.channels.cpu())
    assert torch.equal(c2.s_full.cpu(), c.s_full.cpu())
    q = torch.randn(U, 4, 128, device="cuda").to(torch.bfloat16)
    assert torch.equal(c.decode(q, deterministic=True), c2.decode(q, deterministic=True))
    # idempotent: saving the loaded cache gives the same files
    paths2 = [tmp_path / f"v{u}.qjlc" for u in range(U)]
    Q.save(c2, paths2)
    for a, b in zip(paths, paths2):
        assert a.read_bytes() == b.read_bytes()


def test_fast_path_layouts_are_rejected(cuda, tmp_path):
    c = DeviceKeyCache.create(1, 128, 256, h=8, m_out=64, capacity=128, channels=np.arange(8)[None])
    c.append(torch.randn(1, 4, 128, device="cuda").to(torch.bfloat16),
             torch.randn(1, 4, 128, device="cuda").to(torch.bfloat16))
    with pytest.raises(ValueError):
        Q.save(c, [tmp_path / "x"], magnitudes=np.zeros((1, 128)))


def test_full_size_export_import_round_trip(cuda):
    """C3 shape with reference-format values: export -> import into a fresh cache at a
    row offset is the identity on every byte (size-independent property)."""
    U, n = 16, 32768
    c, _, _ = _u8_cache(U, n, seed=11)
    recs, R = Q.export_records(c.key_desc(), c.value_desc(), 256, 64, n)
    assert R == 180
    d2 = DeviceKeyCache(U, 128, 256, 64, 8, n + 128, value_layout="u8", value_bits=2, value_group=128)
    Q.import_records(recs, n, 256, 64, d2.key_desc(), d2.value_desc(), row_offset=128)
    torch.cuda.synchronize()
    for a, b in ((c.bits_in, d2.bits_in), (c.bits_out, d2.bits_out), (c.norm_in, d2.norm_in),
                 (c.norm_out, d2.norm_out), (c.v_codes, d2.v_codes), (c.v_zero, d2.v_zero),
                 (c.v_scale, d2.v_scale)):
        assert torch.equal(a[:, :n], b[:, 128:128 + n])
    # one unit's records against the oracle's restatement
    u = 9
    h = {k: v[u].cpu() for k, v in _device_arrays(c, n).items()}
    want = O.qjlc_encode(d=128, h=8, m_in=256, m_out=64, value_bits=2, seed=0, orthogonalized=True,
                         channels=np.zeros(8), magnitudes=np.zeros(128), bits_in=h["bits_in"].numpy(),
                         norm_in=h["norm_in"].double().numpy(), bits_out=h["bits_out"].numpy(),
                         norm_out=h["norm_out"].double().numpy(), codes=h["codes"].numpy(),
                         zero=h["zero"][:, 0].double().numpy(), scale=h["scale"][:, 0].double().numpy())
    body = want[Q.HEADER_BYTES + 4 * 8 + 8 * 128:]
    assert recs[u, : n * R].cpu().numpy().tobytes() == body
