"""Product host loader (libfsvd_b200.so, CPU only) vs the reference.

read_checkpoint_file -> normalize<float> is the drop-in loader named by the
north star (checkpoint.cpp:134-214, canonical.cpp:155-194). The product's
C++ loader must produce the reference's CanonicalModel<float> bit for bit on
files the reference itself wrote (tests/golden/tiny_*.fsvd), reject the
same malformed inputs with the same error type (FormatError
checkpoint.hpp:21, NormalizeError canonical.hpp:21), and alias shared bases
(canonical.cpp:138-145).
"""
import json
import zlib

import numpy as np
import pytest

from conftest import GOLDEN
from test_oracle import EXPECT, TINY, _shape


@pytest.mark.parametrize("fname", sorted(EXPECT["files"]))
def test_normalize_matches_reference(fsvd, fname):
    info = EXPECT["files"][fname]
    can = fsvd.Canonical.load_file(GOLDEN / fname)
    cfg = can.config
    assert (cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.d_head, cfg.d_ff, cfg.vocab) == (
        TINY.n_layers, TINY.d_model, TINY.n_heads, TINY.d_head, TINY.d_ff, TINY.vocab)
    assert can.capacity == 256
    for name, crc in info["normalized_crc32"].items():
        t = can.tensor(name, _shape(name, info["ranks"]))
        assert f"{zlib.crc32(t.tobytes()) & 0xFFFFFFFF:08x}" == crc, name
    for key, r in info["ranks"].items():
        l, p = key.split(".")
        assert can.rank(int(l), p) == r
    assert can.shared_count() == info["shared_basis_table"]


def test_family_c_aliases_shared_bases(fsvd):
    """canonical.cpp:138-145: layers of a group share one A storage."""
    can = fsvd.Canonical.load_file(GOLDEN / "tiny_C.fsvd")
    for p in fsvd.PROJ:
        assert can.aliased(0, 1, p)
    a = fsvd.Canonical.load_file(GOLDEN / "tiny_A.fsvd")
    assert not a.aliased(0, 1, "q")


def test_load_bytes_equals_load_file(fsvd):
    raw = (GOLDEN / "tiny_B.fsvd").read_bytes()
    a = fsvd.Canonical.load_bytes(raw)
    b = fsvd.Canonical.load_file(GOLDEN / "tiny_B.fsvd")
    for name in ("layers.1.q.A", "layers.0.down.B", "head"):
        shp = _shape(name, EXPECT["files"]["tiny_B.fsvd"]["ranks"])
        assert np.array_equal(a.tensor(name, shp), b.tensor(name, shp))


def _corrupt(raw: bytes, pos: int) -> bytes:
    b = bytearray(raw)
    b[pos] ^= 0x5A
    return bytes(b)


def test_format_errors(fsvd):
    """checkpoint.cpp:136-191: magic, version, CRC, truncation -> FormatError."""
    raw = (GOLDEN / "tiny_A.fsvd").read_bytes()
    with pytest.raises(fsvd.FormatError):
        fsvd.Canonical.load_bytes(_corrupt(raw, 0))  # magic
    with pytest.raises(fsvd.FormatError):
        fsvd.Canonical.load_bytes(raw[:6] + b"\x02\x00" + raw[8:])  # version 2
    with pytest.raises(fsvd.FormatError, match="checksum"):
        fsvd.Canonical.load_bytes(_corrupt(raw, len(raw) - 3))  # payload byte
    with pytest.raises(fsvd.FormatError):
        fsvd.Canonical.load_bytes(raw[: len(raw) // 2])  # truncated
    with pytest.raises(fsvd.FormatError):
        fsvd.Canonical.load_file(GOLDEN / "does_not_exist.fsvd")


def test_normalize_errors(fsvd):
    """canonical.cpp: a family-B zero scale entry -> NormalizeError."""
    raw = bytearray((GOLDEN / "tiny_B.fsvd").read_bytes())
    hlen = int.from_bytes(raw[8:12], "little")
    hdr = json.loads(raw[12:12 + hlen])
    base = (12 + hlen + 63) // 64 * 64
    ent = next(t for t in hdr["tensors"] if t["name"] == "layers.0.q.scale")
    off = base + ent["offset"]
    raw[off:off + 4] = np.float32(0).tobytes()
    ent["crc32"] = zlib.crc32(bytes(raw[off:off + 4 * ent["shape"][0]])) & 0xFFFFFFFF
    new_hdr = json.dumps(hdr, separators=(",", ":")).encode()
    payload = bytes(raw[base:])  # tensor offsets are payload-relative (checkpoint.hpp:3-7)
    head = bytes(raw[:8]) + len(new_hdr).to_bytes(4, "little") + new_hdr
    head += b"\0" * ((len(head) + 63) // 64 * 64 - len(head))
    with pytest.raises(fsvd.NormalizeError, match="zero"):
        fsvd.Canonical.load_bytes(head + payload)


def test_synthetic_roundtrip_through_fsvd15(fsvd, tmp_path):
    """Synthetic generator -> FSVD15 file -> loader == in-memory canonical (all families)."""
    cfg = fsvd.ModelConfig(2, 64, 2, 32, 160, 96)
    for fam in "ABCD":
        spec = fsvd.SynthSpec(cfg, capacity=128, family=fam, rho=0.5, seed=4, rank_jitter=0.3 if fam in "BD" else 0)
        p = tmp_path / f"s_{fam}.fsvd"
        fsvd.write_synthetic(spec, p)
        a = fsvd.Canonical.load_file(p)
        b = fsvd.Canonical.synthetic(spec)
        for l in range(2):
            for proj in fsvd.PROJ:
                assert a.rank(l, proj) == b.rank(l, proj)
                r = a.rank(l, proj)
                din = cfg.d_ff if proj == "down" else cfg.d_model
                dout = cfg.d_ff if proj in ("up", "gate") else cfg.d_model
                for w, shp in (("A", (din, r)), ("B", (r, dout))):
                    nm = f"layers.{l}.{proj}.{w}"
                    assert np.array_equal(a.tensor(nm, shp), b.tensor(nm, shp)), (fam, nm)


def test_synthetic_matches_oracle_generator(fsvd, oracle_mod):
    """include/fsvd/synth.hpp is restated independently in the oracle."""
    cfg = fsvd.ModelConfig(2, 64, 2, 32, 160, 96)
    for fam in "ABCD":
        spec = fsvd.SynthSpec(cfg, capacity=128, family=fam, rho=0.5, seed=9, conditioned=True,
                              rank_jitter=0.3 if fam in "BD" else 0)
        a = fsvd.Canonical.synthetic(spec)
        o = oracle_mod.OracleModel.synthetic(spec)
        for l in range(2):
            for proj in fsvd.PROJ:
                r = a.rank(l, proj)
                assert o.rank(l, fsvd.PROJ.index(proj)) == r
                din = cfg.d_ff if proj == "down" else cfg.d_model
                nm = f"layers.{l}.{proj}.A"
                assert np.array_equal(a.tensor(nm, (din, r)), o.tensor(nm, (din, r))), (fam, nm)
        assert np.array_equal(a.tensor("head", (64, 96)), o.tensor("head", (64, 96)))


def test_route_ffn_auto(fsvd):
    """eager -> no_merge, per_layer -> packed; explicit wins."""
    assert fsvd.route_ffn_auto("eager") == "no_merge"
    assert fsvd.route_ffn_auto("per_layer") == "packed"
    assert fsvd.route_ffn_auto("full_step") == "packed"
    assert fsvd.route_ffn_auto("eager", "packed") == "packed"
    assert fsvd.route_ffn_auto("per_layer", "no_merge") == "no_merge"
