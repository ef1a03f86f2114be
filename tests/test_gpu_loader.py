"""Streaming FSVD15 -> GPU loader (runtime.cu load_streaming, the fsvd_model_load
default) vs the host path read_checkpoint_file -> normalize<float> -> upload
(FSVD_LOADER=canonical): device factors bitwise equal for reference-written
files (families A, B, C) and generated ones (D, heterogeneous ranks, LLaMA-7B
width), the same FormatError / NormalizeError behaviour, and the host memory
it holds (pinned staging only -- no CanonicalModel<float> copy of the file)."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu


def _load_both(fsvd, path, dtype):
    os.environ["FSVD_LOADER"] = "canonical"
    try:
        ref = fsvd.Model.load(path, dtype=dtype)
    finally:
        del os.environ["FSVD_LOADER"]
    got = fsvd.Model.load(path, dtype=dtype)
    return ref, got


def _header(path):
    with open(path, "rb") as f:
        pre = f.read(12)
        hlen = struct.unpack("<I", pre[8:12])[0]
        return json.loads(f.read(hlen))


def _rank(hdr, layer, proj):
    """Rank of (layer, proj) from the FSVD15 index (the A-like factor's columns)."""
    shapes = {e["name"]: e["shape"] for e in hdr["tensors"]}
    fam = hdr["family"]
    if fam == "C":
        return shapes[f"shared.{proj}.{hdr['layer_groups'][layer]}.A"][1]
    return shapes[f"layers.{layer}.{proj}." + {"A": "A", "B": "Uf", "D": "U"}[fam]][1]


def _same_factors(fsvd, path, a, b, layers=None):
    cfg = a.config
    hdr = _header(path)
    for layer in (range(cfg.n_layers) if layers is None else layers):
        for p in fsvd.PROJ:
            din = cfg.d_ff if p == "down" else cfg.d_model
            dout = cfg.d_ff if p in ("up", "gate") else cfg.d_model
            r = _rank(hdr, layer, p)
            for which, shape in (("A", (din, r)), ("B", (r, dout))):
                fa = a.factor(layer, p, which, shape)
                fb = b.factor(layer, p, which, shape)
                assert np.array_equal(fa.view(np.uint32), fb.view(np.uint32)), (layer, p, which)


@pytest.mark.parametrize("fname", ["tiny_A.fsvd", "tiny_B.fsvd", "tiny_C.fsvd", "tiny_A_rho1.fsvd"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_streaming_equals_canonical_reference_files(fsvd, fname, dtype):
    ref, got = _load_both(fsvd, GOLDEN / fname, dtype)
    _same_factors(fsvd, GOLDEN / fname, ref, got)
    assert ref.info()["decode_weight_bytes"] == got.info()["decode_weight_bytes"]
    # whole-model check through the runtime: identical logits
    cfg = ref.config
    prompt = np.arange(9, dtype=np.int32)[None] % cfg.vocab
    la = fsvd.Session(ref, batch=1, capacity=64, plan="full_step").prefill(prompt)
    lb = fsvd.Session(got, batch=1, capacity=64, plan="full_step").prefill(prompt)
    assert np.array_equal(la.view(np.uint32), lb.view(np.uint32))
    st = fsvd.Model.last_load_stats()
    assert st["payload_bytes"] > 0 and st["seconds"] > 0


@pytest.mark.parametrize("family", ["B", "D"])
def test_streaming_generated_heterogeneous_ranks(fsvd, tmp_path, family):
    cfg = fsvd.ModelConfig(3, 256, 4, 64, 704, 1000)
    spec = fsvd.SynthSpec(cfg, capacity=128, family=family, rho=0.5, seed=9, rank_jitter=0.3)
    path = tmp_path / f"gen_{family}.fsvd"
    fsvd.write_synthetic(spec, path)
    ref, got = _load_both(fsvd, path, "bf16")
    _same_factors(fsvd, path, ref, got)


def test_streaming_7b_width(fsvd, tmp_path):
    """LLaMA-7B width (d 4096, d_ff 11008, rho 0.6), 4 layers, full vocab: a
    2.6 GB f32 file. Bitwise equal to the host path; host memory stays at the
    pinned staging (the host path holds the file, the Checkpoint and the
    CanonicalModel<float>)."""
    cfg = fsvd.ModelConfig(4, 4096, 32, 128, 11008, 32000)
    spec = fsvd.SynthSpec(cfg, capacity=1024, family="A", rho=0.6, seed=5)
    path = tmp_path / "w7b.fsvd"
    fsvd.write_synthetic(spec, path)
    size = path.stat().st_size
    # the streaming load in a fresh process: its peak RSS is CUDA context + pinned staging
    code = ("import json, resource, sys; sys.path.insert(0, %r); import paper_2605_08314_b200 as F; "
            "rss = lambda: resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024; "
            "t = F.Model.synthetic(F.SynthSpec(F.ModelConfig(1, 128, 4, 32, 256, 512), capacity=64)); r0 = rss(); "
            "m = F.Model.load(%r, dtype='bf16'); st = F.Model.last_load_stats(); "
            "st['rss0'] = r0; st['maxrss'] = rss(); print(json.dumps(st))"
            % (str(ROOT), str(path)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    st = json.loads(r.stdout.strip().splitlines()[-1])
    gbs = st["payload_bytes"] / st["seconds"] / 1e9
    grow = st["maxrss"] - st["rss0"]
    print(f"streaming load: {size / 1e9:.2f} GB in {st['seconds']:.2f} s = {gbs:.1f} GB/s, pinned staging "
          f"{st['pinned_bytes'] / 2**20:.0f} MiB, peak RSS {st['rss0'] / 2**20:.0f} MiB (CUDA context) -> "
          f"{st['maxrss'] / 2**20:.0f} MiB")
    assert st["payload_bytes"] >= size * 0.99
    assert grow < size / 2  # the load holds the pinned staging, nowhere near a host copy of the weights
    got = fsvd.Model.load(path, dtype="bf16")
    os.environ["FSVD_LOADER"] = "canonical"
    try:
        ref = fsvd.Model.load(path, dtype="bf16")
    finally:
        del os.environ["FSVD_LOADER"]
    _same_factors(fsvd, path, ref, got, layers=[0, 3])


def test_streaming_errors(fsvd, tmp_path):
    raw = bytearray((GOLDEN / "tiny_B.fsvd").read_bytes())
    bad = tmp_path / "crc.fsvd"
    c = bytearray(raw)
    c[len(c) - 3] ^= 0xFF
    bad.write_bytes(bytes(c))
    with pytest.raises(fsvd.FormatError, match="checksum"):
        fsvd.Model.load(bad)
    with pytest.raises(fsvd.FormatError):
        fsvd.Model.load(tmp_path / "missing.fsvd")
    trunc = tmp_path / "trunc.fsvd"
    trunc.write_bytes(bytes(raw[: len(raw) // 2]))
    with pytest.raises(fsvd.FormatError):
        fsvd.Model.load(trunc)
    # a zero whitening scale is a NormalizeError (canonical.cpp), found before any upload
    hlen = struct.unpack("<I", raw[8:12])[0]
    hdr = json.loads(raw[12:12 + hlen])
    base = (12 + hlen + 63) // 64 * 64
    ent = next(e for e in hdr["tensors"] if e["name"].endswith(".scale"))
    vec = np.frombuffer(raw, dtype=np.float32, count=int(np.prod(ent["shape"])), offset=base + ent["offset"]).copy()
    vec[0] = 0.0
    import zlib

    ent["crc32"] = zlib.crc32(vec.tobytes())
    text = json.dumps(hdr, separators=(",", ":")).encode()
    nbase = (12 + len(text) + 63) // 64 * 64
    payload = bytearray(raw[base:])
    payload[ent["offset"]: ent["offset"] + vec.nbytes] = vec.tobytes()
    out = raw[:8] + struct.pack("<I", len(text)) + text + b"\0" * (nbase - 12 - len(text)) + bytes(payload)
    z = tmp_path / "zero.fsvd"
    z.write_bytes(bytes(out))
    with pytest.raises(fsvd.NormalizeError, match="zero"):
        fsvd.Model.load(z)
