#!/usr/bin/env python3
"""Freeze outputs of the REFERENCE itself as golden fixtures.

    python tests/golden/make_golden.py          # needs /root/reference (builds oracle/_ref)

The GPU box has no /root/reference, so everything the parity tests need from
the real reference is generated here and committed:

  primitives.json   reference math on seeded inputs: SplitMix64 stream
                    (tensor.hpp:35-62; KAT test_tensor.cpp:12-15), rank_for_ratio
                    (compress.cpp:68-80), rmsnorm (math.hpp:16-25), rope_inplace
                    (math.hpp:30-44), online_softmax_attend (math.hpp:104-129),
                    argmax_greedy (math.hpp:132-140), gemv via kern::Ops
                    (kernels_scalar.cpp:11-21), dense_model_checksum (model.cpp:113-130)
  tiny_{A,B,C}.fsvd FSVD15 checkpoints written by the reference's own compressor
                    (compress.cpp:243-256 -> write_checkpoint checkpoint.cpp:85-132)
                    from generate_toy_dense(TINY, seed 7); A also at rho=1
  tiny_expect.json  per-tensor CRC-32 of the reference normalize<float> output of
                    each file (canonical.cpp:155-194), shared_basis_table sizes,
                    and dense_forward_all logits (model.cpp:204-285, f64) of the
                    dense model the files were compressed from.

Every value is produced by calling the reference (oracle/_ref/libfsvd_ref.so,
compiled from /root/reference by oracle/Makefile); nothing is computed by the
restated oracle or the product.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
import zlib
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402

# tiny decoder: L=2, d=64, H=2 (d_h 32), d_ff=160, V=96
TINY = dict(n_layers=2, d_model=64, n_heads=2, d_head=32, d_ff=160, vocab=96)
TINY_SEED = 7
TINY_TOKENS = [3, 17, 88, 41, 0, 95, 12, 12, 60, 33, 7, 71]
DESK = dict(n_layers=4, d_model=256, n_heads=8, d_head=32, d_ff=1024, vocab=1024)  # model.cpp:29-32


def c6c2(cfg):
    c6 = (C.c_uint64 * 6)(cfg["n_layers"], cfg["d_model"], cfg["n_heads"], cfg["d_head"], cfg["d_ff"], cfg["vocab"])
    c2 = np.array([10000.0, 1e-5], dtype=np.float64)
    return c6, c2


def hexd(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def hexf(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float32).astype(np.float64).ravel()]


def dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def ok(rc, r):
    if rc != 0:
        raise RuntimeError(r.ref_last_error().decode())


def primitives(r) -> dict:
    out: dict = {}
    # the semantic kernel table (kernels_scalar.cpp); the oracle restates it
    r.ref_force_variant(b"scalar")
    out["variant"] = r.ref_active_variant().decode()
    out["rng"] = {str(s): [f"{r.ref_rng_u64(s, k):016x}" for k in range(6)] for s in (0, 1, 42, 0xDEADBEEF)}
    out["rank_for_ratio"] = [[rho, m, n, int(r.ref_rank_for_ratio(rho, m, n))]
                             for rho in (0.5, 0.6, 1.0, 0.25)
                             for (m, n) in ((256, 256), (256, 1024), (1024, 256), (4096, 4096), (4096, 11008),
                                            (11008, 4096), (5120, 5120), (5120, 13824), (64, 160))]
    rng = np.random.default_rng(3)
    # rmsnorm f64 + f32 (test_tensor.cpp:87-99 uses n=33)
    x = rng.uniform(-2, 2, 33)
    g = rng.uniform(0.5, 1.5, 33)
    y = np.empty(33)
    r.ref_rmsnorm_f64(dp(y), dp(x), dp(g), 33, 1e-5)
    xf, gf = x.astype(np.float32), g.astype(np.float32)
    yf = np.empty(33, np.float32)
    r.ref_rmsnorm_f32(fp(yf), fp(xf), fp(gf), 33, np.float32(1e-5))
    out["rmsnorm"] = {"x": hexd(x), "g": hexd(g), "eps": 1e-5, "y64": hexd(y), "xf": hexf(xf), "gf": hexf(gf),
                      "y32": hexf(yf)}
    # rope at several positions (d_h 64 and 128), f64 and f32
    ropes = []
    for d, pos in ((64, 0.0), (64, 1.0), (64, 37.0), (128, 511.0), (128, 4607.0), (128, 8191.0)):
        v = rng.uniform(-1, 1, d)
        w = v.copy()
        r.ref_rope_f64(dp(w), d, pos, 10000.0)
        vf = v.astype(np.float32)
        wf = vf.copy()
        r.ref_rope_f32(fp(wf), d, pos, 10000.0)
        ropes.append({"d": d, "pos": pos, "v": hexd(v), "out64": hexd(w), "vf": hexf(vf), "out32": hexf(wf)})
    out["rope"] = ropes
    # online softmax over blocks (test_tensor.cpp:173-233: d=8, scale 0.35)
    att = []
    for seed, rows, d, blocks in ((11, 64, 8, [16, 16, 16, 16]), (23, 21, 8, [3, 5, 1, 7, 5]), (5, 130, 64, [64, 64, 2])):
        rr = np.random.default_rng(seed)
        q, k, v = rr.uniform(-1, 1, d), rr.uniform(-1, 1, (rows, d)), rr.uniform(-1, 1, (rows, d))
        o = np.empty(d)
        bl = (C.c_uint64 * len(blocks))(*blocks)
        ok(r.ref_online_attend_f64(dp(q), dp(np.ascontiguousarray(k)), dp(np.ascontiguousarray(v)), d, 0.35, bl,
                                   len(blocks), dp(o)), r)
        att.append({"rows": rows, "d": d, "blocks": blocks, "scale": 0.35, "q": hexd(q), "k": hexd(k), "v": hexd(v),
                    "out": hexd(o)})
    out["online_attend"] = att
    # argmax ties -> lowest index (test_tensor.cpp:140-149)
    am = []
    for vec in ([1.0, 3.0, 3.0, 2.0], [-1.0, -1.0], [0.5], [2.0, 1.0, 2.0, 2.0]):
        a = np.array(vec, dtype=np.float64)
        am.append({"x": vec, "idx": int(r.ref_argmax_f64(dp(a), a.size))})
    out["argmax"] = am
    # gemv via the reference's kern::Ops (scalar table, forced above)
    m, n = 37, 29
    xv = rng.uniform(-1, 1, m).astype(np.float32)
    A = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    yv = np.empty(n, np.float32)
    r.ref_gemv_f32(fp(yv), fp(xv), fp(A), m, n)
    out["gemv_f32"] = {"m": m, "n": n, "x": hexf(xv), "a": hexf(A), "y": hexf(yv)}
    # dense toy checksum (model.cpp:113-130); desk seed 1 = 0x54BA8A2A [SURVEY probe]
    cs = C.c_uint32()
    c6, c2 = c6c2(DESK)
    ok(r.ref_dense_checksum(c6, dp(c2), 1, C.byref(cs)), r)
    out["desk_checksum_seed1"] = f"{cs.value:08x}"
    c6, c2 = c6c2(TINY)
    ok(r.ref_dense_checksum(c6, dp(c2), TINY_SEED, C.byref(cs)), r)
    out["tiny_checksum"] = f"{cs.value:08x}"
    return out


def tensor_names(cfg):
    names = ["embedding", "head", "final_gamma"]
    for l in range(cfg["n_layers"]):
        names += [f"layers.{l}.attn_gamma", f"layers.{l}.mlp_gamma", f"layers.{l}.a_ug"]
        names += [f"layers.{l}.{p}.{w}" for p in ("q", "k", "v", "o", "up", "gate", "down") for w in "AB"]
    return names


def tensor_count(cfg, name, ranks):
    d, dff, V = cfg["d_model"], cfg["d_ff"], cfg["vocab"]
    if name in ("embedding", "head"):
        return V * d
    if name == "final_gamma" or name.endswith("gamma"):
        return d
    parts = name.split(".")
    l = int(parts[1])
    if parts[2] == "a_ug":
        return d * (ranks[(l, "up")] + ranks[(l, "gate")])
    p, w = parts[2], parts[3]
    din = dff if p == "down" else d
    dout = dff if p in ("up", "gate") else d
    return (din if w == "A" else dout) * ranks[(l, p)]


def checkpoints(r) -> dict:
    expect: dict = {"config": TINY, "seed": TINY_SEED, "tokens": TINY_TOKENS, "files": {}}
    c6, c2 = c6c2(TINY)
    cases = [("tiny_A.fsvd", "A", 0.5), ("tiny_B.fsvd", "B", 0.5), ("tiny_C.fsvd", "C", 0.5),
             ("tiny_A_rho1.fsvd", "A", 1.0)]
    for fname, fam, rho in cases:
        path = HERE / fname
        ok(r.ref_compress_to_file(c6, dp(c2), 256, TINY_SEED, fam.encode(), rho, 2, str(path).encode()), r)
        raw = path.read_bytes()
        # ranks from the header (checkpoint.hpp:3-7: magic, u16 version, u32 header_len, json)
        hlen = int.from_bytes(raw[8:12], "little")
        hdr = json.loads(raw[12:12 + hlen])
        ranks = {}
        for t in hdr["tensors"]:
            nm, shp = t["name"], t["shape"]
            parts = nm.split(".")
            if nm.startswith("layers.") and len(parts) == 4 and parts[3] in ("A", "Uf", "B", "Vt"):
                pr = parts[2]
                ranks[(int(parts[1]), pr)] = shp[0] if parts[3] in ("B", "Vt") else shp[1]
            elif nm.startswith("shared."):
                pass
        if fam == "C":  # shared bases: rank of A from shared.{p}.{g}.A, B carries it too
            for t in hdr["tensors"]:
                parts = t["name"].split(".")
                if t["name"].startswith("layers.") and len(parts) == 4 and parts[3] == "B":
                    ranks[(int(parts[1]), parts[2])] = t["shape"][0]
        crcs = {}
        for nm in tensor_names(TINY):
            n = tensor_count(TINY, nm, ranks)
            buf = np.empty(n, np.float32)
            ok(r.ref_normalize_tensor(str(path).encode(), nm.encode(), fp(buf), n), r)
            crcs[nm] = f"{zlib.crc32(buf.tobytes()) & 0xFFFFFFFF:08x}"
        sc = C.c_uint64()
        ok(r.ref_shared_count(str(path).encode(), C.byref(sc)), r)
        rt = HERE / ("_rt_" + fname)
        ok(r.ref_roundtrip(str(path).encode(), str(rt).encode()), r)
        same = rt.read_bytes() == raw
        rt.unlink()
        expect["files"][fname] = {
            "family": fam, "rho": rho, "bytes": len(raw), "file_crc32": f"{zlib.crc32(raw) & 0xFFFFFFFF:08x}",
            "ranks": {f"{l}.{p}": v for (l, p), v in sorted(ranks.items())},
            "normalized_crc32": crcs, "shared_basis_table": sc.value, "roundtrip_identical": same,
        }
    # dense gold forward of the model the files were compressed from (f64)
    toks = np.array(TINY_TOKENS, dtype=np.int32)
    lg = np.empty((toks.size, TINY["vocab"]), dtype=np.float64)
    ok(r.ref_dense_forward_all(c6, dp(c2), TINY_SEED, toks.ctypes.data_as(C.POINTER(C.c_int32)), toks.size, dp(lg)), r)
    np.save(HERE / "tiny_dense_logits.npy", lg)
    return expect


def main():
    oracle.build(ref=True)
    r = oracle.ref()
    prims = primitives(r)
    (HERE / "primitives.json").write_text(json.dumps(prims, indent=1) + "\n")
    exp = checkpoints(r)
    (HERE / "tiny_expect.json").write_text(json.dumps(exp, indent=1) + "\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
