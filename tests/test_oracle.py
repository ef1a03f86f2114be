"""CPU oracle pinned against the reference (no GPU).

The oracle (oracle/fsvd_oracle.cpp) is the checker for every GPU parity test,
so it is pinned first:
  * against golden vectors frozen from the reference itself
    (tests/golden/make_golden.py calls oracle/_ref, the reference compiled
    from /root/reference) -- these run everywhere, including the GPU box;
  * against the live reference when oracle/_ref is built here;
  * against SPEC invariants the reference states but never tests:
    rho=1 losslessness vs dense_forward_all, cached == no-cache
    (SPEC.md:544), packed == no_merge.
Mirrors proj/tests/test_tensor.cpp (KATs at :12-15, :44-54, :87-99, :106-133,
:140-149, :173-233).
"""
import ctypes as C
import json

import numpy as np
import pytest

from conftest import GOLDEN

PRIM = json.loads((GOLDEN / "primitives.json").read_text())
EXPECT = json.loads((GOLDEN / "tiny_expect.json").read_text())


def unhex(xs, dt=np.float64):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64).astype(dt)


def dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class Cfg:
    def __init__(self, d):
        self.n_layers, self.d_model, self.n_heads = d["n_layers"], d["d_model"], d["n_heads"]
        self.d_head, self.d_ff, self.vocab = d["d_head"], d["d_ff"], d["vocab"]
        self.rope_base, self.norm_eps = 10000.0, 1e-5


TINY = Cfg(EXPECT["config"])


# ------------------------------------------------------------ primitives --
def test_splitmix64_kat(oracle_mod):
    """test_tensor.cpp:12-15: Rng64(0).next_u64() == 0xE220A8397B1DCDAF."""
    L = oracle_mod.lib()
    assert L.oracle_rng_u64(0, 0) == 0xE220A8397B1DCDAF
    for seed, vals in PRIM["rng"].items():
        for k, v in enumerate(vals):
            assert L.oracle_rng_u64(int(seed), k) == int(v, 16), (seed, k)


def test_rank_for_ratio(oracle_mod):
    """compress.cpp:68-80, incl. the 7B/13B ranks the bench uses (1229/1791, 1536/2242)."""
    L = oracle_mod.lib()
    for rho, m, n, r in PRIM["rank_for_ratio"]:
        assert L.oracle_rank_for_ratio(rho, m, n) == r, (rho, m, n)
    assert L.oracle_rank_for_ratio(0.6, 4096, 4096) == 1229
    assert L.oracle_rank_for_ratio(0.6, 4096, 11008) == 1791
    assert L.oracle_rank_for_ratio(0.6, 5120, 5120) == 1536


def test_rmsnorm_bitwise(oracle_mod):
    g = PRIM["rmsnorm"]
    L = oracle_mod.lib()
    x, gam = unhex(g["x"]), unhex(g["g"])
    y = np.empty_like(x)
    L.oracle_rmsnorm_f64(dp(y), dp(x), fp(gam.astype(np.float32)), x.size, g["eps"])
    # the oracle takes f32 gammas (canonical weights are floats): compare with
    # the f32 path bitwise and the f64 path to f32-gamma rounding
    xf, gf = unhex(g["xf"], np.float32), unhex(g["gf"], np.float32)
    yf = np.empty_like(xf)
    L.oracle_rmsnorm_f32(fp(yf), fp(xf), fp(gf), xf.size, np.float32(g["eps"]))
    assert np.array_equal(yf.view(np.uint32), unhex(g["y32"], np.float32).view(np.uint32))
    assert np.allclose(y, unhex(g["y64"]), rtol=1e-6)


def test_rope_bitwise(oracle_mod):
    """math.hpp:30-44: interleaved pairs, angle in double; f64 bitwise."""
    L = oracle_mod.lib()
    for case in PRIM["rope"]:
        v = unhex(case["v"])
        L.oracle_rope_f64(dp(v), case["d"], case["pos"], 10000.0)
        assert np.array_equal(v, unhex(case["out64"])), case["pos"]
        if case["pos"] == 0.0:
            assert np.array_equal(v, unhex(case["v"]))  # test_tensor.cpp:106-112 identity


def test_online_attend(oracle_mod):
    """math.hpp:56-129 and test_tensor.cpp:173-233 (<= 1e-12, partition invariance)."""
    L = oracle_mod.lib()
    for case in PRIM["online_attend"]:
        d, rows = case["d"], case["rows"]
        q, k, v = unhex(case["q"]), unhex(case["k"]).reshape(rows, d), unhex(case["v"]).reshape(rows, d)
        want = unhex(case["out"])
        for blocks in (case["blocks"], [rows], [1] * rows):
            o = np.empty(d)
            bl = (C.c_uint64 * len(blocks))(*blocks)
            L.oracle_online_attend_f64(dp(q), dp(k), dp(v), rows, d, case["scale"], bl, len(blocks), dp(o))
            if blocks == case["blocks"]:
                assert np.array_equal(o, want)
            assert np.abs(o - want).max() <= 1e-12
        # naive softmax oracle (oracles.hpp:30-60)
        s = k @ q * case["scale"]
        w = np.exp(s - s.max())
        assert np.abs(w @ v / w.sum() - want).max() <= 1e-12


def test_argmax_ties_lowest(oracle_mod):
    L = oracle_mod.lib()
    for case in PRIM["argmax"]:
        a = np.array(case["x"], dtype=np.float64)
        assert L.oracle_argmax_f64(dp(a), a.size) == case["idx"]


def test_gemv_per_column_order(oracle_mod):
    """kernels.hpp:8-11: every column accumulates over k in index order --
    the oracle's column-parallel gemv is bitwise the reference scalar kernel."""
    g = PRIM["gemv_f32"]
    m, n = g["m"], g["n"]
    x, a = unhex(g["x"], np.float32), unhex(g["a"], np.float32).reshape(m, n)
    L = oracle_mod.lib()
    for threads in (1, 4):
        oracle_mod.set_threads(threads)
        y = np.empty(n, np.float32)
        L.oracle_gemv_f32(fp(y), fp(x), fp(a), m, n)
        assert np.array_equal(y.view(np.uint32), unhex(g["y"], np.float32).view(np.uint32))
    oracle_mod.set_threads(1)


# ------------------------------------------------------- checkpoints ------
@pytest.mark.parametrize("fname", sorted(EXPECT["files"]))
def test_loader_matches_reference_normalize(oracle_mod, fname):
    """canonical.cpp:155-194: the oracle's normalize of a reference-written
    FSVD15 file equals the reference's normalize<float> bitwise (per-tensor
    CRC-32 of the reference output, frozen in tiny_expect.json)."""
    import zlib

    info = EXPECT["files"][fname]
    om = oracle_mod.OracleModel.load_file(GOLDEN / fname, TINY)
    ranks = {k: v for k, v in info["ranks"].items()}
    for name, crc in info["normalized_crc32"].items():
        shape = _shape(name, ranks)
        t = om.tensor(name, shape)
        assert f"{zlib.crc32(t.tobytes()) & 0xFFFFFFFF:08x}" == crc, name
    assert om.shared_instances() == info["shared_basis_table"]


def _shape(name, ranks):
    d, dff, V = TINY.d_model, TINY.d_ff, TINY.vocab
    if name in ("embedding", "head"):
        return (V, d) if name == "embedding" else (d, V)
    if name.endswith("gamma"):
        return (d,)
    parts = name.split(".")
    l = parts[1]
    if parts[2] == "a_ug":
        return (d, ranks[f"{l}.up"] + ranks[f"{l}.gate"])
    p, w = parts[2], parts[3]
    din = dff if p == "down" else d
    dout = dff if p in ("up", "gate") else d
    r = ranks[f"{l}.{p}"]
    return (din, r) if w == "A" else (r, dout)


def test_rho1_lossless_vs_dense_gold(oracle_mod):
    """SPEC.md:543 acceptance #1: a rho=1 factorization through the oracle's
    no-cache forward reproduces the reference dense_forward_all (model.cpp:204-285)."""
    om = oracle_mod.OracleModel.load_file(GOLDEN / "tiny_A_rho1.fsvd", TINY)
    toks = np.array(EXPECT["tokens"], dtype=np.int32)
    got = om.forward_nocache(toks, f64=True)
    want = np.load(GOLDEN / "tiny_dense_logits.npy")
    # factors are f32 on disk (checkpoint.cpp:102): A.B == W to ~1e-7 relative
    assert oracle_mod.rel_err(got, want) <= 1e-5


@pytest.mark.parametrize("fname", ["tiny_A.fsvd", "tiny_B.fsvd", "tiny_C.fsvd"])
def test_cached_equals_nocache(oracle_mod, fname):
    """SPEC.md:544 acceptance #2: prefill + decode_step == no-cache forward (f64, 1e-12)."""
    om = oracle_mod.OracleModel.load_file(GOLDEN / fname, TINY)
    toks = np.array(EXPECT["tokens"], dtype=np.int32)
    full = om.forward_nocache(toks, f64=True)
    s = om.session(f64=True, capacity=64)
    got = [s.prefill(toks[:5])]
    for t in toks[5:]:
        got.append(s.decode_step(int(t)))
    got = np.stack(got)
    assert oracle_mod.rel_err(got, full[4:]) <= 1e-12
    assert s.position == toks.size


def test_packed_equals_no_merge_oracle(oracle_mod):
    """SPEC.md:547 acceptance #5 (f64: packing is an exact column concat)."""
    om = oracle_mod.OracleModel.load_file(GOLDEN / "tiny_C.fsvd", TINY)
    toks = np.array(EXPECT["tokens"], dtype=np.int32)
    a = om.session(f64=True, ffn="no_merge", capacity=64).prefill(toks)
    b = om.session(f64=True, ffn="packed", capacity=64).prefill(toks)
    assert np.array_equal(a, b)


def test_f32_mode_close_to_f64(oracle_mod):
    om = oracle_mod.OracleModel.load_file(GOLDEN / "tiny_B.fsvd", TINY)
    toks = np.array(EXPECT["tokens"], dtype=np.int32)
    a = om.session(f64=True, capacity=64).prefill(toks)
    b = om.session(f64=False, capacity=64).prefill(toks)
    assert oracle_mod.rel_err(b, a) <= 1e-5


def test_oracle_capacity_errors(oracle_mod):
    om = oracle_mod.OracleModel.load_file(GOLDEN / "tiny_A.fsvd", TINY)
    s = om.session(f64=True, capacity=8)
    with pytest.raises(oracle_mod.OracleError):
        s.prefill(np.arange(9, dtype=np.int32))
    s.prefill(np.arange(8, dtype=np.int32))
    with pytest.raises(oracle_mod.OracleError):
        s.decode_step(1)


# ------------------------------------------------ live reference (here) --
def test_oracle_vs_live_reference(oracle_mod, ref):
    """When oracle/_ref is built (this container), re-derive the golden
    primitives from the reference and compare with the oracle directly."""
    L = oracle_mod.lib()
    rng = np.random.default_rng(99)
    for d, pos in ((64, 3.0), (128, 4607.0), (128, 1.0e4)):
        v = rng.uniform(-1, 1, d)
        a, b = v.copy(), v.copy()
        L.oracle_rope_f64(dp(a), d, pos, 10000.0)
        ref.ref_rope_f64(dp(b), d, pos, 10000.0)
        assert np.array_equal(a, b)
    for k in range(8):
        assert L.oracle_rng_u64(123, k) == ref.ref_rng_u64(123, k)
    ref.ref_force_variant(b"scalar")
    m, n = 300, 70
    x = rng.uniform(-1, 1, m).astype(np.float32)
    a = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    y1, y2 = np.empty(n, np.float32), np.empty(n, np.float32)
    L.oracle_gemv_f32(fp(y1), fp(x), fp(a), m, n)
    ref.ref_gemv_f32(fp(y2), fp(x), fp(a), m, n)
    assert np.array_equal(y1.view(np.uint32), y2.view(np.uint32))
