"""CPU oracle bindings -- TEST INFRASTRUCTURE ONLY.

Loads oracle/_build/liboracle.so (the C++ restatement in fsvd_oracle.cpp) and,
when present, oracle/_ref/libfsvd_ref.so (the reference itself compiled from
/root/reference by oracle/Makefile). Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"
REF_LIB = HERE / "_ref" / "libfsvd_ref.so"
REFERENCE_TREE = Path("/root/reference/proj")

_o = None
_r = None


def build(ref: bool | None = None) -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    if ref or (ref is None and REFERENCE_TREE.exists()):
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


def lib() -> C.CDLL:
    global _o
    if _o is None:
        if not LIB.exists():
            build(ref=False)
        L = C.CDLL(str(LIB))
        vp, u64, dp, i32p = C.c_void_p, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_int32)
        sig = {
            "oracle_last_error": ([], C.c_char_p),
            "oracle_set_threads": ([C.c_int], None),
            "oracle_set_ref_gemv": ([vp], None),
            "oracle_load_file": ([C.c_char_p], vp),
            "oracle_synthetic": ([C.POINTER(u64), dp, u64, C.c_char, C.c_double, u64, u64, C.c_int, C.c_double], vp),
            "oracle_free_model": ([vp], None),
            "oracle_shared_instances": ([vp], u64),
            "oracle_rank": ([vp, u64, C.c_int], u64),
            "oracle_tensor": ([vp, C.c_char_p, C.POINTER(C.c_float), u64], C.c_int),
            "oracle_session": ([vp, C.c_int, C.c_int, u64], vp),
            "oracle_free_session": ([vp], None),
            "oracle_clone_session": ([vp], vp),
            "oracle_prefill": ([vp, i32p, u64, dp], C.c_int),
            "oracle_decode": ([vp, C.c_int32, dp], C.c_int),
            "oracle_generate": ([vp, i32p, u64, u64, i32p], C.c_int),
            "oracle_forward_nocache": ([vp, C.c_int, i32p, u64, dp], C.c_int),
            "oracle_read_kv": ([vp, u64, C.c_int, u64, u64, dp], C.c_int),
            "oracle_position": ([vp], u64),
            "oracle_rope_f64": ([dp, u64, C.c_double, C.c_double], None),
            "oracle_rmsnorm_f64": ([dp, dp, C.POINTER(C.c_float), u64, C.c_double], None),
            "oracle_rmsnorm_f32": ([C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float), u64,
                                    C.c_float], None),
            "oracle_gemv_f32": ([C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float), u64, u64], None),
            "oracle_online_attend_f64": ([dp, dp, dp, u64, u64, C.c_double, C.POINTER(u64), u64, dp], None),
            "oracle_rng_u64": ([u64, u64], u64),
            "oracle_rank_for_ratio": ([C.c_double, u64, u64], u64),
            "oracle_argmax_f64": ([dp, u64], u64),
        }
        for name, (a, r) in sig.items():
            f = getattr(L, name)
            f.argtypes = a
            f.restype = r
        _o = L
    return _o


def ref_available() -> bool:
    return REF_LIB.exists()


def ref() -> C.CDLL:
    """The reference implementation (oracle/_ref), compiled from its own sources."""
    global _r
    if _r is None:
        if not REF_LIB.exists():
            raise RuntimeError("oracle/_ref/libfsvd_ref.so not built (needs /root/reference)")
        L = C.CDLL(str(REF_LIB))
        vp, u64, dp, i32p, fp = C.c_void_p, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_float)
        sig = {
            "ref_last_error": ([], C.c_char_p),
            "ref_force_variant": ([C.c_char_p], C.c_int),
            "ref_active_variant": ([], C.c_char_p),
            "ref_gemv_f32_ptr": ([], vp),
            "ref_gemv_f32": ([fp, fp, fp, u64, u64], None),
            "ref_gemv_f64": ([dp, dp, dp, u64, u64], None),
            "ref_rmsnorm_f64": ([dp, dp, dp, u64, C.c_double], None),
            "ref_rmsnorm_f32": ([fp, fp, fp, u64, C.c_float], None),
            "ref_rope_f64": ([dp, u64, C.c_double, C.c_double], None),
            "ref_rope_f32": ([fp, u64, C.c_double, C.c_double], None),
            "ref_online_attend_f64": ([dp, dp, dp, u64, C.c_double, C.POINTER(u64), u64, dp], C.c_int),
            "ref_argmax_f64": ([dp, u64], u64),
            "ref_rng_u64": ([u64, u64], u64),
            "ref_rank_for_ratio": ([C.c_double, u64, u64], u64),
            "ref_dense_checksum": ([C.POINTER(u64), dp, u64, C.POINTER(C.c_uint32)], C.c_int),
            "ref_compress_to_file": ([C.POINTER(u64), dp, u64, u64, C.c_char, C.c_double, u64, C.c_char_p], C.c_int),
            "ref_dense_forward_all": ([C.POINTER(u64), dp, u64, i32p, u64, dp], C.c_int),
            "ref_normalize_tensor": ([C.c_char_p, C.c_char_p, fp, u64], C.c_int),
            "ref_shared_count": ([C.c_char_p, C.POINTER(u64)], C.c_int),
            "ref_roundtrip": ([C.c_char_p, C.c_char_p], C.c_int),
        }
        for name, (a, r) in sig.items():
            f = getattr(L, name)
            f.argtypes = a
            f.restype = r
        _r = L
    return _r


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def cfg_arrays(cfg):
    c6 = (C.c_uint64 * 6)(cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.d_head, cfg.d_ff, cfg.vocab)
    c2 = np.array([cfg.rope_base, cfg.norm_eps], dtype=np.float64)
    return c6, c2


class OracleError(RuntimeError):
    pass


def _ok(rc: int):
    if rc != 0:
        raise OracleError(lib().oracle_last_error().decode())


class OracleModel:
    """Canonical model as the oracle sees it (normalize<float> weights)."""

    def __init__(self, h, cfg):
        if not h:
            raise OracleError(lib().oracle_last_error().decode())
        self._h = h
        self.cfg = cfg

    @classmethod
    def load_file(cls, path, cfg):
        return cls(lib().oracle_load_file(str(path).encode()), cfg)

    @classmethod
    def synthetic(cls, spec):
        c6, c2 = cfg_arrays(spec.config)
        h = lib().oracle_synthetic(c6, _dp(c2), spec.capacity, spec.family.encode(), spec.rho, spec.group_size,
                                   spec.seed, 1 if spec.conditioned else 0, spec.rank_jitter)
        return cls(h, spec.config)

    def tensor(self, name, shape):
        out = np.empty(shape, dtype=np.float32)
        _ok(lib().oracle_tensor(self._h, name.encode(), _fp(out), out.size))
        return out

    def rank(self, layer, proj):
        return int(lib().oracle_rank(self._h, layer, proj))

    def shared_instances(self):
        return int(lib().oracle_shared_instances(self._h))

    def forward_nocache(self, tokens, f64=True):
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        out = np.empty((t.size, self.cfg.vocab), dtype=np.float64)
        _ok(lib().oracle_forward_nocache(self._h, 1 if f64 else 0, _ip(t), t.size, _dp(out)))
        return out

    def session(self, f64=True, ffn="no_merge", capacity=8192):
        return OracleSession(self, f64, ffn, capacity)

    def __del__(self):
        if getattr(self, "_h", None) and _o is not None:
            _o.oracle_free_model(self._h)
            self._h = None


class OracleSession:
    def __init__(self, model: OracleModel, f64: bool, ffn: str, capacity: int, _handle=None):
        self.model = model
        self._h = _handle or lib().oracle_session(model._h, 1 if f64 else 0, 2 if ffn == "packed" else 1, capacity)

    def clone(self) -> "OracleSession":
        """Independent copy (KV cache + position): fork a shared prompt prefix."""
        return OracleSession(self.model, True, "", 0, _handle=lib().oracle_clone_session(self._h))

    def prefill(self, tokens):
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        out = np.empty(self.model.cfg.vocab, dtype=np.float64)
        _ok(lib().oracle_prefill(self._h, _ip(t), t.size, _dp(out)))
        return out

    def decode_step(self, token):
        out = np.empty(self.model.cfg.vocab, dtype=np.float64)
        _ok(lib().oracle_decode(self._h, int(token), _dp(out)))
        return out

    def generate(self, prompt, max_new):
        t = np.ascontiguousarray(np.asarray(prompt, dtype=np.int32))
        out = np.zeros(max_new, dtype=np.int32)
        _ok(lib().oracle_generate(self._h, _ip(t), t.size, max_new, _ip(out)))
        return out

    def read_kv(self, layer, which, pos0, n):
        out = np.empty((n, self.model.cfg.d_model), dtype=np.float64)
        _ok(lib().oracle_read_kv(self._h, layer, 1 if which == "V" else 0, pos0, n, _dp(out)))
        return out

    @property
    def position(self):
        return int(lib().oracle_position(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _o is not None:
            _o.oracle_free_session(self._h)
            self._h = None


def set_threads(n: int) -> None:
    lib().oracle_set_threads(n)


def rel_err(got, ref) -> float:
    """max over rows of max|d| / max|ref| (logits are ~1e-2 and
    nearly tied under the reference init, so per-element relative error is
    ill-conditioned)."""
    got = np.atleast_2d(np.asarray(got, dtype=np.float64))
    ref = np.atleast_2d(np.asarray(ref, dtype=np.float64))
    num = np.abs(got - ref).max(axis=1)
    den = np.abs(ref).max(axis=1)
    return float((num / np.maximum(den, 1e-300)).max())
