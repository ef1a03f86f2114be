"""B200-native FlashSVD runtime -- Python host mirror of the reference API.

The product is libfsvd_b200.so (sm_100a kernels + C++ loader/runtime behind
the C ABI in include/fsvd_c.h). This module is a thin ctypes binding that
mirrors the reference's names and error behaviour (proj/include/fsvd/*.hpp,
SPEC.md runtime :283-382) so tests and the benchmark read like the
reference's own: ``prefill(tokens) -> logits``, ``decode_step(token) ->
logits``, ``generate(prompt, max_new) -> tokens``, typed errors
``CapacityError``/``ShapeError``/``FormatError``/...

There is no fallback: if the shared library is missing this module raises on
first use.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libfsvd_b200.so"

# ----------------------------------------------------------------- errors --


class FsvdError(RuntimeError):
    status = 12


class ShapeError(FsvdError):  # tensor.hpp:17
    status = 1


class RankError(FsvdError):
    status = 2


class NumericError(FsvdError):
    status = 3


class CapacityError(FsvdError):  # tensor.hpp:26
    status = 4


class ConfigError(FsvdError):
    status = 5


class FormatError(FsvdError):  # checkpoint.hpp:21
    status = 6


class NormalizeError(FsvdError):  # canonical.hpp:21
    status = 7


class CalibrationError(FsvdError):
    status = 8


class CudaError(FsvdError):
    status = 9


class OutOfMemoryError(FsvdError):
    status = 10


class InvalidArgument(FsvdError):
    status = 11


_ERRORS = {e.status: e for e in (ShapeError, RankError, NumericError, CapacityError, ConfigError, FormatError,
                                 NormalizeError, CalibrationError, CudaError, OutOfMemoryError, InvalidArgument)}

# ------------------------------------------------------------------ enums --
DTYPE = {"f32": 0, "fp32": 0, "float32": 0, "bf16": 1, "bfloat16": 1}
FFN = {"auto": 0, "no_merge": 1, "packed": 2}
PLAN = {"eager": 0, "per_layer": 1, "full_step": 2, "split": 3}
ATTN = {"dense_kv": 0, "lowrank_history": 1}
FFN_NAMES = {v: k for k, v in FFN.items()}
PLAN_NAMES = {v: k for k, v in PLAN.items()}
PROJ = ("q", "k", "v", "o", "up", "gate", "down")


class _Config(C.Structure):
    _fields_ = [("n_layers", C.c_uint64), ("d_model", C.c_uint64), ("n_heads", C.c_uint64), ("d_head", C.c_uint64),
                ("d_ff", C.c_uint64), ("vocab", C.c_uint64), ("rope_base", C.c_double), ("norm_eps", C.c_double)]


class _Synth(C.Structure):
    _fields_ = [("config", _Config), ("capacity", C.c_uint64), ("family", C.c_char), ("rho", C.c_double),
                ("group_size", C.c_uint64), ("seed", C.c_uint64), ("conditioned", C.c_int32),
                ("rank_jitter", C.c_double)]


class _Opts(C.Structure):
    _fields_ = [("batch", C.c_uint32), ("capacity", C.c_uint64), ("ffn", C.c_int), ("plan", C.c_int),
                ("attn_route", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("dispatches", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("graph_launches", C.c_uint64), ("allocs", C.c_uint64), ("copy_bytes", C.c_uint64),
                ("last_dispatches", C.c_uint64), ("recon_flops", C.c_uint64)]


@dataclass(frozen=True)
class ModelConfig:
    """reference proj/include/fsvd/model.hpp:18-29"""
    n_layers: int
    d_model: int
    n_heads: int
    d_head: int
    d_ff: int
    vocab: int
    rope_base: float = 10000.0
    norm_eps: float = 1e-5

    def _c(self) -> _Config:
        return _Config(self.n_layers, self.d_model, self.n_heads, self.d_head, self.d_ff, self.vocab, self.rope_base,
                       self.norm_eps)

    @staticmethod
    def _from(c: _Config) -> "ModelConfig":
        return ModelConfig(c.n_layers, c.d_model, c.n_heads, c.d_head, c.d_ff, c.vocab, c.rope_base, c.norm_eps)


PRESETS = {
    "desk": (ModelConfig(4, 256, 8, 32, 1024, 1024), 8192),
    "bench": (ModelConfig(8, 512, 8, 64, 2048, 4096), 8192),
    "tiny": (ModelConfig(4, 256, 4, 64, 1024, 1024), 8192),
    "llama7b": (ModelConfig(32, 4096, 32, 128, 11008, 32000), 8192),
    "llama13b": (ModelConfig(40, 5120, 40, 128, 13824, 32000), 8192),
}


@dataclass
class SynthSpec:
    """include/fsvd/synth.hpp SynthSpec"""
    config: ModelConfig
    capacity: int = 8192
    family: str = "A"
    rho: float = 0.6
    group_size: int = 2
    seed: int = 1
    conditioned: bool = False
    rank_jitter: float = 0.0

    def _c(self) -> _Synth:
        return _Synth(self.config._c(), self.capacity, self.family.encode(), self.rho, self.group_size, self.seed,
                      1 if self.conditioned else 0, self.rank_jitter)


# ---------------------------------------------------------------- library --
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2605_08314_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, u64, i32, f32p, i32p = C.c_void_p, C.c_uint64, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_int32)
    sig = {
        "fsvd_last_error": ([], C.c_char_p),
        "fsvd_version": ([], C.c_char_p),
        "fsvd_canonical_load_file": ([C.c_char_p, C.POINTER(vp)], C.c_int),
        "fsvd_canonical_load_bytes": ([C.c_char_p, C.c_size_t, C.POINTER(vp)], C.c_int),
        "fsvd_canonical_synthetic": ([C.POINTER(_Synth), C.POINTER(vp)], C.c_int),
        "fsvd_canonical_config": ([vp, C.POINTER(_Config), C.POINTER(u64)], C.c_int),
        "fsvd_canonical_rank": ([vp, u64, C.c_uint32, C.POINTER(u64)], C.c_int),
        "fsvd_canonical_copy": ([vp, C.c_char_p, f32p, u64], C.c_int),
        "fsvd_canonical_shared_count": ([vp, C.POINTER(u64)], C.c_int),
        "fsvd_canonical_aliased": ([vp, u64, u64, C.c_uint32, i32p], C.c_int),
        "fsvd_canonical_destroy": ([vp], C.c_int),
        "fsvd_synthetic_write_file": ([C.POINTER(_Synth), C.c_char_p], C.c_int),
        "fsvd_canonical_write_file": ([vp, C.c_char_p], C.c_int),
        "fsvd_model_load": ([C.c_char_p, C.c_int, i32, C.POINTER(vp)], C.c_int),
        "fsvd_last_load_stats": ([C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], C.c_int),
        "fsvd_model_from_canonical": ([vp, C.c_int, i32, C.POINTER(vp)], C.c_int),
        "fsvd_model_synthetic": ([C.POINTER(_Synth), C.c_int, i32, C.POINTER(vp)], C.c_int),
        "fsvd_model_info": ([vp, C.POINTER(_Config), C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)], C.c_int),
        "fsvd_model_copy_factor": ([vp, u64, C.c_uint32, i32, f32p, u64], C.c_int),
        "fsvd_model_destroy": ([vp], C.c_int),
        "fsvd_route_ffn_auto": ([C.c_int, C.c_int, C.POINTER(C.c_int)], C.c_int),
        "fsvd_session_create": ([vp, C.POINTER(_Opts), C.POINTER(vp)], C.c_int),
        "fsvd_prefill": ([vp, i32p, u64, f32p], C.c_int),
        "fsvd_decode_step": ([vp, i32p, f32p], C.c_int),
        "fsvd_generate": ([vp, i32p, u64, u64, i32p], C.c_int),
        "fsvd_prefill_device": ([vp, vp, u64, vp], C.c_int),
        "fsvd_decode_step_device": ([vp, vp, vp], C.c_int),
        "fsvd_decode_steps_device": ([vp, C.c_uint64, vp], C.c_int),
        "fsvd_generate_device": ([vp, vp, u64, u64, vp], C.c_int),
        "fsvd_session_sync": ([vp], C.c_int),
        "fsvd_session_stream": ([vp, C.POINTER(vp)], C.c_int),
        "fsvd_session_position": ([vp, C.POINTER(u64)], C.c_int),
        "fsvd_session_reset": ([vp], C.c_int),
        "fsvd_session_stats": ([vp, C.POINTER(_Stats)], C.c_int),
        "fsvd_session_resolved": ([vp, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
        "fsvd_session_read_kv": ([vp, u64, u64, i32, u64, u64, f32p], C.c_int),
        "fsvd_session_engine": ([vp, i32p, i32p, i32p, i32p], C.c_int),
        "fsvd_session_trace": ([vp, C.POINTER(u64), u64, i32p, i32p], C.c_int),
        "fsvd_session_destroy": ([vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def exported_symbols() -> list[str]:
    return ["fsvd_last_error", "fsvd_version", "fsvd_canonical_load_file", "fsvd_canonical_load_bytes",
            "fsvd_canonical_synthetic", "fsvd_canonical_config", "fsvd_canonical_rank", "fsvd_canonical_copy",
            "fsvd_canonical_shared_count", "fsvd_canonical_aliased", "fsvd_canonical_destroy",
            "fsvd_canonical_write_file", "fsvd_synthetic_write_file", "fsvd_model_load", "fsvd_last_load_stats", "fsvd_model_from_canonical",
            "fsvd_model_synthetic",
            "fsvd_model_info", "fsvd_model_copy_factor", "fsvd_model_destroy", "fsvd_route_ffn_auto",
            "fsvd_session_create", "fsvd_prefill", "fsvd_decode_step", "fsvd_generate", "fsvd_prefill_device",
            "fsvd_decode_step_device", "fsvd_decode_steps_device", "fsvd_generate_device", "fsvd_session_sync", "fsvd_session_stream",
            "fsvd_session_position", "fsvd_session_reset", "fsvd_session_stats", "fsvd_session_resolved",
            "fsvd_session_read_kv", "fsvd_session_engine", "fsvd_session_trace", "fsvd_session_destroy"]


def _check(status: int) -> None:
    if status != 0:
        msg = lib().fsvd_last_error().decode(errors="replace")
        raise _ERRORS.get(status, FsvdError)(msg)


def _f32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def route_ffn_auto(plan: str, ffn: str = "auto") -> str:
    """SPEC.md:419-427 route_ffn_auto(plan_mode) with explicit override precedence."""
    out = C.c_int()
    _check(lib().fsvd_route_ffn_auto(PLAN[plan], FFN[ffn], C.byref(out)))
    return FFN_NAMES[out.value]


# ------------------------------------------------------ host canonical model --
class Canonical:
    """Host CanonicalModel<float> from read_checkpoint_file -> normalize<float>."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def load_file(cls, path) -> "Canonical":
        h = C.c_void_p()
        _check(lib().fsvd_canonical_load_file(str(path).encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def load_bytes(cls, data: bytes) -> "Canonical":
        h = C.c_void_p()
        _check(lib().fsvd_canonical_load_bytes(data, len(data), C.byref(h)))
        return cls(h)

    @classmethod
    def synthetic(cls, spec: SynthSpec) -> "Canonical":
        h = C.c_void_p()
        s = spec._c()
        _check(lib().fsvd_canonical_synthetic(C.byref(s), C.byref(h)))
        return cls(h)

    @property
    def config(self) -> ModelConfig:
        c, cap = _Config(), C.c_uint64()
        _check(lib().fsvd_canonical_config(self._h, C.byref(c), C.byref(cap)))
        return ModelConfig._from(c)

    @property
    def capacity(self) -> int:
        c, cap = _Config(), C.c_uint64()
        _check(lib().fsvd_canonical_config(self._h, C.byref(c), C.byref(cap)))
        return cap.value

    def rank(self, layer: int, proj) -> int:
        p = PROJ.index(proj) if isinstance(proj, str) else proj
        r = C.c_uint64()
        _check(lib().fsvd_canonical_rank(self._h, layer, p, C.byref(r)))
        return r.value

    def tensor(self, name: str, shape) -> np.ndarray:
        out = np.empty(shape, dtype=np.float32)
        _check(lib().fsvd_canonical_copy(self._h, name.encode(), _f32p(out), out.size))
        return out

    def write_file(self, path) -> None:
        """Normalized model -> family-A FSVD15 file (canonical.cpp export_family_a)."""
        _check(lib().fsvd_canonical_write_file(self._h, str(path).encode()))

    def shared_count(self) -> int:
        n = C.c_uint64()
        _check(lib().fsvd_canonical_shared_count(self._h, C.byref(n)))
        return n.value

    def aliased(self, l0: int, l1: int, proj) -> bool:
        p = PROJ.index(proj) if isinstance(proj, str) else proj
        o = C.c_int32()
        _check(lib().fsvd_canonical_aliased(self._h, l0, l1, p, C.byref(o)))
        return bool(o.value)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fsvd_canonical_destroy(self._h)
            self._h = None


def write_synthetic(spec: SynthSpec, path) -> None:
    s = spec._c()
    _check(lib().fsvd_synthetic_write_file(C.byref(s), str(path).encode()))


# ------------------------------------------------------------ device model --
class Model:
    """Device-resident model (immutable; backs any number of sessions)."""

    def __init__(self, handle, dtype: str):
        self._h = handle
        self.dtype = dtype

    @classmethod
    def load(cls, path, dtype: str = "bf16", device: int = 0) -> "Model":
        """FSVD15 file -> device (streaming loader; FSVD_LOADER=canonical: host normalize + upload)."""
        h = C.c_void_p()
        _check(lib().fsvd_model_load(str(path).encode(), DTYPE[dtype], device, C.byref(h)))
        return cls(h, dtype)

    @staticmethod
    def last_load_stats() -> dict:
        """seconds / payload bytes / pinned staging bytes of this thread's last Model.load."""
        sec, nb, pb = C.c_double(), C.c_uint64(), C.c_uint64()
        _check(lib().fsvd_last_load_stats(C.byref(sec), C.byref(nb), C.byref(pb)))
        return {"seconds": sec.value, "payload_bytes": nb.value, "pinned_bytes": pb.value}

    @classmethod
    def from_canonical(cls, canon: Canonical, dtype: str = "bf16", device: int = 0) -> "Model":
        h = C.c_void_p()
        _check(lib().fsvd_model_from_canonical(canon._h, DTYPE[dtype], device, C.byref(h)))
        return cls(h, dtype)

    @classmethod
    def synthetic(cls, spec: SynthSpec, dtype: str = "bf16", device: int = 0) -> "Model":
        h = C.c_void_p()
        s = spec._c()
        _check(lib().fsvd_model_synthetic(C.byref(s), DTYPE[dtype], device, C.byref(h)))
        return cls(h, dtype)

    def info(self) -> dict:
        c, cap, wb, db = _Config(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().fsvd_model_info(self._h, C.byref(c), C.byref(cap), C.byref(wb), C.byref(db)))
        return {"config": ModelConfig._from(c), "capacity": cap.value, "weight_bytes": wb.value,
                "decode_weight_bytes": db.value}

    @property
    def config(self) -> ModelConfig:
        return self.info()["config"]

    def factor(self, layer: int, proj, which: str, shape) -> np.ndarray:
        p = PROJ.index(proj) if isinstance(proj, str) else proj
        out = np.empty(shape, dtype=np.float32)
        _check(lib().fsvd_model_copy_factor(self._h, layer, p, 1 if which == "B" else 0, _f32p(out), out.size))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fsvd_model_destroy(self._h)
            self._h = None


@dataclass
class StepStats:
    """SPEC.md:299-302 StepStats (+ device counters)."""
    steps: int
    dispatches: int
    kernel_launches: int
    graph_launches: int
    allocs: int
    copy_bytes: int
    last_dispatches: int
    recon_flops: int = 0  # lowrank_history route: K/V reconstruction FLOPs


class Session:
    """SPEC.md:293-298 Session: KV cache + workspace + plans for `batch`
    independent sequences advanced in lock step on one GPU."""

    def __init__(self, model: Model, batch: int = 1, capacity: int = 0, ffn: str = "auto", plan: str = "eager",
                 attn_route: str = "dense_kv"):
        self.model = model
        self.batch = batch
        self._cfg = model.config
        h = C.c_void_p()
        o = _Opts(batch, capacity, FFN[ffn], PLAN[plan], ATTN[attn_route])
        _check(lib().fsvd_session_create(model._h, C.byref(o), C.byref(h)))
        self._h = h

    # -- SPEC.md:305 prefill(session, tokens) -> logits (last position)
    def prefill(self, tokens) -> np.ndarray:
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32).reshape(self.batch, -1))
        out = np.empty((self.batch, self._cfg.vocab), dtype=np.float32)
        _check(lib().fsvd_prefill(self._h, _i32p(t), t.shape[1], _f32p(out)))
        return out

    # -- SPEC.md:314 decode_step(session, token) -> logits
    def decode_step(self, tokens) -> np.ndarray:
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32).reshape(self.batch))
        out = np.empty((self.batch, self._cfg.vocab), dtype=np.float32)
        _check(lib().fsvd_decode_step(self._h, _i32p(t), _f32p(out)))
        return out

    # -- SPEC.md:341 generate(session, prompt, max_new) -> tokens
    def generate(self, prompt, max_new: int) -> np.ndarray:
        t = np.ascontiguousarray(np.asarray(prompt, dtype=np.int32).reshape(self.batch, -1))
        out = np.zeros((self.batch, max_new), dtype=np.int32)
        _check(lib().fsvd_generate(self._h, _i32p(t), t.shape[1], max_new, _i32p(out)))
        return out

    # device-pointer entry points (asynchronous on the session stream)
    def prefill_device(self, d_tokens: int, T: int, d_logits: int = 0) -> None:
        _check(lib().fsvd_prefill_device(self._h, C.c_void_p(d_tokens), T, C.c_void_p(d_logits or None)))

    def decode_step_device(self, d_tokens: int = 0, d_logits: int = 0) -> None:
        _check(lib().fsvd_decode_step_device(self._h, C.c_void_p(d_tokens or None), C.c_void_p(d_logits or None)))

    def decode_steps_device(self, n: int, d_out: int = 0) -> None:
        """n greedy decode steps on the device (megakernel: one launch per <= 256 steps)."""
        _check(lib().fsvd_decode_steps_device(self._h, n, C.c_void_p(d_out or None)))

    def generate_device(self, d_prompt: int, T: int, max_new: int, d_out: int) -> None:
        _check(lib().fsvd_generate_device(self._h, C.c_void_p(d_prompt), T, max_new, C.c_void_p(d_out)))

    def sync(self) -> None:
        _check(lib().fsvd_session_sync(self._h))

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(lib().fsvd_session_stream(self._h, C.byref(s)))
        return s.value or 0

    @property
    def position(self) -> int:
        p = C.c_uint64()
        _check(lib().fsvd_session_position(self._h, C.byref(p)))
        return p.value

    def reset(self) -> None:
        _check(lib().fsvd_session_reset(self._h))

    def stats(self) -> StepStats:
        s = _Stats()
        _check(lib().fsvd_session_stats(self._h, C.byref(s)))
        return StepStats(s.steps, s.dispatches, s.kernel_launches, s.graph_launches, s.allocs, s.copy_bytes,
                         s.last_dispatches, s.recon_flops)

    def resolved(self) -> tuple[str, str]:
        f, p = C.c_int(), C.c_int()
        _check(lib().fsvd_session_resolved(self._h, C.byref(f), C.byref(p)))
        return FFN_NAMES[f.value], PLAN_NAMES[p.value]

    def engine(self) -> dict:
        v = [C.c_int32() for _ in range(4)]
        _check(lib().fsvd_session_engine(self._h, *[C.byref(x) for x in v]))
        # kind 1: persistent decode megakernel (B <= 2); 2: batched layer engine
        return {"megakernel": v[0].value == 1, "batched": v[0].value == 2, "stage_bytes": v[1].value,
                "stages": v[2].value, "attn_splits": v[3].value}

    def trace(self, max_phases: int = 4096) -> np.ndarray:
        """[grid, phases, 8] ns stamps of the last traced full step (FSVD_TRACE=1)."""
        buf = np.zeros(148 * 2 * max_phases * 16 + 8192 * 4, dtype=np.uint64)
        ph, g = C.c_int32(), C.c_int32()
        _check(lib().fsvd_session_trace(self._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size,
                                        C.byref(ph), C.byref(g)))
        self.chunk_trace = buf[g.value * ph.value * 16: g.value * ph.value * 16 + 8192 * 4].reshape(8192, 4)
        return buf[: g.value * ph.value * 16].reshape(g.value, ph.value, 16)

    def read_kv(self, layer: int, b: int, which: str, pos0: int, npos: int) -> np.ndarray:
        out = np.empty((npos, self._cfg.d_model), dtype=np.float32)
        _check(lib().fsvd_session_read_kv(self._h, layer, b, 1 if which == "V" else 0, pos0, npos, _f32p(out)))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fsvd_session_destroy(self._h)
            self._h = None
