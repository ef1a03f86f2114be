"""In-tree build of libfsvd_b200.so (sm_100a) -- no JIT cache, no torch.

    python -m paper_2605_08314_b200.build [-v] [--force]

Host C++ (loader, normalizer, synthetic generator, C ABI) is compiled with
g++ -std=c++20; CUDA sources with nvcc -gencode arch=compute_100a,code=sm_100a
-lineinfo. The shared library lands next to this file so it travels to the GPU
box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libfsvd_b200.so"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def json_include_dir() -> Path:
    """nlohmann/json 3.11.3 -- the header the reference vendors (checkpoint.hpp:14)."""
    cands = [
        Path(sys.prefix) / "lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann",
        Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"),
    ]
    for c in cands:
        if (c / "json.hpp").exists():
            return c
    import glob

    hits = glob.glob(str(Path(sys.prefix) / "lib/python3*/site-packages/**/nlohmann/json.hpp"), recursive=True)
    if hits:
        return Path(hits[0]).parent
    raise RuntimeError("nlohmann json.hpp not found (needed by the FSVD15 header parser)")


HOST_SOURCES = ["host/model.cpp", "host/checkpoint.cpp", "host/canonical.cpp", "host/synth.cpp", "host/cpu_kernels.cpp",
                "capi/capi.cpp"]
CUDA_SOURCES = [
    "cuda/decode_mk.cu",
    "cuda/attention.cu",
    "cuda/attn_tc.cu",
    "cuda/gemm_simt.cu",
    "cuda/gemm_tc.cu",
    "cuda/gemm.cu",
    "cuda/misc.cu",
    "host/runtime.cu",
]
HEADERS = sorted(str(p) for p in list((CSRC).rglob("*.h")) + list(CSRC.rglob("*.cuh")) + list((ROOT / "include").rglob("*.h*")))


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    if src.stat().st_mtime > t:
        return True
    return any(Path(h).stat().st_mtime > t for h in HEADERS)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build step failed ({r.returncode}):\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr, flush=True)


def build(verbose: bool = False, force: bool = False) -> Path:
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    BUILD.mkdir(exist_ok=True)
    inc = ["-I", str(ROOT / "include"), "-I", str(json_include_dir()), "-I", str(CUDA_HOME / "include")]
    jobs = []
    objs = []
    for s in HOST_SOURCES:
        src = CSRC / s
        obj = BUILD / (s.replace("/", "_") + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            jobs.append(["g++", "-std=c++20", "-O3", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
                         "-Wno-unused-parameter", *inc, "-c", str(src), "-o", str(obj)])
    for s in CUDA_SOURCES:
        src = CSRC / s
        obj = BUILD / (s.replace("/", "_") + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            jobs.append([NVCC, *ARCH, "-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
                         "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr", *inc,
                         "-c", str(src), "-o", str(obj)])
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    if force or jobs or not LIB.exists():
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread", "-ldl", "-lrt"], verbose)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="--force" in sys.argv)
    print(LIB)
