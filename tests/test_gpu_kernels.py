"""Kernel-level GPU checks of the round-2 kernels, through the product library
(libfsvd_b200.so) and small CUDA drivers under tools/:

* tcgen05 prefill flash attention (attn_tc.cu) against an fp64 reference over
  history offsets, batch, d_head 64 / 128 and NaN-poisoned cache rows past the
  history (tools/attn_check.cu);
* the cluster split-K (K splits of one tile reduced through DSMEM inside the
  GEMM) bitwise against the reduction-kernel path at equal splits, for the
  decode-sized swap GEMM (M = 16) and the M = 512 prefill tiles incl. CTA pairs
  (tools/gemm_sweep.cu modes cred / cred512)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

NVCC = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
LIB = ROOT / "paper_2605_08314_b200"


def _build(src, out):
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++20", "-I", str(ROOT / "include"),
           str(ROOT / "tools" / src), "-o", str(out), "-L", str(LIB), "-lfsvd_b200", f"-Xlinker", f"-rpath={LIB}"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr


def test_attn_tcgen05_vs_fp64(tmp_path):
    exe = tmp_path / "attn_check"
    _build("attn_check.cu", exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "all ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("m,mode", [(16, "cred"), (512, "cred512")])
def test_cluster_split_k_bitwise(tmp_path, m, mode):
    exe = tmp_path / "gemm_sweep"
    _build("gemm_sweep.cu", exe)
    r = subprocess.run([str(exe), str(m), "8" if mode == "cred" else "4", mode], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    checks = [l for l in r.stdout.splitlines() if l.startswith("PAIRCHECK")]
    print("\n".join(checks))
    assert len(checks) >= 8
    assert all(l.endswith("bitwise") for l in checks), [l for l in checks if not l.endswith("bitwise")]
    assert "error" not in r.stdout.lower()
