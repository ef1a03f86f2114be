"""The C-ABI boundary (include/fsvd_c.h) without a GPU: the library loads,
exports every declared entry point, and maps errors to the reference's
exception types (tensor.hpp:17-31, checkpoint.hpp:21, canonical.hpp:21)."""
import re
import subprocess

import pytest

from conftest import ROOT


def declared():
    hdr = (ROOT / "include" / "fsvd_c.h").read_text()
    return sorted(set(re.findall(r"\b(fsvd_[a-z0-9_]+)\s*\(", hdr)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("fsvd_model_load", "fsvd_session_create", "fsvd_prefill", "fsvd_decode_step", "fsvd_generate",
                 "fsvd_canonical_load_file", "fsvd_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(fsvd):
    lib = fsvd.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    assert set(fsvd.exported_symbols()) <= exported
    # no torch in the boundary
    dyn = subprocess.run(["readelf", "-d", str(lib)], capture_output=True, text=True, check=True).stdout
    assert "torch" not in dyn and "c10" not in dyn


def test_binding_covers_header(fsvd):
    assert sorted(fsvd.exported_symbols()) == declared()


def test_errors_cross_the_boundary_as_status(fsvd):
    import ctypes as C

    L = fsvd.lib()
    h = C.c_void_p()
    st = L.fsvd_canonical_load_file(b"/nonexistent/file.fsvd", C.byref(h))
    assert st == fsvd.FormatError.status
    assert b"nonexistent" in L.fsvd_last_error()
    assert L.fsvd_prefill(None, None, 1, None) == fsvd.InvalidArgument.status
    with pytest.raises(fsvd.InvalidArgument):
        fsvd._check(L.fsvd_session_reset(None))
    assert fsvd.lib().fsvd_version()


def test_cpp_wrapper_rethrows_reference_exceptions(fsvd, tmp_path):
    """include/fsvd/runtime.hpp: C++ callers keep catch (fsvd::FormatError&)."""
    exe = tmp_path / "wrapper_check"
    cmd = ["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), str(ROOT / "tests/cpp/wrapper_check.cpp"),
           "-o", str(exe), "-L", str(fsvd.LIB_PATH.parent), "-lfsvd_b200",
           f"-Wl,-rpath,{fsvd.LIB_PATH.parent}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def test_cpu_operator_api_matches_reference_golden(fsvd, tmp_path):
    """include/fsvd/kernels.hpp + math.hpp (the reference's kern::Ops registry
    and math layer, kernels.hpp:18-62 / math.hpp:16-140) compile against this
    tree, link to libfsvd_b200.so, and reproduce the reference's own scalar
    outputs bit for bit (tests/golden/primitives.json)."""
    from paper_2605_08314_b200.build import json_include_dir

    exe = tmp_path / "cpu_ops_check"
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", str(ROOT / "include"), "-I", str(json_include_dir()),
           str(ROOT / "tests/cpp/cpu_ops_check.cpp"), "-o", str(exe), "-L", str(fsvd.LIB_PATH.parent), "-lfsvd_b200",
           f"-Wl,-rpath,{fsvd.LIB_PATH.parent}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe), str(ROOT / "tests/golden/primitives.json")], capture_output=True, text=True)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
