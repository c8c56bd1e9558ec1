"""The C-ABI library loads without a GPU and exports every entry point that
include/fireiron_b200.h declares; errors map to anvil::ErrorKind ordinals."""
import ctypes as C
import os
import re
import subprocess

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "fireiron_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fi_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(fi):
    syms = declared_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", fi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fi_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(fi.lib, s)


def test_version_and_error_channel(fi):
    assert fi.lib.fi_version().decode().startswith("fireiron_b200")
    buf = C.create_string_buffer(256)
    n = fi.lib.fi_script_print(b"not a script", buf, 256)
    assert n == -22  # ParseError = ErrorKind ordinal 21 + 1
    assert "ParseError" in fi._native.last_error()


def test_plan_create_rejects_null(fi):
    h = C.c_void_p()
    assert fi.lib.fi_plan_create(None, 0, 0, 0, 0, 0, C.byref(h)) == 104


def test_plan_create_reports_invalid_tree_kind(fi):
    h = C.c_void_p()
    rc = fi.lib.fi_plan_create(b"spec MatMul(64,64,8)(GL,GL,GL)(Kernel)\ndone\n", 0, 0, 0, 0, 0, C.byref(h))
    assert rc == 23  # InvalidTree: lowering an invalid tree (program.hpp:631-632)
    assert "NoExecutableMatch" in fi._native.last_error()


def test_status_names(fi):
    from paper_2003_06324_b200._native import status_name
    assert status_name(1) == "ZeroDim" and status_name(24) == "IoError" and status_name(101) == "NvrtcError"


def test_library_has_no_link_time_cuda_driver_dependency(fi):
    out = subprocess.run(["ldd", fi.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcuda.so" not in out and "libnvrtc" not in out
