"""The drop-in C++ shim (include/commdet/gpu.hpp) run by a reference-style
caller (tests/cpp/shim_kat.cpp, built by `make shim`)."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

pytestmark = pytest.mark.gpu


def test_cpp_shim_kats():
    exe = os.path.join(ROOT, "build", "shim_kat")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "shim"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
