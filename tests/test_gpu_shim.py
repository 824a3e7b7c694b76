"""The drop-in C++ shim (include/commdet/gpu.hpp) run by a reference-style
caller (tests/cpp/shim_kat.cpp, built by `make shim`)."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

pytestmark = pytest.mark.gpu


def test_cpp_shim_kats(tmp_path):
    # always compiled against the current headers (a stale binary would
    # disagree with the C ABI's struct layouts); same recipe as `make shim`
    exe = str(tmp_path / "shim_kat")
    lib_dir = os.path.join(ROOT, "paper_1304_4453_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_kat.cpp"), "-o", exe, "-L" + lib_dir,
                    "-lcommdet_cuda", "-Wl,-rpath," + lib_dir], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
