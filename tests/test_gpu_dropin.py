"""The C++ drop-in header (include/esp/esp.hpp) compiled with g++ against
libesp_b200.so and run on the GPU: reference-style unit tests."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_dropin(esp, gpu, tmp_path):
    exe = tmp_path / "test_dropin"
    libdir = os.path.dirname(esp.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-L", libdir,
                    "-lesp_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
