"""The C++ host side over the C-ABI (include/wc4dvar_gpu.hpp): compile tests/cpp/test_cpp_api.cpp
with g++ against libwc4dvar_gpu.so (and the CPU oracle as its checker) and run it on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_api(tmp_path):
    exe = str(tmp_path / "test_cpp_api")
    libdir, orcdir = os.path.join(ROOT, "paper_2101_07249_b200"), os.path.join(ROOT, "oracle")
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp",
           "test_cpp_api.cpp"), "-L", libdir, "-lwc4dvar_gpu", "-L", orcdir, "-loracle",
           f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{orcdir}", "-o", exe]
    b = subprocess.run(cmd, capture_output=True, text=True)
    assert b.returncode == 0, b.stderr[-3000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "0 failed" in r.stdout
