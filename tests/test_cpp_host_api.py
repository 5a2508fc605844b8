"""The C++ host API (include/netsort_b200.hpp): compiled against the library
on CPU (host-side checks run here), run in full on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp")
BIN = os.path.join(ROOT, "build", "test_host_api")


def build_binary():
    from paper_2503_05934_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", SRC, "-o", BIN, "-L", libdir,
                    "-lnetsort_b200", f"-Wl,-rpath,{libdir}", "-L/usr/local/cuda/lib64",
                    "-lcudart"], check=True)
    return BIN


def test_cpp_host_api_builds_and_host_checks_pass():
    b = build_binary()
    out = subprocess.run([b, "--no-gpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_cpp_host_api_on_gpu():
    b = build_binary()
    out = subprocess.run([b], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASSED" in out.stdout
