"""The C++ drop-in mirror (include/groot_aigsage.hpp) compiled and run like a
reference user's program: host-only checks on CPU, the full device pipeline on GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_aigsage_api.cpp")
PKG = os.path.join(ROOT, "paper_2511_18297_b200")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    from paper_2511_18297_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2511_18297_b200 import build
        build.build()
    out = str(tmp_path_factory.mktemp("cpp") / "test_api")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", SRC,
           "-L", PKG, "-lgroot_b200", f"-Wl,-rpath,{PKG}", "-o", out]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return out


def test_cpp_api_host(binary):
    res = subprocess.run([binary], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr + res.stdout
    assert "host checks ok" in res.stdout


@pytest.mark.gpu
def test_cpp_api_device(binary):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    res = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr + res.stdout
    assert "device checks ok" in res.stdout
