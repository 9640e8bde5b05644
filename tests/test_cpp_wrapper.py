"""Builds the C++ drop-in test program (tests/cpp/test_b200_api.cpp, written
like the reference's GTest suites) against include/vie_b200.hpp; runs it on
the GPU.  The compile check needs no GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "test_b200_api")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_exe():
    import __graft_entry__

    __graft_entry__.build()
    pkg = os.path.join(ROOT, "paper_1811_00484_b200")
    orc = os.path.join(ROOT, "oracle")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", os.path.join(ROOT, "tests", "cpp", "test_b200_api.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", orc, "-I", os.path.join(CUDA, "include"),
           "-L", pkg, "-lvie_b200", "-L", orc, "-loracle", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{orc}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}", "-o", EXE]
    subprocess.run(cmd, check=True)
    return EXE


def test_cpp_wrapper_compiles():
    assert os.path.exists(build_exe())


@pytest.mark.gpu
def test_cpp_wrapper_parity_on_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = build_exe()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") >= 25 and "FAIL" not in out.stdout
