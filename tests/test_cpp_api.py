"""Builds tests/cpp/test_dfa2_api.cpp against include/dfa2/*.hpp and
libdfa2_b200.so (the reference's C++ operator API, drop-in) and runs it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dfa2_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2503_22796_b200")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "test_dfa2_api")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
                    "-L", LIBDIR, "-ldfa2_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return out


def _run(binary, mode):
    r = subprocess.run([binary, mode], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cpp_api_host_cases(binary):
    _run(binary, "host")


@pytest.mark.gpu
def test_cpp_api_gpu_cases(binary):
    _run(binary, "gpu")
