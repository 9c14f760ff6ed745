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


def test_generate_is_bit_identical_to_reference(binary, tmp_path):
    """dfa2::generate (C++ drop-in) hashes to the same bytes as the
    reference's generate() on the same configs (tests/golden/
    gen_workload_golden.py), so pipelines and calibration runs see the
    reference's exact inputs."""
    import hashlib
    import json

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "workload_golden.json")))
    for g in gold:
        path = str(tmp_path / "w.bin")
        r = subprocess.run([binary, "dump-workload", *map(str, g["config"]), path], capture_output=True, timeout=600)
        assert r.returncode == 0, r.stderr
        assert hashlib.sha256(open(path, "rb").read()).hexdigest() == g["sha256"], g["config"]
