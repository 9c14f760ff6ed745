"""The C-ABI from plain C (tests/c/capi_from_c.c): compiled with gcc against
include/dfa2c.h and libdfa2_b200.so only, then run on the GPU — the boundary
a cgo / JNI / N-API binding uses, exercised without C++ or torch."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def test_c_caller_runs_a_layer_through_the_c_abi(tmp_path):
    gcc = shutil.which("gcc")
    if not gcc:
        pytest.skip("gcc not found")
    lib = os.path.join(ROOT, "paper_2503_22796_b200")
    exe = tmp_path / "capi_from_c"
    subprocess.run([gcc, "-std=c99", "-O2", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
                    os.path.join(ROOT, "tests", "c", "capi_from_c.c"), "-L", lib, "-ldfa2_b200",
                    "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{lib}",
                    f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi from C ok" in r.stdout
