"""Builds the in-tree native library (no JIT cache; the .so travels with the repo).

    python -m paper_2503_22796_b200.build

Produces paper_2503_22796_b200/libdfa2_b200.so: the sm_100a kernels
(tcgen05 / TMA / TMEM), the C-ABI of include/dfa2c.h and the host C++
dfa2:: API of include/dfa2/ (csrc/host/), with the CUDA runtime linked
statically so the library is self-contained for ctypes / cgo / JNI callers.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdfa2_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["attn_sm100.cu", "rse_sm100.cu", "convert_sm100.cu", "reference_sm100.cu", "workload_sm100.cu"]
CPP_SOURCES = ["dfa2c.cpp", "json_lite.cpp", "plansolver.cpp", "nccl_dl.cpp", "workload_dev.cpp"]


def _sources():
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES + CPP_SOURCES]
    host = os.path.join(CSRC, "host")
    if os.path.isdir(host):
        srcs += sorted(os.path.join(host, f) for f in os.listdir(host) if f.endswith(".cpp"))
    return srcs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    deps = _sources()
    for d in (CSRC, os.path.join(ROOT, "include"), os.path.join(ROOT, "include", "dfa2")):
        if os.path.isdir(d):
            deps += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".h", ".cuh", ".hpp"))]
    if not force and not _stale(out, deps):
        return out
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++20", "-shared", "-cudart", "static",
           "-Xcompiler", "-fPIC,-fvisibility=hidden,-fvisibility-inlines-hidden", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *[f"-D{d}" for d in defines], "-o", out + ".tmp", *_sources(), "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


CLI = os.path.join(HERE, "bin", "dfa2")
CLI_SOURCES = [os.path.join(CSRC, "cli", "dfa2_main.cpp"), os.path.join(CSRC, "json_lite.cpp")]


def build_cli(force: bool = False) -> str:
    """The `dfa2` command-line front end (calibrate | run | verify | bench |
    workload, the reference CLI's subcommands) linked against libdfa2_b200.so."""
    deps = CLI_SOURCES + [LIB, os.path.join(CSRC, "json_lite.h")]
    inc = os.path.join(ROOT, "include", "dfa2")
    deps += [os.path.join(inc, f) for f in os.listdir(inc)]
    if not force and not _stale(CLI, deps):
        return CLI
    os.makedirs(os.path.dirname(CLI), exist_ok=True)
    cmd = [os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *CLI_SOURCES, "-o", CLI + ".tmp", "-L", HERE, "-ldfa2_b200", "-Wl,-rpath,$ORIGIN/.."]
    subprocess.run(cmd, check=True)
    os.replace(CLI + ".tmp", CLI)
    return CLI


def build_tools(force: bool = False) -> str:
    """tools/cpp_api_bench_bin: times the C++ drop-in dfa2::multi_strategy_attention
    with host f32 tensors (the reference's calling convention; bench.py's
    e2e_cpp_f32)."""
    src = os.path.join(ROOT, "tools", "cpp_api_bench.cpp")
    exe = os.path.join(ROOT, "tools", "cpp_api_bench_bin")
    inc = os.path.join(ROOT, "include", "dfa2")
    deps = [src, LIB] + [os.path.join(inc, f) for f in os.listdir(inc)]
    if not force and not _stale(exe, deps):
        return exe
    cmd = [os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o",
           exe + ".tmp", "-L", HERE, "-ldfa2_b200", "-Wl,-rpath,$ORIGIN/../paper_2503_22796_b200"]
    subprocess.run(cmd, check=True)
    os.replace(exe + ".tmp", exe)
    return exe


if __name__ == "__main__":
    # python -m paper_2503_22796_b200.build [--force] [-v] [--out PATH] [-DNAME=VAL ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else LIB
    defs = [a[2:] for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv or bool(defs), verbose="-v" in argv, out=out, defines=defs))
    if out == LIB:
        print(build_cli(force="--force" in argv))
