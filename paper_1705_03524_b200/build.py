"""Compile libswg.so (the sm_100a kernels + C-ABI) in-tree.

    python -m paper_1705_03524_b200.build [--verbose]

nvcc cross-compiles for sm_100a without a GPU.  The library is written to
paper_1705_03524_b200/lib/libswg.so (git-ignored; gpurun ships it to the GPU
box).  -fmad=false keeps every fp64 multiply and add separately rounded, as
the reference's SSE2 build does.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libswg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["swg_abi.cu", "k_build.cu", "k_sweep.cu", "k_stream.cu", "k_brute.cu", "k_decay.cu", "k_exp.cu"]
HEADERS = ["swg_internal.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "-Xcompiler", "-fPIC,-O2",
    "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


CPP_DIR = os.path.join(PKG, "cpp")
CPP_SOURCES = ["core.cpp", "tables.cpp", "engine.cpp", "matching.cpp", "pgm.cpp", "bench.cpp"]
CPP_LIB = os.path.join(LIBDIR, "libswih_b200.so")
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra",
             "-I" + os.path.join(ROOT, "include"), "-I" + CPP_DIR]


def build_cpp(verbose: bool = False, force: bool = False) -> str:
    """The reference-compatible C++ API (include/swih/*.hpp) over libswg."""
    build(verbose, force)
    hdrs = [os.path.join(ROOT, "include", "swih", h)
            for h in os.listdir(os.path.join(ROOT, "include", "swih"))]
    srcs = [os.path.join(CPP_DIR, s) for s in CPP_SOURCES] + [os.path.join(CPP_DIR, "runtime.hpp")]
    if force or _stale(CPP_LIB, srcs + hdrs + [LIB]):
        cmd = [CXX, *CXX_FLAGS, "-shared", *[os.path.join(CPP_DIR, s) for s in CPP_SOURCES],
               "-o", CPP_LIB, "-L" + LIBDIR, "-lswg", "-Wl,-rpath,$ORIGIN"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return CPP_LIB


def build_cpp_tests(verbose: bool = False) -> str:
    """tests/cpp/test_api.cpp against libswih_b200.so (binary in tests/cpp/build)."""
    build_cpp(verbose)
    tdir = os.path.join(ROOT, "tests", "cpp")
    out = os.path.join(tdir, "build", "test_api")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    deps = [os.path.join(tdir, "test_api.cpp"), os.path.join(tdir, "minitest.hpp"), CPP_LIB]
    if _stale(out, deps):
        cmd = [CXX, *CXX_FLAGS, os.path.join(tdir, "test_api.cpp"), "-o", out,
               "-L" + LIBDIR, "-lswih_b200", "-lswg", "-Wl,-rpath," + LIBDIR, "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    tool = os.path.join(tdir, "build", "io_tool")
    if _stale(tool, [os.path.join(tdir, "io_tool.cpp"), CPP_LIB]):
        subprocess.run([CXX, *CXX_FLAGS, os.path.join(tdir, "io_tool.cpp"), "-o", tool,
                        "-L" + LIBDIR, "-lswih_b200", "-lswg", "-Wl,-rpath," + LIBDIR,
                        "-lpthread"], check=True)
    return out


def build(verbose: bool = False, force: bool = False, variant: str = "",
          defines=()) -> str:
    """variant/defines: an A/B build (lib/libswg_<variant>.so, -D flags)."""
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(PKG, "build" + ("_" + variant if variant else ""))
    os.makedirs(objdir, exist_ok=True)
    deps_common = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "swg.h")]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + deps_common):
            cmd = [NVCC, *NVCC_FLAGS, *["-D" + d for d in defines], "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    lib = LIB if not variant else os.path.join(LIBDIR, f"libswg_{variant}.so")
    if force or _stale(lib, objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib,
               "-Xcompiler", "-fPIC"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    build_cpp(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    if "--tests" in sys.argv:
        print(build_cpp_tests(verbose="--verbose" in sys.argv))
    print(LIB)
    print(CPP_LIB)
