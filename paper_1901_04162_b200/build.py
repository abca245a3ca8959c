"""In-tree build of libgk.so (sm_100a) with nvcc.

``python -m paper_1901_04162_b200.build`` compiles csrc/ into
paper_1901_04162_b200/libgk.so.  The .so is git-ignored but travels to the
GPU box with the gpurun snapshot; nothing is JIT-compiled at import time.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libgk.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler",
          "-ffp-contract=off", "-I", os.path.join(ROOT, "include")]

# build.cu must round exactly like the reference (no FMA contraction)
SOURCES = {
    "build.cu": ["-fmad=false"],
    "fill.cu": [],
    "fill_mo1.cu": [],
    "fill_mo3.cu": [],
    "fill_mo4.cu": [],
    "fill_mo6.cu": [],
    "fill_mo7.cu": [],
    "eval.cu": [],
    "abi.cu": [],
    "host.cpp": [],
    "edges.cu": [],
    "comm.cu": [],
}
HEADERS = ["gk_device.cuh", "gk_internal.h", "fill_kernels.cuh", "fill_sweep.cuh"]


def _newer(src_files, target) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(f) > t for f in src_files)


def _compile(name: str, extra: list[str], verbose: bool) -> str:
    src = os.path.join(CSRC, name)
    obj = os.path.join(OBJ, name + ".o")
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "gk", "gk.h")]
    if not _newer(deps, obj):
        return obj
    if name.endswith(".cpp"):
        cmd = [NVCC, "-x", "cu", *ARCH, *COMMON, *extra, "-c", src, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{r.stdout}\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda kv: _compile(kv[0], kv[1], verbose), SOURCES.items()))
    if _newer(objs, LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_cpp_test()
    build_tools()
    return LIB


CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_adapter.cpp")
CPP_TEST_BIN = os.path.join(OBJ, "test_adapter")


def build_cpp_test() -> str:
    """The C++ adapter test (include/gk/gk.hpp over libgk.so), host g++ only."""
    deps = [CPP_TEST_SRC, LIB, os.path.join(ROOT, "include", "gk", "gk.hpp")]
    if _newer(deps, CPP_TEST_BIN):
        cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), CPP_TEST_SRC,
               "-o", CPP_TEST_BIN, "-L", PKG, "-lgk", "-Wl,-rpath,$ORIGIN/.."]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed for test_adapter:\n{r.stderr}")
    return CPP_TEST_BIN


TOOL_SRC = os.path.join(PKG, "tools", "gk_sharded_fill.cpp")
TOOL_BIN = os.path.join(OBJ, "gk_sharded_fill")


def build_tools() -> str:
    """The C++ multi-GPU driver (tools/gk_sharded_fill.cpp): host g++ over the
    C ABI + the CUDA runtime, linked against libgk.so."""
    deps = [TOOL_SRC, LIB, os.path.join(ROOT, "include", "gk", "gk.h")]
    if _newer(deps, TOOL_BIN):
        cuda = os.path.dirname(os.path.dirname(os.path.realpath(NVCC)))
        cmd = ["g++", "-std=c++20", "-O2", "-pthread", "-I", os.path.join(ROOT, "include"),
               "-I", os.path.join(cuda, "include"), TOOL_SRC, "-o", TOOL_BIN, "-L", PKG, "-lgk",
               "-L", os.path.join(cuda, "lib64"), "-lcudart", "-Wl,-rpath,$ORIGIN/..",
               "-Wl,-rpath," + os.path.join(cuda, "lib64")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed for gk_sharded_fill:\n{r.stderr}")
    return TOOL_BIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
