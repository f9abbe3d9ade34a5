"""Builds the in-tree shared library libnegf_b200.so (host plan C++ + sm_100a
CUDA kernels + C ABI) with nvcc.  The .so lives next to this file so it
travels with the repository snapshot to the GPU box."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnegf_b200.so")
OBJDIR = os.path.join(ROOT, "build", "negf_b200")
SOURCES = ["tree.cpp", "plan.cpp", "kernels.cu", "capi.cu", "lead.cu", "output.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O3", f"-I{os.path.join(ROOT, 'include')}"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".hpp")]
    headers.append(os.path.join(ROOT, "include", "negf_gpu.h"))
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJDIR, src + ".o")
        objs.append(o)
        if _newer(o, [s] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
            if verbose and src.endswith(".cu"):
                cmd.insert(1, "-Xptxas=-v")
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
    if _newer(LIB, objs):
        # Static cudart: the library brings its own runtime and shares the
        # device's primary context with torch through the driver.
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl", "-lpthread", "-lrt"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    build_example(verbose)
    return LIB


EXAMPLE_SRC = os.path.join(ROOT, "examples", "negf_solve.cpp")
EXAMPLE_BIN = os.path.join(ROOT, "examples", "negf_solve")


def build_example(verbose: bool = False) -> str:
    """The C++ host program on the C ABI alone (examples/negf_solve.cpp)."""
    if os.path.exists(EXAMPLE_SRC) and _newer(EXAMPLE_BIN, [EXAMPLE_SRC, LIB, os.path.join(ROOT, "include", "negf_gpu.h")]):
        cmd = [os.environ.get("CXX", "g++"), "-std=c++17", "-O2", "-Wall", f"-I{os.path.join(ROOT, 'include')}",
               EXAMPLE_SRC, f"-L{HERE}", "-lnegf_b200", "-Wl,-rpath,$ORIGIN/../paper_1305_1070_b200",
               "-o", EXAMPLE_BIN]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return EXAMPLE_BIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
