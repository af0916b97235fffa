"""Build libmgm.so in-tree for sm_100a (nvcc + g++; no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libmgm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler",
                  "-ffp-contract=off", "-Xptxas", "-v"]
SOURCES = [
    ("host_setup.cpp", ["g++", "-O3", "-ffp-contract=off", "-fPIC", "-std=c++17", "-pthread",
                        "-I/usr/local/cuda/include"]),
    ("setup_kernels.cu", [NVCC] + NVFLAGS + ["-fmad=false"]),
    ("mgm.cu", [NVCC] + NVFLAGS),
]


def _newer(src_paths, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in src_paths)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "mgm.h"))
    objs = []
    for src, cmd in SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _newer([sp] + headers, obj):
            full = cmd + ["-c", sp, "-o", obj]
            r = subprocess.run(full, capture_output=True, text=True)
            if verbose or r.returncode:
                sys.stderr.write(" ".join(full) + "\n" + r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError(f"compilation of {src} failed")
    if force or _newer(objs, LIB):
        tmp = LIB + ".tmp%d" % os.getpid()
        full = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lpthread", "-ldl"]
        r = subprocess.run(full, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(" ".join(full) + "\n" + r.stdout + r.stderr)
            raise RuntimeError("link of libmgm.so failed")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
