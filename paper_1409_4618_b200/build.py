"""Build libefem.so in-tree with nvcc for sm_100a (no JIT cache).

The .so lives next to this file so it travels with the repo snapshot to the
GPU box and is the file the tests / bench / smoke load.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["mesh.cu", "dofs.cu", "assemble.cu", "api.cu", "fan2d.cu", "dist2d.cu", "part.cu", "integrate.cu", "p1.cu"]
LIB = os.path.join(HERE, "libefem.so")
BUILD_DIR = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

def _nccl_dir():
    """The NCCL that torch loads (the venv's nvidia-nccl wheel): libefem.so
    links the same libnccl.so.2, so one NCCL lives in the process."""
    try:
        import nvidia.nccl as m

        d = list(m.__path__)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    except Exception:
        pass
    raise RuntimeError("nccl.h / libnccl.so.2 not found (nvidia-nccl wheel)")


NCCL = _nccl_dir()
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xcompiler", "-fPIC",
         "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(NCCL, "include")]
LINK = ["-L" + os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "efem.h"))
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD_DIR, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC] + FLAGS + ["-c", s, "-o", o])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB] + objs + LINK)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
