"""In-tree build of the CUDA library (sm_100a) -- `python -m paper_2105_01827_b200.build`."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "gala_lib.cu")
OUT = os.path.join(HERE, "_lib", "libgala_b200.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("gala_lib.cu", "gala_kernels.cuh", "gala_device.cuh")] + [
    os.path.join(HERE, "..", "include", "gala_b200.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


CUDA_LIB = "/usr/local/cuda/lib64"
LINK = ["-L" + CUDA_LIB, "-Xlinker", "-rpath=" + CUDA_LIB]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    extra = os.environ.get("GALA_NVCC_EXTRA", "").split()   # experiments only (e.g. -DGTC_PROF)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", OUT, SRC, *LINK]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
