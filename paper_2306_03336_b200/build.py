"""In-tree build of libdtb_b200.so for sm_100a (and nothing else).

-fmad=false plus explicit __dmul_rn/__dadd_rn keeps every product and sum
separately rounded, the reference's bitwise contract (kernel.py:3-11).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libdtb_b200.so")
SOURCES = ["dtb_kernels.cu", "dtb_plan.cpp"]
HEADERS = ["dtb_core.cuh", "dtb_pipe.cuh", "dtb_plan.h",
           os.path.join("..", "..", "include", "dtb_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    deps += [os.path.join(CSRC, f) for f in os.listdir(CSRC)]  # any csrc file
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_native(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *[os.path.join(CSRC, s) for s in SOURCES], "-o", OUT + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose=True))
