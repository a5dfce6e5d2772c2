"""In-tree build of libdtb_b200.so for sm_100a (and nothing else).

-fmad=false plus explicit __dmul_rn/__dadd_rn keeps every product and sum
separately rounded, the reference's bitwise contract (kernel.py:3-11).
The translation units (one per kernel family and element type, the host
runtime, the planner) compile in parallel and link into one shared object.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libdtb_b200.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["dtb_resident_f64.cu", "dtb_resident_f32.cu", "dtb_pipe_f64.cu", "dtb_pipe_f32.cu",
           "dtb_stream.cu", "dtb_host.cu", "dtb_plan.cpp"]
HEADER = os.path.join(HERE, "..", "include", "dtb_b200.h")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def _deps() -> list[str]:
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [HEADER, __file__]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(d) > t for d in _deps() if os.path.exists(d))


def build_native(force: bool = False, verbose: bool = False, defines: tuple[str, ...] = (),
                 out: str | None = None) -> str:
    """Compile every translation unit (in parallel) and link the library.
    ``defines`` (e.g. ``("DTB_PIPE_PROBE=1",)``) and ``out`` build debug
    variants beside the product library."""
    target = out or OUT
    if out is None and not defines and not force and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    tag = "_".join(d.replace("=", "") for d in defines) or "product"
    objdir = os.path.join(OBJ, tag)
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src: str) -> str:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *dflags, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs,
           "-o", target + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    outp = next((a[6:] for a in sys.argv[1:] if a.startswith("--out=")), None)
    print(build_native(force="--force" in sys.argv, verbose=True, defines=defs, out=outp))
