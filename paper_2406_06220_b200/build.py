"""Build the C-ABI shared library `libll.so` in-tree for sm_100a.

    python -m paper_2406_06220_b200.build          # nvcc, a few tens of seconds

The library is plain CUDA C++ (no torch headers); the Python binding loads it
with ctypes.  Flags: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libll.so")
SOURCES = [os.path.join(HERE, "csrc", "ll_api.cu"), os.path.join(HERE, "csrc", "ll_gather.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("common.cuh", "linear.cuh", "decode.cuh", "gemm_tc.cuh")] + \
    [os.path.join(ROOT, "include", "ll.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-ldl"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    """Build libll.so; variant="timeline" builds libll_timeline.so with the
    per-warp clock64 timeline hooks compiled in (tools/timeline.py)."""
    lib = LIB if not variant else os.path.join(HERE, f"libll_{variant}.so")
    if not force and os.path.exists(lib) and not any(os.path.getmtime(d) > os.path.getmtime(lib) for d in DEPS):
        return lib
    defs = {"": [], "timeline": ["-DLL_TIMELINE"], "trace": ["-DLL_DEBUG_TRACE"]}.get(variant)
    if defs is None:   # experiment variants: "timeline_exp1" -> -DLL_TIMELINE -DLL_EXP1
        defs = ["-DLL_" + v.upper() for v in variant.split("_")]
    tmp = f"{lib}.tmp{os.getpid()}"   # per process: concurrent ranks may build at once; os.replace is atomic
    cmd = [NVCC] + FLAGS + defs + ["-I", os.path.join(ROOT, "include"), "-o", tmp] + SOURCES
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libll.so")
    if verbose:
        sys.stderr.write(r.stderr)
    if not variant:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
            fh.write(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
