"""Build libdmv3d.so in-tree with nvcc for sm_100a (no torch, no JIT cache).

    python -m paper_2605_18052_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdmv3d.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]

SOURCES = ["api.cu", "render_simt.cu", "render_tc.cu", "elementwise.cu", "backward.cu", "backward_tc.cu"]
HEADERS = ["common.cuh", "kernels.h", "tc_ptx.cuh", "simt_common.cuh"]


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths if os.path.exists(p)), default=0)


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB,
          objdir: str = BUILD) -> str:
    """Compile csrc/*.cu for sm_100a into `lib`.  `defines` (e.g. ["DMV3D_PHASES"]) build an
    instrumented variant into its own object directory and library name."""
    os.makedirs(objdir, exist_ok=True)
    hdr_time = _newest([os.path.join(CSRC, h) for h in HEADERS] +
                       [os.path.join(ROOT, "include", "dmv3d.h")])
    objs, jobs = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
                os.path.getmtime(src), hdr_time):
            cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for cmd, r in zip(jobs, results):
            if verbose or r.returncode:
                sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError(f"nvcc failed for {cmd[-3]}")
    if force or jobs or not os.path.exists(lib):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart"]
        subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
