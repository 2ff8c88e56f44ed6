"""Build the in-tree C-ABI library ``_lib/libbatchsim_b200.so`` with nvcc for sm_100a.

No torch extension machinery: the product is a plain shared library whose ``extern "C"``
entry points are declared in ``include/batchsim_b200.h``; Python binds it with ctypes
(``_native.py``).  Parity-critical translation units (pose algebra, rasterizer setup) are
compiled with ``-fmad=false`` so their float arithmetic rounds like numpy's; the step
kernel may contract to FMA.

Usage: ``python -m paper_2410_00425_b200.build_native [--force] [-v]``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB_NAME = "libbatchsim_b200.so"
LIB_PATH = os.path.join(OUT_DIR, LIB_NAME)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
          "-I" + os.path.join(ROOT, "include")]
if os.environ.get("BS_PHASE_TIMING"):  # developer instrumentation build (tools/phase_timing.py)
    COMMON.append("-DBS_PHASE_TIMING")
# Per-file extra flags.  NOFMA: numpy-order arithmetic must not be contracted.
NOFMA = ["-fmad=false"]
SOURCES = {
    "pose.cu": NOFMA,
    "sim.cu": [],
    "step.cu": [],
    "raster.cu": NOFMA,
    "vision_ops.cu": NOFMA,
    "capi.cu": [],
}


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the batchsim-b200 CUDA library cannot be built")


def _deps_mtime() -> float:
    newest = os.path.getmtime(os.path.join(ROOT, "include", "batchsim_b200.h"))
    for f in os.listdir(CSRC):
        if f.endswith((".cuh", ".h")):
            newest = max(newest, os.path.getmtime(os.path.join(CSRC, f)))
    return newest


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source for sm_100a and link the shared library; returns its path."""
    nvcc = _nvcc()
    os.makedirs(OUT_DIR, exist_ok=True)
    hdr_time = _deps_mtime()
    sources = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    objs = []
    jobs = []
    for src in sources:
        spath = os.path.join(CSRC, src)
        obj = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
        objs.append(obj)
        stale = force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
            os.path.getmtime(spath), hdr_time)
        if stale:
            cmd = [nvcc, *ARCH, *COMMON, *SOURCES[src], "-c", spath, "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(run, jobs))
    newest_obj = max(os.path.getmtime(o) for o in objs)
    if force or jobs or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest_obj:
        tmp = LIB_PATH + ".tmp"
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
        run(cmd)
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
