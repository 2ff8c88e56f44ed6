"""Build the in-tree C-ABI library ``_lib/libbatchsim_b200.so`` with nvcc for sm_100a.

No torch extension machinery: the product is a plain shared library whose ``extern "C"``
entry points are declared in ``include/batchsim_b200.h``; Python binds it with ctypes
(``_native.py``).  Parity-critical translation units (pose algebra, rasterizer setup) are
compiled with ``-fmad=false`` so their float arithmetic rounds like numpy's; the step
kernel may contract to FMA.

Usage: ``python -m paper_2410_00425_b200.build_native [--force] [-v]``.
"""

from __future__ import annotations

import hashlib
import json
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
if os.environ.get("BS_EXTRA_NVCC"):  # developer A/B variants (tools/gpu_lib_ab.sh), e.g. -DBS_NO_L2_PREFETCH
    COMMON.extend(os.environ["BS_EXTRA_NVCC"].split())
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


def _digest(src: str) -> str:
    """Content hash of one translation unit's inputs: the source, every header it can include
    and the exact nvcc flags (so a stale object is detected even when file mtimes lie, e.g.
    after a snapshot copy)."""
    h = hashlib.sha256()
    h.update(" ".join(ARCH + COMMON + SOURCES[src]).encode())
    files = [os.path.join(CSRC, src), os.path.join(ROOT, "include", "batchsim_b200.h")]
    files += sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
    for f in files:
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


STAMP = os.path.join(OUT_DIR, "build_stamp.json")


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source for sm_100a and link the shared library; returns its path.
    An object is rebuilt when its content digest (source + headers + flags) changed."""
    nvcc = _nvcc()
    os.makedirs(OUT_DIR, exist_ok=True)
    try:
        with open(STAMP) as fh:
            stamp = json.load(fh)
    except (OSError, ValueError):
        stamp = {}
    sources = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    objs = []
    jobs = []
    for src in sources:
        spath = os.path.join(CSRC, src)
        obj = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
        objs.append(obj)
        digest = _digest(src)
        stale = force or not os.path.exists(obj) or stamp.get(src) != digest
        stamp[src] = digest
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
    link_digest = hashlib.sha256("".join(stamp[s] for s in sources).encode()).hexdigest()
    if force or jobs or not os.path.exists(LIB_PATH) or stamp.get("__lib__") != link_digest:
        tmp = LIB_PATH + ".tmp"
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
        run(cmd)
        os.replace(tmp, LIB_PATH)
    stamp["__lib__"] = link_digest
    with open(STAMP, "w") as fh:
        json.dump(stamp, fh, indent=1)
    return LIB_PATH


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
