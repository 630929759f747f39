"""Build the native library in-tree: paper_2011_10570_b200/_lib/libamr_b200.so.

One nvcc per source (in parallel) compiles the sm_100a kernels (amr_kernels.cu,
amr_wavelet.cu) and the host C++ mesh builder (amr_mesh.cpp); one link makes
the C-ABI shared library that Python loads with ctypes.  Flags that matter for parity:
  -fmad=false            no FMA contraction in device code (numpy rounds every op)
  -ffp-contract=off      same for the host C++ (interpolation weights)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libamr_b200.so")
INCLUDE = os.path.abspath(os.path.join(HERE, "..", "include"))
SOURCES = ["amr_kernels.cu", "amr_wavelet.cu", "amr_mesh.cpp"]
HEADERS = ["amr_stage_pipe.cuh", "amr_stage_blob.cuh", "amr_stage_cross.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(INCLUDE, "amr_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile if stale.  AMR_NVCC_FLAGS adds flags (e.g. -DAMR_MIN_BLOCKS=2
    for tuning experiments)."""
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    extra = os.environ.get("AMR_NVCC_FLAGS", "").split()
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", *extra,
              "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O2", "-I", INCLUDE]
    if verbose:
        common.insert(1, "-Xptxas=-v")
    # one nvcc per source, in parallel, then one link
    procs = []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, os.path.splitext(src)[0] + ".o")
        cmd = [*common, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    objs = []
    for cmd, obj, pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{out}\n{err}")
        if verbose:
            sys.stderr.write(err)
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lgomp"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({' '.join(cmd)}):\n{proc.stdout}\n{proc.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
