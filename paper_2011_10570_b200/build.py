"""Build the native library in-tree: paper_2011_10570_b200/_lib/libamr_b200.so.

One nvcc per source (in parallel) compiles the sm_100a kernels (amr_kernels.cu,
amr_wavelet.cu, amr_octree.cu) and the host C++ mesh builder (amr_mesh.cpp); one link makes
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
SOURCES = ["amr_kernels.cu", "amr_wavelet.cu", "amr_octree.cu", "amr_devmesh.cu", "amr_devprog.cu", "amr_mesh.cpp", "amr_programs.cpp"]
# the stage-kernel launcher, compiled once per (dim, ppo, lts) in parallel
INSTANCES = [(d, p, l) for d in (2, 3) for p in (5, 7, 9) for l in (0, 1)]
INST_SRC = "amr_stage_inst.cu"
HEADERS = ["amr_common.cuh", "amr_async.cuh", "amr_stage_cross.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS + [INST_SRC]] + [os.path.join(INCLUDE, "amr_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Compile if stale.  AMR_NVCC_FLAGS adds flags (e.g. -DAMR_CROSS_MINB=5
    for tuning experiments); ``out`` builds a variant library elsewhere (load
    it with AMR_LIB_PATH)."""
    lib_path = out or LIB
    objdir = os.path.dirname(lib_path) if out else LIBDIR
    if not force and not out and not _stale():
        return LIB
    os.makedirs(objdir, exist_ok=True)
    extra = os.environ.get("AMR_NVCC_FLAGS", "").split()
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", *extra,
              "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O2", "-I", INCLUDE]
    if verbose:
        common.insert(1, "-Xptxas=-v")
    # one nvcc per source and per stage-kernel instance, in parallel, then one link
    jobs = [([os.path.join(CSRC, src)], os.path.join(objdir, os.path.splitext(src)[0] + ".o")) for src in SOURCES]
    for d, p, l in INSTANCES:
        jobs.append(([f"-DAMR_INST_DIM={d}", f"-DAMR_INST_PPO={p}", f"-DAMR_INST_LTS={l}", os.path.join(CSRC, INST_SRC)],
                     os.path.join(objdir, f"amr_stage_{d}_{p}_{l}.o")))
    # heaviest first (3D ppo 9), at most one job per core
    jobs.sort(key=lambda j: -sum(int(a.split("=")[1]) for a in j[0] if a.startswith("-DAMR_INST_")))
    width = max(1, min(len(jobs), os.cpu_count() or 4))
    objs, running = [], []

    def reap(item):
        cmd, obj, pr = item
        out, err = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{out}\n{err}")
        if verbose:
            sys.stderr.write(err)
        objs.append(obj)

    for srcs, obj in jobs:
        while len(running) >= width:
            reap(running.pop(0))
        cmd = [*common, "-c", *srcs, "-o", obj]
        running.append((cmd, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    for item in running:
        reap(item)
    cmd = [NVCC, *ARCH, "-shared", "-o", lib_path + ".tmp", *objs, "-lgomp"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({' '.join(cmd)}):\n{proc.stdout}\n{proc.stderr}")
    os.replace(lib_path + ".tmp", lib_path)
    return lib_path


if __name__ == "__main__":
    o = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=o[0] if o else None))
