"""cfg5 (BASELINE configs[4], ~5.6e8 zip nodes, 1.22 M leaves) on one GPU: setup
timings, a few LTS slices and one GTS step, rates by CUDA events.  Usage:
python tools/cfg5_try.py [config] [slices]"""
import os
import resource
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import build_mesh, units_per_round  # noqa: E402
from paper_2011_10570_b200.stepper import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
n_sl = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rss = lambda: resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6  # noqa: E731
t0 = time.time()
cfg, mesh = build_mesh(name, 1, "lts")
t1 = time.time()
print(f"{name}: tree + mesh {t1 - t0:.1f} s, {len(mesh.tree)} leaves, {mesh.n_nodes} zip nodes, host rss {rss():.1f} GB, "
      f"device {torch.cuda.memory_allocated() / 1e9:.1f} GB", flush=True)
for mode in ("lts", "gts"):
    t2 = time.time()
    eng = Engine(mesh, tableau=cfg.tableau, cfl=cfg.cfl, mode=mode, nonlinear=cfg.nonlinear)
    t3 = time.time()
    eng.initialize(cfg.chi0(), device_eval=True)
    t4 = time.time()
    print(f"{mode}: engine {t3 - t2:.1f} s, initialize {t4 - t3:.1f} s, host rss {rss():.1f} GB, "
          f"device {torch.cuda.memory_allocated() / 1e9:.1f} GB", flush=True)
    counts = np.diff(mesh.leaf_starts)
    cad = eng._leaf_cadence
    n = n_sl if mode == "lts" else 2
    eng.advance_slice()  # warm
    units = 0
    for i in range(eng.i_fine, eng.i_fine + n):
        el = eng._eligible_cadences(i)
        units += eng.p * int(counts[np.isin(cad, el)].sum())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        eng.advance_slice()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    z = eng.current_zip_device()
    mx = float(z[0].abs().max())
    fin = bool(torch.isfinite(z[0]).all()) and bool(torch.isfinite(z[1]).all())
    print(f"{mode}: {n} slices {ms:.1f} ms, {units / ms / 1e6:.2f} G updates/s, max|chi| {mx:.6f}, finite {fin}", flush=True)
    del eng, z
    import gc

    gc.collect()
    torch.cuda.empty_cache()
