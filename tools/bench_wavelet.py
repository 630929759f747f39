"""Benchmark of the wavelet refinement criterion.

Workload: every leaf of a uniform level-6 3D tree (262 144 octants) on
[-1,1]^3, nodes_per_dim 7 (the reference default), field tests' gauss3.
  * device: amr_wavelet_coeff on device-resident samples (720 MB > L2),
    CUDA events around K launches; roofline = 8 B x npd^3 read + 8 B coeff +
    4 B level + 1 B flag per octant against measured HBM GB/s;
  * e2e: W.refine_flags(f, tree, policy) — host sampling + f, H2D, kernel,
    D2H of the flags — wall time;
  * cpu: oracle/amr_oracle.c ora_wavelet_coeff on the same samples (C +
    OpenMP, all host cores): the reference's arithmetic restated.
One JSON line on stdout.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2011_10570_b200 import wavelet as W  # noqa: E402
from paper_2011_10570_b200.octree import uniform_tree  # noqa: E402
from wavelet_fields import FIELDS  # noqa: E402


def main(steps=20, warmup=3, level=6, npd=7):
    dim, L = 3, level
    tree = uniform_tree(dim, L, level)
    an, lv = tree.arrays()
    lo, hi = (-1.0,) * 3, (1.0,) * 3
    f = FIELDS["gauss3"]
    pol = W.RefinePolicy(tolerance=1e-4, min_level=1, max_level=L + 1)
    n = len(an)
    vals = W._sample_values(f, W._sample_axes(an.astype(np.int64), lv, L, lo, hi, npd), npd)
    dv = torch.from_numpy(vals).cuda()
    dl = torch.from_numpy(lv).cuda()
    for _ in range(warmup):
        W.coefficients_from_values(dv, npd, dim, dl, pol)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        W.coefficients_from_values(dv, npd, dim, dl, pol)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    bytes_per = 8 * npd ** dim + 8 + 4 + 1
    gbs = bytes_per * n / (ms * 1e-3) / 1e9
    peak = 6456.8
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    # e2e through the drop-in API (host f, pinned H2D, kernel, D2H)
    W.refine_codes(f, tree, pol, npd, lo, hi)
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        codes = W.refine_codes(f, tree, pol, npd, lo, hi)
    e2e_s = (time.perf_counter() - t0) / reps
    # the same call with on-device sampling: f written with torch ops
    ft = lambda x, y, z: torch.exp(-((x - 0.3) ** 2 + y ** 2 + (z + 0.1) ** 2) / 0.02)  # noqa: E731
    W.refine_codes(ft, tree, pol, npd, lo, hi, device_eval=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        W.refine_codes(ft, tree, pol, npd, lo, hi, device_eval=True)
    dev_s = (time.perf_counter() - t0) / reps
    out = {
        "metric": "wavelet coefficients + flags (octants/s)", "value": n / (ms * 1e-3), "unit": "octants/s",
        "ms_per_launch": ms, "octants": n, "nodes_per_dim": npd, "dim": dim,
        "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                     "bytes_per_octant": bytes_per},
        "e2e": {"value": n / e2e_s, "unit": "octants/s", "s_per_call": e2e_s,
                "h2d_bytes": int(vals.nbytes + 4 * n), "d2h_bytes": int(9 * n)},
        "e2e_device_sampling": {"value": n / dev_s, "unit": "octants/s", "s_per_call": dev_s,
                                "note": "refine_codes(device_eval=True): coordinates and f (torch ops) on the GPU"},
        "flags_hist": {str(k): int(v) for k, v in zip(*np.unique(codes, return_counts=True))},
    }
    # predicate-driven construction (wavelet.py:127-144 through octree.construct):
    # one launch per level, samples on the device
    from paper_2011_10570_b200.octree import SfcOrdering, construct

    pp = W.RefinePolicy(tolerance=1e-6, min_level=2, max_level=8)
    pred = W.refinement_predicate(ft, pp, npd, lo, hi, device_eval=True)
    construct(pred, 3, 8, SfcOrdering("morton", 3, 8))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    built = construct(pred, 3, 8, SfcOrdering("morton", 3, 8))
    tc = time.perf_counter() - t0
    an_b, lv_b = built.arrays()
    # octants visited by the level-synchronous construction: leaves + internal
    # nodes of the complete octree ((leaves - 1) / 7)
    hist = np.bincount(lv_b, minlength=9)
    tested = int(len(lv_b) + (len(lv_b) - 1) // 7)
    out["construct"] = {"leaves": int(len(lv_b)), "octants_tested": tested, "s": tc,
                        "octants_per_s": tested / tc, "levels": [int(x) for x in hist],
                        "note": "construct(refinement_predicate(gauss3 in torch, tol 1e-6, levels 2..8, npd 7, "
                                "device_eval=True)), Morton order, one launch per level"}
    if "--no-cpu" not in sys.argv:
        from oracle import oracle as O

        sub = vals[: n // 4]
        t0 = time.perf_counter()
        O.wavelet_coeffs(sub, npd, dim)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": len(sub) / dt, "unit": "octants/s", "cores": len(os.sched_getaffinity(0)),
                               "kind": "port", "sample": f"{len(sub)} octants, oracle ora_wavelet_coeff (C+OpenMP)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
