"""Benchmark: RK-stage zip-node updates/s of the LTS/GTS octree wave solver on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One *step* = one LTS coarse round (2^dL fine slices) of BASELINE configs[1]
("cfg2": 3D linear wave, levels 3-7, ppo 9, RK4, CFL 0.25) — the largest
workload the metric is quoted on for one GPU.  Unit of work = one RK stage
applied to one zip node; LTS counts the units it executes.
Alongside: the GTS engine over the same simulated time (the LTS-vs-GTS wall
speedup), the stage kernel's HBM roofline (68 algorithmic bytes per unit,
CUDA events per launch), an end-to-end number through the public API with
host buffers, the CPU oracle ("port" of the reference; the reference itself is
pure Python and absent on the GPU box) timed on the host cores, and the SM
clocks sampled during the timed region.

N > 1: launched by torch.distributed.run, one rank per GPU, weighted Morton
partition across ranks (mesh.pmap), ghost leaves over NCCL after every stage;
time = max over ranks, value = all ranks' units / time ("weak" in the sense
that each rank owns a contiguous 1/N of the weighted leaves of a fixed mesh
is strong scaling — reported as "strong").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_UNIT = 68.0  # RK4, 2 x fp64 vars, per zip-node stage update


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clock/throttle sampling (100 ms) for the whole run; samples are
    attributed to the timed windows by timestamp."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.windows = []

    def start(self):
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.time(), ln.strip()))

    def window(self):
        """Context manager marking one timed region."""
        sampler = self

        class _W:
            def __enter__(self):
                self.t0 = time.time()
                return self

            def __exit__(self, *exc):
                sampler.windows.append((self.t0, time.time()))

        return _W()

    def stop(self):
        if self.proc is not None:
            time.sleep(0.25)  # let the last window's samples arrive
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.th.join(timeout=2)

    def summary(self):
        sm, mx, reasons, n_all = [], None, set(), 0
        for t, ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            n_all += 1
            # a sample read at t describes the ~100 ms before it
            if not any(a - 0.05 <= t <= b + 0.15 for a, b in self.windows):
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "samples_total": n_all}


def _workload(name: str) -> str:
    from paper_2011_10570_b200.configs import CONFIGS

    c = CONFIGS[name]
    src = {False: "linear", "cubic": "cubic", "sin": "sin"}[c.nonlinear]
    levels = {"cfg1": "3-6", "cfg2": "3-7", "cfg3": "4-9", "cfg4": "2-13", "cfg5": "4-12"}.get(name, "?")
    return (f"{name}: {c.dim}D {src} wave on [-1,1]^{c.dim}, levels {levels}, ppo {c.ppo}, pad {c.pad}, "
            f"{c.tableau.upper()}, CFL {c.cfl}; step = one LTS coarse round")


def _speedup_model(mesh, work_ratio):
    from paper_2011_10570_b200.perfmodel import estimate, histogram_from_mesh

    est = estimate(histogram_from_mesh(mesh.blocks))
    return {"perfmodel_speedup": est.speedup, "perfmodel_bound": est.bound,
            "zip_node_work_ratio": work_ratio}


def _ncu_traffic():
    """DRAM bytes per stage launch from the committed ncu capture
    (profiles/traffic.json, written by tools/ncu_traffic.py from one
    `ncu --set full` run of tools/profile_stage.py on cfg2)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return float(d["lts_bytes_per_launch"]), (
            f"ncu dram__bytes_read+write per LTS stage launch ({d['source']}); "
            f"algorithmic bytes of the same launches: {d['lts_algorithmic_bytes_per_launch']:.3e}")
    except Exception:
        return None, "no committed ncu capture"


def build_mesh(cfg_name, ranks, mode):
    from paper_2011_10570_b200.configs import CONFIGS
    from paper_2011_10570_b200.mesh import Domain, Mesh
    from paper_2011_10570_b200.octree import SfcOrdering, balance_2to1, construct
    from paper_2011_10570_b200.partition import tree_weights, weighted_partition

    c = CONFIGS[cfg_name]
    tree = balance_2to1(construct(c.refine, c.dim, c.max_depth, SfcOrdering("morton", c.dim, c.max_depth)))
    pmap = weighted_partition(tree, tree_weights(tree, mode), ranks) if ranks > 1 else None
    return c, Mesh(tree, points_per_octant=c.ppo, pad=c.pad, pmap=pmap, domain=Domain(c.domain_lo, c.domain_hi))


def units_per_round(eng, rank_only=True):
    """Zip-node stage updates one LTS round executes (this rank's leaves)."""
    mesh = eng.mesh
    counts = np.diff(mesh.leaf_starts)
    if eng._dist is not None and rank_only:
        owners = mesh.pmap.owners(len(counts))
        counts = np.where(owners == eng.rank, counts, 0)
    by_cad = {}
    for c, n in zip(eng._leaf_cadence.tolist(), counts.tolist()):
        by_cad[c] = by_cad.get(c, 0) + n
    total = 0
    launches = 0
    for i in range(eng.schedule.slices_per_round):
        el = eng._eligible_cadences(i)
        total += eng.p * sum(by_cad.get(c, 0) for c in el)
        launches += eng.launches_per_slice(i)
    return total, launches


def time_rounds(eng, steps, torch, dist, per_launch=False):
    """Device time of `steps` rounds; optional per-launch CUDA events (profiling pass)."""
    dev = eng.device
    stream = torch.cuda.current_stream(dev)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches = []
    if per_launch:
        from paper_2011_10570_b200 import _native

        L, P = eng._lib, eng._prm
        orig = L.amr_stage

        def timed(prm, strm):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rc = orig(prm, strm)
            e1.record(stream)
            launches.append((e0, e1, int(P.n_tiles)))
            return rc

        eng._lib = type("L", (), {"amr_stage": staticmethod(timed), "amr_iface": staticmethod(L.amr_iface)})()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    n_slices = eng.schedule.slices_per_round
    for _ in range(steps):
        if per_launch:  # eager slices so every launch can be bracketed by events
            for _ in range(n_slices):
                eng.advance_slice()
        else:  # the public API: one coarse round (CUDA-graph replay after warm-up)
            eng.lts_coarse_step()
    end.record(stream)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    if per_launch:
        eng._lib = L
    ms = start.elapsed_time(end)
    return ms, [(a.elapsed_time(b), n) for a, b, n in launches]


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2011_10570_b200.stepper import Engine

    clk = ClockSampler(local).start()
    t0 = time.time()
    cfg, mesh = build_mesh(args.config, world, "lts")
    t_mesh = time.time() - t0
    chi0 = cfg.chi0()
    res = {}
    engines = {}
    for mode in ("lts", "gts"):
        eng = Engine(mesh, tableau=cfg.tableau, cfl=cfg.cfl, mode=mode, nonlinear=cfg.nonlinear, device=dev)
        eng.initialize(chi0)
        engines[mode] = eng
        units, launches = units_per_round(eng)
        for _ in range(args.warmup):
            eng.lts_coarse_step() if mode == "lts" else [eng.gts_step() for _ in range(eng.schedule.slices_per_round)]
        with clk.window():
            if mode == "lts":
                ms, _ = time_rounds(eng, args.steps, torch, dist)
            else:
                n = engines["lts"].schedule.slices_per_round
                if dist is not None:
                    dist.barrier()
                torch.cuda.synchronize(dev)
                s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s_ev.record()
                for _ in range(args.steps * n):
                    eng.gts_step()
                e_ev.record()
                torch.cuda.synchronize(dev)
                if dist is not None:
                    dist.barrier()
                ms = s_ev.elapsed_time(e_ev)
        if mode == "gts":  # a GTS "step" covers the same simulated time: 2^dL fine slices
            n = engines["lts"].schedule.slices_per_round
            units, launches = units * n, launches * n
        t = torch.tensor([ms, float(units)], dtype=torch.float64, device=dev)
        if dist is not None:
            tmax = t.clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            tsum = t.clone()
            dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
            ms_all, units_all = float(tmax[0]), float(tsum[1])
        else:
            ms_all, units_all = ms, float(units)
        res[mode] = dict(ms=ms_all, units_per_step=units_all, launches_per_step=launches)

    # roofline: profiling pass (per-launch CUDA events) of the headline engine
    eng = engines["lts"]
    _, per = time_rounds(eng, 1, torch, None if dist is None else dist, per_launch=True)
    counts = np.diff(mesh.leaf_starts)
    # algorithmic bytes per launch = 68 B x owned nodes of the launched tiles
    tiles = eng._rank_list[0].tiles
    cum = np.concatenate([[0], np.cumsum(counts[tiles])])
    k_ms = sum(m for m, _ in per)
    k_bytes = sum(BYTES_PER_UNIT * cum[n] for _, n in per)
    peak, peak_src = _peaks()
    achieved = k_bytes / (k_ms * 1e-3) / 1e9 if k_ms > 0 else 0.0
    traffic, traffic_note = _ncu_traffic()
    # same for GTS launches (all tiles)
    geng = engines["gts"]
    _, gper = time_rounds(geng, 1, torch, None if dist is None else dist, per_launch=True)
    g_ms = sum(m for m, _ in gper)
    g_bytes = sum(BYTES_PER_UNIT * cum[n] for _, n in gper) if gper else 0.0
    g_ach = g_bytes / (g_ms * 1e-3) / 1e9 if g_ms > 0 else 0.0

    # e2e through the public API with host buffers (pinned), LTS
    z_host = torch.from_numpy(eng.current_zip()).pin_memory()
    z_out = torch.empty_like(z_host).pin_memory()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    te0 = time.perf_counter()
    ew = clk.window()
    ew.__enter__()
    for _ in range(args.steps):
        eng.load_zip(z_host)
        eng.lts_coarse_step()
        z_out.copy_(eng.current_zip_device(), non_blocking=True)
        torch.cuda.synchronize(dev)
    te = time.perf_counter() - te0
    ew.__exit__(None, None, None)
    clk.stop()
    tt = torch.tensor([te], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    te = float(tt[0])

    lts, gts = res["lts"], res["gts"]
    value = lts["units_per_step"] * args.steps / (lts["ms"] * 1e-3)
    gts_value = gts["units_per_step"] * args.steps / (gts["ms"] * 1e-3)
    out = {
        "metric": "RK-stage zip-node updates/s (LTS, executed)",
        "value": value,
        "unit": "updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": lts["ms"] / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic ({args.config} mesh and Gaussian initial data, seeded; no dataset exists for this path)",
        "config": {
            "workload": _workload(args.config),
            "leaves": len(mesh.tree.leaves), "zip_nodes": mesh.n_nodes,
            "l2_policy": "inputs larger than L2 (state u0,u1,K0..K3 = "
                         f"{6 * 16 * mesh.n_nodes / 1e6:.0f} MB > 126 MB)",
            "parallelism": f"weighted Morton partition x{world}" if world > 1 else "1 GPU",
            "mesh_build_s": round(t_mesh, 2),
        },
        "gts": {"value": gts_value, "ms_per_step": gts["ms"] / args.steps,
                "units_per_step": gts["units_per_step"]},
        "lts_vs_gts_wall_speedup": gts["ms"] / lts["ms"],
        # the reference's work model (perfmodel.py:52-71) and the zip-node work ratio, beside the measured speedup
        "lts_vs_gts_model": _speedup_model(mesh, gts["units_per_step"] / lts["units_per_step"]),
        "lts_gts_equivalent_rate": gts["units_per_step"] * args.steps / (lts["ms"] * 1e-3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_note": traffic_note,
                     "peak_source": peak_src,
                     "kernel": f"amr_stage (stage_cross, {eng._threads} threads/CTA): fused unzip on the owned cross + RHS + zip [+ RK combine]",
                     "bytes_per_unit": BYTES_PER_UNIT,
                     "launches": len(per), "kernel_ms_per_round": k_ms,
                     "gts_achieved": g_ach, "gts_frac": g_ach / peak},
        "e2e": {"value": lts["units_per_step"] * args.steps / te, "unit": "updates/s",
                "h2d_bytes_per_step": int(2 * 8 * mesh.n_nodes), "d2h_bytes_per_step": int(2 * 8 * mesh.n_nodes)},
        "gpu_launches": int(lts["launches_per_step"] * args.steps),
        "clocks": clk.summary(),
    }
    if rank == 0:
        out["remesh_criterion"] = _remesh_criterion(eng)
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args, rounds=1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def _oracle_setup(cfg_name):
    from oracle import oracle as O

    from paper_2011_10570_b200.configs import CONFIGS

    c = CONFIGS[cfg_name]
    a, lv = O.construct(c.refine, c.dim, c.max_depth)
    a, lv = O.balance(c.dim, c.max_depth, a, lv)
    m = O.OracleMesh(c.dim, c.max_depth, a, lv, c.ppo, c.pad, c.domain_lo, c.domain_hi)
    e = O.OracleEngine(m, c.tableau, c.cfl, "lts", c.nonlinear)
    e.initialize(c.chi0())
    return c, m, e


def _oracle_units(m, e):
    counts = np.diff(m.leaf_starts)
    lr, _, ll = m.blocks()
    cad = np.empty(len(counts), dtype=np.int64)
    for (a, b), lvl in zip(lr, ll):
        cad[a:b] = lvl
    R = 1 << (e.l_max - e.l_min)
    tot = 0
    for i in range(R):
        el = cad >= (e.l_max - ((i & -i).bit_length() - 1 if i else e.l_max))
        tot += e.p * int(np.sum(counts[el]))
    return tot, R


def _remesh_criterion(eng, reps=10):
    """Wavelet remesh criterion on the evolved solution,
    outside the timed region: the leaf-lattice gather + amr_wavelet_coeff
    (nodes_per_dim = ppo) over every leaf, CUDA events on the current stream.
    The full-size kernel roofline is tools/bench_wavelet.py's."""
    import torch

    from paper_2011_10570_b200.wavelet import RefinePolicy, coefficients_from_values

    m = eng.mesh
    pol = RefinePolicy(tolerance=1e-3, min_level=0, max_level=m.L)
    lv = torch.from_numpy(m.tree.arrays()[1].astype(np.int32)).to(eng.device)
    z = eng.current_zip_device()
    lat = m.leaf_lattice_device(z, 0)
    s, e, k = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        lat = m.leaf_lattice_device(z, 0)
    k.record()
    for _ in range(reps):
        _, codes = coefficients_from_values(lat, m.ppo, m.dim, lv, pol)
    e.record()
    torch.cuda.synchronize()
    hist = torch.bincount((codes.to(torch.int64) + 1), minlength=3).tolist()
    return {"leaves": int(lat.shape[0]), "nodes_per_dim": m.ppo, "ms_leaf_lattice": s.elapsed_time(k) / reps,
            "ms_wavelet_kernel": k.elapsed_time(e) / reps, "flags_coarsen_keep_refine": hist}


def cpu_baseline(args, rounds=1):
    """The oracle port timed on this host's cores on a bounded sample."""
    c, m, e = _oracle_setup(args.config)
    units, R = _oracle_units(m, e)
    t0 = time.perf_counter()
    for _ in range(rounds * R):
        e.advance_slice()
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
    return {"value": units * rounds / dt, "unit": "updates/s", "cores": cores, "kind": "port",
            "sample": f"{rounds} LTS round(s) of {args.config} ({units * rounds} zip-node stage updates), "
                      "oracle/amr_oracle.c (C+OpenMP restatement of amrlts.stepper), mesh build excluded"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    c, m, e = _oracle_setup(args.config)
    units, R = _oracle_units(m, e)
    for _ in range(args.warmup * R):
        e.advance_slice()
    t0 = time.perf_counter()
    for _ in range(args.steps * R):
        e.advance_slice()
    dt = time.perf_counter() - t0
    value = units * args.steps / dt
    cores = int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
    print(json.dumps({
        "impl": "reference", "metric": "RK-stage zip-node updates/s (LTS, executed)", "value": value,
        "unit": "updates/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (BASELINE configs[1])",
        "config": {"workload": _workload(args.config), "zip_nodes": m.n_nodes},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} LTS rounds of {args.config} on the oracle port "
                                   "(the reference amrlts is pure Python and not present on the GPU box)"},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
