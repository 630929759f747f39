"""Generate golden fixtures by running the UNMODIFIED reference package.

Run here (where /root/reference exists):

    python tests/golden/make_golden.py [case ...]

Each case imports ``amrlts`` read-only from /root/reference/pkg/src, builds a
tree / partition / mesh with the reference's own functions and steps its own
``Engine``.  The outputs are committed as ``tests/golden/<case>.npz`` so the
GPU box (which has no /root/reference) can check parity against them.

The cubic source ``-chi^3`` does not exist in the reference (SURVEY.md §0
finding 2).  It is added as a documented *oracle extension*: the reference
``wave_rhs`` is wrapped so that ``dphi -= (chi*chi)*chi`` on every interior
point except the physical-face rows, which reproduces "source before face
overwrite" (wave.py:161-169).  Nothing else is patched.

Large snapshots are stored as (sha256 of the exact bytes with -0 -> +0, a
strided sample, per-variable max|.|) to keep fixtures small.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import amrlts.stepper as ref_stepper  # noqa: E402
from amrlts import rkcorrect, wave  # noqa: E402
from amrlts.mesh import Domain, Mesh  # noqa: E402
from amrlts.octree import SfcOrdering, balance_2to1, construct, random_tree, uniform_tree  # noqa: E402
from amrlts.partition import build_exchange_plan, tree_weights, weighted_partition  # noqa: E402
from amrlts.stepper import Engine  # noqa: E402

from paper_2011_10570_b200.configs import CONFIGS  # noqa: E402

_ORIG_RHS = ref_stepper.wave_rhs


def cubic_rhs(y, geom, nonlinear, k_chi, k_phi, f0_chi=0.0, f0_phi=0.0):
    """Oracle extension: linear reference RHS, then -chi^3 off the face rows."""
    out = _ORIG_RHS(y, geom, False, k_chi, k_phi, f0_chi, f0_phi)
    if nonlinear:
        g = geom.pad
        dim = y[0].ndim
        chi = y[0][(slice(g, -g),) * dim]
        src = (chi * chi) * chi
        mask = np.ones(chi.shape, dtype=bool)
        n = chi.shape[0]
        for axis, side in geom.faces:
            sel = [slice(None)] * dim
            sel[axis] = 0 if side == 0 else n - 1
            mask[tuple(sel)] = False
        out[1][mask] = out[1][mask] - src[mask]
    return out


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a, dtype=np.float64) + 0.0
    return hashlib.sha256(a.tobytes()).hexdigest()


def tree_arrays(tree):
    anchors = np.array([k.anchor for k in tree.leaves], dtype=np.int64).reshape(len(tree.leaves), tree.dim)
    levels = np.array([k.level for k in tree.leaves], dtype=np.int64)
    return anchors, levels


def mesh_arrays(mesh, with_gathers=True):
    out = {
        "n_nodes": np.int64(mesh.n_nodes),
        "leaf_slices": mesh.leaf_slices.astype(np.int64),
        "leaf_gids": mesh.leaf_gids.astype(np.int64),
        "node_coords": mesh.node_coords.astype(np.int64),
        "block_root_anchor": np.array([b.root.anchor for b in mesh.blocks], dtype=np.int64),
        "block_root_level": np.array([b.root.level for b in mesh.blocks], dtype=np.int64),
        "block_leaf_level": np.array([b.leaf_level for b in mesh.blocks], dtype=np.int64),
        "block_leaf_range": np.array([b.leaf_range for b in mesh.blocks], dtype=np.int64),
        "block_owner": np.array([b.owner_rank for b in mesh.blocks], dtype=np.int64),
        "finest_spacing": np.float64(mesh.finest_spacing()),
    }
    reads = [np.asarray(mesh.block_read_leaves(b.index), dtype=np.int64) for b in mesh.blocks]
    out["block_read_ptr"] = np.concatenate([[0], np.cumsum([len(r) for r in reads])]).astype(np.int64)
    out["block_read"] = np.concatenate(reads).astype(np.int64)
    digs = []
    hist = {}
    for G in mesh.gathers:
        h = hashlib.sha256()
        h.update(np.asarray(G.indptr, dtype=np.int64).tobytes())
        h.update(np.asarray(G.indices, dtype=np.int64).tobytes())
        h.update(np.asarray(G.data, dtype=np.float64).tobytes())
        digs.append(h.hexdigest())
        for k, v in zip(*np.unique(np.diff(G.indptr), return_counts=True)):
            hist[int(k)] = hist.get(int(k), 0) + int(v)
    out["gather_digests"] = np.array(digs)
    out["gather_nnz_hist"] = np.array(sorted(hist.items()), dtype=np.int64)
    if with_gathers:
        ptr, idx, dat, rows = [0], [], [], [0]
        for G in mesh.gathers:
            base = ptr[-1]
            ptr.extend((np.asarray(G.indptr[1:], dtype=np.int64) + base).tolist())
            idx.append(np.asarray(G.indices, dtype=np.int64))
            dat.append(np.asarray(G.data, dtype=np.float64))
            rows.append(rows[-1] + G.shape[0])
        out["g_indptr"] = np.array(ptr, dtype=np.int64)
        out["g_indices"] = np.concatenate(idx)
        out["g_data"] = np.concatenate(dat)
        out["g_block_rows"] = np.array(rows, dtype=np.int64)
    return out


def plan_arrays(plan, prefix):
    rows = []
    for (s, r), items in sorted(plan.entries.items()):
        for e in items:
            rows.append((s, r, e.leaf, e.node_start, e.node_stop, e.sender_block, len(e.receiver_blocks)))
    return {prefix: np.array(rows, dtype=np.int64).reshape(-1, 7)}


def store_field(out, key, z, full):
    z = np.asarray(z)
    if full:
        out[key] = z.copy()
    else:
        out[key + "__sha"] = np.array(digest(z))
        out[key + "__sample"] = z[:, ::7].copy()
        out[key + "__absmax"] = np.max(np.abs(z), axis=1)


def make_engine(mesh, cfg_tableau, mode, nonlinear):
    if nonlinear == "cubic":
        ref_stepper.wave_rhs = cubic_rhs
        nl = True
    else:
        ref_stepper.wave_rhs = _ORIG_RHS
        nl = bool(nonlinear)
    return Engine(mesh, tableau=cfg_tableau, cfl=0.25, mode=mode, nonlinear=nl)


def run_fields(out, mesh, chi0, runs, full):
    """runs: list of (tag, tableau, mode, nonlinear, checkpoints in fine slices)."""
    for tag, tab, mode, nl, checkpoints in runs:
        t0 = time.time()
        eng = make_engine(mesh, tab, mode, nl)
        eng.initialize(chi0)
        if "z0" not in out and "z0__sha" not in out:
            store_field(out, "z0", eng.current_zip(), full)
        for cp in checkpoints:
            eng.run_to(cp)
            store_field(out, f"{tag}_i{cp}", eng.current_zip(), full)
            if mode == "lts" and cp == eng.schedule.slices_per_round:
                out[f"{tag}_point_steps_round"] = np.int64(eng.counters.point_steps)
        out[f"{tag}_dt_fine"] = np.float64(eng.dt_fine)
        ref_stepper.wave_rhs = _ORIG_RHS
        print(f"  {tag}: {time.time() - t0:.1f}s", flush=True)


def config_case(name, runs, full, parts=((2, "lts"), (3, "lts"), (4, "lts"), (8, "lts"), (4, "gts")),
                with_gathers=True):
    cfg = CONFIGS[name]
    order = SfcOrdering("morton", cfg.dim, cfg.max_depth)
    pre = construct(cfg.refine, cfg.dim, cfg.max_depth, order)
    tree = balance_2to1(pre)
    out = {"meta": np.array(json.dumps({"case": name, "dim": cfg.dim, "max_depth": cfg.max_depth,
                                         "ppo": cfg.ppo, "pad": cfg.pad}))}
    out["pre_anchor"], out["pre_level"] = tree_arrays(pre)
    out["anchor"], out["level"] = tree_arrays(tree)
    for R, mode in parts:
        pm = weighted_partition(tree, tree_weights(tree, mode), R)
        out[f"part_{mode}_{R}"] = np.array(pm.rank_ranges, dtype=np.int64)
    dom = Domain(cfg.domain_lo, cfg.domain_hi)
    t0 = time.time()
    mesh = Mesh(tree, points_per_octant=cfg.ppo, pad=cfg.pad, domain=dom)
    print(f"  mesh {time.time() - t0:.1f}s n_nodes={mesh.n_nodes}", flush=True)
    out.update(mesh_arrays(mesh, with_gathers))
    pm = weighted_partition(tree, tree_weights(tree, "lts"), 4)
    mesh4 = Mesh(tree, points_per_octant=cfg.ppo, pad=cfg.pad, pmap=pm, domain=dom)
    out["r4_block_leaf_range"] = np.array([b.leaf_range for b in mesh4.blocks], dtype=np.int64)
    out["r4_block_owner"] = np.array([b.owner_rank for b in mesh4.blocks], dtype=np.int64)
    out.update(plan_arrays(build_exchange_plan(mesh4, pm), "r4_plan"))
    run_fields(out, mesh, cfg.chi0(), runs, full)
    return out


def small_cases():
    """Reference-test style meshes: DOM2 = [-10,10]^2 (non-dyadic h), ppo 5/7,
    random trees; rk3 (the reference default tableau)."""
    out = {}
    dom2 = Domain((-10.0, -10.0), (10.0, 10.0))

    def ball_refine(key, rad=3.0, top_level=4, base=2, lo=-10.0, hi=10.0):
        if key.level < base:
            return True
        if key.level >= top_level:
            return False
        scale = (hi - lo) / (1 << key.max_depth)
        mins = [lo + a * scale for a in key.anchor]
        maxs = [lo + (a + key.side) * scale for a in key.anchor]
        d2 = sum(0.0 if m <= 0.0 <= M else min(m * m, M * M) for m, M in zip(mins, maxs))
        return d2 < rad * rad

    # (a) ball tree, DOM2, ppo 5, rk3 LTS/GTS + 3-rank partition (test_stepper style)
    tree = balance_2to1(construct(lambda k: ball_refine(k), 2, 4))
    a_anchor, a_level = tree_arrays(tree)
    out["ball_anchor"], out["ball_level"] = a_anchor, a_level
    mesh = Mesh(tree, points_per_octant=5, pad=2, domain=dom2)
    for k, v in mesh_arrays(mesh).items():
        out["ball_" + k] = v
    chi0 = wave.gaussian_pulse((0.0, 0.0), 0.8, 1.0)
    sub = {}
    run_fields(sub, mesh, chi0, [
        ("lts_rk3", "rk3", "lts", False, [1, 4, 8]),
        ("gts_rk3", "rk3", "gts", False, [1, 4]),
        ("lts_rk4", "rk4", "lts", False, [4, 8]),
        ("lts_rk2", "rk2", "lts", False, [4]),
        ("lts_euler", "euler", "lts", False, [4]),
        ("lts_sin", "rk3", "lts", "sin", [4]),
        ("lts_cubic", "rk4", "lts", "cubic", [4]),
    ], full=True)
    for k, v in sub.items():
        out["ball_" + k] = v
    # (b) random trees (test_mesh style), dims 2/3, default domain [0, 2^L]
    rng = np.random.default_rng(5)
    for dim in (2, 3):
        for t in range(2):
            tr = random_tree(rng, dim, 4 if dim == 2 else 3, ordering=SfcOrdering("morton", dim, 4 if dim == 2 else 3))
            for ppo in (5, 7):
                key = f"rnd{dim}d{t}_p{ppo}_"
                if t == 0 or ppo == 5:
                    an, lv = tree_arrays(tr)
                    out[key + "anchor"], out[key + "level"] = an, lv
                    m = Mesh(tr, points_per_octant=ppo, pad=2)
                    for k, v in mesh_arrays(m).items():
                        out[key + k] = v
    # (c) uniform tree, 4-rank gts partition (seams), ppo 5
    ut = uniform_tree(2, 3, 2, SfcOrdering("morton", 2, 3))
    pm = weighted_partition(ut, tree_weights(ut, "gts"), 4)
    m = Mesh(ut, points_per_octant=5, pad=2, pmap=pm, domain=dom2)
    for k, v in mesh_arrays(m).items():
        out["uni_" + k] = v
    # (d) constants: stencil weights and the RK4 transfer matrices the cfg1 run uses
    for nm in ("_D2_CENTER", "_D2_EDGE0", "_D2_EDGE1", "_D1_CENTER", "_D1_EDGE0", "_D1_EDGE1"):
        out["w" + nm] = getattr(wave, nm)
    tab = rkcorrect.get_tableau("rk4")
    dtf = 1.0 / 1024
    for key in [(0, 1, 2), (0, 2, 1), (0, 2, 4), (0, 4, 2), (1, 2, 1), (2, 4, 2), (1, 4, 1), (3, 4, 1)]:
        M = rkcorrect.stage_transfer_matrix(tab, key[0] * dtf, key[1] * dtf, key[2] * dtf)
        out["M_%d_%d_%d" % key] = M
    return out


CASES = {
    "cfg1": lambda: config_case("cfg1", [
        ("gts_rk4", "rk4", "gts", False, [1, 8, 512]),
        ("lts_rk4", "rk4", "lts", False, [1, 2, 8, 64, 512]),
        ("lts_cubic", "rk4", "lts", "cubic", [8, 64]),
        ("gts_cubic", "rk4", "gts", "cubic", [8]),
        ("lts_sin", "rk4", "lts", "sin", [8]),
        ("lts_rk3", "rk3", "lts", False, [8]),
    ], full=True),
    "mini3d": lambda: config_case("mini3d", [
        ("gts_rk4", "rk4", "gts", False, [1, 4]),
        ("lts_rk4", "rk4", "lts", False, [1, 4, 16]),
        ("lts_cubic", "rk4", "lts", "cubic", [4]),
    ], full=False, with_gathers=False),
    "small": small_cases,
}


def main(argv):
    names = argv or list(CASES)
    for name in names:
        path = os.path.join(HERE, f"{name}.npz")
        print(f"[golden] {name}", flush=True)
        t0 = time.time()
        data = CASES[name]()
        np.savez_compressed(path, **data)
        print(f"[golden] {name} -> {path} ({os.path.getsize(path) / 1e6:.2f} MB, {time.time() - t0:.0f}s)")


if __name__ == "__main__":
    main(sys.argv[1:])
