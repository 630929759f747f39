"""Goldens at BASELINE scale (test infrastructure; run here, where /root/reference exists).

    python tests/golden/make_golden_scale.py trees [cfg ...]   # reference construct/balance/partition
    python tests/golden/make_golden_scale.py fields [cfg ...]  # C oracle fields (oracle/, pinned in test_oracle.py)

Two kinds of fixture, both small enough to commit:

* ``scale_trees.json``: for cfg2..cfg5, digests of the leaf keys and levels
  *before* and *after* 2:1 balance, and the R = 2, 4, 8 partition cuts with
  LTS and GTS weights, computed by the UNMODIFIED reference (``amrlts.octree.
  construct`` / ``balance_2to1`` / ``amrlts.partition.weighted_partition``,
  octree.py:249-330, partition.py:20-91) on the frozen config predicates.
* ``scale_<cfg>.npz``: field snapshots of the C oracle (a restatement of
  ``amrlts.stepper.Engine``, bit-identical to the reference on every golden in
  tests/golden/*.npz — see tests/test_oracle.py) after one GTS step, one LTS
  coarse round, a pre-boundary time and (cfg2) the final time T = 1.0.  Each
  snapshot is (sha256 of the exact bytes with -0 -> +0, a strided sample,
  per-variable max|.|); the GPU tests compare the digest bit for bit and
  report the sampled relative error on a mismatch.  The Python reference cannot
  build these meshes (SURVEY §0 finding 6: > 25 min for cfg2's Mesh alone),
  so the oracle is the checker at this scale.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)

from paper_2011_10570_b200.configs import CONFIGS  # noqa: E402

# (mode, fine slices, label) snapshots per config.  cfg2: one round = 16
# slices, T = 1.0 = 2048 slices, T = 0.5 pre-boundary.  cfg3: one round = 32
# slices; 8 rounds (T = 0.125) is before the pulses reach the faces.  cfg4: a
# round is 2^(13-3) = 1024 slices (T ~ 0.0078, pre-boundary).  cfg5: one GTS
# step and the first LTS slices.
SNAPSHOTS = {
    "cfg2": [("gts", [1, 1024, 2048]), ("lts", [16, 1024, 2048]), ("lts-cubic", [16])],
    "cfg3": [("gts", [1]), ("lts", [32, 256])],
    "cfg4": [("gts", [1]), ("lts", [1024])],
    "cfg5": [("gts", [1]), ("lts", [4])],
}


def digest(z: np.ndarray) -> str:
    z = np.ascontiguousarray(z, dtype=np.float64) + 0.0
    return hashlib.sha256(z.tobytes()).hexdigest()


def tree_digest(anchors, levels) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(anchors, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(levels, dtype=np.int64).tobytes())
    return h.hexdigest()


def make_trees(names):
    sys.path.insert(0, REF)
    from amrlts.octree import SfcOrdering, balance_2to1, construct
    from amrlts.partition import tree_weights, weighted_partition

    path = os.path.join(HERE, "scale_trees.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        c = CONFIGS[name]
        t0 = time.time()
        raw = construct(c.refine, c.dim, c.max_depth, SfcOrdering("morton", c.dim, c.max_depth))
        t1 = time.time()
        bal = balance_2to1(raw)
        t2 = time.time()
        rec = {}
        for tag, tr in (("raw", raw), ("balanced", bal)):
            an = np.array([k.anchor for k in tr.leaves], dtype=np.int64)
            lv = np.array([k.level for k in tr.leaves], dtype=np.int64)
            rec[tag] = {"n": len(lv), "sha": tree_digest(an, lv),
                        "levels": {int(l): int(n) for l, n in zip(*np.unique(lv, return_counts=True))}}
        parts = {}
        for mode in ("lts", "gts"):
            w = tree_weights(bal, mode)
            for R in (2, 4, 8):
                pm = weighted_partition(bal, w, R)
                parts[f"{mode}{R}"] = [list(map(int, r)) for r in pm.rank_ranges]
        rec["partitions"] = parts
        rec["seconds"] = {"construct": round(t1 - t0, 1), "balance": round(t2 - t1, 1)}
        out[name] = rec
        print(name, rec["balanced"]["n"], rec["seconds"], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


def make_fields(names):
    from oracle import oracle as O

    for name in names:
        c = CONFIGS[name]
        t0 = time.time()
        an, lv = O.construct(c.refine, c.dim, c.max_depth)
        an, lv = O.balance(c.dim, c.max_depth, an, lv)
        m = O.OracleMesh(c.dim, c.max_depth, an, lv, c.ppo, c.pad, c.domain_lo, c.domain_hi)
        print(name, "oracle mesh", len(lv), "leaves", m.n_nodes, "nodes", round(time.time() - t0, 1), "s", flush=True)
        stride = max(1, m.n_nodes // 10000)
        data = {"n_nodes": np.int64(m.n_nodes), "n_leaves": np.int64(len(lv)), "stride": np.int64(stride),
                "leaf_slices_sha": np.array(hashlib.sha256(
                    np.ascontiguousarray(m.leaf_slices, dtype=np.int64).tobytes()).hexdigest())}
        for spec, slices in SNAPSHOTS[name]:
            mode, _, nl = spec.partition("-")
            nonlinear = nl or c.nonlinear
            e = O.OracleEngine(m, c.tableau, c.cfl, mode, nonlinear)
            e.initialize(c.chi0())
            for s in slices:
                t1 = time.time()
                e.run_to(s)
                z = e.current_zip()
                key = f"{spec}_{s}"
                data[key + "__sha"] = np.array(digest(z))
                data[key + "__sample"] = np.ascontiguousarray(z[:, ::stride])
                data[key + "__max"] = np.max(np.abs(z), axis=1)
                print(name, key, "max", data[key + "__max"], round(time.time() - t1, 1), "s", flush=True)
            del e
        # AMR_GOLDEN_OUT: write elsewhere (cfg4 needs more host memory than this container has: it is
        # generated on the GPU box, whose copy of the repo is scratch, and brought back in gpurun_out/)
        np.savez_compressed(os.path.join(os.environ.get("AMR_GOLDEN_OUT", HERE), f"scale_{name}.npz"), **data)
        del m


if __name__ == "__main__":
    what, names = sys.argv[1], sys.argv[2:] or ["cfg2", "cfg3", "cfg4", "cfg5"]
    {"trees": make_trees, "fields": make_fields}[what](names)
