"""Octree build and 2:1 balance on the device (csrc/amr_octree.cu, octree.DeviceOctree).

With a CUDA device, ``construct`` and ``balance_2to1`` run as key-array rounds
on the GPU.  They must give the reference's leaves: the BASELINE configs against
the digests of the UNMODIFIED reference's construct / balance_2to1
(tests/golden/scale_trees.json, cfg2..cfg5: up to 1.22 M leaves) and against
the reference goldens of cfg1 / mini3d; random trees, 2D and 3D, Morton and
Hilbert, against the host ripple (amr_balance) and a brute-force balance check."""
import hashlib
import itertools
import json
import os
import time

import numpy as np
import pytest

from conftest import GOLDEN, golden

from paper_2011_10570_b200 import octree as OT
from paper_2011_10570_b200.configs import CONFIGS
from paper_2011_10570_b200.octree import OctKey, SfcOrdering, balance_2to1, construct, random_tree

pytestmark = pytest.mark.gpu

TREES = json.load(open(os.path.join(GOLDEN, "scale_trees.json")))


def _digest(tree):
    a, lv = tree.arrays()
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(lv, dtype=np.int64).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_device_trees_match_reference_digests(cuda, name):
    assert OT._device() is not None
    c = CONFIGS[name]
    want = TREES[name]
    t0 = time.time()
    raw = construct(c.refine, c.dim, c.max_depth, SfcOrdering("morton", c.dim, c.max_depth))
    t1 = time.time()
    bal = balance_2to1(raw)
    t2 = time.time()
    print(f"{name}: construct {t1 - t0:.2f} s, balance {t2 - t1:.2f} s, {len(bal)} leaves")
    assert len(raw) == want["raw"]["n"] and _digest(raw) == want["raw"]["sha"]
    assert len(bal) == want["balanced"]["n"] and _digest(bal) == want["balanced"]["sha"]
    assert bal.balanced and not raw.balanced


@pytest.mark.parametrize("name", ["cfg1", "mini3d"])
def test_device_trees_match_reference_goldens(cuda, name):
    gd = golden(name)
    c = CONFIGS[name]
    raw = construct(c.refine, c.dim, c.max_depth, SfcOrdering("morton", c.dim, c.max_depth))
    bal = balance_2to1(raw)
    for pre, tr in (("pre_", raw), ("", bal)):
        a, lv = tr.arrays()
        assert np.array_equal(a, gd[pre + "anchor"]) and np.array_equal(lv, gd[pre + "level"]), pre


def _brute_balanced(tree):
    a, lv = tree.arrays()
    side = (1 << (tree.max_depth - lv.astype(np.int64)))
    lo, hi = a.astype(np.int64), a.astype(np.int64) + side[:, None]
    for i in range(len(lv)):
        touch = np.all((lo <= hi[i]) & (lo[i] <= hi), axis=1)
        if np.any(np.abs(lv[touch] - lv[i]) > 1):
            return False
    return True


@pytest.mark.parametrize("dim,depth,kind", [(2, 6, "morton"), (3, 5, "morton"), (2, 5, "hilbert"), (3, 4, "hilbert")])
def test_device_balance_equals_host_ripple_on_random_trees(cuda, dim, depth, kind):
    for seed in range(6):
        rng = np.random.default_rng(seed)
        raw = random_tree(rng, dim, depth, n_clusters=4, balance=False, ordering=SfcOrdering(kind, dim, depth))
        dev = balance_2to1(raw)
        host = OT._balance_host(raw)
        assert _digest(dev) == _digest(host), (seed, len(dev), len(host))
        assert _brute_balanced(dev)
        # the device construct (callable predicate, one call per octant) equals the host construct
        if kind == "morton":
            seeds = [(tuple(int(x) for x in rng.integers(0, 1 << depth, dim)), int(rng.integers(2, depth + 1)))
                     for _ in range(3)]

            def refine(k: OctKey) -> bool:
                return k.level < 1 or any(k.level < d and all(a <= c < a + k.side for a, c in zip(k.anchor, cell))
                                          for cell, d in seeds)

            got = construct(refine, dim, depth, SfcOrdering("morton", dim, depth))
            want = OT._construct_host(refine, dim, depth, SfcOrdering("morton", dim, depth))
            assert _digest(got) == _digest(want)


def test_device_keys_roundtrip_and_order(cuda):
    import torch

    rng = np.random.default_rng(3)
    tree = random_tree(rng, 3, 6, n_clusters=5, ordering=SfcOrdering("morton", 3, 6))
    a, lv = tree.arrays()
    perm = rng.permutation(len(lv))
    t = OT.DeviceOctree.from_arrays(a[perm], lv[perm], 3, 6)
    t.sort()
    a2, lv2 = t.octants()
    assert np.array_equal(a2.cpu().numpy(), a) and np.array_equal(lv2.cpu().numpy(), lv)
    # ancestors sort before descendants with the same anchor code
    k = torch.tensor([(0 << 6) | 3, (0 << 6) | 1, (7 << 6) | 2], dtype=torch.int64)
    assert torch.sort(k).values.tolist() == [1, 3, (7 << 6) | 2]
