"""Generate tests/golden/wavelet.npz by running the UNMODIFIED reference
``amrlts.wavelet`` (read-only, /root/reference/pkg/src).

    python tests/golden/make_golden_wavelet.py

Cases (fields from tests/wavelet_fields.py, domain [-1,1]^D):
  * W<npd>: _lagrange_matrix(xs[::2], xs) for npd 3..15;
  * <case>_anchors/_levels/_values/_coeff/_codes: every leaf of a random
    tree, the reference's samples (octant_samples + f), its
    wavelet_coefficient and refine_flags (1 refine / 0 keep / -1 coarsen);
  * <case>_tree_anchors/_levels: construct(refinement_predicate(...)) leaves.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..")))

from amrlts.octree import SfcOrdering, construct, random_tree  # noqa: E402
from amrlts.wavelet import (Flag, RefinePolicy, _lagrange_matrix, octant_samples, refine_flags,  # noqa: E402
                            refinement_predicate, wavelet_coefficient)

from wavelet_fields import FIELDS  # noqa: E402

CODE = {Flag.REFINE: 1, Flag.KEEP: 0, Flag.COARSEN: -1}

# name: (field, dim, max_depth, npd, tree seed, unused, tolerance, min_level, max_level)
CASES = {
    "g2n7": ("gauss2", 2, 7, 7, 1, 6, 1e-4, 1, 6),
    "t2n5": ("trig2", 2, 6, 5, 2, 5, 1e-5, 0, 5),
    "c2n9": ("cubic2", 2, 5, 9, 3, 5, 1e-12, 0, 4),
    "g3n7": ("gauss3", 3, 6, 7, 4, 4, 1e-4, 1, 5),
    "t3n3": ("trig3", 3, 5, 3, 5, 4, 1e-3, 0, 4),
    "r3n9": ("rough3", 3, 5, 9, 6, 3, 1e-3, 1, 4),
}


def main():
    out = {}
    for npd in range(3, 16, 2):
        xs = np.linspace(0.0, 1.0, npd)
        out[f"W{npd}"] = _lagrange_matrix(xs[::2], xs)
    lo = (-1.0, -1.0, -1.0)
    hi = (1.0, 1.0, 1.0)
    for name, (fname, dim, L, npd, seed, lmax, tol, mnl, mxl) in CASES.items():
        f = FIELDS[fname]
        tree = random_tree(np.random.default_rng(seed), dim, L, n_clusters=3, base_level=1,
                           ordering=SfcOrdering("morton", dim, L))
        keys = tree.leaves
        vals = np.stack([np.asarray(f(*octant_samples(k, lo[:dim], hi[:dim], npd)), dtype=float).reshape(-1)
                         for k in keys])
        coeff = np.array([wavelet_coefficient(f, k, npd, lo[:dim], hi[:dim]) for k in keys])
        pol = RefinePolicy(tolerance=tol, min_level=mnl, max_level=mxl)
        codes = np.array([CODE[x] for x in refine_flags(f, tree, pol, npd, lo[:dim], hi[:dim])], dtype=np.int8)
        pred = refinement_predicate(f, pol, npd, lo[:dim], hi[:dim])
        built = construct(pred, dim, min(L, mxl + 1), SfcOrdering("morton", dim, min(L, mxl + 1)))
        out[f"{name}_meta"] = np.array([dim, L, npd, mnl, mxl, min(L, mxl + 1)], dtype=np.int64)
        out[f"{name}_tol"] = np.array([tol])
        out[f"{name}_field"] = np.array(fname)
        out[f"{name}_anchors"] = np.array([k.anchor for k in keys], dtype=np.int32)
        out[f"{name}_levels"] = np.array([k.level for k in keys], dtype=np.int32)
        out[f"{name}_values"] = vals
        out[f"{name}_coeff"] = coeff
        out[f"{name}_codes"] = codes
        out[f"{name}_tree_anchors"] = np.array([k.anchor for k in built.leaves], dtype=np.int32)
        out[f"{name}_tree_levels"] = np.array([k.level for k in built.leaves], dtype=np.int32)
        print(name, len(keys), "leaves;", np.bincount(codes + 1), "codes;", len(built.leaves), "built leaves")
    # a larger case without the samples (the GPU test re-samples through the
    # product's host path, pinned above): every leaf of a 3D random tree
    f = FIELDS["trig3"]
    L = 6
    tree = random_tree(np.random.default_rng(11), 3, L, n_clusters=6, base_level=4,
                       ordering=SfcOrdering("morton", 3, L))
    keys = tree.leaves
    pol = RefinePolicy(tolerance=6e-6, min_level=2, max_level=6)
    out["scale_meta"] = np.array([3, L, 7, 2, 6], dtype=np.int64)
    out["scale_anchors"] = np.array([k.anchor for k in keys], dtype=np.int32)
    out["scale_levels"] = np.array([k.level for k in keys], dtype=np.int32)
    out["scale_coeff"] = np.array([wavelet_coefficient(f, k, 7, lo, hi) for k in keys])
    out["scale_codes"] = np.array([CODE[x] for x in refine_flags(f, tree, pol, 7, lo, hi)], dtype=np.int8)
    print("scale", len(keys), "leaves;", np.bincount(out["scale_codes"] + 1), "codes")
    np.savez_compressed(os.path.join(HERE, "wavelet.npz"), **out)


if __name__ == "__main__":
    main()
