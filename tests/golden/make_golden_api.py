"""Goldens for the API kernels (run here, where /root/reference exists):

    python tests/golden/make_golden_api.py

``Mesh.unzip`` (mesh.py:413-420) and ``wave_rhs`` (wave.py:147-201) of the
UNMODIFIED reference on two meshes: the reference tests' [-10,10]^2 ball tree
(2D, ppo 5) and mini3d (3D, ppo 9, non-trivial domain faces), for a
synthetic zip field spanning seven decades (exact integer arithmetic, rebuilt
by the tests).  Stored: every block's padded unzip array (2D: flat with
offsets; 3D: sha256 per block) and, per block, the linear and the
sin-nonlinear RHS of that padded array (all blocks in 2D; the physical-face
blocks and a few interior ones in 3D).  -> tests/golden/api.npz
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from amrlts import wave  # noqa: E402
from amrlts.mesh import Domain, Mesh  # noqa: E402
from amrlts.octree import SfcOrdering, balance_2to1, construct  # noqa: E402

from paper_2011_10570_b200.configs import CONFIGS  # noqa: E402


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


def synthetic_zip(n: int) -> np.ndarray:
    """A (2, n) field spanning seven decades from exact integer arithmetic
    (bit-portable: no libm, no RNG stream): the tests rebuild it."""
    i = np.arange(n, dtype=np.int64)
    out = np.empty((2, n))
    for v, mul in enumerate((2654435761, 40503)):
        h = (i * mul + 12345 * (v + 1)) % (1 << 20) - (1 << 19)
        out[v] = (h.astype(np.float64) / 1024.0) * np.array([1e-3, 1e-2, 0.1, 1.0, 10.0, 100.0, 1e3])[(i + v) % 7]
    return out


def sha(a) -> str:
    import hashlib

    return hashlib.sha256((np.ascontiguousarray(a, dtype=np.float64) + 0.0).tobytes()).hexdigest()


def case(tag, mesh, rng, rhs_blocks, full_unzip=True):
    out = {}
    z = synthetic_zip(mesh.n_nodes)
    blocks = mesh.unzip(z)
    if full_unzip:
        out[f"{tag}_unzip"] = np.concatenate([b.reshape(2, -1) for b in blocks], axis=1)
    out[f"{tag}_unzip_sha"] = np.array([sha(b) for b in blocks])
    out[f"{tag}_unzip_off"] = np.concatenate([[0], np.cumsum([b[0].size for b in blocks])]).astype(np.int64)
    r_eps = mesh.finest_spacing()
    ids = list(rhs_blocks(mesh))
    out[f"{tag}_rhs_blocks"] = np.array(ids, dtype=np.int64)
    for nl in (False, True):
        res = []
        for i in ids:
            geom = wave.block_geometry(mesh, mesh.blocks[i], r_eps)
            res.append(wave.wave_rhs(blocks[i], geom, nl, 1.0, 2.0).reshape(2, -1))
        out[f"{tag}_rhs_{'sin' if nl else 'lin'}"] = np.concatenate(res, axis=1)
    return out


def main():
    rng = np.random.default_rng(20260)
    out = {}
    tree = balance_2to1(construct(lambda k: ball_refine(k), 2, 4))
    mesh = Mesh(tree, points_per_octant=5, pad=2, domain=Domain((-10.0, -10.0), (10.0, 10.0)))
    out.update(case("ball", mesh, rng, lambda m: range(len(m.blocks))))
    c = CONFIGS["mini3d"]
    tree = balance_2to1(construct(c.refine, c.dim, c.max_depth, SfcOrdering("morton", c.dim, c.max_depth)))
    mesh = Mesh(tree, points_per_octant=c.ppo, pad=c.pad, domain=Domain(c.domain_lo, c.domain_hi))

    def pick(m):
        face = [b.index for b in m.blocks if m.block_domain_faces(b)]
        inner = [b.index for b in m.blocks if not m.block_domain_faces(b)]
        return sorted(face[:10] + inner[:6])

    out.update(case("mini3d", mesh, rng, pick, full_unzip=False))
    np.savez_compressed(os.path.join(HERE, "api.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
