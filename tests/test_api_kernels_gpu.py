"""The API-side kernels against reference arrays (tests/golden/api.npz, made by
tests/golden/make_golden_api.py from the UNMODIFIED reference):

* ``Mesh.unzip`` (amr_gather_rows) == the reference's padded block arrays
  (mesh.py:413-420), bit for bit, 2D ppo 5 and 3D ppo 9;
* ``wave.wave_rhs`` (amr_block_rhs) == the reference's ``wave_rhs``
  (wave.py:147-201) on those padded arrays: linear bit for bit (interior,
  biased rows, radiative faces), sin-nonlinear within 1e-12 relative (libm vs
  CUDA sin, the north_star one-step tolerance);
* ``zip(unzip(z)) == z`` (reference test_mesh.py:114-125).
"""
import hashlib

import numpy as np
import pytest

from conftest import golden, rel_linf
from helpers import config_mesh

from paper_2011_10570_b200 import wave
from paper_2011_10570_b200.mesh import Domain, Mesh
from paper_2011_10570_b200.octree import balance_2to1, construct

pytestmark = pytest.mark.gpu


def synthetic_zip(n):
    i = np.arange(n, dtype=np.int64)
    out = np.empty((2, n))
    for v, mul in enumerate((2654435761, 40503)):
        h = (i * mul + 12345 * (v + 1)) % (1 << 20) - (1 << 19)
        out[v] = (h.astype(np.float64) / 1024.0) * np.array([1e-3, 1e-2, 0.1, 1.0, 10.0, 100.0, 1e3])[(i + v) % 7]
    return out


def _sha(a):
    return hashlib.sha256((np.ascontiguousarray(a, dtype=np.float64) + 0.0).tobytes()).hexdigest()


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


def _meshes():
    tree = balance_2to1(construct(lambda k: ball_refine(k), 2, 4))
    yield "ball", Mesh(tree, points_per_octant=5, pad=2, domain=Domain((-10.0, -10.0), (10.0, 10.0)))
    yield "mini3d", config_mesh("mini3d")


@pytest.mark.parametrize("tag", ["ball", "mini3d"])
def test_unzip_and_rhs_match_reference(cuda, tag):
    gd = golden("api")
    mesh = dict(_meshes())[tag]
    z = synthetic_zip(mesh.n_nodes)
    blocks = mesh.unzip(z)
    off = gd[f"{tag}_unzip_off"]
    assert len(blocks) == len(off) - 1
    assert [_sha(b) for b in blocks] == [str(s) for s in gd[f"{tag}_unzip_sha"]]
    if f"{tag}_unzip" in gd.files:
        flat = np.concatenate([b.reshape(2, -1) for b in blocks], axis=1)
        assert np.array_equal(flat, gd[f"{tag}_unzip"])
    assert np.array_equal(mesh.zip(blocks), z)  # zip o unzip is the identity
    r_eps = mesh.finest_spacing()
    for nl, key in ((False, "lin"), (True, "sin")):
        want = gd[f"{tag}_rhs_{key}"]
        pos = 0
        for i in gd[f"{tag}_rhs_blocks"].tolist():
            geom = wave.block_geometry(mesh, mesh.blocks[i], r_eps)
            got = wave.wave_rhs(blocks[i], geom, nl, 1.0, 2.0).reshape(2, -1)
            w = want[:, pos: pos + got.shape[1]]
            pos += got.shape[1]
            if nl:
                assert rel_linf(got, w) <= 1e-12, (tag, i)
            else:
                assert np.array_equal(got, w), (tag, i, rel_linf(got, w))
        assert pos == want.shape[1]
