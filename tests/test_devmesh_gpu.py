"""Node registry, tile tables and interpolation rows built on the device
(csrc/amr_devmesh.cu) against the host passes (amr_mesh_build), bit for bit:
leaf_slices, leaf_gids, the n x E unzip table, the hanging-point codes and
every interpolation row (gids and weight bits), on cfg1 (2D), mini3d, random
2D/3D trees at ppo 5/7/9, and the BASELINE 3D configs cfg2/cfg3.  The host
passes are themselves pinned to the reference's registry and gather CSRs
(tests/test_structure_golden.py).  With a device present, Mesh uses the device
builder: the engine parity tests run on its tables."""
import time

import numpy as np
import pytest

from helpers import config_tree

from paper_2011_10570_b200 import _native
from paper_2011_10570_b200.configs import CONFIGS
from paper_2011_10570_b200.mesh import Domain, Mesh, device_tables
from paper_2011_10570_b200.octree import SfcOrdering, random_tree

pytestmark = pytest.mark.gpu
C = _native.C


def _host_tables(mesh):
    L, h = mesh._nm.lib, mesh._nm.h
    td = mesh.tile_data()
    return dict(starts=mesh.leaf_starts, leaf_gids=mesh.leaf_gids.astype(np.int32), table=td["table"],
                row_ptr=td["interp_ptr"], gid=td["interp_gid"][: td["interp_ptr"][-1]],
                w=td["interp_w"][: td["interp_ptr"][-1]])


def _compare(tree, ppo, cuda, monkeypatch):
    monkeypatch.setenv("AMR_HOST_MESH", "1")
    t0 = time.time()
    host = Mesh(tree, points_per_octant=ppo, pad=2)
    assert not host._nm.on_device
    want = _host_tables(host)
    t1 = time.time()
    got = {k: v.cpu().numpy() for k, v in device_tables(tree, ppo, 2, cuda).items()}
    t2 = time.time()
    for k in ("starts", "leaf_gids", "table", "row_ptr", "gid"):
        assert np.array_equal(got[k].reshape(-1), np.asarray(want[k]).reshape(-1)), k
    assert got["w"].tobytes() == np.ascontiguousarray(want["w"]).tobytes()  # weight bits
    monkeypatch.delenv("AMR_HOST_MESH")
    dev = Mesh(tree, points_per_octant=ppo, pad=2)
    assert dev._nm.on_device and dev.n_nodes == host.n_nodes
    assert [(b.root, b.leaf_level, b.leaf_range) for b in dev.blocks] == \
        [(b.root, b.leaf_level, b.leaf_range) for b in host.blocks]
    assert np.array_equal(dev.node_coords, host.node_coords)
    return t1 - t0, t2 - t1


@pytest.mark.parametrize("name", ["cfg1", "mini3d", "cfg2", "cfg3"])
def test_device_tables_equal_host_tables(cuda, monkeypatch, name):
    import torch

    c = CONFIGS[name]
    th, td = _compare(config_tree(name), c.ppo, torch.device("cuda", 0), monkeypatch)
    print(f"{name}: host passes {th:.2f} s, device passes {td:.2f} s")


@pytest.mark.parametrize("dim,depth,ppo", [(2, 5, 5), (2, 5, 9), (3, 4, 5), (3, 4, 7), (3, 4, 9)])
def test_device_tables_random_trees(cuda, monkeypatch, dim, depth, ppo):
    import torch

    for seed in range(3):
        tree = random_tree(np.random.default_rng(seed), dim, depth, n_clusters=4,
                           ordering=SfcOrdering("morton", dim, depth))
        _compare(tree, ppo, torch.device("cuda", 0), monkeypatch)


def test_hilbert_trees_use_the_host_builder(cuda):
    tree = random_tree(np.random.default_rng(1), 2, 4)  # default ordering: Hilbert
    mesh = Mesh(tree, points_per_octant=5, pad=2)
    assert not mesh._nm.on_device


@pytest.mark.parametrize("name", ["cfg1", "mini3d"])
def test_device_node_coordinates_and_initial_data(cuda, name):
    """node_physical_device == node_physical bit for bit; Engine.initialize(device_eval=True)
    differs from the host evaluation only by the rounding of exp (CUDA vs libm)."""
    from helpers import config_mesh

    from paper_2011_10570_b200.stepper import Engine

    c = CONFIGS[name]
    mesh = config_mesh(name)
    xs = mesh.node_physical_device()
    want = mesh.node_physical()
    for d in range(mesh.dim):
        assert np.array_equal(xs[d].cpu().numpy(), want[:, d])
    a = Engine(mesh, tableau="rk4", mode="lts")
    b = Engine(mesh, tableau="rk4", mode="lts")
    a.initialize(c.chi0())
    b.initialize(c.chi0(), device_eval=True)
    za, zb = a.current_zip(), b.current_zip()
    assert np.max(np.abs(za - zb)) <= 4e-16 * max(1.0, np.max(np.abs(za)))
