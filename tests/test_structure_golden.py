"""Integer parity against reference goldens: Morton construct, 2:1 balance,
weighted partition, node registry (gids, leaf slices, coordinates), maximal
blocks, every gather CSR (bit-exact weights), read sets and exchange plans.
CPU only: the mesh builder is host C++ in the same C-ABI library."""
import numpy as np
import pytest

from conftest import gather_digests, golden
from helpers import config_mesh, config_tree

from paper_2011_10570_b200.configs import CONFIGS
from paper_2011_10570_b200.mesh import Domain, Mesh
from paper_2011_10570_b200.octree import LinearOctree, SfcOrdering, construct
from paper_2011_10570_b200.partition import build_exchange_plan, tree_weights, weighted_partition


def _check_mesh(mesh, gd, prefix=""):
    g = lambda k: gd[prefix + k]  # noqa: E731
    assert mesh.n_nodes == int(g("n_nodes"))
    assert np.array_equal(mesh.leaf_slices, g("leaf_slices"))
    assert np.array_equal(mesh.leaf_gids, g("leaf_gids"))
    assert np.array_equal(mesh.node_coords, g("node_coords"))
    assert np.array_equal(np.array([b.leaf_range for b in mesh.blocks]).reshape(-1, 2), g("block_leaf_range"))
    assert np.array_equal(np.array([b.root.level for b in mesh.blocks]), g("block_root_level"))
    assert np.array_equal(np.array([b.leaf_level for b in mesh.blocks]), g("block_leaf_level"))
    assert np.array_equal(np.array([b.root.anchor for b in mesh.blocks]).reshape(len(mesh.blocks), -1),
                          g("block_root_anchor").reshape(len(mesh.blocks), -1))
    assert mesh.finest_spacing() == float(g("finest_spacing"))
    assert gather_digests(mesh) == list(g("gather_digests"))
    reads = np.concatenate([mesh.block_read_leaves(b.index) for b in mesh.blocks])
    assert np.array_equal(reads, g("block_read"))


@pytest.mark.parametrize("name", ["cfg1", "mini3d"])
def test_construct_and_balance_bit_exact(name):
    gd = golden(name)
    c = CONFIGS[name]
    pre = construct(c.refine, c.dim, c.max_depth, SfcOrdering("morton", c.dim, c.max_depth))
    a, lv = pre.arrays()
    assert np.array_equal(a, gd["pre_anchor"]) and np.array_equal(lv, gd["pre_level"])
    tree = config_tree(name)
    a, lv = tree.arrays()
    assert np.array_equal(a, gd["anchor"]) and np.array_equal(lv, gd["level"])


@pytest.mark.parametrize("name", ["cfg1", "mini3d"])
def test_partition_bit_exact(name):
    gd = golden(name)
    tree = config_tree(name)
    for key in gd.files:
        if key.startswith("part_"):
            _, mode, R = key.split("_")
            pm = weighted_partition(tree, tree_weights(tree, mode), int(R))
            assert np.array_equal(np.array(pm.rank_ranges), gd[key]), key


@pytest.mark.parametrize("name", ["cfg1", "mini3d"])
def test_mesh_registry_and_gathers_bit_exact(name):
    _check_mesh(config_mesh(name), golden(name))


@pytest.mark.parametrize("name", ["cfg1", "mini3d"])
def test_rank_split_blocks_and_exchange_plan(name):
    gd = golden(name)
    tree = config_tree(name)
    pm = weighted_partition(tree, tree_weights(tree, "lts"), 4)
    c = CONFIGS[name]
    mesh = Mesh(tree, points_per_octant=c.ppo, pad=2, pmap=pm, domain=Domain(c.domain_lo, c.domain_hi))
    assert np.array_equal(np.array([b.leaf_range for b in mesh.blocks]), gd["r4_block_leaf_range"])
    assert np.array_equal(np.array([b.owner_rank for b in mesh.blocks]), gd["r4_block_owner"])
    rows = []
    for (s, r), items in sorted(build_exchange_plan(mesh, pm).entries.items()):
        for e in items:
            rows.append((s, r, e.leaf, e.node_start, e.node_stop, e.sender_block, len(e.receiver_blocks)))
    assert np.array_equal(np.array(rows, dtype=np.int64).reshape(-1, 7), gd["r4_plan"])


def _tree(gd, prefix, dim, L):
    return LinearOctree.from_arrays(gd[prefix + "anchor"], gd[prefix + "level"], dim, L,
                                    SfcOrdering("morton", dim, L), balanced=True)


def test_reference_test_meshes_bit_exact():
    gd = golden("small")
    tree = _tree(gd, "ball_", 2, 4)
    _check_mesh(Mesh(tree, points_per_octant=5, pad=2, domain=Domain((-10.0, -10.0), (10.0, 10.0))), gd, "ball_")
    for dim, L in ((2, 4), (3, 3)):
        for t in range(2):
            for ppo in (5, 7):
                pre = f"rnd{dim}d{t}_p{ppo}_"
                if pre + "anchor" not in gd.files:
                    continue
                _check_mesh(Mesh(_tree(gd, pre, dim, L), points_per_octant=ppo, pad=2), gd, pre)
    ut = _tree(gd, "uni_", 2, 3) if "uni_anchor" in gd.files else None
    if ut is not None:
        pm = weighted_partition(ut, tree_weights(ut, "gts"), 4)
        _check_mesh(Mesh(ut, points_per_octant=5, pad=2, pmap=pm, domain=Domain((-10.0, -10.0), (10.0, 10.0))),
                    gd, "uni_")


def test_random_trees_regenerate_identically():
    """random_tree draws the same seeds and yields the same balanced leaves."""
    from paper_2011_10570_b200.octree import random_tree

    gd = golden("small")
    rng = np.random.default_rng(5)
    for dim in (2, 3):
        for t in range(2):
            L = 4 if dim == 2 else 3
            tr = random_tree(rng, dim, L, ordering=SfcOrdering("morton", dim, L))
            a, lv = tr.arrays()
            pre = f"rnd{dim}d{t}_p5_"
            assert np.array_equal(a, gd[pre + "anchor"]) and np.array_equal(lv, gd[pre + "level"])


def test_stencil_weights_bit_exact():
    from paper_2011_10570_b200 import wave

    gd = golden("small")
    for nm in ("_D2_CENTER", "_D2_EDGE0", "_D2_EDGE1", "_D1_CENTER", "_D1_EDGE0", "_D1_EDGE1"):
        assert np.array_equal(getattr(wave, nm).view(np.int64), gd["w" + nm].view(np.int64)), nm


def test_transfer_matrices_bit_exact():
    from paper_2011_10570_b200.rkcorrect import get_tableau, stage_transfer_matrix

    gd = golden("small")
    tab = get_tableau("rk4")
    dtf = 1.0 / 1024
    for k in gd.files:
        if k.startswith("M_"):
            d, f, t = (int(x) for x in k[2:].split("_"))
            M = stage_transfer_matrix(tab, d * dtf, f * dtf, t * dtf)
            assert np.array_equal(M.view(np.int64), gd[k].view(np.int64)), k
