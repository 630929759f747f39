"""The native program builder (csrc/amr_programs.cpp) produces exactly the
bytes of the numpy specification (tileprog.build_programs): heads, tails,
interface pairs and the weight table, for LTS and GTS cadences."""
import numpy as np
import pytest

from helpers import config_mesh

from paper_2011_10570_b200 import tileprog as TP


@pytest.mark.parametrize("name,lts", [("cfg1", True), ("cfg1", False), ("mini3d", True), ("mini3d", False),
                                      ("cfg2", True)])
def test_native_programs_equal_numpy(name, lts):
    mesh = config_mesh(name)
    td = mesh.tile_data()
    n = len(mesh.tree.leaves)
    leaf_cad = td["level"].astype(np.int32) if lts else np.full(n, int(td["level"].max()), np.int32)
    node_cad = np.repeat(leaf_cad.astype(np.uint8), np.diff(td["starts"]))
    tiles = np.arange(n)[np.lexsort((np.arange(n), -leaf_cad))]
    want = TP.build_programs(td, tiles, leaf_cad, node_cad, lts)
    got = TP.build_programs_native(mesh, tiles, leaf_cad, lts)
    for k in ("max_head", "max_slots", "max_tail", "n_iface", "n_rows", "n_cells"):
        assert got[k] == want[k], k
    for k in ("heads", "tail", "if_gid", "if_cad", "wtab"):
        assert np.array_equal(np.asarray(got[k]), np.asarray(want[k])), k


def test_native_programs_subset_of_tiles():
    """A rank's tile subset (here every other leaf) encodes like the numpy path."""
    mesh = config_mesh("cfg1")
    td = mesh.tile_data()
    n = len(mesh.tree.leaves)
    leaf_cad = td["level"].astype(np.int32)
    node_cad = np.repeat(leaf_cad.astype(np.uint8), np.diff(td["starts"]))
    mine = np.arange(0, n, 2)
    tiles = mine[np.lexsort((mine, -leaf_cad[mine]))]
    want = TP.build_programs(td, tiles, leaf_cad, node_cad, True)
    got = TP.build_programs_native(mesh, tiles, leaf_cad, True)
    for k in ("heads", "tail", "if_gid", "if_cad", "wtab"):
        assert np.array_equal(np.asarray(got[k]), np.asarray(want[k])), k
