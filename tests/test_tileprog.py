"""CPU checks of the per-tile stage programs (paper_2011_10570_b200/tileprog.py):
decoding a tile's program must give back, cell for cell, the mesh's unzip
table on the owned cross — copies, LTS interface pairs and the hanging rows
with their taps in ascending-gid order (mesh.py:316-351, 391-393)."""
import numpy as np
import pytest

from helpers import config_mesh

from paper_2011_10570_b200 import tileprog as TP


def _programs(name, lts=True):
    mesh = config_mesh(name)
    td = mesh.tile_data()
    n_leaves = len(mesh.tree.leaves)
    leaf_cad = td["level"].astype(np.int32)
    node_cad = np.repeat(leaf_cad.astype(np.uint8), np.diff(td["starts"]))
    mine = np.arange(n_leaves)
    tiles = mine[np.lexsort((mine, -leaf_cad[mine]))]
    P = TP.build_programs(td, tiles, leaf_cad, node_cad, lts)
    return mesh, td, tiles, leaf_cad, node_cad, P


@pytest.mark.parametrize("name,lts", [("cfg1", True), ("cfg1", False), ("mini3d", True)])
def test_programs_decode_to_the_unzip_table(name, lts):
    mesh, td, tiles, leaf_cad, node_cad, P = _programs(name, lts)
    cells = TP.cross_cells(mesh.dim, mesh.ppo)
    ptr, gid, w = td["interp_ptr"], td["interp_gid"], td["interp_w"]
    starts = td["starts"]
    NI = mesh.ppo ** mesh.dim
    n_checked = 0
    for t, leaf in enumerate(tiles):
        dec = TP.decode(P, t)
        g0, g1 = starts[leaf], starts[leaf + 1]
        assert (dec["g0"], dec["n_own"]) == (g0, g1 - g0)
        row = td["table"][leaf]
        cell_src = dec["cells"]
        cell_row = {c: taps for c, taps in dec["rows"]}
        # every owned node is a copy of itself
        own_cells = {int(cells[e]) for e in range(NI) if g0 <= row[e] < g1}
        assert len(own_cells) == g1 - g0
        cad = leaf_cad[leaf]
        for e, c in enumerate(cells):
            c = int(c)
            v = int(row[e])
            if c in cell_src:
                s = cell_src[c]
                if isinstance(s, tuple):  # interface pair: same node, reader cadence = this tile's
                    assert lts and v >= 0 and node_cad[v] != cad
                    assert P["if_gid"][s[1]] == v and (P["if_cad"][s[1]] & 0xFF) == cad
                else:
                    assert s == v and (not lts or node_cad[v] == cad)
                n_checked += 1
            elif c in cell_row:
                assert v <= -2
                r = -v - 2
                want = list(zip(gid[ptr[r]:ptr[r + 1]].tolist(), w[ptr[r]:ptr[r + 1]].tolist()))
                got = [(s, wt) for s, wt in cell_row[c] if s is not None]
                pads = [(s, wt) for s, wt in cell_row[c] if s is None]
                assert all(wt == 0.0 for _, wt in pads) and len(cell_row[c]) % 4 == 0
                got_g = [(P["if_gid"][s[1]] if isinstance(s, tuple) else s) for s, _ in got]
                assert got_g == [g for g, _ in want] and [wt for _, wt in got] == [wt for _, wt in want]
            else:
                assert v == -1 or c not in own_cells  # never read by an owned stencil
        for c in own_cells:
            assert cell_src[c] in range(g0, g1)
    assert n_checked > 0


def test_program_buckets_and_needed_set():
    mesh, td, tiles, leaf_cad, node_cad, P = _programs("mini3d")
    h = P["heads"].view(np.int32)
    for t in range(len(tiles)):
        dec = TP.decode(P, t)
        b8, b4, b2, b1 = dec["buckets"]
        assert b8 + b4 + b2 + b1 == h[t, 3]
    # the owned cross: at most the stencil cross, at least the owned nodes
    assert P["n_cells"] < len(tiles) * TP.cross_cells(3, 9).size
    assert P["n_cells"] >= mesh.n_nodes


def test_needed_set_covers_every_stencil_read():
    """Brute force on a 2D tile set: every cell any owned node's stencil (centred
    or biased) reads is in the owned cross."""
    mesh = config_mesh("cfg1")
    td = mesh.tile_data()
    n = len(mesh.tree.leaves)
    tiles = np.arange(n)
    starts = td["starts"]
    table = td["table"].astype(np.int64)
    ppo, L = mesh.ppo, mesh.L
    a3 = td["anchor3"].astype(np.int64)
    side = 1 << (L - td["level"].astype(np.int64))
    faces = np.zeros(n, dtype=np.int64)
    for d in range(2):
        faces |= (a3[:, d] == 0).astype(np.int64) << (2 * d)
        faces |= ((a3[:, d] + side) == (1 << L)).astype(np.int64) << (2 * d + 1)
    need = TP.owned_cross(table, starts[:-1], starts[1:], faces, 2, ppo)
    cells = TP.cross_cells(2, ppo)
    RS = TP.box_strides(2, ppo)[0]
    for t in tiles:
        have = set(cells[need[t]].tolist())
        for e in range(ppo * ppo):
            if not starts[t] <= table[t, e] < starts[t + 1]:
                continue
            pos = [cells[e] // RS - 2, cells[e] % RS - 2]
            for d in range(2):
                lo, hi = (faces[t] >> (2 * d)) & 1, (faces[t] >> (2 * d + 1)) & 1
                p = pos[d]
                if lo and p <= 1:
                    offs = range(-p, 6 - p)
                elif hi and p >= ppo - 2:
                    offs = range(ppo - 6 - p, ppo - p)
                else:
                    offs = range(-2, 3)
                for o in offs:
                    q = list(pos)
                    q[d] += o
                    assert (q[0] + 2) * RS + q[1] + 2 in have, (t, e, d, o)
