"""CPU checks of the compact tile blobs of the pipelined stage kernel
(paper_2011_10570_b200/tileprog.py): decoding every blob must give back the
tile table and interpolation program it was built from, exactly."""
import numpy as np
import pytest

from helpers import config_mesh

from paper_2011_10570_b200 import tileprog as TP
from paper_2011_10570_b200.stepper import Engine


def _programs(name, lts=True):
    mesh = config_mesh(name)
    td = mesh.tile_data()
    n_leaves = len(mesh.tree.leaves)
    leaf_cad = td["level"].astype(np.int32)
    node_cad = np.repeat(leaf_cad.astype(np.uint8), np.diff(td["starts"]))
    mine = np.arange(n_leaves)
    tiles = mine[np.lexsort((mine, -leaf_cad[mine]))].astype(np.int32)
    table, prog = Engine._tile_programs(td, tiles, node_cad, leaf_cad, lts=lts)
    n_iface = prog.pop("n_iface")
    B = TP.build_blobs(table, prog, n_iface, td["starts"], td["anchor3"], mesh.ppo ** mesh.dim, mesh.ppo + 4)
    return mesh, table, prog, B


def _decode_source(base, off):
    """table value of a (base, offset) source: a gid, or an interface pair code"""
    return base + off if base >= 0 else TP.IFACE_BASE - (-base - 1 + off)


@pytest.mark.parametrize("name", ["cfg1", "mini3d"])
def test_blobs_decode_to_the_tile_programs(name):
    mesh, table, prog, B = _programs(name)
    blob, off = B["blob"], B["blob_off"]
    nt, E = table.shape
    cells = prog["cross_cells"].astype(np.int64)
    cell_to_e = {int(c): e for e, c in enumerate(cells)}
    assert B["max_blob"] == int(B["blob_head"].max())
    heads = B["heads"]
    assert heads.shape == (nt, B["max_blob"])
    for t in range(nt):  # the fixed-stride copy of every head
        hb = int(B["blob_head"][t])
        assert np.array_equal(heads[t, :hb], blob.view(np.uint8)[off[t]:off[t] + hb])
        assert not heads[t, hb:].any()
    for t in range(nt):
        b = blob[off[t] // 2: off[t + 1] // 2]
        h = b[:32].view(np.int32)
        g0, n_own, lmeta, nrun, nslot, nrow, nbase, ln = h[:8]
        assert ln == len(b) and h[15] * 8 == off[t] // 2
        assert B["blob_head"][t] == 2 * h[11]
        bases = b[32:32 + 2 * nbase].view(np.int32)
        runs = b[32 + ((2 * nbase + 7) // 8) * 8:][:2 * nrun].view(np.uint32)
        got = np.full(E, -9, dtype=np.int64)
        for w in runs.astype(np.int64):
            cell, ln_, code = w & 0xFFF, ((w >> 12) & 15) + 1, w >> 16
            bi, o = code >> 10, code & 1023
            for i in range(ln_):
                e = cell_to_e[cell + i]
                got[e] = -1 if bi == 63 else _decode_source(int(bases[bi]), o + i)
        want = table[t].astype(np.int64)
        hang = (want <= -2) & (want > TP.IFACE_BASE)
        assert np.array_equal(got[~hang], want[~hang]), t
        assert np.all(got[hang] == -9)
        faces = (lmeta >> 16) & 0x3F
        if faces:  # face tiles keep per-entry codes (hanging row r -> offset r + 1)
            ent = b[h[11]:h[11] + E].astype(np.int64)
            r = ent[hang] & 1023
            assert np.all(ent[hang] >> 10 == 63) and np.array_equal(r - 1, -want[hang] - 2)
        # slots
        sl = b[h[12]:h[12] + nslot].astype(np.int64)
        sg = prog["slot_gid"][prog["tile_slot_ptr"][t]:prog["tile_slot_ptr"][t + 1]].astype(np.int64)
        for k in range(nslot):
            v = _decode_source(int(bases[sl[k] >> 10]), int(sl[k] & 1023))
            assert (v if v >= 0 else -(TP.IFACE_BASE - v) - 1) == sg[k]
        # rows and taps
        rows = b[h[13]:h[13] + 2 * nrow].view(np.uint32)
        taps = b[h[14]:].astype(np.int64)
        i0 = prog["tile_in_ptr"][t]
        for r in range(nrow):
            w = int(rows[r])
            assert (w & 0xFFF) == prog["in_cell"][i0 + r]
            k0, k1 = prog["in_tap_ptr"][i0 + r], prog["in_tap_ptr"][i0 + r + 1]
            nq, q0 = (w >> 12) & 31, w >> 17
            assert 4 * nq == k1 - k0
            tt = prog["tap"][k0:k1].astype(np.int64)
            tw = taps[4 * q0: 4 * q0 + 4 * nq]
            assert np.array_equal(tw >> 6, tt >> 16) and np.array_equal(tw & 63, tt & 0xFFFF)


def test_cell_entries_inverts_the_cross():
    cells = np.array([5, 0, 7], dtype=np.uint16)
    inv = TP.cell_entries(cells, 2, 1)  # a 5x5 box
    assert inv[5] == 0 and inv[0] == 1 and inv[7] == 2
    assert np.all(np.delete(inv, [0, 5, 7]) == 0xFFFF)
