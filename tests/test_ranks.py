"""Host side of the multi-rank engine (CPU): per-rank layouts and programs,
shipment lists, and a world-size-2 gloo run of the shipment protocol.

The engine's ranks (stepper._Rank) hold owned + ghost leaves only, so every
node id in a rank's stage programs is rewritten to the rank's layout.  These
tests decode the rewritten programs and map them back: they must read exactly
the zip nodes the single-rank programs read.  The shipment lists must deliver
every ghost leaf from its owner, and the packed prefix protocol (finest cadence
first) must fill exactly the ghosts of the leaves that stepped.  The device
path is tests/test_ranks_gpu.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import config_mesh

from paper_2011_10570_b200 import tileprog
from paper_2011_10570_b200.stepper import _Link, _Rank, _ship_lists


def _ranks(mesh, lts=True, split=False):
    lv = mesh.tree.arrays()[1].astype(np.int32)
    cad = lv if lts else np.full_like(lv, lv.max())
    rr = mesh.pmap.rank_ranges
    ranks = {r: _Rank(mesh, cad, lts, int(lv.max()), r, np.arange(*rr[r])) for r in range(len(rr))}
    lists = _ship_lists({r: rk.ghosts for r, rk in ranks.items()}, rr)
    for r, rk in ranks.items():
        rk.split = split
        sent = [v for (q, _), v in lists.items() if q == r]
        rk.layout(np.unique(np.concatenate(sent)) if sent else np.zeros(0, np.int64))
    return cad, ranks, lists


def _decoded(prog_like, t, l2g, if_gid, if_cad):
    d = tileprog.decode(prog_like, t)

    def g(src):
        if src is None:
            return None
        if isinstance(src, tuple):
            i = src[1]
            return ("pair", int(l2g[if_gid[i]]), int(if_cad[i]))
        return int(l2g[src])

    cells = {c: g(s) for c, s in d["cells"].items()}
    rows = sorted((c, tuple((g(s), w) for s, w in taps)) for c, taps in d["rows"])
    return int(l2g[d["g0"]]) if d["n_own"] else None, d["n_own"], cells, rows


@pytest.mark.parametrize("name,R,lts,split", [("cfg1", 2, True, False), ("cfg1", 3, True, True), ("cfg1", 8, True, False),
                                              ("cfg1", 4, False, False), ("mini3d", 4, True, True)])
def test_rank_programs_read_the_same_nodes(name, R, lts, split):
    mesh = config_mesh(name, ranks=R)
    cad, ranks, lists = _ranks(mesh, lts, split)
    one = _Rank(mesh, cad, lts, int(cad.max()), 0, np.arange(len(cad)))
    one.layout(np.zeros(0, np.int64))
    assert one.identity and one.l2g is None
    ident = np.arange(mesh.n_nodes)
    ref = {}
    for t, leaf in enumerate(one.tiles):
        ref[int(leaf)] = _decoded(one.host, t, ident, one.host["if_gid"], one.host["if_cad"])
    seen = 0
    for r, rk in ranks.items():
        assert not rk.identity
        # local layout: owned + ghosts in leaf order, l2g a bijection onto their gids
        want = np.concatenate([np.arange(mesh.leaf_starts[l], mesh.leaf_starts[l + 1]) for l in rk.local_leaves])
        assert np.array_equal(rk.l2g, want)
        assert rk.n_boundary == int(np.isin(rk.tiles, np.concatenate(
            [v for (q, _), v in lists.items() if q == r] or [np.zeros(0, np.int64)])).sum())
        # launch groups: (boundary | interior) x (full | lean), back to back, each finest cadence first;
        # with `split` the tiles on a physical face are the full groups
        an, lvl = mesh.tree.arrays()
        side = 1 << (mesh.L - lvl.astype(np.int64))
        on_face = np.any((an == 0) | (an + side[:, None] == (1 << mesh.L)), axis=1)
        pos = 0
        for part in (True, False):
            for full in (True, False):
                off, prefix = rk.groups[(part, full)]
                assert off == pos
                grp = rk.tiles[off: off + prefix[0]]
                pos += len(grp)
                assert np.all(np.diff(cad[grp]) <= 0)
                assert np.all((np.arange(off, off + len(grp)) < rk.n_boundary) == part)
                if split:
                    assert np.all(on_face[grp] == full)
                else:
                    assert not full or len(grp) == 0
                for c in range(int(cad.max()) + 1):
                    assert prefix[c] == int(np.sum(cad[grp] >= c))
        assert pos == len(rk.tiles)
        for t, leaf in enumerate(rk.tiles):
            got = _decoded(rk.host, t, rk.l2g, rk.host["if_gid"], rk.host["if_cad"])
            assert got == ref[int(leaf)], (r, int(leaf))
            seen += 1
    assert seen == len(cad)


@pytest.mark.parametrize("R", [2, 4, 8])
def test_ship_lists_deliver_every_ghost_once(R):
    mesh = config_mesh("cfg1", ranks=R)
    cad, ranks, lists = _ranks(mesh)
    owners = mesh.pmap.owners(len(cad))
    for r, rk in ranks.items():
        got = np.sort(np.concatenate([v for (q, rr_), v in lists.items() if rr_ == r] or [np.zeros(0, np.int64)]))
        assert np.array_equal(got, rk.ghosts)
        assert len(rk.ghosts) > 0
        for (q, rr_), v in lists.items():
            if rr_ == r:
                assert np.all(owners[v] == q)
    # the owned cross reads a subset of the reference plan's block footprints (partition.py:147-175)
    plan = mesh.exchange_plan()
    for (q, r), v in lists.items():
        assert set(v.tolist()) <= {e.leaf for e in plan.entries.get((q, r), [])}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _np_move(rg, k, tot, rows, buf, unpack):
    """numpy statement of amr_ghost_pack / amr_ghost_unpack on (n_rows, n_local) rows."""
    start = rg.start.numpy()
    off = rg.off_host
    for j in range(k):
        a, n = int(start[j]), int(off[j + 1] - off[j])
        for r in range(rows.shape[0]):
            if unpack:
                rows[r, a:a + n] = buf[r * tot + off[j]: r * tot + off[j] + n]
            else:
                buf[r * tot + off[j]: r * tot + off[j] + n] = rows[r, a:a + n]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = config_mesh("cfg1", ranks=world)
        cad = mesh.tree.arrays()[1].astype(np.int32)
        rr = mesh.pmap.rank_ranges
        rk = _Rank(mesh, cad, True, int(cad.max()), rank, np.arange(*rr[rank]))
        gathered = [None] * world
        dist.all_gather_object(gathered, rk.ghosts.tolist())
        lists = _ship_lists({r: np.asarray(g, dtype=np.int64) for r, g in enumerate(gathered)}, rr)
        sent = [v for (s, _), v in lists.items() if s == rank]
        rk.layout(np.unique(np.concatenate(sent)) if sent else np.zeros(0, np.int64))
        cpu = torch.device("cpu")
        out = {r: _Link(v, cad, mesh.leaf_starts, rk.leaf_lstart, None, cpu, 2) for (s, r), v in lists.items() if s == rank}
        inc = {s: _Link(v, cad, mesh.leaf_starts, None, rk.leaf_lstart, cpu, 2) for (s, r), v in lists.items() if r == rank}
        truth = np.stack([rk.l2g.astype(np.float64), -rk.l2g.astype(np.float64)])
        own = np.zeros(rk.n_local, dtype=bool)
        own[rk.own_l0: rk.own_l0 + rk.own_g1 - rk.own_g0] = True
        ok = {}
        for tag, cmin in (("all", int(cad.min())), ("finest", int(cad.max()))):
            rows = np.where(own[None, :], truth, np.nan)
            ops, recvs = [], []
            for r, lk in out.items():
                k, tot = lk.send.prefix(cmin)
                if k:
                    buf = np.empty(2 * tot)
                    _np_move(lk.send, k, tot, rows, buf, False)
                    ops.append(dist.P2POp(dist.isend, torch.from_numpy(buf), r))
            for s, lk in inc.items():
                k, tot = lk.recv.prefix(cmin)
                if k:
                    hb = torch.empty(2 * tot, dtype=torch.float64)
                    ops.append(dist.P2POp(dist.irecv, hb, s))
                    recvs.append((lk, k, tot, hb))
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for lk, k, tot, hb in recvs:
                _np_move(lk.recv, k, tot, rows, hb.numpy(), True)
            expect = own.copy()
            for l in rk.ghosts:
                if cad[l] >= cmin:
                    expect[rk.leaf_lstart[l]: rk.leaf_lstart[l] + mesh.leaf_starts[l + 1] - mesh.leaf_starts[l]] = True
            ok[tag] = bool(np.array_equal(rows[:, expect], truth[:, expect]) and np.all(np.isnan(rows[:, ~expect])))
            ok[tag + "_n"] = int(expect.sum() - own.sum())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_shipments():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r]["all"] and res[r]["finest"], res
        assert res[r]["all_n"] > res[r]["finest_n"] > 0
