"""World-size-2 gloo test of the multi-rank ghost exchange (CPU, no GPU).

Each rank owns the weighted-Morton leaf range of cfg1 for 2 ranks and writes
only its own zip rows; after the exchange every ghost leaf the reference
exchange plan routes to a rank must hold the owner's values, and nothing else
may change.  This is the transport the Engine runs over NCCL after every stage
and step (stepper.GhostExchange)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from helpers import config_mesh

        from paper_2011_10570_b200.stepper import GhostExchange

        mesh = config_mesh("cfg1", ranks=world, mode="lts")
        owners = mesh.pmap.owners(len(mesh.tree.leaves))
        levels = mesh.tree.arrays()[1]
        n = mesh.n_nodes
        truth = np.stack([np.arange(n, dtype=np.float64), -np.arange(n, dtype=np.float64)])  # (2, n) zip layout
        node_owner = np.repeat(owners, np.diff(mesh.leaf_starts))
        t = torch.full((2, n), float("nan"), dtype=torch.float64)
        mine = torch.from_numpy(node_owner == rank)
        t[:, mine] = torch.from_numpy(truth)[:, mine]
        gx = GhostExchange(mesh.exchange_plan(), levels, mesh.leaf_starts, rank, None, torch.device("cpu"))
        gx.swap_from_cadence(t, int(levels.min()))
        got = t.numpy().T
        truth = truth.T
        expect_rows = np.zeros(n, dtype=bool)
        expect_rows[node_owner == rank] = True
        for peer, leaves in gx.recv.items():
            for l in leaves:
                expect_rows[mesh.leaf_starts[l]:mesh.leaf_starts[l + 1]] = True
        ok_vals = np.array_equal(got[expect_rows], truth[expect_rows])
        ok_rest = bool(np.all(np.isnan(got[~expect_rows])))
        # exact-cadence swap: only finest-level ghosts move
        t2 = torch.full((2, n), float("nan"), dtype=torch.float64)
        t2[:, mine] = torch.from_numpy(truth.T)[:, mine]
        lmax = int(levels.max())
        gx.swap_cadence(t2, lmax)
        fine_rows = np.zeros(n, dtype=bool)
        for peer, leaves in gx.recv.items():
            for l in leaves[levels[leaves] == lmax]:
                fine_rows[mesh.leaf_starts[l]:mesh.leaf_starts[l + 1]] = True
        g2 = t2.numpy().T
        ok_fine = np.array_equal(g2[fine_rows], truth[fine_rows]) and bool(
            np.all(np.isnan(g2[~fine_rows & (node_owner != rank)])))
        n_recv = int(sum(len(v) for v in gx.recv.values()))
        q.put((rank, ok_vals, ok_rest, ok_fine, n_recv))
    finally:
        dist.destroy_process_group()


def test_ghost_exchange_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_vals, ok_rest, ok_fine, n_recv in res:
        assert n_recv > 0, rank
        assert ok_vals and ok_rest and ok_fine, (rank, ok_vals, ok_rest, ok_fine)
