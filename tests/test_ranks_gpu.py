"""Multi-rank engine on the device (reference: rank_records + _ship,
stepper.py:158-161, 318-333; test_stepper.py:234-245 rank-count invariance).

A partitioned mesh runs as R simulated ranks in one process: each rank holds
only its owned and ghost leaves, launches its own tiles (boundary tiles first),
and ghosts move after every stage and step through amr_ghost_pack ->
buffer copy -> amr_ghost_unpack.  Results must be bit-identical to one rank, for
any R, in eager slices and in CUDA-graph replay; cutting the shipments must
break that (so the test has teeth).  A 2-process gloo run on the same device
covers the torch.distributed transport (host staging instead of NCCL)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import compare_field, golden
from helpers import config_mesh, config_tree

from paper_2011_10570_b200.configs import CONFIGS
from paper_2011_10570_b200.stepper import Engine

pytestmark = pytest.mark.gpu


def _run(mesh, c, mode, nl, rounds, graphs=True):
    eng = Engine(mesh, tableau="rk4", cfl=c.cfl, mode=mode, nonlinear=nl)
    eng.use_graphs = graphs
    eng.initialize(c.chi0())
    outs = []
    for _ in range(rounds):
        if mode == "lts":
            eng.lts_coarse_step()
        else:
            eng.gts_step()
        outs.append(eng.current_zip())
    return eng, outs


@pytest.mark.parametrize("R", [2, 3, 4, 8])
@pytest.mark.parametrize("mode,nl", [("lts", False), ("gts", False), ("lts", "cubic")])
def test_cfg1_rank_count_invariance(cuda, R, mode, nl):
    c = CONFIGS["cfg1"]
    tree = config_tree("cfg1")
    _, want = _run(config_mesh("cfg1", tree=tree), c, mode, nl, 4)
    eng, got = _run(config_mesh("cfg1", ranks=R, mode=mode, tree=tree), c, mode, nl, 4)
    assert len(eng._rank_list) == R and eng.comm_bytes > 0
    assert all(len(rk.ghosts) for rk in eng._rank_list)
    assert sum(rk.n_local for rk in eng._rank_list) < R * eng.mesh.n_nodes  # owned + ghosts, not the global layout
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_cfg1_ranks_match_reference_golden(cuda):
    """R = 4 simulated ranks against the reference's own fields (cfg1 LTS, first checkpoint)."""
    gd = golden("cfg1")
    c = CONFIGS["cfg1"]
    eng = Engine(config_mesh("cfg1", ranks=4), tableau="rk4", cfl=c.cfl, mode="lts")
    eng.initialize(c.chi0())
    for i in (1, 2, 8, 64):
        eng.run_to(i)
        exact, rel = compare_field(eng.current_zip(), gd, f"lts_rk4_i{i}")
        assert exact, (i, rel)


def test_eager_slices_equal_graph_replay_with_ranks(cuda):
    c = CONFIGS["mini3d"]
    mesh = config_mesh("mini3d", ranks=4)
    _, a = _run(mesh, c, "lts", "cubic", 4, graphs=True)
    _, b = _run(mesh, c, "lts", "cubic", 4, graphs=False)
    _, w = _run(config_mesh("mini3d"), c, "lts", "cubic", 4)
    for x, y, z in zip(a, b, w):
        assert np.array_equal(x, y) and np.array_equal(x, z)


def test_without_shipments_results_differ(cuda, monkeypatch):
    from paper_2011_10570_b200 import stepper

    c = CONFIGS["cfg1"]
    tree = config_tree("cfg1")
    _, want = _run(config_mesh("cfg1", tree=tree), c, "lts", False, 1)
    monkeypatch.setattr(stepper._LocalTransport, "ship", lambda self, i, s, cmin: None)
    _, got = _run(config_mesh("cfg1", ranks=2, tree=tree), c, "lts", False, 1, graphs=False)
    assert not np.array_equal(got[0], want[0])


@pytest.mark.parametrize("R", [2, 4, 8])
def test_cfg2_rank_count_invariance(cuda, R):
    """BASELINE configs[1] at full size: R simulated ranks == 1 rank, bit for bit,
    after two LTS rounds (the second is a graph replay)."""
    c = CONFIGS["cfg2"]
    tree = config_tree("cfg2")
    _, want = _run(config_mesh("cfg2", tree=tree), c, "lts", False, 2)
    eng, got = _run(config_mesh("cfg2", ranks=R, tree=tree), c, "lts", False, 2)
    assert eng.comm_bytes > 0
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_profile_phase_buckets(cuda):
    c = CONFIGS["cfg1"]
    eng = Engine(config_mesh("cfg1", ranks=2), tableau="rk4", cfl=c.cfl, mode="lts", profile=True)
    eng.initialize(c.chi0())
    eng.lts_coarse_step()
    ms = eng.phase_ms()
    assert ms["rhs"] > 0 and ms["time_interp"] > 0 and ms["comm"] > 0
    from paper_2011_10570_b200 import report

    row = report.phase_row(eng)
    assert row[0] == 2 and row[1] == 0.0 and row[3] == ms["rhs"]
    work = report.work_rows(eng)
    nb = {lvl: sum(1 for b in eng.mesh.blocks if b.leaf_level == lvl) for lvl in (3, 4, 5, 6)}
    assert [w[0] for w in work] == [3, 4, 5, 6]
    assert [w[2] for w in work] == [nb[lvl] * (1 << (lvl - 3)) for lvl in (3, 4, 5, 6)]  # block-steps of one round
    assert report.parse_csv(report.to_csv(report.PHASES, [row]))[0] == list(report.PHASES)


WORKER = r"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.join(os.environ["AMR_ROOT"], "tests")); sys.path.insert(0, os.environ["AMR_ROOT"])
from helpers import config_mesh
from paper_2011_10570_b200.configs import CONFIGS
from paper_2011_10570_b200.stepper import Engine
dist.init_process_group("gloo")
torch.cuda.set_device(0)
c = CONFIGS["cfg1"]
eng = Engine(config_mesh("cfg1", ranks=dist.get_world_size()), tableau="rk4", cfl=c.cfl, mode="lts", process_group=True)
assert len(eng._rank_list) == 1 and eng.rank == dist.get_rank()
eng.initialize(c.chi0())
for _ in range(2):
    eng.lts_coarse_step()
z = eng.current_zip()
if dist.get_rank() == 0:
    np.save(os.environ["AMR_OUT"], z)
    assert eng.comm_bytes > 0
dist.barrier()
dist.destroy_process_group()
"""


def test_two_processes_gloo_on_one_device(cuda, tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    out = tmp_path / "z.npy"
    env = dict(os.environ, AMR_ROOT=root, AMR_OUT=str(out))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)]
    pr = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert pr.returncode == 0, pr.stdout[-2000:] + pr.stderr[-4000:]
    c = CONFIGS["cfg1"]
    _, want = _run(config_mesh("cfg1"), c, "lts", False, 2)
    assert np.array_equal(np.load(out), want[-1])


def test_more_ranks_than_leaves(cuda):
    """Empty ranks (weighted_partition with more ranks than the weights can split) run and change nothing."""
    from paper_2011_10570_b200.mesh import Domain, Mesh
    from paper_2011_10570_b200.octree import SfcOrdering, uniform_tree
    from paper_2011_10570_b200.partition import tree_weights, weighted_partition
    from paper_2011_10570_b200.wave import gaussian_pulse

    tree = uniform_tree(2, 2, 1, SfcOrdering("morton", 2, 2))
    dom = Domain((-1.0, -1.0), (1.0, 1.0))
    pm = weighted_partition(tree, tree_weights(tree, "lts"), 8)
    assert pm.has_empty_ranks
    outs = []
    for pmap in (None, pm):
        eng = Engine(Mesh(tree, points_per_octant=5, pad=2, pmap=pmap, domain=dom), tableau="rk4", mode="lts")
        eng.initialize(gaussian_pulse((0.1, -0.2), 0.3, 1.0))
        for _ in range(3):
            eng.lts_coarse_step()
        outs.append(eng.current_zip())
    assert np.array_equal(outs[0], outs[1])
