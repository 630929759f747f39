"""GPU parity against goldens produced by the unmodified reference Engine.

Tolerances (BASELINE.json north_star): relative L-inf <= 1e-12 after one
step / round, <= 1e-10 at the final time.  The kernels follow the reference's
operation order, so linear and cubic runs are expected to be bit-exact; the
sin source differs by libm-vs-CUDA ulps and is held to the tolerance only.
"""
import numpy as np
import pytest

from conftest import compare_field, golden
from helpers import config_mesh

from paper_2011_10570_b200.configs import CONFIGS
from paper_2011_10570_b200.mesh import Domain, Mesh
from paper_2011_10570_b200.octree import LinearOctree, SfcOrdering
from paper_2011_10570_b200.stepper import Engine
from paper_2011_10570_b200.wave import gaussian_pulse

pytestmark = pytest.mark.gpu

RUNS = {  # tag -> (tableau, mode, nonlinear)
    "gts_rk4": ("rk4", "gts", False), "lts_rk4": ("rk4", "lts", False),
    "lts_cubic": ("rk4", "lts", "cubic"), "gts_cubic": ("rk4", "gts", "cubic"),
    "lts_sin": ("rk4", "lts", "sin"), "lts_rk3": ("rk3", "lts", False),
    "gts_rk3": ("rk3", "gts", False), "lts_rk2": ("rk2", "lts", False), "lts_euler": ("euler", "lts", False),
}


def _checkpoints(gd, prefix, tag):
    out = []
    for k in gd.files:
        if k.startswith(f"{prefix}{tag}_i"):
            stem = k[len(prefix) + len(tag) + 2:].split("__")[0]
            if stem.isdigit():
                out.append(int(stem))
    return sorted(set(out))


def _run_case(mesh, chi0, gd, prefix, tag, results, runs=RUNS):
    tab, mode, nl = runs[tag]
    eng = Engine(mesh, tableau=tab, cfl=0.25, mode=mode, nonlinear=nl)
    eng.initialize(chi0)
    assert eng.dt_fine == float(gd[f"{prefix}{tag}_dt_fine"])
    for cp in _checkpoints(gd, prefix, tag):
        eng.run_to(cp)
        exact, rel = compare_field(eng.current_zip(), gd, f"{prefix}{tag}_i{cp}")
        results.append((tag, cp, exact, rel))
    return eng


def _assert_results(results, final_tol=1e-10, first_tol=1e-12):
    for tag, cp, exact, rel in results:
        tol = first_tol if cp <= 8 else final_tol
        assert rel <= tol, (tag, cp, rel)
        if "sin" not in tag:
            assert exact, f"{tag} at slice {cp} not bit-exact (rel {rel:.3e})"


@pytest.mark.parametrize("tag", ["gts_rk4", "lts_rk4", "lts_cubic", "gts_cubic", "lts_sin", "lts_rk3"])
def test_cfg1_fields_match_reference(cuda, tag):
    gd = golden("cfg1")
    mesh = config_mesh("cfg1")
    results = []
    _run_case(mesh, CONFIGS["cfg1"].chi0(), gd, "", tag, results)
    print(results)
    _assert_results(results)


@pytest.mark.parametrize("tag", ["gts_rk4", "lts_rk4", "lts_cubic"])
def test_mini3d_fields_match_reference(cuda, tag):
    gd = golden("mini3d")
    mesh = config_mesh("mini3d")
    results = []
    _run_case(mesh, CONFIGS["mini3d"].chi0(), gd, "", tag, results)
    print(results)
    _assert_results(results)


@pytest.mark.parametrize("tag", ["lts_rk3", "gts_rk3", "lts_rk4", "lts_rk2", "lts_euler", "lts_sin", "lts_cubic"])
def test_ball_dom2_fields_match_reference(cuda, tag):
    """Reference-test geometry: [-10,10]^2, ppo 5 (non-dyadic h: true divisions)."""
    gd = golden("small")
    tree = LinearOctree.from_arrays(gd["ball_anchor"], gd["ball_level"], 2, 4, SfcOrdering("morton", 2, 4), True)
    mesh = Mesh(tree, points_per_octant=5, pad=2, domain=Domain((-10.0, -10.0), (10.0, 10.0)))
    results = []
    runs = dict(RUNS, lts_sin=("rk3", "lts", "sin"))  # make_golden.small_cases runs sin with rk3
    _run_case(mesh, gaussian_pulse((0.0, 0.0), 0.8, 1.0), gd, "ball_", tag, results, runs)
    print(results)
    _assert_results(results)


def test_graph_replayed_rounds_equal_eager(cuda):
    """lts_coarse_step replays captured CUDA graphs (two round parities); the
    result must be bit-identical to eager slices and to the reference."""
    gd = golden("cfg1")
    mesh = config_mesh("cfg1")
    outs, counts = [], []
    for graphs in (True, False):
        eng = Engine(mesh, tableau="rk4", cfl=0.25, mode="lts")
        eng.use_graphs = graphs
        eng.initialize(CONFIGS["cfg1"].chi0())
        for _ in range(8):  # eager warm-up rounds, capture, replays of both parities
            eng.lts_coarse_step()
        assert eng.i_fine == 64
        outs.append(eng.current_zip())
        counts.append((eng.counters.point_steps, dict(eng.counters.steps_by_level)))
    assert np.array_equal(outs[0], outs[1])
    assert counts[0] == counts[1]
    exact, rel = compare_field(outs[0], gd, "lts_rk4_i64")
    assert exact, rel


@pytest.mark.parametrize("threads", [128, 256])
@pytest.mark.parametrize("cfg,tag", [("cfg1", "gts_rk4"), ("cfg1", "lts_rk4"), ("cfg1", "lts_sin"),
                                     ("mini3d", "lts_rk4"), ("mini3d", "lts_cubic"), ("mini3d", "gts_rk4")])
def test_stage_kernel_block_shapes_match_reference(cuda, monkeypatch, cfg, tag, threads):
    """The owned-cross stage kernel with 128- and 256-thread CTAs (AMR_THREADS)
    is held to the same goldens."""
    monkeypatch.setenv("AMR_THREADS", str(threads))
    gd = golden(cfg)
    mesh = config_mesh(cfg)
    results = []
    eng = _run_case(mesh, CONFIGS[cfg].chi0(), gd, "", tag, results)
    assert eng._threads == threads
    _assert_results(results)


def test_unencodable_mesh_raises(cuda, monkeypatch):
    """A mesh that does not fit the compact per-tile encoding (here: a forced
    1-source-group limit) is refused with a ValueError, never run on a fallback."""
    monkeypatch.setenv("AMR_MAX_BASES", "1")  # read by the native program builder
    mesh = config_mesh("cfg1")
    with pytest.raises(ValueError, match="source groups"):
        Engine(mesh, tableau="rk4", mode="lts")


def test_async_current_zip_matches(cuda):
    """Engine.current_zip_to (the pipelined e2e read-back) returns the same
    bits as current_zip, and later load_zip/steps do not disturb a copy in
    flight."""
    import torch

    c = CONFIGS["cfg1"]
    eng = Engine(config_mesh("cfg1"), tableau="rk4", cfl=0.25, mode="lts", nonlinear=False, device=cuda)
    eng.initialize(c.chi0())
    eng.lts_coarse_step()
    want = eng.current_zip()
    out = torch.empty((2, eng.mesh.n_nodes), dtype=torch.float64).pin_memory()
    ev = eng.current_zip_to(out, torch.cuda.Stream(cuda))
    eng.load_zip(np.zeros_like(want))  # overwrite the live buffers right away
    eng.lts_coarse_step()
    ev.synchronize()
    assert np.array_equal(out.numpy(), want)


@pytest.mark.parametrize("name,nl", [("cfg1", False), ("mini3d", "cubic")])
def test_reload_after_steps_equals_a_fresh_engine(cuda, name, nl):
    """load_zip leaves the stage buffers of the previous run in place (every K_j is
    rewritten at slice 0 before anything reads it): a reloaded engine must step
    exactly like a fresh one, in eager slices and through the captured round graphs."""
    c = CONFIGS[name]
    mesh = config_mesh(name)
    fresh = Engine(mesh, tableau="rk4", cfl=c.cfl, mode="lts", nonlinear=nl, device=cuda)
    fresh.initialize(c.chi0())
    z0 = fresh.current_zip()
    used = Engine(mesh, tableau="rk4", cfl=c.cfl, mode="lts", nonlinear=nl, device=cuda)
    used.load_zip(3.0 * z0 + 0.25)  # another field, a few rounds: stale K, Y, u_pre everywhere
    for _ in range(3):
        used.lts_coarse_step()
    used.load_zip(z0)
    for _ in range(2):
        fresh.lts_coarse_step()
        used.lts_coarse_step()
        assert np.array_equal(fresh.current_zip(), used.current_zip())
    used.load_zip(z0)
    fresh.load_zip(z0)
    used.run_to(5)
    fresh.run_to(5)
    assert np.array_equal(fresh.current_zip(), used.current_zip())
