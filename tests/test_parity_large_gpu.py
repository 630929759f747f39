"""GPU parity at BASELINE sizes against the CPU oracle (oracle/, pinned to
reference goldens in tests/test_oracle.py), plus size-independent properties.

cfg2 (configs[1], 3.67 M zip nodes) is compared bit for bit after one LTS
coarse round and after GTS steps.  Properties checked at full size:
uniform-mesh LTS == GTS bit-exact (a reference test, test_stepper.py:150-161),
the zero field as a fixed point, and linearity of the linear operator
(rank-count invariance at this size: tests/test_ranks_gpu.py)."""
import numpy as np
import pytest

from conftest import rel_linf
from helpers import config_mesh, config_tree

from paper_2011_10570_b200.configs import CONFIGS
from paper_2011_10570_b200.mesh import Domain, Mesh
from paper_2011_10570_b200.octree import SfcOrdering, uniform_tree
from paper_2011_10570_b200.stepper import Engine, compare_round

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg2():
    from oracle import oracle as O

    c = CONFIGS["cfg2"]
    tree = config_tree("cfg2")
    a, lv = tree.arrays()
    om = O.OracleMesh(c.dim, c.max_depth, a, lv, c.ppo, c.pad, c.domain_lo, c.domain_hi)
    return c, tree, config_mesh("cfg2", tree=tree), om


@pytest.mark.parametrize("mode,nl,slices", [("lts", False, 16), ("gts", False, 2), ("lts", "cubic", 16)])
def test_cfg2_matches_oracle_bit_exact(cuda, cfg2, mode, nl, slices):
    from oracle import oracle as O

    c, tree, mesh, om = cfg2
    assert mesh.n_nodes == om.n_nodes
    assert np.array_equal(mesh.leaf_slices, om.leaf_slices)
    eng = Engine(mesh, tableau="rk4", cfl=0.25, mode=mode, nonlinear=nl)
    eng.initialize(c.chi0())
    ref = O.OracleEngine(om, "rk4", 0.25, mode, nl)
    ref.initialize(c.chi0())
    assert eng.dt_fine == ref.dt_fine
    eng.run_to(slices)
    ref.run_to(slices)
    got, want = eng.current_zip(), ref.current_zip()
    assert rel_linf(got, want) <= 1e-12
    assert np.array_equal(got, want)


def test_uniform_3d_lts_equals_gts_bit_exact(cuda):
    tree = uniform_tree(3, 4, 4, SfcOrdering("morton", 3, 4))
    mesh = Mesh(tree, points_per_octant=9, pad=2, domain=Domain((-1.0,) * 3, (1.0,) * 3))
    chi0 = CONFIGS["mini3d"].chi0()
    lts = Engine(mesh, tableau="rk4", mode="lts")
    gts = Engine(mesh, tableau="rk4", mode="gts")
    lts.initialize(chi0)
    gts.initialize(chi0)
    for _ in range(3):
        assert compare_round(lts, gts) == 0.0


def test_zero_field_fixed_point_full_size(cuda, cfg2):
    _, _, mesh, _ = cfg2
    eng = Engine(mesh, tableau="rk4", mode="lts", nonlinear="cubic")
    eng.initialize(lambda *xs: 0 * xs[0])
    eng.lts_coarse_step()
    assert not np.any(eng.current_zip())


def test_linearity_full_size(cuda, cfg2):
    """The linear operator: E(a z1 + b z2) == a E(z1) + b E(z2) to rounding."""
    c, _, mesh, _ = cfg2
    xyz = mesh.node_physical()
    z1 = np.stack([np.exp(-np.sum(xyz ** 2, axis=1) / 0.01), np.zeros(mesh.n_nodes)])
    z2 = np.stack([np.sin(3 * xyz[:, 0]) * np.cos(2 * xyz[:, 1]), np.cos(xyz[:, 2])])
    outs = []
    for z in (z1, z2, 2.0 * z1 - 0.5 * z2):
        eng = Engine(mesh, tableau="rk4", mode="lts")
        eng.load_zip(z)
        eng.lts_coarse_step()
        outs.append(eng.current_zip())
    assert rel_linf(outs[2], 2.0 * outs[0] - 0.5 * outs[1]) <= 1e-12
