"""Behaviour of the public API on the device, stated the way the reference's own
suite states it (pkg/tests/test_stepper.py, test_wave.py, test_mesh.py: the
checks that need Engine stepping, Mesh.unzip or wave_rhs and therefore a GPU
here).  These are this repo's statements of those properties, on its own
meshes; bit-level parity with the reference is in the golden tests."""
import numpy as np
import pytest

from paper_2011_10570_b200.mesh import Domain, Mesh, field_csv_rows, write_block_vtk
from paper_2011_10570_b200.octree import OctKey, SfcOrdering, balance_2to1, construct, uniform_tree
from paper_2011_10570_b200.perfmodel import estimate, histogram_from_mesh
from paper_2011_10570_b200.stepper import Engine, compare_round, lts_single_stage_engine
from paper_2011_10570_b200.wave import analytic_linear, block_geometry, gaussian_pulse, plane_pulse, wave_rhs

pytestmark = pytest.mark.gpu
DOM = Domain((-10.0, -10.0), (10.0, 10.0))


def _uniform(dim=2, level=2, lo=-10.0, hi=10.0, ppo=5):
    tree = uniform_tree(dim, level, level, SfcOrdering("morton", dim, level))
    return Mesh(tree, points_per_octant=ppo, pad=2, domain=Domain((lo,) * dim, (hi,) * dim))


def _centre_refined(depth=4, base=2, radius=3.0, ppo=5, dom=DOM):
    def near(key: OctKey) -> bool:
        if key.level < base:
            return True
        scale = (dom.hi[0] - dom.lo[0]) / (1 << key.max_depth)
        d2 = 0.0
        for a in key.anchor:
            lo, hi = dom.lo[0] + a * scale, dom.lo[0] + (a + key.side) * scale
            d2 += 0.0 if lo <= 0.0 <= hi else min(lo * lo, hi * hi)
        return key.level < depth and d2 < radius * radius

    tree = balance_2to1(construct(near, 2, depth, SfcOrdering("morton", 2, depth)))
    return Mesh(tree, points_per_octant=ppo, pad=2, domain=dom)


def _padded(mesh, fchi, fphi):
    """Per-block padded (2, ...) arrays of analytic fields (no unzip involved)."""
    out = []
    for b in mesh.blocks:
        grids = np.meshgrid(*mesh.block_axes(b), indexing="ij")
        out.append(np.stack([fchi(*grids), fphi(*grids)]))
    return out


# ---------------------------------------------------------------- wave_rhs
def test_rhs_of_the_zero_state_is_zero(cuda):
    mesh = _uniform()
    y = _padded(mesh, lambda x, y: 0 * x, lambda x, y: 0 * x)
    for b in mesh.blocks:
        assert not np.any(wave_rhs(y[b.index], block_geometry(mesh, b, 1e-9), False, 1.0, 2.0))


@pytest.mark.parametrize("dim", [2, 3])
def test_rhs_laplacian_of_a_quadratic_is_exact(cuda, dim):
    mesh = _uniform(dim=dim, level=1 if dim == 3 else 2, lo=1.0, hi=5.0)
    y = _padded(mesh, lambda *xs: sum(x * x for x in xs), lambda *xs: 3.0 + 0 * xs[0])
    b = mesh.blocks[0]
    out = wave_rhs(y[0], block_geometry(mesh, b, 1e-9), False, 1.0, 2.0)
    inner = (slice(1, b.interior_n - 1),) * dim  # off the radiative faces (one block covers the domain)
    assert np.allclose(out[0][inner], 3.0, rtol=0, atol=1e-12)          # dchi = phi
    assert np.allclose(out[1][inner], 2.0 * dim, rtol=1e-10)            # dphi = laplacian, biased rows included


def test_rhs_sin_source_closed_form_and_odd(cuda):
    mesh = _uniform(lo=2.0, hi=6.0)
    b = mesh.blocks[0]
    geom = block_geometry(mesh, b, 1e-9)
    inner = (slice(1, b.interior_n - 1),) * 2
    outs = []
    for c in (0.5, -0.5):
        y = _padded(mesh, lambda x, y, c=c: c + 0 * x, lambda x, y: 0 * x)
        outs.append(wave_rhs(y[0], geom, True, 1.0, 2.0)[1][inner])
    want = -np.sin(2 * 0.5) / geom.r2_reg[inner]
    assert np.allclose(outs[0], want, rtol=1e-12)
    assert np.allclose(outs[0], -outs[1], rtol=1e-12)


def test_radiative_faces(cuda):
    """On a physical face both variables relax: constant state f0 = 0 decays with -k f;
    a 1/r profile gives -1/r^2 - 1/r (one-sided 4th-order rows, wave.py:173-201)."""
    mesh = _uniform(lo=2.0, hi=6.0)
    b = mesh.blocks[0]
    geom = block_geometry(mesh, b, 1e-9)
    n = b.interior_n
    face = (0, slice(1, n - 1))
    y = _padded(mesh, lambda x, y: 1.5 + 0 * x, lambda x, y: -0.25 + 0 * x)
    out = wave_rhs(y[0], geom, False, 1.0, 2.0)
    assert np.allclose(out[0][face], -1.0 * 1.5, atol=1e-12) and np.allclose(out[1][face], -2.0 * -0.25, atol=1e-12)
    y = _padded(mesh, lambda x, y: 1.0 / np.sqrt(x * x + y * y), lambda x, y: 0 * x)
    out = wave_rhs(y[0], geom, False, 1.0, 2.0)
    r = geom.r[face]
    assert np.max(np.abs(out[0][face] - (-1.0 / r ** 2 - 1.0 / r))) < 5e-4


# ---------------------------------------------------------------- unzip
def test_unzip_padding_copies_and_cubics(cuda):
    """Same-level padding is a copy of the neighbour's nodes; padding interpolated from a
    coarser leaf reproduces cubics (4-point Lagrange), and zip(unzip(z)) == z."""
    mesh = _centre_refined()
    xy = mesh.node_physical()
    poly = lambda x, y: 0.3 + x - 2 * y + 0.5 * x * y + 0.25 * x ** 3 - 0.125 * x * y * y  # noqa: E731
    z = np.stack([poly(xy[:, 0], xy[:, 1]), np.arange(mesh.n_nodes, dtype=float)])
    blocks = mesh.unzip(z)
    assert np.array_equal(mesh.zip(blocks), z)
    for b, arr in zip(mesh.blocks, blocks):
        gx, gy = np.meshgrid(*mesh.block_axes(b), indexing="ij")
        inside = (gx >= DOM.lo[0]) & (gx <= DOM.hi[0]) & (gy >= DOM.lo[1]) & (gy <= DOM.hi[1])
        g, n = b.pad, b.interior_n
        cross = np.zeros_like(inside)
        cross[g:g + n, :] = True
        cross[:, g:g + n] = True
        sel = inside & cross  # the stencil cross; corner padding is filled too but never read
        assert np.max(np.abs(arr[0][sel] - poly(gx, gy)[sel])) <= 1e-9 * np.max(np.abs(z[0]))
        assert np.all(arr[0][~inside] == 0.0)  # outside the domain: empty rows


def test_vtk_and_csv_rows(cuda):
    mesh = _uniform()
    blocks = mesh.unzip(np.stack([np.arange(mesh.n_nodes, dtype=float), np.zeros(mesh.n_nodes)]))
    text = write_block_vtk(mesh, mesh.blocks[0], blocks[0][0])
    assert text.startswith("# vtk DataFile") and "RECTILINEAR_GRID" in text
    rows = list(field_csv_rows(mesh, blocks))
    assert len(rows) == sum(b.interior_points for b in mesh.blocks) and len(rows[0]) == 4


# ---------------------------------------------------------------- engine
@pytest.mark.parametrize("mode", ["lts", "gts"])
def test_zero_field_is_a_fixed_point(cuda, mode):
    eng = Engine(_centre_refined(), mode=mode, tableau="rk3")
    eng.initialize(lambda x, y: 0 * x)
    for _ in range(eng.schedule.slices_per_round):
        eng.advance_slice()
    assert not np.any(eng.current_zip())


def test_mode_and_schedule_errors(cuda):
    mesh = _centre_refined()
    gts = Engine(mesh, mode="gts")
    gts.initialize(gaussian_pulse((0.0, 0.0), 0.8, 1.0))
    with pytest.raises(ValueError, match="CFL"):
        gts.gts_step(dt=2.0 * gts.dt_fine)
    gts.gts_step(dt=gts.dt_fine)
    lts = Engine(mesh, mode="lts")
    lts.initialize(gaussian_pulse((0.0, 0.0), 0.8, 1.0))
    with pytest.raises(RuntimeError):
        lts.gts_step()
    lts.advance_slice()
    with pytest.raises(RuntimeError, match="synchron"):
        lts.lts_coarse_step()
    with pytest.raises(ValueError):
        Engine(mesh, mode="both")
    with pytest.raises(ValueError):
        lts_single_stage_engine(mesh, tableau="rk3")


def test_uniform_mesh_lts_equals_gts_bit_for_bit(cuda):
    mesh = _uniform(level=3)
    a, b = Engine(mesh, mode="lts", tableau="rk3"), Engine(mesh, mode="gts", tableau="rk3")
    for e in (a, b):
        e.initialize(gaussian_pulse((0.0, 0.0), 2.0, 1.0))
    for _ in range(4):
        assert compare_round(a, b) == 0.0


def test_counters_follow_the_work_model(cuda):
    """After one coarse round: a level-l block has stepped 2^(l - l_min) times, and the
    point-steps are perfmodel's W_lts (LTS) and W_gts (GTS) (stepper.py:451-453, perfmodel.py:52-71)."""
    mesh = _centre_refined()
    lts, gts = Engine(mesh, mode="lts"), Engine(mesh, mode="gts")
    for e in (lts, gts):
        e.initialize(gaussian_pulse((0.0, 0.0), 0.8, 1.0))
    lts.lts_coarse_step()
    for _ in range(lts.schedule.slices_per_round):
        gts.gts_step()
    lmin = min(b.leaf_level for b in mesh.blocks)
    nb = {}
    for b in mesh.blocks:
        nb[b.leaf_level] = nb.get(b.leaf_level, 0) + 1
    assert dict(lts.counters.steps_by_level) == {lvl: n << (lvl - lmin) for lvl, n in nb.items()}
    est = estimate(histogram_from_mesh(mesh.blocks))
    assert lts.counters.point_steps == est.w_lts and gts.counters.point_steps == est.w_gts
    assert sum(lts.counters.rhs_evals.values()) == lts.p * sum(n << (lvl - lmin) for lvl, n in nb.items())


def test_lts_tracks_gts_while_the_interfaces_are_quiet(cuda):
    mesh = _centre_refined()
    lts, gts = Engine(mesh, mode="lts", tableau="rk3"), Engine(mesh, mode="gts", tableau="rk3")
    for e in (lts, gts):
        e.initialize(gaussian_pulse((0.0, 0.0), 0.4, 1.0))  # exp(-56) at the first level interface
    assert lts.schedule.delta_l >= 1
    assert compare_round(lts, gts) <= 1e-12


def test_plane_wave_error_drops_with_resolution(cuda):
    """chi(x, t) = (f(x - t) + f(x + t)) / 2 for a plane pulse, away from the faces
    (whose radiative rows assume a radial wave): the error at the same physical
    time falls with the mesh depth."""
    errs = []
    for level in (4, 5):
        mesh = _uniform(level=level, lo=-40.0, hi=40.0, ppo=5)
        eng = Engine(mesh, mode="gts", tableau="rk3", cfl=0.25)
        prof = lambda x: np.exp(-(x ** 2) / 4.0)  # noqa: E731
        eng.initialize(plane_pulse(0.0, 2.0, 1.0))
        for _ in range(int(round(0.5 / eng.dt_fine))):
            eng.gts_step()
        xy = mesh.node_physical()
        mid = (np.abs(xy[:, 0]) < 20.0) & (np.abs(xy[:, 1]) < 20.0)
        errs.append(np.max(np.abs(eng.current_zip()[0][mid] - analytic_linear(prof, eng.time, xy[mid, 0]))))
    assert errs[1] < errs[0] / 2.0 and errs[0] < 0.05


def test_single_stage_scheme(cuda):
    """The pseudo-timestep neighbour scheme (stepper.py:175-196): on a uniform mesh it is
    GTS Euler bit for bit; next to finer blocks a block steps at their cadence."""
    mesh = _uniform(level=3)
    a = lts_single_stage_engine(mesh)
    b = Engine(mesh, mode="gts", tableau="euler")
    for e in (a, b):
        e.initialize(gaussian_pulse((0.0, 0.0), 2.0, 1.0))
    assert compare_round(a, b) == 0.0
    mesh = _centre_refined()
    eng = lts_single_stage_engine(mesh)
    promoted = [b.index for b in mesh.blocks if eng.cadence[b.index] > b.leaf_level]
    assert promoted and all(eng.cadence[i] == mesh.blocks[i].leaf_level + 1 for i in promoted)
    eng.initialize(gaussian_pulse((0.0, 0.0), 0.8, 1.0))
    for _ in range(eng.schedule.slices_per_round):
        eng.advance_slice()
    i = promoted[0]
    assert eng.counters.rhs_evals[i] == 1 << (eng.cadence[i] - min(eng.cadence))
