"""Wavelet refinement criterion on the GPU (amr_wavelet_coeff) against the
reference's goldens and the oracle, plus the reference's own test_wavelet.py
cases through the drop-in API."""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from paper_2011_10570_b200 import wavelet as W
from paper_2011_10570_b200.octree import OctKey, SfcOrdering, construct, uniform_tree
from wavelet_fields import FIELDS

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

G = golden("wavelet")
CASES = sorted(k[: -len("_meta")] for k in G.files if k.endswith("_meta") and not k.startswith("scale"))
LO, HI = (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)
CODE = {W.Flag.REFINE: 1, W.Flag.KEEP: 0, W.Flag.COARSEN: -1}


@pytest.mark.parametrize("case", CASES)
def test_device_coefficients_bit_exact(case):
    dim, L, npd = (int(x) for x in G[f"{case}_meta"][:3])
    v = torch.from_numpy(G[f"{case}_values"]).cuda()
    c, _ = W.coefficients_from_values(v, npd, dim)
    assert np.array_equal(c.cpu().numpy(), G[f"{case}_coeff"])


@pytest.mark.parametrize("case", CASES)
def test_refine_flags_and_coefficients_api(case):
    dim, L, npd, mnl, mxl, _ = (int(x) for x in G[f"{case}_meta"])
    f = FIELDS[str(G[f"{case}_field"])]
    an, lv = G[f"{case}_anchors"], G[f"{case}_levels"]
    c = W.wavelet_coefficients(f, an, lv, L, npd, LO[:dim], HI[:dim])
    assert np.array_equal(c, G[f"{case}_coeff"])
    from paper_2011_10570_b200.octree import LinearOctree

    tree = LinearOctree([OctKey(tuple(int(x) for x in a), int(l), L) for a, l in zip(an, lv)], dim, L,
                        SfcOrdering("morton", dim, L))
    pol = W.RefinePolicy(tolerance=float(G[f"{case}_tol"][0]), min_level=mnl, max_level=mxl)
    flags = W.refine_flags(f, tree, pol, npd, LO[:dim], HI[:dim])
    assert np.array_equal(np.array([CODE[x] for x in flags], dtype=np.int8), G[f"{case}_codes"])
    k = 0  # single-octant entry point
    assert W.wavelet_coefficient(f, tree.leaves[k], npd, LO[:dim], HI[:dim]) == G[f"{case}_coeff"][k]


@pytest.mark.parametrize("case", CASES)
def test_predicate_construction_matches_reference(case):
    dim, L, npd, mnl, mxl, Lb = (int(x) for x in G[f"{case}_meta"])
    f = FIELDS[str(G[f"{case}_field"])]
    pol = W.RefinePolicy(tolerance=float(G[f"{case}_tol"][0]), min_level=mnl, max_level=mxl)
    tree = construct(W.refinement_predicate(f, pol, npd, LO[:dim], HI[:dim]), dim, Lb, SfcOrdering("morton", dim, Lb))
    an, lv = tree.arrays()
    assert np.array_equal(an, G[f"{case}_tree_anchors"]) and np.array_equal(lv, G[f"{case}_tree_levels"])


@pytest.mark.parametrize("dim,npd", [(2, 3), (2, 7), (2, 15), (3, 5), (3, 7), (3, 9), (3, 11)])
def test_random_values_vs_oracle(dim, npd):
    """Values spanning 1e+-20, signed zeros, inf and NaN, many octants (several
    warps per CTA, grid-stride loop)."""
    rng = np.random.default_rng(dim * 100 + npd)
    n = 20000 if dim == 2 else 3000
    v = rng.standard_normal((n, npd ** dim)) * np.exp(rng.uniform(-46, 46, (n, 1)))
    v[1, 3] = np.nan
    v[2, 0] = np.inf
    v[3, :] = -0.0
    v[4, 5] = -np.inf
    v[5, 1] = np.nan  # an even-index-free slot (odd node) only
    c, _ = W.coefficients_from_values(torch.from_numpy(v).cuda(), npd, dim)
    want = O.wavelet_coeffs(v, npd, dim)
    got = c.cpu().numpy()
    assert np.array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(got[~np.isnan(got)], want[~np.isnan(want)])


def test_device_flags_modes():
    rng = np.random.default_rng(7)
    n, npd, dim = 5000, 7, 3
    v = rng.standard_normal((n, npd ** dim)) * np.exp(rng.uniform(-12, 2, (n, 1)))
    lv = rng.integers(0, 8, n).astype(np.int32)
    pol = W.RefinePolicy(tolerance=1e-2, coarsen_factor=0.25, min_level=2, max_level=6)
    c, fl = W.coefficients_from_values(torch.from_numpy(v).cuda(), npd, dim, torch.from_numpy(lv).cuda(), pol)
    want = O.wavelet_coeffs(v, npd, dim)
    assert np.array_equal(c.cpu().numpy(), want)
    assert np.array_equal(fl.cpu().numpy(), O.wavelet_flag_codes(want, lv, 1e-2, 0.25, 2, 6))
    _, sp = W.coefficients_from_values(torch.from_numpy(v).cuda(), npd, dim, torch.from_numpy(lv).cuda(), pol,
                                       mode="predicate")
    exp = np.where(lv < 2, 1, np.where(lv >= 6, 0, (want > 1e-2).astype(np.int8)))
    assert np.array_equal(sp.cpu().numpy(), exp)


def test_empty_and_chunked():
    assert W.wavelet_coefficients(FIELDS["gauss2"], np.zeros((0, 2)), 0, 4).shape == (0,)
    # more octants than one host chunk: exercises the double-buffered stream
    tree = uniform_tree(3, 6, 6)
    an, lv = tree.arrays()
    old = W._CHUNK_VALUES
    W._CHUNK_VALUES = 343 * 10000
    try:
        got = W.wavelet_coefficients(FIELDS["trig3"], an, lv, 6, 7, LO, HI)
    finally:
        W._CHUNK_VALUES = old
    sel = np.arange(0, len(an), 997)
    vals = np.stack([O.wavelet_samples(FIELDS["trig3"], tuple(int(x) for x in an[i]), int(lv[i]), 6, 7, LO, HI)
                     .reshape(-1) for i in sel])
    assert np.array_equal(got[sel], O.wavelet_coeffs(vals, 7, 3))


# --- the reference's own tests (tests/test_wavelet.py), through the drop-in API

def root2d(max_depth=2):
    return OctKey((0, 0), 0, max_depth)


def test_linear_field_reproduced():
    for f in (lambda x, y: 2 * x - 3 * y + 1, lambda x, y: x, lambda x, y: 0 * x + 5):
        assert W.wavelet_coefficient(f, root2d(), 7) <= 1e-13


def test_quadratic_hand_value_three_nodes():
    c = W.wavelet_coefficient(lambda x, y: x ** 2, OctKey((0, 0), 0, 1), 3, domain_lo=(0.0, 0.0),
                              domain_hi=(1.0, 1.0))
    assert c == pytest.approx(0.25, abs=1e-14)


def test_cubic_reproduced_with_seven_nodes():
    f = lambda x, y: x ** 3 - 2 * x * y ** 2 + y ** 3  # noqa: E731
    assert W.wavelet_coefficient(f, root2d(), 7) <= 1e-12 * 8.0 ** 3


def test_distant_gaussian_small():
    f = lambda x, y: np.exp(-((x - 6.0) ** 2 + y ** 2))  # noqa: E731
    assert W.wavelet_coefficient(f, OctKey((0, 0), 2, 2), 7) < 1e-5


def test_constant_field_coarsens():
    tree = uniform_tree(2, 3, 2)
    flags = W.refine_flags(lambda x, y: 0 * x + 3.0, tree, W.RefinePolicy(tolerance=1e-5, min_level=0, max_level=3))
    assert all(f is W.Flag.COARSEN for f in flags)
    flags2 = W.refine_flags(lambda x, y: 0 * x + 3.0, tree, W.RefinePolicy(tolerance=1e-5, min_level=2, max_level=3))
    assert all(f is W.Flag.KEEP for f in flags2)


def test_gaussian_flags_concentrate_on_pulse():
    tree = uniform_tree(2, 4, 2)
    f = lambda x, y: np.exp(-(x ** 2 + y ** 2))  # noqa: E731
    flags = W.refine_flags(f, tree, W.RefinePolicy(tolerance=1e-5, min_level=0, max_level=4),
                           domain_lo=(-10.0, -10.0), domain_hi=(10.0, 10.0))
    for key, flag in zip(tree.leaves, flags):
        cx = -10.0 + (key.anchor[0] + key.side / 2) / 16 * 20
        cy = -10.0 + (key.anchor[1] + key.side / 2) / 16 * 20
        if flag is W.Flag.REFINE:
            assert cx * cx + cy * cy < 50.0
        if cx * cx + cy * cy > 120.0:
            assert flag is not W.Flag.REFINE


def test_max_level_clamps_refine():
    tree = uniform_tree(2, 2, 2)
    flags = W.refine_flags(lambda x, y: np.sin(3 * x) * np.cos(2 * y), tree,
                           W.RefinePolicy(tolerance=1e-12, min_level=0, max_level=2))
    assert all(f is W.Flag.KEEP for f in flags)


@pytest.mark.parametrize("scale", [1.5, 3.0, 17.25, 1e4])
def test_flags_invariant_under_joint_scaling(scale):
    tree = uniform_tree(2, 3, 1)
    f = lambda x, y: np.exp(-((x - 4) ** 2 + (y - 4) ** 2) / 2.0)  # noqa: E731
    fs = lambda x, y: scale * f(x, y)  # noqa: E731
    base = W.RefinePolicy(tolerance=1e-4, min_level=0, max_level=3)
    scaled = W.RefinePolicy(tolerance=1e-4 * scale, min_level=0, max_level=3)
    assert W.refine_flags(f, tree, base) == W.refine_flags(fs, tree, scaled)


def test_predicate_drives_construction():
    f = lambda x, y: np.exp(-(x ** 2 + y ** 2) / 0.5)  # noqa: E731
    pol = W.RefinePolicy(tolerance=1e-4, min_level=1, max_level=4)
    tree = construct(W.refinement_predicate(f, pol, domain_lo=(-10.0, -10.0), domain_hi=(10.0, 10.0)), 2, 4)
    assert tree.min_level() >= 1 and tree.max_level() == 4
    for key in tree.leaves:
        if key.level == 4:
            cx = -10.0 + (key.anchor[0] + key.side / 2) / 16 * 20
            cy = -10.0 + (key.anchor[1] + key.side / 2) / 16 * 20
            assert cx * cx + cy * cy < 30.0


# --- the criterion on the evolved solution (remesh at synchronised times)

def test_leaf_lattice_matches_unzip_and_engine_flags():
    """Mesh.leaf_lattice_device equals the leaf's sub-box of Mesh.unzip (the
    reference-pinned gather), and Engine.wavelet_flags equals the oracle's
    coefficients and refine_flags rule on those samples."""
    from helpers import config_mesh
    from paper_2011_10570_b200.configs import CONFIGS
    from paper_2011_10570_b200.stepper import Engine

    mesh = config_mesh("cfg1")
    c = CONFIGS["cfg1"]
    eng = Engine(mesh, tableau="rk4", cfl=0.25, mode="lts", nonlinear=False, device=torch.device("cuda", 0))
    eng.initialize(c.chi0())
    eng.lts_coarse_step()
    z = eng.current_zip()
    lat = mesh.leaf_lattice_device(torch.from_numpy(z).cuda(), 0).cpu().numpy()
    blocks = mesh.unzip(z)
    ppo = mesh.ppo
    an, lv = mesh.tree.arrays()
    for i in range(0, len(an), 5):
        b = mesh.blocks[mesh.leaf_block[i]]
        org = mesh._block_org(b)
        step = mesh.leaf_spacing(b.leaf_level)
        off = [(int(an[i, d]) * mesh.scale - int(org[d])) // step for d in range(mesh.dim)]
        sub = blocks[mesh.leaf_block[i]][0][tuple(slice(o, o + ppo) for o in off)]
        assert np.array_equal(lat[i].reshape(sub.shape), sub + 0.0), i
    pol = W.RefinePolicy(tolerance=1e-3, min_level=3, max_level=6)
    coeff, codes = eng.wavelet_flags(pol)
    want = O.wavelet_coeffs(lat, ppo, mesh.dim)
    assert np.array_equal(coeff, want)
    assert np.array_equal(codes, O.wavelet_flag_codes(want, lv, 1e-3, 0.1, 3, 6))


# --- device-side sampling (device_eval=True: f gets CUDA tensors)

@pytest.mark.parametrize("dim,npd,L", [(2, 7, 7), (3, 5, 6), (3, 9, 5)])
def test_device_sample_coordinates_bit_exact(dim, npd, L):
    from paper_2011_10570_b200.octree import random_tree
    rng = np.random.default_rng(dim * 10 + npd)
    n = 300
    lv = rng.integers(0, L + 1, n).astype(np.int32)
    an = np.stack([(rng.integers(0, 1 << L, n) >> (L - lv)) << (L - lv) for _ in range(dim)], axis=1).astype(np.int64)
    lo, hi = (-1.0, -0.5, -2.0)[:dim], (1.0, 3.0, 0.25)[:dim]
    axes = W._sample_axes(an, lv, L, lo, hi, npd)
    for d in range(dim):
        host = W._sample_values(lambda *g: g[d], axes, npd)
        dev = W._device_samples(torch, lambda *g: g[d], torch.from_numpy(an).cuda(), torch.from_numpy(lv).cuda(),
                                L, lo, hi, npd)
        assert np.array_equal(dev.cpu().numpy(), host)


def test_device_eval_matches_host_path():
    """Fields of products and sums only (no transcendental) round the same in
    numpy and torch, so the device-sampled path must give the host path's bits."""
    f = lambda x, y, z: x * x * y - 0.5 * z * x + y * z * z * z + 0.25  # noqa: E731
    tree = uniform_tree(3, 4, 4)
    pol = W.RefinePolicy(tolerance=1e-4, min_level=1, max_level=4)
    host = W.refine_codes(f, tree, pol, 7, LO, HI)
    dev = W.refine_codes(f, tree, pol, 7, LO, HI, device_eval=True)
    assert np.array_equal(host, dev)
    an, lv = tree.arrays()
    assert np.array_equal(W.wavelet_coefficients(f, an, lv, 4, 7, LO, HI),
                          W.wavelet_coefficients(f, an, lv, 4, 7, LO, HI, device_eval=True))
    g = lambda x, y: x * y * y - 3.0 * x + y  # noqa: E731
    p2 = W.RefinePolicy(tolerance=1e-6, min_level=0, max_level=5)
    t_host = construct(W.refinement_predicate(g, p2, 5, LO[:2], HI[:2]), 2, 5, SfcOrdering("morton", 2, 5))
    t_dev = construct(W.refinement_predicate(g, p2, 5, LO[:2], HI[:2], device_eval=True), 2, 5,
                      SfcOrdering("morton", 2, 5))
    assert [k for k in t_host.leaves] == [k for k in t_dev.leaves]


def test_reference_coefficients_at_scale():
    """4 278 leaves of a 3D random tree: the reference's own coefficients and
    flags (no samples stored; the product's host sampling re-creates them)."""
    dim, L, npd, mnl, mxl = (int(x) for x in G["scale_meta"])
    an, lv = G["scale_anchors"], G["scale_levels"]
    c = W.wavelet_coefficients(FIELDS["trig3"], an, lv, L, npd, LO, HI)
    assert np.array_equal(c, G["scale_coeff"])
    from paper_2011_10570_b200.octree import LinearOctree

    tree = LinearOctree([OctKey(tuple(int(x) for x in a), int(l), L) for a, l in zip(an, lv)], dim, L,
                        SfcOrdering("morton", dim, L))
    codes = W.refine_codes(FIELDS["trig3"], tree, W.RefinePolicy(tolerance=6e-6, min_level=mnl, max_level=mxl),
                           npd, LO, HI)
    assert np.array_equal(codes, G["scale_codes"])
