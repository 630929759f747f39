"""Wavelet refinement criterion: oracle and host logic against goldens made by
the reference itself (tests/golden/make_golden_wavelet.py).  CPU only."""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from paper_2011_10570_b200 import _native
from paper_2011_10570_b200 import wavelet as W
from wavelet_fields import FIELDS

G = golden("wavelet")
CASES = sorted(k[: -len("_meta")] for k in G.files if k.endswith("_meta") and not k.startswith("scale"))
LO, HI = (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)


@pytest.mark.parametrize("npd", range(3, 16, 2))
def test_lagrange_matrix_bits(npd):
    xs = np.linspace(0.0, 1.0, npd)
    want = G[f"W{npd}"]
    assert np.array_equal(W._lagrange_matrix(xs[::2], xs), want)
    assert np.array_equal(O.lagrange_matrix(xs[::2], xs), want)


@pytest.mark.parametrize("case", CASES)
def test_oracle_coefficients_pinned(case):
    dim, L, npd = (int(x) for x in G[f"{case}_meta"][:3])
    got = O.wavelet_coeffs(G[f"{case}_values"], npd, dim)
    assert np.array_equal(got, G[f"{case}_coeff"])


@pytest.mark.parametrize("case", CASES)
def test_oracle_samples_and_flags_pinned(case):
    dim, L, npd, mnl, mxl, _ = (int(x) for x in G[f"{case}_meta"])
    f = FIELDS[str(G[f"{case}_field"])]
    an, lv = G[f"{case}_anchors"], G[f"{case}_levels"]
    for i in range(0, len(an), 7):
        v = O.wavelet_samples(f, tuple(int(a) for a in an[i]), int(lv[i]), L, npd, LO[:dim], HI[:dim])
        assert np.array_equal(v.reshape(-1), G[f"{case}_values"][i])
    codes = O.wavelet_flag_codes(G[f"{case}_coeff"], lv, float(G[f"{case}_tol"][0]), 0.1, mnl, mxl)
    assert np.array_equal(codes, G[f"{case}_codes"])


@pytest.mark.parametrize("case", CASES)
def test_host_batched_sampling_bits(case):
    """The product's vectorised sampling (all octants in one f call) gives
    the reference's per-octant samples bit for bit."""
    dim, L, npd = (int(x) for x in G[f"{case}_meta"][:3])
    f = FIELDS[str(G[f"{case}_field"])]
    an, lv = G[f"{case}_anchors"].astype(np.int64), G[f"{case}_levels"]
    axes = W._sample_axes(an, lv, L, LO[:dim], HI[:dim], npd)
    assert np.array_equal(W._sample_values(f, axes, npd), G[f"{case}_values"])


def test_validation():
    # wavelet.py:82-83 and :33-39, the reference's test_wavelet.py:52-66
    key = W.OctKey((0, 0), 0, 2)
    for npd in (4, 1, 2):
        with pytest.raises(ValueError):
            W.wavelet_coefficient(lambda x, y: x, key, npd)
    with pytest.raises(ValueError):
        W.RefinePolicy(tolerance=-1.0)
    with pytest.raises(ValueError):
        W.RefinePolicy(tolerance=1e-3, coarsen_factor=1.5)
    with pytest.raises(ValueError):
        W.RefinePolicy(tolerance=1e-3, min_level=4, max_level=2)


def test_predicate_level_clamps_without_device():
    """Levels outside [min_level, max_level) are decided without sampling f
    (wavelet.py:137-140), so they need no GPU."""
    pol = W.RefinePolicy(tolerance=1e-3, min_level=2, max_level=4)

    def boom(*a):
        raise AssertionError("f must not be evaluated")

    pred = W.refinement_predicate(boom, pol)
    an = np.zeros((3, 2), dtype=np.int64)
    assert pred.batch(an, 1, 6).all()
    assert not pred.batch(an, 4, 6).any()


def test_abi_exports_wavelet():
    assert "amr_wavelet_coeff" in _native.SIGNATURES
    assert hasattr(_native.lib(), "amr_wavelet_coeff")


@pytest.mark.parametrize("dim,npd,L", [(2, 7, 7), (3, 5, 6), (3, 9, 5)])
def test_device_sampling_formula_on_cpu_tensors(dim, npd, L):
    """The device_eval sampling (torch ops, tensor/tensor divisions) gives the
    numpy coordinates bit for bit; checked here with CPU tensors."""
    import torch

    rng = np.random.default_rng(dim * 7 + npd)
    n = 200
    lv = rng.integers(0, L + 1, n).astype(np.int32)
    an = np.stack([(rng.integers(0, 1 << L, n) >> (L - lv)) << (L - lv) for _ in range(dim)], axis=1).astype(np.int64)
    lo, hi = (-1.0, -0.5, -2.0)[:dim], (1.0, 3.0, 0.25)[:dim]
    axes = W._sample_axes(an, lv, L, lo, hi, npd)
    for d in range(dim):
        host = W._sample_values(lambda *g: g[d], axes, npd)
        dev = W._device_samples(torch, lambda *g: g[d], torch.from_numpy(an), torch.from_numpy(lv), L, lo, hi, npd)
        assert np.array_equal(dev.numpy(), host)


def test_oracle_at_scale_pinned():
    """4 278 leaves of a 3D random tree: the oracle's per-octant samples and
    coefficients against the reference's (golden 'scale' case)."""
    dim, L, npd, mnl, mxl = (int(x) for x in G["scale_meta"])
    an, lv = G["scale_anchors"], G["scale_levels"]
    vals = np.stack([O.wavelet_samples(FIELDS["trig3"], tuple(int(x) for x in a), int(l), L, npd, LO, HI).reshape(-1)
                     for a, l in zip(an, lv)])
    c = O.wavelet_coeffs(vals, npd, dim)
    assert np.array_equal(c, G["scale_coeff"])
    assert np.array_equal(O.wavelet_flag_codes(c, lv, 6e-6, 0.1, mnl, mxl), G["scale_codes"])
