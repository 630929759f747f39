"""Wave system, radiative boundaries, initial data — drop-in for ``amrlts.wave``.

    d(chi)/dt = phi
    d(phi)/dt = Laplacian(chi) - source(chi)

with source ``c*sin(2 chi)/r^2`` (the reference's nonlinear term,
wave.py:162-163) or ``chi^3`` (BASELINE.json configs 3 and 5; an extension,
see DESIGN.md).  ``wave_rhs`` evaluates the operator on one padded block with
the sm_100a kernel (``amr_block_rhs``) — the same device code the fused
stage kernel uses — so there is one RHS implementation and it is on the GPU.

The stencil weights are produced by Fornberg's recursion with the same
floating-point operation order as the reference, so they match its arrays
bit for bit (four entries differ from correctly rounded fractions by an ulp;
the centred 2nd-derivative stencil is bitwise asymmetric).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native


def fornberg_weights(m: int, offsets) -> np.ndarray:
    """Weights of the m-th derivative at 0 on integer ``offsets`` (Fornberg 1988).

    Every product/quotient is formed in the order the reference evaluates it
    (wave.py:22-44) so the resulting doubles are identical."""
    xs = [float(v) for v in offsets]
    npts = len(xs)
    tab = np.zeros((npts, m + 1))
    tab[0, 0] = 1.0
    prod_prev = 1.0
    x_now = xs[0]
    for i in range(1, npts):
        top = min(i, m)
        prod = 1.0
        x_prev, x_now = x_now, xs[i]
        for j in range(i):
            gap = xs[i] - xs[j]
            prod *= gap
            if j == i - 1:
                for k in range(top, 0, -1):
                    tab[i, k] = prod_prev * (k * tab[i - 1, k - 1] - x_prev * tab[i - 1, k]) / prod
                tab[i, 0] = -prod_prev * x_prev * tab[i - 1, 0] / prod
            for k in range(top, 0, -1):
                tab[j, k] = (x_now * tab[j, k] - k * tab[j, k - 1]) / gap
            tab[j, 0] = x_now * tab[j, 0] / gap
        prod_prev = prod
    return tab[:, m]


_D2_CENTER = fornberg_weights(2, range(-2, 3))
_D2_EDGE0 = fornberg_weights(2, range(0, 6))
_D2_EDGE1 = fornberg_weights(2, range(-1, 5))
_D1_CENTER = fornberg_weights(1, range(-2, 3))
_D1_EDGE0 = fornberg_weights(1, range(0, 5))
_D1_EDGE1 = fornberg_weights(1, range(-1, 4))

NONLINEAR_CODES = {False: 0, None: 0, "none": 0, True: 1, "sin": 1, "cubic": 2}


def nonlinear_code(nonlinear) -> int:
    try:
        return NONLINEAR_CODES[nonlinear]
    except (KeyError, TypeError):
        raise ValueError(f"nonlinear must be False/True/'sin'/'cubic', got {nonlinear!r}") from None


def fill_weights(p) -> None:
    """Copy the reference stencil arrays into an AmrStageParams."""
    for name, arr in (("d2c", _D2_CENTER), ("d2e0", _D2_EDGE0), ("d2e1", _D2_EDGE1),
                      ("d1c", _D1_CENTER), ("d1e0", _D1_EDGE0), ("d1e1", _D1_EDGE1)):
        dst = getattr(p, name)
        for i, v in enumerate(arr):
            dst[i] = float(v)


def _row_stencils(order: int, n: int, lo: bool, hi: bool):
    """Per interior row along one axis: (offsets, weights) of the stencil the
    reference applies (centred, then the biased rows near physical faces)."""
    if order == 2:
        centred, e0, e1, r0, r1 = _D2_CENTER, _D2_EDGE0, _D2_EDGE1, range(0, 6), range(-1, 5)
    else:
        centred, e0, e1, r0, r1 = _D1_CENTER, _D1_EDGE0, _D1_EDGE1, range(0, 5), range(-1, 4)
    rows = [(list(range(-2, 3)), list(centred))] * n
    sign = (-1) ** order
    if lo:
        rows[0], rows[1] = (list(r0), list(e0)), (list(r1), list(e1))
    if hi:
        rows[n - 1] = ([-o for o in r0], [w * sign for w in e0])
        rows[n - 2] = ([-o for o in r1], [w * sign for w in e1])
    return rows


def derivative_axis(arr: np.ndarray, axis: int, h: float, pad: int, order: int,
                    lo_boundary: bool, hi_boundary: bool) -> np.ndarray:
    """Host utility (not on the engine path): the 1D derivative of
    wave.py:67-109 over the interior of a padded numpy array; each row sums
    its stencil terms left to right and divides by h**order."""
    moved = np.moveaxis(np.asarray(arr, dtype=float), axis, 0)
    inner = (slice(None),) + (slice(pad, -pad),) * (moved.ndim - 1)
    core = moved[inner]
    n = moved.shape[0] - 2 * pad
    out = np.empty((n,) + core.shape[1:])
    for i, (offs, wts) in enumerate(_row_stencils(order, n, lo_boundary, hi_boundary)):
        acc = None
        for o, w in zip(offs, wts):
            term = w * core[pad + i + o]
            acc = term if acc is None else acc + term
        out[i] = acc / h ** order
    return np.moveaxis(out, 0, axis)


@dataclass
class BlockGeometry:
    h: float
    axes_interior: list[np.ndarray]
    r2_reg: np.ndarray
    r: np.ndarray
    faces: list[tuple[int, int]]
    pad: int
    r_eps: float = 0.0


def block_geometry(mesh, block, r_eps: float) -> BlockGeometry:
    """Per-block constants of the operator (wave.py:124-144)."""
    axes = mesh.block_axes(block)
    g, n, dim = block.pad, block.interior_n, mesh.dim
    inner = []
    for d in range(dim):
        shape = [1] * dim
        shape[d] = n
        inner.append(axes[d][g: g + n].reshape(shape))
    r2 = sum(a ** 2 for a in inner)
    return BlockGeometry(h=mesh.block_spacing(block), axes_interior=inner, r2_reg=np.maximum(r2, r_eps ** 2),
                         r=np.maximum(np.sqrt(r2), r_eps), faces=mesh.block_domain_faces(block), pad=g,
                         r_eps=r_eps)


def wave_rhs(y: np.ndarray, geom: BlockGeometry, nonlinear, k_chi: float, k_phi: float,
             f0_chi: float = 0.0, f0_phi: float = 0.0) -> np.ndarray:
    """(dchi, dphi) on the block interior from padded ``y`` — on the GPU."""
    import torch

    y = np.ascontiguousarray(y, dtype=np.float64)
    dim = y.ndim - 1
    g = geom.pad
    n = y.shape[1] - 2 * g
    if g != 2:
        raise ValueError("wave_rhs kernel implements pad=2")
    dev = torch.device("cuda")
    yd = torch.from_numpy(y).to(dev)
    coords = np.stack([np.asarray(geom.axes_interior[d]).reshape(-1) for d in range(dim)]).astype(np.float64)
    cd = torch.from_numpy(np.ascontiguousarray(coords)).to(dev)
    out = torch.empty((2,) + (n,) * dim, dtype=torch.float64, device=dev)
    faces = 0
    for axis, side in geom.faces:
        faces |= 1 << (2 * axis + side)
    prm = _native.AmrStageParams()
    fill_weights(prm)
    r_eps = geom.r_eps if geom.r_eps else float(np.sqrt(np.min(geom.r2_reg)))
    prm.r_eps2 = r_eps ** 2
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(_native.lib().amr_block_rhs(dim, n, g, yd.data_ptr(), out.data_ptr(), geom.h, geom.h ** 2,
                                              cd.data_ptr(), r_eps, faces, nonlinear_code(nonlinear),
                                              k_chi, k_phi, f0_chi, f0_phi, _native.C.byref(prm), stream),
                  "amr_block_rhs")
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# initial data and reference solutions (host)
# ---------------------------------------------------------------------------


def gaussian_pulse(center, width, amplitude):
    def chi0(*xs):
        r2 = sum((x - c) ** 2 for x, c in zip(xs, center))
        return amplitude * np.exp(-r2 / width ** 2)

    return chi0


def plane_pulse(center_x, width, amplitude):
    def chi0(*xs):
        return amplitude * np.exp(-((xs[0] - center_x) ** 2) / width ** 2)

    return chi0


def analytic_linear(profile, t: float, x):
    return 0.5 * (profile(x - t) + profile(x + t))


def norms(a: np.ndarray, b: np.ndarray) -> tuple[float, float]:
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        raise ValueError(f"mesh mismatch: {a.shape} vs {b.shape}")
    diff = a - b
    l2 = float(np.sqrt(np.mean(diff ** 2)))
    linf = float(np.max(np.abs(diff))) if diff.size else 0.0
    return l2, linf
