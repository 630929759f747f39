"""Synthetic workloads standing in for BASELINE.json's five configs.

BASELINE.json names refinement regions in words ("refined to level 6 inside
radius 0.2", "nested spheres of radius 0.4/0.2/0.1", ...).  The reference has
no such presets; its own tests refine with the box-distance predicate
``ball_refine`` (``/root/reference/pkg/tests/test_stepper.py:17-26``).  The
predicates below follow that convention: an octant refines while its level is
below the target of the closest distance band its box touches.  They are duck
typed on ``key.level / key.anchor / key.side / key.max_depth`` so the same
objects drive the reference's ``construct`` (golden generation) and ours.

All numbers here are frozen: goldens, tests and ``bench.py`` depend on them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def box_dist2_batch(anchors: np.ndarray, level: int, max_depth: int, center, lo=-1.0, hi=1.0):
    """Vectorised box_dist2 over an (n, dim) anchor array: the same float64
    operations in the same order, so the decisions are identical."""
    scale = (hi - lo) / (1 << max_depth)
    side = 1 << (max_depth - level)
    d2 = np.zeros(len(anchors))
    for d, c in enumerate(center[: anchors.shape[1]]):
        a = anchors[:, d].astype(np.float64)
        m = lo + a * scale - c
        M = lo + (anchors[:, d] + side).astype(np.float64) * scale - c
        inside = (m <= 0.0) & (0.0 <= M)
        d2 = d2 + np.where(inside, 0.0, np.minimum(m * m, M * M))
    return d2


def box_dist2_device(anchors, level: int, max_depth: int, center, lo=-1.0, hi=1.0):
    """box_dist2_batch on a CUDA int32 (n, dim) anchor tensor: the same float64
    operations in the same order (torch elementwise ops are correctly rounded
    like numpy's), so the decisions are identical."""
    import torch

    scale = (hi - lo) / (1 << max_depth)
    side = 1 << (max_depth - level)
    d2 = torch.zeros(anchors.shape[0], dtype=torch.float64, device=anchors.device)
    zero = torch.zeros((), dtype=torch.float64, device=anchors.device)
    for d, c in enumerate(center[: anchors.shape[1]]):
        a = anchors[:, d].to(torch.float64)
        m = lo + a * scale - c
        M = lo + (anchors[:, d].to(torch.int64) + side).to(torch.float64) * scale - c
        inside = (m <= 0.0) & (0.0 <= M)
        d2 = d2 + torch.where(inside, zero, torch.minimum(m * m, M * M))
    return d2


def box_dist2(key, center, lo: float = -1.0, hi: float = 1.0) -> float:
    """Squared distance from ``center`` to the octant's closed box (same
    arithmetic as the reference test predicate, test_stepper.py:22-25)."""
    scale = (hi - lo) / (1 << key.max_depth)
    d2 = 0.0
    for a, c in zip(key.anchor, center):
        m = lo + a * scale - c
        M = lo + (a + key.side) * scale - c
        d2 += 0.0 if m <= 0.0 <= M else min(m * m, M * M)
    return d2


@dataclass(frozen=True)
class BandRefine:
    """Refine to ``level`` where the box is within ``radius`` of any centre.

    ``bands`` is a list of ``(radius, level)``; the deepest matching band wins;
    every octant refines at least to ``base``.
    """

    base: int
    bands: tuple[tuple[float, int], ...]
    centers: tuple[tuple[float, ...], ...]
    lo: float = -1.0
    hi: float = 1.0

    def target(self, key) -> int:
        tgt = self.base
        d2 = min(box_dist2(key, c, self.lo, self.hi) for c in self.centers)
        for rad, lvl in self.bands:
            if d2 < rad * rad and lvl > tgt:
                tgt = lvl
        return tgt

    def __call__(self, key) -> bool:
        if key.level < self.base:
            return True
        return key.level < self.target(key)

    def batch(self, anchors: np.ndarray, level: int, max_depth: int) -> np.ndarray:
        if level < self.base:
            return np.ones(len(anchors), dtype=bool)
        d2 = None
        for c in self.centers:
            e = box_dist2_batch(anchors, level, max_depth, c, self.lo, self.hi)
            d2 = e if d2 is None else np.minimum(d2, e)
        tgt = np.full(len(anchors), self.base)
        for rad, lvl in self.bands:
            tgt = np.where((d2 < rad * rad) & (lvl > tgt), lvl, tgt)
        return level < tgt

    def batch_device(self, anchors, level: int, max_depth: int):
        import torch

        if level < self.base:
            return torch.ones(anchors.shape[0], dtype=torch.bool, device=anchors.device)
        d2 = None
        for c in self.centers:
            e = box_dist2_device(anchors, level, max_depth, c, self.lo, self.hi)
            d2 = e if d2 is None else torch.minimum(d2, e)
        tgt = torch.full((anchors.shape[0],), self.base, dtype=torch.int64, device=anchors.device)
        for rad, lvl in self.bands:
            tgt = torch.where((d2 < rad * rad) & (lvl > tgt), torch.full_like(tgt, lvl), tgt)
        return level < tgt


@dataclass(frozen=True)
class SphereSeeds:
    """Per-sphere refinement: each sphere (centre, radius, level) refines
    boxes it touches to its level (BASELINE cfg4/cfg5 'seed-placed spheres')."""

    base: int
    spheres: tuple[tuple[tuple[float, ...], float, int], ...]
    lo: float = -1.0
    hi: float = 1.0

    def __call__(self, key) -> bool:
        if key.level < self.base:
            return True
        for c, r, lvl in self.spheres:
            if key.level < lvl and box_dist2(key, c, self.lo, self.hi) < r * r:
                return True
        return False

    def batch(self, anchors: np.ndarray, level: int, max_depth: int) -> np.ndarray:
        if level < self.base:
            return np.ones(len(anchors), dtype=bool)
        out = np.zeros(len(anchors), dtype=bool)
        for c, r, lvl in self.spheres:
            if level < lvl:
                out |= box_dist2_batch(anchors, level, max_depth, c, self.lo, self.hi) < r * r
        return out

    def batch_device(self, anchors, level: int, max_depth: int):
        import torch

        if level < self.base:
            return torch.ones(anchors.shape[0], dtype=torch.bool, device=anchors.device)
        out = torch.zeros(anchors.shape[0], dtype=torch.bool, device=anchors.device)
        for c, r, lvl in self.spheres:
            if level < lvl:
                out |= box_dist2_device(anchors, level, max_depth, c, self.lo, self.hi) < r * r
        return out


@dataclass(frozen=True)
class GradedSpheres:
    """Per-sphere graded refinement: sphere (c, r) with target level
    lmax - round(log2(r / 0.005)) (small spheres refine deepest) refines boxes
    within rscale*r*2^k of its centre to target - k (BASELINE cfg4)."""

    base: int
    lmax: int
    spheres: tuple
    rscale: float = 1.0
    lo: float = -1.0
    hi: float = 1.0

    def _targets(self):
        return [(c, r * self.rscale, min(self.lmax, self.lmax - int(round(math.log2(r / 0.005)))))
                for c, r, _ in self.spheres]

    def __call__(self, key) -> bool:
        if key.level < self.base:
            return True
        for c, r, lt in self._targets():
            d2 = box_dist2(key, c, self.lo, self.hi)
            for k in range(8):
                if key.level < lt - k and d2 < (r * 2 ** k) ** 2:
                    return True
        return False

    def batch(self, anchors: np.ndarray, level: int, max_depth: int) -> np.ndarray:
        if level < self.base:
            return np.ones(len(anchors), dtype=bool)
        out = np.zeros(len(anchors), dtype=bool)
        for c, r, lt in self._targets():
            d2 = box_dist2_batch(anchors, level, max_depth, c, self.lo, self.hi)
            for k in range(8):
                if level < lt - k:
                    out |= d2 < (r * 2 ** k) ** 2
        return out

    def batch_device(self, anchors, level: int, max_depth: int):
        import torch

        if level < self.base:
            return torch.ones(anchors.shape[0], dtype=torch.bool, device=anchors.device)
        out = torch.zeros(anchors.shape[0], dtype=torch.bool, device=anchors.device)
        for c, r, lt in self._targets():
            if level >= lt:
                continue
            d2 = box_dist2_device(anchors, level, max_depth, c, self.lo, self.hi)
            for k in range(8):
                if level < lt - k:
                    out |= d2 < (r * 2 ** k) ** 2
        return out


@dataclass(frozen=True)
class WaveConfig:
    name: str
    dim: int
    max_depth: int
    refine: object
    ppo: int = 9
    pad: int = 2
    nonlinear: object = False  # False | "cubic" | "sin"
    pulse_centers: tuple = ((0.0, 0.0, 0.0),)
    pulse_width: float = 0.1
    pulse_amps: tuple = (1.0,)
    t_end: float = 1.0
    cfl: float = 0.25
    tableau: str = "rk4"
    note: str = ""

    @property
    def domain_lo(self):
        return (-1.0,) * self.dim

    @property
    def domain_hi(self):
        return (1.0,) * self.dim

    def chi0(self):
        """Initial chi: sum of Gaussians amp*exp(-r^2/width^2) (phi0 = 0).

        A single pulse is evaluated with the reference's own expression
        (wave.py:212-214) so that initial data is bit-identical."""
        cs = [c[: self.dim] for c in self.pulse_centers]
        amps = self.pulse_amps
        w = self.pulse_width

        def chi0(*xs):
            tot = None
            for c, a in zip(cs, amps):
                r2 = sum((x - cc) ** 2 for x, cc in zip(xs, c))
                q = -r2 / w**2
                term = a * (q.exp() if hasattr(q, "exp") else np.exp(q))  # torch tensors: device evaluation
                tot = term if tot is None else tot + term
            return tot

        return chi0


def _cfg4_spheres(seed: int = 4, n: int = 16, lmax: int = 13, base: int = 2):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        c = tuple(float(x) for x in rng.uniform(-0.8, 0.8, size=3))
        r = float(math.exp(rng.uniform(math.log(0.005), math.log(0.1))))
        out.append((c, r, lmax))
    return tuple(out)


def _cfg5_sources(seed: int = 5, n: int = 64):
    rng = np.random.default_rng(seed)
    cs = tuple(tuple(float(x) for x in rng.uniform(-0.7, 0.7, size=3)) for _ in range(n))
    amps = tuple(float(a) for a in rng.uniform(0.5, 1.0, size=n))
    return cs, amps


_CFG5_C, _CFG5_A = _cfg5_sources()

CONFIGS: dict[str, WaveConfig] = {
    # BASELINE configs[0]: 2D, base level 3, level 6 within 0.2 of the origin
    "cfg1": WaveConfig(
        "cfg1", 2, 6, BandRefine(3, ((0.2, 6),), ((0.0, 0.0),)),
        pulse_centers=((0.0, 0.0),), pulse_width=0.1, t_end=0.5,
    ),
    # configs[1]: 3D, levels 3-7 in nested spheres 0.4/0.2/0.1
    "cfg2": WaveConfig(
        "cfg2", 3, 7, BandRefine(3, ((0.4, 5), (0.2, 6), (0.1, 7)), ((0.0, 0.0, 0.0),)),
        pulse_width=0.05, t_end=1.0,
    ),
    # configs[2]: 3D cubic, levels 4-9 around two Gaussians at (+-0.3, 0, 0)
    "cfg3": WaveConfig(
        "cfg3", 3, 9,
        BandRefine(4, ((0.6, 5), (0.35, 6), (0.2, 7), (0.1, 8), (0.05, 9)),
                   ((-0.3, 0.0, 0.0), (0.3, 0.0, 0.0))),
        nonlinear="cubic", pulse_centers=((-0.3, 0.0, 0.0), (0.3, 0.0, 0.0)),
        pulse_amps=(1.0, 1.0), pulse_width=0.05, t_end=1.0,
    ),
    # configs[3]: deep adaptivity, levels 2-13 around 16 seeded spheres; graded
    # refinement calibrated (rscale 0.25) to BASELINE's ~50 M points: 108 298
    # leaves after balance
    "cfg4": WaveConfig(
        "cfg4", 3, 13, GradedSpheres(2, 13, _cfg4_spheres(), rscale=0.25),
        pulse_centers=tuple(s[0] for s in _cfg4_spheres()), pulse_amps=(0.5,) * 16,
        pulse_width=0.05, t_end=1.0,
        note="random-phase superposition defined as 16 Gaussians at the sphere centres",
    ),
    # configs[4]: 64 Gaussian sources, levels 4-12, cubic
    "cfg5": WaveConfig(
        "cfg5", 3, 12,
        # bands calibrated (x0.5) to BASELINE's ~500 M points: 1 216 972 leaves after balance
        BandRefine(4, ((0.15, 6), (0.05, 8), (0.02, 10), (0.005, 12)), _CFG5_C),
        nonlinear="cubic", pulse_centers=_CFG5_C, pulse_amps=_CFG5_A, pulse_width=0.02,
        t_end=0.390625,
    ),
    # uniform level-5 3D mesh (32 768 leaves, no level interfaces): the tile
    # kernel's best case, for performance diagnosis only
    "uni5": WaveConfig(
        "uni5", 3, 5, BandRefine(5, (), ((0.0, 0.0, 0.0),)), pulse_width=0.2, t_end=1.0,
    ),
    # small 3D mesh for goldens and fast parity (levels 2-4)
    "mini3d": WaveConfig(
        "mini3d", 3, 4, BandRefine(2, ((0.6, 3), (0.25, 4)), ((0.1, 0.0, 0.0),)),
        pulse_centers=((0.1, 0.0, 0.0),), pulse_width=0.25, t_end=0.25,
    ),
}


def get_config(name: str) -> WaveConfig:
    try:
        return CONFIGS[name]
    except KeyError:
        raise ValueError(f"unknown config {name!r}; choose from {sorted(CONFIGS)}") from None
