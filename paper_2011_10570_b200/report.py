"""CSV reporting in the reference's schemas.

The reference package ships no CLI; its specification fixes the data shapes a
driver emits.  These helpers produce exactly those rows from an ``Engine`` /
``Mesh``:

===============================  ==========================================
``step,time,l2,linf``            error time series (paper Fig. 9)
``ranks,blk_sync,time_interp,``  phase profile (Figs. 10/12); device
``rhs,comm``                     milliseconds from ``Engine(profile=True)``
``level,alpha,steps``            work per level (block-interior points, steps)
``rank,octants,weight``          partition report (Fig. 8)
``L,W_lts,W_gts,S,S_bound``      speed-up model beside a measured S (Table 2)
===============================  ==========================================

``blk_sync`` (the reference's unzip/zip bucket, stepper.py:72-84) has no
separate kernel here: unzip, RHS and zip are one fused launch, booked under
``rhs``; the column is kept, with 0, so files keep the reference's header.
"""
from __future__ import annotations

import csv
import io
from typing import Iterable, Sequence

import numpy as np

from .perfmodel import estimate, histogram_from_mesh
from .wave import norms

TIME_SERIES = ("step", "time", "l2", "linf")
PHASES = ("ranks", "blk_sync", "time_interp", "rhs", "comm")
WORK = ("level", "alpha", "steps")
PARTITION = ("rank", "octants", "weight")
ESTIMATE = ("L", "W_lts", "W_gts", "S", "S_bound")


def to_csv(header: Sequence[str], rows: Iterable[Sequence]) -> str:
    """CSV text; floats are written with repr precision so files parse back losslessly."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(header)
    for r in rows:
        w.writerow([repr(float(v)) if isinstance(v, (float, np.floating)) else v for v in r])
    return buf.getvalue()


def parse_csv(text: str) -> tuple[list[str], list[list[str]]]:
    rows = list(csv.reader(io.StringIO(text)))
    return rows[0], rows[1:]


def time_series_row(engine, reference_zip: np.ndarray, var: int = 0) -> tuple:
    """One ``step,time,l2,linf`` row: the engine's field against a reference field."""
    l2, linf = norms(engine.current_zip()[var], np.asarray(reference_zip)[var])
    return (engine.i_fine, engine.time, l2, linf)


def phase_row(engine) -> tuple:
    """``ranks,blk_sync,time_interp,rhs,comm`` in device milliseconds (engine built with profile=True)."""
    ms = engine.phase_ms()
    return (engine.mesh.pmap.ranks, 0.0, ms.get("time_interp", 0.0), ms.get("rhs", 0.0), ms.get("comm", 0.0))


def work_rows(engine) -> list[tuple]:
    """``level,alpha,steps``: block-interior points per level and the steps those blocks took since reset_work."""
    alpha: dict[int, int] = {}
    for b in engine.mesh.blocks:
        alpha[b.leaf_level] = alpha.get(b.leaf_level, 0) + b.interior_points
    steps = engine.counters.steps_by_level
    return [(lvl, alpha[lvl], int(steps.get(lvl, 0))) for lvl in sorted(alpha)]


def partition_rows(mesh) -> list[tuple]:
    pm = mesh.pmap
    return [(r, b - a, float(pm.rank_weights[r])) for r, (a, b) in enumerate(pm.rank_ranges)]


def estimate_row(mesh) -> tuple:
    h = histogram_from_mesh(mesh.blocks)
    e = estimate(h)
    return (h.L, e.w_lts, e.w_gts, e.speedup, e.bound)
