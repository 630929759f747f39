"""Global and local (multirate) RK stepping on the GPU — drop-in for ``amrlts.stepper``.

Same driver semantics as the reference engine (stepper.py:105-514): time is
counted in fine slices of ``dt_fine = cfl * dx_finest``; a block of cadence
level c steps every ``2**(l_max - c)`` slices; at a slice all eligible blocks
run the RK stage loop in lockstep, reading neighbours through the stage
transfer algebra where step sizes or times differ.

B200 design:
* state lives on the device in the reference's (nvars, n_nodes) zip layout
  (SoA): two u buffers and p stage buffers.  A leaf's live buffer is the parity of
  its step count, so ``u_pre <- u_curr`` costs nothing, and the record fields
  ``t0``/``dt_units`` are implied by the schedule;
* tiles are sorted by cadence (finest first), so the eligible set of any
  slice is a prefix of the tile list — one launch per stage per slice;
* each stage is one launch of the fused unzip + time-interpolation + RHS +
  zip kernel (``amr_stage``); the last stage also does the RK combine;
* per-slice LTS coefficients (transfer matrices, parities, dt products) are
  computed once per slice phase on the host and kept on the device.
* multi-GPU: one process per GPU, contiguous weighted-Morton leaf ranges,
  every rank holds the full zip layout (180 GB HBM makes that cheap), and the
  ghost leaves of the reference's exchange plan move over NCCL after every
  stage (``GhostExchange``), exactly where the reference calls ``_ship``.
"""
from __future__ import annotations

import os
import time
from collections import defaultdict
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .mesh import Mesh
from .partition import ExchangePlan
from .rkcorrect import ButcherTableau, get_tableau, stage_transfer_matrix
from .wave import fill_weights, nonlinear_code

C = _native.C


@dataclass
class TimeLevelSchedule:
    """Eligibility of blocks over the fine-slice phases of one coarse round (stepper.py:34-69)."""

    block_levels: list[int]
    l_max: int
    l_min: int

    @property
    def delta_l(self) -> int:
        return self.l_max - min(self.block_levels)

    @property
    def slices_per_round(self) -> int:
        return 1 << self.delta_l

    def period(self, block: int) -> int:
        return 1 << (self.l_max - self.block_levels[block])

    def eligible(self, i: int) -> list[int]:
        return [b for b in range(len(self.block_levels)) if i % self.period(b) == 0]

    def phase(self, i: int) -> int:
        if i % self.slices_per_round == 0:
            return self.delta_l
        tz = (i & -i).bit_length() - 1
        return min(tz, self.delta_l)

    def step_start(self, i: int, block: int) -> int:
        p = self.period(block)
        return (i // p) * p

    def steps_per_round(self, block: int) -> int:
        return self.slices_per_round // self.period(block)


class WorkCounters:
    """Work and phase counters (stepper.py:72-84).

    The engine advances per-cadence tallies once per slice; the per-block and
    per-level views of the reference are materialised on access."""

    def __init__(self, block_cadence=(), block_level=(), block_points=(), block_rank=(), stages=1):
        self._bc = np.asarray(block_cadence, dtype=np.int64)
        self._bl = np.asarray(block_level, dtype=np.int64)
        self._bp = np.asarray(block_points, dtype=np.int64)
        self._br = np.asarray(block_rank, dtype=np.int64)
        self._p = stages
        self._steps_total = defaultdict(int)  # cadence -> steps since construction
        self._steps_work = defaultdict(int)   # cadence -> steps since reset_work
        self.phases = defaultdict(float)

    def _tally(self, cadences) -> None:
        for c in cadences:
            self._steps_total[c] += 1
            self._steps_work[c] += 1

    def reset_work(self) -> None:
        self._steps_work = defaultdict(int)

    def _per_block(self, tally) -> np.ndarray:
        out = np.zeros(len(self._bc), dtype=np.int64)
        for c, n in tally.items():
            out[self._bc == c] = n
        return out

    @property
    def rhs_evals(self):
        steps = self._per_block(self._steps_total)
        return defaultdict(int, {int(b): int(self._p * s) for b, s in enumerate(steps) if s})

    @property
    def rhs_by_rank(self):
        steps = self._per_block(self._steps_total)
        out = defaultdict(int)
        for r, s in zip(self._br.tolist(), steps.tolist()):
            if s:
                out[r] += self._p * s
        return out

    @property
    def point_steps(self) -> int:
        return int(np.sum(self._per_block(self._steps_work) * self._bp))

    @property
    def point_steps_by_rank(self):
        steps = self._per_block(self._steps_work) * self._bp
        out = defaultdict(int)
        for r, s in zip(self._br.tolist(), steps.tolist()):
            if s:
                out[r] += s
        return out

    @property
    def steps_by_level(self):
        steps = self._per_block(self._steps_work)
        out = defaultdict(int)
        for lvl, s in zip(self._bl.tolist(), steps.tolist()):
            if s:
                out[lvl] += s
        return out


def _pow2_exact(x: float) -> bool:
    m, _ = np.frexp(x)
    return x > 0 and m == 0.5


class Engine:
    """Wave-system timestepper over a block mesh, global or local mode, on one GPU
    (or one GPU per rank under torch.distributed)."""

    NVARS = 2

    def __init__(self, mesh: Mesh, tableau: str | ButcherTableau = "rk3", cfl: float = 0.25,
                 mode: str = "lts", nonlinear=False, k_chi: float = 1.0, k_phi: float = 2.0,
                 threads: int = 1, single_stage_neighbors: bool = False, device=None, process_group=None):
        import torch

        if mode not in ("lts", "gts"):
            raise ValueError("mode must be 'lts' or 'gts'")
        self.mesh = mesh
        self.tab = get_tableau(tableau) if isinstance(tableau, str) else tableau
        self.p = self.tab.stages
        if self.p > _native.AMR_MAXP:
            raise ValueError(f"at most {_native.AMR_MAXP} stages are supported")
        self.cfl = cfl
        self.mode = mode
        self.nonlinear = nonlinear
        self._nl = nonlinear_code(nonlinear)
        self.k_chi = k_chi
        self.k_phi = k_phi
        self.threads = threads
        self.dt_fine = cfl * mesh.finest_spacing()
        levels = [b.leaf_level for b in mesh.blocks]
        self.l_max = max(levels)
        self.l_min = min(levels)
        if self.l_max >= _native.AMR_MAXL:
            raise ValueError(f"levels above {_native.AMR_MAXL - 1} are not supported")
        if single_stage_neighbors:
            if self.p != 1:
                raise ValueError("the pseudo-timestep neighbor scheme supports single-stage tableaus only")
            cadence = self._promoted_cadence(levels)
        elif mode == "gts":
            cadence = [self.l_max] * len(levels)
        else:
            cadence = list(levels)
        self.cadence = cadence
        self.schedule = TimeLevelSchedule(cadence, self.l_max, self.l_min)
        self.dt_units = [1 << (self.l_max - c) for c in cadence]
        self._full_plan = None
        self._partial_plans = None
        self.counters = WorkCounters(cadence, levels, [b.interior_points for b in mesh.blocks],
                                     [b.owner_rank for b in mesh.blocks], self.p)
        self.i_fine = 0
        self._r_eps = mesh.finest_spacing()
        self._transfer_cache: dict = {}
        self._coef_cache: dict = {}

        # -- distribution ---------------------------------------------------------
        self._dist = None
        self.rank = 0
        if process_group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()
                                         and torch.distributed.get_world_size() > 1):
            ws = torch.distributed.get_world_size(process_group)
            if ws != mesh.pmap.ranks:
                raise ValueError(f"mesh is partitioned for {mesh.pmap.ranks} ranks, process group has {ws}")
            self.rank = torch.distributed.get_rank(process_group)
            self._dist = process_group if process_group is not None else torch.distributed.group.WORLD

        # -- device state ---------------------------------------------------------------
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise RuntimeError("the engine runs on CUDA devices only (no CPU path)")
        self._lib = _native.lib()
        td = mesh.tile_data()
        n_leaves = len(mesh.tree.leaves)
        leaf_cad = np.empty(n_leaves, dtype=np.int32)
        for b in mesh.blocks:
            leaf_cad[b.leaf_range[0]: b.leaf_range[1]] = cadence[b.index]
        self._leaf_cadence = leaf_cad
        counts = np.diff(td["starts"])
        node_cad = np.repeat(leaf_cad.astype(np.uint8), counts)
        owners = mesh.pmap.owners(n_leaves)
        mine = np.nonzero(owners == self.rank)[0] if self._dist is not None else np.arange(n_leaves)
        order = np.lexsort((mine, -leaf_cad[mine]))
        tiles = mine[order].astype(np.int32)
        lts_kernel = mode == "lts" or any(c != self.l_max for c in cadence)
        self._init_programs(td, tiles, leaf_cad, node_cad, lts_kernel)
        n = mesh.n_nodes
        # the reference's (nvars, n_nodes) zip layout, SoA: chi row then phi row.
        # Rows are padded to an even stride ld > n (16-byte aligned rows; the
        # kernel bulk-prefetches 16-byte aligned supersets of a tile's owned range)
        ld = (n + 2) // 2 * 2
        self._ld = ld
        dev = self.device
        self._U_store = [torch.zeros((2, ld), dtype=torch.float64, device=dev) for _ in range(2)]
        self._K_store = torch.zeros((self.p, 2, ld), dtype=torch.float64, device=dev)
        self._U = [u[:, :n] for u in self._U_store]
        self._K = self._K_store[:, :, :n]
        # verbatim stage sources, double-buffered by stage parity
        self._Y_store = torch.zeros((2, 2, ld), dtype=torch.float64, device=dev)
        self._Y = self._Y_store[:, :, :n]
        self._node_cad_t = self._d["node_cad"].long()
        self._vt = [[j for j in range(s_) if self.tab.a[s_][j] != 0.0] for s_ in range(self.p)]
        self._prm = self._make_params()
        self._exchange = _EngineExchange(self) if self._dist is not None else None

    def _init_programs(self, td, tiles, leaf_cad, node_cad, lts):
        """The stage kernel's per-tile programs (tileprog.py) on the device."""
        import torch

        from . import tileprog

        prog = tileprog.build_programs_native(self.mesh, tiles, leaf_cad, lts)  # == tileprog.build_programs
        tcad = leaf_cad[tiles]
        self._prefix = {c: int(np.sum(tcad >= c)) for c in range(self.l_max + 1)}
        n_iface = prog["n_iface"]
        self._if_prefix = {c: int(np.sum((prog["if_cad"][:n_iface] & 0xFF) >= c)) for c in range(self.l_max + 1)}
        self._n_iface = n_iface
        dev = self.device
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        pad = lambda a: a if len(a) else np.zeros(1, a.dtype)  # noqa: E731
        self._d = dict(tiles=T(tiles.astype(np.int32)), node_cad=T(node_cad), heads=T(prog["heads"]),
                       tail=T(prog["tail"]), wtab=T(prog["wtab"]), if_gid=T(pad(prog["if_gid"])),
                       if_cad=T(pad(prog["if_cad"])))
        self._max_slots = prog["max_slots"]
        self._max_head = prog["max_head"]
        self._max_tail = prog["max_tail"]
        self._ibuf = torch.zeros((2, max(n_iface, 1)), dtype=torch.float64, device=dev)
        self._threads = int(os.environ.get("AMR_THREADS", "256"))



    # -- setup -------------------------------------------------------------------------
    def _promoted_cadence(self, levels: list[int]) -> list[int]:
        """Single-stage scheme: a block touching finer blocks steps at the finest
        touching cadence (stepper.py:175-196)."""
        boxes = []
        for b in self.mesh.blocks:
            lo = np.array(b.root.anchor)
            boxes.append((lo, lo + b.root.side))
        cadence = list(levels)
        for i in range(len(levels)):
            for j in range(len(levels)):
                if i == j or levels[j] <= levels[i]:
                    continue
                if all(boxes[i][0][d] <= boxes[j][1][d] and boxes[j][0][d] <= boxes[i][1][d]
                       for d in range(self.mesh.dim)):
                    cadence[i] = max(cadence[i], levels[j])
        return cadence

    def _make_params(self) -> _native.AmrStageParams:
        m = self.mesh
        P = _native.AmrStageParams()
        P.dim, P.ppo, P.pad = m.dim, m.ppo, m.pad
        P.lts = 1 if self.mode == "lts" or any(c != self.l_max for c in self.cadence) else 0
        P.n_stages = self.p
        P.nonlinear = self._nl
        P.n_nodes = m.n_nodes
        P.ld = self._ld
        d = self._d
        P.max_slots = self._max_slots
        P.if_gid, P.if_cad, P.ibuf = d["if_gid"].data_ptr(), d["if_cad"].data_ptr(), self._ibuf.data_ptr()
        P.n_iface_total = self._n_iface
        P.wtab, P.n_wtab = d["wtab"].data_ptr(), int(d["wtab"].numel())
        P.heads, P.max_head, P.tail = d["heads"].data_ptr(), self._max_head, d["tail"].data_ptr()
        P.threads = self._threads
        P.max_tail = self._max_tail
        P.U0, P.U1, P.K = self._U[0].data_ptr(), self._U[1].data_ptr(), self._K.data_ptr()
        P.Y = self._Y.data_ptr()
        for s in range(self.p):
            for j in range(self.p):
                a = self.tab.a[s][j]
                P.g_cstage[s][j] = self.dt_fine * a if (j < s and a != 0.0) else 0.0
            w = self.tab.w[s]
            P.g_comb[s] = (1 * self.dt_fine) * w if w != 0.0 else 0.0
        P.max_depth = m.L
        P.top_nodes = m.top_nodes
        for dd in range(m.dim):
            P.lo[dd] = m.domain.lo[dd]
            P.extent[dd] = m.domain.extent(dd)
        for lvl in range(_native.AMR_MAXL):
            if lvl > m.L:
                continue
            h = m.level_spacing(lvl)
            h2 = h ** 2
            P.h[lvl], P.h2[lvl] = h, h2
            P.h2_pow2[lvl] = 1 if _pow2_exact(h2) else 0
            P.inv_h2[lvl] = 1.0 / h2 if P.h2_pow2[lvl] else 0.0
        P.r_eps = self._r_eps
        P.r_eps2 = self._r_eps ** 2
        P.k_chi, P.k_phi, P.f0_chi, P.f0_phi = self.k_chi, self.k_phi, 0.0, 0.0
        fill_weights(P)
        return P

    # -- plans (API parity; built lazily: they need every block's gather support) --
    @property
    def full_plan(self) -> ExchangePlan:
        if self._full_plan is None:
            self._full_plan = self.mesh.exchange_plan()
        return self._full_plan

    @property
    def partial_plans(self) -> list[ExchangePlan]:
        if self._partial_plans is None:
            cad = self.cadence
            self._partial_plans = [
                self.full_plan.restrict({b for b in range(len(cad)) if cad[b] >= self.l_max - k})
                for k in range(self.schedule.delta_l + 1)
            ]
        return self._partial_plans

    # -- state I/O -----------------------------------------------------------------------
    def initialize(self, chi0, phi0=None) -> None:
        xyz = self.mesh.node_physical()
        coords = [xyz[:, d] for d in range(self.mesh.dim)]
        z = np.zeros((self.NVARS, self.mesh.n_nodes))
        z[0] = np.asarray(chi0(*coords), dtype=float)
        if phi0 is not None:
            z[1] = np.asarray(phi0(*coords), dtype=float)
        self.load_zip(z)

    def load_zip(self, z) -> None:
        """Load a (2, n_nodes) zip field (host numpy or device tensor): u_pre = u_curr = z, K = 0."""
        import torch

        if not isinstance(z, torch.Tensor):
            z = torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64))
        if tuple(z.shape) != (self.NVARS, self.mesh.n_nodes):
            raise ValueError(f"zip field must be (2, {self.mesh.n_nodes}), got {tuple(z.shape)}")
        # straight into the live buffer (one host->device copy; pinned host
        # memory makes it a DMA), then device-side into the other parity
        self._U[0].copy_(z.to(dtype=torch.float64), non_blocking=True)
        self._U[1].copy_(self._U[0])
        self._K.zero_()
        self.i_fine = 0

    @property
    def time(self) -> float:
        return self.i_fine * self.dt_fine

    def _cur_parity(self, i: int, cad: int) -> int:
        per = 1 << (self.l_max - cad)
        return ((i + per - 1) // per) & 1

    def current_zip_device(self):
        """(2, n_nodes) float64 device tensor of every leaf's u_curr."""
        import torch

        i = self.i_fine
        key = tuple(self._cur_parity(i, c) for c in range(self.l_max + 1))
        cache = self.__dict__.setdefault("_sel_cache", {})
        sel = cache.get(key)
        if sel is None:  # which u buffer is live, per node: a function of the cadence parities only
            par = torch.tensor(key, device=self.device)
            sel = cache[key] = par[self._node_cad_t].bool().unsqueeze(0)
        return torch.where(sel, self._U[1], self._U[0])

    def current_zip(self) -> np.ndarray:
        return self.current_zip_device().cpu().numpy()

    def current_zip_to(self, out, copy_stream=None):
        """Asynchronous current_zip: copy the live (2, n_nodes) field into the
        pinned host tensor ``out`` on ``copy_stream`` (ordered after the work
        already queued on the current stream) and return the CUDA event that
        marks its completion.  The engine's buffers are free for the next
        load_zip/step at once: the copy reads a snapshot, so the device->host
        transfer of one step overlaps the host->device load of the next."""
        import torch

        cur = torch.cuda.current_stream(self.device)
        # two preallocated device snapshots, alternating: no allocation (and
        # no allocator-deferred frees) per call; a snapshot is rewritten only
        # after the copy that read it two calls ago has finished
        st = self.__dict__.get("_snap")
        if st is None:
            st = self.__dict__["_snap"] = [[torch.empty_like(self._U[0]), None] for _ in range(2)]
            self.__dict__["_snap_i"] = 0
        j = self.__dict__["_snap_i"]
        self.__dict__["_snap_i"] = j ^ 1
        buf, prev = st[j]
        if prev is not None:
            cur.wait_event(prev)
        live = self.current_zip_device()
        buf.copy_(live)
        cs = copy_stream if copy_stream is not None else cur
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            out.copy_(buf, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(cs)
        st[j][1] = ev
        return ev

    def wavelet_flags(self, policy, var: int = 0):
        """Remesh criterion on the evolved solution, on the device: the
        wavelet coefficient (wavelet.py:70-105) of every leaf's own ppo^dim
        lattice of variable ``var`` and refine_flags' decision
        (wavelet.py:108-124).  Returns (coeff, codes) host arrays, codes
        1 refine / 0 keep / -1 coarsen.  The paper remeshes only when all
        blocks are synchronised (end of a coarse round)."""
        import torch

        from .wavelet import coefficients_from_values

        lat = self.mesh.leaf_lattice_device(self.current_zip_device(), var)
        lv = torch.from_numpy(self.mesh.tree.arrays()[1].astype(np.int32)).to(lat.device)
        c, f = coefficients_from_values(lat, self.mesh.ppo, self.mesh.dim, lv, policy)
        return c.cpu().numpy(), f.cpu().numpy()

    # -- correction algebra ----------------------------------------------------------------
    def _transfer(self, delta_units: int, from_units: int, to_units: int):
        if delta_units == 0 and from_units == to_units:
            return None
        key = (delta_units, from_units, to_units)
        M = self._transfer_cache.get(key)
        if M is None:
            M = stage_transfer_matrix(self.tab, delta_units * self.dt_fine, from_units * self.dt_fine,
                                      to_units * self.dt_fine)
            if delta_units == 0:
                M = np.tril(M)
            self._transfer_cache[key] = M
        return M

    def _slice_coef(self, i: int):
        """Device AmrSliceCoef for slice i.

        It depends on i only through (i mod round, round parity): the coarsest
        cadence steps once per round, so its live-buffer parity flips every round."""
        import torch

        R = self.schedule.slices_per_round
        key = (i % R, (i // R) & 1)
        t = self._coef_cache.get(key)
        if t is not None:
            return t
        cf = _native.AmrSliceCoef()
        cads = sorted(set(self.cadence))
        tab, p = self.tab, self.p
        for c in cads:
            cf.cur[c] = self._cur_parity(i, c)
        for cr in cads:
            to = 1 << (self.l_max - cr)
            if i % to:
                continue  # reader not eligible at this slice
            dt_to = to * self.dt_fine
            for s in range(p):
                for j in range(s):
                    a = tab.a[s][j]
                    cf.cstage[cr][s][j] = dt_to * a if a != 0.0 else 0.0
            dt = to * self.dt_fine
            for s, w in enumerate(tab.w):
                cf.comb[cr][s] = (dt * w) if w != 0.0 else 0.0
            for cs in cads:
                per = 1 << (self.l_max - cs)
                if i % per == 0:
                    if per == to:
                        cf.mode[cr][cs] = 0
                        continue
                    cf.mode[cr][cs] = 1
                    M = self._transfer(0, per, to)
                else:
                    delta = i - (i // per) * per
                    cf.mode[cr][cs] = 2
                    Mv = self._transfer(0, per, delta)
                    for a_ in range(p):
                        for b_ in range(p):
                            cf.Mv[cr][cs][a_][b_] = float(Mv[a_, b_])
                    dtd = delta * self.dt_fine
                    for q, w in enumerate(tab.w):
                        cf.dtw[cr][cs][q] = (dtd * w) if w != 0.0 else 0.0
                    M = self._transfer(delta, per, to)
                for a_ in range(p):
                    for b_ in range(p):
                        cf.M[cr][cs][a_][b_] = float(M[a_, b_])
        raw = np.frombuffer(bytes(cf), dtype=np.uint8).copy()
        t = torch.from_numpy(raw).to(self.device)
        self._coef_cache[key] = t
        return t

    # -- the slice ------------------------------------------------------------------------------
    def _eligible_cadences(self, i: int) -> list[int]:
        return [c for c in sorted(set(self.cadence)) if i % (1 << (self.l_max - c)) == 0]

    def advance_slice(self) -> None:
        """Advance every block eligible at the current fine slice by one of its steps."""
        import torch

        i = self.i_fine
        elig = self._eligible_cadences(i)
        n_tiles = self._prefix[min(elig)] if elig else 0
        P = self._prm
        P.n_tiles = n_tiles
        P.n_iface = self._if_prefix[min(elig)] if elig else 0

        if P.lts:
            P.coef = self._slice_coef(i).data_ptr()
        else:
            P.gts_cur = i & 1
        stream = torch.cuda.current_stream(self.device).cuda_stream
        t0 = time.perf_counter()
        for s in range(self.p):
            P.stage = s
            vt = self._vt[s + 1] if s + 1 < self.p else []  # the writer forms stage s+1's sources
            P.n_vt = len(vt)
            for t, j in enumerate(vt):
                P.vt_j[t] = j
            if n_tiles:
                if P.n_iface:
                    rc = self._lib.amr_iface(C.byref(P), stream)
                    if rc:
                        _native.check(rc, "amr_iface")
                rc = self._lib.amr_stage(C.byref(P), stream)
                if rc:
                    _native.check(rc, "amr_stage")
            if self._exchange is not None:
                self._exchange.after_stage(i, s, elig)
        if self._exchange is not None:
            self._exchange.after_step(i, elig)
        self.counters.phases["rhs"] += time.perf_counter() - t0
        self.counters._tally(elig)
        self.i_fine += 1

    # -- public stepping --------------------------------------------------------------------------
    def gts_step(self, dt: float | None = None) -> None:
        if self.mode != "gts":
            raise RuntimeError("engine not in global-stepping mode")
        if dt is not None and dt > self.dt_fine * (1.0 + 1e-12):
            raise ValueError(f"step {dt} violates the CFL bound {self.dt_fine} (= cfl * dx_finest)")
        self.advance_slice()

    def lts_coarse_step(self) -> None:
        if self.i_fine % self.schedule.slices_per_round != 0:
            raise RuntimeError("blocks are not synchronized at a coarse time")
        R = self.schedule.slices_per_round
        if self.use_graphs and self._dist is None:
            self._replay_round(R)
            return
        for _ in range(R):
            self.advance_slice()

    # -- CUDA graphs ----------------------------------------------------------------------
    use_graphs = True

    def _replay_round(self, R: int) -> None:
        """One coarse round as a captured CUDA graph.  The launch sequence of a
        round depends only on the round parity (coefficient blocks, buffer
        parities), so two graphs cover every round.  The first round runs
        eagerly (kernel attributes, coefficient blocks); both graphs are then
        recorded (capture does not execute) and every later round replays."""
        import torch

        if not hasattr(self, "_graphs"):
            self._graphs = {}
        if not self._graphs:
            for _ in range(R):
                self.advance_slice()
            i_next = self.i_fine
            for i in range(i_next, i_next + 2 * R):  # coefficient blocks of both parities
                if self._prm.lts:
                    self._slice_coef(i)
            torch.cuda.synchronize(self.device)
            for start in (i_next, i_next + R):
                graph = torch.cuda.CUDAGraph()
                self.i_fine = start
                with torch.cuda.graph(graph):
                    for _ in range(R):
                        self.advance_slice()
                self._untally_round(start, R)
                self._graphs[(start // R) & 1] = graph
            self.i_fine = i_next
            return
        i0 = self.i_fine
        self._graphs[(i0 // R) & 1].replay()
        self._tally_round(i0, R)
        self.i_fine = i0 + R

    def _tally_round(self, i0: int, R: int) -> None:
        for i in range(i0, i0 + R):
            self.counters._tally(self._eligible_cadences(i))

    def _untally_round(self, i0: int, R: int) -> None:
        for i in range(i0, i0 + R):
            for c in self._eligible_cadences(i):
                self.counters._steps_total[c] -= 1
                self.counters._steps_work[c] -= 1

    def run_to(self, i_fine_target: int) -> None:
        while self.i_fine < i_fine_target:
            self.advance_slice()

    def launches_per_slice(self, i: int) -> int:
        """Kernel launches advance_slice(i) issues (stage + LTS interface passes)."""
        el = self._eligible_cadences(i)
        if not el:
            return 0
        return self.p * (2 if self._if_prefix[min(el)] else 1)

    def close(self):
        self._exchange = None


def lts_single_stage_engine(mesh: Mesh, **kw) -> Engine:
    kw.setdefault("tableau", "euler")
    tab = kw["tableau"]
    stages = get_tableau(tab).stages if isinstance(tab, str) else tab.stages
    if stages != 1:
        raise ValueError("the pseudo-timestep neighbor scheme supports single-stage tableaus only")
    return Engine(mesh, mode="lts", single_stage_neighbors=True, **kw)


def compare_round(lts: Engine, gts: Engine) -> float:
    """One LTS coarse round vs the matching GTS span; max |chi_lts - chi_gts|."""
    n = lts.schedule.slices_per_round
    lts.lts_coarse_step()
    for _ in range(n):
        gts.gts_step()
    a = lts.current_zip()
    b = gts.current_zip()
    return float(np.max(np.abs(a[0] - b[0])))


class GhostExchange:
    """Ghost-leaf transport between ranks over torch.distributed (NCCL on GPUs,
    gloo in the CPU tests).

    The reference ships whole leaf records after every stage and step
    (stepper.py:318-361, partition.py:182-207).  Here only the record fields
    that changed move: K_s of the leaves that just ran stage s, and their new
    u after the step; t0/dt_units follow from the schedule and u_pre is the
    other parity buffer the receiver already holds.  Which leaves go to which
    rank is the reference's exchange plan (block gather footprints); since
    every rank keeps the global zip layout, a shipment is a set of contiguous
    gid ranges gathered into one buffer per peer."""

    def __init__(self, plan: ExchangePlan, leaf_cadence: np.ndarray, leaf_starts: np.ndarray, rank: int,
                 group=None, device=None):
        self.group = group
        self.rank = rank
        self.cad = np.asarray(leaf_cadence)
        self.starts = np.asarray(leaf_starts)
        self.device = device
        self.send, self.recv = {}, {}
        for (s, r), items in plan.entries.items():
            leaves = np.array([e.leaf for e in items], dtype=np.int64)
            if s == rank:
                self.send[r] = leaves
            if r == rank:
                self.recv[s] = leaves
        self.peers = sorted(set(self.send) | set(self.recv))
        self._idx = {}

    @classmethod
    def for_engine(cls, eng: "Engine") -> "GhostExchange":
        return cls(eng.full_plan, eng._leaf_cadence, eng.mesh.leaf_starts, eng.rank, eng._dist, eng.device)

    def _index(self, kind, peer, sel_key, select):
        import torch

        key = (kind, peer, sel_key)
        if key not in self._idx:
            leaves = (self.send if kind == "s" else self.recv).get(peer)
            idx = None
            if leaves is not None:
                sel = leaves[select(self.cad[leaves])]
                if len(sel):
                    idx = torch.from_numpy(np.concatenate(
                        [np.arange(self.starts[l], self.starts[l + 1]) for l in sel])).to(self.device)
            self._idx[key] = idx
        return self._idx[key]

    def swap(self, tensor, sel_key, select) -> None:
        """Ship the zip nodes (last axis) of the selected leaves owned here to
        every peer that reads them."""
        import torch
        import torch.distributed as dist

        ax = tensor.dim() - 1
        ops, bufs = [], []
        for peer in self.peers:
            si = self._index("s", peer, sel_key, select)
            ri = self._index("r", peer, sel_key, select)
            if si is not None:
                ops.append(dist.P2POp(dist.isend, tensor.index_select(ax, si).contiguous(), peer, self.group))
            if ri is not None:
                rb = torch.empty(tuple(tensor.shape[:-1]) + (len(ri),), dtype=tensor.dtype, device=tensor.device)
                ops.append(dist.P2POp(dist.irecv, rb, peer, self.group))
                bufs.append((ri, rb))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for ri, rb in bufs:
            tensor.index_copy_(ax, ri, rb)

    def swap_from_cadence(self, tensor, min_cad: int) -> None:
        self.swap(tensor, ("ge", min_cad), lambda c: c >= min_cad)

    def swap_cadence(self, tensor, cad: int) -> None:
        self.swap(tensor, ("eq", cad), lambda c: c == cad)


class _EngineExchange:
    """Engine hooks: K_s after each stage, the new u after the step."""

    def __init__(self, eng: Engine):
        self.eng = eng
        self.gx = GhostExchange.for_engine(eng)

    def after_stage(self, i: int, s: int, elig: list[int]) -> None:
        if elig:
            t0 = time.perf_counter()
            self.gx.swap_from_cadence(self.eng._K[s], min(elig))
            if s + 1 < self.eng.p:  # the verbatim sources the owners formed for stage s+1
                self.gx.swap_from_cadence(self.eng._Y[(s + 1) & 1], min(elig))
            self.eng.counters.phases["comm"] += time.perf_counter() - t0

    def after_step(self, i: int, elig: list[int]) -> None:
        t0 = time.perf_counter()
        for c in elig:  # each cadence wrote the buffer of its new parity
            self.gx.swap_cadence(self.eng._U[self.eng._cur_parity(i + 1, c)], c)
        self.eng.counters.phases["comm"] += time.perf_counter() - t0
