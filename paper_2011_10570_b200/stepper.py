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
  computed once per slice phase on the host and kept on the device;
* ranks: a partitioned mesh (``mesh.pmap.ranks > 1``) runs as R ranks, each
  holding only its owned leaves plus the ghost leaves its tiles read
  (``_Rank``).  Without a process group the R ranks are simulated in this
  process on one device (the reference's ``rank_records``, stepper.py:158-161)
  and ghosts move by device copies; under ``torch.distributed`` each process
  owns one rank and the same packed shipments move over NCCL.  Either way the
  shipments happen exactly where the reference calls ``_ship``
  (stepper.py:430,455): after every stage and after the step, for the leaves
  that stepped.  A rank launches the tiles other ranks read first, so the
  shipment overlaps its interior tiles.
"""
from __future__ import annotations

import os
from collections import defaultdict
from dataclasses import dataclass

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


def _as_tensors(prog: dict) -> dict:
    """The program arrays as torch tensors (CPU for the host builder's numpy
    arrays, CUDA for the device builder's), so one code path lays them out."""
    import torch

    out = dict(prog)
    for k in ("heads", "tail", "if_gid", "if_cad", "wtab"):
        v = prog[k]
        if not isinstance(v, torch.Tensor):
            v = np.ascontiguousarray(v)
            if v.dtype == np.uint16:
                v = v.view(np.int16)
            v = torch.from_numpy(v)
        out[k] = v
    return out


def _head_words(heads):
    """(n, max_head / 4) int32 view of the heads."""
    import torch

    return heads.view(torch.int32).reshape(heads.shape[0], -1)


def _base_mask(h32, nt: int):
    """The source-group base words of the first nt heads and the mask of the real (>= 0) ones."""
    import torch

    W = min(63, h32.shape[1] - 16)
    bases = h32[:nt, 16:16 + W]
    valid = (torch.arange(W, device=h32.device)[None, :] < h32[:nt, 6][:, None]) & (bases >= 0)
    return bases, valid


def _source_leaves(prog: dict, starts: np.ndarray, tile_leaves: np.ndarray) -> np.ndarray:
    """Sorted leaves whose zip nodes the programs read (their own tiles included):
    the positive source bases of every head, and the source nodes of the
    interface pairs."""
    import torch

    heads = prog["heads"]
    nt = len(tile_leaves)
    out = [np.asarray(tile_leaves, dtype=np.int64)]
    st = torch.from_numpy(np.ascontiguousarray(starts)).to(heads.device)
    if nt:
        bases, valid = _base_mask(_head_words(heads), nt)
        vals = torch.unique(bases[valid]).to(torch.int64)
        out.append((torch.searchsorted(st, vals, right=True) - 1).cpu().numpy())
    if prog["n_iface"]:
        g = torch.unique(prog["if_gid"][: prog["n_iface"]]).to(torch.int64)
        out.append((torch.searchsorted(st, g, right=True) - 1).cpu().numpy())
    return np.unique(np.concatenate(out))


class _Rank:
    """One rank's share of the mesh on a device: its tiles' stage programs, the
    zip rows of its owned leaves and of the ghost leaves those tiles read
    (owned + ghosts in leaf order, so a leaf is one contiguous range), and the
    launches of one RK stage."""

    def __init__(self, mesh: Mesh, leaf_cad: np.ndarray, lts_kernel: bool, l_max: int, rank: int, owned: np.ndarray):
        self.mesh, self.cad, self.l_max = mesh, leaf_cad, l_max
        self.rank = rank
        self.owned = np.asarray(owned, dtype=np.int64)
        self.split = False  # set by the engine: launch the lean kernel instance on tiles off the physical faces
        self.merge = os.environ.get("AMR_MERGE", "1") == "1"  # one launch when all tiles of a part step
        self.lts_kernel = lts_kernel
        self.slots = 4 * 148  # resident stage-kernel CTAs; set by the engine from the device's SM count
        cad = leaf_cad
        order = np.lexsort((self.owned, -cad[self.owned]))
        self.tiles = self.owned[order]  # cadence order; reordered by layout()
        from . import tileprog

        if not len(self.tiles):  # an empty rank (more ranks than the weights can split)
            prog = dict(heads=np.zeros((1, 64), np.uint8), tail=np.zeros(8, np.uint16), max_head=64,
                        max_slots=0, max_tail=0, if_gid=np.zeros(0, np.int32), if_cad=np.zeros(0, np.int32),
                        n_iface=0, wtab=np.zeros(1), n_rows=0, n_cells=0)
        elif mesh._nm.on_device and os.environ.get("AMR_HOST_PROGRAMS") != "1":
            # tables were built on the device: so are the programs (byte-identical to the host builder)
            prog = tileprog.build_programs_device(mesh, self.tiles.astype(np.int32), cad, lts_kernel)
        else:
            prog = tileprog.build_programs_native(mesh, self.tiles.astype(np.int32), cad, lts_kernel)
        self.prog = _as_tensors(prog)
        self.src_leaves = _source_leaves(self.prog, mesh.leaf_starts, self.tiles)
        own_mask = np.zeros(len(cad) + 1, dtype=bool)
        own_mask[self.owned] = True
        self.ghosts = self.src_leaves[~own_mask[self.src_leaves]]

    # -- layout ---------------------------------------------------------------------
    def layout(self, boundary_leaves: np.ndarray) -> None:
        """Host side: fix the launch order (tiles other ranks read first, each
        part finest cadence first) and the local node layout (owned + ghost
        leaves in leaf order), and rewrite the programs' node ids to it."""
        mesh = self.mesh
        cad = self.cad
        starts = mesh.leaf_starts
        n_leaves = len(cad)
        prog = self.prog
        # launch order: [boundary | interior], each finest cadence first
        is_b = np.zeros(n_leaves, dtype=bool)
        is_b[np.asarray(boundary_leaves, dtype=np.int64)] = True
        tb = is_b[self.tiles]
        import torch

        # tiles on a physical face need the full kernel instance (biased and radiative rows); with
        # `split` they form a second group after the lean tiles of each part
        an, lv = mesh.tree.arrays()
        side = (1 << (mesh.L - lv[self.tiles].astype(np.int64)))[:, None]
        a = an[self.tiles].astype(np.int64)
        on_face = np.any((a == 0) | (a + side == (1 << mesh.L)), axis=1) if len(self.tiles) else np.zeros(0, bool)
        tf = on_face if self.split else np.zeros(len(self.tiles), dtype=bool)
        perm = np.lexsort((self.tiles, -cad[self.tiles], ~tf, ~tb))
        self.tiles = self.tiles[perm]
        pdev = prog["heads"].device
        heads = prog["heads"][torch.from_numpy(perm).to(pdev)] if len(perm) else prog["heads"]
        tcad = cad[self.tiles]
        tb, tf = tb[perm], tf[perm]
        self.n_boundary = int(tb.sum())
        levels = range(self.l_max + 2)
        self.prefix_b = [int(np.sum(tcad[tb] >= c)) for c in levels]
        self.prefix_i = [int(np.sum(tcad[~tb] >= c)) for c in levels]
        # launch groups: (boundary | interior) x (full | lean), each finest cadence first.  The full
        # group comes first so that, when every tile of a part steps, one launch of the full instance
        # covers both groups with the long face tiles at the front of the grid (launch_plan)
        self.groups = {}
        off = 0
        for part, pm in ((True, tb), (False, ~tb)):
            for full, fm in ((True, tf), (False, ~tf)):
                sel = pm & fm
                self.groups[(part, full)] = (off, [int(np.sum(tcad[sel] >= c)) for c in levels])
                off += int(sel.sum())
        n_iface = prog["n_iface"]
        self.n_iface = n_iface
        rcad = (prog["if_cad"][:n_iface] & 0xFF).cpu().numpy() if n_iface else np.zeros(0, np.int64)
        self.if_prefix = [int(np.sum(rcad >= c)) for c in levels]
        # local layout: owned + ghost leaves in leaf order
        self.local_leaves = np.union1d(self.owned, self.ghosts)
        counts = (starts[1:] - starts[:-1])[self.local_leaves]
        lstart = np.zeros(len(self.local_leaves) + 1, dtype=np.int64)
        np.cumsum(counts, out=lstart[1:])
        self.n_local = int(lstart[-1])
        if self.n_local >= 2 ** 31 - 2:
            raise ValueError("a rank holds more than 2^31 zip nodes; partition the mesh over more ranks")
        self.leaf_lstart = np.full(n_leaves, -1, dtype=np.int64)
        self.leaf_lstart[self.local_leaves] = lstart[:-1]
        self.identity = self.n_local == mesh.n_nodes and len(self.local_leaves) == n_leaves
        if_gid = prog["if_gid"]
        if not self.identity:
            st = torch.from_numpy(np.ascontiguousarray(starts)).to(pdev)
            ls = torch.from_numpy(self.leaf_lstart).to(pdev)
            h32 = _head_words(heads)
            nt = len(self.tiles)
            if nt:
                h32[:nt, 0] = ls[torch.from_numpy(self.tiles).to(pdev)].to(torch.int32)
                bases, valid = _base_mask(h32, nt)
                old = bases[valid].to(torch.int64)
                lf = torch.searchsorted(st, old, right=True) - 1
                new = ls[lf]
                if bool(torch.any(st[lf] != old)) or bool(torch.any(new < 0)):
                    raise RuntimeError("stage programs read a leaf outside the rank's layout")
                bases[valid] = new.to(torch.int32)
            if n_iface:
                g = if_gid[:n_iface].to(torch.int64)
                lf = torch.searchsorted(st, g, right=True) - 1
                if_gid = (ls[lf] + (g - st[lf])).to(torch.int32)
            # local node -> global gid (load_zip)
            self.l2g = np.repeat(starts[self.local_leaves] - lstart[:-1], counts) + np.arange(self.n_local)
        else:
            self.l2g = None
        a, b = (int(self.owned[0]), int(self.owned[-1]) + 1) if len(self.owned) else (0, 0)
        self.own_g0, self.own_g1 = int(starts[a]), int(starts[b])  # owned gids (global), contiguous
        self.own_l0 = int(self.leaf_lstart[a]) if len(self.owned) else 0
        self.progt = dict(heads=heads, tail=prog["tail"], wtab=prog["wtab"], if_gid=if_gid, if_cad=prog["if_cad"])
        self.max_head, self.max_tail, self.max_slots = prog["max_head"], prog["max_tail"], prog["max_slots"]
        self.stats = dict(n_rows=prog["n_rows"], n_cells=prog["n_cells"])
        self.prog = None
        # the owned leaves as ranges of equal cadence (current_zip)
        oc = cad[self.owned]
        first = np.concatenate([[0], np.flatnonzero(np.diff(oc)) + 1]).astype(np.int64) if len(oc) else \
            np.zeros(0, np.int64)
        r_start = self.leaf_lstart[self.owned[first]] if len(oc) else np.zeros(0, np.int64)
        r_end = np.append(r_start[1:], self.own_l0 + (self.own_g1 - self.own_g0)) if len(oc) else r_start
        self.own_ranges_host = (r_start, r_end - r_start, oc[first] if len(oc) else np.zeros(0, np.int64))

    @property
    def host(self) -> dict:
        """The laid-out programs as numpy arrays (tests, tileprog.decode)."""
        h = self.progt
        out = {k: h[k].cpu().numpy() for k in ("heads", "wtab", "if_gid", "if_cad")}
        out["tail"] = h["tail"].cpu().numpy().view(np.uint16)
        return out

    def upload(self, eng: "Engine") -> None:
        """Device side: programs, zip rows (u0, u1, K, Y), interface buffer."""
        import torch

        self.eng = eng
        dev = eng.device
        pad = lambda x: x if x.numel() else torch.zeros(1, dtype=x.dtype)  # noqa: E731
        h = self.progt
        self.d = {k: pad(h[k]).contiguous().to(dev) for k in ("heads", "tail", "wtab", "if_gid", "if_cad")}
        self.progt = None
        n_iface = self.n_iface
        n = self.n_local
        # rows padded to an even stride ld > n (16-byte aligned rows; the kernel
        # bulk-prefetches 16-byte aligned supersets of a tile's owned range)
        self.ld = ld = (n + 2) // 2 * 2
        p = eng.p
        self.U_store = [torch.zeros((2, ld), dtype=torch.float64, device=dev) for _ in range(2)]
        self.K_store = torch.zeros((p, 2, ld), dtype=torch.float64, device=dev)
        self.Y_store = torch.zeros((2, 2, ld), dtype=torch.float64, device=dev)  # by stage parity
        self.U = [u[:, :n] for u in self.U_store]
        self.K = self.K_store[:, :, :n]
        self.Y = self.Y_store[:, :, :n]
        self.ibuf = torch.zeros((p, 2, max(n_iface, 1)), dtype=torch.float64, device=dev)  # one slab per stage
        self.prm = self._make_params()
        self.own_ranges = _Ranges(*self.own_ranges_host, dev)

    def _make_params(self) -> _native.AmrStageParams:
        eng = self.eng
        m = eng.mesh
        P = _native.AmrStageParams()
        P.dim, P.ppo, P.pad = m.dim, m.ppo, m.pad
        P.lts = 1 if eng._lts_kernel else 0
        P.n_stages = eng.p
        P.nonlinear = eng._nl
        P.n_nodes = self.n_local
        P.ld = self.ld
        d = self.d
        P.max_slots = self.max_slots
        P.if_gid, P.if_cad = d["if_gid"].data_ptr(), d["if_cad"].data_ptr()
        P.ibuf = P.ibuf0 = self.ibuf.data_ptr()
        P.n_iface_total = self.n_iface
        P.wtab, P.n_wtab = d["wtab"].data_ptr(), int(d["wtab"].numel())
        P.heads, P.max_head, P.tail = d["heads"].data_ptr(), self.max_head, d["tail"].data_ptr()
        P.threads = eng._threads
        P.max_tail = self.max_tail
        P.U0, P.U1, P.K = self.U_store[0].data_ptr(), self.U_store[1].data_ptr(), self.K_store.data_ptr()
        P.Y = self.Y_store.data_ptr()
        tab = eng.tab
        for s in range(eng.p):
            for j in range(eng.p):
                a = tab.a[s][j]
                P.g_cstage[s][j] = eng.dt_fine * a if (j < s and a != 0.0) else 0.0
            w = tab.w[s]
            P.g_comb[s] = (1 * eng.dt_fine) * w if w != 0.0 else 0.0
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
        P.r_eps = eng._r_eps
        P.r_eps2 = eng._r_eps ** 2
        P.k_chi, P.k_phi, P.f0_chi, P.f0_phi = eng.k_chi, eng.k_phi, 0.0, 0.0
        fill_weights(P)
        self.heads_ptr = d["heads"].data_ptr()
        return P

    # -- launches ---------------------------------------------------------------------
    def begin_stage(self, i: int, s: int, cmin: int) -> None:
        """Stage parameters of (slice i, stage s) and the LTS interface pass."""
        eng = self.eng
        P = self.prm
        if P.lts:
            P.coef = eng._slice_coef(i).data_ptr()
            R = eng.schedule.slices_per_round
            mask, cstage, comb = eng._coef_host[(i % R, (i // R) & 1)]
            P.l_cur_mask = mask
            for c, rows in cstage.items():
                for j in range(eng.p):
                    P.l_cnext[c][j] = rows[s + 1][j] if s + 1 < eng.p else 0.0
                    P.l_comb[c][j] = comb[c][j]
        else:
            P.gts_cur = i & 1
        P.stage = s
        vt = eng._vt[s + 1] if s + 1 < eng.p else []  # the writer forms stage s+1's sources
        P.n_vt = len(vt)
        for t, j in enumerate(vt):
            P.vt_j[t] = j
        P.n_iface = self.if_prefix[cmin]
        P.ibuf = self.ibuf.data_ptr() + s * 2 * max(self.n_iface, 1) * 8
        # stage 0 also fills every stage of the pairs whose source is not stepping at this slice;
        # later stages redo only the pairs whose source steps too — none when one cadence steps alone
        P.if_phase = 1 if s == 0 else 2
        if P.n_iface and (self.prefix_b[cmin] or self.prefix_i[cmin]) and (s == 0 or eng._n_eligible(i) > 1):
            with eng._phase("time_interp"):
                rc = eng._lib.amr_iface(C.byref(P), eng._stream())
            if rc:
                _native.check(rc, "amr_iface")

    def launch_plan(self, cmin: int, boundary: bool):
        """(first tile, tiles, lean instance?) of the stage launches of one part at cadence >= cmin.
        Lean tiles, then the face tiles (full instance).  When every tile of the part steps, both
        groups go in one launch of the full instance instead: the face tiles are about 3x a normal
        tile, and at the front of a mixed grid they overlap the rest, where a launch of their own
        leaves most of the SMs idle."""
        (off_f, pre_f), (off_l, pre_l) = self.groups[(boundary, True)], self.groups[(boundary, False)]
        n_f, n_l = pre_f[cmin], pre_l[cmin]
        if self.merge and n_f and n_l and n_f == pre_f[0] and n_l == pre_l[0]:
            # LTS: the full instance runs a lean tile about 3 % slower, and a face launch of several
            # waves is already well packed: merge when the idle slots of its last wave (x 3 tile times)
            # outweigh that (cfg2: 296 face tiles of 7 344, merged; cfg3: not).  GTS: always one launch
            idle = -n_f % self.slots
            if not self.lts_kernel or 100 * idle > n_l:
                return [(off_f, n_f + n_l, False)]
        return [(o, n, lean) for o, n, lean in ((off_l, n_l, self.split), (off_f, n_f, False)) if n]

    def launch_tiles(self, cmin: int, boundary: bool) -> None:
        P = self.prm
        for off, n, lean in self.launch_plan(cmin, boundary):
            P.n_tiles = n
            P.heads = self.heads_ptr + off * self.max_head
            P.lean = 1 if lean else 0
            with self.eng._phase("rhs"):
                rc = self.eng._lib.amr_stage(C.byref(P), self.eng._stream())
            if rc:
                _native.check(rc, "amr_stage")

    # -- state I/O ----------------------------------------------------------------------
    def load(self, zd) -> None:
        """u_pre = u_curr = the rank's nodes of the global device field zd.  K is left as it
        is: at slice 0 every leaf steps, so each K_j is written before anything reads it
        (same-step stage sources read K_j only for j below the running stage; virtual
        substeps read the K of a source's last completed step, and the first of those is
        slice 0's), and the reference's ``K = 0`` (stepper.py:224) is never observable."""
        import torch

        if self.identity:
            self.U[0].copy_(zd, non_blocking=True)
        else:
            if not hasattr(self, "_l2g_d"):
                self._l2g_d = torch.from_numpy(self.l2g).to(self.eng.device)
            self.U[0].copy_(zd.index_select(1, self._l2g_d))
        self.U[1].copy_(self.U[0])

    def shipment_rows(self, s: int, i: int):
        """(row0, row1, parity per cadence) of the record fields that changed in
        stage s of slice i: K_s (LTS interface readers need it), and the next
        stage's verbatim source or, after the last stage, the new u."""
        eng = self.eng
        ld = self.ld
        rows0, rows1 = [], []
        if self.prm.lts:
            k = self.K_store.data_ptr() + s * 2 * ld * 8
            rows0 += [k, k + ld * 8]
            rows1 += [k, k + ld * 8]
        par = [0] * _native.AMR_MAXL
        if s + 1 < eng.p:
            y = self.Y_store.data_ptr() + ((s + 1) & 1) * 2 * ld * 8
            rows0 += [y, y + ld * 8]
            rows1 += [y, y + ld * 8]
        else:
            u0, u1 = self.U_store[0].data_ptr(), self.U_store[1].data_ptr()
            rows0 += [u0, u0 + ld * 8]
            rows1 += [u1, u1 + ld * 8]
            for c in range(eng.l_max + 1):  # each cadence wrote the buffer of its new parity
                par[c] = eng._cur_parity(i + 1, c) if self.prm.lts else (i + 1) & 1
        return rows0, rows1, par


class _Ranges:
    """Whole-leaf zip ranges of one rank's layout, finest cadence first, on the
    device, with the prefix sizes per minimum cadence."""

    def __init__(self, start, length, cad, device):
        import torch

        start = np.asarray(start, dtype=np.int64)
        length = np.asarray(length, dtype=np.int64)
        cad = np.asarray(cad, dtype=np.int64)
        self.n = len(start)
        off = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(length, out=off[1:])
        self.total = int(off[-1])
        self.off_host = off
        self.cad_host = cad
        T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(device)  # noqa: E731
        self.start = T(start if self.n else np.zeros(1, np.int64))
        self.off = T(off)
        self.cad = T((cad if self.n else np.zeros(1, np.int64)).astype(np.int32))

    def prefix(self, cmin: int):
        """(ranges, nodes) with cadence >= cmin; ranges must be sorted finest first."""
        k = int(np.sum(self.cad_host >= cmin))
        return k, int(self.off_host[k])

    def move(self, n_ranges: int, total: int, rows0, rows1, par, buf_ld: int = 0) -> _native.AmrGhostMove:
        M = _native.AmrGhostMove()
        M.n_ranges, M.total, M.buf_ld = n_ranges, total, buf_ld
        M.start, M.off, M.cad = self.start.data_ptr(), self.off.data_ptr(), self.cad.data_ptr()
        M.n_rows = len(rows0)
        for r, (a, b) in enumerate(zip(rows0, rows1)):
            M.row0[r], M.row1[r] = a, b
        for c, v in enumerate(par):
            M.par[c] = v
        return M


class _Link:
    """Shipments of one (sender, receiver) pair: the sender's leaves the
    receiver's tiles read, finest cadence first, as ranges of each side's layout."""

    def __init__(self, leaves, cad, starts, send_lstart, recv_lstart, device, rows_max):
        import torch

        leaves = np.asarray(leaves, dtype=np.int64)
        order = np.lexsort((leaves, -cad[leaves]))
        leaves = leaves[order]
        self.leaves = leaves
        length = (starts[1:] - starts[:-1])[leaves]
        lc = cad[leaves]
        self.send = _Ranges(send_lstart[leaves], length, lc, device) if send_lstart is not None else None
        self.recv = _Ranges(recv_lstart[leaves], length, lc, device) if recv_lstart is not None else None
        total = int(length.sum())
        self.total = total
        self.sbuf = torch.empty(max(rows_max * total, 1), dtype=torch.float64, device=device) \
            if send_lstart is not None else None
        self.rbuf = torch.empty(max(rows_max * total, 1), dtype=torch.float64, device=device) \
            if recv_lstart is not None else None


def _ship_lists(need: dict, rank_ranges) -> dict:
    """{(sender, receiver): leaves} from each receiver's ghost-leaf list."""
    out = {}
    for r, ghosts in need.items():
        ghosts = np.asarray(ghosts, dtype=np.int64)
        for q, (a, b) in enumerate(rank_ranges):
            if q == r:
                continue
            sel = ghosts[(ghosts >= a) & (ghosts < b)]
            if len(sel):
                out[(q, r)] = sel
    return out


class _LocalTransport:
    """Simulated ranks in one process (the reference's rank_records,
    stepper.py:158-161, 318-333): every shipment is packed from the sender's
    rows, copied buffer to buffer, and unpacked into the receiver's ghost rows,
    all on the engine's stream."""

    def __init__(self, eng: "Engine", ranks: dict, lists: dict):
        self.eng = eng
        self.ranks = ranks
        cad, starts = eng._leaf_cadence, eng.mesh.leaf_starts
        self.links = {(q, r): _Link(lv, cad, starts, ranks[q].leaf_lstart, ranks[r].leaf_lstart, eng.device, 4)
                      for (q, r), lv in sorted(lists.items())}
        self.bytes_moved = 0

    def ship(self, i: int, s: int, cmin: int) -> None:
        eng = self.eng
        lib, st = eng._lib, eng._stream()
        with eng._phase("comm"):
            for (q, r), lk in self.links.items():
                k, tot = lk.send.prefix(cmin)
                if not k:
                    continue
                rows0, rows1, par = self.ranks[q].shipment_rows(s, i)
                _native.check(lib.amr_ghost_pack(C.byref(lk.send.move(k, tot, rows0, rows1, par)),
                                                 lk.sbuf.data_ptr(), st), "amr_ghost_pack")
                n = len(rows0) * tot
                lk.rbuf[:n].copy_(lk.sbuf[:n])  # the wire
                rows0, rows1, par = self.ranks[r].shipment_rows(s, i)
                _native.check(lib.amr_ghost_unpack(C.byref(lk.recv.move(k, tot, rows0, rows1, par)),
                                                   lk.rbuf.data_ptr(), st), "amr_ghost_unpack")
                self.bytes_moved += 8 * n

    def finish(self) -> None:
        pass


class _DistTransport:
    """One rank per process over torch.distributed: NCCL point-to-point between
    GPUs (device buffers, a side stream so the interior tiles overlap the
    shipment), or gloo through host staging (CPU-side tests)."""

    def __init__(self, eng: "Engine", rk: _Rank, lists: dict, group):
        import torch
        import torch.distributed as dist

        self.eng, self.rk, self.group = eng, rk, group
        cad, starts = eng._leaf_cadence, eng.mesh.leaf_starts
        me = rk.rank
        self.out = {r: _Link(lv, cad, starts, rk.leaf_lstart, None, eng.device, 4)
                    for (q, r), lv in sorted(lists.items()) if q == me}
        self.inc = {q: _Link(lv, cad, starts, None, rk.leaf_lstart, eng.device, 4)
                    for (q, r), lv in sorted(lists.items()) if r == me}
        self.host = dist.get_backend(group) != "nccl"
        self.global_rank = (lambda r: dist.get_global_rank(group, r)) if group is not dist.group.WORLD else (lambda r: r)
        self.comm = torch.cuda.Stream(eng.device)
        self.bytes_moved = 0

    def ship(self, i: int, s: int, cmin: int) -> None:
        import torch
        import torch.distributed as dist

        eng, rk = self.eng, self.rk
        lib = eng._lib
        cur = torch.cuda.current_stream(eng.device)
        self.comm.wait_stream(cur)  # the boundary tiles of this stage are queued on `cur`
        rows0, rows1, par = rk.shipment_rows(s, i)
        nr = len(rows0)
        with eng._phase("comm"), torch.cuda.stream(self.comm):
            st = self.comm.cuda_stream
            ops, recvs = [], []
            for r, lk in self.out.items():
                k, tot = lk.send.prefix(cmin)
                if not k:
                    continue
                _native.check(lib.amr_ghost_pack(C.byref(lk.send.move(k, tot, rows0, rows1, par)),
                                                 lk.sbuf.data_ptr(), st), "amr_ghost_pack")
                buf = lk.sbuf[: nr * tot]
                if self.host:
                    buf = buf.cpu()
                ops.append(dist.P2POp(dist.isend, buf, self.global_rank(r), self.group))
                self.bytes_moved += 8 * nr * tot
            for q, lk in self.inc.items():
                k, tot = lk.recv.prefix(cmin)
                if not k:
                    continue
                buf = lk.rbuf[: nr * tot]
                hb = torch.empty(nr * tot, dtype=torch.float64) if self.host else buf
                ops.append(dist.P2POp(dist.irecv, hb, self.global_rank(q), self.group))
                recvs.append((lk, k, tot, buf, hb))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()  # NCCL: orders the comm stream after the transfer (no host block)
            for lk, k, tot, buf, hb in recvs:
                if self.host:
                    buf.copy_(hb)
                _native.check(lib.amr_ghost_unpack(C.byref(lk.recv.move(k, tot, rows0, rows1, par)),
                                                   buf.data_ptr(), st), "amr_ghost_unpack")

    def finish(self) -> None:
        """The next launches on the engine's stream see the unpacked ghosts."""
        import torch

        torch.cuda.current_stream(self.eng.device).wait_stream(self.comm)


class Engine:
    """Wave-system timestepper over a block mesh, global or local mode, on one GPU:
    all ranks of a partitioned mesh simulated in-process, or one rank per
    process under torch.distributed (``process_group``)."""

    NVARS = 2

    def __init__(self, mesh: Mesh, tableau: str | ButcherTableau = "rk3", cfl: float = 0.25,
                 mode: str = "lts", nonlinear=False, k_chi: float = 1.0, k_phi: float = 2.0,
                 threads: int = 1, single_stage_neighbors: bool = False, device=None, process_group=None,
                 profile: bool = False):
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
        self._coef_host: dict = {}
        self._prof = [] if profile else None
        if profile:
            self.use_graphs = False

        # -- device -------------------------------------------------------------------
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise RuntimeError("the engine runs on CUDA devices only (no CPU path)")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._lib = _native.lib()
        self._threads = int(os.environ.get("AMR_THREADS", "256"))
        n_leaves = len(mesh.tree)
        leaf_cad = np.empty(n_leaves, dtype=np.int32)
        for b in mesh.blocks:
            leaf_cad[b.leaf_range[0]: b.leaf_range[1]] = cadence[b.index]
        self._leaf_cadence = leaf_cad
        self._lts_kernel = mode == "lts" or any(c != self.l_max for c in cadence)
        self._vt = [[j for j in range(s_) if self.tab.a[s_][j] != 0.0] for s_ in range(self.p)]

        # -- ranks ----------------------------------------------------------------------
        # distributed (one rank here) only with an explicit process group, or when
        # the default group's size is the mesh's rank count; otherwise a
        # partitioned mesh runs as simulated ranks in this process
        R = mesh.pmap.ranks
        dist = torch.distributed
        self._dist = None
        self.rank = 0
        if process_group is not None:
            if process_group is True:
                process_group = dist.group.WORLD
            ws = dist.get_world_size(process_group)
            if ws != R:
                raise ValueError(f"mesh is partitioned for {R} ranks, process group has {ws}")
            self._dist = process_group
            self.rank = dist.get_rank(process_group)
        elif R > 1 and process_group is None and dist.is_available() and dist.is_initialized() \
                and dist.get_world_size() == R:
            self._dist = dist.group.WORLD
            self.rank = dist.get_rank()
        rr = mesh.pmap.rank_ranges
        with torch.cuda.device(self.device):
            if self._dist is not None:
                local = {self.rank: _Rank(mesh, leaf_cad, self._lts_kernel, self.l_max, self.rank, np.arange(*rr[self.rank]))}
                gathered = [None] * R
                dist.all_gather_object(gathered, local[self.rank].ghosts.tolist(), group=self._dist)
                need = {r: np.asarray(g, dtype=np.int64) for r, g in enumerate(gathered)}
            elif R > 1:
                local = {r: _Rank(mesh, leaf_cad, self._lts_kernel, self.l_max, r, np.arange(*rr[r])) for r in range(R)}
                need = {r: rk.ghosts for r, rk in local.items()}
            else:
                local = {0: _Rank(mesh, leaf_cad, self._lts_kernel, self.l_max, 0, np.arange(n_leaves))}
                need = {}
            lists = _ship_lists(need, rr) if need else {}
            # GTS engines use the split only for its tile order (face tiles first, one launch)
            split = self._nl != 1 and os.environ.get("AMR_SPLIT", "1") == "1" \
                and (self._lts_kernel or os.environ.get("AMR_SPLIT_GTS", "1") == "1")
            slots = 4 * torch.cuda.get_device_properties(self.device).multi_processor_count
            for r, rk in local.items():
                rk.split = split
                rk.slots = slots
                sent = [lv for (q, _), lv in lists.items() if q == r]
                rk.layout(np.unique(np.concatenate(sent)) if sent else np.zeros(0, np.int64))
                rk.upload(self)
            self._ranks = local
            self._rank_list = [local[r] for r in sorted(local)]
            if self._dist is not None:
                self._transport = _DistTransport(self, local[self.rank], lists, self._dist)
            elif R > 1:
                self._transport = _LocalTransport(self, local, lists)
            else:
                self._transport = None
        self.ghost_lists = lists

    # single-rank views kept for tools and tests
    @property
    def _prm(self):
        return self._rank_list[0].prm

    @property
    def _d(self):
        rk = self._rank_list[0]
        return dict(rk.d, tiles=rk.tiles)

    @property
    def _U(self):
        return self._rank_list[0].U

    @property
    def _K(self):
        return self._rank_list[0].K

    @property
    def _prefix(self):
        rk = self._rank_list[0]
        return {c: rk.prefix_b[c] + rk.prefix_i[c] for c in range(self.l_max + 1)}

    def _stream(self) -> int:
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

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

    # -- phase timing (stepper.py:72-84 buckets, on the device) ---------------------------
    def _phase(self, name: str):
        return _PhaseTimer(self, name) if self._prof is not None else _NO_TIMER

    def phase_ms(self) -> dict:
        """Device milliseconds per phase bucket since construction (profile=True):
        ``time_interp`` (LTS interface pass), ``rhs`` (the fused unzip + RHS + zip
        stage kernel, which also covers the reference's ``blk_sync``), ``comm``."""
        import torch

        if self._prof is None:
            raise RuntimeError("construct the engine with profile=True")
        torch.cuda.synchronize(self.device)
        for name, a, b in self._prof:
            self.counters.phases[name] += a.elapsed_time(b) * 1e-3
        self._prof.clear()
        return {k: 1e3 * v for k, v in self.counters.phases.items()}

    # -- state I/O -----------------------------------------------------------------------
    def initialize(self, chi0, phi0=None, device_eval: bool = False) -> None:
        """Evaluate initial data on the zip nodes and load all state
        (stepper.py:198-211).  ``device_eval``: evaluate ``chi0`` / ``phi0``
        (elementwise, written with array methods or torch ops) on device coordinates
        instead of numpy on the host — for meshes where a host pass over every
        node is the slow part (cfg5); transcendentals then round as CUDA's, not
        libm's, so the data is not bit-identical to the host evaluation."""
        if device_eval:
            import torch

            with torch.cuda.device(self.device):
                xs = self.mesh.node_physical_device()
                n = self.mesh.n_nodes
                z = torch.zeros((self.NVARS, n), dtype=torch.float64, device=self.device)
                step = 1 << 26  # nodes per evaluation (elementwise functions): bounded temporaries
                for a in range(0, n, step):
                    part = [x[a:a + step] for x in xs]
                    z[0, a:a + step] = chi0(*part)
                    if phi0 is not None:
                        z[1, a:a + step] = phi0(*part)
                del xs
            self.load_zip(z)
            return
        xyz = self.mesh.node_physical()
        coords = [xyz[:, d] for d in range(self.mesh.dim)]
        z = np.zeros((self.NVARS, self.mesh.n_nodes))
        z[0] = np.asarray(chi0(*coords), dtype=float)
        if phi0 is not None:
            z[1] = np.asarray(phi0(*coords), dtype=float)
        self.load_zip(z)

    def load_zip(self, z) -> None:
        """Load a (2, n_nodes) zip field (host numpy, pinned host or device tensor):
        u_pre = u_curr = z, time 0 (stepper.py:213-230)."""
        import torch

        if not isinstance(z, torch.Tensor):
            z = torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64))
        if tuple(z.shape) != (self.NVARS, self.mesh.n_nodes):
            raise ValueError(f"zip field must be (2, {self.mesh.n_nodes}), got {tuple(z.shape)}")
        z = z.to(dtype=torch.float64)
        with torch.cuda.device(self.device):
            one = self._rank_list[0]
            if len(self._rank_list) == 1 and one.identity:
                one.load(z)  # straight into the live buffer: one host->device DMA
            else:
                zd = z.to(self.device, non_blocking=True)
                for rk in self._rank_list:
                    rk.load(zd)
        self.i_fine = 0

    @property
    def time(self) -> float:
        return self.i_fine * self.dt_fine

    def _cur_parity(self, i: int, cad: int) -> int:
        per = 1 << (self.l_max - cad)
        return ((i + per - 1) // per) & 1

    def current_zip_device(self, out=None):
        """(2, n_nodes) float64 device tensor of every leaf's u_curr: each rank's
        owned ranges read from the buffer of their cadence's parity (one gather
        launch per rank).  Under torch.distributed the ranks' parts are summed
        into the global field (every other entry is zero)."""
        import torch

        n = self.mesh.n_nodes
        i = self.i_fine
        with torch.cuda.device(self.device):
            if out is None:
                out = torch.empty((2, n), dtype=torch.float64, device=self.device)
            if self._dist is not None:
                out.zero_()  # the other ranks' entries: summed in below
            par = [(self._cur_parity(i, c) if self._lts_kernel else i & 1) if c <= self.l_max else 0
                   for c in range(_native.AMR_MAXL)]
            st = self._stream()
            for rk in self._rank_list:
                rg = rk.own_ranges
                if not rg.total:
                    continue
                u0, u1, ld = rk.U_store[0].data_ptr(), rk.U_store[1].data_ptr(), rk.ld
                M = rg.move(rg.n, rg.total, [u0, u0 + 8 * ld], [u1, u1 + 8 * ld], par, buf_ld=n)
                _native.check(self._lib.amr_ghost_pack(C.byref(M), out.data_ptr() + 8 * rk.own_g0, st),
                              "amr_ghost_pack")
            if self._dist is not None:
                torch.distributed.all_reduce(out, group=self._dist)
        return out

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
            st = self.__dict__["_snap"] = [
                [torch.empty((2, self.mesh.n_nodes), dtype=torch.float64, device=self.device), None] for _ in range(2)]
            self.__dict__["_snap_i"] = 0
        j = self.__dict__["_snap_i"]
        self.__dict__["_snap_i"] = j ^ 1
        buf, prev = st[j]
        if prev is not None:
            cur.wait_event(prev)
        self.current_zip_device(out=buf)
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
        # the entries the stage kernel takes by value (same bits)
        mask = 0
        for c in cads:
            mask |= (cf.cur[c] & 1) << c
        self._coef_host[key] = (mask,
                                {c: [[cf.cstage[c][s][j] for j in range(p)] for s in range(p)] for c in cads},
                                {c: [cf.comb[c][j] for j in range(p)] for c in cads})
        return t

    # -- the slice ------------------------------------------------------------------------------
    def _eligible_cadences(self, i: int) -> list[int]:
        return [c for c in sorted(set(self.cadence)) if i % (1 << (self.l_max - c)) == 0]

    def _n_eligible(self, i: int) -> int:
        return len(self._eligible_cadences(i))

    def advance_slice(self) -> None:
        """Advance every block eligible at the current fine slice by one of its steps.

        Per stage and rank: the LTS interface pass, the tiles other ranks read,
        the shipment of what they wrote (K_s and the next stage's verbatim
        source, or the new u after the last stage) while the interior tiles
        run; the next stage starts when the ghosts have landed."""
        import torch

        i = self.i_fine
        elig = self._eligible_cadences(i)
        if elig:
            cmin = min(elig)
            tr = self._transport
            with torch.cuda.device(self.device):
                for s in range(self.p):
                    for rk in self._rank_list:
                        rk.begin_stage(i, s, cmin)
                        rk.launch_tiles(cmin, True)
                    if tr is not None:
                        tr.ship(i, s, cmin)
                    for rk in self._rank_list:
                        rk.launch_tiles(cmin, False)
                    if tr is not None:
                        tr.finish()
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
        if self.use_graphs and self._graphable():
            self._replay_round(R)
            return
        for _ in range(R):
            self.advance_slice()

    # -- CUDA graphs ----------------------------------------------------------------------
    use_graphs = True

    def _graphable(self) -> bool:
        """Single-rank and simulated-rank rounds are pure launch sequences on one
        stream.  NCCL shipments can be captured too (AMR_GRAPH_NCCL=1); that
        path has not run on multi-GPU hardware, so it is opt-in."""
        if self._dist is None:
            return True
        return (not self._transport.host) and os.environ.get("AMR_GRAPH_NCCL") == "1"

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
                if self._lts_kernel:
                    self._slice_coef(i)
            torch.cuda.synchronize(self.device)
            moved = self._transport.bytes_moved if self._transport is not None else 0
            for start in (i_next, i_next + R):
                graph = torch.cuda.CUDAGraph()
                self.i_fine = start
                with torch.cuda.graph(graph):
                    for _ in range(R):
                        self.advance_slice()
                self._untally_round(start, R)
                self._graphs[(start // R) & 1] = graph
            if self._transport is not None:
                self._round_bytes = (self._transport.bytes_moved - moved) // 2
                self._transport.bytes_moved = moved
            self.i_fine = i_next
            return
        i0 = self.i_fine
        self._graphs[(i0 // R) & 1].replay()
        self._tally_round(i0, R)
        if self._transport is not None:
            self._transport.bytes_moved += self._round_bytes
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
        """Stage-path kernel launches advance_slice(i) issues on this process
        (LTS interface passes and stage kernels; shipments not counted)."""
        el = self._eligible_cadences(i)
        if not el:
            return 0
        c = min(el)
        n = 0
        for rk in self._rank_list:
            tiles = len(rk.launch_plan(c, True)) + len(rk.launch_plan(c, False))
            iface = (1 if len(el) == 1 else self.p) if tiles and rk.if_prefix[c] else 0
            n += self.p * tiles + iface
        return n

    @property
    def comm_bytes(self) -> int:
        """Ghost bytes shipped so far (sent by the ranks held in this process)."""
        return self._transport.bytes_moved if self._transport is not None else 0

    def close(self):
        self._transport = None


class _PhaseTimer:
    def __init__(self, eng: Engine, name: str):
        self.eng, self.name = eng, name

    def __enter__(self):
        import torch

        self.a = torch.cuda.Event(enable_timing=True)
        self.a.record(torch.cuda.current_stream(self.eng.device))
        return self

    def __exit__(self, *exc):
        import torch

        b = torch.cuda.Event(enable_timing=True)
        b.record(torch.cuda.current_stream(self.eng.device))
        self.eng._prof.append((self.name, self.a, b))
        return False


class _NoTimer:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_NO_TIMER = _NoTimer()


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
