"""TEST INFRASTRUCTURE ONLY — CPU oracle for the LTS/GTS octree wave path.

A restatement of the reference ``amrlts`` algorithms (``/root/reference/pkg/src/amrlts``):
tree construction (pure Python, octree.py:249-271), 2:1 balance, maximal
blocks, node registry, gathers and the record-based LTS/GTS stepper (C, see
``amr_oracle.c`` for the file:line map), and the stage-transfer algebra
(numpy, rkcorrect.py:80-121).  Pinned against goldens generated from the
reference itself (tests/test_oracle.py).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline leg may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
MAXP = 4
_LIB = None

_i32p, _i64p, _f64p, _vp = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_void_p


def build() -> str:
    src = os.path.join(HERE, "amr_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(src) > os.path.getmtime(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _LIB
    if _LIB is None:
        if os.path.exists(os.path.join(HERE, "amr_oracle.c")):
            try:
                build()
            except (OSError, subprocess.CalledProcessError):
                pass
        L = C.CDLL(LIB_PATH)
        sig = {
            "ora_wavelet_coeff": ([C.c_int, C.c_int, C.c_int64, _f64p, _f64p, _f64p], C.c_int),
            "ora_morton_sort": ([C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _i64p], C.c_int),
            "ora_balance": ([C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _i64p], _vp),
            "ora_tree_fetch": ([_vp, _i32p, _i32p], C.c_int),
            "ora_tree_free": ([_vp], None),
            "ora_mesh_build": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _i32p, _f64p, _f64p],
                               _vp),
            "ora_mesh_free": ([_vp], None),
            "ora_mesh_n_nodes": ([_vp], C.c_int64),
            "ora_mesh_n_blocks": ([_vp], C.c_int64),
            "ora_mesh_leaf_starts": ([_vp, _i64p], C.c_int),
            "ora_mesh_leaf_gids": ([_vp, _i64p], C.c_int),
            "ora_mesh_node_coords": ([_vp, _i32p], C.c_int),
            "ora_mesh_blocks": ([_vp, _i64p, _i32p, _i32p], C.c_int),
            "ora_mesh_block_gather": ([_vp, C.c_int64, _i64p, _i64p, _i64p, _i64p, _f64p], C.c_int),
            "ora_engine_new": ([_vp, C.c_int, _f64p, _f64p, C.c_double, C.c_int, C.c_int, C.c_double, C.c_double,
                                _f64p], _vp),
            "ora_engine_free": ([_vp], None),
            "ora_engine_dt_fine": ([_vp], C.c_double),
            "ora_engine_load": ([_vp, _f64p], C.c_int),
            "ora_engine_current": ([_vp, _f64p], C.c_int),
            "ora_engine_advance": ([_vp, C.c_int64, _i64p, _f64p], C.c_int),
            "ora_last_error": ([], C.c_char_p),
        }
        for k, (a, r) in sig.items():
            f = getattr(L, k)
            f.argtypes, f.restype = a, r
        _LIB = L
    return _LIB


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


# ----------------------------------------------------------------------------- octree
def construct(refine, dim: int, max_depth: int):
    """Top-down DFS refinement, Morton sorted (octree.py:249-271). Returns (anchors, levels)."""
    from types import SimpleNamespace

    leaves = []
    stack = [((0,) * dim, 0)]
    while stack:
        anchor, level = stack.pop()
        key = SimpleNamespace(anchor=anchor, level=level, max_depth=max_depth, side=1 << (max_depth - level))
        if level < max_depth and refine(key):
            half = 1 << (max_depth - level - 1)
            for code in range(1 << dim):
                stack.append((tuple(a + ((code >> d) & 1) * half for d, a in enumerate(anchor)), level + 1))
        else:
            leaves.append((anchor, level))
    an = np.array([a for a, _ in leaves], dtype=np.int32).reshape(-1, dim)
    lv = np.array([l for _, l in leaves], dtype=np.int32)
    perm = np.empty(len(lv), dtype=np.int64)
    lib().ora_morton_sort(dim, max_depth, len(lv), _p(an, C.c_int32), _p(lv, C.c_int32), _p(perm, C.c_int64))
    return an[perm], lv[perm]


def balance(dim: int, max_depth: int, anchors, levels):
    """balance_2to1 restated (octree.py:289-330); Morton sorted output."""
    an = np.ascontiguousarray(anchors, dtype=np.int32)
    lv = np.ascontiguousarray(levels, dtype=np.int32)
    n = C.c_int64(0)
    h = lib().ora_balance(dim, max_depth, len(lv), _p(an, C.c_int32), _p(lv, C.c_int32), C.byref(n))
    a2 = np.empty((n.value, dim), dtype=np.int32)
    l2 = np.empty(n.value, dtype=np.int32)
    lib().ora_tree_fetch(h, _p(a2, C.c_int32), _p(l2, C.c_int32))
    lib().ora_tree_free(h)
    return a2, l2


def partition(levels, ranks: int, mode: str):
    """weighted_partition restated (partition.py:20-91): rank ranges."""
    levels = np.asarray(levels)
    w = np.ones(len(levels)) if mode == "gts" else np.array([float(1 << int(l - levels.min())) for l in levels])
    total = float(np.sum(w))
    prefix = np.cumsum(w)
    cuts = [0]
    for r in range(1, ranks):
        cut = int(np.searchsorted(prefix, total * r / ranks)) + 1
        cuts.append(min(max(cut, cuts[-1]), len(w)))
    cuts.append(len(w))
    return [(cuts[r], cuts[r + 1]) for r in range(ranks)]


# ----------------------------------------------------------------------------- mesh
class OracleMesh:
    def __init__(self, dim, max_depth, anchors, levels, ppo=9, pad=2, lo=None, hi=None, owners=None):
        self.dim, self.L, self.ppo, self.pad = dim, max_depth, ppo, pad
        self.anchors = np.ascontiguousarray(anchors, dtype=np.int32)
        self.levels = np.ascontiguousarray(levels, dtype=np.int32)
        lo = np.array(lo if lo is not None else [0.0] * dim, dtype=np.float64)
        hi = np.array(hi if hi is not None else [float(1 << max_depth)] * dim, dtype=np.float64)
        own = None if owners is None else np.ascontiguousarray(owners, dtype=np.int32)
        self.h = lib().ora_mesh_build(dim, max_depth, ppo, pad, len(self.levels), _p(self.anchors, C.c_int32),
                                      _p(self.levels, C.c_int32), None if own is None else _p(own, C.c_int32),
                                      _p(lo, C.c_double), _p(hi, C.c_double))
        if not self.h:
            raise RuntimeError(lib().ora_last_error().decode())
        self.lo, self.hi = lo, hi
        self.n_nodes = int(lib().ora_mesh_n_nodes(self.h))
        n = len(self.levels)
        st = np.empty(n + 1, dtype=np.int64)
        lib().ora_mesh_leaf_starts(self.h, _p(st, C.c_int64))
        self.leaf_starts = st
        self.leaf_slices = np.stack([st[:-1], st[1:]], axis=1)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_mesh_free(self.h)
            self.h = None

    @property
    def leaf_gids(self):
        g = np.empty((len(self.levels), self.ppo ** self.dim), dtype=np.int64)
        lib().ora_mesh_leaf_gids(self.h, _p(g, C.c_int64))
        return g

    @property
    def node_coords(self):
        c = np.empty((self.n_nodes, self.dim), dtype=np.int32)
        lib().ora_mesh_node_coords(self.h, _p(c, C.c_int32))
        return c.astype(np.int64)

    def blocks(self):
        nb = int(lib().ora_mesh_n_blocks(self.h))
        lr = np.empty((nb, 2), dtype=np.int64)
        rl = np.empty(nb, dtype=np.int32)
        ll = np.empty(nb, dtype=np.int32)
        lib().ora_mesh_blocks(self.h, _p(lr, C.c_int64), _p(rl, C.c_int32), _p(ll, C.c_int32))
        return lr, rl, ll

    def block_gather(self, b):
        rows, nnz = C.c_int64(0), C.c_int64(0)
        lib().ora_mesh_block_gather(self.h, b, C.byref(rows), C.byref(nnz), None, None, None)
        ptr = np.empty(rows.value + 1, dtype=np.int64)
        col = np.empty(nnz.value, dtype=np.int64)
        val = np.empty(nnz.value, dtype=np.float64)
        lib().ora_mesh_block_gather(self.h, b, C.byref(rows), C.byref(nnz), _p(ptr, C.c_int64), _p(col, C.c_int64),
                                    _p(val, C.c_double))
        return ptr, col, val

    def node_physical(self):
        top = (self.ppo - 1) << self.L
        nc = self.node_coords
        return np.stack([self.lo[d] + (nc[:, d] / top) * (self.hi[d] - self.lo[d]) for d in range(self.dim)], axis=1)


# ----------------------------------------------------------------------------- RK algebra
TABLEAUS = {
    "euler": ([[0.0]], [1.0]),
    "rk2": ([[0.0, 0.0], [0.5, 0.0]], [0.0, 1.0]),
    "rk3": ([[0.0, 0.0, 0.0], [0.5, 0.0, 0.0], [-1.0, 2.0, 0.0]], [1 / 6, 2 / 3, 1 / 6]),
    "rk4": ([[0.0] * 4, [0.5, 0.0, 0.0, 0.0], [0.0, 0.5, 0.0, 0.0], [0.0, 0.0, 1.0, 0.0]],
            [1 / 6, 1 / 3, 1 / 3, 1 / 6]),
}


def transfer_matrix(a, delta, dt_from, dt_to):
    """C P(dt_to) B(delta) P(dt_from)^-1 C^-1 (rkcorrect.py:80-121)."""
    p = len(a)
    Cm = np.zeros((p, p))
    Cm[:, 0] = 1.0
    for j in range(1, p):
        for i in range(p):
            Cm[i, j] = sum(a[i][m] * Cm[m, j - 1] for m in range(i))
    B = np.zeros((p, p))
    for i in range(p):
        for j in range(i, p):
            B[i, j] = delta ** (j - i) / math.factorial(j - i)
    P_to = np.diag([dt_to ** j for j in range(p)])
    return Cm @ P_to @ B @ np.diag([dt_from ** -j for j in range(p)]) @ np.linalg.inv(Cm)


class OracleEngine:
    """Reference Engine restated (stepper.py:105-487), single rank."""

    def __init__(self, mesh: OracleMesh, tableau="rk4", cfl=0.25, mode="lts", nonlinear=False,
                 k_chi=1.0, k_phi=2.0):
        a, w = TABLEAUS[tableau]
        self.a, self.w, self.p = a, w, len(w)
        self.mesh, self.mode = mesh, mode
        nl = {False: 0, None: 0, True: 1, "sin": 1, "cubic": 2}[nonlinear]
        st = np.zeros(32)
        for off, arr in zip((0, 5, 11, 17, 22, 27), _stencils()):
            st[off:off + len(arr)] = arr
        aa = np.zeros(self.p * self.p)
        for i in range(self.p):
            for j in range(self.p):
                aa[i * self.p + j] = a[i][j]
        ww = np.array(w, dtype=np.float64)
        self.h = lib().ora_engine_new(mesh.h, self.p, _p(aa, C.c_double), _p(ww, C.c_double), cfl,
                                      1 if mode == "lts" else 0, nl, k_chi, k_phi, _p(st, C.c_double))
        self.dt_fine = float(lib().ora_engine_dt_fine(self.h))
        _, _, ll = mesh.blocks()
        self.l_max, self.l_min = int(ll.max()), int(ll.min())
        self.cads = sorted(set(ll.tolist())) if mode == "lts" else [self.l_max]
        self.i_fine = 0
        self._cache = {}

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_engine_free(self.h)
            self.h = None

    def initialize(self, chi0):
        xyz = self.mesh.node_physical()
        z = np.zeros((2, self.mesh.n_nodes))
        z[0] = chi0(*[xyz[:, d] for d in range(self.mesh.dim)])
        self.load_zip(z)

    def load_zip(self, z):
        z = np.ascontiguousarray(z, dtype=np.float64)
        lib().ora_engine_load(self.h, _p(z, C.c_double))
        self.i_fine = 0

    def current_zip(self):
        z = np.empty((2, self.mesh.n_nodes))
        lib().ora_engine_current(self.h, _p(z, C.c_double))
        return z

    def _keys(self, i):
        keys, mats = [], []
        for cr in self.cads:
            to = 1 << (self.l_max - cr)
            if i % to:
                continue
            for cs in self.cads:
                per = 1 << (self.l_max - cs)
                if i % per == 0:
                    if per != to:
                        keys.append((0, per, to))
                else:
                    d = i % per
                    keys += [(d, per, to), (0, per, d)]
        for k in keys:
            M = self._cache.get(k)
            if M is None:
                M = transfer_matrix(self.a, k[0] * self.dt_fine, k[1] * self.dt_fine, k[2] * self.dt_fine)
                if k[0] == 0:
                    M = np.tril(M)
                self._cache[k] = M
            pad = np.zeros((MAXP, MAXP))
            pad[: self.p, : self.p] = M
            mats.append(pad)
        k = np.array(keys, dtype=np.int64).reshape(-1, 3)
        m = np.array(mats, dtype=np.float64).reshape(-1, MAXP, MAXP)
        return k, m

    def advance_slice(self):
        k, m = self._keys(self.i_fine)
        k = np.ascontiguousarray(k)
        m = np.ascontiguousarray(m)
        lib().ora_engine_advance(self.h, len(k), _p(k, C.c_int64), _p(m, C.c_double))
        self.i_fine += 1

    def run_to(self, i):
        while self.i_fine < i:
            self.advance_slice()


def _stencils():
    """Fornberg weights, same recursion and op order as wave.py:22-54 (restated)."""
    def fw(m, offsets):
        x = [float(v) for v in offsets]
        n = len(x)
        c = np.zeros((n, m + 1))
        c[0, 0] = 1.0
        c1, c4 = 1.0, x[0]
        for i in range(1, n):
            mn = min(i, m)
            c2, c5, c4 = 1.0, c4, x[i]
            for j in range(i):
                c3 = x[i] - x[j]
                c2 *= c3
                if j == i - 1:
                    for k in range(mn, 0, -1):
                        c[i, k] = c1 * (k * c[i - 1, k - 1] - c5 * c[i - 1, k]) / c2
                    c[i, 0] = -c1 * c5 * c[i - 1, 0] / c2
                for k in range(mn, 0, -1):
                    c[j, k] = (c4 * c[j, k] - k * c[j, k - 1]) / c3
                c[j, 0] = c4 * c[j, 0] / c3
            c1 = c2
        return c[:, m]

    return [fw(2, range(-2, 3)), fw(2, range(0, 6)), fw(2, range(-1, 5)),
            fw(1, range(-2, 3)), fw(1, range(0, 5)), fw(1, range(-1, 4))]


# ---------------------------------------------------------------------------
# wavelet refinement criterion (wavelet.py:41-144), restated

def lagrange_matrix(src, dst, max_points=4):
    """Sliding-window Lagrange weights, wavelet.py:41-54 (same window rule and product order)."""
    npts = min(max_points, len(src))
    out = np.zeros((len(dst), len(src)))
    for i, x in enumerate(dst):
        j0 = max(0, min(int(np.searchsorted(src, x) - npts // 2), len(src) - npts))
        for a in range(npts):
            w = 1.0
            for b in range(npts):
                if a != b:
                    w *= (x - src[j0 + b]) / (src[j0 + a] - src[j0 + b])
            out[i, j0 + a] = w
    return out


def wavelet_samples(f, anchor, level, max_depth, npd, domain_lo=None, domain_hi=None):
    """f on one octant's closed npd^dim grid, wavelet.py:57-67,86-92."""
    dim = len(anchor)
    lo_d = (0.0,) * dim if domain_lo is None else domain_lo
    hi_d = (float(1 << max_depth),) * dim if domain_hi is None else domain_hi
    top = float(1 << max_depth)
    side = 1 << (max_depth - level)
    axes = [np.linspace(lo_d[d] + (anchor[d] / top) * (hi_d[d] - lo_d[d]),
                        lo_d[d] + ((anchor[d] + side) / top) * (hi_d[d] - lo_d[d]), npd) for d in range(dim)]
    return np.asarray(f(*np.meshgrid(*axes, indexing="ij")), dtype=float)


def wavelet_coeffs(values, npd, dim):
    """Coefficients of (n, npd^dim) samples through the C restatement."""
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, npd ** dim)
    xs = np.linspace(0.0, 1.0, npd)
    W = np.ascontiguousarray(lagrange_matrix(xs[::2], xs))
    out = np.zeros(v.shape[0])
    rc = lib().ora_wavelet_coeff(dim, npd, v.shape[0], v.ctypes.data_as(_f64p), W.ctypes.data_as(_f64p),
                                 out.ctypes.data_as(_f64p))
    if rc:
        raise ValueError(lib().ora_last_error().decode())
    return out


def wavelet_flag_codes(coeff, levels, tolerance, coarsen_factor, min_level, max_level):
    """refine_flags' rule, wavelet.py:118-123: 1 refine, 0 keep, -1 coarsen."""
    out = np.zeros(len(coeff), dtype=np.int8)
    for i, (c, lv) in enumerate(zip(coeff, levels)):
        if c > tolerance and lv < max_level:
            out[i] = 1
        elif c < coarsen_factor * tolerance and lv > min_level:
            out[i] = -1
    return out
