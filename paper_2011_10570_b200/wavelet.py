"""Interpolation-residual ("wavelet") refinement criterion — drop-in for
``amrlts.wavelet`` (wavelet.py:1-144), with the per-octant coefficient on the
GPU.

The coefficient of an octant is how badly a field is rebuilt from the
even-index subset of an odd tensor grid of samples: 4-point Lagrange windows
one axis after the other, max-norm of the mismatch on the remaining nodes
(wavelet.py:70-105).  Here all octants of a tree (or of one construction
level) go through ONE launch of ``amr_wavelet_coeff`` (csrc/amr_wavelet.cu),
which also applies the refine/keep/coarsen rule or the construction predicate.

Host side: the sample coordinates (``np.linspace`` per octant and axis, the
reference's own expressions, vectorised over octants) and the call of the
user's field function ``f`` — a Python callable, as in the reference — in
chunks streamed through pinned buffers to the device.  When the sampled
field is already on the device (a solution on the leaf lattice, say), the
``*_from_values`` entry points skip the host entirely.

Results are bit-identical to the reference: the kernel reproduces its
np.tensordot (OpenBLAS dgemm) arithmetic, see tests/test_wavelet*.py.
"""
from __future__ import annotations

from dataclasses import dataclass
import os
from enum import Enum
from typing import Callable

import numpy as np

from . import _native
from .octree import LinearOctree, OctKey

_CHUNK_VALUES = 1 << 22  # samples per host->device chunk (32 MiB of fp64)
# Threads evaluating f on host chunks.  f is called on chunked (n, npd, ...) coordinate
# arrays; the reference calls it once per octant on (npd,)*dim grids, in order.  For an
# elementwise f (every reference test and BASELINE predicate) the samples are the same
# bits either way.  An f that is not elementwise or not thread-safe must not be batched:
# AMR_WAVELET_WORKERS=1 evaluates chunks one at a time, and `_probe_elementwise` refuses
# an f whose values on an octant change with the rest of the batch.
_HOST_WORKERS = max(1, int(os.environ.get("AMR_WAVELET_WORKERS", "8")))
_PINNED: list = []


def _pinned(count: int, numel: int):
    """Reusable pinned staging buffers (pinning is slow; keep them across calls)."""
    import torch

    global _PINNED
    if len(_PINNED) < count or (_PINNED and _PINNED[0].numel() < numel):
        _PINNED = [torch.empty(max(numel, _PINNED[0].numel() if _PINNED else 0), dtype=torch.float64).pin_memory()
                   for _ in range(max(count, len(_PINNED)))]
    return _PINNED[:count]


class Flag(Enum):
    """wavelet.py:19-22."""

    REFINE = "refine"
    KEEP = "keep"
    COARSEN = "coarsen"


_FLAG_OF_CODE = {1: Flag.REFINE, 0: Flag.KEEP, -1: Flag.COARSEN}


@dataclass(frozen=True)
class RefinePolicy:
    """Thresholds and level clamps (wavelet.py:25-39), same validation."""

    tolerance: float
    coarsen_factor: float = 0.1
    min_level: int = 0
    max_level: int = 31

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if not 0 < self.coarsen_factor < 1:
            raise ValueError("coarsen_factor must be in (0, 1)")
        if self.min_level > self.max_level:
            raise ValueError("min_level must not exceed max_level")


def _lagrange_matrix(src: np.ndarray, dst: np.ndarray, max_points: int = 4) -> np.ndarray:
    """Sliding-window Lagrange interpolation matrix (wavelet.py:41-54).

    Host constant (npd x nc), computed with the reference's window rule and
    product order so the device kernel sees the reference's weight bits.
    """
    npts = min(max_points, len(src))
    out = np.zeros((len(dst), len(src)))
    for i, x in enumerate(dst):
        j0 = int(np.searchsorted(src, x) - npts // 2)
        j0 = max(0, min(j0, len(src) - npts))
        xs = src[j0: j0 + npts]
        for a in range(npts):
            w = 1.0
            for b in range(npts):
                if a != b:
                    w *= (x - xs[b]) / (xs[a] - xs[b])
            out[i, j0 + a] = w
    return out


def _check_npd(nodes_per_dim: int) -> None:
    if nodes_per_dim < 3 or nodes_per_dim % 2 == 0:
        raise ValueError("nodes_per_dim must be odd and >= 3")
    if nodes_per_dim > 15:
        raise ValueError("nodes_per_dim > 15 is not supported by the device kernel")


def _domain(dim: int, max_depth: int, domain_lo, domain_hi):
    if domain_lo is None:
        domain_lo = (0.0,) * dim
    if domain_hi is None:
        domain_hi = (float(1 << max_depth),) * dim
    return tuple(domain_lo), tuple(domain_hi)


def octant_samples(key: OctKey, domain_lo, domain_hi, nodes_per_dim: int):
    """Physical tensor-grid coordinates covering the octant (wavelet.py:57-67)."""
    top = float(1 << key.max_depth)
    axes = []
    for d in range(key.dim):
        lo = domain_lo[d] + (key.anchor[d] / top) * (domain_hi[d] - domain_lo[d])
        hi = domain_lo[d] + ((key.anchor[d] + key.side) / top) * (domain_hi[d] - domain_lo[d])
        axes.append(np.linspace(lo, hi, nodes_per_dim))
    return np.meshgrid(*axes, indexing="ij")


def _sample_axes(anchors: np.ndarray, levels: np.ndarray, max_depth: int, domain_lo, domain_hi,
                 npd: int) -> list[np.ndarray]:
    """Per-octant sample axes, [dim] x (n, npd): octant_samples' expressions
    elementwise over octants (same fp64 operations, same np.linspace)."""
    top = float(1 << max_depth)
    side = np.left_shift(np.int64(1), max_depth - levels.astype(np.int64))
    out = []
    for d in range(anchors.shape[1]):
        a = anchors[:, d].astype(np.int64)
        ext = domain_hi[d] - domain_lo[d]
        lo = domain_lo[d] + (a / top) * ext
        hi = domain_lo[d] + ((a + side) / top) * ext
        out.append(np.linspace(lo, hi, npd, axis=-1))
    return out


def _sample_values(f: Callable, axes: list[np.ndarray], npd: int) -> np.ndarray:
    """f on every octant's meshgrid(ij), one call per chunk: (n, npd^dim)."""
    dim = len(axes)
    n = axes[0].shape[0]
    shape = (n,) + (npd,) * dim
    grids = []
    for d, ax in enumerate(axes):
        view = ax.reshape((n,) + tuple(npd if e == d else 1 for e in range(dim)))
        grids.append(np.ascontiguousarray(np.broadcast_to(view, shape)))
    vals = np.asarray(f(*grids), dtype=float)
    if vals.shape != shape:  # f returned a broadcastable array (e.g. a constant)
        vals = np.array(np.broadcast_to(vals, shape))
    if n > 1:
        _probe_elementwise(f, grids, vals, shape)
    return vals.reshape(n, -1)


def _probe_elementwise(f: Callable, grids, vals: np.ndarray, shape) -> None:
    """The reference evaluates f octant by octant; batching is only the same
    function for an elementwise f.  Check it on the first octant of the batch."""
    one = np.asarray(f(*[g[:1] for g in grids]), dtype=float)
    one = np.broadcast_to(one, (1,) + tuple(shape[1:]))
    if not np.array_equal(one, vals[:1], equal_nan=True):
        raise ValueError("the field function is not elementwise: its values on one octant change when octants "
                         "are batched; evaluate it per octant (wavelet_coefficient) instead")


_LAUNCHERS: dict = {}


def _launcher(dim: int, npd: int, device=None) -> "_Launcher":
    """One _Launcher (and one upload of W) per (dim, npd, device)."""
    import torch

    dev = torch.device("cuda") if device is None else torch.device(device)
    if dev.type == "cuda" and dev.index is None and torch.cuda.is_available():
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (dim, npd, str(dev))
    L = _LAUNCHERS.get(key)
    if L is None:
        L = _LAUNCHERS[key] = _Launcher(dim, npd, dev)
    return L


class _Launcher:
    """Device constants and the launch of amr_wavelet_coeff."""

    def __init__(self, dim: int, npd: int, device=None):
        import torch

        if not torch.cuda.is_available():
            raise _native.NativeError("wavelet coefficients run on the GPU; no CUDA device is available")
        self.torch = torch
        self.dim, self.npd = dim, npd
        self.dev = torch.device("cuda") if device is None else torch.device(device)
        xs = np.linspace(0.0, 1.0, npd)
        self.W = torch.from_numpy(np.ascontiguousarray(_lagrange_matrix(xs[::2], xs))).to(self.dev)
        self.lib = _native.lib()

    def launch(self, values, levels, mode, policy, coeff, flags, stream) -> None:
        tol = cthr = 0.0
        lo, hi = 0, 0
        if policy is not None:
            tol = float(policy.tolerance)
            cthr = float(policy.coarsen_factor * policy.tolerance)
            lo, hi = int(policy.min_level), int(policy.max_level)
        n = values.shape[0]
        _native.check(self.lib.amr_wavelet_coeff(
            self.dim, self.npd, n, values.data_ptr(), self.W.data_ptr(),
            levels.data_ptr() if levels is not None else None, mode, tol, cthr, lo, hi,
            coeff.data_ptr() if coeff is not None else None,
            flags.data_ptr() if flags is not None else None, stream), "amr_wavelet_coeff")


def _device_samples(torch, f, anchors_d, levels_d, max_depth, domain_lo, domain_hi, npd):
    """_sample_axes + _sample_values on the device: the same fp64 operations
    one kernel each (no contraction), so the coordinates equal numpy's bit for
    bit; ``f`` gets CUDA tensors (torch ops) and its values never leave HBM."""
    n, dim = anchors_d.shape
    top = float(1 << max_depth)
    side = torch.bitwise_left_shift(torch.ones_like(levels_d, dtype=torch.int64), max_depth - levels_d.to(torch.int64))
    ar = torch.arange(npd, dtype=torch.float64, device=anchors_d.device)
    shape = (n,) + (npd,) * dim
    grids = []
    for d in range(dim):
        a = anchors_d[:, d]
        ext = domain_hi[d] - domain_lo[d]
        # true divisions by tensors: torch turns "tensor / python scalar" into
        # a multiplication by the reciprocal, which is not numpy's rounding
        lo = (a.to(torch.float64) / torch.full_like(ar[:1], top)) * ext + domain_lo[d]
        hi = ((a + side).to(torch.float64) / torch.full_like(ar[:1], top)) * ext + domain_lo[d]
        step = (hi - lo) / torch.full_like(ar[:1], float(npd - 1))  # np.linspace: arange*step + start, last = stop
        ax = ar[None, :] * step[:, None]
        ax = ax + lo[:, None]
        ax[:, -1] = hi
        view = ax.reshape((n,) + tuple(npd if e == d else 1 for e in range(dim)))
        grids.append(view.expand(shape).contiguous())
    vals = f(*grids)
    vals = torch.as_tensor(vals, dtype=torch.float64, device=anchors_d.device)
    return vals.expand(shape).reshape(n, -1).contiguous()


def _run(f: Callable, anchors: np.ndarray, levels: np.ndarray, max_depth: int, npd: int, domain_lo, domain_hi,
         mode: int, policy, device=None, device_eval: bool = False):
    """Stream f's samples to the device chunk by chunk; return (coeff, flags)
    as host arrays (flags None without a policy).  device_eval: sample on the
    device, ``f`` called with CUDA tensors."""
    _check_npd(npd)
    n, dim = anchors.shape
    L = _launcher(dim, npd, device)
    torch = L.torch
    nv = npd ** dim
    coeff = torch.empty(n, dtype=torch.float64, device=L.dev)
    flags = lvl = None
    if policy is not None:
        flags = torch.empty(n, dtype=torch.int8, device=L.dev)
        lvl = torch.from_numpy(np.array(levels, dtype=np.int32)).to(L.dev)
    if device_eval:
        stream = torch.cuda.current_stream(L.dev).cuda_stream
        an_d = torch.from_numpy(np.ascontiguousarray(anchors, dtype=np.int64)).to(L.dev)
        lv_d = torch.from_numpy(np.array(levels, dtype=np.int32)).to(L.dev)
        chunk = max(1, (_CHUNK_VALUES * 4) // nv)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            vals = _device_samples(torch, f, an_d[s:e], lv_d[s:e], max_depth, domain_lo, domain_hi, npd)
            L.launch(vals, lvl[s:e] if lvl is not None else None, mode, policy, coeff[s:e],
                     flags[s:e] if flags is not None else None, stream)
        return coeff.cpu().numpy(), (flags.cpu().numpy() if flags is not None else None)
    chunk = max(1, _CHUNK_VALUES // nv)
    stream = torch.cuda.current_stream(L.dev)
    spans = [(s, min(n, s + chunk)) for s in range(0, n, chunk)]
    workers = max(1, min(_HOST_WORKERS, len(spans)))
    host = _pinned(min(workers + 1, len(spans)), min(chunk, n) * nv)
    dbuf = [torch.empty(min(chunk, n) * nv, dtype=torch.float64, device=L.dev) for _ in range(min(2, len(spans)))]
    done = [None] * len(host)

    def fill(b, s, e):  # host worker: samples + f straight into pinned buffer b
        vals = _sample_values(f, _sample_axes(anchors[s:e], levels[s:e], max_depth, domain_lo, domain_hi, npd), npd)
        np.copyto(host[b][: (e - s) * nv].numpy().reshape(e - s, nv), vals)

    def issue(b, s, e, c):
        db = dbuf[c % len(dbuf)][: (e - s) * nv]
        db.copy_(host[b][: (e - s) * nv], non_blocking=True)
        L.launch(db.view(e - s, nv), lvl[s:e] if lvl is not None else None, mode, policy, coeff[s:e],
                 flags[s:e] if flags is not None else None, stream.cuda_stream)
        done[b] = torch.cuda.Event()
        done[b].record(stream)

    from concurrent.futures import ThreadPoolExecutor

    pending = []
    with ThreadPoolExecutor(workers) as ex:  # numpy ufuncs release the GIL
        for c, (s, e) in enumerate(spans):
            b = c % len(host)
            if done[b] is not None:
                done[b].synchronize()  # the H2D copy out of this pinned buffer has finished
            pending.append((ex.submit(fill, b, s, e), b, s, e, c))
            while len(pending) >= len(host) or (c == len(spans) - 1 and pending):
                fut, pb, ps, pe, pc = pending.pop(0)
                fut.result()
                issue(pb, ps, pe, pc)
    c_host = coeff.cpu().numpy()
    f_host = flags.cpu().numpy() if flags is not None else None
    return c_host, f_host


def wavelet_coefficients(f: Callable, anchors: np.ndarray, levels, max_depth: int, nodes_per_dim: int = 7,
                         domain_lo=None, domain_hi=None, *, device_eval: bool = False) -> np.ndarray:
    """wavelet_coefficient of many octants at once (anchors (n, dim) in
    finest-cell units, levels scalar or (n,)): fp64 array (n,)."""
    _check_npd(nodes_per_dim)
    anchors = np.asarray(anchors, dtype=np.int64)
    if len(anchors) == 0:
        return np.zeros(0)
    anchors = anchors.reshape(len(anchors), -1)
    levels = np.broadcast_to(np.asarray(levels, dtype=np.int32), (len(anchors),))
    lo, hi = _domain(anchors.shape[1], max_depth, domain_lo, domain_hi)
    return _run(f, anchors, levels, max_depth, nodes_per_dim, lo, hi, 0, None, device_eval=device_eval)[0]


def wavelet_coefficient(f: Callable, key: OctKey, nodes_per_dim: int = 7, domain_lo=None,
                        domain_hi=None) -> float:
    """Max interpolation residual of ``f`` on the octant's odd-index nodes
    (wavelet.py:70-105).  ``f`` takes one coordinate array per dimension."""
    _check_npd(nodes_per_dim)
    a = np.asarray([key.anchor], dtype=np.int64)
    return float(wavelet_coefficients(f, a, key.level, key.max_depth, nodes_per_dim, domain_lo, domain_hi)[0])


def refine_flags(f: Callable, tree: LinearOctree, policy: RefinePolicy, nodes_per_dim: int = 7,
                 domain_lo=None, domain_hi=None, *, device_eval: bool = False) -> list[Flag]:
    """Per-leaf refine/keep/coarsen decision (wavelet.py:108-124), one launch
    for the whole tree.  device_eval=True samples on the GPU and calls ``f``
    with CUDA tensors (write ``f`` with torch ops)."""
    codes = refine_codes(f, tree, policy, nodes_per_dim, domain_lo, domain_hi, device_eval=device_eval)
    return [_FLAG_OF_CODE[int(c)] for c in codes]


def refine_codes(f: Callable, tree: LinearOctree, policy: RefinePolicy, nodes_per_dim: int = 7,
                 domain_lo=None, domain_hi=None, *, device_eval: bool = False) -> np.ndarray:
    """refine_flags as an int8 array: 1 refine, 0 keep, -1 coarsen."""
    _check_npd(nodes_per_dim)
    if len(tree) == 0:
        return np.zeros(0, dtype=np.int8)
    anchors, levels = tree.arrays()
    lo, hi = _domain(tree.dim, tree.max_depth, domain_lo, domain_hi)
    return _run(f, anchors.astype(np.int64), levels, tree.max_depth, nodes_per_dim, lo, hi, 0, policy,
                device_eval=device_eval)[1]


class _WaveletPredicate:
    """refinement_predicate (wavelet.py:127-144) with the ``batch`` hook that
    octree.construct uses to test a whole level in one launch."""

    def __init__(self, f, policy, nodes_per_dim, domain_lo, domain_hi, device_eval=False):
        _check_npd(nodes_per_dim)
        self.f, self.policy, self.npd, self.device_eval = f, policy, nodes_per_dim, device_eval
        self.domain_lo, self.domain_hi = domain_lo, domain_hi

    def __call__(self, key: OctKey) -> bool:
        return bool(self.batch(np.asarray([key.anchor], dtype=np.int64), key.level, key.max_depth)[0])

    def batch(self, anchors: np.ndarray, level: int, max_depth: int) -> np.ndarray:
        n = len(anchors)
        p = self.policy
        # the reference evaluates f only for min_level <= level < max_level
        if level < p.min_level:
            return np.ones(n, dtype=bool)
        if level >= p.max_level or n == 0:
            return np.zeros(n, dtype=bool)
        anchors = np.asarray(anchors, dtype=np.int64).reshape(n, -1)
        lo, hi = _domain(anchors.shape[1], max_depth, self.domain_lo, self.domain_hi)
        levels = np.full(n, level, dtype=np.int32)
        return _run(self.f, anchors, levels, max_depth, self.npd, lo, hi, 1, p,
                    device_eval=self.device_eval)[1].astype(bool)


def refinement_predicate(f: Callable, policy: RefinePolicy, nodes_per_dim: int = 7, domain_lo=None,
                         domain_hi=None, *, device_eval: bool = False) -> Callable[[OctKey], bool]:
    """Predicate for top-down construction driven by the coefficient
    (wavelet.py:127-144)."""
    return _WaveletPredicate(f, policy, nodes_per_dim, domain_lo, domain_hi, device_eval)


# ---------------------------------------------------------------------------
# device-resident samples (no host work): the remesh-at-synchronised-times
# use, where the field already lives in HBM

def coefficients_from_values(values, nodes_per_dim: int, dim: int, levels=None, policy: RefinePolicy | None = None,
                             mode: str = "flags"):
    """Coefficients (and, with ``policy``, flags) of device-resident samples.

    values: CUDA fp64 tensor (n, npd^dim) or (n, npd, ..., npd); levels: CUDA
    int32 (n,) when a policy is given.  mode "flags" applies refine_flags'
    rule (int8 1/0/-1), "predicate" the construction predicate (1/0).
    Returns (coeff, flags-or-None) as CUDA tensors, stream-ordered on the
    current stream.
    """
    import torch

    _check_npd(nodes_per_dim)
    if mode not in ("flags", "predicate"):
        raise ValueError("mode must be 'flags' or 'predicate'")
    L = _launcher(dim, nodes_per_dim, values.device)
    nv = nodes_per_dim ** dim
    if values.dtype != torch.float64 or not values.is_cuda or values.numel() % nv:
        raise ValueError("values must be a CUDA float64 tensor of n * nodes_per_dim**dim samples")
    v = values.reshape(-1, nv).contiguous()
    n = v.shape[0]
    coeff = torch.empty(n, dtype=torch.float64, device=v.device)
    flags = None
    if policy is not None:
        if levels is None:
            raise ValueError("flags need per-octant levels")
        levels = levels.to(device=v.device, dtype=torch.int32).contiguous()
        flags = torch.empty(n, dtype=torch.int8, device=v.device)
    L.launch(v, levels if policy is not None else None, 0 if mode == "flags" else 1, policy, coeff, flags,
             torch.cuda.current_stream(v.device).cuda_stream)
    return coeff, flags
