"""Block decomposition, node registry and zip/unzip — drop-in for ``amrlts.mesh``.

The registry and every gather table are built by the native mesh builder
(``amr_mesh_build``, C++).  Two views are exposed:

* the reference's public view — maximal uniform ``blocks`` split at rank cuts,
  per-block scipy CSR ``gathers``, ``zip_positions``, ``leaf_gids``,
  ``node_coords`` (built lazily; API/debug only, mesh.py:153-492);
* the engine's view — one *leaf tile* per leaf (ppo^D nodes + the 2-deep
  stencil cross), as int32 unzip tables plus shared interpolation rows
  (``tile_data``).  Leaf tiles reproduce maximal-block results bit for bit
  because a gather row depends only on the lattice point it samples.

``unzip`` runs on the GPU (``amr_gather_rows``); there is no CPU gather.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from .octree import LinearOctree, OctKey
from .partition import ExchangePlan, PartitionMap, build_exchange_plan

C = _native.C


@dataclass(frozen=True)
class Domain:
    lo: tuple[float, ...]
    hi: tuple[float, ...]

    def extent(self, d: int) -> float:
        return self.hi[d] - self.lo[d]


@dataclass(frozen=True)
class Block:
    """Uniform patch: a root octant whose descendant leaves share ``leaf_level`` (mesh.py:48-84)."""

    index: int
    root: OctKey
    leaf_level: int
    leaf_range: tuple[int, int]
    points_per_octant: int
    pad: int
    owner_rank: int

    @property
    def dim(self) -> int:
        return self.root.dim

    @property
    def interior_n(self) -> int:
        return (self.points_per_octant - 1) * (1 << (self.leaf_level - self.root.level)) + 1

    @property
    def interior_points(self) -> int:
        return self.interior_n ** self.dim

    @property
    def padded_n(self) -> int:
        return self.interior_n + 2 * self.pad

    @property
    def padded_shape(self) -> tuple[int, ...]:
        return (self.padded_n,) * self.dim

    @property
    def interior_slices(self) -> tuple[slice, ...]:
        return (slice(self.pad, self.pad + self.interior_n),) * self.dim


def decompose_blocks(tree: LinearOctree, points_per_octant: int = 7, pad: int = 2,
                     pmap: PartitionMap | None = None) -> list[Block]:
    """Maximal uniform blocks split at rank cuts (mesh.py:87-135), native recursion."""
    owners = pmap.owners(len(tree)) if pmap is not None else np.zeros(len(tree), dtype=int)
    return _blocks_from_native(_NativeMesh(tree, points_per_octant, 2, owners, registry=False), tree,
                               points_per_octant, pad)


class _NotMortonOrder(ValueError):
    """The leaf order is another curve's: the device builder (leaf index = key position) does not apply."""


def device_tables(tree: LinearOctree, ppo: int, pad: int, device) -> dict:
    """Node registry, leaf-tile table and interpolation rows of a Morton-ordered
    balanced tree, built on the device (csrc/amr_devmesh.cu; the passes of
    mesh.py:214-398).  Returns device tensors: ``starts`` (leaf_slices),
    ``leaf_gids`` [n, ppo^dim], ``table`` [n, E], the sorted lattice ``codes`` of
    the hanging points and their rows as CSR (``row_ptr``, ``gid``, ``w``).
    Prefix sums and the sort/unique of the codes are torch's (cub)."""
    import torch

    L = _native.lib()
    dim, depth = tree.dim, tree.max_depth
    an, lv = tree.arrays()
    n = len(lv)
    P = ppo ** dim
    E = int(L.amr_tile_entries(dim, ppo))
    with torch.cuda.device(device):
        st = torch.cuda.current_stream(device).cuda_stream
        a_d = torch.from_numpy(np.ascontiguousarray(an, dtype=np.int32)).to(device)
        l_d = torch.from_numpy(np.ascontiguousarray(lv, dtype=np.int32)).to(device)
        keys = torch.empty(n, dtype=torch.int64, device=device)
        _native.check(L.amr_oct_keys(dim, depth, n, a_d.data_ptr(), l_d.data_ptr(), keys.data_ptr(), st), "amr_oct_keys")
        if n > 1 and not bool(torch.all(keys[1:] > keys[:-1])):
            raise _NotMortonOrder("leaves are not in Morton order")
        geo = (dim, depth, ppo, pad, n, keys.data_ptr(), a_d.data_ptr(), l_d.data_ptr())
        err = torch.zeros(1, dtype=torch.int32, device=device)
        status = torch.empty((n, P), dtype=torch.int8, device=device)
        owner = torch.empty((n, P), dtype=torch.int32, device=device)
        counts = torch.empty(n, dtype=torch.int64, device=device)
        _native.check(L.amr_dm_ownership(*geo, status.data_ptr(), owner.data_ptr(), counts.data_ptr(),
                                         err.data_ptr(), st), "amr_dm_ownership")
        if int(err[0]):
            raise ValueError("leaf point outside every leaf: tree is not complete")
        starts = torch.zeros(n + 1, dtype=torch.int64, device=device)
        torch.cumsum(counts, 0, out=starts[1:])
        if int(starts[-1]) >= 2 ** 31:
            raise ValueError("more than 2^31 zip nodes: int32 gids overflow")
        leaf_gids = torch.empty((n, P), dtype=torch.int32, device=device)
        _native.check(L.amr_dm_gids(*geo, status.data_ptr(), owner.data_ptr(), starts.data_ptr(),
                                    leaf_gids.data_ptr(), st), "amr_dm_gids")
        del status, owner
        table = torch.empty((n, E), dtype=torch.int32, device=device)
        n_hang = torch.empty(n, dtype=torch.int32, device=device)
        _native.check(L.amr_dm_table(*geo, leaf_gids.data_ptr(), table.data_ptr(), n_hang.data_ptr(), st),
                      "amr_dm_table")
        hang_end = torch.cumsum(n_hang.to(torch.int64), 0)
        total_h = int(hang_end[-1]) if n else 0
        hang_off = hang_end - n_hang
        pos = torch.empty(max(total_h, 1), dtype=torch.int64, device=device)
        code = torch.empty(max(total_h, 1), dtype=torch.int64, device=device)
        _native.check(L.amr_dm_hang_list(*geo, table.data_ptr(), hang_off.data_ptr(), pos.data_ptr(),
                                         code.data_ptr(), st), "amr_dm_hang_list")
        codes = torch.unique(code[:total_h])  # sorted
        nr = codes.numel()
        _native.check(L.amr_dm_table_rows(total_h, pos.data_ptr(), code.data_ptr(), nr, codes.data_ptr(),
                                          table.data_ptr(), st), "amr_dm_table_rows")
        del pos, code
        cnt = torch.empty(max(nr, 1), dtype=torch.int32, device=device)
        _native.check(L.amr_dm_rows(*geo, leaf_gids.data_ptr(), nr, codes.data_ptr(), None, cnt.data_ptr(), None, None,
                                    err.data_ptr(), st), "amr_dm_rows")
        row_ptr = torch.zeros(nr + 1, dtype=torch.int64, device=device)
        if nr:
            torch.cumsum(cnt[:nr].to(torch.int64), 0, out=row_ptr[1:])
        nnz = int(row_ptr[-1])
        gid = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
        w = torch.empty(max(nnz, 1), dtype=torch.float64, device=device)
        _native.check(L.amr_dm_rows(*geo, leaf_gids.data_ptr(), nr, codes.data_ptr(), row_ptr.data_ptr(), cnt.data_ptr(),
                                    gid.data_ptr(), w.data_ptr(), err.data_ptr(), st), "amr_dm_rows")
        e = int(err[0])
        if e:
            raise ValueError("device mesh builder: " + ("lattice point outside the domain during interpolation"
                                                        if e & 1 else "interpolation row exceeds the builder's limits"))
    return dict(starts=starts, leaf_gids=leaf_gids, table=table, codes=codes, row_ptr=row_ptr, gid=gid[:nnz], w=w[:nnz],
                anchors=a_d, levels=l_d)


class _NativeMesh:
    """Owning handle around AmrMesh*: built by the host passes (amr_mesh_build),
    or around tables built on the device (``device=...``, Morton order)."""

    def __init__(self, tree: LinearOctree, ppo: int, pad: int, owners, registry: bool = True, device=None):
        anchors, levels = tree.arrays()
        self.lib = _native.lib()
        own = np.ascontiguousarray(owners, dtype=np.int32)
        self.on_device = device is not None
        self.tables = None  # device tensors of the tables when they were built there
        self._full = True
        if device is not None:
            try:
                self.tables = device_tables(tree, ppo, pad, device)
            except _NotMortonOrder:  # leaves along another curve: the host passes index them themselves
                device = None
                self.on_device = False
        if device is not None:
            # a light handle (blocks, leaf slices); host copies of the big tables only when an
            # API view asks for them (full()) — the engine works on the device tensors
            self._args = (tree.dim, tree.max_depth, ppo, pad, len(levels), anchors, levels, own)
            self._full = False
            self.h = self._from_tables(full=False)
        else:
            self.h = self.lib.amr_mesh_build(tree.dim, tree.max_depth, ppo, pad, len(levels),
                                             _native.ptr(anchors, C.c_int32), _native.ptr(levels, C.c_int32),
                                             _native.ptr(own, C.c_int32), 0)
        if not self.h:
            raise ValueError(_native.last_error())

    def _from_tables(self, full: bool):
        dim, depth, ppo, pad, n, anchors, levels, own = self._args
        p32, p64 = (lambda a: _native.ptr(a, C.c_int32)), (lambda a: _native.ptr(a, C.c_int64))
        t = self.tables
        starts = np.ascontiguousarray(t["starts"].cpu().numpy())
        if not full:
            return self.lib.amr_mesh_from_tables(dim, depth, ppo, pad, n, p32(anchors), p32(levels), p32(own),
                                                 p64(starts), None, None, 0, None, None, None, None)
        h = {k: np.ascontiguousarray(t[k].cpu().numpy()) for k in ("leaf_gids", "table", "codes", "row_ptr", "gid", "w")}
        return self.lib.amr_mesh_from_tables(
            dim, depth, ppo, pad, n, p32(anchors), p32(levels), p32(own), p64(starts), p32(h["leaf_gids"]),
            p32(h["table"]), len(h["codes"]), p64(h["codes"]), p64(h["row_ptr"]),
            p32(h["gid"] if len(h["gid"]) else np.zeros(1, np.int32)),
            _native.ptr(h["w"] if len(h["w"]) else np.zeros(1), C.c_double))

    def full(self):
        """The handle with host copies of every table (API views, the host program builder)."""
        if not self._full:
            h = self._from_tables(full=True)
            if not h:
                raise ValueError(_native.last_error())
            old, self.h = self.h, h
            self.lib.amr_mesh_free(old)
            self._full = True
        return self.h

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            self.lib.amr_mesh_free(h)


def _blocks_from_native(nm: _NativeMesh, tree, ppo, pad) -> list[Block]:
    L = nm.lib
    nb = L.amr_mesh_n_blocks(nm.h)
    dim = tree.dim
    ra = np.empty((nb, dim), dtype=np.int32)
    rl = np.empty(nb, dtype=np.int32)
    ll = np.empty(nb, dtype=np.int32)
    lr = np.empty((nb, 2), dtype=np.int64)
    ow = np.empty(nb, dtype=np.int32)
    _native.check(L.amr_mesh_blocks(nm.h, _native.ptr(ra, C.c_int32), _native.ptr(rl, C.c_int32),
                                    _native.ptr(ll, C.c_int32), _native.ptr(lr, C.c_int64),
                                    _native.ptr(ow, C.c_int32)), "amr_mesh_blocks")
    return [Block(index=i, root=OctKey(tuple(int(x) for x in ra[i]), int(rl[i]), tree.max_depth),
                  leaf_level=int(ll[i]), leaf_range=(int(lr[i, 0]), int(lr[i, 1])),
                  points_per_octant=ppo, pad=pad, owner_rank=int(ow[i]))
            for i in range(nb)]


class Mesh:
    """Node registry, gather/scatter plans and synchronization maps (mesh.py:153-492)."""

    def __init__(self, tree: LinearOctree, points_per_octant: int = 7, pad: int = 2,
                 pmap: PartitionMap | None = None, domain: Domain | None = None):
        if not tree.balanced:
            raise ValueError("mesh construction requires a 2:1 balanced tree")
        if points_per_octant < 5 or points_per_octant % 2 == 0:
            raise ValueError("points_per_octant must be odd and >= 5")
        if pad < 1 or pad > points_per_octant - 1:
            raise ValueError("pad must be in [1, points_per_octant - 1]")
        if pad != 2:
            raise ValueError("the B200 engine implements the reference's 5-point stencil reach: pad must be 2")
        self.tree = tree
        self.dim = tree.dim
        self.L = tree.max_depth
        self.ppo = points_per_octant
        self.pad = pad
        self.scale = points_per_octant - 1
        self.top_nodes = self.scale << self.L
        if (self.top_nodes + 1) ** self.dim >= 2**62:
            raise ValueError("max_depth too large for the node lattice encoding")
        if domain is None:
            domain = Domain((0.0,) * self.dim, (float(1 << self.L),) * self.dim)
        self.domain = domain
        if pmap is None:
            w = np.ones(len(tree))
            pmap = PartitionMap([(0, len(tree))], w, np.array([float(len(tree))]))
        self.pmap = pmap
        owners = pmap.owners(len(tree))
        # registry, tile tables and interpolation rows: on the device when there is one
        # (Morton order), else the host passes; both give the same tables
        # (tests/test_devmesh_gpu.py).  AMR_HOST_MESH=1 forces the host builder.
        import os

        from .octree import _device

        dev = None if os.environ.get("AMR_HOST_MESH") == "1" else _device()
        if dev is not None and (tree.ordering.kind != "morton" or tree.dim * tree.max_depth > 57):
            dev = None
        self._nm = _NativeMesh(tree, points_per_octant, pad, owners, device=dev)
        L = self._nm.lib
        self.blocks = _blocks_from_native(self._nm, tree, points_per_octant, pad)
        n_leaves = len(tree)
        self.leaf_block = np.empty(n_leaves, dtype=int)
        for b in self.blocks:
            self.leaf_block[b.leaf_range[0]: b.leaf_range[1]] = b.index
        self.n_nodes = int(L.amr_mesh_n_nodes(self._nm.h))
        starts = np.empty(n_leaves + 1, dtype=np.int64)
        _native.check(L.amr_mesh_leaf_starts(self._nm.h, _native.ptr(starts, C.c_int64)), "leaf_starts")
        self.leaf_starts = starts
        self.leaf_slices = np.stack([starts[:-1], starts[1:]], axis=1)
        self._leaf_gids = None
        self._node_coords = None
        self._zip_positions = None
        self._gathers = None
        self._block_read = None
        self._tile = None
        self._plan: ExchangePlan | None = None
        self._unzip_dev = None

    # -- registry views --------------------------------------------------------
    @property
    def leaf_gids(self) -> np.ndarray:
        if self._leaf_gids is None:
            g = np.empty((len(self.tree), self.ppo ** self.dim), dtype=np.int32)
            _native.check(self._nm.lib.amr_mesh_leaf_gids(self._nm.full(), _native.ptr(g, C.c_int32)), "leaf_gids")
            self._leaf_gids = g.astype(np.int64)
        return self._leaf_gids

    @property
    def node_coords(self) -> np.ndarray:
        if self._node_coords is None:
            c = np.empty((self.n_nodes, self.dim), dtype=np.int32)
            _native.check(self._nm.lib.amr_mesh_node_coords(self._nm.full(), _native.ptr(c, C.c_int32)), "node_coords")
            self._node_coords = c.astype(np.int64)
        return self._node_coords

    def leaf_spacing(self, level: int) -> int:
        return 1 << (self.L - level)

    def _leaf_points(self, key: OctKey) -> np.ndarray:
        s = self.leaf_spacing(key.level)
        axes = [a * self.scale + s * np.arange(self.ppo) for a in key.anchor]
        grid = np.meshgrid(*axes, indexing="ij")
        return np.stack([g.ravel() for g in grid], axis=-1).astype(np.int64)

    def _block_org(self, b: Block) -> np.ndarray:
        s = self.leaf_spacing(b.leaf_level)
        return np.array(b.root.anchor, dtype=np.int64) * self.scale - b.pad * s

    @property
    def zip_positions(self) -> list[np.ndarray]:
        """Per leaf: flat padded-block positions of its owned nodes (mesh.py:270-277)."""
        if self._zip_positions is None:
            gids = self.leaf_gids
            out = []
            for i, key in enumerate(self.tree.leaves):
                a, e = self.leaf_slices[i]
                owned = (gids[i] >= a) & (gids[i] < e)
                pts = self._leaf_points(key)[owned]
                b = self.blocks[self.leaf_block[i]]
                rel = (pts - self._block_org(b)) // self.leaf_spacing(b.leaf_level)
                out.append(np.ravel_multi_index(rel.T, b.padded_shape).astype(np.int64))
            self._zip_positions = out
        return self._zip_positions

    def lookup_gids(self, codes: np.ndarray) -> np.ndarray:
        m = self.top_nodes + 1
        coords = self.node_coords
        all_codes = coords[:, 0].copy()
        for d in range(1, self.dim):
            all_codes = all_codes * m + coords[:, d]
        order = np.argsort(all_codes, kind="stable")
        sc = all_codes[order]
        codes = np.asarray(codes, dtype=np.int64)
        pos = np.clip(np.searchsorted(sc, codes), 0, max(len(sc) - 1, 0))
        hit = sc[pos] == codes if len(sc) else np.zeros(codes.shape, dtype=bool)
        return np.where(hit, order[pos], -1)

    # -- gathers ------------------------------------------------------------------
    def _block_csr(self, b: int):
        L = self._nm.lib
        self._nm.full()
        rows, nnz = C.c_int64(0), C.c_int64(0)
        _native.check(L.amr_mesh_block_gather(self._nm.h, b, C.byref(rows), C.byref(nnz), None, None, None),
                      "block_gather")
        ptr = np.empty(rows.value + 1, dtype=np.int64)
        col = np.empty(nnz.value, dtype=np.int64)
        val = np.empty(nnz.value, dtype=np.float64)
        _native.check(L.amr_mesh_block_gather(self._nm.h, b, C.byref(rows), C.byref(nnz),
                                              _native.ptr(ptr, C.c_int64), _native.ptr(col, C.c_int64),
                                              _native.ptr(val, C.c_double)), "block_gather")
        return ptr, col, val

    @property
    def gathers(self):
        """Per-block scipy CSR (padded points x n_nodes), rows sorted by gid."""
        if self._gathers is None:
            import scipy.sparse as sp

            out = []
            for b in self.blocks:
                ptr, col, val = self._block_csr(b.index)
                out.append(sp.csr_matrix((val, col, ptr), shape=(len(ptr) - 1, self.n_nodes)))
            self._gathers = out
        return self._gathers

    def _read_sets(self):
        if self._block_read is None:
            starts = self.leaf_slices[:, 0]
            reads = []
            for b in self.blocks:
                _, col, _ = self._block_csr(b.index)
                support = np.unique(col)
                reads.append(np.unique(np.searchsorted(starts, support, side="right") - 1))
            self._block_read = reads
        return self._block_read

    def leaf_node_slice(self, leaf: int) -> tuple[int, int]:
        a, b = self.leaf_slices[leaf]
        return int(a), int(b)

    def block_read_leaves(self, block_index: int) -> np.ndarray:
        return self._read_sets()[block_index]

    def zeros_zip(self, nvars: int = 1) -> np.ndarray:
        return np.zeros((nvars, self.n_nodes))

    def unzip(self, zip_values: np.ndarray) -> list[np.ndarray]:
        """Padded per-block arrays gathered from the zipped field, on the GPU."""
        import torch

        z = np.atleast_2d(np.asarray(zip_values, dtype=np.float64))
        nv = z.shape[0]
        dev = torch.device("cuda")
        if self._unzip_dev is None:
            ptrs, cols, vals, offs = [np.zeros(1, dtype=np.int64)], [], [], [0]
            base = 0
            for b in self.blocks:
                ptr, col, val = self._block_csr(b.index)
                ptrs.append(ptr[1:] + base)
                base += len(col)
                cols.append(col)
                vals.append(val)
                offs.append(offs[-1] + len(ptr) - 1)
            self._unzip_dev = (
                torch.from_numpy(np.concatenate(ptrs)).to(dev),
                torch.from_numpy(np.concatenate(cols) if cols else np.zeros(0, np.int64)).to(dev),
                torch.from_numpy(np.concatenate(vals) if vals else np.zeros(0)).to(dev),
                offs,
            )
        ptr_d, col_d, val_d, offs = self._unzip_dev
        zd = torch.from_numpy(np.ascontiguousarray(z)).to(dev)
        n_rows = offs[-1]
        out = torch.empty((nv, n_rows), dtype=torch.float64, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _native.check(self._nm.lib.amr_gather_rows(n_rows, ptr_d.data_ptr(), col_d.data_ptr(), val_d.data_ptr(),
                                                   nv, zd.data_ptr(), self.n_nodes, out.data_ptr(), n_rows,
                                                   stream), "amr_gather_rows")
        host = out.cpu().numpy()
        return [np.ascontiguousarray(host[:, offs[i]:offs[i + 1]].reshape(nv, *b.padded_shape))
                for i, b in enumerate(self.blocks)]

    def zip(self, block_arrays: Sequence[np.ndarray]) -> np.ndarray:
        """Zipped field from block interiors, owners win (mesh.py:422-432)."""
        nvars = block_arrays[0].shape[0]
        out = np.empty((nvars, self.n_nodes))
        zp = self.zip_positions
        for i in range(len(self.tree)):
            a, b = self.leaf_slices[i]
            if b == a:
                continue
            arr = block_arrays[self.leaf_block[i]].reshape(nvars, -1)
            out[:, a:b] = arr[:, zp[i]]
        return out

    def leaf_lattice_device(self, zd, var: int = 0):
        """(n_leaves, ppo^dim) CUDA tensor: every leaf's own ppo^dim lattice
        nodes (ij order, last axis fastest) from a (nvars, n_nodes) CUDA zip
        field.  Shared/owned nodes are copies, hanging nodes are the
        reference's interpolation rows (0 + sum w*z in ascending-gid order,
        mesh.py:355-398, amr_gather_rows), i.e. the interior of Mesh.unzip
        restricted to the leaf.  Feeds the wavelet criterion on the solution
        (wavelet.coefficients_from_values with nodes_per_dim = ppo)."""
        import torch

        dev = zd.device
        lt = self.__dict__.get("_lattice_dev")
        if lt is None or lt[0].device != dev:
            td = self.tile_data()
            NI = self.ppo ** self.dim
            tab = td["table"][:, :NI].astype(np.int64)
            hang = tab <= -2
            rows = (-tab[hang] - 2)
            iptr = td["interp_ptr"]
            ptr = np.zeros(len(rows) + 1, dtype=np.int64)
            np.cumsum(iptr[rows + 1] - iptr[rows], out=ptr[1:])
            lens = iptr[rows + 1] - iptr[rows]
            take = np.repeat(iptr[rows] - ptr[:-1], lens) + np.arange(int(ptr[-1]), dtype=np.int64)
            col = td["interp_gid"][take].astype(np.int64)
            w = td["interp_w"][take]
            hidx = np.flatnonzero(hang.reshape(-1)).astype(np.int64)  # integer index: no mask->nonzero sync
            lt = (torch.from_numpy(np.where(hang, 0, tab)).to(dev), torch.from_numpy(hidx).to(dev),
                  torch.from_numpy(ptr).to(dev), torch.from_numpy(col).to(dev), torch.from_numpy(w).to(dev),
                  len(rows))
            self.__dict__["_lattice_dev"] = lt
        tab_d, hidx_d, ptr_d, col_d, w_d, nh = lt
        row = zd[var].contiguous()
        out = row[tab_d]
        if nh:
            hv = torch.empty(nh, dtype=torch.float64, device=dev)
            stream = torch.cuda.current_stream(dev).cuda_stream
            _native.check(self._nm.lib.amr_gather_rows(nh, ptr_d.data_ptr(), col_d.data_ptr(), w_d.data_ptr(), 1,
                                                       row.data_ptr(), row.numel(), hv.data_ptr(), nh, stream),
                          "amr_gather_rows")
            out.view(-1).index_copy_(0, hidx_d, hv)
        return out

    # -- engine view ---------------------------------------------------------------
    def device_tables(self):
        """The registry and tile tables as device tensors (built there, or
        uploaded from the host builder's arrays), for the device program builder."""
        if self._nm.tables is None:
            import torch

            dev = torch.device("cuda", torch.cuda.current_device())
            td = self.tile_data()
            an, lv = self.tree.arrays()
            T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
            nnz = int(td["interp_ptr"][-1])
            self._nm.tables = dict(starts=T(self.leaf_starts), table=T(td["table"]), row_ptr=T(td["interp_ptr"]),
                                   gid=T(td["interp_gid"][:max(nnz, 1)]), w=T(td["interp_w"][:max(nnz, 1)]),
                                   anchors=T(an.astype(np.int32)), levels=T(lv.astype(np.int32)))
        return self._nm.tables

    def tile_data(self) -> dict:
        """Leaf-tile unzip tables for the stage kernel (see include/amr_b200.h)."""
        if self._tile is None:
            L = self._nm.lib
            self._nm.full()
            n = len(self.tree)
            E = int(L.amr_tile_entries(self.dim, self.ppo))
            table = np.empty((n, E), dtype=np.int32)
            _native.check(L.amr_mesh_tile_table(self._nm.h, _native.ptr(table, C.c_int32)), "tile_table")
            nr = int(L.amr_mesh_interp_rows(self._nm.h))
            nz = int(L.amr_mesh_interp_nnz(self._nm.h))
            iptr = np.empty(nr + 1, dtype=np.int64)
            igid = np.empty(max(nz, 1), dtype=np.int32)
            iw = np.empty(max(nz, 1), dtype=np.float64)
            _native.check(L.amr_mesh_interp_csr(self._nm.h, _native.ptr(iptr, C.c_int64),
                                                _native.ptr(igid, C.c_int32), _native.ptr(iw, C.c_double)),
                          "interp_csr")
            anchors, levels = self.tree.arrays()
            a3 = np.zeros((n, 3), dtype=np.int32)
            a3[:, : self.dim] = anchors
            self._tile = dict(table=table, entries=E, interp_ptr=iptr, interp_gid=igid, interp_w=iw,
                              anchor3=a3, level=levels.astype(np.int32), starts=self.leaf_starts,
                              dim=self.dim, ppo=self.ppo, max_depth=self.L)
        return self._tile

    # -- sync maps -------------------------------------------------------------------
    def exchange_plan(self) -> ExchangePlan:
        if self._plan is None:
            self._plan = build_exchange_plan(self, self.pmap)
        return self._plan

    def level_blocks(self, min_level: int) -> set[int]:
        return {b.index for b in self.blocks if b.leaf_level >= min_level}

    def build_sync_maps(self) -> tuple[ExchangePlan, list[ExchangePlan]]:
        full = self.exchange_plan()
        l_max = max(b.leaf_level for b in self.blocks)
        l_min = min(b.leaf_level for b in self.blocks)
        return full, [full.restrict(self.level_blocks(l_max - k)) for k in range(l_max - l_min + 1)]

    # -- physical coordinates ----------------------------------------------------------
    def node_physical(self) -> np.ndarray:
        out = np.empty((self.n_nodes, self.dim))
        nc = self.node_coords
        for d in range(self.dim):
            out[:, d] = self.domain.lo[d] + (nc[:, d] / self.top_nodes) * self.domain.extent(d)
        return out

    def node_physical_device(self):
        """node_physical as per-axis float64 CUDA tensors, from the device
        registry (each leaf's owned lattice points scattered to their gids):
        the same ``lo + (coord / top_nodes) * extent`` operations, no host pass
        over the nodes (cfg5: 6e8 nodes)."""
        import torch

        t = self.device_tables()
        if "leaf_gids" not in t:
            dev = t["table"].device
            t["leaf_gids"] = torch.from_numpy(self.leaf_gids.astype(np.int32)).to(dev)
        lg, st = t["leaf_gids"], t["starts"]
        dev = lg.device
        n, P = lg.shape
        coords = [torch.empty(self.n_nodes, dtype=torch.float64, device=dev) for _ in range(self.dim)]
        kk = torch.arange(P, device=dev)
        locs = [((kk // self.ppo ** (self.dim - 1 - d)) % self.ppo)[None, :] for d in range(self.dim)]
        chunk = 1 << 15  # leaves per pass: temporaries stay small next to an engine's state
        for a in range(0, n, chunk):
            b = min(n, a + chunk)
            g = lg[a:b]
            own = (g >= st[a:b, None]) & (g < st[a + 1:b + 1, None])
            idx = g[own].to(torch.int64)
            s = (torch.ones((), dtype=torch.int64, device=dev) << (self.L - t["levels"][a:b].to(torch.int64)))[:, None]
            for d in range(self.dim):
                c = t["anchors"][a:b, d].to(torch.int64)[:, None] * self.scale + s * locs[d]
                coords[d][idx] = c[own].to(torch.float64)
        out = []
        top = torch.full((), float(self.top_nodes), dtype=torch.float64, device=dev)
        for d in range(self.dim):
            ext = torch.full((), self.domain.extent(d), dtype=torch.float64, device=dev)
            x = coords[d]
            x.div_(top).mul_(ext).add_(self.domain.lo[d])  # lo + (coord / top) * extent, in place
            out.append(x)
        return out

    def block_axes(self, block: Block) -> list[np.ndarray]:
        s = self.leaf_spacing(block.leaf_level)
        org = self._block_org(block)
        return [self.domain.lo[d] + ((org[d] + s * np.arange(block.padded_n)) / self.top_nodes) * self.domain.extent(d)
                for d in range(self.dim)]

    def level_spacing(self, level: int) -> float:
        return self.domain.extent(0) * self.leaf_spacing(level) / self.top_nodes

    def block_spacing(self, block: Block) -> float:
        return self.level_spacing(block.leaf_level)

    def finest_spacing(self) -> float:
        return min(self.block_spacing(b) for b in self.blocks)

    def block_domain_faces(self, block: Block) -> list[tuple[int, int]]:
        out = []
        side = block.root.side
        for d in range(self.dim):
            if block.root.anchor[d] == 0:
                out.append((d, 0))
            if block.root.anchor[d] + side == (1 << self.L):
                out.append((d, 1))
        return out


def write_block_vtk(mesh: Mesh, block: Block, values: np.ndarray, name: str = "field") -> str:
    """Legacy-VTK ASCII rectilinear grid of one block's interior (mesh.py:500-525)."""
    axes = mesh.block_axes(block)
    g, n = block.pad, block.interior_n
    inner = [ax[g: g + n] for ax in axes]
    if mesh.dim == 2:
        inner.append(np.zeros(1))
    dims = [len(a) for a in inner]
    lines = ["# vtk DataFile Version 2.0", f"block {block.index}", "ASCII", "DATASET RECTILINEAR_GRID",
             f"DIMENSIONS {dims[0]} {dims[1]} {dims[2]}"]
    for label, ax in zip(("X", "Y", "Z"), inner):
        lines.append(f"{label}_COORDINATES {len(ax)} double")
        lines.append(" ".join(f"{v:.17g}" for v in ax))
    interior = values[block.interior_slices]
    lines += [f"POINT_DATA {interior.size}", f"SCALARS {name} double", "LOOKUP_TABLE default"]
    lines.extend(f"{v:.17g}" for v in interior.transpose(*range(mesh.dim - 1, -1, -1)).ravel())
    return "\n".join(lines) + "\n"


def field_csv_rows(mesh: Mesh, block_arrays: Sequence[np.ndarray], var: int = 0):
    """Rows ``block_id,i,j[,k],value`` over block interiors (mesh.py:528-533)."""
    for b in mesh.blocks:
        interior = block_arrays[b.index][var][b.interior_slices]
        for idx in np.ndindex(*interior.shape):
            yield (b.index, *idx, interior[idx])
