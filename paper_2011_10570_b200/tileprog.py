"""Per-tile stage programs of the stage kernel (``amr_stage``, csrc/amr_stage_cross.cuh).

One leaf = one tile.  A tile computes the RHS only at the zip nodes it owns
(its contiguous gid range ``leaf_slices[leaf]``), so it needs the stage input
only on the **owned cross**: the owned nodes and the cells within two steps of
one of them along a single axis (the 4th-order stencil's reach; the biased
rows at physical faces stay inside the leaf).  Everything else of the
reference's padded block is never read.  On cfg2 that is
1 257 of the 1 701 stencil-cross cells of a tile and 70 of its 144 hanging
rows.

The program of a tile is two byte strings:

* the **head** (fixed stride ``max_head`` bytes, so the kernel bulk-copies it
  into shared memory with one ``cp.async.bulk`` and no offset lookup):

  ========  ==============================================================
  header    16 int32: g0, n_own, level | cadence<<8 | faces<<16, n_runs,
            n_slots, n_rows, n_bases, tail bytes, anchor[3], run counts of the
            8/4/2/1-lane buckets (two uint16 per word, words 11-12), tail
            offset (16-byte units, word 14), taps offset inside the tail
            (uint16 units, word 15)
  bases     int32 per source group: a source leaf's first gid (>= 0), or,
            for LTS interface pairs, -(first pair of the (reader cadence,
            source leaf) group) - 1
  runs      uint32 per copy run: box cell | (length-1) << 12 | code << 16,
            code = base index << 10 | offset of the first source node.  A run
            is z-consecutive box cells fed by consecutive nodes of one source
            group, at most 8 long.  Runs are bucketed by length (5-8, 3-4, 2,
            1 -> 8, 4, 2, 1 lanes per run) so a warp copies 32 nodes per
            instruction with lanes walking along runs (coalesced, balanced)
  slots     uint16 per unique interpolation source node, same code
  ========  ==============================================================

* the **tail** (read through L2, bulk-prefetched at tile start): hanging rows
  (uint32: box cell | n_quads << 12 | quad offset << 17), longest first, and
  their taps (uint16: slot << 6 | weight id), each row padded to a multiple of
  4 taps with (zero slot, weight 0), which leaves the ascending-gid running
  sum of ``_point_weights`` (mesh.py:316-351) unchanged.

Unzip semantics (``Mesh.unzip``, mesh.py:413-420): a copy cell is a zip node,
a hanging cell is an interpolation row ``0 + sum w_k src(g_k)`` in ascending
gid order, and a cell outside the domain is never read by the owned stencils.
At LTS level interfaces a source node whose cadence differs from the reader's
is an **interface pair** (node, reader cadence): its stage source (transfer
matrices, virtual substeps; ``Engine._stage_source``, stepper.py:274-314) is
formed once per stage by ``iface_kernel`` and read like a copy.

All numpy, vectorised over tiles; built once per mesh (Engine construction).
"""
from __future__ import annotations

import os

import numpy as np

HDR_WORDS = 16        # int32 words in the header
MAX_BASES = 63        # source groups per tile (6-bit base index)
RUN_MAX = 8           # longest run
ROW_STRIDE = 13       # box row stride in doubles (amr_common.cuh Tile::RS; AMR_RS overrides both, for experiments)
BUCKET_LANES = (8, 4, 2, 1)


class ProgramError(ValueError):
    """The mesh does not fit the compact per-tile encoding."""


def _r16(nbytes):
    return (np.asarray(nbytes, dtype=np.int64) + 15) // 16 * 16


def cross_cells(dim: int, ppo: int, pad: int = 2) -> np.ndarray:
    """Padded-box cell of every stencil-cross entry, in the enumeration of the
    mesh's tile table (amr_mesh.cpp cross_entry_local): the ppo^dim interior
    in C order, then per axis the 2*pad layers below and above."""
    NI, NF = ppo ** dim, ppo ** (dim - 1)
    E = NI + dim * 2 * pad * NF
    e = np.arange(E, dtype=np.int64)
    loc = np.zeros((E, dim), dtype=np.int64)
    inner = e < NI
    r = e[inner].copy()
    for d in range(dim - 1, -1, -1):
        loc[inner, d] = pad + r % ppo
        r //= ppo
    h = ~inner
    r = e[h] - NI
    axis = r // (2 * pad * NF)
    r = r % (2 * pad * NF)
    layer = r // NF
    within = r % NF
    sub = np.zeros((len(r), dim), dtype=np.int64)
    for d in range(dim - 1, -1, -1):
        others = axis != d
        sub[others, d] = pad + within[others] % ppo
        within = np.where(others, within // ppo, within)
    sub[np.arange(len(r)), axis] = np.where(layer < pad, layer, ppo + layer)
    loc[h] = sub
    strides = box_strides(dim, ppo)
    cell = np.zeros(E, dtype=np.int64)
    for d in range(dim):
        cell += loc[:, d] * strides[d]
    return cell


def box_strides(dim: int, ppo: int, pad: int = 2) -> tuple:
    """Strides of the shared-memory stencil box (the kernel's Tile::RS):
    rows of the last axis padded to ROW_STRIDE doubles."""
    NP = ppo + 2 * pad
    rs = max(int(os.environ.get("AMR_RS", ROW_STRIDE)), NP)
    return (NP * rs, rs, 1) if dim == 3 else (rs, 1)


def box_cells(dim: int, ppo: int, pad: int = 2) -> int:
    return (ppo + 2 * pad) ** (dim - 2) * box_strides(dim, ppo, pad)[-2] * (ppo + 2 * pad)


def owned_cross(table: np.ndarray, g0: np.ndarray, g1: np.ndarray, faces: np.ndarray, dim: int,
                ppo: int) -> np.ndarray:
    """(n_tiles, E) mask of the cross entries the owned stencils read: the
    centred rows' +-1, +-2 along each axis, and at a physical face the biased
    rows' 6-point windows (wave.py:57-109; first-derivative rows read a subset)."""
    cells = cross_cells(dim, ppo)
    NI = ppo ** dim
    bs = box_strides(dim, ppo)
    cell2e = np.full(box_cells(dim, ppo), -1, dtype=np.int64)
    cell2e[cells] = np.arange(len(cells))
    core = table[:, :NI]
    own = (core >= g0[:, None]) & (core < g1[:, None])
    need = np.zeros(table.shape, dtype=bool)
    need[:, :NI] = own
    k = np.arange(NI)
    for d in range(dim):
        stride = bs[d]
        pos = (k // ppo ** (dim - 1 - d)) % ppo
        for o in (-2, -1, 1, 2):
            tgt = cell2e[cells[:NI] + o * stride]
            need[:, tgt] |= own
        lo = ((faces >> (2 * d)) & 1).astype(bool)
        hi = ((faces >> (2 * d + 1)) & 1).astype(bool)
        for o in range(-5, 6):
            inside = (pos + o >= 0) & (pos + o < ppo)
            at_lo = inside & (pos <= 1)
            at_hi = inside & (pos >= ppo - 2)
            for sel, fl in ((at_lo, lo), (at_hi, hi)):
                if not sel.any() or not fl.any():
                    continue
                src = np.nonzero(sel)[0]
                tgt = cell2e[cells[src] + o * stride]
                need[np.ix_(fl, tgt)] |= own[np.ix_(fl, src)]
    return need


def build_programs(td: dict, tiles: np.ndarray, leaf_cad: np.ndarray, node_cad: np.ndarray,
                   lts: bool) -> dict:
    """Programs of ``tiles`` (launch order) from the mesh's tile tables.

    Returns heads (n_tiles, max_head) uint8, tail (uint16), max_head,
    max_slots, the interface pairs (if_gid, if_cad = reader cadence | source
    cadence << 8, sorted finest reader first) and the weight table wtab."""
    dim, ppo, L = td["dim"], td["ppo"], td["max_depth"]
    starts = np.asarray(td["starts"], dtype=np.int64)
    tiles = np.asarray(tiles, dtype=np.int64)
    nt = len(tiles)
    table = td["table"][tiles].astype(np.int64)
    E = table.shape[1]
    g0, g1 = starts[tiles], starts[tiles + 1]
    a3 = np.asarray(td["anchor3"], dtype=np.int64)[tiles]
    faces = np.zeros(nt, dtype=np.int64)
    side = 1 << (L - td["level"][tiles].astype(np.int64))
    for d in range(dim):
        faces |= (a3[:, d] == 0).astype(np.int64) << (2 * d)
        faces |= ((a3[:, d] + side) == (1 << L)).astype(np.int64) << (2 * d + 1)
    need = owned_cross(table, g0, g1, faces, dim, ppo)
    cells = cross_cells(dim, ppo)
    tcad = leaf_cad[tiles].astype(np.int64)

    # ---- hanging rows (needed only), longest first within a tile
    ptr, gid, w = td["interp_ptr"], td["interp_gid"], td["interp_w"]
    t_idx, e_idx = np.nonzero((table <= -2) & need)
    rows = -table[t_idx, e_idx] - 2
    cnt = ptr[rows + 1] - ptr[rows]
    o = np.lexsort((e_idx, -cnt, t_idx))
    t_idx, e_idx, rows, cnt = t_idx[o], e_idx[o], rows[o], cnt[o]
    n_in = len(rows)
    tile_in_ptr = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(np.bincount(t_idx, minlength=nt), out=tile_in_ptr[1:])
    padded = (cnt + 3) // 4 * 4
    in_tap_ptr = np.zeros(n_in + 1, dtype=np.int64)
    np.cumsum(padded, out=in_tap_ptr[1:])
    n_real = int(cnt.sum())
    within = np.arange(n_real) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    src_idx = np.repeat(ptr[rows], cnt) + within
    dst_idx = np.repeat(in_tap_ptr[:-1], cnt) + within
    tap_gid = gid[src_idx].astype(np.int64)
    tap_tile = np.repeat(t_idx, cnt)
    if n_real:
        key, inv = np.unique((tap_tile << 32) | tap_gid, return_inverse=True)
    else:
        key, inv = np.zeros(0, np.int64), np.zeros(0, np.int64)
    slot_tile = key >> 32
    slot_gid = key & 0xFFFFFFFF
    tile_slot_ptr = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(np.bincount(slot_tile, minlength=nt), out=tile_slot_ptr[1:])
    n_slots = np.diff(tile_slot_ptr)
    max_slots = int(n_slots.max()) if nt else 0
    if max_slots >= 1023:
        raise ProgramError(f"a tile reads {max_slots} interpolation sources (> 1022)")
    local_slot = inv - tile_slot_ptr[tap_tile]
    wtab, widx = np.unique(np.concatenate([w[src_idx], [0.0]]), return_inverse=True)
    if len(wtab) > 64:
        raise ProgramError(f"{len(wtab)} distinct interpolation weights (> 64)")
    zero_w = int(widx[-1])
    tap = np.zeros(int(in_tap_ptr[-1]), dtype=np.int64)
    npad = padded - cnt
    pad_in = np.repeat(np.arange(n_in), npad)
    pad_pos = np.repeat(in_tap_ptr[:-1] + cnt, npad) + (
        np.arange(int(npad.sum())) - np.repeat(np.cumsum(npad) - npad, npad))
    tap[pad_pos] = (n_slots[t_idx[pad_in]] << 6) | zero_w
    tap[dst_idx] = (local_slot << 6) | widx[:-1]

    # ---- copy entries (needed, non-hanging, inside the domain) and slots;
    #      LTS interface pairs where the source cadence differs from the reader's
    ct, ce = np.nonzero((table >= 0) & need)
    cg = table[ct, ce]
    s_tile = slot_tile
    if lts:
        cm = node_cad[cg].astype(np.int64) != tcad[ct]
        sm = node_cad[slot_gid].astype(np.int64) != tcad[s_tile] if len(slot_gid) else np.zeros(0, bool)
        keys = np.concatenate([((31 - tcad[ct[cm]]) << 32) | cg[cm],
                               ((31 - tcad[s_tile[sm]]) << 32) | slot_gid[sm]])
    else:
        cm = np.zeros(len(cg), bool)
        sm = np.zeros(len(slot_gid), bool)
        keys = np.zeros(0, np.int64)
    if len(keys):
        ukeys, pinv = np.unique(keys, return_inverse=True)
        if_gid = ukeys & 0xFFFFFFFF
        if_cad = (31 - (ukeys >> 32)) | (node_cad[if_gid].astype(np.int64) << 8)
        ne = int(cm.sum())
        c_pair = np.zeros(len(cg), np.int64)
        c_pair[cm] = pinv[:ne]
        s_pair = np.zeros(len(slot_gid), np.int64)
        s_pair[sm] = pinv[ne:]
        # pair groups: (reader cadence, source leaf); pairs of one group are contiguous
        if_leaf = np.searchsorted(starts, if_gid, side="right") - 1
        gkey = ((ukeys >> 32) << 40) | if_leaf
        new = np.ones(len(ukeys), dtype=bool)
        new[1:] = gkey[1:] != gkey[:-1]
        grp_start = np.maximum.accumulate(np.where(new, np.arange(len(ukeys)), 0))
    else:
        if_gid = np.zeros(0, np.int64)
        if_cad = np.zeros(0, np.int64)
        c_pair = np.zeros(len(cg), np.int64)
        s_pair = np.zeros(len(slot_gid), np.int64)
        grp_start = np.zeros(0, np.int64)

    def encode(v, is_pair, pair):
        base = np.empty(len(v), dtype=np.int64)
        off = np.empty(len(v), dtype=np.int64)
        lf = np.searchsorted(starts, v[~is_pair], side="right") - 1
        base[~is_pair] = starts[lf]
        off[~is_pair] = v[~is_pair] - starts[lf]
        gs = grp_start[pair[is_pair]]
        base[is_pair] = -gs - 1
        off[is_pair] = pair[is_pair] - gs
        return base, off

    e_base, e_off = encode(cg, cm, c_pair)
    s_base, s_off = encode(slot_gid, sm, s_pair)
    if (len(e_off) and e_off.max() >= 1024) or (len(s_off) and s_off.max() >= 1024):
        raise ProgramError("source offset >= 1024")

    # ---- per-tile base tables
    bkey = np.concatenate([(ct << 33) | (e_base + (1 << 32)), (s_tile << 33) | (s_base + (1 << 32))])
    ukey, binv = np.unique(bkey, return_inverse=True)
    u_tile = ukey >> 33
    u_base = (ukey & ((1 << 33) - 1)) - (1 << 32)
    bptr = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(np.bincount(u_tile, minlength=nt), out=bptr[1:])
    nbase = np.diff(bptr)
    if nt and int(nbase.max()) > MAX_BASES:
        raise ProgramError(f"a tile reads {int(nbase.max())} source groups (> {MAX_BASES})")
    b_idx = (np.arange(len(ukey)) - bptr[u_tile])[binv]
    e_code = (b_idx[:len(cg)] << 10) | e_off
    s_code = (b_idx[len(cg):] << 10) | s_off

    # ---- copy runs: sort by (tile, cell), cut where cells or sources stop
    #      being consecutive (or a box row ends), at most RUN_MAX long
    rc = cells[ce]
    o = np.lexsort((rc, ct))
    rt, rc, rcode = ct[o], rc[o], e_code[o]
    brk = np.ones(len(rt), dtype=bool)
    brk[1:] = ((rt[1:] != rt[:-1]) | (rc[1:] != rc[:-1] + 1) | (rc[1:] % box_strides(dim, ppo)[-2] == 0)
               | ((rcode[1:] >> 10) != (rcode[:-1] >> 10)) | ((rcode[1:] & 1023) != (rcode[:-1] & 1023) + 1))
    rid = np.cumsum(brk) - 1
    first = np.nonzero(brk)[0]
    pos = np.arange(len(rt)) - first[rid]
    brk |= (pos % RUN_MAX) == 0
    first = np.nonzero(brk)[0]
    rlen = np.diff(np.append(first, len(rt)))
    r_tile = rt[first]
    r_word = rc[first] | ((rlen - 1) << 12) | (rcode[first] << 16)
    bucket = np.select([rlen > 4, rlen > 2, rlen > 1], [0, 1, 2], 3)
    o = np.lexsort((rc[first], bucket, r_tile))
    r_tile, r_word, bucket = r_tile[o], r_word[o], bucket[o]
    nrun = np.bincount(r_tile, minlength=nt)
    rptr = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(nrun, out=rptr[1:])
    bcnt = np.zeros((nt, 4), dtype=np.int64)
    np.add.at(bcnt, (r_tile, bucket), 1)

    # ---- heads: header, bases, runs, slots (16-byte aligned sections)
    off_base = 4 * HDR_WORDS
    off_run = off_base + _r16(4 * nbase)
    off_slot = off_run + _r16(4 * nrun)
    head_len = off_slot + _r16(2 * n_slots)
    max_head = int(head_len.max()) if nt else 64
    # ---- tails: rows, taps
    nrow = np.diff(tile_in_ptr)
    cell_in = cells[e_idx]
    nq = (in_tap_ptr[1:] - in_tap_ptr[:-1]) // 4
    tile_tap0 = in_tap_ptr[tile_in_ptr[:-1]]
    t_r = t_idx
    qoff = (in_tap_ptr[:-1] - tile_tap0[t_r]) // 4 if n_in else np.zeros(0, np.int64)
    if n_in and (nq.max() > 31 or qoff.max() >= (1 << 15) or cell_in.max() >= (1 << 12)):
        raise ProgramError("hanging row does not fit the packed row word")
    if nt and nrow.max() >= 1024:
        raise ProgramError("more than 1023 hanging rows in one tile")
    row_word = cell_in | (nq << 12) | (qoff << 17)
    ntap = np.diff(np.append(tile_tap0, int(in_tap_ptr[-1])))
    rows_b = _r16(4 * nrow)
    tail_len = rows_b + _r16(2 * ntap)
    tail_start = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(tail_len, out=tail_start[1:])
    if int(tail_start[-1]) // 16 >= (1 << 31):
        raise ProgramError("tile tails exceed 32 GB")

    heads = np.zeros((max(nt, 1), max_head // 4), dtype=np.uint32)
    lmeta = td["level"][tiles].astype(np.int64) | (tcad << 8) | (faces << 16)
    hdr = np.stack([g0, g1 - g0, lmeta, nrun, n_slots, nrow, nbase, tail_len,
                    a3[:, 0], a3[:, 1], a3[:, 2], bcnt[:, 0] | (bcnt[:, 1] << 16), bcnt[:, 2] | (bcnt[:, 3] << 16),
                    np.zeros(nt, np.int64), tail_start[:nt] // 16, rows_b // 2], axis=1)
    if nt:
        heads[:nt, :HDR_WORDS] = hdr.astype(np.int64).astype(np.uint32)
        heads[u_tile, off_base // 4 + (np.arange(len(ukey)) - bptr[u_tile])] = \
            u_base.astype(np.int32).view(np.uint32)
        heads[r_tile, off_run[r_tile] // 4 + (np.arange(len(r_word)) - rptr[r_tile])] = r_word.astype(np.uint32)
        h16 = heads.view(np.uint16)
        ls = np.arange(len(s_code)) - tile_slot_ptr[s_tile]
        h16[s_tile, off_slot[s_tile] // 2 + ls] = s_code.astype(np.uint16)
    tail = np.zeros(max(int(tail_start[-1]) // 2, 8), dtype=np.uint16)
    t32 = tail.view(np.uint32)
    if n_in:
        lr = np.arange(n_in) - tile_in_ptr[t_r]
        t32[tail_start[t_r] // 4 + lr] = row_word.astype(np.uint32)
    if len(tap):
        t_t = np.repeat(np.arange(nt, dtype=np.int64), ntap)
        lt = np.arange(len(tap)) - tile_tap0[t_t]
        tail[(tail_start[t_t] + rows_b[t_t]) // 2 + lt] = tap.astype(np.uint16)
    return dict(heads=heads.view(np.uint8), tail=tail, max_head=max_head, max_slots=max_slots,
                max_tail=int(tail_len.max()) if nt else 0,
                if_gid=if_gid.astype(np.int32), if_cad=if_cad.astype(np.int32), n_iface=len(if_gid),
                wtab=wtab.astype(np.float64), n_rows=n_in, n_cells=int(need.sum()))


def decode(prog: dict, t: int) -> dict:
    """A tile's program back as {box cell: source} (source = gid, or
    ('pair', i) for interface pair i) plus its rows [(cell, [(slot source,
    weight)...])] — the inverse of build_programs, for tests."""
    h8 = prog["heads"][t]
    h = h8.view(np.int32)
    nrun, nslot, nrow, nbase = int(h[3]), int(h[4]), int(h[5]), int(h[6])
    bases = h[HDR_WORDS:HDR_WORDS + nbase].astype(np.int64)
    off_run = 4 * HDR_WORDS + int(_r16(4 * nbase))
    off_slot = off_run + int(_r16(4 * nrun))
    runs = h8[off_run:off_run + 4 * nrun].view(np.uint32).astype(np.int64)
    slots = h8[off_slot:off_slot + 2 * nslot].view(np.uint16).astype(np.int64)

    def src(code, i=0):
        b, o = bases[code >> 10], (code & 1023) + i
        return int(b + o) if b >= 0 else ("pair", int(-b - 1 + o))

    cells = {}
    for wd in runs:
        for i in range(((wd >> 12) & 7) + 1):
            cells[int((wd & 0xFFF) + i)] = src(wd >> 16, i)
    slot_src = [src(c) for c in slots]
    tail = prog["tail"]
    t0 = int(h[14]) * 8
    rw = tail[t0:t0 + 2 * nrow].view(np.uint32).astype(np.int64)
    taps = tail[t0 + int(h[15]):].astype(np.int64)
    wt = prog["wtab"]
    rows = []
    for wd in rw:
        nq, q0 = (wd >> 12) & 31, wd >> 17
        tt = taps[4 * q0: 4 * q0 + 4 * nq]
        rows.append((int(wd & 0xFFF), [(slot_src[s] if s < nslot else None, float(wt[k]))
                                       for s, k in zip(tt >> 6, tt & 63)]))
    b = [int(x) & 0xFFFF for x in h[11:13]] + [int(x) >> 16 for x in h[11:13]]
    return dict(g0=int(h[0]), n_own=int(h[1]), cells=cells, rows=rows,
                buckets=(b[0], b[2], b[1], b[3]))


def build_programs_native(mesh, tiles: np.ndarray, leaf_cad: np.ndarray, lts: bool, n_threads: int = 0) -> dict:
    """build_programs through the native builder (csrc/amr_programs.cpp), from
    the mesh's own leaf tables (no host copy of the n_leaves x E table); the
    same dict, byte for byte (tests/test_programs_native.py)."""
    import ctypes as C

    from . import _native

    L = _native.lib()
    tiles = np.ascontiguousarray(tiles, dtype=np.int32)
    cad = np.ascontiguousarray(leaf_cad, dtype=np.int32)
    h = L.amr_programs_build(mesh._nm.full(), len(tiles), _native.ptr(tiles, C.c_int32), _native.ptr(cad, C.c_int32),
                             1 if lts else 0, box_strides(mesh.dim, mesh.ppo)[-2], n_threads)
    if not h:
        raise ProgramError(_native.last_error())
    try:
        info = np.zeros(9, dtype=np.int64)
        L.amr_programs_info(h, _native.ptr(info, C.c_int64))
        nt, max_head, max_tail, max_slots, n_iface, n_wtab, n_tail, n_rows, n_cells = (int(x) for x in info)
        heads = np.empty((max(nt, 1), max_head), dtype=np.uint8)
        tail = np.empty(n_tail, dtype=np.uint16)
        if_gid = np.empty(max(n_iface, 1), dtype=np.int32)
        if_cad = np.empty(max(n_iface, 1), dtype=np.int32)
        wtab = np.empty(n_wtab, dtype=np.float64)
        L.amr_programs_fetch(h, heads.ctypes.data, tail.ctypes.data, if_gid.ctypes.data, if_cad.ctypes.data,
                             wtab.ctypes.data)
    finally:
        L.amr_programs_free(h)
    return dict(heads=heads, tail=tail, max_head=max_head, max_slots=max_slots, max_tail=max_tail,
                if_gid=if_gid[:n_iface], if_cad=if_cad[:n_iface], n_iface=n_iface, wtab=wtab, n_rows=n_rows,
                n_cells=n_cells)


def build_programs_device(mesh, tiles: np.ndarray, leaf_cad: np.ndarray, lts: bool, device=None) -> dict:
    """build_programs on the device (csrc/amr_devprog.cu) from the mesh's
    device tables (``Mesh.device_tables``): the same dict, byte for byte
    (tests/test_devprog_gpu.py), with ``heads``, ``tail``, ``if_gid``,
    ``if_cad`` and ``wtab`` as CUDA tensors.  One thread per tile; the
    sort/unique of the interface-pair keys and of the used weights are torch's."""
    import ctypes as C

    import torch

    from . import _native

    L = _native.lib()
    tabs = mesh.device_tables()
    device = tabs["table"].device if device is None else device
    dim, ppo = mesh.dim, mesh.ppo
    nt = len(tiles)
    n_leaves = len(leaf_cad)
    E = tabs["table"].shape[1]
    NI = ppo ** dim
    cells = cross_cells(dim, ppo)
    bs = box_strides(dim, ppo)
    cell2e = np.full(box_cells(dim, ppo), -1, dtype=np.int32)
    cell2e[cells] = np.arange(len(cells), dtype=np.int32)
    pos = np.zeros((NI, 3), dtype=np.int16)
    k = np.arange(NI)
    for d in range(dim):
        pos[:, d] = (k // ppo ** (dim - 1 - d)) % ppo
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
    with torch.cuda.device(device):
        st = torch.cuda.current_stream(device).cuda_stream
        d_cell, d_c2e, d_pos = T(cells.astype(np.int32)), T(cell2e), T(pos)
        d_tiles, d_cad = T(np.asarray(tiles, dtype=np.int32)), T(np.asarray(leaf_cad, dtype=np.int32))
        A = _native.AmrDevProg()
        A.dim, A.max_depth, A.ppo, A.lts, A.row_stride = dim, mesh.L, ppo, 1 if lts else 0, bs[-2]
        A.max_bases = int(os.environ.get("AMR_MAX_BASES", "0"))
        A.n_leaves, A.n_tiles = n_leaves, nt
        A.table, A.starts = tabs["table"].data_ptr(), tabs["starts"].data_ptr()
        A.anchors, A.levels = tabs["anchors"].data_ptr(), tabs["levels"].data_ptr()
        A.leaf_cad, A.tiles = d_cad.data_ptr(), d_tiles.data_ptr()
        A.row_ptr, A.gid, A.w = tabs["row_ptr"].data_ptr(), tabs["gid"].data_ptr(), tabs["w"].data_ptr()
        A.cell, A.cell2e, A.pos = d_cell.data_ptr(), d_c2e.data_ptr(), d_pos.data_ptr()
        threads = 128
        blocks = max(1, min((nt + threads - 1) // threads, 148 * 4))
        n_rows_mesh = tabs["row_ptr"].numel() - 1
        need = torch.empty((max(nt, 1), E), dtype=torch.uint8, device=device)
        row_used = torch.zeros(max(n_rows_mesh, 1), dtype=torch.uint8, device=device)
        n_keys = torch.zeros(max(nt, 1), dtype=torch.int64, device=device)
        _native.check(L.amr_dp_need(C.byref(A), need.data_ptr(), row_used.data_ptr(), n_keys.data_ptr(), blocks,
                                    threads, st), "amr_dp_need")
        # interface pairs: unique (reader cadence, gid) keys, finest reader first
        ukeys = torch.zeros(0, dtype=torch.int64, device=device)
        if lts and nt:
            ends = torch.cumsum(n_keys[:nt], 0)
            total = int(ends[-1])
            if total:
                keys = torch.empty(total, dtype=torch.int64, device=device)
                off = ends - n_keys[:nt]
                _native.check(L.amr_dp_keys(C.byref(A), need.data_ptr(), off.data_ptr(), keys.data_ptr(), blocks,
                                            threads, st), "amr_dp_keys")
                ukeys = torch.unique(keys)
        n_iface = ukeys.numel()
        if n_iface:
            if_gid = ukeys & 0xFFFFFFFF
            hi = ukeys >> 32
            leaf = torch.searchsorted(tabs["starts"], if_gid, right=True) - 1
            if_cad = (31 - hi) | (d_cad[leaf].to(torch.int64) << 8)
            new = torch.ones(n_iface, dtype=torch.bool, device=device)
            new[1:] = (hi[1:] != hi[:-1]) | (leaf[1:] != leaf[:-1])
            idx = torch.arange(n_iface, dtype=torch.int64, device=device)
            grp_start = torch.cummax(torch.where(new, idx, torch.zeros_like(idx)), 0).values
        else:
            if_gid = if_cad = grp_start = torch.zeros(0, dtype=torch.int64, device=device)
        # weights of the used rows
        counts = tabs["row_ptr"][1:] - tabs["row_ptr"][:-1]
        used_w = tabs["w"][torch.repeat_interleave(row_used[:n_rows_mesh].bool(), counts)] if n_rows_mesh else \
            torch.zeros(0, dtype=torch.float64, device=device)
        wtab = torch.unique(torch.cat([torch.zeros(1, dtype=torch.float64, device=device), used_w]))
        if wtab.numel() > 64:
            raise ProgramError(f"{wtab.numel()} distinct interpolation weights (> 64)")
        gs = grp_start if n_iface else torch.zeros(1, dtype=torch.int64, device=device)
        uk = ukeys if n_iface else torch.zeros(1, dtype=torch.int64, device=device)
        A.n_iface, A.ukeys, A.grp_start = n_iface, uk.data_ptr(), gs.data_ptr()
        A.n_wtab, A.wtab = wtab.numel(), wtab.data_ptr()
        nb = C.c_int64(0)
        L.amr_dp_scratch_bytes(blocks * threads, C.byref(nb))
        scratch = torch.empty(nb.value, dtype=torch.uint8, device=device)
        sizes = torch.zeros((max(nt, 1), 5), dtype=torch.int64, device=device)
        err = torch.zeros(1, dtype=torch.int32, device=device)
        _native.check(L.amr_dp_encode(C.byref(A), need.data_ptr(), scratch.data_ptr(), sizes.data_ptr(), None, 0,
                                      None, None, err.data_ptr(), blocks, threads, st), "amr_dp_encode")
        e = int(err[0])
        if e:
            raise ProgramError("programs: a tile reads more source groups than the encoding holds (> 63)" if e & 2
                               else "programs: a tile reads too many interpolation sources (> 1022)" if e & 1
                               else "programs: tile does not fit the compact encoding")
        max_head = max(64, int(sizes[:nt, 0].max())) if nt else 64
        tail_end = torch.cumsum(sizes[:, 1], 0)
        tail_total = int(tail_end[nt - 1]) if nt else 0
        if tail_total // 16 >= (1 << 31):
            raise ProgramError("tile tails exceed 32 GB")
        tail_off = tail_end - sizes[:, 1]
        heads = torch.zeros((max(nt, 1), max_head), dtype=torch.uint8, device=device)
        tail = torch.zeros(max(tail_total // 2, 8), dtype=torch.int16, device=device)
        _native.check(L.amr_dp_encode(C.byref(A), need.data_ptr(), scratch.data_ptr(), sizes.data_ptr(),
                                      heads.data_ptr(), max_head, tail_off.data_ptr(), tail.data_ptr(), err.data_ptr(),
                                      blocks, threads, st), "amr_dp_encode")
        if int(err[0]):
            raise ProgramError("hanging row does not fit the packed row word")
        tot = sizes[:nt].sum(0) if nt else torch.zeros(5, dtype=torch.int64)
        return dict(heads=heads, tail=tail, max_head=max_head, max_slots=int(sizes[:nt, 2].max()) if nt else 0,
                    max_tail=int(sizes[:nt, 1].max()) if nt else 0, if_gid=if_gid.to(torch.int32),
                    if_cad=if_cad.to(torch.int32), n_iface=n_iface, wtab=wtab, n_rows=int(tot[3]),
                    n_cells=int(tot[4]))
