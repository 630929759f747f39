"""Per-tile program blobs of the blob stage kernels (amr_stage, AMR_KERNEL 1 and 2).

One blob per leaf tile, in launch order, 16-byte aligned.  The kernel fetches
its head (header, bases, runs, slot codes) with a single bulk copy
(``cp.async.bulk``) into a shared-memory ring two tiles ahead; the tail (face
entry codes, rows, taps) is bulk-prefetched into L2 and read from there.  It re-encodes the tile table and the
tile's interpolation program (``Engine._tile_programs``) compactly:

=========  =================================================================
section    contents
=========  =================================================================
header     16 int32: g0, n_own, level | cadence<<8 | faces<<16, n_runs, n_slots,
           n_rows, n_bases, blob length (uint16 units), anchor[3], the
           uint16 offsets of the entry/slot/row/tap sections, and the blob's
           own offset in the blob array (16-byte units)
bases      int32 per source group: a source leaf's first gid (>= 0), or, for
           LTS interface pairs, -(first pair of the (reader cadence, source
           leaf) group) - 1
runs       uint32 per copy run: smem cell | (length-1) << 12 | code << 16,
           code = base index << 10 | offset of the first source; base index
           63 is special: offset 0 = outside the domain (zeros).  Runs cover
           every non-hanging stencil-cross entry, z-consecutive cells with
           consecutive sources, longest first
slots      uint16 per unique interpolation source, same code
entries    face tiles only: uint16 code per stencil-cross entry (offset r+1
           of base 63 = the tile's hanging row r), for the phi lookups of the
           radiative rows
rows       uint32 per hanging row: smem cell | n_quads << 12 | quad offset << 17
taps       uint16 per tap: slot << 6 | weight id, rows padded to 4 taps with
           (zero slot, weight 0) exactly as the int32 program
=========  =================================================================

A source leaf owns at most ppo^D nodes (< 1024) and a (cadence, leaf) pair
group at most as many, so every offset fits 10 bits.  Tables are static: the
encoding is built once per mesh (all numpy, vectorised over tiles).
"""
from __future__ import annotations

import numpy as np

IFACE_BASE = -(1 << 20)  # AMR_IFACE_BASE in amr_kernels.cu
HDR_WORDS = 16           # int32 words in the header
SPECIAL = 63             # base index of outside / hanging codes
MAX_BASES = 63


def _pad8(n):
    return (np.asarray(n, dtype=np.int64) + 7) // 8 * 8


class BlobError(ValueError):
    """The mesh does not fit the compact encoding (the kernel falls back to v17)."""


def build_blobs(table: np.ndarray, prog: dict, n_iface: int, starts: np.ndarray, anchor3: np.ndarray,
                n_interior: int, n_pad: int) -> dict:
    """Blobs for every tile of ``table`` (launch order).

    ``table``/``prog`` are the outputs of ``Engine._tile_programs``; ``starts``
    the leaf gid offsets (leaf_slices), ``anchor3`` the leaf anchors,
    ``n_interior`` = ppo^D and ``n_pad`` = ppo + 4 (the box edge)."""
    cross_cells = prog["cross_cells"]
    nt, E = table.shape
    starts = np.asarray(starts, dtype=np.int64)
    meta = prog["tile_meta"].astype(np.int64)
    tsp = prog["tile_slot_ptr"].astype(np.int64)
    tip = prog["tile_in_ptr"].astype(np.int64)
    itp = prog["in_tap_ptr"].astype(np.int64)
    ttp = prog["tile_tap_ptr"].astype(np.int64)
    n_slot_tot = int(tsp[-1])
    n_in = int(tip[-1])
    n_tap = int(ttp[-1])
    slot_gid = prog["slot_gid"][:n_slot_tot].astype(np.int64)
    if len(prog["wtab"]) > 64:
        raise BlobError("more than 64 distinct interpolation weights")

    # -- interface pair groups: pairs sorted by (reader cadence desc, gid), so
    #    the pairs of one (cadence, source leaf) are contiguous
    if n_iface:
        if_gid = prog["if_gid"][:n_iface].astype(np.int64)
        if_cad = prog["if_cad"][:n_iface].astype(np.int64) & 0xFF  # reader cadence
        if_leaf = np.searchsorted(starts, if_gid, side="right") - 1
        gkey = (if_cad << 40) | if_leaf
        new = np.ones(n_iface, dtype=bool)
        new[1:] = gkey[1:] != gkey[:-1]
        grp_start = np.maximum.accumulate(np.where(new, np.arange(n_iface), 0))
    else:
        grp_start = np.zeros(0, np.int64)

    def encode_src(v: np.ndarray, is_pair: np.ndarray):
        """(base value, offset) of gids (is_pair False) or interface pairs."""
        base = np.empty(len(v), dtype=np.int64)
        off = np.empty(len(v), dtype=np.int64)
        g = v[~is_pair]
        lf = np.searchsorted(starts, g, side="right") - 1
        base[~is_pair] = starts[lf]
        off[~is_pair] = g - starts[lf]
        p = v[is_pair]
        gs = grp_start[p]
        base[is_pair] = -gs - 1
        off[is_pair] = p - gs
        return base, off

    # entries
    ent = table.astype(np.int64)
    t_e = np.repeat(np.arange(nt, dtype=np.int64), E)
    flat = ent.reshape(-1)
    is_copy = flat >= 0
    is_pair = flat <= IFACE_BASE
    is_src = is_copy | is_pair
    src_v = np.where(is_pair, IFACE_BASE - flat, flat)[is_src]
    e_base, e_off = encode_src(src_v, is_pair[is_src])
    # slots
    t_s = np.repeat(np.arange(nt, dtype=np.int64), np.diff(tsp))
    s_pair = slot_gid < 0
    s_base, s_off = encode_src(np.where(s_pair, -slot_gid - 1, slot_gid), s_pair)

    # per-tile base tables
    bkey = np.concatenate([(t_e[is_src] << 33) | (e_base + (1 << 32)),
                           (t_s << 33) | (s_base + (1 << 32))])
    ukey, inv = np.unique(bkey, return_inverse=True)
    u_tile = ukey >> 33
    u_base = (ukey & ((1 << 33) - 1)) - (1 << 32)
    bptr = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(np.bincount(u_tile, minlength=nt), out=bptr[1:])
    nbase = np.diff(bptr)
    if nt and int(nbase.max()) > MAX_BASES:
        raise BlobError(f"a tile reads {int(nbase.max())} source groups (> {MAX_BASES})")
    local_b = np.arange(len(ukey)) - bptr[u_tile]
    b_idx = local_b[inv]
    ne_src = int(is_src.sum())
    if (len(e_off) and e_off.max() >= 1024) or (len(s_off) and s_off.max() >= 1024):
        raise BlobError("source offset >= 1024")

    code = np.full(nt * E, SPECIAL << 10, dtype=np.int64)  # outside by default
    code[is_src] = (b_idx[:ne_src] << 10) | e_off
    hang = (flat <= -2) & ~is_pair
    row_local = -flat[hang] - 2
    if len(row_local) and row_local.max() + 1 >= 1024:
        raise BlobError("more than 1022 hanging rows in one tile")
    code[hang] = (SPECIAL << 10) | (row_local + 1)
    s_code = (b_idx[ne_src:] << 10) | s_off

    # rows and taps
    nrow = np.diff(tip)
    faces = (meta[:, 2] >> 16) & 0x3F
    if nt and int(nrow[faces != 0].max(initial=0)) > n_interior:
        # face tiles keep the phi of their hanging rows in the owned-phi array
        raise BlobError("face tile with more hanging rows than interior nodes")
    t_r = np.repeat(np.arange(nt, dtype=np.int64), nrow)
    cell = prog["in_cell"][:n_in].astype(np.int64)
    nq = (itp[1:] - itp[:-1]) // 4
    qoff = (itp[:-1] - ttp[t_r]) // 4 if n_in else np.zeros(0, np.int64)
    if n_in and (nq.max() > 31 or qoff.max() >= (1 << 15) or cell.max() >= (1 << 12)):
        raise BlobError("hanging row does not fit the packed row word")
    row_word = (cell | (nq << 12) | (qoff << 17)).astype(np.uint32)
    tap32 = prog["tap"][:n_tap].astype(np.int64)
    t_slot = tap32 >> 16
    t_w = tap32 & 0xFFFF
    if n_tap and (t_slot.max() >= 1024 or t_w.max() >= 64):
        raise BlobError("tap slot >= 1024 or weight id >= 64")
    tap16 = ((t_slot << 6) | t_w).astype(np.uint16)
    ntap = np.diff(ttp)

    # copy runs: the non-hanging cross entries of a tile sorted by smem cell
    # and cut into runs of z-consecutive cells whose sources are consecutive
    # nodes of one source group (or zeros), at most 16 long; longest first
    cross_cells = np.asarray(cross_cells, dtype=np.int64)
    code2 = code.reshape(nt, E)
    keep = ~hang.reshape(nt, E)
    rt, re_ = np.nonzero(keep)
    rc = cross_cells[re_]
    rcode = code2[rt, re_]
    o = np.lexsort((rc, rt))
    rt, rc, rcode = rt[o], rc[o], rcode[o]
    rb, ro = rcode >> 10, rcode & 1023
    brk = np.ones(len(rt), dtype=bool)
    brk[1:] = ((rt[1:] != rt[:-1]) | (rc[1:] != rc[:-1] + 1) | (rc[1:] % n_pad == 0) | (rb[1:] != rb[:-1])
               | ((rb[1:] != SPECIAL) & (ro[1:] != ro[:-1] + 1)))
    rid = np.cumsum(brk) - 1
    first = np.nonzero(brk)[0]
    pos = np.arange(len(rt)) - first[rid]
    brk |= (pos % 16) == 0
    first = np.nonzero(brk)[0]
    rlen = np.diff(np.append(first, len(rt)))
    r_tile = rt[first]
    r_word = (rc[first] | ((rlen - 1) << 12) | (rcode[first] << 16)).astype(np.uint32)
    o = np.lexsort((-rlen, r_tile))
    r_tile, r_word = r_tile[o], r_word[o]
    nrun = np.bincount(r_tile, minlength=nt)
    rptr = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(nrun, out=rptr[1:])

    # section sizes in uint16 units
    nslot = np.diff(tsp)
    sz_hdr = 2 * HDR_WORDS
    sz_base = _pad8(2 * nbase)
    sz_run = _pad8(2 * nrun)
    sz_ent = np.where(faces != 0, int(_pad8(E)), 0)  # entry codes: face tiles only (phi lookups)
    sz_slot = _pad8(nslot)
    sz_row = _pad8(2 * nrow)
    sz_tap = _pad8(ntap)
    off_base = np.full(nt, sz_hdr, dtype=np.int64)
    off_run = off_base + sz_base
    off_slot = off_run + sz_run
    off_ent = off_slot + sz_slot
    off_row = off_ent + sz_ent
    off_tap = off_row + sz_row
    length = off_tap + sz_tap
    if nt and int(length.max()) >= (1 << 20):
        raise BlobError("tile blob too large")
    tstart = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(length, out=tstart[1:])
    blob = np.zeros(max(int(tstart[-1]), 8), dtype=np.uint16)
    b32 = blob.view(np.uint32)

    # header
    a3 = np.asarray(anchor3, dtype=np.int64)[meta[:, 3]]
    hdr = np.stack([meta[:, 0], meta[:, 1] - meta[:, 0], meta[:, 2], nrun, nslot, nrow, nbase, length,
                    a3[:, 0], a3[:, 1], a3[:, 2], off_ent, off_slot, off_row, off_tap,
                    tstart[:nt] // 8], axis=1)
    idx = (tstart[:nt, None] // 2 + np.arange(HDR_WORDS)[None, :]).reshape(-1)
    b32[idx] = hdr.reshape(-1).astype(np.int64).astype(np.uint32)
    # bases (int32)
    if len(ukey):
        b32[(tstart[u_tile] + off_base[u_tile]) // 2 + local_b] = u_base.astype(np.int32).view(np.uint32)
    # entries
    # runs
    if len(r_word):
        lr_ = np.arange(len(r_word)) - rptr[r_tile]
        b32[(tstart[r_tile] + off_run[r_tile]) // 2 + lr_] = r_word
    # entry codes of face tiles
    ft = np.nonzero(faces != 0)[0]
    if len(ft):
        blob[(tstart[ft] + off_ent[ft])[:, None] + np.arange(E)[None, :]] = code2[ft].astype(np.uint16)
    # slots
    if n_slot_tot:
        ls = np.arange(n_slot_tot) - tsp[t_s]
        blob[tstart[t_s] + off_slot[t_s] + ls] = s_code.astype(np.uint16)
    # rows
    if n_in:
        lr = np.arange(n_in) - tip[t_r]
        b32[(tstart[t_r] + off_row[t_r]) // 2 + lr] = row_word
    # taps
    if n_tap:
        t_t = np.repeat(np.arange(nt, dtype=np.int64), ntap)
        lt = np.arange(n_tap) - ttp[t_t]
        blob[tstart[t_t] + off_tap[t_t] + lt] = tap16
    if int(tstart[-1]) // 8 >= (1 << 31):
        raise BlobError("tile blobs exceed 32 GB")
    head = (off_ent * 2).astype(np.int32)  # header, bases, runs, slots: staged in shared memory
    tail = (length - off_ent) * 2          # face entry codes, rows, taps: read through L2
    # the heads again at a fixed stride (the per-tile kernel copies without an offset lookup)
    mh = int(head.max()) if nt else 16
    hstart = tstart[:nt] * 2
    heads = np.zeros((max(nt, 1), mh), dtype=np.uint8)
    bb = blob.view(np.uint8)
    if nt:
        within = np.arange(mh)[None, :]
        src = np.minimum(hstart[:, None] + within, len(bb) - 1)
        heads[:nt] = np.where(within < head[:, None], bb[src], 0)
    return dict(blob=blob, blob_off=(tstart * 2).astype(np.int64), blob_head=head, heads=heads,
                max_blob=int(head.max()) if nt else 16, max_tail=int(tail.max()) if nt else 0,  # tail: info
                max_rows=int(nrow.max()) if nt else 0)


def cell_entries(cross_cells: np.ndarray, dim: int, ppo: int) -> np.ndarray:
    """Inverse of the cross enumeration: stencil-cross entry of each padded-box
    cell (0xFFFF off the cross)."""
    NS = (ppo + 4) ** dim
    out = np.full(NS, 0xFFFF, dtype=np.uint16)
    out[np.asarray(cross_cells, dtype=np.int64)] = np.arange(len(cross_cells), dtype=np.uint16)
    return out
