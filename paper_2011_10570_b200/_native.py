"""ctypes binding of the C ABI in include/amr_b200.h.

The library is built in-tree (paper_2011_10570_b200/_lib/libamr_b200.so) and
is mandatory: there is no Python or CPU fallback for anything it provides.
If it cannot be loaded (or built, when nvcc is present) every caller raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

AMR_MAXL = 16
AMR_MAXP = 4

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p


class AmrSliceCoef(C.Structure):
    _fields_ = [
        ("cur", C.c_int32 * AMR_MAXL),
        ("mode", (C.c_int32 * AMR_MAXL) * AMR_MAXL),
        ("cstage", ((C.c_double * AMR_MAXP) * AMR_MAXP) * AMR_MAXL),
        ("comb", (C.c_double * AMR_MAXP) * AMR_MAXL),
        ("M", (((C.c_double * AMR_MAXP) * AMR_MAXP) * AMR_MAXL) * AMR_MAXL),
        ("Mv", (((C.c_double * AMR_MAXP) * AMR_MAXP) * AMR_MAXL) * AMR_MAXL),
        ("dtw", ((C.c_double * AMR_MAXP) * AMR_MAXL) * AMR_MAXL),
    ]


class AmrStageParams(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("ppo", C.c_int), ("pad", C.c_int),
        ("lts", C.c_int), ("stage", C.c_int), ("n_stages", C.c_int),
        ("nonlinear", C.c_int), ("gts_cur", C.c_int),
        ("n_tiles", C.c_int64), ("n_nodes", C.c_int64), ("ld", C.c_int64),
        ("heads", _vp), ("tail", _vp), ("max_head", C.c_int), ("max_tail", C.c_int), ("max_slots", C.c_int), ("threads", C.c_int), ("lean", C.c_int), ("probe", _vp),
        ("wtab", _vp), ("n_wtab", C.c_int),
        ("n_iface", C.c_int64), ("n_iface_total", C.c_int64), ("if_gid", _vp), ("if_cad", _vp), ("ibuf", _vp), ("ibuf0", _vp), ("if_phase", C.c_int),
        ("n_vt", C.c_int), ("vt_j", C.c_int * AMR_MAXP), ("Y", _vp),
        ("U0", _vp), ("U1", _vp), ("K", _vp),
        ("coef", _vp),
        ("l_cur_mask", C.c_uint32),
        ("l_cnext", (C.c_double * AMR_MAXP) * AMR_MAXL),
        ("l_comb", (C.c_double * AMR_MAXP) * AMR_MAXL),
        ("g_cstage", (C.c_double * AMR_MAXP) * AMR_MAXP),
        ("g_comb", C.c_double * AMR_MAXP),
        ("max_depth", C.c_int),
        ("top_nodes", C.c_int64),
        ("lo", C.c_double * 3), ("extent", C.c_double * 3),
        ("h", C.c_double * AMR_MAXL), ("h2", C.c_double * AMR_MAXL),
        ("h2_pow2", C.c_int32 * AMR_MAXL),
        ("inv_h2", C.c_double * AMR_MAXL),
        ("r_eps", C.c_double), ("r_eps2", C.c_double),
        ("k_chi", C.c_double), ("k_phi", C.c_double), ("f0_chi", C.c_double), ("f0_phi", C.c_double),
        ("d2c", C.c_double * 5), ("d2e0", C.c_double * 6), ("d2e1", C.c_double * 6),
        ("d1c", C.c_double * 5), ("d1e0", C.c_double * 5), ("d1e1", C.c_double * 5),
    ]


AMR_GHOST_ROWS = 8


class AmrDevProg(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("max_depth", C.c_int), ("ppo", C.c_int), ("lts", C.c_int), ("row_stride", C.c_int),
        ("n_wtab", C.c_int), ("max_bases", C.c_int),
        ("n_leaves", C.c_int64), ("n_tiles", C.c_int64), ("n_iface", C.c_int64),
        ("table", _vp), ("starts", _vp), ("anchors", _vp), ("levels", _vp), ("leaf_cad", _vp), ("tiles", _vp),
        ("row_ptr", _vp), ("gid", _vp), ("w", _vp), ("cell", _vp), ("cell2e", _vp), ("pos", _vp),
        ("ukeys", _vp), ("grp_start", _vp), ("wtab", _vp),
    ]


class AmrGhostMove(C.Structure):
    _fields_ = [
        ("n_ranges", C.c_int64), ("total", C.c_int64),
        ("start", _vp), ("off", _vp), ("cad", _vp),
        ("n_rows", C.c_int), ("buf_ld", C.c_int64),
        ("row0", _vp * AMR_GHOST_ROWS), ("row1", _vp * AMR_GHOST_ROWS),
        ("par", C.c_int32 * AMR_MAXL),
    ]


# every symbol the header declares (checked by tests/test_native_abi.py)
SIGNATURES = {
    "amr_last_error": ([], C.c_char_p),
    "amr_abi_version": ([], C.c_int),
    "amr_morton_sort": ([C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _i64p], C.c_int),
    "amr_balance": ([C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _i64p], _vp),
    "amr_oct_keys": ([C.c_int, C.c_int, C.c_int64, _vp, _vp, _vp, _vp], C.c_int),
    "amr_oct_octants": ([C.c_int, C.c_int, C.c_int64, _vp, _vp, _vp, _vp], C.c_int),
    "amr_oct_split": ([C.c_int, C.c_int, C.c_int64, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "amr_oct_balance_mark": ([C.c_int, C.c_int, C.c_int64, _vp, _vp, _vp], C.c_int),
    "amr_tree_fetch": ([_vp, _i32p, _i32p], C.c_int),
    "amr_tree_free": ([_vp], None),
    "amr_mesh_build": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _i32p, C.c_int], _vp),
    "amr_dm_ownership": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64] + [_vp] * 8, C.c_int),
    "amr_dm_gids": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64] + [_vp] * 8, C.c_int),
    "amr_dm_table": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64] + [_vp] * 7, C.c_int),
    "amr_dm_hang_list": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64] + [_vp] * 8, C.c_int),
    "amr_dm_table_rows": ([C.c_int64, _vp, _vp, C.c_int64, _vp, _vp, _vp], C.c_int),
    "amr_dm_rows": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, _vp, _vp, _vp, _vp, C.c_int64] + [_vp] * 7,
                    C.c_int),
    "amr_mesh_from_tables": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, _i32p, _i32p, _i32p, _i64p, _i32p,
                              _i32p, C.c_int64, _i64p, _i64p, _i32p, _f64p], _vp),
    "amr_mesh_free": ([_vp], None),
    "amr_mesh_n_nodes": ([_vp], C.c_int64),
    "amr_mesh_leaf_starts": ([_vp, _i64p], C.c_int),
    "amr_mesh_leaf_gids": ([_vp, _i32p], C.c_int),
    "amr_mesh_node_coords": ([_vp, _i32p], C.c_int),
    "amr_tile_entries": ([C.c_int, C.c_int], C.c_int64),
    "amr_mesh_tile_table": ([_vp, _i32p], C.c_int),
    "amr_mesh_interp_rows": ([_vp], C.c_int64),
    "amr_mesh_interp_nnz": ([_vp], C.c_int64),
    "amr_mesh_interp_csr": ([_vp, _i64p, _i32p, _f64p], C.c_int),
    "amr_mesh_n_blocks": ([_vp], C.c_int64),
    "amr_programs_build": ([_vp, C.c_int64, _i32p, _i32p, C.c_int, C.c_int, C.c_int], _vp),
    "amr_programs_info": ([_vp, _i64p], C.c_int),
    "amr_programs_fetch": ([_vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "amr_programs_free": ([_vp], None),
    "amr_dp_scratch_bytes": ([C.c_int, _i64p], C.c_int),
    "amr_dp_need": ([C.POINTER(AmrDevProg), _vp, _vp, _vp, C.c_int, C.c_int, _vp], C.c_int),
    "amr_dp_keys": ([C.POINTER(AmrDevProg), _vp, _vp, _vp, C.c_int, C.c_int, _vp], C.c_int),
    "amr_dp_encode": ([C.POINTER(AmrDevProg), _vp, _vp, _vp, _vp, C.c_int64, _vp, _vp, _vp, C.c_int, C.c_int, _vp],
                      C.c_int),
    "amr_mesh_blocks": ([_vp, _i32p, _i32p, _i32p, _i64p, _i32p], C.c_int),
    "amr_mesh_block_gather": ([_vp, C.c_int64, _i64p, _i64p, _i64p, _i64p, _f64p], C.c_int),
    "amr_stage": ([C.POINTER(AmrStageParams), _vp], C.c_int),
    "amr_iface": ([C.POINTER(AmrStageParams), _vp], C.c_int),
    "amr_stage_params_layout": ([_i64p, C.c_int], C.c_int),
    "amr_gather_rows": ([C.c_int64, _vp, _vp, _vp, C.c_int, _vp, C.c_int64, _vp, C.c_int64, _vp], C.c_int),
    "amr_block_rhs": ([C.c_int, C.c_int, C.c_int, _vp, _vp, C.c_double, C.c_double, _vp, C.c_double,
                       C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                       C.POINTER(AmrStageParams), _vp], C.c_int),
    "amr_ghost_pack": ([C.POINTER(AmrGhostMove), _vp, _vp], C.c_int),
    "amr_ghost_unpack": ([C.POINTER(AmrGhostMove), _vp, _vp], C.c_int),
    "amr_wavelet_coeff": ([C.c_int, C.c_int, C.c_int64, _vp, _vp, _vp, C.c_int, C.c_double, C.c_double,
                           C.c_int, C.c_int, _vp, _vp, _vp], C.c_int),
}

LAYOUT_FIELDS = ["n_tiles", "heads", "max_tail", "probe", "wtab", "n_iface", "ibuf", "vt_j", "Y", "coef", "g_cstage",
                 "g_comb", "max_depth", "top_nodes", "lo", "h2_pow2", "inv_h2", "r_eps", "f0_phi", "d2c", "d1e1"]

_LIB = None


class NativeError(RuntimeError):
    pass


def lib() -> C.CDLL:
    """Load (building first if stale and nvcc is available) the native library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("AMR_LIB_PATH") or _build.LIB  # override: kernel-variant experiments (tools/)
    nvcc = os.path.exists(_build.NVCC)
    if nvcc and os.path.isdir(_build.CSRC) and not os.environ.get("AMR_LIB_PATH"):
        _build.build()
    if not os.path.exists(path):
        raise NativeError(
            f"native library {path} is missing and cannot be built (nvcc: {nvcc}); "
            "run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = C.CDLL(path)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = L
    return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().amr_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed (code {rc}): {msg}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def last_error() -> str:
    return lib().amr_last_error().decode(errors="replace")
