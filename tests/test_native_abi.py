"""The C-ABI library loads on a CPU-only host and exports every symbol declared
in include/amr_b200.h (no device calls here)."""
import os
import re

from conftest import ROOT

from paper_2011_10570_b200 import _native


def _declared():
    src = open(os.path.join(ROOT, "include", "amr_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(amr_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = _native.lib()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.SIGNATURES), set(names) ^ set(_native.SIGNATURES)


def test_abi_version_and_struct_sizes():
    import ctypes

    lib = _native.lib()
    assert lib.amr_abi_version() == 1
    # AmrSliceCoef layout: 16 + 256 int32 then doubles
    assert ctypes.sizeof(_native.AmrSliceCoef) == 4 * (16 + 256) + 8 * (16 * 16 + 16 * 4 + 2 * 16 * 16 * 16 + 16 * 16 * 4)


def test_native_errors_map_to_valueerror():
    import numpy as np
    import pytest

    from paper_2011_10570_b200.mesh import Mesh
    from paper_2011_10570_b200.octree import uniform_tree

    with pytest.raises(ValueError):
        Mesh(uniform_tree(2, 2, 1), points_per_octant=6)
    with pytest.raises(ValueError):
        Mesh(uniform_tree(2, 2, 1), points_per_octant=5, pad=3)


def test_stage_params_layout_matches_ctypes():
    """The ctypes mirror of AmrStageParams has the compiled struct's size and
    field offsets (a silent mismatch would feed the kernel garbage)."""
    import ctypes

    import numpy as np

    out = np.zeros(64, dtype=np.int64)
    n = _native.lib().amr_stage_params_layout(_native.ptr(out, ctypes.c_int64), 64)
    assert n == 1 + len(_native.LAYOUT_FIELDS)
    S = _native.AmrStageParams
    assert out[0] == ctypes.sizeof(S)
    for i, f in enumerate(_native.LAYOUT_FIELDS):
        assert out[1 + i] == getattr(S, f).offset, f
