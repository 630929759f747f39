"""Pin the CPU oracle (oracle/, test infrastructure) against reference goldens.

The oracle is what the GPU tests compare against beyond the golden cases, and
bench.py's CPU baseline, so it must reproduce the reference bit for bit first."""
import numpy as np
import pytest

from conftest import compare_field, golden

from oracle import oracle as O
from paper_2011_10570_b200.configs import CONFIGS


def _oracle_mesh(name):
    c = CONFIGS[name]
    a, lv = O.construct(c.refine, c.dim, c.max_depth)
    pre = (a, lv)
    a, lv = O.balance(c.dim, c.max_depth, a, lv)
    return pre, (a, lv), O.OracleMesh(c.dim, c.max_depth, a, lv, c.ppo, c.pad, c.domain_lo, c.domain_hi)


@pytest.mark.parametrize("name", ["cfg1", "mini3d"])
def test_oracle_tree_and_registry(name):
    gd = golden(name)
    pre, tree, m = _oracle_mesh(name)
    assert np.array_equal(pre[0], gd["pre_anchor"]) and np.array_equal(pre[1], gd["pre_level"])
    assert np.array_equal(tree[0], gd["anchor"]) and np.array_equal(tree[1], gd["level"])
    assert m.n_nodes == int(gd["n_nodes"])
    assert np.array_equal(m.leaf_slices, gd["leaf_slices"])
    assert np.array_equal(m.leaf_gids, gd["leaf_gids"])
    assert np.array_equal(m.node_coords, gd["node_coords"])
    lr, rl, ll = m.blocks()
    assert np.array_equal(lr, gd["block_leaf_range"])
    assert np.array_equal(rl, gd["block_root_level"]) and np.array_equal(ll, gd["block_leaf_level"])


def test_oracle_gathers_cfg1():
    gd = golden("cfg1")
    _, _, m = _oracle_mesh("cfg1")
    rows = gd["g_block_rows"]
    for b in range(len(rows) - 1):
        ptr, col, val = m.block_gather(b)
        r0, r1 = rows[b], rows[b + 1]
        want_ptr = gd["g_indptr"][r0:r1 + 1]
        assert np.array_equal(ptr, want_ptr - want_ptr[0])
        assert np.array_equal(col, gd["g_indices"][want_ptr[0]:want_ptr[-1]])
        assert np.array_equal(val.view(np.int64), gd["g_data"][want_ptr[0]:want_ptr[-1]].view(np.int64))


def test_oracle_partition():
    gd = golden("cfg1")
    for k in gd.files:
        if k.startswith("part_"):
            _, mode, R = k.split("_")
            assert np.array_equal(np.array(O.partition(gd["level"], int(R), mode)), gd[k])


@pytest.mark.parametrize("name,tag,tab,mode,nl", [
    ("cfg1", "gts_rk4", "rk4", "gts", False), ("cfg1", "lts_rk4", "rk4", "lts", False),
    ("cfg1", "lts_cubic", "rk4", "lts", "cubic"), ("cfg1", "gts_cubic", "rk4", "gts", "cubic"),
    ("cfg1", "lts_rk3", "rk3", "lts", False), ("cfg1", "lts_sin", "rk4", "lts", "sin"),
    ("mini3d", "gts_rk4", "rk4", "gts", False), ("mini3d", "lts_rk4", "rk4", "lts", False),
    ("mini3d", "lts_cubic", "rk4", "lts", "cubic"),
])
def test_oracle_fields_bit_exact(name, tag, tab, mode, nl):
    gd = golden(name)
    _, _, m = _oracle_mesh(name)
    e = O.OracleEngine(m, tab, 0.25, mode, nl)
    e.initialize(CONFIGS[name].chi0())
    assert e.dt_fine == float(gd[f"{tag}_dt_fine"])
    cps = sorted({int(k[len(tag) + 2:].split("__")[0]) for k in gd.files if k.startswith(tag + "_i")})
    for cp in cps:
        e.run_to(cp)
        exact, rel = compare_field(e.current_zip(), gd, f"{tag}_i{cp}")
        assert rel <= 1e-12, (cp, rel)
        if nl != "sin":  # glibc sin vs numpy's vectorised sin may differ by an ulp
            assert exact, (cp, rel)


def test_oracle_reference_test_geometry():
    """[-10,10]^2 ball tree, ppo 5, rk3/rk2/euler (non-dyadic h)."""
    from paper_2011_10570_b200.wave import gaussian_pulse

    gd = golden("small")
    m = O.OracleMesh(2, 4, gd["ball_anchor"], gd["ball_level"], 5, 2, (-10.0, -10.0), (10.0, 10.0))
    for tag, tab, mode, nl in [("lts_rk3", "rk3", "lts", False), ("gts_rk3", "rk3", "gts", False),
                               ("lts_rk2", "rk2", "lts", False), ("lts_euler", "euler", "lts", False),
                               ("lts_cubic", "rk4", "lts", "cubic")]:
        e = O.OracleEngine(m, tab, 0.25, mode, nl)
        e.initialize(gaussian_pulse((0.0, 0.0), 0.8, 1.0))
        for cp in sorted({int(k[len("ball_" + tag) + 2:]) for k in gd.files
                          if k.startswith(f"ball_{tag}_i")}):
            e.run_to(cp)
            exact, rel = compare_field(e.current_zip(), gd, f"ball_{tag}_i{cp}")
            assert exact, (tag, cp, rel)
