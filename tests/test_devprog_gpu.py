"""Per-tile stage programs built on the device (csrc/amr_devprog.cu) against
the host builder (amr_programs.cpp, itself byte-identical to the numpy
statement tileprog.build_programs): heads, tails, interface pairs, weight
table and the scalar sizes must agree byte for byte, for whole meshes and for
the tile subsets of a partition, LTS and GTS."""
import time

import numpy as np
import pytest

from helpers import config_mesh

from paper_2011_10570_b200 import tileprog

pytestmark = pytest.mark.gpu


def _same(dev, host, nt):
    for k in ("max_head", "max_slots", "max_tail", "n_iface", "n_rows", "n_cells"):
        assert dev[k] == host[k], (k, dev[k], host[k])
    assert np.array_equal(dev["heads"].cpu().numpy()[:nt], host["heads"][:nt])
    assert dev["tail"].cpu().numpy().view(np.uint16).tobytes() == host["tail"].tobytes()
    assert np.array_equal(dev["if_gid"].cpu().numpy(), host["if_gid"])
    assert np.array_equal(dev["if_cad"].cpu().numpy(), host["if_cad"])
    assert dev["wtab"].cpu().numpy().tobytes() == host["wtab"].tobytes()


@pytest.mark.parametrize("name,lts", [("cfg1", True), ("cfg1", False), ("mini3d", True), ("cfg2", True), ("cfg2", False),
                                      ("cfg3", True)])
def test_device_programs_equal_host_programs(cuda, name, lts):
    mesh = config_mesh(name)
    lv = mesh.tree.arrays()[1].astype(np.int32)
    cad = lv if lts else np.full_like(lv, lv.max())
    tiles = np.lexsort((np.arange(len(lv)), -cad)).astype(np.int32)
    t0 = time.time()
    host = tileprog.build_programs_native(mesh, tiles, cad, lts)
    t1 = time.time()
    dev = tileprog.build_programs_device(mesh, tiles, cad, lts)
    import torch

    torch.cuda.synchronize()
    t2 = time.time()
    print(f"{name} lts={lts}: host {t1 - t0:.2f} s, device {t2 - t1:.2f} s")
    _same(dev, host, len(tiles))


def test_device_programs_of_a_rank_subset(cuda):
    mesh = config_mesh("cfg1", ranks=3)
    lv = mesh.tree.arrays()[1].astype(np.int32)
    for a, b in mesh.pmap.rank_ranges:
        own = np.arange(a, b)
        tiles = own[np.lexsort((own, -lv[own]))].astype(np.int32)
        _same(tileprog.build_programs_device(mesh, tiles, lv, True), tileprog.build_programs_native(mesh, tiles, lv, True),
              len(tiles))


def test_device_programs_refuse_unencodable_meshes(cuda, monkeypatch):
    monkeypatch.setenv("AMR_MAX_BASES", "1")
    mesh = config_mesh("cfg1")
    lv = mesh.tree.arrays()[1].astype(np.int32)
    tiles = np.lexsort((np.arange(len(lv)), -lv)).astype(np.int32)
    with pytest.raises(ValueError, match="source groups"):
        tileprog.build_programs_device(mesh, tiles, lv, True)
