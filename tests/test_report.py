"""CSV schemas of SPEC.md:217,449,564 (host side; the phase profile runs in test_ranks_gpu.py)."""
import numpy as np

from helpers import config_mesh

from paper_2011_10570_b200 import report
from paper_2011_10570_b200.perfmodel import estimate, histogram_from_mesh


def test_partition_and_estimate_rows_roundtrip():
    mesh = config_mesh("cfg1", ranks=4)
    rows = report.partition_rows(mesh)
    assert [r[0] for r in rows] == [0, 1, 2, 3]
    assert sum(r[1] for r in rows) == len(mesh.tree)
    assert np.isclose(sum(r[2] for r in rows), float(np.sum(mesh.pmap.weights)))
    text = report.to_csv(report.PARTITION, rows)
    hdr, back = report.parse_csv(text)
    assert hdr == ["rank", "octants", "weight"]
    assert [float(b[2]) for b in back] == [r[2] for r in rows]  # lossless
    e = estimate(histogram_from_mesh(mesh.blocks))
    row = report.estimate_row(mesh)
    assert row == (3, e.w_lts, e.w_gts, e.speedup, e.bound)
    hdr, back = report.parse_csv(report.to_csv(report.ESTIMATE, [row]))
    assert hdr == list(report.ESTIMATE) and float(back[0][3]) == e.speedup


def test_headers_match_spec():
    assert report.TIME_SERIES == ("step", "time", "l2", "linf")
    assert report.PHASES == ("ranks", "blk_sync", "time_interp", "rhs", "comm")
    assert report.WORK == ("level", "alpha", "steps")
