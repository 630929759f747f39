"""Emit the reference's CSV reports (paper_2011_10570_b200/report.py)
for one config: phases.csv (device ms per phase bucket for R = 1, 2, 4, 8 simulated ranks
over a few LTS rounds), work.csv, partition.csv, estimate.csv, and series.csv (LTS vs
GTS: step,time,l2,linf of chi, the Table-1-shaped comparison).
Usage: python tools/report_csv.py [config] [out_dir] [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import build_mesh  # noqa: E402
from paper_2011_10570_b200 import report  # noqa: E402
from paper_2011_10570_b200.stepper import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
os.makedirs(out, exist_ok=True)
phases, work, part, est = [], None, None, None
for R in (1, 2, 4, 8):
    cfg, mesh = build_mesh(name, R, "lts")
    eng = Engine(mesh, tableau=cfg.tableau, cfl=cfg.cfl, mode="lts", nonlinear=cfg.nonlinear, profile=True)
    eng.initialize(cfg.chi0())
    eng.lts_coarse_step()  # warm
    eng.phase_ms()
    eng.counters.phases.clear()
    eng.counters.reset_work()
    for _ in range(rounds):
        eng.lts_coarse_step()
    phases.append(report.phase_row(eng))
    if R == 8:
        work, part, est = report.work_rows(eng), report.partition_rows(mesh), report.estimate_row(mesh)
cfg, mesh = build_mesh(name, 1, "lts")
lts = Engine(mesh, tableau=cfg.tableau, cfl=cfg.cfl, mode="lts", nonlinear=cfg.nonlinear)
gts = Engine(mesh, tableau=cfg.tableau, cfl=cfg.cfl, mode="gts", nonlinear=cfg.nonlinear)
series = []
for e in (lts, gts):
    e.initialize(cfg.chi0())
for _ in range(rounds):
    lts.lts_coarse_step()
    gts.run_to(lts.i_fine)
    series.append(report.time_series_row(lts, gts.current_zip()))
for fn, hdr, rows in (("phases", report.PHASES, phases), ("work", report.WORK, work), ("partition", report.PARTITION, part),
                      ("estimate", report.ESTIMATE, [est]), ("series", report.TIME_SERIES, series)):
    with open(os.path.join(out, f"{name}_{fn}.csv"), "w") as f:
        f.write(report.to_csv(hdr, rows))
    print(fn, rows if fn != "work" else rows[:3])
