"""Per-phase timeline of the stage kernel (build with -DAMR_PHASE_PROBE into a
variant library, load it with AMR_LIB_PATH).  Thread 0 of every CTA stamps
%globaltimer at: 0 start, 1 head landed, 2 gathers issued, 3 gathers landed,
4 rows done, 5 own RHS done, 6 all RHS done.  Prints mean phase durations and
CTA lifetimes for one GTS stage and one LTS round-start stage on cfg2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import build_mesh  # noqa: E402
from paper_2011_10570_b200.stepper import Engine  # noqa: E402

cfg, mesh = build_mesh(os.environ.get("CFG", "cfg2"), 1, "lts")
for mode in ("gts", "lts"):
    eng = Engine(mesh, tableau="rk4", cfl=0.25, mode=mode, nonlinear=cfg.nonlinear)
    eng.initialize(cfg.chi0())
    for _ in range(eng.schedule.slices_per_round):
        eng.advance_slice()
    nt = len(eng._rank_list[0].tiles)
    buf = torch.zeros((nt, 8), dtype=torch.int64, device="cuda")
    eng._prm.probe = buf.data_ptr()
    for stage_of_interest in range(eng.p):
        buf.zero_()
        # run slices until the round start, probe stage `stage_of_interest`
        P = eng._prm
        lib = eng._lib
        orig = lib.amr_stage
        calls = []

        def hook(prm, st, orig=orig):
            calls.append(1)
            P.probe = buf.data_ptr() if len(calls) - 1 == stage_of_interest else None
            return orig(prm, st)
        eng._lib = type("L", (), {"amr_stage": staticmethod(hook), "amr_iface": staticmethod(lib.amr_iface)})()
        eng.advance_slice()
        eng._lib = lib
        torch.cuda.synchronize()
        t = buf.cpu().numpy().astype(np.float64)
        tpc = int(os.environ.get("TPC", "1"))
        idx = np.arange(len(t))
        ok = t[:, 0] > 0
        t0 = t[ok, 0].min()
        span = (t[ok, 6].max() - t0) / 1e3
        names = ["head", "gather-issue", "gather-wait", "rows", "rhs(own)", "rhs(all)"]
        for j in range(tpc):  # j-th tile of its CTA
            tj = t[ok & (idx % tpc == j)]
            life = (tj[:, 6] - tj[:, 0]) / 1e3
            d = np.diff(tj[:, :7], axis=1) / 1e3
            print(f"{mode} stage {stage_of_interest} tile {j}/{tpc}: {len(tj)} tiles, span {span:.1f} us, "
                  f"mean tile life {life.mean():.2f} us; " +
                  ", ".join(f"{n} {v:.2f}" for n, v in zip(names, d.mean(axis=0))))
    eng._prm.probe = None
