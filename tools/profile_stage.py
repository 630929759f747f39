"""Short driver for ncu: 1 warm LTS round + 1 GTS step, then the profiled
launches between cudaProfilerStart/Stop (run ncu with --profile-from-start off):
an LTS round start (all tiles), the next LTS slice (finest level only) and a
GTS step.  Run plain first, then under ncu (see profiles/README.md)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import build_mesh  # noqa: E402
from paper_2011_10570_b200.stepper import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
args = ap.parse_args()
cfg, mesh = build_mesh(args.config, 1, "lts")
lts = Engine(mesh, tableau="rk4", cfl=0.25, mode="lts", nonlinear=cfg.nonlinear)
gts = Engine(mesh, tableau="rk4", cfl=0.25, mode="gts", nonlinear=cfg.nonlinear)
for e in (lts, gts):
    e.initialize(cfg.chi0())
lts.lts_coarse_step()   # 16 slices x 4 launches
gts.gts_step()          # 4 launches
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off: only the launches below are profiled
lts.advance_slice()     # round start: all tiles (cfg2: 4 launches of the full instance, face tiles first; cfg3/cfg4: 4 lean + 4 full)
lts.advance_slice()     # next slice: finest level only (4 launches)
gts.gts_step()          # all tiles, GTS kernel (4 launches)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", mesh.n_nodes)
