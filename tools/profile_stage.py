"""Short driver for ncu: cfg2 mesh, 1 warm LTS round + 1 GTS step, then
`--n` profiled slices (LTS slice 0 = all tiles, LTS slice 1 = finest only,
GTS step).  Run plain first, then under ncu (see profiles/README.md)."""
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
lts.advance_slice()     # slice 16 = round start: all tiles (profiled: launches 68..71)
lts.advance_slice()     # slice 17: finest level only (72..75)
gts.gts_step()          # all tiles, GTS kernel (76..79)
torch.cuda.synchronize()
print("ok", mesh.n_nodes)
