"""Per-phase cycle counts of the persistent stage kernel (debug counters, P.dbg).

Runs cfg2 (or --config), warms one GTS step and one LTS round, then runs one
GTS stage-1 launch with the counters on and prints, per phase, the mean and
max over warps of cycles per tile:
  issue (heads + gathers of j+2), wait (tile j+1 landed), syncA, rows (j+1),
  rhs (j), syncB."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

os.environ["AMR_KERNEL"] = "1"  # the probe instruments the persistent pipelined kernel

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import build_mesh  # noqa: E402
from paper_2011_10570_b200.stepper import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--mode", default="gts")
ap.add_argument("--skip", type=int, default=0, help="ablation bits: 1 gathers, 2 rows, 4 RHS (results invalid)")
args = ap.parse_args()
cfg, mesh = build_mesh(args.config, 1, "lts")
eng = Engine(mesh, tableau="rk4", cfl=0.25, mode=args.mode, nonlinear=cfg.nonlinear)
eng.initialize(cfg.chi0())
eng.use_graphs = False
eng.advance_slice()
torch.cuda.synchronize()
NW = 16
buf = torch.zeros((148 * 4 * NW, 8), dtype=torch.int64, device="cuda")
eng._prm.dbg = buf.data_ptr()
eng._prm.dbg_skip = args.skip
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
eng.advance_slice()
ev[1].record()
torch.cuda.synchronize()
eng._prm.dbg = None
eng._prm.dbg_skip = 0
print(f"slice time {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (skip={args.skip})")
b = buf.cpu().numpy()
b = b[b[:, 6] > 0]
names = ["issue", "wait", "syncA", "rows", "rhs", "syncB"]
# summed over the slice's stage launches
per = b[:, :6] / b[:, 6:7]
print("warps", len(b), "tiles/CTA", b[:, 6].mean())
for i, nm in enumerate(names):
    print(f"{nm:6s} mean {per[:, i].mean():8.0f}  max {per[:, i].max():8.0f}  cycles/tile")
print("total  mean", per.sum(1).mean())
w = np.arange(len(b)) % NW
print("per warp index (cycles/tile): issue wait rows rhs syncB")
for i in range(NW):
    m = per[w == i].mean(0)
    print(f"  warp {i:2d}: " + " ".join(f"{m[k]:6.0f}" for k in (0, 1, 3, 4, 5)))
