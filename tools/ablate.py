"""Ablation timing of the stage kernel (results invalid by construction):
GTS slice time on cfg2 with field gathers (1), hanging-row sums (2) and the
RHS/epilogue (4) switched off in any combination (P.dbg_skip).
The per-tile kernel's ablation hooks are compiled only with -DAMR_ABLATE:
  AMR_NVCC_FLAGS=-DAMR_ABLATE python -m paper_2011_10570_b200.build --force
  python tools/ablate.py [--kernel 0|1] [--mode gts|lts]
  python -m paper_2011_10570_b200.build --force      # back to the product build"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--kernel", default="0")
ap.add_argument("--mode", default="gts")
ap.add_argument("--config", default="cfg2")
args = ap.parse_args()
os.environ["AMR_KERNEL"] = args.kernel

import torch  # noqa: E402

from bench import build_mesh  # noqa: E402
from paper_2011_10570_b200.stepper import Engine  # noqa: E402

cfg, mesh = build_mesh(args.config, 1, "lts")
eng = Engine(mesh, tableau="rk4", cfl=0.25, mode=args.mode, nonlinear=cfg.nonlinear)
eng.initialize(cfg.chi0())
eng.use_graphs = False
R = eng.schedule.slices_per_round if args.mode == "lts" else 4
for _ in range(R):
    eng.advance_slice()
torch.cuda.synchronize()
for skip in (0, 1, 2, 4, 3, 5, 6, 7):
    eng._prm.dbg_skip = skip
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(R):  # warm
        eng.advance_slice()
    ev[0].record()
    for _ in range(R):
        eng.advance_slice()
    ev[1].record()
    torch.cuda.synchronize()
    print(f"kernel {args.kernel} {args.mode} skip={skip}: {ev[0].elapsed_time(ev[1]) * 1e3 / R:8.1f} us per slice")
eng._prm.dbg_skip = 0
