"""cfg5 on one GPU: the weighted-Morton R-rank engine (simulated ranks) against the
single-rank engine, bit for bit, after a few LTS slices.  The engines are built one
after the other (each holds ~85 GB).  Usage: python tools/cfg5_ranks.py [config] [R] [slices]"""
import gc
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import build_mesh  # noqa: E402
from paper_2011_10570_b200.stepper import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n_sl = int(sys.argv[3]) if len(sys.argv) > 3 else 4
digests = []
for ranks in (1, R):
    t0 = time.time()
    cfg, mesh = build_mesh(name, ranks, "lts")
    eng = Engine(mesh, tableau=cfg.tableau, cfl=cfg.cfl, mode="lts", nonlinear=cfg.nonlinear)
    eng.initialize(cfg.chi0(), device_eval=True)
    t1 = time.time()
    for _ in range(n_sl):
        eng.advance_slice()
    z = eng.current_zip_device()
    torch.cuda.synchronize()
    h = hashlib.sha256((z.cpu().numpy() + 0.0).tobytes()).hexdigest()
    digests.append(h)
    ghosts = sum(len(rk.ghosts) for rk in eng._rank_list)
    local = sum(rk.n_local for rk in eng._rank_list)
    print(f"{name} R={ranks}: setup {t1 - t0:.1f} s, {len(mesh.tree)} leaves, {mesh.n_nodes} nodes, local nodes over ranks "
          f"{local} ({local / mesh.n_nodes:.3f}x), ghost leaves {ghosts}, ghost bytes shipped {eng.comm_bytes}, "
          f"{n_sl} slices, sha256 {h[:16]}", flush=True)
    del eng, z, mesh
    gc.collect()
    torch.cuda.empty_cache()
print("bit-identical" if digests[0] == digests[1] else "MISMATCH")
sys.exit(0 if digests[0] == digests[1] else 1)
