"""Small driver for compute-sanitizer (tools/sanitize.sh): one eager LTS round of
cfg1 (single rank and 2 simulated ranks, cubic source), one GTS step, the
device octree build, and the wavelet criterion on the result."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import torch  # noqa: E402
from helpers import config_mesh  # noqa: E402

from paper_2011_10570_b200.configs import CONFIGS  # noqa: E402
from paper_2011_10570_b200.stepper import Engine  # noqa: E402
from paper_2011_10570_b200.wavelet import RefinePolicy  # noqa: E402

c = CONFIGS["cfg1"]
for ranks in (1, 2):
    mesh = config_mesh("cfg1", ranks=ranks)  # device construct + balance
    eng = Engine(mesh, tableau="rk4", cfl=c.cfl, mode="lts", nonlinear="cubic")
    eng.use_graphs = False
    eng.initialize(c.chi0())
    eng.lts_coarse_step()
    z = eng.current_zip()
g = Engine(config_mesh("cfg1"), tableau="rk4", cfl=c.cfl, mode="gts")
g.initialize(c.chi0())
g.gts_step()
coeff, codes = eng.wavelet_flags(RefinePolicy(tolerance=1e-3, min_level=3, max_level=6))
torch.cuda.synchronize()
print("ok", float(abs(z).max()), int((codes != 0).sum()))
