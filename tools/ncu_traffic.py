"""Write profiles/traffic.json from an ncu report of tools/profile_stage.py:
average DRAM bytes (read+write) per LTS stage launch over the profiled LTS
launches (slices 16 and 17), beside their algorithmic bytes (68 B/unit)."""
import csv
import json
import subprocess
import re
import sys


def _is_lts(name: str) -> bool:
    """stage_cross<DIM, PPO, LTS, NT, NTH, FULL> as ncu prints it (demangled forms vary)."""
    m = re.search(r"stage_(?:kernel|blob|pipe|cross)<\(?\w*\)?(\d+), \(?\w*\)?(\d+), \(?\w*\)?(\w+)", name)
    return bool(m) and m.group(3) in ("1", "true")


def _is_full(name: str) -> bool:
    args = re.search(r"stage_cross<([^>]*)>", name)
    last = args.group(1).split(",")[-1].strip() if args else "1"
    return re.sub(r"\(\w+\)", "", last) in ("1", "true")

import numpy as np


def main(rep, out="profiles/traffic.json", cfg="cfg2"):
    q = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                        "dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size"],
                       capture_output=True, text=True).stdout
    rows = list(csv.reader(q.splitlines()))
    hdr, units = rows[0], rows[1]
    i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    i_n, i_g = hdr.index("Kernel Name"), hdr.index("launch__grid_size")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    lts = []
    for r in rows[2:]:
        if _is_lts(r[i_n]):
            lts.append((float(r[i_r]) * scale[units[i_r]] + float(r[i_w]) * scale[units[i_w]], int(float(r[i_g])),
                        _is_full(r[i_n])))
    # algorithmic bytes: 68 B x owned nodes of the launched tiles.  The LTS engine launches the lean
    # kernel instance (last template argument false) on the tiles off the physical faces and the full
    # one on the rest, each group finest cadence first: a launch is a prefix of its group.
    sys.path.insert(0, ".")
    from bench import build_mesh
    from paper_2011_10570_b200.stepper import Engine

    c, mesh = build_mesh(cfg, 1, "lts")
    rk = Engine(mesh, tableau=c.tableau, cfl=c.cfl, mode="lts", nonlinear=c.nonlinear)._rank_list[0]
    counts = np.diff(mesh.leaf_starts)
    cum = np.concatenate([[0], np.cumsum(counts[rk.tiles])])

    def alg_bytes(grid, full):
        off = rk.groups[(False, full)][0]
        return 68.0 * (cum[off + grid] - cum[off])

    alg = [alg_bytes(g, f) for _, g, f in lts]
    d = {"source": rep.split("/")[-1], "config": cfg, "lts_launches": len(lts),
         "lts_bytes_per_launch": float(np.mean([b for b, _, _ in lts])),
         "lts_algorithmic_bytes_per_launch": float(np.mean(alg)),
         "ratio": float(np.sum([b for b, _, _ in lts]) / np.sum(alg))}
    json.dump(d, open(out, "w"), indent=1)
    print(d)


if __name__ == "__main__":
    main(sys.argv[1], *sys.argv[2:4])
