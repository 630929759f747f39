"""Summarise an ncu report: one row per profiled launch (duration, DRAM bytes, throughput, occupancy)."""
import csv
import subprocess
import re
import sys


def _is_lts(name: str) -> bool:
    """stage_{kernel,blob,pipe}<DIM, PPO, LTS, NT> as ncu prints it (demangled forms vary)."""
    m = re.search(r"stage_(?:kernel|blob|pipe|cross)<\(?\w*\)?(\d+), \(?\w*\)?(\d+), \(?\w*\)?(\w+)", name)
    return bool(m) and m.group(3) in ("1", "true")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "lts__t_sector_hit_rate.pct",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    print("| # | kernel | grid | regs | time us | DRAM rd MB | DRAM wr MB | DRAM % | L2 hit % | L1 hit % | SM % | warps % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for n, r in enumerate(rows[2:]):
        name = r[idx["Kernel Name"]]
        lts = _is_lts(name)
        args = re.search(r"stage_cross<([^>]*)>", name)
        last = re.sub(r"\(\w+\)", "", args.group(1).split(",")[-1].strip()) if args else "1"
        short = "stage" + ("_lts" if lts else "_gts") + ("" if last in ("1", "true") else "_lean")
        def g(m, scale=1.0):
            try:
                return float(r[idx[m]]) * scale
            except (KeyError, ValueError):
                return float("nan")
        unit_t = rows[1][idx["gpu__time_duration.sum"]]
        t = g("gpu__time_duration.sum") * (1000.0 if unit_t == "ms" else 1.0)
        ur = rows[1][idx["dram__bytes_read.sum"]]
        sc = {"Gbyte": 1000.0, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}.get(ur, 1.0)
        uw = rows[1][idx["dram__bytes_write.sum"]]
        sw = {"Gbyte": 1000.0, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}.get(uw, 1.0)
        print(f"| {n} | {short} | {int(g('launch__grid_size'))} | {int(g('launch__registers_per_thread'))} | {t:.1f} | "
              f"{g('dram__bytes_read.sum', sc):.1f} | {g('dram__bytes_write.sum', sw):.1f} | "
              f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | {g('lts__t_sector_hit_rate.pct'):.1f} | "
              f"{g('l1tex__t_sector_hit_rate.pct'):.1f} | {g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
