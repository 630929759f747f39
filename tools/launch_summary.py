"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv log) by kernel.
usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def key_of(name: str) -> str:
    m = re.search(r"(stage_cross|iface_kernel|gather_rows_kernel|block_rhs_kernel|pack_kernel)", name)
    if m:
        k = m.group(1)
        if k.startswith("stage"):
            lts = re.search(r"stage_\w+<\(?\w*\)?\d+, \(?\w*\)?\d+, \(?\w*\)?(\w+)", name)
            k += " (LTS)" if lts and lts.group(1) in ("1", "true") else " (GTS)"
        return k
    return "torch: " + name.split("(")[0].replace("void ", "").split("<")[0]


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    I = {h: i for i, h in enumerate(rows[0])}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if r[I["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = key_of(r[I["Kernel Name"]])
        tot[k] += float(r[I["Metric Value"]]) * UNIT.get(r[I["Metric Unit"]], 1.0)
        cnt[k] += 1
    T = sum(tot.values()) or 1.0
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| {k} | {cnt[k]} | {v:.0f} | {100 * v / T:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
