"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv log) by kernel.
usage: python tools/launch_summary.py launches.csv

Kernels are grouped: "step" = what a timed bench step launches (stage kernel, LTS
interface pass, ghost moves), "setup" = the one-off tree / mesh / program builders,
"torch" = library kernels (state copies, prefix sums, sorts, the wavelet side line)."""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
STEP = ("stage_cross", "iface_kernel", "ghost_move_kernel")
SETUP = ("ownership_kernel", "owned_gids_kernel", "shared_gids_kernel", "table_kernel", "hang_list_kernel",
         "table_rows_kernel", "rows_kernel", "need_kernel", "keys_kernel", "encode_kernel", "octants_kernel",
         "split_kernel", "balance_mark_kernel")
OURS = STEP + SETUP + ("gather_rows_kernel", "block_rhs_kernel", "wavelet_kernel")


def key_of(name: str):
    m = re.search("(" + "|".join(OURS) + ")", name)
    if m:
        k = m.group(1)
        group = "step" if k in STEP else "setup" if k in SETUP else "api"
        if k == "stage_cross":
            lts = re.search(r"stage_cross<\(?\w*\)?\d+, \(?\w*\)?\d+, \(?\w*\)?(\w+)", name)
            k += " (LTS)" if lts and lts.group(1) in ("1", "true") else " (GTS)"
        return group, k
    short = name.split("(")[0].replace("void ", "")
    return "torch", "torch: " + (short.split("<")[0] or short)[:60]


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
    gsum = collections.Counter()
    for (g, _), v in tot.items():
        gsum[g] += v
    T = sum(tot.values()) or 1.0
    print("| group | kernel | launches | total us | share of all | share of group |\n|---|---|---|---|---|---|")
    for (g, k), v in sorted(tot.items(), key=lambda kv: (-gsum[kv[0][0]], -kv[1])):
        print(f"| {g} | {k} | {cnt[(g, k)]} | {v:.0f} | {100 * v / T:.1f}% | {100 * v / gsum[g]:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
