"""Per-CUDA-source-line instruction and stall-sample totals of one profiled launch.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX SKIP [TOP]
(needs a report captured with --import-source on from a -lineinfo build)."""
import csv
import subprocess
import sys


def main(path, regex, skip, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                          "--launch-skip", str(skip), "--launch-count", "1", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    data = []
    fname = ""
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ie = hdr.index("Instructions Executed")
            ss = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue
        try:
            data.append((float(r[ie]), float(r[ss]), f"{fname}:{r[0]}", r[1]))
        except ValueError:
            pass
    ti = sum(d[0] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")
    print("  inst%  stall%  line  source")
    for d in sorted(data, key=lambda d: -(d[0] / ti + d[1] / ts))[:top]:
        print(f"{100 * d[0] / ti:6.1f} {100 * d[1] / ts:6.1f}  {d[2]:>22}  {d[3].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 40)
