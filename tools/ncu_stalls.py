"""Top stall reasons and hottest SASS lines of one profiled launch (ncu source page)."""
import collections
import csv
import subprocess
import sys


def main(path, regex, skip):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                          "--launch-skip", str(skip), "--launch-count", "1", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    print(rows[0][:2])
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    S = idx["Warp Stall Sampling (All Samples)"]
    data = [r for r in rows[2:] if len(r) > S and r[S].isdigit()]
    seen = set()
    uniq = []
    for r in data:
        if r[0] in seen:
            continue
        seen.add(r[0])
        uniq.append(r)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    for r in uniq:
        for s in stalls:
            try:
                tot[s] += int(r[idx[s]])
            except ValueError:
                pass
    T = sum(tot.values()) or 1
    print("stalls:", ", ".join(f"{s[6:]} {100 * c / T:.0f}%" for s, c in tot.most_common(8)))
    for r in sorted(uniq, key=lambda r: -int(r[S]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 12]:
        top = max(stalls, key=lambda s: int(r[idx[s]]) if r[idx[s]].isdigit() else 0)
        print(f"{r[S]:>6} {r[1].strip()[:64]:64s} {top[6:]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]))
