"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel
launch counts, device time and share.  With --window solve:N the summary covers the N-th
complete paraexp_solve (each solve ends with exactly one unpack_kernel launch).
Usage: python tools/launch_summary.py launches.csv [--window solve:2] > summary.csv"""
import csv
import re
import sys


def rows(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = list(csv.reader(lines))
    hdr = r[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    out = []
    for row in r[1:]:
        if row[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", row[ki]).replace("void ", "")
        out.append((name, float(row[vi].replace(",", ""))))
    return out


def main():
    path = sys.argv[1]
    win = None
    if "--window" in sys.argv:
        win = sys.argv[sys.argv.index("--window") + 1]
    L = rows(path)
    if win and win.startswith("solve:"):
        n = int(win.split(":")[1])
        ends = [q for q, (k, _) in enumerate(L) if k.startswith("pe::unpack_kernel")]
        lo = ends[n - 2] + 1 if n >= 2 else 0
        L = L[lo:ends[n - 1] + 1]
    tot = sum(t for _, t in L)
    agg = {}
    for k, t in L:
        c, s = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, s + t)
    w = csv.writer(sys.stdout)
    w.writerow(["kernel", "launches", "total_ns", "mean_ns", "share"])
    for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        w.writerow([k, c, int(s), int(s / c), f"{s / tot:.4f}"])
    print(f"# {len(L)} launches, {tot / 1e6:.3f} ms device time (ncu: serialised, cold-cache)", file=sys.stderr)


if __name__ == "__main__":
    main()
