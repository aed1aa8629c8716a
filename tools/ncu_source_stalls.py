"""Summarise `ncu --page source --csv` (SASS view with warp-stall sampling) per kernel: total
samples by stall reason and the hottest instructions.  Usage: python tools/ncu_source_stalls.py
file.csv[.gz] [kernel-substring] [top]"""
import csv
import gzip
import io
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    rows = list(csv.reader(io.StringIO(raw)))
    kernels, cur = [], None
    i = 0
    while i < len(rows):
        r = rows[i]
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "hdr": rows[i + 1], "rows": []}
            kernels.append(cur)
            i += 2
            continue
        if cur is not None and r:
            cur["rows"].append(r)
        i += 1
    seen = set()
    for k in kernels:
        if want not in k["name"] or k["name"] in seen:
            continue
        seen.add(k["name"])
        hdr = k["hdr"]
        stall_cols = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        tot = defaultdict(float)
        insts = []
        si = hdr.index("Warp Stall Sampling (All Samples)")
        for r in k["rows"]:
            try:
                s = float(r[si])
            except (ValueError, IndexError):
                continue
            for j in stall_cols:
                try:
                    tot[hdr[j]] += float(r[j])
                except ValueError:
                    pass
            insts.append((s, r[0], r[1].strip(), {hdr[j][6:]: r[j] for j in stall_cols if r[j] not in ("0", "")}))
        total = sum(tot.values())
        print(f"== {k['name'][:120]}\n   samples {total:.0f}, instructions {len(insts)}")
        for n, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
            print(f"   {n:28s} {v / total * 100:5.1f}%")
        print("   hottest instructions:")
        for s, addr, src, st in sorted(insts, key=lambda x: -x[0])[:top]:
            print(f"   {s / total * 100:5.2f}%  {src[:58]:58s} {st}")


if __name__ == "__main__":
    main()
