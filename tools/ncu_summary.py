"""Summarise an ncu --set full report (.ncu-rep) into the numbers DESIGN.md / bench.py use:
per launch duration, DRAM read/write bytes, achieved DRAM GB/s, shared-memory wavefronts and
bank conflicts, occupancy.  Usage: python tools/ncu_summary.py rep.ncu-rep [algorithmic_bytes]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"us": 1e-6, "ns": 1e-9, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    out = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = float(row[i].replace(",", "")) if row[i] not in ("", "n/a") else None
                u = units[i]
                if v is not None and u in SCALE:
                    v *= SCALE[u]
                    u = "s" if u in ("us", "ns", "ms") else "B"
                d[k] = v
        t, rd, wr = d["gpu__time_duration.sum"], d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        d["dram_bytes"] = rd + wr
        d["dram_GBps"] = (rd + wr) / t / 1e9
        if alg:
            d["algorithmic_bytes"] = alg
            d["traffic_over_algorithmic"] = (rd + wr) / alg
            d["algorithmic_GBps"] = alg / t / 1e9
        out.append(d)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
