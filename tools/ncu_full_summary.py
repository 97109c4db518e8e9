#!/usr/bin/env python
"""Key metrics of ncu --set full captures (one row per captured launch) as CSV.
Usage: python tools/ncu_full_summary.py rep1.ncu-rep [rep2 ...] > summary.csv"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]


def main():
    w = csv.writer(sys.stdout)
    w.writerow(["report", "kernel"] + METRICS)
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if not rows:
            continue
        h = rows[0]
        idx = {m: h.index(m) for m in METRICS if m in h}
        units = rows[1]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")][:60]
            w.writerow([rep.split("/")[-1], name] +
                       [f"{r[idx[m]]} {units[idx[m]]}".strip() if m in idx else "" for m in METRICS])


if __name__ == "__main__":
    main()
