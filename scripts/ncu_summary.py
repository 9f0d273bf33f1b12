#!/usr/bin/env python
"""Key metrics of ncu --set full reports (one line per metric and launch).
usage: ncu_summary.py LABEL=report.ncu-rep[:launch_labels,...] ..."""

import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__registers_per_thread"]


def main():
    for arg in sys.argv[1:]:
        label, rest = arg.split("=", 1)
        path, _, labs = rest.partition(":")
        labels = labs.split(",") if labs else []
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for k, vals in enumerate(rows[2:]):
            name = labels[k] if k < len(labels) else f"{label}#{k}"
            for m in METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    print(f"{name:<14} {m:<70} {vals[i]:>14} {units[i]}")


if __name__ == "__main__":
    main()
