#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
`bench.py --steps 1 --warmup W --no-graph ...`: per kernel, launches per step
(= launches / runs), mean duration and share of the serialised step.

usage: summarize_launches.py launches.csv RUNS [title] [KEY=label1,label2,...]
The optional KEY=labels splits a kernel that runs several times per layer
(e.g. grouped_gemm_kernel=QKV+RoPE,O-proj,GEMM1,GEMM2): its i-th launch gets
label i % len(labels)."""

import csv
import sys
from collections import OrderedDict


def main():
    path, runs = sys.argv[1], int(sys.argv[2])
    title = sys.argv[3] if len(sys.argv) > 3 else ""
    split_key, split_labels = None, []
    if len(sys.argv) > 4 and "=" in sys.argv[4]:
        split_key, lab = sys.argv[4].split("=", 1)
        split_labels = lab.split(",")
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
        name = r["Kernel Name"]
        if name.startswith("at::") or name.startswith("void at::") or "pack_w13" in name:
            continue  # torch set-up kernels (weights, inputs) and weight packing: not in the step
        rows.append((name, us))
    agg = OrderedDict()
    seen = 0
    for name, us in rows:
        short = name.split("(")[0].replace("void ", "").replace("msi::", "").replace("(anonymous namespace)::", "")
        if split_key and split_key in short:
            short = f"{short} [{split_labels[seen % len(split_labels)]}]"
            seen += 1
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(v[1] for v in agg.values()) / runs
    if title:
        print(f"# {title}")
    print(f"# {len(rows)} launches over {runs} runs; serialised cold-cache ncu durations")
    print(f"{'kernel':<60} {'n/step':>7} {'avg_us':>9} {'share':>7}")
    for k, (n, t) in agg.items():
        print(f"{k[:60]:<60} {n / runs:>7.2f} {t / n:>9.1f} {100 * t / runs / total:>6.1f}%")
    print(f"{'step total (serialised)':<60} {'':>7} {total:>9.1f}")


if __name__ == "__main__":
    main()
