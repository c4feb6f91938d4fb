#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration.sum per launch, --csv) by kernel.

    python scripts/summarize_launches.py gpurun_out/launches_cfg4.csv [--skip-prefix at::]

ncu's per-launch times are cold-cache and serialised: compare each kernel's SHARE of
the step with the share bench.py measures live (CUDA events), not the absolutes.
"""
import argparse
import collections
import csv
import sys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--skip-prefix", default="void at::", help="drop torch's own kernels (allocator fills)")
    a = ap.parse_args()
    rows = []
    with open(a.csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if a.skip_prefix and name.startswith(a.skip_prefix):
            continue
        short = name.split("(")[0].replace("void ", "").replace("mpf::", "").replace("(anonymous namespace)::", "")
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        rows.append((short, r["Grid Size"], r["Block Size"], ns))
    agg = collections.OrderedDict()
    for short, grid, block, ns in rows:
        e = agg.setdefault(short, [0, 0.0])
        e[0] += 1
        e[1] += ns
    tot = sum(v[1] for v in agg.values())
    print(f"# {a.csv}: {len(rows)} launches of this repo's kernels, {tot / 1e6:.3f} ms total (cold-cache, serialised)")
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:8d} {ns / 1e6:10.3f} {ns / tot:7.1%}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
