#!/usr/bin/env python
"""Summarise an `ncu --page raw --csv` export (optionally .gz): per launch, duration,
DRAM traffic and throughput, tensor-pipe activity, occupancy and the top stall reasons.

    python scripts/ncu_summary.py gpurun_out/ncu_cfg5_raw.csv.gz [--stalls]
"""
import argparse
import csv
import gzip
import io
import sys


def load(path):
    f = io.TextIOWrapper(gzip.open(path), "utf-8") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    hdr = rows[0]
    return hdr, rows[1], rows[2:]


def num(s):
    try:
        return float(s.replace(",", ""))
    except Exception:
        return float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--stalls", action="store_true")
    a = ap.parse_args()
    hdr, units, rows = load(a.csv)
    ix = {h: i for i, h in enumerate(hdr)}
    scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
             "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def g(r, k):
        if k not in ix:
            return float("nan")
        return num(r[ix[k]]) * scale.get(units[ix[k]], 1.0)

    print(f"# {a.csv}")
    print(f"{'#':>3s} {'kernel':34s} {'grid':>14s} {'us':>9s} {'DRAM MB':>9s} {'GB/s':>7s} {'dram%':>6s} "
          f"{'tc%':>6s} {'sm%':>6s} {'occ%':>6s} {'regs':>5s}")
    for n, r in enumerate(rows):
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("mpf::", "")
        name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")[:34]
        us = g(r, "gpu__time_duration.sum") * 1e6
        mb = (g(r, "dram__bytes_read.sum") + g(r, "dram__bytes_write.sum")) / 1e6
        print(f"{n:3d} {name:34s} {r[ix['Grid Size']]:>14s} {us:9.1f} {mb:9.1f} {mb / max(us, 1e-9) * 1e3:7.0f} "
              f"{g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{g(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{g(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{g(r, 'launch__registers_per_thread'):5.0f}")
        if a.stalls:
            st = [(h, num(r[i])) for h, i in ix.items()
                  if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
            if not st:
                st = [(h, num(r[i])) for h, i in ix.items()
                      if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
            st = sorted([s for s in st if s[1] == s[1]], key=lambda s: -s[1])[:5]
            print("      stalls: " + ", ".join(f"{h.split('stalled_')[-1].split('.')[0]}={v:.2f}" for h, v in st))
    return 0


if __name__ == "__main__":
    sys.exit(main())
