#!/usr/bin/env python
"""Hot SASS lines of an `ncu --page source --csv --print-source sass` export (.gz ok):
top instructions by warp-stall samples, with a little context."""
import csv
import gzip
import io
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = io.TextIOWrapper(gzip.open(path), "utf-8") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
print(rows[0][1][:100])
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) > ix["Instructions Executed"] and r[ix["Warp Stall Sampling (All Samples)"]].isdigit()]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
print("total samples", tot)
hot = sorted(range(len(body)), key=lambda i: -int(body[i][ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]
for i in sorted(hot):
    r = body[i]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{i:5d} {s:7d} {100.0 * s / max(tot, 1):5.1f}%  ex={r[ix['Instructions Executed']]:>9s}  {r[ix['Source']].strip()[:90]}")
