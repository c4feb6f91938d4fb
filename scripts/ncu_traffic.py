#!/usr/bin/env python
"""Map an `ncu --set full` capture of one training step (scripts/run_step.py, raw page
CSV) onto the library's launch order (run_step.py --order-json) and write, per
(workload, kernel, layer): DRAM bytes per launch, ncu duration, tensor-pipe and DRAM
utilisation.  Merges into profiles/ncu_traffic.json (read by bench.py) and prints a table.

    python scripts/ncu_traffic.py cfg4 gpurun_out/ncu_cfg4_raw.csv.gz gpurun_out/order_cfg4.json
"""
import csv
import gzip
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    wl, raw, order = sys.argv[1], sys.argv[2], sys.argv[3]
    f = io.TextIOWrapper(gzip.open(raw), "utf-8") if raw.endswith(".gz") else open(raw)
    rows = list(csv.reader(f))
    hdr, units, body = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def g(r, k):
        if k not in ix or r[ix[k]] in ("", "n/a"):
            return float("nan")
        return float(r[ix[k]].replace(",", "")) * SCALE.get(units[ix[k]], 1.0)

    ours = [r for r in body if not r[ix["Kernel Name"]].lstrip("void ").startswith("at::")]
    seq = json.load(open(order))
    if len(ours) != len(seq):
        print(f"warning: {len(ours)} profiled launches vs {len(seq)} library launches; mapping by order", file=sys.stderr)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    print(f"{'kernel':18s} {'L':>3s} {'ncu us':>9s} {'DRAM MB':>9s} {'alg MB':>9s} {'DRAM/alg':>8s} {'dram%':>6s} {'tc%':>6s}  name")
    # one library launch can be several kernels: the swapped-role weight gradient in passes
    # (consecutive wgrad_tc_swap_kernel launches) -> merge them into that launch's row
    merged, i = [], 0
    extra = len(ours) - len(seq)
    for name, *_ in seq:
        if i >= len(ours):
            break
        grp = [ours[i]]
        i += 1
        while (extra > 0 and name == "wgrad_tc" and i < len(ours) and "wgrad_tc_swap_kernel" in ours[i][ix["Kernel Name"]]
               and "wgrad_tc_swap_kernel" in grp[0][ix["Kernel Name"]]):
            grp.append(ours[i])
            i += 1
            extra -= 1
        merged.append(grp)
    for (name, layer, ms, flops, nbytes), grp in zip(seq, merged):
        r = grp[0]
        dram = sum(g(x, "dram__bytes_read.sum") + g(x, "dram__bytes_write.sum") for x in grp)
        us = sum(g(x, "gpu__time_duration.sum") for x in grp) * 1e6
        if len(grp) > 1:
            name_note = f" ({len(grp)} passes)"
        else:
            name_note = ""
        table[f"{wl}:{name}:{layer}"] = dram
        kn = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("mpf::", "")[:40] + name_note
        print(f"{name:18s} {layer:3d} {us:9.1f} {dram / 1e6:9.1f} {nbytes / 1e6:9.1f} {dram / max(nbytes, 1):8.2f} "
              f"{g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{g(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):6.1f}  {kn}")
    with open(path, "w") as fo:
        json.dump(table, fo, indent=1, sort_keys=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
