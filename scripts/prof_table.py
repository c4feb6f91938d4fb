#!/usr/bin/env python
"""Print bench.py --profile-json tables: per (kernel, layer) live CUDA-event time and
achieved algorithmic TFLOP/s and GB/s."""
import json
import sys

for path in sys.argv[1:]:
    d = json.load(open(path))
    ks = sorted(d["kernels"], key=lambda r: -r["total_ms"])
    tot = sum(r["total_ms"] for r in ks)
    ov = f", overlapped step {d['overlapped_step_ms']:.3f} ms" if "overlapped_step_ms" in d else ""
    print(f"{path}: step {d['step_ms']:.3f} ms{ov}, kernels sum {tot / max(1, ks[0]['launches']):.3f} ms/step")
    for r in ks[:int(sys.argv[0] and 30)]:
        ms = r["total_ms"] / r["launches"]
        fl = r["flops"] / ms / 1e9 if r["flops"] else 0
        bw = r["bytes"] / ms / 1e6
        print(f'  {r["name"]:18s} L{r["layer"]:2d} n={r["launches"]:3d} ms={ms:8.3f} share={r["total_ms"] / tot:5.1%} '
              f'TF/s={fl:7.1f} GB/s={bw:7.0f}')
