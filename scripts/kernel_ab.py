#!/usr/bin/env python
"""A/B of kernel-selection flags (MPF_FLAG_*): per-kernel live CUDA-event times of the same
training step under each flag set.  Usage:
    python scripts/kernel_ab.py --workload cfg4 --flags 0 256 --match head wgrad
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import mpf_synth as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--flags", type=lambda s: int(s, 0), nargs="+", default=[0])
    ap.add_argument("--match", nargs="*", default=[])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--json", default="")
    ap.add_argument("--images", type=int, default=0, help="0 = the config's global batch")
    a = ap.parse_args()
    import torch
    from paper_1302_1690_b200 import _lib as L
    from paper_1302_1690_b200.net import MPFNet
    cfg = S.CONFIGS[a.workload]
    B = a.images or cfg.global_batch
    im, lb = S.make_batch(cfg, list(range(B)))
    img, lab = torch.tensor(im, device="cuda"), torch.tensor(lb, device="cuda")
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=B)
    net.set_params(S.init_params(cfg).astype(np.float32))
    out = {}
    for fl in a.flags:
        net.set_flags(fl | L.MPF_FLAG_SERIAL)
        for _ in range(2):
            net.train_step(img, lab)
        torch.cuda.synchronize()
        net.profile_begin(100000)
        for _ in range(a.steps):
            net.train_step(img, lab)
        torch.cuda.synchronize()
        st = net.profile_end()
        rows = sorted(st, key=lambda r: -r["total_ms"])
        tot = sum(r["total_ms"] for r in rows) / a.steps
        print(f"{a.workload} flags=0x{fl:x}: kernels {tot:.3f} ms/step")
        for r in rows:
            if a.match and not any(m in r["name"] for m in a.match):
                continue
            ms = r["total_ms"] / r["launches"]
            extra = f"{r['flops'] / ms / 1e9:7.1f} TF/s" if r["name"].endswith("_tc") else f"{r['bytes'] / ms / 1e6:7.0f} GB/s"
            print(f"   {r['name']:18s} L{r['layer']:2d} {ms:8.3f} ms  {extra}")
        out[hex(fl)] = {"step_ms": tot, "kernels": rows}
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
