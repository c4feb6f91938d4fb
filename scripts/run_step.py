#!/usr/bin/env python
"""One training step of a BASELINE config through the C ABI, for profilers.

    python scripts/run_step.py --workload cfg5 [--warmup 1] [--images N]

The warm-up steps run outside the profiled range; the measured step is bracketed by
cudaProfilerStart/Stop (use `ncu --profile-from-start off`).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import mpf_synth as S  # noqa: E402
from paper_1302_1690_b200.net import MPFNet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--images", type=int, default=0, help="0 = the config's global batch")
    ap.add_argument("--precision", default="tf32")
    ap.add_argument("--order-json", default="", help="write the (kernel, layer) launch order of one step here")
    a = ap.parse_args()
    cfg = S.CONFIGS[a.workload]
    n = a.images or cfg.global_batch
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=n, precision=a.precision)
    net.set_params(S.init_params(cfg).astype(np.float32))
    im, lb = S.make_batch(cfg, list(range(n)))
    img = torch.tensor(im, device="cuda")
    lab = torch.tensor(lb, device="cuda")

    def step():
        net.forward(img)
        net.backward(lab)
        net.sgd_step(cfg.lr, 1.0 / n)

    for _ in range(a.warmup):
        step()
    net.check()
    torch.cuda.synchronize()
    if a.order_json:  # one extra step through the library's own launch timer (not profiled)
        import json
        net.profile_begin(1000)
        step()
        recs = net.profile_end()
        with open(a.order_json, "w") as f:
            json.dump([[r["name"], r["layer"], r["total_ms"], r["flops"], r["bytes"]] for r in recs], f)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    net.check()
    print("ok", a.workload, n)


if __name__ == "__main__":
    main()
