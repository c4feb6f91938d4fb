#!/usr/bin/env python
"""Segmentation (inference) workload of SURVEY §8(f) item 2: same-size per-pixel class
probabilities of whole images — mirror padding, the whole-image forward with
the per-pixel softmax, and the fragment -> pixel reassembly — timed on one GPU.

    python scripts/bench_segment.py --workload cfg4 [--images 8] [--steps 5]

Prints one JSON line: pixels/s (every pixel of the original images is predicted), ms per
batch, and the dominant kernel of the pass with its achieved fraction of the roofline.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import mpf_synth as S  # noqa: E402
from paper_1302_1690_b200.net import MPFNet, mirror_pad  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--images", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    cfg = S.CONFIGS[a.workload]
    n = a.images or cfg.global_batch
    im, _ = S.make_batch(cfg, list(range(n)))
    x = torch.tensor(im, device="cuda")
    H, W = cfg.H, cfg.W
    net = MPFNet(cfg.layers, cfg.P, H + cfg.P - 1, W + cfg.P - 1, max_images=n)
    net.set_params(S.init_params(cfg).astype(np.float32))

    def step():
        return net.predict(mirror_pad(x, cfg.P))

    for _ in range(a.warmup):
        out = step()
    torch.cuda.synchronize()
    assert out.shape == (n, net.geom.classes, H, W)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    net.profile_begin(200 * a.steps)
    for _ in range(a.steps):
        step()
    torch.cuda.synchronize()
    stats = sorted(net.profile_end(), key=lambda r: -r["total_ms"])
    dom = stats[0]
    avg = dom["total_ms"] / dom["launches"]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    if dom["name"].endswith("_tc"):
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * 0.5
        roof = {"bound": "tensor", "achieved": dom["flops"] / avg / 1e9, "peak": peak, "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": dom["bytes"] / avg / 1e6, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = f"{dom['name']}[layer {dom['layer']}]"
    line = {"metric": "segmented pixels/sec (mirror pad + whole-image forward + softmax + fragments->pixels)",
            "value": n * H * W / (ms / 1e3), "unit": "px/s", "ms_per_batch": ms, "images": n,
            "config": {"workload": a.workload, "image": [H, W], "patch": cfg.P, "padded": [H + cfg.P - 1, W + cfg.P - 1]},
            "dtype": "tf32", "data": "synthetic", "roofline": roof,
            "kernels": [{"name": r["name"], "layer": r["layer"], "ms": r["total_ms"] / a.steps} for r in stats[:12]]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
