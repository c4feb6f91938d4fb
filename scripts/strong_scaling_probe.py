#!/usr/bin/env python
"""Per-GPU step time at the per-GPU batch of an N-GPU run with a fixed global batch
(strong scaling, R14): time one GPU's share (B_g / N images) and report the implied
scaling efficiency t(B_g) / (N * t(B_g / N)), allreduce excluded (one 2.2 MB NCCL call).

    python scripts/strong_scaling_probe.py --workload cfg4
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


def time_step(cfg, n, steps=5, warmup=3, graph=False):
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=n)
    net.set_params(S.init_params(cfg).astype(np.float32))
    im, lb = S.make_batch(cfg, list(range(n)))
    img, lab = torch.tensor(im, device="cuda"), torch.tensor(lb, device="cuda")

    def step():
        net.train_step(img, lab)
        net.sgd_step(cfg.lr, 1.0 / n)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    run = step
    if graph:  # the whole step replayed as one CUDA graph (bench.py's timed loop)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        g.replay()
        torch.cuda.synchronize()
        run = g.replay
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays of the step")
    a = ap.parse_args()
    cfg = S.CONFIGS[a.workload]
    B = cfg.global_batch
    t_full = time_step(cfg, B, graph=a.graph)
    for N in (2, 4, 8):
        t = time_step(cfg, B // N, graph=a.graph)
        print(f"{a.workload}{' (graph)' if a.graph else ''}: N={N} per-GPU {B // N} images {t:.3f} ms vs "
              f"{t_full:.3f} ms for {B}: efficiency {t_full / (N * t):.3f}")


if __name__ == "__main__":
    main()
