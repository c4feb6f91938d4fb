#!/usr/bin/env python
"""Armijo-safeguarded step timed on one GPU: ms per step and the
loss evaluations it took, next to the plain SGD step of the same batch.

    python scripts/bench_armijo.py --workload cfg4 [--alpha0 0.01]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import mpf_synth as S  # noqa: E402
from paper_1302_1690_b200.net import MPFNet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--alpha0", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=4)
    a = ap.parse_args()
    cfg = S.CONFIGS[a.workload]
    n = cfg.global_batch
    im, lb = S.make_batch(cfg, list(range(n)))
    x, y = torch.tensor(im, device="cuda"), torch.tensor(lb, device="cuda")
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=n)
    net.set_params(S.init_params(cfg).astype(np.float32))
    for _ in range(2):  # warm-up
        net.train_step(x, y)
        net.sgd_step(cfg.lr, 1.0 / n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        net.train_step(x, y)
        net.sgd_step(cfg.lr, 1.0 / n)
    torch.cuda.synchronize()
    sgd_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    res = []
    t0 = time.perf_counter()
    for _ in range(a.steps):
        res.append(net.armijo_step(x, y, alpha0=a.alpha0))
    torch.cuda.synchronize()
    arm_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    line = {"metric": "Armijo-safeguarded step (wall ms, host line search)", "workload": a.workload, "images": n,
            "alpha0": a.alpha0, "armijo_ms": arm_ms, "sgd_step_ms": sgd_ms,
            "evals": [r["evals"] for r in res], "alpha": [r["alpha"] for r in res],
            "loss": [[r["loss0"], r["loss"]] for r in res]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
