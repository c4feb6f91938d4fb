#!/usr/bin/env python
"""Full-batch L-BFGS timed on one GPU: wall ms per
iteration (evaluations = forward + backward of the whole batch), the evaluations it took,
the loss trajectory, and the two-loop direction alone (device time of its passes, by CUDA
events, with the pairs stored so far), next to the plain SGD step of the same batch.

    python scripts/bench_lbfgs.py --workload cfg4 [--memory 10] [--iters 12]
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
from paper_1302_1690_b200.net import Lbfgs, MPFNet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--memory", type=int, default=10)
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--alpha0", type=float, default=0.05)
    a = ap.parse_args()
    cfg = S.CONFIGS[a.workload]
    n = cfg.global_batch
    im, lab = S.make_batch(cfg, list(range(n)))
    x, y = torch.tensor(im, device="cuda"), torch.tensor(lab, device="cuda")
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=n)
    p0 = S.init_params(cfg).astype(np.float32)
    net.set_params(p0)
    for _ in range(2):
        net.train_step(x, y)
        net.sgd_step(cfg.lr, 1.0 / n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(4):
        net.train_step(x, y)
        net.sgd_step(cfg.lr, 1.0 / n)
    torch.cuda.synchronize()
    sgd_ms = (time.perf_counter() - t0) * 1e3 / 4
    net.set_params(p0)
    net.zero_grads()
    lb = Lbfgs(net, memory=a.memory)
    recs, times = [], []
    for _ in range(a.iters):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        recs.append(lb.step(x, y, alpha0=a.alpha0))
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
    # the two-loop alone, with the pairs now stored (direction() only re-derives v)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dms = []
    for _ in range(10):
        torch.cuda.synchronize()
        e0.record(torch.cuda.default_stream())
        lb.direction()
        e1.record(torch.cuda.default_stream())
        torch.cuda.synchronize()
        dms.append(e0.elapsed_time(e1))
    k, nparams = recs[-1]["pairs"], net.geom.n_params
    passes = 2 * k + 1
    bytes_dir = passes * nparams * (4 + 4 + 16)  # x, z fp32 read; v fp64 read + write
    dmed = float(np.median(dms))
    line = {"metric": "full-batch L-BFGS iteration (wall ms)", "workload": a.workload, "images": n,
            "memory": a.memory, "n_params": nparams, "sgd_step_ms": sgd_ms,
            "iter_ms": times, "evals": [r["evals"] for r in recs], "alpha": [r["alpha"] for r in recs],
            "loss": [r["loss"] for r in recs], "loss0": recs[0]["loss0"], "pairs": k,
            "direction_ms_median": dmed, "direction_passes": passes, "direction_alg_bytes": bytes_dir,
            "direction_GBps": bytes_dir / (dmed * 1e-3) / 1e9}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
