#!/usr/bin/env python
"""Interleaved timing of the device-resident step (train_step + sgd_step on HBM inputs) and the
host-buffer step (mpf_train_step_host: pinned H2D copies + loss D2H inside), to separate the
e2e gap from clock drift:  python scripts/e2e_ab.py --workload cfg5 --rounds 4 --steps 5"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import mpf_synth as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import torch
    from paper_1302_1690_b200.net import MPFNet
    cfg = S.CONFIGS[a.workload]
    B = cfg.global_batch
    im, lb = S.make_batch(cfg, list(range(B)))
    d_im, d_lb = torch.tensor(im, device="cuda"), torch.tensor(lb, device="cuda")
    h_im, h_lb = torch.tensor(im).pin_memory(), torch.tensor(lb).pin_memory()
    h_loss = torch.zeros(B, dtype=torch.float32).pin_memory()
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=B)
    net.set_params(S.init_params(cfg).astype(np.float32))
    s = torch.cuda.current_stream()

    def dev_step():
        net.train_step(d_im, d_lb)
        net.sgd_step(cfg.lr, 1.0 / B)

    def host_step():
        net.train_step_host(h_im, h_lb, h_loss, apply_sgd=True, lr=cfg.lr, grad_scale=1.0 / B)

    def copy_only():  # the H2D copies of one step alone
        d_im.copy_(h_im, non_blocking=True)
        d_lb.copy_(h_lb, non_blocking=True)

    res = {"device": [], "host": [], "copies": []}
    for fn in (dev_step, host_step):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    for _ in range(a.rounds):
        for name, fn in (("device", dev_step), ("host", host_step), ("copies", copy_only)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.steps):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) / a.steps)
    for k, v in res.items():
        print(f"{a.workload} {k:7s} ms/step: min {min(v):.3f} mean {np.mean(v):.3f}  {[round(x, 3) for x in v]}")


if __name__ == "__main__":
    main()
