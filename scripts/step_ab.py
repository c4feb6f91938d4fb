#!/usr/bin/env python
"""A/B of kernel-selection flags (MPF_FLAG_*) on the whole overlapped training step (side
stream on, unlike kernel_ab.py's serialised per-kernel tables): forward + backward + SGD,
eager launches, CUDA-event time per step; the flag sets alternate round by round so clock
drift hits them alike.

    python scripts/step_ab.py --workload cfg4 --flags 0 0x800 --rounds 4 --steps 3
"""
import argparse
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
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--images", type=int, default=0, help="0 = the config's global batch")
    a = ap.parse_args()
    import torch
    from paper_1302_1690_b200.net import MPFNet
    cfg = S.CONFIGS[a.workload]
    B = a.images or cfg.global_batch
    im, lb = S.make_batch(cfg, list(range(B)))
    img, lab = torch.tensor(im, device="cuda"), torch.tensor(lb, device="cuda")
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=B)
    net.set_params(S.init_params(cfg).astype(np.float32))
    times = {fl: [] for fl in a.flags}

    def step():
        net.train_step(img, lab)
        net.sgd_step(cfg.lr, 1.0 / B)

    for r in range(a.rounds):
        for fl in a.flags:
            net.set_flags(fl)
            for _ in range(2):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                step()
            e1.record()
            torch.cuda.synchronize()
            times[fl].append(e0.elapsed_time(e1) / a.steps)
    for fl in a.flags:
        t = np.array(times[fl])
        print(f"{a.workload} n={B} flags={fl:#x}: {t.mean():.3f} ms/step (min {t.min():.3f}, rounds {np.round(t, 3).tolist()})")


if __name__ == "__main__":
    main()
