#!/usr/bin/env python
"""The README's Python API example, runnable: one call of every public entry point on a
BASELINE workload (default cfg2, small), printing what each returned.

    python scripts/api_tour.py [--workload cfg4]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import mpf_synth as S  # noqa: E402
from paper_1302_1690_b200.net import Lbfgs, MPFNet, mirror_pad  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    a = ap.parse_args()
    cfg = S.CONFIGS[a.workload]
    n = cfg.global_batch
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=n)
    net.set_params(S.init_params(cfg))
    images, labels = (torch.tensor(x, device="cuda") for x in S.make_batch(cfg, range(n)))

    loss = net.train_step(images, labels)
    print("train_step: per-image losses", [round(float(v), 4) for v in loss])
    net.sgd_step(cfg.lr, 1.0 / n)
    r = net.armijo_step(images, labels, alpha0=0.01)
    print("armijo_step:", r)
    try:
        w, counts = net.class_weights_auto(labels)
        print("class_weights_auto:", [round(v, 4) for v in w], counts)
    except Exception as e:  # a class absent from this batch is an invalid input
        print("class_weights_auto:", e)
    print("lbfgs step:", Lbfgs(net, memory=10).step(images, labels))
    probs = net.predict(images)
    print("predict:", tuple(probs.shape), "sums to 1:", bool(torch.allclose(probs.sum(1), torch.ones(1, device="cuda"))))
    seg = MPFNet(cfg.layers, cfg.P, cfg.H + cfg.P - 1, cfg.W + cfg.P - 1, max_images=n)
    seg.set_params(net.get_params())
    full = seg.predict(mirror_pad(images, cfg.P))
    print("same-size segmentation:", tuple(full.shape), "for images", tuple(images.shape))
    assert full.shape[-2:] == images.shape[-2:]


if __name__ == "__main__":
    main()
