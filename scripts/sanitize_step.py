#!/usr/bin/env python
"""One small training step (forward, loss, backward, SGD, fragments -> pixels) of cfg1 and of
cfg2's net on a 100^2 image, for compute-sanitizer (racecheck / synccheck / initcheck /
memcheck) runs over every kernel of the path: the tcgen05/TMA convolutions and weight
gradients (CTA pairs, multi-tap, M = 64 tiles), the MPF kernels, the head and the reductions.
    compute-sanitizer --tool racecheck python scripts/sanitize_step.py
"""
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import mpf_synth as S  # noqa: E402


def main():
    import torch
    from paper_1302_1690_b200.net import MPFNet
    cases = [S.CONFIGS["cfg1"], dataclasses.replace(S.CONFIGS["cfg2"], H=100, W=100),
             dataclasses.replace(S.CONFIGS["cfg4"], H=126, W=126)]
    for cfg in cases:
        im, lb = S.make_batch(cfg, [0, 1])
        net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=2)
        net.set_params(S.init_params(cfg).astype(np.float32))
        img, lab = torch.tensor(im, device="cuda"), torch.tensor(lb, device="cuda")
        probs = net.forward(img, want_probs=True)
        loss = net.backward(lab)
        net.sgd_step(cfg.lr, 0.5)
        net.fragments_to_pixels(probs, 2, cfg.classes)
        net.train_step(img, lab)
        net.check()
        torch.cuda.synchronize()
        print(cfg.name, cfg.H, "loss", loss.cpu().numpy())


if __name__ == "__main__":
    main()
