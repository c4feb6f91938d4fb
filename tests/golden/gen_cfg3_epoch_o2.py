"""Writes tests/golden/cfg3_epoch_o2.npz: the oracle's (O2, fp64) one epoch of per-image
SGD on configs[2] (cfg3: 64 images of 512^2, the cfg2 architecture; "updating the weights
after every image"; reading R14), for the GPU epoch test
(tests/test_gpu_parity.py::test_cfg3_epoch_vs_o2).

Calls only oracle/ (O2 = Alg. 1-4 written out, pinned by tests/test_oracle_pins.py) and the
seeded input generators of mpf_synth; nothing here comes from the CUDA path.

    python tests/golden/gen_cfg3_epoch_o2.py          # ~8 min on 8 cores

Stored: loss[i] = mean MCCE of image i at the parameters before step i (R8), theta0 (the
seeded initial parameters, fp64), theta_final after the 64 steps theta <- theta - lr g_i.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import mpf_synth as S  # noqa: E402
from oracle import o2  # noqa: E402


def main():
    cfg = S.CONFIGS["cfg3"]
    theta0 = S.init_params(cfg).astype(np.float32).astype(np.float64)  # the GPU starts from the fp32 copy
    theta = theta0.copy()
    losses = np.zeros(cfg.n_images)
    t0 = time.time()
    for i in range(cfg.n_images):
        images, labels = S.make_batch(cfg, [i])
        ls, cnt, g, _ = o2.train_image(cfg.layers, theta, images[0].astype(np.float64), labels[0], P=cfg.P)
        losses[i] = ls / cnt
        theta = theta - cfg.lr * (g / cnt)
        print(f"step {i}: loss {losses[i]:.6f} ({time.time() - t0:.0f} s)", flush=True)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg3_epoch_o2.npz")
    np.savez_compressed(out, loss=losses, theta0=theta0, theta_final=theta, lr=cfg.lr)
    print("wrote", out)


if __name__ == "__main__":
    main()
