#!/usr/bin/env python
"""Maximum-size probe: the cfg4 net bound for 16 images of 1024^2 (the FC1 activations and
deltas hold 2.8e9 fp32 elements each: beyond 2^31) against the same net bound for 8.  The 16
images are the bench's 8 images twice, so per-image losses must repeat the 8-image run's and
the gradient sum must be twice its gradient sum, up to the order of the fp32 partial sums and
the length of the tensor-core accumulation chains (conv_tc.cu wgrad_splits caps them at 160 K
positions; before the cap the FC1 weight gradient of the two runs differed by 2.1e-3, the
chains of the 16-image run being twice as long).
Usage: python scripts/big_batch_probe.py [n_big] [workload]   (default 16 cfg4; e.g. 32 cfg5)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import mpf_synth as S  # noqa: E402


def main():
    import torch
    from paper_1302_1690_b200.net import MPFNet
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    cfg = S.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "cfg4"]
    im, lb = S.make_batch(cfg, list(range(8)))
    params = S.init_params(cfg).astype(np.float32)

    def run(n):
        reps = n // 8
        net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=n)
        print(f"n={n}: bytes {net.bytes}", flush=True)
        net.set_params(params)
        img = torch.tensor(np.concatenate([im] * reps), device="cuda")
        lab = torch.tensor(np.concatenate([lb] * reps), device="cuda")
        loss = net.train_step(img, lab)
        torch.cuda.synchronize()
        net.check()
        out = loss.cpu().numpy().copy(), net.grads.double().cpu().numpy().copy()
        del net, img, lab
        torch.cuda.empty_cache()
        return out

    l8, g8 = run(8)
    lN, gN = run(nb)
    reps = nb // 8
    dl = np.abs(lN - np.tile(l8, reps)).max()
    rel = np.linalg.norm(gN - reps * g8) / np.linalg.norm(reps * g8)
    print(f"per-image losses: max |diff| {dl:.3e} (losses {l8[:3]} ...)")
    print(f"gradient sum vs {reps} x the 8-image sum: rel L2 {rel:.3e}")
    from tests.gpu_common import param_slices
    for nm, sl in param_slices(cfg.layers):
        e = np.linalg.norm(gN[sl] - reps * g8[sl]) / max(np.linalg.norm(reps * g8[sl]), 1e-30)
        print(f"   {nm}: {e:.3e}")
    ok = dl <= 1e-6 and rel <= 2e-4
    print("OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
