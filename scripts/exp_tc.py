"""Experiment: tcgen05 conv vs the SIMT conv on the same net, and TF32 error sources.

Run on a GPU box:  python scripts/exp_tc.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mpf_synth as S  # noqa: E402
from paper_1302_1690_b200 import MPF_TAPE_VALUE  # noqa: E402
from paper_1302_1690_b200.net import MPFNet  # noqa: E402
from tests.gpu_common import gpu_step, oracle_step, param_slices, rel_l2  # noqa: E402


def run(cfg, H, n, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: v for k, v in env.items() if v is not None})
    for k, v in env.items():
        if v is None:
            os.environ.pop(k, None)
    try:
        rng = np.random.default_rng(0)
        images, labels = S.make_batch(cfg, range(n)) if H == cfg.H else (
            rng.standard_normal((n, 1, H, H)).astype(np.float32), None)
        if labels is None:
            labels = S.random_labels(rng, n, H - cfg.P + 1, H - cfg.P + 1, cfg.classes, 0.0)
        params = S.init_params(cfg)
        net = MPFNet(cfg.layers, cfg.P, H, H, max_images=n, precision="tf32", debug_keep=True)
        g = gpu_step(cfg.layers, cfg.P, images, labels, params, "tf32", net=net)
        outs = {}
        net.set_params(params.astype(np.float32))
        net.forward(g["img"])
        torch.cuda.synchronize()
        for l, ly in enumerate(cfg.layers[:-1]):
            if ly.kind != S.POOL:
                outs[l] = net.debug_tape(l, MPF_TAPE_VALUE, n).cpu().numpy()
        return g, outs, images, labels, params
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    for name, H, n in [("cfg2", 128, 2), ("cfg5", 120, 1), ("cfg4", 200, 1), ("cfg3", 200, 1)]:
        cfg = S.CONFIGS[name]
        ref, ref_out, *_ = run(cfg, H, n, {"MPF_DISABLE_TC": "1"})
        for bm in ("0",):
            try:
                g, outs, *_ = run(cfg, H, n, {"MPF_DISABLE_TC": None, "MPF_TC_BASE_MODE": bm})
            except Exception as e:  # noqa: BLE001
                print(name, "base_mode", bm, "ERROR", e)
                continue
            fe = {l: f"{rel_l2(outs[l], ref_out[l]):.1e}" for l in outs}
            ge = {nm: f"{rel_l2(g['grad_sum'][sl], ref['grad_sum'][sl]):.1e}" for nm, sl in param_slices(cfg.layers)}
            print(f"{name} H={H} base_mode={bm}: conv outputs vs SIMT {fe}; grads vs SIMT {ge}", flush=True)
    # error source: cfg1 tf32 with forward operands unrounded
    cfg = S.CONFIGS["cfg1"]
    images, labels = S.make_batch(cfg, [0])
    params = S.init_params(cfg)
    o = oracle_step(cfg.layers, cfg.P, images.astype(np.float64), labels, params, engine="o1")
    for env in ({}, {"MPF_DEBUG_FWD_FP32": "1"}):
        os.environ.update(env)
        g = gpu_step(cfg.layers, cfg.P, images, labels, params, "tf32")
        for k in env:
            os.environ.pop(k)
        errs = {nm: f"{rel_l2(g['grad_sum'][sl], o['grad_sum'][sl]):.1e}" for nm, sl in param_slices(cfg.layers)}
        print("cfg1 tf32", env, errs, flush=True)
    # timing of TC vs SIMT on a cfg4 image
    cfg = S.CONFIGS["cfg4"]
    images, labels = S.make_batch(cfg, [0])
    params = S.init_params(cfg).astype(np.float32)
    for env in ({"MPF_DISABLE_TC": "1"}, {}):
        os.environ.update(env)
        net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=1)
        net.set_params(params)
        img = torch.tensor(images, device="cuda")
        lab = torch.tensor(labels, device="cuda")
        for _ in range(2):
            net.forward(img)
            net.backward(lab)
        torch.cuda.synchronize()
        net.profile_begin(1000)
        net.forward(img)
        net.backward(lab)
        st = net.profile_end()
        for k in env:
            os.environ.pop(k)
        st.sort(key=lambda r: -r["total_ms"])
        print("cfg4 1 image", env, "total ms", round(sum(r["total_ms"] for r in st), 2))
        for r in st[:12]:
            rate = r["flops"] / r["total_ms"] / 1e9 if r["flops"] else r["bytes"] / r["total_ms"] / 1e6
            print(f"   {r['name']:>16} L{r['layer']:<2} {r['total_ms']:8.3f} ms  {rate:9.1f} {'TF/s' if r['flops'] else 'GB/s'}")


if __name__ == "__main__":
    main()
