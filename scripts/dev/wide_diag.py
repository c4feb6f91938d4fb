"""Diagnostic sweep: first-layer gradient error vs O2 (fp32 path) on small variants."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import mpf_synth as S
from oracle import o2
from tests.gpu_common import gpu_step, rel_l2, param_slices

def run(layers, P, cin, H, W, seed=0, prec="fp32"):
    rng = np.random.default_rng(seed)
    images = rng.standard_normal((1, cin, H, W)).astype(np.float32)
    labels = S.random_labels(rng, 1, H - P + 1, W - P + 1, layers[-1].n_out)
    params = S.init_params(layers, seed, in_channels=cin)
    g = gpu_step(layers, P, images, labels, params, prec)
    ls, cnt, gr, pr = o2.train_image(layers, params, images[0].astype(np.float64), labels[0], P=P, in_channels=cin)
    out = {}
    for nm, sl in param_slices(layers):
        out[nm] = rel_l2(g["grad_sum"][sl], gr[sl] / cnt)
    out["probs"] = rel_l2(g["probs"][0], pr)
    return out

T, L = S.TANH, S.LOGISTIC
act = int(sys.argv[1]) if len(sys.argv) > 1 else T
cases = {
  "c3-c2-mp2 cin4": ((S.C(3, 36, act), S.C(2, 44, act), S.MP(2), S.F(2, 40, act), S.F(1, 5, S.IDENTITY)), 7, 4),
  "c3-c2-mp2 cin1": ((S.C(3, 36, act), S.C(2, 44, act), S.MP(2), S.F(2, 40, act), S.F(1, 5, S.IDENTITY)), 7, 1),
  "c3-mp2 cin4": ((S.C(3, 36, act), S.MP(2), S.F(2, 40, act), S.F(1, 5, S.IDENTITY)), 6, 4),
  "c3-mp2 cin1": ((S.C(3, 36, act), S.MP(2), S.F(2, 40, act), S.F(1, 5, S.IDENTITY)), 6, 1),
  "c3x8-mp2 cin4": ((S.C(3, 8, act), S.MP(2), S.F(2, 8, act), S.F(1, 5, S.IDENTITY)), 6, 4),
  "c1-mp2 cin4": ((S.C(1, 16, act), S.MP(2), S.F(2, 8, act), S.F(1, 3, S.IDENTITY)), 4, 4),
}
for nm, (layers, P, cin) in cases.items():
    r = run(layers, P, cin, P + 60, P + 50)
    print(nm, {k: f"{v:.2e}" for k, v in r.items()}, flush=True)
