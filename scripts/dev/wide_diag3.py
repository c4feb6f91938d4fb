"""Bisect the logistic-activation gradient error (fp32 path) over architecture variants."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import mpf_synth as S
from oracle import o2
from tests.gpu_common import gpu_step, rel_l2, param_slices

def build(blocks, s, fcs, act):
    size = s
    for convs, kp in reversed(blocks):
        size *= kp
        for kc, _ in reversed(convs):
            size += kc - 1
    layers = []
    for convs, kp in blocks:
        layers += [S.C(kc, n, act) for kc, n in convs] + [S.MP(kp)]
    layers.append(S.F(s, fcs[0], act))
    for f in fcs[1:-1]:
        layers.append(S.F(1, f, act))
    layers.append(S.F(1, fcs[-1], S.IDENTITY))
    return tuple(layers), size

def run(layers, P, cin, prec="fp32", extra=40):
    rng = np.random.default_rng(7)
    H, W = P + extra, P + extra + 7
    images = rng.standard_normal((1, cin, H, W)).astype(np.float32)
    labels = S.random_labels(rng, 1, H - P + 1, W - P + 1, layers[-1].n_out)
    params = S.init_params(layers, 5, in_channels=cin)
    g = gpu_step(layers, P, images, labels, params, prec)
    ls, cnt, gr, pr = o2.train_image(layers, params, images[0].astype(np.float64), labels[0], P=P, in_channels=cin)
    r = {nm: f"{rel_l2(g['grad_sum'][sl], gr[sl] / cnt):.0e}" for nm, sl in param_slices(layers)}
    r["probs"] = f"{rel_l2(g['probs'][0], pr):.0e}"
    if os.environ.get("DIAG_TAPS"):
        cinl = cin
        for (nm, sl), lay in zip(param_slices(layers), [l for l in layers for _ in (0, 1) if l.kind != S.POOL]):
            if not nm.startswith("W") or lay.kind == S.POOL:
                continue
            gg, oo = g['grad_sum'][sl], gr[sl] / cnt
            k = lay.k
            try:
                a = gg.reshape(lay.n_out, -1, k, k); b = oo.reshape(lay.n_out, -1, k, k)
            except Exception:
                continue
            tap = [[f"{rel_l2(a[:, :, i, j], b[:, :, i, j]):.0e}" for j in range(k)] for i in range(k)]
            print("   ", nm, "per-tap rel err", tap, "mean|g|", f"{np.abs(b).mean():.1e}", "mean diff", f"{(a-b).mean():.1e}")
    r["loss"] = f"{abs(g['loss'][0] - ls / cnt) / abs(ls / cnt):.0e}"
    return r

L, T = S.LOGISTIC, S.TANH
variants = {
  "C noC1 T": ([([(3, 36), (2, 44)], 2), ([(2, 68)], 2)], 2, [40, 5], T),
  "A full L": ([([(3, 36), (2, 44)], 2), ([(2, 68), (1, 24)], 2)], 2, [40, 5], L),
  "A full T": ([([(3, 36), (2, 44)], 2), ([(2, 68), (1, 24)], 2)], 2, [40, 5], T),
  "C noC1 L": ([([(3, 36), (2, 44)], 2), ([(2, 68)], 2)], 2, [40, 5], L),
  "D 1lvl L": ([([(2, 68), (1, 24)], 2)], 2, [40, 5], L),
  "E C1 L": ([([(1, 24)], 2)], 2, [40, 5], L),
  "F 2lvl simple L": ([([(3, 36)], 2), ([(2, 68)], 2)], 2, [40, 5], L),
  "G 2lvl simple T": ([([(3, 36)], 2), ([(2, 68)], 2)], 2, [40, 5], T),
  "H 1lvl L": ([([(3, 36)], 2)], 2, [40, 5], L),
}
if __name__ != '__main__':
    sel = []
else:
    sel = sys.argv[1:] or list(variants)
for nm, (blocks, s, fcs, act) in variants.items():
    if nm.split()[0] not in sel:
        continue
    layers, P = build(blocks, s, fcs, act)
    for env in ["", "MPF_DISABLE_TC", "MPF_BWD_SLIDE"]:
        if env:
            os.environ[env] = "1"
        print(nm, env or "default", "P", P, run(layers, P, 1), flush=True)
        if env:
            os.environ.pop(env)
