"""Reproduce test_wide_random_archs_vs_o2 seeds and bisect (fp32 path)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import mpf_synth as S
from oracle import o2
from tests.gpu_common import gpu_step, rel_l2, param_slices
src = open(os.path.join(os.path.dirname(__file__), "..", "..", "tests", "test_gpu_parity.py")).read()
i = src.find("def _wide_arch"); j = src.find("@pytest.mark.parametrize", i)
ns = {"S": S, "np": np}; exec(src[i:j], ns)

def run(layers, P, cin, images, labels, params, prec="fp32"):
    g = gpu_step(layers, P, images, labels, params, prec)
    n = images.shape[0]
    gs = np.zeros_like(params)
    for k in range(n):
        ls, cnt, gr, pr = o2.train_image(layers, params, images[k].astype(np.float64), labels[k], P=P, in_channels=cin)
        gs += gr / cnt
    return {nm: f"{rel_l2(g['grad_sum'][sl], gs[sl]):.1e}" for nm, sl in param_slices(layers)}

for seed in [int(a) for a in sys.argv[1:]]:
    rng = np.random.default_rng(900 + seed)
    layers, P = ns["_wide_arch"](rng)
    cin = 4 if seed % 2 else 1
    n = int(rng.integers(1, 3))
    H, W = int(rng.integers(P + 40, P + 140)), int(rng.integers(P + 40, P + 140))
    images = rng.standard_normal((n, cin, H, W)).astype(np.float32)
    labels = S.random_labels(rng, n, H - P + 1, W - P + 1, layers[-1].n_out)
    params = S.init_params(layers, seed, in_channels=cin)
    print("seed", seed, "act", layers[0].act, "P", P, "n", n, H, W, [(l.kind, l.k, l.n_out) for l in layers], flush=True)
    print("  exact       ", run(layers, P, cin, images, labels, params), flush=True)
    print("  1 image     ", run(layers, P, cin, images[:1], labels[:1], params), flush=True)
    print("  params*0.5  ", run(layers, P, cin, images[:1], labels[:1], params * 0.5), flush=True)
    os.environ["MPF_DISABLE_TC"] = "1"
    print("  no TC       ", run(layers, P, cin, images[:1], labels[:1], params), flush=True)
    os.environ.pop("MPF_DISABLE_TC")
    Hs, Ws = P + 10, P + 12
    print("  small image ", run(layers, P, cin, np.ascontiguousarray(images[:1, :, :Hs, :Ws]),
                              np.ascontiguousarray(labels[:1, :Hs - P + 1, :Ws - P + 1]), params), flush=True)
