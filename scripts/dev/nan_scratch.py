"""Fill the scratch arena (and the tape) with NaN before a step: any read of a scratch or
tape byte that the step did not write first shows up as a NaN gradient."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import mpf_synth as S
from paper_1302_1690_b200.net import MPFNet
sys.path.insert(0, os.path.dirname(__file__))
from wide_diag3 import build, variants  # noqa

for nm in sys.argv[1:]:
    blocks, s, fcs, act = variants[nm]
    layers, P = build(blocks, s, fcs, act)
    rng = np.random.default_rng(7)
    H, W = P + 40, P + 47
    x = torch.tensor(rng.standard_normal((1, 1, H, W)).astype(np.float32), device="cuda")
    y = torch.tensor(S.random_labels(rng, 1, H - P + 1, W - P + 1, layers[-1].n_out), device="cuda")
    for prec in ("fp32", "tf32"):
        net = MPFNet(layers, P, H, W, max_images=1, precision=prec)
        net.set_params(S.init_params(layers, 5).astype(np.float32))
        for fill in ("scratch", "tape", "both"):
            if fill in ("scratch", "both"):
                net.scratch.view(torch.float32).fill_(float("nan"))
            if fill in ("tape", "both"):
                net.tape.view(torch.float32)[: net.tape.numel() // 4].fill_(float("nan"))
            net.zero_grads()
            net.forward(x)
            net.backward(y)
            torch.cuda.synchronize()
            g = net.grads.cpu().numpy()
            print(nm, prec, fill, "NaN grads:", int(np.isnan(g).sum()), "of", g.size, flush=True)
