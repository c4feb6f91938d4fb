import os, sys, ctypes
import numpy as np, torch
sys.path.insert(0, '.')
import mpf_synth as S
from paper_1302_1690_b200.net import MPFNet
from paper_1302_1690_b200 import _lib as L

cfg = S.CONFIGS["cfg2"]
images, labels = S.make_batch(cfg, [3])
params = S.init_params(cfg)
net = MPFNet(cfg.layers, cfg.P, 128, 128, max_images=1, debug_keep=True)
net.set_params(params.astype(np.float32))
img = torch.tensor(images, device="cuda"); lab = torch.tensor(labels, device="cuda")
g = net.geom
Lh = g.n_layers - 1
F, gr, gc, Ch = g.frag[Lh], g.rows[Lh], g.cols[Lh], g.chans[Lh]
print("h grid", F, gr, gc, Ch)
# unfused: probs per position and h
probs = net.forward(img, want_probs=True)
h = net.debug_tape(Lh - 1, L.MPF_TAPE_VALUE, 1).cpu().numpy()   # [F, vr, vc, Ch] compact
pr = probs.cpu().numpy()  # [F, vr, vc, C]
# fused
net.zero_grads()
loss = net.train_step(img, lab)
torch.cuda.synchronize()
per_img = F * net.geom.rows[Lh] * 0
nrow = F * h.shape[1] * 0
# the fused path's grid: FC1 output stored on its input grid (gr_in x gc_in)
gri, gci = g.rows[Lh - 1], g.cols[Lh - 1]
print("input grid of FC1", gri, gci, "valid", h.shape[1], h.shape[2])
rows = F * gri * gci
rl = torch.empty(rows, dtype=torch.float32, device="cuda")
L.check(net.lib.mpf_debug_scratch(net.h, 0, ctypes.c_void_p(rl.data_ptr()), rows * 4, None), "dbg")
rl = rl.cpu().numpy().reshape(F, gri, gci)
# expected per-position loss: -log p[label] with the fragment->pixel label map
from oracle import o2
lossmap = np.zeros((F, h.shape[1], h.shape[2]))
ks = [L2.k for L2 in cfg.layers if L2.kind == S.POOL]
for f in range(F):
    for i in range(h.shape[1]):
        for j in range(h.shape[2]):
            yy, xx, rf = i, j, f
            for kq in reversed(ks):
                d = rf % (kq * kq); rf //= kq * kq
                yy = d // kq + kq * yy; xx = d % kq + kq * xx
            if yy < cfg.out_rows and xx < cfg.out_cols:
                t = labels[0, yy, xx]
                if t != 255:
                    lossmap[f, i, j] = -np.log(pr[f, i, j, t])
fused = rl[:, :h.shape[1], :h.shape[2]]
d = np.abs(fused - lossmap)
print("loss sum fused", fused.sum(), "expected", lossmap.sum(), "max abs diff", d.max())
idx = np.argwhere(d > 1e-3)
print("n bad", len(idx), "of", lossmap.size, idx[:10])
print("bad by i", np.bincount(idx[:, 1], minlength=h.shape[1]) if len(idx) else None)
print("bad by j", np.bincount(idx[:, 2], minlength=h.shape[2]) if len(idx) else None)
print("bad by f", np.bincount(idx[:, 0], minlength=F)[:16] if len(idx) else None)
