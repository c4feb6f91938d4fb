"""Helpers shared by the GPU parity tests: run the CUDA path through the C ABI and
the oracle on the same seeded inputs, and compare element by element."""
from __future__ import annotations

import numpy as np

import mpf_synth as S
import oracle
from oracle import o2

# north_star tolerance: relative L2 error 5e-3 (TF32 tensor cores, fp32 accumulate), per
# tensor (reading R17).  fp32 mode must be far tighter.
TOL_TF32 = 5e-3
TOL_FP32 = 1e-3  # fp32 arithmetic; a rare argmax flip vs fp64 can still move early-layer grads ~1e-4


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def param_slices(layers, in_channels=1):
    out, off, c = [], 0, in_channels
    for i, L in enumerate(layers):
        if L.kind == S.POOL:
            continue
        n = L.n_out * c * L.k * L.k
        out.append((f"W{i}", slice(off, off + n)))
        out.append((f"b{i}", slice(off + n, off + n + L.n_out)))
        off += n + L.n_out
        c = L.n_out
    return out


def gpu_step(layers, P, images, labels, params, precision="tf32", lr=0.01, class_w=None, debug_keep=False,
             net=None):
    """forward (+probs) -> backward -> sgd on the GPU. Returns dict of numpy results."""
    import torch
    from paper_1302_1690_b200.net import MPFNet
    n, cin, H, W = images.shape
    if net is None:
        net = MPFNet(layers, P, H, W, max_images=n, in_channels=cin, precision=precision, debug_keep=debug_keep)
    net.set_params(params.astype(np.float32))
    net.zero_grads()
    img = torch.tensor(images, dtype=torch.float32, device="cuda").contiguous()
    lab = torch.tensor(labels, dtype=torch.uint8, device="cuda").contiguous()
    probs_frag = net.forward(img, want_probs=True)
    loss = net.backward(lab, class_w)
    grads = net.grads.clone()
    p0 = net.params.clone()
    net.sgd_step(lr, 1.0 / n)
    net.check()
    pix = net.fragments_to_pixels(probs_frag, n, net.geom.classes)
    torch.cuda.synchronize()
    return dict(net=net, probs=pix.cpu().numpy(), probs_frag=probs_frag.cpu().numpy(), loss=loss.cpu().numpy(),
                grad_sum=grads.cpu().numpy().astype(np.float64), params0=p0.cpu().numpy(),
                params1=net.params.cpu().numpy(), img=img, lab=lab)


def oracle_step(layers, P, images, labels, params, engine="o2", class_w=None, pix=None, threads=None):
    """Per image: probs [C, O_H, O_W] (O2) and per-image mean loss / gradient."""
    n = images.shape[0]
    probs, losses, grads = [], [], []
    for i in range(n):
        if engine == "o2":
            ls, cnt, g, pr = o2.train_image(layers, params, images[i], labels[i], class_w, P=P)
        else:
            ls, cnt, g, pr = oracle.o1_image(layers, P, params, images[i], labels[i], class_w,
                                             None if pix is None else pix[i], threads)
        probs.append(pr)
        losses.append(ls / cnt if cnt else 0.0)
        grads.append(g / cnt if cnt else np.zeros_like(params))
    return dict(probs=probs, loss=np.array(losses), grads=grads, grad_sum=np.sum(grads, axis=0))


def compare_step(layers, g, o, tol, what=""):
    """Per-tensor rel L2 of probs, loss, every W/b gradient; returns the worst."""
    errs = {}
    if isinstance(o["probs"][0], np.ndarray) and o["probs"][0].ndim == 3:
        errs["probs"] = rel_l2(g["probs"], np.stack(o["probs"]))
    errs["loss"] = rel_l2(g["loss"], o["loss"])
    for name, sl in param_slices(layers):
        errs["g" + name] = rel_l2(g["grad_sum"][sl], o["grad_sum"][sl])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"{what}: rel L2 above {tol}: {bad} (all: {errs})"
    return errs
