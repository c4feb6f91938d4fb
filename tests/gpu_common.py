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


def _tf32_round(t):
    """Round to TF32 on the fp32 bit pattern, nearest with ties to even, as the GPU's
    cvt.rn.tf32 does (finite inputs: the rounding model sees no Inf/NaN)."""
    import torch
    b = t.detach().float().contiguous().view(torch.int32)
    lsb = (b >> 13) & 1
    return ((b + 0x0FFF + lsb) & ~0x1FFF).view(torch.float32).to(t.dtype)


def rounding_model_grads(layers, params, images, labels, prec):
    """Expected rounding error of the GPU arithmetic, for deriving per-tensor tolerances on
    random architectures (reading R22; not a reference for the values): the same network
    as a dilated-convolution model (every patch output of the whole image, SURVEY.md §4
    item 4) in CPU torch, fp32 arithmetic, with every convolution operand and every
    gradient flowing into one rounded to TF32 when prec == "tf32" (tensor-core inputs;
    fp32 accumulation).  Returns the mean over images of the per-image mean-loss gradient."""
    import torch
    import torch.nn.functional as Fn

    class _R(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x):
            return _tf32_round(x)

        @staticmethod
        def backward(ctx, g):
            return _tf32_round(g)

    rnd = _R.apply if prec == "tf32" else (lambda v: v)
    n = images.shape[0]
    total = np.zeros(len(params))
    for i in range(n):
        th = torch.tensor(np.asarray(params, np.float32), requires_grad=True)
        x = torch.tensor(np.asarray(images[i], np.float32))[None]
        d, off, c = 1, 0, images.shape[1]
        for L in layers:
            if L.kind == S.POOL:
                x = Fn.max_pool2d(x, L.k, stride=1, dilation=d)
                d *= L.k
                continue
            nw = L.n_out * c * L.k * L.k
            W = th[off:off + nw].reshape(L.n_out, c, L.k, L.k)
            b = th[off + nw:off + nw + L.n_out]
            off += nw + L.n_out
            c = L.n_out
            x = Fn.conv2d(rnd(x), rnd(W), b, dilation=d)
            if L.act == S.TANH:
                x = torch.tanh(x)
            elif L.act == S.LOGISTIC:
                x = torch.sigmoid(x)
        logp = torch.log_softmax(x[0], dim=0)
        t = torch.tensor(np.asarray(labels[i]).astype(np.int64))
        m = t != 255
        tt = torch.where(m, t, torch.zeros_like(t))
        nll = -logp.gather(0, tt[None])[0]
        loss = (nll * m).sum() / m.sum().clamp(min=1)
        loss.backward()
        total += th.grad.double().numpy()
    return total


def o2_image_worker(args):
    """One image through the literal whole-image oracle O2 in a worker process (spawned: the
    parent holds a CUDA context).  args = (layers, params, image [cin, H, W] fp64, labels,
    P, want_idx).  Returns (loss_sum, n_lab, grad_sum, probs, idx) with idx the O2 argmax
    tensors of every pool layer (a list per layer of [C, nh, nw] uint8 per output fragment)
    when want_idx, else None."""
    layers, params, image, labels, P, want_idx = args
    ls, cnt, g, pr = o2.train_image(layers, params, image, labels, P=P)
    idx = None
    if want_idx:
        _, idxs = o2.forward_dense(layers, params, image)
        idx = [None if ix is None else [m.astype(np.uint8) for m in ix] for ix in idxs]
    return ls, cnt, g, pr, idx


def o2_images_parallel(layers, params, images, labels, P, want_idx=()):
    """O2 on several images in parallel worker processes (BLAS threads split between them)."""
    import concurrent.futures as cf
    import multiprocessing as mp
    import os
    n = images.shape[0]
    cores = len(os.sched_getaffinity(0))
    old = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in old:
        os.environ[k] = str(max(1, cores // n))
    try:
        with cf.ProcessPoolExecutor(max_workers=n, mp_context=mp.get_context("spawn")) as ex:
            jobs = [ex.submit(o2_image_worker, (layers, params, images[i].astype(np.float64), labels[i], P,
                                                i in want_idx)) for i in range(n)]
            return [j.result() for j in jobs]
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def argmax_flips(net, layers, o2_idx, n_frag_images):
    """Per pool layer: pooled cells whose GPU argmax (tape of the last forward, image 0)
    differs from O2's argmax on its own fp64 forward, over O2's ragged fragment extents
    (reading R16: end to end, TF32 rounding can flip near-ties; reported, not asserted).
    Returns {layer: (flips, cells)}."""
    from paper_1302_1690_b200 import MPF_TAPE_ARGMAX
    out = {}
    for l, ly in enumerate(layers):
        if ly.kind != S.POOL:
            continue
        gpu = net.debug_tape(l, MPF_TAPE_ARGMAX, n_frag_images).cpu().numpy()  # [n*F, rows, cols, C]
        flips = cells = 0
        for f, m in enumerate(o2_idx[l]):
            C_, nh, nw = m.shape
            g = gpu[f, :nh, :nw, :].transpose(2, 0, 1)
            flips += int(np.count_nonzero(g != m))
            cells += m.size
        out[l] = (flips, cells)
    return out
