"""Oracles for the MPF whole-image training path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything under
``oracle/``.  The product path (``paper_1302_1690_b200``) never does; it fails
loudly when its CUDA library is missing.  The two share no code: the only common
import is ``mpf_synth`` (seeded input generators, no method arithmetic).

O1 (``o1_patch.c``): the plain definition — naive patch-by-patch MPCNN training
    in fp64 C.
O2 (``o2_fragments.py``): the paper's whole-image algorithm literally
    (Alg. 1-4) on ragged fragment lists in fp64 numpy.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): SPEC/PAPER worked examples
(tests/golden/), closed forms (fragment count, output count, coverage audit),
finite differences, O1 == O2 (two independent programs from the paper), and the
library special case ``torch.nn.functional.conv2d(dilation=...)`` +
``max_pool2d(stride=1, dilation=...)`` + autograd in fp64 (an independent third
reference).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from . import o2_fragments as o2  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "o1_patch.c")
_LIB = os.path.join(_HERE, "_build", "libo1.so")
_lock = threading.Lock()
_lib = None


class O1Layer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("k", ctypes.c_int), ("n_out", ctypes.c_int),
                ("act", ctypes.c_int)]


def build_o1(force: bool = False) -> str:
    """Compile o1_patch.c with gcc (plain -O2; the oracle is never tuned)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_o1())
            lib.o1_n_params.restype = ctypes.c_long
            lib.o1_n_params.argtypes = [ctypes.POINTER(O1Layer), ctypes.c_int, ctypes.c_int, ctypes.c_int]
            lib.o1_image.restype = ctypes.c_int
            dp = ctypes.POINTER(ctypes.c_double)
            lib.o1_image.argtypes = [ctypes.POINTER(O1Layer), ctypes.c_int, ctypes.c_int, ctypes.c_int, dp,
                                     dp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_ubyte), dp,
                                     ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int, dp, dp,
                                     ctypes.POINTER(ctypes.c_long), dp]
            _lib = lib
    return _lib


def _layers_c(layers):
    arr = (O1Layer * len(layers))()
    for i, L in enumerate(layers):
        arr[i].kind, arr[i].k, arr[i].n_out, arr[i].act = L.kind, L.k, L.n_out, L.act
    return arr


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def o1_n_params(layers, P, in_channels=1) -> int:
    return int(_load().o1_n_params(_layers_c(layers), len(layers), in_channels, P))


def o1_image(layers, P, params, image, labels=None, class_w=None, pix=None, threads=None,
             need_grad=True, need_probs=True):
    """O1 on one image.  image [C,H,W] or [H,W]; labels [O_H,O_W] uint8 (255 = ignore);
    pix: linear output indices to process (None = all).  Returns
    (loss_sum, n_lab, grad_sum or None, probs [n_pix, C] or None)."""
    lib = _load()
    image = np.ascontiguousarray(image, np.float64)
    if image.ndim == 2:
        image = image[None]
    cin, H, W = image.shape
    params = np.ascontiguousarray(params, np.float64)
    npar = lib.o1_n_params(_layers_c(layers), len(layers), cin, P)
    if npar < 0:
        raise ValueError("O1: invalid architecture / patch size")
    if npar != params.size:
        raise ValueError(f"O1: expected {npar} parameters, got {params.size}")
    O_H, O_W = H - P + 1, W - P + 1
    if pix is not None:
        pix = np.ascontiguousarray(pix, np.int32)
        n_pix = pix.size
    else:
        n_pix = O_H * O_W
    C = layers[-1].n_out
    grad = np.zeros(npar) if need_grad else None
    probs = np.zeros((n_pix, C)) if need_probs else None
    loss = ctypes.c_double(0.0)
    nlab = ctypes.c_long(0)
    lab = None
    if labels is not None:
        labels = np.ascontiguousarray(labels, np.uint8)
        assert labels.shape == (O_H, O_W)
        lab = labels.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte))
    cw = np.ascontiguousarray(class_w, np.float64) if class_w is not None else None
    st = lib.o1_image(_layers_c(layers), len(layers), cin, P, _dp(params), _dp(image), H, W, lab, _dp(cw),
                      pix.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) if pix is not None else None,
                      n_pix, int(threads or default_threads()), _dp(grad), ctypes.byref(loss),
                      ctypes.byref(nlab), _dp(probs))
    if st == 3:
        raise ValueError("O1: label out of range")
    if st != 0:
        raise RuntimeError(f"O1 failed with status {st}")
    return loss.value, nlab.value, grad, probs


def train_step(layers, P, params, images, labels, class_w=None, lr=0.01, pix=None, threads=None,
               engine="o1"):
    """One SGD step on a global batch (R8, R14): per-image loss/gradient = mean over its
    labelled pixels; step gradient = mean over images; theta <- theta - lr * g.

    engine: "o1" (patch-by-patch C) or "o2" (literal Alg. 1-4, numpy).
    pix: optional list (per image) of linear output indices (O1 only).
    Returns dict(loss=[n], n_lab=[n], grad=[n_params] step gradient, params=new params)."""
    params = np.asarray(params, np.float64)
    images = np.asarray(images)
    n = images.shape[0]
    g = np.zeros_like(params)
    losses, nl = [], []
    for i in range(n):
        if engine == "o1":
            ls, cnt, gs, _ = o1_image(layers, P, params, images[i], labels[i], class_w,
                                      None if pix is None else pix[i], threads, need_probs=False)
        else:
            ls, cnt, gs, _ = o2.train_image(layers, params, images[i], labels[i], class_w, P)
        if cnt > 0:
            g += gs / cnt
            losses.append(ls / cnt)
        else:
            losses.append(0.0)
        nl.append(cnt)
    g /= n
    return {"loss": np.array(losses), "n_lab": np.array(nl), "grad": g, "params": params - lr * g}
