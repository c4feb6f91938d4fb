"""ORACLE O2 — the paper's whole-image algorithm, literally, on ragged fragments, fp64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA
path.  It follows PAPER.md §3 step by step in the paper's order and notation:

  * a storage F = {U_i f_i} is a list of fragments, each a stack of maps
    (§3.1); the input storage holds one fragment, the image;
  * every layer is applied to every fragment and the outputs are united
    (Alg. 1);
  * an MPF layer emits, per input fragment, one fragment per offset (r, c) of the
    k x k pooling kernel, MP_fwd(f(r:end, c:end), P), together with the argmax
    indices mpIDXS (Alg. 3).  Offsets are enumerated row-major
    (reading R2), partial blocks are dropped (floor rule, R5), ties go to the
    first maximum in row-major scan (R6);
  * the loss derivative w.r.t. the whole output image x_hat is formed first
    (PAPER.md:110-113), here MCCE with softmax (R15);
  * MPF backward places every output fragment's delta at its argmax in the source
    fragment and *accumulates* (Alg. 4, read as R3;
    Fig. 2 PAPER.md:143-145 "summed together");
  * parameter gradients are the sum over fragments of the per-fragment gradient
    (Alg. 2, with the layer input passed as in R4).

Library primitives used as single steps: numpy.tensordot (a matrix product) for
the per-(ky, kx) tap of a cross-correlation, numpy.argmax (first occurrence) for
the block maximum.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

CONV, POOL, FC = 0, 1, 2
TANH, IDENTITY, LOGISTIC = 0, 1, 2


@dataclass
class Fragment:
    """A stack of maps [C, h, w] and its offset lineage [(r, c, k), ...]."""
    maps: np.ndarray
    lineage: List[Tuple[int, int, int]] = field(default_factory=list)


def storage_from_image(image: np.ndarray) -> List[Fragment]:
    """Input storage of cardinality 1 holding the image."""
    img = np.asarray(image, np.float64)
    if img.ndim == 2:
        img = img[None]
    if img.size == 0:
        raise ValueError("empty image")
    return [Fragment(img.copy(), [])]


def expected_fragment_count(pool_factors) -> int:
    """|F_out| = |F_in| k^2 per MPF layer."""
    n = 1
    for k in pool_factors:
        if k < 1:
            raise ValueError("pool factor must be >= 1")
        n *= k * k
    return n


def lineage_to_pixel(lineage, m: int, n: int) -> Tuple[int, int]:
    """row = r1 + k1*(r2 + k2*(... (rL + kL*m))); col likewise."""
    row, col = m, n
    for (r, c, k) in reversed(lineage):
        row = r + k * row
        col = c + k * col
    return row, col


def _act(act, v):
    if act == TANH:
        return np.tanh(v)
    if act == LOGISTIC:
        return 1.0 / (1.0 + np.exp(-v))
    return v


def _act_d(act, y):
    if act == TANH:
        return 1.0 - y * y
    if act == LOGISTIC:
        return y * (1.0 - y)
    return np.ones_like(y)


# --------------------------------------------------------------------------- C / FC

def conv_fwd(f: Fragment, W: np.ndarray, b: np.ndarray, act: int) -> Fragment:
    """l->fwd(f) of a C (or FC-as-k x k-correlation) layer: valid cross-correlation,
    full connectivity, + bias, then the activation (R10, R12)."""
    x = f.maps
    co, ci, kr, kc = W.shape
    if x.shape[0] != ci:
        raise ValueError("channel mismatch")
    h, w = max(x.shape[1] - kr + 1, 0), max(x.shape[2] - kc + 1, 0)
    s = np.zeros((co, h, w))  # a fragment with no complete window stays empty (floor rule)
    for ky in range(kr):
        for kx in range(kc):
            s += np.tensordot(W[:, :, ky, kx], x[:, ky:ky + h, kx:kx + w], axes=(1, 0))
    s += b[:, None, None]
    return Fragment(_act(act, s), list(f.lineage))


def conv_grad(f_in: Fragment, f_out: Fragment, f_delta: Fragment, W: np.ndarray, act: int,
              need_input_delta: bool = True):
    """l->grad(f_delta) for one fragment (Alg. 2 body, R4): returns (gW, gb, delta_in).
    The activation derivative is taken from the stored output."""
    x = f_in.maps
    co, ci, kr, kc = W.shape
    dp = f_delta.maps * _act_d(act, f_out.maps)
    h, w = dp.shape[1], dp.shape[2]
    if h == 0 or w == 0:
        return np.zeros_like(W), np.zeros(co), (np.zeros_like(x) if need_input_delta else None)
    gW = np.zeros_like(W)
    for ky in range(kr):
        for kx in range(kc):
            gW[:, :, ky, kx] = np.tensordot(dp, x[:, ky:ky + h, kx:kx + w], axes=([1, 2], [1, 2]))
    gb = dp.sum(axis=(1, 2))
    din = None
    if need_input_delta:
        din = np.zeros_like(x)
        for ky in range(kr):
            for kx in range(kc):
                din[:, ky:ky + h, kx:kx + w] += np.tensordot(W[:, :, ky, kx], dp, axes=(0, 0))
    return gW, gb, din


# --------------------------------------------------------------------------- MP / MPF

def MP_fwd(maps: np.ndarray, k: int):
    """Non-overlapping k x k max pooling of a map stack, floor rule (R5).
    Returns (pooled [C, nh, nw], idx [C, nh, nw]) with idx = dy*k + dx, first max (R6)."""
    Cc, h, w = maps.shape
    nh, nw = h // k, w // k  # may be 0: the offset has no complete block (floor rule, R5)
    blk = maps[:, :nh * k, :nw * k].reshape(Cc, nh, k, nw, k).transpose(0, 1, 3, 2, 4)
    blk = blk.reshape(Cc, nh, nw, k * k)
    idx = np.argmax(blk, axis=3)  # first occurrence of the maximum
    pooled = np.take_along_axis(blk, idx[..., None], axis=3)[..., 0]
    return pooled, idx


def MP_bkp(delta: np.ndarray, idx: np.ndarray, k: int, shape) -> np.ndarray:
    """Place each pooled cell's delta at its recorded argmax."""
    out = np.zeros(shape)
    Cc, nh, nw = delta.shape
    dy, dx = idx // k, idx % k
    cc, ii, jj = np.meshgrid(np.arange(Cc), np.arange(nh), np.arange(nw), indexing="ij")
    np.add.at(out, (cc, ii * k + dy, jj * k + dx), delta)
    return out


def mpf_fwd(storage: List[Fragment], k: int):
    """Alg. 3: for each input fragment i, for j = 1..k^2: [r, c] = offset j (row-major, R2);
    [a, b] = MP_fwd(f_i(r:end, c:end), P); F_out U= a; mpIDXS U= b."""
    F_out, mpIDXS = [], []
    for f in storage:
        for j in range(k * k):
            r, c = divmod(j, k)
            a, b = MP_fwd(f.maps[:, r:, c:], k)
            F_out.append(Fragment(a, f.lineage + [(r, c, k)]))
            mpIDXS.append(b)
    return F_out, mpIDXS


def mpf_bkp(F_in: List[Fragment], F_delta_out: List[Fragment], mpIDXS, k: int) -> List[Fragment]:
    """Alg. 4 (R3): the output storage has as many fragments as F_in; for source
    fragment s and offset j the delta of output fragment s*k^2 + j is placed at its
    argmax inside f_s(r:end, c:end) and accumulated."""
    F_delta = [Fragment(np.zeros_like(f.maps), list(f.lineage)) for f in F_in]
    for i, fd in enumerate(F_delta_out):
        s, j = divmod(i, k * k)          # findSourceFragment(i, j)
        r, c = divmod(j, k)
        sub_shape = F_in[s].maps[:, r:, c:].shape
        F_delta[s].maps[:, r:, c:] += MP_bkp(fd.maps, mpIDXS[i], k, sub_shape)
    return F_delta


# --------------------------------------------------------------------------- network

def split_params(layers, params, in_channels=1):
    """Views (W, b) per parameterised layer in canonical order."""
    out, off, c = [], 0, in_channels
    for L in layers:
        if L.kind in (CONV, FC):
            n = L.n_out * c * L.k * L.k
            W = params[off:off + n].reshape(L.n_out, c, L.k, L.k)
            off += n
            b = params[off:off + L.n_out]
            off += L.n_out
            out.append((W, b))
            c = L.n_out
        else:
            out.append(None)
    if off != len(params):
        raise ValueError(f"parameter count mismatch: {off} != {len(params)}")
    return out


def forward_dense(layers, params, image, in_channels=1):
    """Whole-image forward (Alg. 1 per layer, Alg. 3 for MPF). Returns the tape:
    list of storages (input of every layer + final), and the mpIDXS per layer."""
    wb = split_params(layers, np.asarray(params, np.float64), in_channels)
    S = storage_from_image(image)
    tape, idxs = [S], []
    for L, p in zip(layers, wb):
        if L.kind == POOL:
            S, ix = mpf_fwd(S, L.k)
            idxs.append(ix)
        else:
            W, b = p
            S = [conv_fwd(f, W, b, L.act) for f in S]  # Alg. 1: F_out = F_out U l->fwd(f_i)
            idxs.append(None)
        tape.append(S)
    return tape, idxs


def defragment(storage: List[Fragment], O_H: int, O_W: int, audit: bool = True) -> np.ndarray:
    """Scatter every fragment value to lineage_to_pixel coordinates."""
    Cc = storage[0].maps.shape[0]
    out = np.zeros((Cc, O_H, O_W))
    cnt = np.zeros((O_H, O_W), np.int64)
    for f in storage:
        _, h, w = f.maps.shape
        for m in range(h):
            for n in range(w):
                y, x = lineage_to_pixel(f.lineage, m, n)
                if y < O_H and x < O_W:
                    out[:, y, x] = f.maps[:, m, n]
                    cnt[y, x] += 1
                elif audit:
                    raise AssertionError(f"fragment position maps outside the output grid: {(y, x)}")
    if audit and not np.all(cnt == 1):
        raise AssertionError("defragment write-count audit failed")
    return out


def _softmax(z):
    z = z - z.max(axis=0, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=0, keepdims=True)


def train_image(layers, params, image, labels, class_w=None, P=None, in_channels=1, need_grad=True):
    """Whole image: forward, MCCE over labelled output pixels, backward.

    Returns (loss_sum, n_lab, grad_sum, probs[C, O_H, O_W]) with the same
    conventions as O1 (sums over labelled pixels; R8 divides by n_lab later)."""
    params = np.asarray(params, np.float64)
    image = np.asarray(image, np.float64)
    if image.ndim == 2:
        image = image[None]
    H, W = image.shape[1:]
    O_H, O_W = labels.shape if labels is not None else (H - P + 1, W - P + 1)
    wb = split_params(layers, params, in_channels)
    tape, idxs = forward_dense(layers, params, image, in_channels)
    final = tape[-1]
    Cc = final[0].maps.shape[0]
    probs = np.zeros((Cc, O_H, O_W))
    loss, n_lab = 0.0, 0
    # dL/dx_hat per fragment (first step of back-propagation)
    deltas = []
    for f in final:
        p = _softmax(f.maps)
        d = np.zeros_like(p)
        _, h, w = p.shape
        for m in range(h):
            for n in range(w):
                y, x = lineage_to_pixel(f.lineage, m, n)
                if y >= O_H or x >= O_W:
                    continue
                probs[:, y, x] = p[:, m, n]
                if labels is None:
                    continue
                t = int(labels[y, x])
                if t == 255:
                    continue
                if t >= Cc:
                    raise ValueError("label out of range")
                wt = 1.0 if class_w is None else float(class_w[t])
                loss += -wt * np.log(p[t, m, n])
                n_lab += 1
                d[:, m, n] = wt * p[:, m, n]
                d[t, m, n] -= wt
        deltas.append(Fragment(d, list(f.lineage)))
    if not need_grad:
        return loss, n_lab, None, probs
    grads = [None] * len(layers)
    Fd = deltas
    for li in range(len(layers) - 1, -1, -1):
        L = layers[li]
        F_in, F_out = tape[li], tape[li + 1]
        if L.kind == POOL:
            Fd = mpf_bkp(F_in, Fd, idxs[li], L.k)
        else:
            W, b = wb[li]
            gW, gb = np.zeros_like(W), np.zeros_like(b)
            new = []
            for fi, fo, fd in zip(F_in, F_out, Fd):      # Alg. 2: g = g + l->grad(f_i^delta)
                a, bb, din = conv_grad(fi, fo, fd, W, L.act, need_input_delta=li > 0)
                gW += a
                gb += bb
                new.append(Fragment(din, list(fi.lineage)) if din is not None else None)
            grads[li] = (gW, gb)
            Fd = new
    flat = np.concatenate([np.concatenate([g[0].ravel(), g[1]]) for g in grads if g is not None])
    return loss, n_lab, flat, probs


def auto_class_weights(labels: np.ndarray, C: int) -> Tuple[np.ndarray, np.ndarray]:
    """Per-class loss weights of the unbalanced-data MCCE (SURVEY §8(f) item 3,
    the inverse-frequency rule w_c = N / (C n_c) of SPEC.md:417-421).  labels: any shape,
    uint8, 255 = ignored.  Returns (weights fp64 [C], counts int [C]); raises on an
    absent class."""
    lab = np.asarray(labels).reshape(-1)
    lab = lab[lab < C]
    counts = np.bincount(lab.astype(np.int64), minlength=C)[:C]
    if np.any(counts == 0):
        raise ValueError("auto class weights: a class has no labelled pixel")
    N = counts.sum()
    return N / (C * counts.astype(np.float64)), counts


def mirror_pad(image: np.ndarray, P: int) -> np.ndarray:
    """Same-size output: the image [..., H, W] mirror-padded by floor((P-1)/2)
    before and P-1-floor((P-1)/2) after each spatial axis, reflecting about the border pixel
    without repeating it (numpy's 'reflect' mode; reading R20)."""
    pt = (P - 1) // 2
    pads = [(0, 0)] * (image.ndim - 2) + [(pt, P - 1 - pt), (pt, P - 1 - pt)]
    return np.pad(image, pads, mode="reflect")


def armijo_step(eval_loss_grad, eval_loss, theta: np.ndarray, alpha0: float, beta: float, c: float,
                max_backtracks: int):
    """Armijo-safeguarded gradient step, written out: L0, g at
    theta; alpha = alpha0, alpha0 beta, ...; accept the first theta - alpha g with
    L <= L0 - c alpha ||g||^2; else keep theta.  Returns (theta_new, alpha or 0, L, accepted,
    evaluations)."""
    L0, g = eval_loss_grad(theta)
    g2 = float(np.dot(g.ravel(), g.ravel()))
    alpha = alpha0
    for it in range(max_backtracks + 1):
        t = theta - alpha * g
        L = eval_loss(t)
        if np.isfinite(L) and L <= L0 - c * alpha * g2:
            return t, alpha, L, True, it + 1
        alpha *= beta
    return theta, 0.0, L0, False, max_backtracks + 1


def lbfgs_two_loop(g: np.ndarray, S: List[np.ndarray], Y: List[np.ndarray]) -> np.ndarray:
    """r = H_k g by the L-BFGS two-loop recursion ("two-loop recursion
    direction"; "We use LBFGS"), pairs oldest first, H_k^0 = gamma I with
    gamma = s_{k-1}^T y_{k-1} / y_{k-1}^T y_{k-1} (1 with no pairs; reading R21)."""
    q = g.astype(np.float64).copy()
    a = [0.0] * len(S)
    for i in reversed(range(len(S))):          # newest to oldest
        rho = 1.0 / float(np.dot(S[i], Y[i]))
        a[i] = rho * float(np.dot(S[i], q))
        q = q - a[i] * Y[i]
    gamma = float(np.dot(S[-1], Y[-1])) / float(np.dot(Y[-1], Y[-1])) if S else 1.0
    r = gamma * q
    for i in range(len(S)):                    # oldest to newest
        rho = 1.0 / float(np.dot(S[i], Y[i]))
        b = rho * float(np.dot(Y[i], r))
        r = r + (a[i] - b) * S[i]
    return r


def lbfgs_step(state: dict, theta: np.ndarray, eval_loss_grad, memory: int, alpha0: float, beta: float, c: float,
               max_backtracks: int, sy_min: float = 1e-10):
    """One full-batch L-BFGS iteration, written out:

      (L, g) at theta (kept in `state` from the previous accepted trial);
      d = -H g by the two-loop recursion; if g^T d >= 0, d = -g (steepest descent);
      alpha = alpha0 with no pairs, 1 otherwise (reading R21); backtrack alpha <- beta alpha
      until L(theta + alpha d) <= L + c alpha g^T d (Armijo along d);
      accepted: s = theta_new - theta, y = g_new - g, the pair kept iff s^T y > sy_min,
      the oldest dropped beyond `memory`; exhausted: theta unchanged, pairs cleared (R21).

    state: {"S": [...], "Y": [...], "L": float or None, "g": array or None}, updated in place.
    Returns (theta_new, alpha or 0, L_before, L_after, accepted, evaluations, fallback)."""
    if state.get("g") is None:
        state["L"], state["g"] = eval_loss_grad(theta)
    S, Y = state.setdefault("S", []), state.setdefault("Y", [])
    L0, g = state["L"], state["g"]
    d = -lbfgs_two_loop(g, S, Y)
    gtd = float(np.dot(g, d))
    fallback = not (gtd < 0.0)
    if fallback:
        d = -g
        gtd = -float(np.dot(g, g))
    alpha = alpha0 if not S else 1.0
    for it in range(max_backtracks + 1):
        t = theta + alpha * d
        Lt, gt = eval_loss_grad(t)
        if np.isfinite(Lt) and Lt <= L0 + c * alpha * gtd:
            s, y = t - theta, gt - g
            if float(np.dot(s, y)) > sy_min:
                S.append(s)
                Y.append(y)
                if len(S) > memory:
                    del S[0], Y[0]
            state["L"], state["g"] = Lt, gt
            return t, alpha, L0, Lt, True, it + 1, fallback
        alpha *= beta
    S.clear()
    Y.clear()
    return theta, 0.0, L0, L0, False, max_backtracks + 1, fallback
