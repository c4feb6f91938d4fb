"""Seeded synthetic inputs shared by the oracle and the B200 path.

This module is deliberately *method-free*: it holds the five BASELINE.json
configurations (layer lists, image sizes, batch sizes), the seeded image/label
generators and the weight initialiser.  It contains none of the method's
arithmetic (no convolution, pooling, fragment or loss code), so that the oracle
(`oracle/`) and the product (`paper_1302_1690_b200/`) can both draw their
inputs from it without sharing any computation (task rule ③).

Recipes (DESIGN.md §"Synthetic inputs"):
  * The paper's data (ISBI-2012 EM slices; the proprietary
    ArcelorMittal steel set) is not available.  Seeded
    synthetic images with the BASELINE.json shapes stand in for them; no item of
    either dataset is reproduced.
  * Images are fp32, standardised to mean 0 / variance 1.  Labels are uint8 on
    the *output grid* [O_H, O_W], O = H - P + 1 (reading R7): output
    (y, x) is the patch whose top-left pixel is (y, x); its label is the pixel
    label at the patch centre (y + c, x + c), c = (P - 1) // 2.  255 = ignore.
  * Weights and biases ~ U(+-1/sqrt(fan_in)), fan_in = C_in * k * k (R13),
    drawn once on the host in fp64 (numpy PCG64) and handed identically to
    the oracle and to the GPU path.
  * Seeds: data_seed = 1000 + cfg, weight_seed = 2000 + cfg, per-image seed =
    data_seed * 10**6 + image_index (any rank can generate its own shard).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

try:  # scipy is in the image; the fallback keeps the module importable anyway
    from scipy.ndimage import gaussian_filter as _gauss
except Exception:  # pragma: no cover
    _gauss = None

CONV, POOL, FC = 0, 1, 2
TANH, IDENTITY, LOGISTIC = 0, 1, 2
IGNORE = 255


@dataclass(frozen=True)
class Layer:
    """One layer of an MPCNN (§2).

    kind  CONV: k x k valid cross-correlation + activation (n_out maps)
          POOL: k x k max pooling (an MPF layer in whole-image mode, §3.2)
          FC:   fully-connected over the remaining k x k x C volume (the first
                FC; k = 1 for later FCs), evaluated over fragments as a k x k
                convolution (north_star; reading R12).
    """
    kind: int
    k: int
    n_out: int = 0
    act: int = TANH


def C(k, n, act=TANH):
    return Layer(CONV, k, n, act)


def MP(k):
    return Layer(POOL, k, 0, IDENTITY)


def F(k, n, act=TANH):
    return Layer(FC, k, n, act)


@dataclass(frozen=True)
class Config:
    name: str
    index: int
    P: int                      # patch size = receptive field (R1)
    H: int
    W: int
    n_images: int               # images in the workload
    global_batch: int           # images per SGD step (R14)
    classes: int
    layers: Tuple[Layer, ...]
    recipe: str
    lr: float = 0.01
    in_channels: int = 1
    description: str = ""

    @property
    def out_rows(self) -> int:
        return self.H - self.P + 1

    @property
    def out_cols(self) -> int:
        return self.W - self.P + 1

    @property
    def steps(self) -> int:
        return self.n_images // self.global_batch


CONFIGS = {
    # BASELINE.json configs[0]
    "cfg1": Config("cfg1", 1, 14, 32, 32, 1, 1, 2,
                   (C(3, 4), MP(2), C(3, 8), MP(2), F(2, 16), F(1, 2, IDENTITY)),
                   "iid", description="tiny net, one 32x32 N(0,1) image, ellipse labels"),
    # configs[1]
    "cfg2": Config("cfg2", 2, 44, 128, 128, 8, 8, 2,
                   (C(5, 16), MP(2), C(5, 32), MP(2), C(3, 48), MP(2), F(3, 100), F(1, 2, IDENTITY)),
                   "bandlimited", description="8 x 128^2 band-limited texture, 1-3 ellipse defects"),
    # configs[2]: same architecture, 64 images of 512^2, one epoch of per-image SGD
    "cfg3": Config("cfg3", 3, 44, 512, 512, 64, 1, 2,
                   (C(5, 16), MP(2), C(5, 32), MP(2), C(3, 48), MP(2), F(3, 100), F(1, 2, IDENTITY)),
                   "steel", description="64 x 512^2 steel-like texture, elongated blobs ~3%"),
    # configs[3]: P = 94 is the receptive field of the stated layer list (R1; BASELINE says 96)
    "cfg4": Config("cfg4", 4, 94, 1024, 1024, 256, 8, 5,
                   (C(7, 32), MP(2), C(5, 64), MP(2), C(5, 96), MP(2), C(3, 128), MP(2),
                    F(3, 200), F(1, 5, IDENTITY)),
                   "steel5", description="256 x 1024^2, 4 defect classes + background"),
    # configs[4]: P = 84 is the receptive field of the stated layer list (R1; BASELINE says 90)
    "cfg5": Config("cfg5", 5, 84, 768, 768, 128, 8, 2,
                   (C(4, 24), MP(3), C(4, 48), MP(3), C(3, 64), MP(3), F(2, 128), F(1, 2, IDENTITY)),
                   "bandlimited10", description="128 x 768^2, pooling stress, ~10% positive"),
}


def param_shapes(layers, in_channels: int = 1) -> List[Tuple[Tuple[int, int, int, int], int]]:
    """(W shape [n_out, C_in, k, k], n_bias) for every CONV/FC layer, in layer order.

    Canonical flat order: layer order; within a layer
    W[out][in][kr][kc] row-major, then b[out].
    """
    shapes = []
    c = in_channels
    for L in layers:
        if L.kind in (CONV, FC):
            shapes.append(((L.n_out, c, L.k, L.k), L.n_out))
            c = L.n_out
    return shapes


def n_params(layers, in_channels: int = 1) -> int:
    return sum(int(np.prod(w)) + b for w, b in param_shapes(layers, in_channels))


def init_params(cfg_or_layers, seed: int | None = None, in_channels: int = 1) -> np.ndarray:
    """Flat fp64 parameters, W and b ~ U(+-1/sqrt(fan_in)) (R13)."""
    if isinstance(cfg_or_layers, Config):
        layers, in_channels = cfg_or_layers.layers, cfg_or_layers.in_channels
        seed = 2000 + cfg_or_layers.index if seed is None else seed
    else:
        layers = cfg_or_layers
        seed = 0 if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for (w, b) in param_shapes(layers, in_channels):
        bound = 1.0 / np.sqrt(w[1] * w[2] * w[3])
        out.append(rng.uniform(-bound, bound, size=int(np.prod(w))))
        out.append(rng.uniform(-bound, bound, size=b))
    return np.concatenate(out).astype(np.float64)


# ----------------------------------------------------------------------------
# images and labels
# ----------------------------------------------------------------------------

def _smooth(x, sigma):
    if _gauss is not None:
        return _gauss(x, sigma, mode="wrap")
    # FFT fallback (periodic), same effect
    H, W = x.shape
    sy, sx = (sigma, sigma) if np.isscalar(sigma) else sigma
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.fftfreq(W)[None, :]
    g = np.exp(-2 * (np.pi ** 2) * ((sy * fy) ** 2 + (sx * fx) ** 2))
    return np.real(np.fft.ifft2(np.fft.fft2(x) * g))


def _standardise(x):
    x = x - x.mean()
    s = x.std()
    return x / (s if s > 0 else 1.0)


def _ellipse(H, W, cy, cx, a, b, theta):
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    dy, dx = yy - cy, xx - cx
    c, s = np.cos(theta), np.sin(theta)
    u = (c * dx + s * dy) / a
    v = (-s * dx + c * dy) / b
    return (u * u + v * v) <= 1.0


def _line(H, W, y0, x0, theta, length, width):
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    dy, dx = yy - y0, xx - x0
    c, s = np.cos(theta), np.sin(theta)
    along = c * dx + s * dy
    across = -s * dx + c * dy
    return (np.abs(across) <= width / 2.0) & (np.abs(along) <= length / 2.0)


def make_image(cfg: Config, idx: int) -> Tuple[np.ndarray, np.ndarray]:
    """Seeded image (fp32 [H, W], mean 0 var 1) and per-pixel labels (uint8 [H, W])."""
    seed = (1000 + cfg.index) * 10 ** 6 + idx
    rng = np.random.Generator(np.random.PCG64(seed))
    H, W = cfg.H, cfg.W
    lab = np.zeros((H, W), np.uint8)
    r = cfg.recipe
    if r == "iid":
        img = rng.standard_normal((H, W))
        a, b = rng.uniform(4, 12, 2)
        m = _ellipse(H, W, rng.uniform(0, H), rng.uniform(0, W), a, b, rng.uniform(0, np.pi))
        lab[m] = 1
        return img.astype(np.float32), lab
    if r in ("bandlimited", "bandlimited10"):
        tex = _standardise(_smooth(rng.standard_normal((H, W)), 2.0))
        target = 0.05 if r == "bandlimited" else 0.10
        n_def = int(rng.integers(1, 4))
        area = target * H * W / n_def
        for _ in range(n_def):
            asp = rng.uniform(1.0, 2.5)
            a = np.sqrt(area * asp / np.pi)
            m = _ellipse(H, W, rng.uniform(0, H), rng.uniform(0, W), a, a / asp, rng.uniform(0, np.pi))
            lab[m] = 1
        tex = tex + 1.5 * lab
        return _standardise(tex).astype(np.float32), lab
    if r in ("steel", "steel5"):
        # anisotropic Gaussian-filtered noise with rolling streaks (sigma_row ~1, sigma_col ~6-8)
        tex = _smooth(rng.standard_normal((H, W)), (1.0, rng.uniform(6.0, 8.0)))
        streak = _smooth(rng.standard_normal((H, 1)), (3.0, 0.0)) * 0.8
        tex = _standardise(tex) + streak
        if r == "steel":
            n_def = int(rng.integers(1, 4))
            area = 0.03 * H * W / n_def
            for _ in range(n_def):
                asp = rng.uniform(3.0, 8.0)
                a = np.sqrt(area * asp / np.pi)
                m = _ellipse(H, W, rng.uniform(0, H), rng.uniform(0, W), a, a / asp,
                             rng.uniform(-0.3, 0.3))
                lab[m] = 1
                tex = tex + (2.0 if rng.uniform() < 0.5 else -2.0) * m
            return _standardise(tex).astype(np.float32), lab
        # steel5: classes 1 bright ellipse, 2 dark ellipse, 3 bright line, 4 dark line
        for cls in (1, 2):
            for _ in range(int(rng.integers(1, 3))):
                asp = rng.uniform(2.0, 6.0)
                a = rng.uniform(0.02, 0.06) * H
                m = _ellipse(H, W, rng.uniform(0, H), rng.uniform(0, W), a, a / asp,
                             rng.uniform(0, np.pi))
                lab[m] = cls
                tex = tex + (2.0 if cls == 1 else -2.0) * m
        for cls in (3, 4):
            for _ in range(int(rng.integers(1, 3))):
                m = _line(H, W, rng.uniform(0, H), rng.uniform(0, W), rng.uniform(0, np.pi),
                          rng.uniform(0.2, 0.6) * W, rng.uniform(2.0, 4.0))
                lab[m] = cls
                tex = tex + (2.5 if cls == 3 else -2.5) * m
        return _standardise(tex).astype(np.float32), lab
    raise ValueError(f"unknown recipe {r}")


def output_labels(pix_labels: np.ndarray, P: int) -> np.ndarray:
    """Pixel labels -> labels on the output grid (R7): out[y, x] = pix[y + c, x + c]."""
    H, W = pix_labels.shape
    c = (P - 1) // 2
    return np.ascontiguousarray(pix_labels[c:c + H - P + 1, c:c + W - P + 1])


def make_batch(cfg: Config, indices) -> Tuple[np.ndarray, np.ndarray]:
    """images fp32 [n, 1, H, W]; labels uint8 [n, O_H, O_W] (output grid)."""
    imgs, labs = [], []
    for i in indices:
        im, lb = make_image(cfg, int(i))
        imgs.append(im[None])
        labs.append(output_labels(lb, cfg.P))
    return np.stack(imgs).astype(np.float32), np.stack(labs).astype(np.uint8)


def random_arch_case(rng: np.random.Generator):
    """A small random MPCNN (for randomized oracle/GPU property tests).

    Returns (layers, P).  1-2 pooling layers with k in {2, 3}; the head is one FC
    over the remaining s x s volume, optionally a hidden FC, then the linear FC.
    The patch size P is built backwards from the head so patch-mode geometry is
    exact — this is input generation, not method arithmetic.
    """
    n_pool = int(rng.integers(1, 3))
    classes = int(rng.integers(2, 4))
    s = int(rng.integers(1, 3))
    layers = []
    size = s
    blocks = []
    for _ in range(n_pool):
        kc = int(rng.integers(1, 4))
        kp = int(rng.choice([2, 3]))
        blocks.append((kc, kp, int(rng.integers(2, 5))))
    # walk backwards: FC needs s; before FC a pool (k) after a conv (kc)
    for kc, kp, n in reversed(blocks):
        size = size * kp + kc - 1
    P = size
    for kc, kp, n in blocks:
        layers += [C(kc, n), MP(kp)]
    hidden = int(rng.integers(3, 7))
    layers.append(F(s, hidden))
    if rng.uniform() < 0.5:
        layers.append(F(1, int(rng.integers(2, 5))))
    layers.append(F(1, classes, IDENTITY))
    return tuple(layers), P


def random_labels(rng, n, O_H, O_W, classes, ignore_frac=0.1):
    lab = rng.integers(0, classes, size=(n, O_H, O_W)).astype(np.uint8)
    if ignore_frac > 0:
        lab[rng.uniform(size=lab.shape) < ignore_frac] = IGNORE
    return lab
