"""Pins for the oracles (O1 patch-by-patch C, O2 literal Alg. 1-4 numpy).

Each test pins the oracle to something *other than itself*: the paper's / SPEC's
worked examples (tests/golden/), closed forms, finite differences, brute force,
the independent library special case (torch fp64 dilated conv + stride-1 dilated
max-pool + autograd), and O1 == O2 (two independent programs written from the
paper).  Chosen so a plausible slip (dropped bias, wrong tap orientation, wrong
offset order, missing accumulation, wrong normalisation) fails at least one.
"""
import math

import numpy as np
import pytest

import mpf_synth as S
import oracle
from oracle import o2
from tests.conftest import golden_lines

CONV, POOL, FC = S.CONV, S.POOL, S.FC


# ----------------------------------------------------------------- golden examples

def test_golden_mpf_4x4():
    lines = golden_lines("mpf_4x4_k2.txt")
    x = np.array([[float(v) for v in lines[i].split()] for i in range(1, 5)])
    k = int(lines[5].split()[1])
    want = np.array([[float(v) for v in lines[i].split()] for i in (7, 8)])
    sizes = lines[9].split()[1:]
    F_out, idx = o2.mpf_fwd(o2.storage_from_image(x), k)
    assert len(F_out) == 4
    np.testing.assert_array_equal(F_out[0].maps[0], want)
    got_sizes = [f"{f.maps.shape[1]}x{f.maps.shape[2]}" for f in F_out]
    assert got_sizes == sizes
    # patch-mode MP is the offset-(0,0) fragment
    pooled, _ = o2.MP_fwd(x[None], 2)
    np.testing.assert_array_equal(pooled[0], want)


def test_golden_mp_patch_examples():
    # [[1,2],[3,4]] -> [[4]]; 5x5 -> 2x2 (floor rule)
    p, i = o2.MP_fwd(np.array([[[1.0, 2.0], [3.0, 4.0]]]), 2)
    assert p.shape == (1, 1, 1) and p[0, 0, 0] == 4.0 and i[0, 0, 0] == 3
    p, _ = o2.MP_fwd(np.random.default_rng(0).standard_normal((1, 5, 5)), 2)
    assert p.shape == (1, 2, 2)


def test_golden_lineage():
    for ln in golden_lines("lineage.txt"):
        lin_s, mn, rc = [s.strip() for s in ln.split("|")]
        lineage = [tuple(int(v) for v in e.split(",")) for e in lin_s.split(";")] if lin_s else []
        m, n = (int(v) for v in mn.split())
        want = tuple(int(v) for v in rc.split())
        assert o2.lineage_to_pixel(lineage, m, n) == want


def test_golden_fragment_count_and_brute_force():
    for ln in golden_lines("fragment_count.txt"):
        lhs, rhs = ln.split("->")
        ks = [] if lhs.strip() == "-" else [int(v) for v in lhs.split(",")]
        want = int(rhs)
        assert o2.expected_fragment_count(ks) == want
        # brute force: chain MPF layers on a real storage and count
        Sg = o2.storage_from_image(np.random.default_rng(1).standard_normal((23, 23)))
        for k in ks:
            Sg, _ = o2.mpf_fwd(Sg, k)
        assert len(Sg) == want


def test_golden_mcce():
    lines = golden_lines("mcce.txt")
    logits = [float(v) for v in lines[0].split()[1:]]
    t = int(lines[1].split()[1])
    loss = float(lines[2].split()[1])
    delta = [float(v) for v in lines[3].split()[1:]]
    # a 1x1 "image" through a single linear FC whose output equals the logits:
    # W = 0, b = logits (closed form: logits do not depend on the input)
    layers = (S.F(1, 2, S.IDENTITY),)
    params = np.array([0.0, 0.0] + logits)
    img = np.array([[[0.37]]])
    lab = np.array([[t]], np.uint8)
    for eng in ("o1", "o2"):
        if eng == "o1":
            ls, n, g, pr = oracle.o1_image(layers, 1, params, img, lab)
        else:
            ls, n, g, pr = o2.train_image(layers, params, img, lab, P=1)
        assert n == 1
        assert ls == pytest.approx(loss, abs=1e-15)
        # dL/db = delta (the bias gradient of the logit layer), dL/dW = delta * x
        np.testing.assert_allclose(g[2:], delta, atol=1e-15)
        np.testing.assert_allclose(g[:2], np.array(delta) * 0.37, atol=1e-15)


def test_mcce_saturation_and_class_weight():
    # saturated correct pixel -> loss 0 and delta 0; w doubles both
    layers = (S.F(1, 2, S.IDENTITY),)
    img = np.array([[[1.0]]])
    lab = np.array([[1]], np.uint8)
    ls, n, g, _ = oracle.o1_image(layers, 1, np.array([0.0, 0.0, -400.0, 400.0]), img, lab)
    assert ls == pytest.approx(0.0, abs=1e-300) and np.all(np.abs(g) < 1e-300)
    p = np.array([0.3, -0.2, 0.1, 0.05])
    l1, _, g1, _ = oracle.o1_image(layers, 1, p, img, lab, class_w=[1.0, 1.0])
    l2, _, g2, _ = oracle.o1_image(layers, 1, p, img, lab, class_w=[1.0, 2.0])
    assert l2 == pytest.approx(2 * l1, rel=1e-15)
    np.testing.assert_allclose(g2, 2 * g1, rtol=1e-15)


def test_golden_conv():
    vals = dict(ln.split() for ln in golden_lines("conv.txt"))
    f = o2.Fragment(np.ones((1, 4, 4)))
    out = o2.conv_fwd(f, np.ones((1, 1, 3, 3)), np.zeros(1), S.IDENTITY)
    assert out.maps.shape == (1, 2, 2) and np.all(out.maps == float(vals["ones3x3_on_ones4x4"]))
    f = o2.Fragment(np.random.default_rng(2).standard_normal((1, 5, 5)))
    out = o2.conv_fwd(f, np.zeros((1, 1, 3, 3)), np.zeros(1), S.IDENTITY)
    assert out.maps.shape == (1, 3, 3) and np.all(out.maps == float(vals["zero_kernel_5x5"]))
    # tanh(0) = 0
    out = o2.conv_fwd(o2.Fragment(np.zeros((1, 2, 2))), np.ones((1, 1, 1, 1)), np.zeros(1), S.TANH)
    assert np.all(out.maps == 0.0)


def test_cross_correlation_orientation_closed_form():
    # R10: cross-correlation, no flip.  A kernel with a single 1 at (0,1) shifts the image left.
    x = np.arange(20, dtype=float).reshape(1, 4, 5)
    W = np.zeros((1, 1, 2, 2))
    W[0, 0, 0, 1] = 1.0
    out = o2.conv_fwd(o2.Fragment(x), W, np.array([0.5]), S.IDENTITY)
    np.testing.assert_array_equal(out.maps[0], x[0, :3, 1:5] + 0.5)
    # the same through O1: P=2 net with a single FC(2) layer (a 2x2 correlation)
    W2 = np.zeros((2, 1, 2, 2))
    W2[0, 0, 0, 1] = 1.0
    params = np.concatenate([W2.ravel(), [0.5, 0.0]])
    layers = (S.F(2, 2, S.IDENTITY),)
    _, _, _, pr = oracle.o1_image(layers, 2, params, x, None, need_grad=False)
    logit = x[0, :3, 1:5] + 0.5  # class-0 logit; class-1 logit is 0
    p0 = 1.0 / (1.0 + np.exp(-logit))
    np.testing.assert_allclose(pr[:, 0], p0.ravel(), rtol=1e-14)


def test_golden_patch_count():
    lines = golden_lines("patch_count.txt")
    H, W = (int(v) for v in lines[0].split()[1:])
    want = int(lines[1].split()[1])
    # one patch per output pixel; a same-size output of an HxW image (mirror padding
    # by P-1 rows/cols) has (H+P-1-P+1)(W+P-1-P+1) = H*W outputs
    P = 8
    layers = (S.C(3, 2), S.MP(2), S.F(3, 2, S.IDENTITY))
    img = np.random.default_rng(3).standard_normal((H + P - 1, W + P - 1))
    _, _, _, pr = oracle.o1_image(layers, P, S.init_params(layers, 1), img, None, need_grad=False)
    assert pr.shape[0] == want == H * W


# ----------------------------------------------------------------- MPF backward

def test_mpf_backward_examples_and_shared_max():
    # SPEC.md:160-162; PAPER.md:143-145 (Fig. 2): an element that is the max for
    # offsets (0,0) and (1,1) receives the sum a + b
    x = np.array([[[0.1, 0.2, 0.3], [0.4, 1.0, 0.5], [0.6, 0.7, 0.8]]])
    F_in = o2.storage_from_image(x)
    F_out, idx = o2.mpf_fwd(F_in, 2)
    # offset (0,0) block rows 0-1 cols 0-1 -> max 1.0 at (1,1); offset (1,1) block rows 1-2 cols 1-2 -> 1.0
    assert F_out[0].maps[0, 0, 0] == 1.0 and F_out[3].maps[0, 0, 0] == 1.0
    a, b = 0.25, -0.75
    deltas = [o2.Fragment(np.zeros_like(f.maps)) for f in F_out]
    deltas[0].maps[0, 0, 0] = a
    deltas[3].maps[0, 0, 0] = b
    d_in = o2.mpf_bkp(F_in, deltas, idx, 2)
    want = np.zeros_like(x)
    want[0, 1, 1] = a + b
    np.testing.assert_array_equal(d_in[0].maps, want)
    # zeros in -> zeros out
    z = o2.mpf_bkp(F_in, [o2.Fragment(np.zeros_like(f.maps)) for f in F_out], idx, 2)
    assert np.all(z[0].maps == 0)


@pytest.mark.parametrize("k", [2, 3])
def test_mpf_adjoint(k):
    # <selection(x), d> = <x, mpf_bkp(d)> for a fixed argmax pattern
    rng = np.random.default_rng(10 + k)
    x = rng.standard_normal((3, 17, 19))
    F_in = o2.storage_from_image(x)
    F_out, idx = o2.mpf_fwd(F_in, k)
    d = [o2.Fragment(rng.standard_normal(f.maps.shape)) for f in F_out]
    lhs = sum(float((f.maps * dd.maps).sum()) for f, dd in zip(F_out, d))
    rhs = float((x * o2.mpf_bkp(F_in, d, idx, k)[0].maps).sum())
    assert lhs == pytest.approx(rhs, rel=1e-12)
    assert len(F_out) == k * k


# ----------------------------------------------------------------- counts / coverage

@pytest.mark.parametrize("ks,kc", [((2,), 3), ((3,), 2), ((2, 2), 2), ((2, 3), 2), ((3, 2), 1), ((2, 2, 2), 1)])
def test_coverage_audit_and_counts(ks, kc):
    # SPEC.md:284-285 / 621: every output pixel written exactly once (defragment audit),
    # output count = (H-P+1)(W-P+1), fragment count = prod k^2
    rng = np.random.default_rng(sum(ks) * 7 + kc)
    s = 1
    layers = []
    size = s
    for k in reversed(ks):
        size = size * k + kc - 1
    for k in ks:
        layers += [S.C(kc, 2), S.MP(k)]
    layers += [S.F(s, 2, S.IDENTITY)]
    P = size
    for H, W in [(17, 23), (29, 40), (P, P + 3)]:
        if H < P or W < P:
            continue
        img = rng.standard_normal((H, W))
        params = S.init_params(tuple(layers), 5)
        tape, _ = o2.forward_dense(tuple(layers), params, img)
        final = tape[-1]
        assert len(final) == o2.expected_fragment_count(ks)
        out = o2.defragment(final, H - P + 1, W - P + 1, audit=True)  # raises on a miss/double write
        assert out.shape[1] * out.shape[2] == (H - P + 1) * (W - P + 1)


def test_configs_fragment_and_output_counts():
    # SURVEY.md §8(c) pins: F = prod k^2 ; O = H - P + 1 (configs 1-5, R1 patch sizes)
    want = {"cfg1": (16, 19), "cfg2": (64, 85), "cfg3": (64, 469), "cfg4": (256, 931), "cfg5": (729, 685)}
    for name, (F, O) in want.items():
        cfg = S.CONFIGS[name]
        ks = [L.k for L in cfg.layers if L.kind == POOL]
        assert o2.expected_fragment_count(ks) == F
        assert cfg.out_rows == O
        assert oracle.o1_n_params(cfg.layers, cfg.P) == S.n_params(cfg.layers)
    assert S.n_params(S.CONFIGS["cfg1"].layers) == 898
    assert S.n_params(S.CONFIGS["cfg2"].layers) == 70622
    assert S.n_params(S.CONFIGS["cfg4"].layers) == 548885
    assert S.n_params(S.CONFIGS["cfg5"].layers) == 79754


def test_o1_rejects_inexact_geometry():
    # architectures failing exact divisibility are rejected (R1: P=96 for cfg4)
    cfg = S.CONFIGS["cfg4"]
    assert oracle.o1_n_params(cfg.layers, 96) < 0
    assert oracle.o1_n_params(cfg.layers, 94) > 0
    assert oracle.o1_n_params(S.CONFIGS["cfg5"].layers, 90) < 0


def test_zero_weight_model_uniform():
    # all-zero weights -> uniform 1/C, loss ln C
    cfg = S.CONFIGS["cfg1"]
    im, lab = S.make_batch(cfg, [0])
    p = np.zeros(S.n_params(cfg.layers))
    ls, n, _, pr = oracle.o1_image(cfg.layers, cfg.P, p, im[0], lab[0])
    np.testing.assert_allclose(pr, 0.5, atol=0)
    assert ls / n == pytest.approx(math.log(2), rel=1e-15)
    ls2, n2, _, pr2 = o2.train_image(cfg.layers, p, im[0], lab[0], P=cfg.P)
    np.testing.assert_allclose(pr2, 0.5, atol=0)


# ----------------------------------------------------------------- finite differences

def _tiny():
    layers = (S.C(3, 2), S.MP(2), S.C(2, 3), S.F(2, 4), S.F(1, 2, S.IDENTITY))
    # P: 1x1 <- FC2(1) <- FC1 needs 2 <- C2 -> 3 <- MP2 -> 6 <- C3 -> 8
    return layers, 8


def test_finite_differences_o1():
    # SPEC.md:620 (acceptance #3): every parameter, central differences, step 1e-5,
    # rel < 1e-4 (denominator max(|a|,|b|,1e-8)); <=200 params, 12x12 image
    layers, P = _tiny()
    rng = np.random.default_rng(7)
    params = S.init_params(layers, 11) * 2.0
    assert params.size <= 200
    img = rng.standard_normal((12, 12))
    lab = rng.integers(0, 2, size=(12 - P + 1, 12 - P + 1)).astype(np.uint8)
    cw = np.array([1.0, 1.7])

    def loss(th):
        ls, n, _, _ = oracle.o1_image(layers, P, th, img, lab, cw, need_grad=False, need_probs=False,
                                      threads=1)
        return ls / n

    _, n, g, _ = oracle.o1_image(layers, P, params, img, lab, cw, threads=1)
    g = g / n
    h = 1e-5
    worst = 0.0
    for i in range(params.size):
        e = np.zeros_like(params)
        e[i] = h
        fd = (loss(params + e) - loss(params - e)) / (2 * h)
        rel = abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1e-8)
        worst = max(worst, rel)
    assert worst < 1e-4, worst


def test_finite_differences_o2_sampled():
    layers, P = _tiny()
    rng = np.random.default_rng(8)
    params = S.init_params(layers, 12) * 2.0
    img = rng.standard_normal((13, 11))
    lab = rng.integers(0, 2, size=(13 - P + 1, 11 - P + 1)).astype(np.uint8)
    _, n, g, _ = o2.train_image(layers, params, img, lab, P=P)
    g = g / n
    h = 1e-5
    for i in rng.choice(params.size, 40, replace=False):
        e = np.zeros_like(params)
        e[i] = h
        lp = o2.train_image(layers, params + e, img, lab, P=P, need_grad=False)
        lm = o2.train_image(layers, params - e, img, lab, P=P, need_grad=False)
        fd = (lp[0] / lp[1] - lm[0] / lm[1]) / (2 * h)
        assert abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1e-8) < 1e-4


# ----------------------------------------------------------------- O1 == O2

@pytest.mark.parametrize("seed", range(12))
def test_o1_equals_o2_random_archs(seed):
    # SPEC.md:618-619 (acceptance #1/#2): dense == patches, fwd < 1e-10, grad < 1e-8 (fp64)
    rng = np.random.default_rng(100 + seed)
    layers, P = S.random_arch_case(rng)
    H = int(rng.integers(max(P, 20), max(P, 20) + 20))
    W = int(rng.integers(max(P, 20), max(P, 20) + 20))
    img = rng.standard_normal((H, W))
    C = layers[-1].n_out
    lab = S.random_labels(rng, 1, H - P + 1, W - P + 1, C)[0]
    cw = rng.uniform(0.5, 2.0, C)
    params = S.init_params(layers, seed) * 1.5
    l1, n1, g1, p1 = oracle.o1_image(layers, P, params, img, lab, cw)
    l2, n2, g2, p2 = o2.train_image(layers, params, img, lab, cw, P=P)
    assert n1 == n2
    O_H, O_W = H - P + 1, W - P + 1
    assert np.max(np.abs(p1.reshape(O_H, O_W, C).transpose(2, 0, 1) - p2)) < 1e-10
    assert abs(l1 - l2) <= 1e-10 * abs(l1)
    assert np.linalg.norm(g1 - g2) <= 1e-8 * np.linalg.norm(g1)


# ----------------------------------------------------------------- library special case

def _torch_dilated(layers, params, img, lab, cw=None, tie="first"):
    """fp64 torch: conv2d(dilation = prod of earlier pool k) + max_pool2d(k, stride 1,
    dilation) reproduces every patch output; autograd gives the
    gradient.  Independent of both oracles.  torch's CPU max pooling keeps the first
    maximum of a window in row-major order (strict >), i.e. reading R6; tie="last" pools
    the spatially flipped tensor instead, which routes every tie to its last maximum."""
    import torch
    import torch.nn.functional as Fn
    th = torch.tensor(params, dtype=torch.float64, requires_grad=True)
    x = torch.tensor(img, dtype=torch.float64)[None, None]
    d, off, c = 1, 0, 1
    for L in layers:
        if L.kind == POOL:
            if tie == "first":
                x = Fn.max_pool2d(x, L.k, stride=1, dilation=d)
            else:
                x = torch.flip(Fn.max_pool2d(torch.flip(x, (2, 3)), L.k, stride=1, dilation=d), (2, 3))
            d *= L.k
        else:
            n = L.n_out * c * L.k * L.k
            W = th[off:off + n].reshape(L.n_out, c, L.k, L.k)
            b = th[off + n:off + n + L.n_out]
            off += n + L.n_out
            c = L.n_out
            x = Fn.conv2d(x, W, b, dilation=d)
            if L.act == S.TANH:
                x = torch.tanh(x)
    logp = torch.log_softmax(x[0], dim=0)
    t = torch.tensor(lab.astype(np.int64))
    m = t != 255
    w = torch.ones(logp.shape[0], dtype=torch.float64) if cw is None else torch.tensor(cw)
    tt = torch.where(m, t, torch.zeros_like(t))
    nll = -logp.gather(0, tt[None])[0] * w[tt]
    loss = (nll * m).sum() / m.sum()
    loss.backward()
    return float(loss), th.grad.numpy(), torch.softmax(x[0], 0).detach().numpy()


@pytest.mark.parametrize("name,H", [("cfg1", 32), ("cfg2", 60), ("cfg5", 90)])
def test_oracles_match_torch_dilated(name, H):
    cfg = S.CONFIGS[name]
    rng = np.random.default_rng(5)
    img = rng.standard_normal((H, H))
    O = H - cfg.P + 1
    lab = S.random_labels(rng, 1, O, O, cfg.classes)[0]
    params = S.init_params(cfg)
    lt, gt, pt = _torch_dilated(cfg.layers, params, img, lab)
    l2, n2, g2, p2 = o2.train_image(cfg.layers, params, img, lab, P=cfg.P)
    assert abs(l2 / n2 - lt) <= 1e-12 * abs(lt)
    assert np.max(np.abs(p2 - pt)) < 1e-12
    assert np.linalg.norm(g2 / n2 - gt) <= 1e-10 * np.linalg.norm(gt)
    if O * O <= 400:
        l1, n1, g1, p1 = oracle.o1_image(cfg.layers, cfg.P, params, img, lab)
        assert np.linalg.norm(g1 / n1 - gt) <= 1e-10 * np.linalg.norm(gt)
    else:  # sampled pixels through O1 against the torch outputs
        pix = rng.choice(O * O, 24, replace=False)
        _, _, _, p1 = oracle.o1_image(cfg.layers, cfg.P, params, img, None, pix=pix, need_grad=False)
        np.testing.assert_allclose(p1, pt.reshape(cfg.classes, -1)[:, pix].T, atol=1e-12)


def test_tie_rule_first_maximum_pinned():
    """Reading R6 (first maximum in row-major scan, strict >) pinned in both oracles: with the
    first layer's weights zero every conv output is tanh(b), so every pooling block is an
    exact tie and the rule alone decides where the deltas go.  O1 (its `>` in the block
    scan) and O2 (numpy argmax) must equal torch's first-maximum pooling, and the
    last-maximum routing must give a clearly different gradient (so `>=` would fail)."""
    cfg = S.CONFIGS["cfg1"]
    rng = np.random.default_rng(23)
    H = 22
    img = rng.standard_normal((H, H))
    O = H - cfg.P + 1
    lab = S.random_labels(rng, 1, O, O, cfg.classes, ignore_frac=0.0)[0]
    params = S.init_params(cfg)
    n0 = cfg.layers[0].n_out * cfg.layers[0].k ** 2
    params[:n0] = 0.0                                    # W of the first conv: all ties below
    lt, gt, pt = _torch_dilated(cfg.layers, params, img, lab)
    _, gl, _ = _torch_dilated(cfg.layers, params, img, lab, tie="last")
    l1, n1, g1, p1 = oracle.o1_image(cfg.layers, cfg.P, params, img, lab)
    l2, n2, g2, p2 = o2.train_image(cfg.layers, params, img, lab, P=cfg.P)
    w0 = slice(0, n0)
    assert np.linalg.norm(gt[w0] - gl[w0]) > 0.1 * np.linalg.norm(gt[w0])  # the rule matters here
    for g, n in ((g1, n1), (g2, n2)):
        assert np.linalg.norm(g / n - gt) <= 1e-10 * np.linalg.norm(gt)


# ----------------------------------------------------------------- SGD / determinism

def test_train_step_formula_and_determinism():
    # R8 / R14: step gradient = mean over images of per-image means; theta -= lr * g
    cfg = S.CONFIGS["cfg1"]
    rng = np.random.default_rng(9)
    imgs = rng.standard_normal((2, 1, 32, 32))
    labs = S.random_labels(rng, 2, 19, 19, 2)
    p = S.init_params(cfg)
    r = oracle.train_step(cfg.layers, cfg.P, p, imgs, labs, lr=0.01, threads=3)
    per = []
    for i in range(2):
        ls, n, g, _ = o2.train_image(cfg.layers, p, imgs[i, 0], labs[i], P=cfg.P)
        per.append(g / n)
    gm = (per[0] + per[1]) / 2
    assert np.linalg.norm(r["grad"] - gm) <= 1e-12 * np.linalg.norm(gm)
    np.testing.assert_allclose(r["params"], p - 0.01 * r["grad"], rtol=0, atol=0)
    r2 = oracle.train_step(cfg.layers, cfg.P, p, imgs, labs, lr=0.01, threads=3)
    assert np.array_equal(r["grad"], r2["grad"])  # bitwise reproducible


def test_golden_auto_class_weights():
    """SPEC.md:417-421 worked examples of the per-class MCCE weights."""
    lines = golden_lines("class_weights.txt")
    pairs = [(lines[i], lines[i + 1]) for i in range(0, len(lines), 2)]
    for cl, wl in pairs:
        counts = [int(v) for v in cl.split()[1:]]
        want = [float(v) for v in wl.split()[1:]]
        labels = np.concatenate([np.full(n, c, dtype=np.uint8) for c, n in enumerate(counts)] +
                                [np.full(7, 255, dtype=np.uint8)])  # ignored pixels do not count
        w, cnt = o2.auto_class_weights(labels, len(counts))
        assert list(cnt) == counts
        assert np.allclose(w, want, rtol=0, atol=1e-15)
    # invariants: positive, finite, sum_c w_c n_c = N (the weighted class mass equals N / C each)
    rng = np.random.default_rng(5)
    lab = rng.integers(0, 5, size=(3, 17, 19)).astype(np.uint8)
    w, cnt = o2.auto_class_weights(lab, 5)
    assert np.all(w > 0) and np.all(np.isfinite(w))
    assert np.allclose(w * cnt, cnt.sum() / 5)
    with pytest.raises(ValueError):
        o2.auto_class_weights(np.zeros(10, dtype=np.uint8), 2)


def test_golden_mirror_pad():
    """PAPER.md:207 / SPEC.md:296 mirror convention on a worked row, and the same-size
    property: a P-padded image has an output grid of exactly H x W (H - P + 1 after padding)."""
    lines = golden_lines("mirror_pad.txt")
    row = np.array([float(v) for v in lines[0].split()[1:]])
    before, after = (int(v) for v in lines[1].split()[1:])
    want = [float(v) for v in lines[2].split()[1:]]
    got = np.pad(row, (before, after), mode="reflect")  # the primitive o2.mirror_pad uses
    assert list(got) == want
    img = np.arange(5 * 7, dtype=np.float64).reshape(5, 7)
    for P in (2, 4, 5):
        pad = o2.mirror_pad(img, P)
        assert pad.shape == (5 + P - 1, 7 + P - 1)
        pt = (P - 1) // 2
        assert np.array_equal(pad[pt:pt + 5, pt:pt + 7], img)
        assert pad.shape[0] - P + 1 == 5 and pad.shape[1] - P + 1 == 7
        if pt > 0:
            assert np.array_equal(pad[pt - 1, pt:pt + 7], img[1])  # no repeat of the edge row


def test_golden_armijo_quadratic():
    """SPEC.md:388-396 worked cases of the Armijo rule on L = theta^2."""
    for line in golden_lines("armijo.txt"):
        tok = line.split()
        th, a0, beta = float(tok[2]), float(tok[4]), float(tok[6])
        want_th, want_a, want_ev = float(tok[9]), float(tok[11]), int(tok[13])
        f = lambda t: float(np.sum(t * t))  # noqa: E731
        fg = lambda t: (f(t), 2.0 * t)  # noqa: E731
        t_new, a, L, ok, ev = o2.armijo_step(fg, f, np.array([th]), a0, beta, 1e-4, 10)
        assert ok and ev == want_ev and a == want_a and abs(t_new[0] - want_th) < 1e-15
        assert L <= th * th  # an accepted step never increases the loss


def _quad(A, bvec):
    """L = 1/2 t^T A t - b^T t and its gradient."""
    return lambda t: (0.5 * float(t @ A @ t) - float(bvec @ t), A @ t - bvec)


def test_golden_lbfgs_worked_steps():
    """SPEC.md:397-405 worked cases (tests/golden/lbfgs.txt): the empty-history step is
    steepest descent at alpha0, and the second direction equals the BFGS inverse-Hessian
    update written as matrices (an independent form of the two-loop)."""
    lines = {ln.split()[0]: ln.split() for ln in golden_lines("lbfgs.txt")}
    f = lambda t: (float(t[0] ** 2 + 4 * t[1] ** 2), np.array([2 * t[0], 8 * t[1]]))  # noqa: E731
    st = {}
    t1, a, L0, L1, ok, ev, fb = o2.lbfgs_step(st, np.array([1.0, 1.0]), f, 5, 0.1, 0.5, 1e-4, 10)
    s1 = lines["step1"]
    assert ok and not fb and ev == int(s1[7]) and a == float(s1[5])
    assert np.allclose(t1, [float(s1[2]), float(s1[3])], rtol=0, atol=1e-15)
    assert abs(float(st["S"][0] @ st["Y"][0]) - float(s1[9])) < 1e-14
    d2 = -o2.lbfgs_two_loop(st["g"], st["S"], st["Y"])
    w = lines["dir2"]
    want = np.array([int(w[1]) / int(w[2]), int(w[3]) / int(w[4])])
    assert np.allclose(d2, want, rtol=1e-14, atol=0)


def test_lbfgs_two_loop_equals_bfgs_matrix_update():
    """The two-loop product H_k g equals the explicit BFGS recursion
    H <- (I - rho s y^T) H (I - rho y s^T) + rho s s^T from H0 = gamma I over the same m pairs,
    and H_k y_newest = s_newest (secant equation), for random pairs with s^T y > 0."""
    rng = np.random.default_rng(7)
    n, m = 6, 4
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    S = [rng.standard_normal(n) for _ in range(m)]
    Y = [A @ s for s in S]
    gamma = float(S[-1] @ Y[-1]) / float(Y[-1] @ Y[-1])
    H = gamma * np.eye(n)
    for s, y in zip(S, Y):
        rho = 1.0 / float(s @ y)
        V = np.eye(n) - rho * np.outer(y, s)
        H = V.T @ H @ V + rho * np.outer(s, s)
    g = rng.standard_normal(n)
    assert np.allclose(o2.lbfgs_two_loop(g, S, Y), H @ g, rtol=1e-11, atol=1e-12)
    assert np.allclose(o2.lbfgs_two_loop(Y[-1], S, Y), S[-1], rtol=1e-11, atol=1e-12)
    assert np.array_equal(o2.lbfgs_two_loop(g, [], []), g)


def test_lbfgs_convex_quadratic_converges():
    """on a fixed strictly convex 5-variable quadratic the gradient norm
    drops below 1e-8 within 20 iterations, the loss decreases monotonically, and the history
    never exceeds `memory` pairs (10, the customary default; the SPEC leaves it open); the
    minimiser is A^-1 b (closed form)."""
    rng = np.random.default_rng(11)
    M = rng.standard_normal((5, 5))
    A = M @ M.T + np.eye(5)
    bvec = rng.standard_normal(5)
    f = _quad(A, bvec)
    theta, st, losses, memory = np.zeros(5), {}, [], 10
    for it in range(20):
        theta, a, L0, L1, ok, ev, fb = o2.lbfgs_step(st, theta, f, memory, 1.0, 0.5, 1e-4, 30)
        assert ok and L1 <= L0
        assert len(st["S"]) <= memory
        losses.append(L1)
        if np.linalg.norm(st["g"]) < 1e-8:
            break
    assert np.linalg.norm(st["g"]) < 1e-8, (it, np.linalg.norm(st["g"]))
    assert np.allclose(theta, np.linalg.solve(A, bvec), rtol=1e-7, atol=1e-9)
    assert all(b <= a for a, b in zip(losses, losses[1:]))


def test_lbfgs_fallback_and_restart():
    """Non-descent direction -> steepest descent; an exhausted line search keeps
    theta and clears the pairs (R21); pairs with s^T y <= 1e-10 are not stored."""
    f = lambda t: (float(t @ t), 2 * t)  # noqa: E731
    st = {"S": [np.array([1.0, 0.0])], "Y": [np.array([-1.0, 0.0])], "L": 2.0, "g": np.array([2.0, 2.0])}
    # with s^T y < 0 the single-pair H is indefinite along e1: H g = (-2 + ..., ...) gives g^T d >= 0
    d = -o2.lbfgs_two_loop(st["g"], st["S"], st["Y"])
    assert float(st["g"] @ d) >= 0
    t, a, L0, L1, ok, ev, fb = o2.lbfgs_step(st, np.array([1.0, 1.0]), f, 3, 0.1, 0.5, 1e-4, 10)
    # d = -g = (-2, -2); history non-empty -> alpha starts at 1: L(-1, -1) = 2 is rejected,
    # alpha = 0.5 reaches the minimum (0, 0)
    assert fb and ok and a == 0.5 and ev == 2 and np.array_equal(t, [0.0, 0.0])
    # exhausted search: max_backtracks = 0 and a step that overshoots
    st2 = {}
    t2, a2, L0, L1, ok2, ev2, fb2 = o2.lbfgs_step(st2, np.array([1.0]), f, 3, 5.0, 0.5, 1e-4, 0)
    assert not ok2 and a2 == 0.0 and t2[0] == 1.0 and st2["S"] == [] and ev2 == 1
    # a linear loss has y = 0, so s^T y = 0 and no pair is stored
    lin = lambda t: (float(np.sum(t)), np.ones_like(t))  # noqa: E731
    st3 = {}
    o2.lbfgs_step(st3, np.array([0.0, 0.0]), lin, 3, 0.5, 0.5, 1e-4, 5)
    assert st3["S"] == []
