"""World-size-2 `gloo` tests of the data-parallel host logic (CPU, no GPU).

Each rank computes the per-image mean gradients of ITS shard of a global batch with
the oracle (the GPU kernels are replaced by the oracle here only because there is no
GPU; the sharding, the all-reduce on the flat gradient and the SGD scaling are the
same code bench.py runs), sums them with paper_1302_1690_b200.dist.allreduce_grads,
and must reproduce the single-process full-batch gradient and SGD update.
"""
import os
import socket

import numpy as np
import pytest

import mpf_synth as S
from paper_1302_1690_b200 import dist as D

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch_grad(cfg, indices):
    import oracle
    images, labels = S.make_batch(cfg, indices)
    params = S.init_params(cfg)
    g = np.zeros_like(params)
    for i in range(len(indices)):
        _, n, gi, _ = oracle.o1_image(cfg.layers, cfg.P, params, images[i].astype(np.float64), labels[i],
                                      threads=1, need_probs=False)
        g += gi / n
    return params, g


def _worker(rank, world, port, B, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = S.CONFIGS["cfg1"]
        idx = D.batch_indices(1, B, world, rank)
        params, g = _batch_grad(cfg, idx)
        t = torch.tensor(g)
        D.allreduce_grads(t)
        theta = params - cfg.lr * (1.0 / B) * t.numpy()
        mx = D.max_over_ranks(float(rank + 1))
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.concatenate([t.numpy(), theta, [mx]]))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for B, W in [(8, 1), (8, 2), (8, 4), (8, 8), (6, 3)]:
        owned = [i for r in range(W) for i in D.shard(B, W, r)]
        assert owned == list(range(B))
    assert D.batch_indices(2, 8, 4, 3) == [22, 23]
    with pytest.raises(ValueError):
        D.shard(8, 3, 0)


def test_gloo_world2_gradient_sum_equals_full_batch(tmp_path):
    import torch.multiprocessing as mp
    B, world = 4, 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, B, str(tmp_path)), nprocs=world, start_method="spawn")
    r0, r1 = (np.load(tmp_path / f"r{r}.npy") for r in range(world))
    cfg = S.CONFIGS["cfg1"]
    params, g_full = _batch_grad(cfg, D.batch_indices(1, B, 1, 0))
    n = params.size
    # both ranks hold the same summed gradient and the same updated parameters
    assert np.array_equal(r0, r1)
    assert np.allclose(r0[:n], g_full, rtol=1e-12, atol=1e-14)
    assert np.allclose(r0[n:2 * n], params - cfg.lr * g_full / B, rtol=1e-12, atol=1e-14)
    assert r0[-1] == 2.0  # max over ranks


class _OracleLbfgsOps:
    """dist.lbfgs_iteration ops over numpy + the oracle (there is no GPU here): the
    shard's gradient is summed over ranks with dist.allreduce_grads and the loss with
    dist.all_sum_scalar, exactly as net.Lbfgs.evaluate does on the GPU path."""

    def __init__(self, cfg, images, labels, theta, B, memory):
        self.cfg, self.images, self.labels, self.B, self.m = cfg, images, labels, B, memory
        self.theta, self.have_g, self.L, self.n_pairs = theta.copy(), False, 0.0, 0
        self.S, self.Y = [], []

    def evaluate(self):
        import oracle
        g = np.zeros_like(self.theta)
        L = 0.0
        for i in range(len(self.images)):
            loss, n, gi, _ = oracle.o1_image(self.cfg.layers, self.cfg.P, self.theta, self.images[i].astype(np.float64),
                                             self.labels[i], threads=1, need_probs=False)
            g += gi / n
            L += loss / n
        t = torch.tensor(g)
        D.allreduce_grads(t)
        self.grad = t.numpy() / self.B
        return D.all_sum_scalar(L) / self.B

    def set_gradient(self):
        self.g, self.have_g = self.grad, True

    def direction(self):
        from oracle import o2
        self.theta0 = self.theta.copy()
        self.d = -o2.lbfgs_two_loop(self.g, self.S, self.Y)
        gtd = float(self.g @ self.d)
        fb = not gtd < 0
        if fb:
            self.d, gtd = -self.g, -float(self.g @ self.g)
        return gtd, fb

    def trial(self, alpha):
        self.theta = self.theta0 + alpha * self.d

    def accept(self):
        s, y = self.theta - self.theta0, self.grad - self.g
        self.g = self.grad
        if float(s @ y) > 1e-10:
            self.S.append(s)
            self.Y.append(y)
            if len(self.S) > self.m:
                del self.S[0], self.Y[0]
            self.n_pairs = len(self.S)
            return True
        return False

    def reject(self):
        self.theta = self.theta0
        self.S, self.Y, self.n_pairs = [], [], 0


def _lbfgs_worker(rank, world, port, B, iters, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = S.CONFIGS["cfg1"]
        images, labels = S.make_batch(cfg, D.batch_indices(0, B, world, rank))
        ops = _OracleLbfgsOps(cfg, images, labels, S.init_params(cfg).astype(np.float64), B, 3)
        rec = []
        for _ in range(iters):
            r = D.lbfgs_iteration(ops, 0.5, 0.5, 1e-4, 8)
            rec += [r["loss"], r["alpha"], r["evals"], r["pairs"]]
        np.save(os.path.join(out_dir, f"l{rank}.npy"), np.concatenate([ops.theta, rec]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_lbfgs_equals_full_batch_oracle(tmp_path):
    """Full-batch L-BFGS over two ranks ("full-batch"): the host
    loop dist.lbfgs_iteration with the gradient and loss summed over ranks takes the same
    steps as the single-process oracle o2.lbfgs_step on the whole batch."""
    import torch.multiprocessing as mp
    from oracle import o2
    import oracle
    B, world, iters = 4, 2, 3
    port = _free_port()
    mp.start_processes(_lbfgs_worker, args=(world, port, B, iters, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    r0, r1 = (np.load(tmp_path / f"l{r}.npy") for r in range(world))
    assert np.array_equal(r0, r1)
    cfg = S.CONFIGS["cfg1"]
    images, labels = S.make_batch(cfg, D.batch_indices(0, B, 1, 0))

    def eval_lg(theta):
        g, L = np.zeros_like(theta), 0.0
        for i in range(B):
            loss, n, gi, _ = oracle.o1_image(cfg.layers, cfg.P, theta, images[i].astype(np.float64), labels[i],
                                             threads=1, need_probs=False)
            g += gi / n
            L += loss / n
        return L / B, g / B

    st, theta, rec = {}, S.init_params(cfg).astype(np.float64), []
    for _ in range(iters):
        theta, a, L0, L1, ok, ev, fb = o2.lbfgs_step(st, theta, eval_lg, 3, 0.5, 0.5, 1e-4, 8)
        rec += [L1, a, ev, len(st["S"])]
    n = theta.size
    assert np.allclose(r0[:n], theta, rtol=1e-9, atol=1e-12)
    assert np.allclose(r0[n:], rec, rtol=1e-9, atol=1e-12)
    assert rec[0] < eval_lg(S.init_params(cfg).astype(np.float64))[0]


def _w_offsets(layers):
    off, out = 0, []
    shapes = iter(S.param_shapes(layers))
    for ly in layers:
        if ly.kind == S.POOL:
            out.append(-1)
            continue
        (w, b) = next(shapes)
        out.append(off)
        off += int(np.prod(w)) + b
    return out, off


def test_grad_buckets_tile_the_buffer():
    """The buckets mpf_net_set_grad_hook reports (dist.grad_buckets) cover every gradient
    entry exactly once, in decreasing offset order, the softmax FC with the last hidden
    layer (include/mpf.h; the same plan the library's backward follows)."""
    for name in S.CONFIGS:
        cfg = S.CONFIGS[name]
        woff, n = _w_offsets(cfg.layers)
        b = D.grad_buckets(cfg.layers, woff, n)
        cover = np.zeros(n, int)
        for l, o, c in b:
            cover[o:o + c] += 1
        assert np.all(cover == 1), name
        assert [o for _, o, _ in b] == sorted([o for _, o, _ in b], reverse=True)
        assert b[-1][1] == 0 and b[0][0] == len(cfg.layers) - 2


def _bucket_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = S.CONFIGS["cfg4"]
        woff, n = _w_offsets(cfg.layers)
        g = torch.tensor(np.random.default_rng(rank).standard_normal(n))
        full = g.clone()
        D.allreduce_grads(full)
        br = D.BucketAllReduce(g)
        for l, o, c in D.grad_buckets(cfg.layers, woff, n):  # what the library's backward calls
            br(l, o, c, None)
        br.wait()
        np.save(os.path.join(out_dir, f"b{rank}.npy"), np.stack([g.numpy(), full.numpy()]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bucketed_allreduce_equals_flat(tmp_path):
    """Per-bucket all-reduces started from the gradient-ready hook (dist.BucketAllReduce)
    give exactly the flat all-reduce of the whole buffer (fp64, two ranks)."""
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_bucket_worker, args=(2, port, str(tmp_path)), nprocs=2, start_method="spawn")
    for r in range(2):
        g, full = np.load(tmp_path / f"b{r}.npy")
        assert np.array_equal(g, full)


def _peer_table_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    recs = [None] * world
    # what PeerExchange all-gathers: (rank, 64-byte IPC handle, offset, buffer bytes)
    dist.all_gather_object(recs, (rank, bytes([rank]) * 64, 256 * rank, 4096))
    table = D.peer_table(recs, rank, world)
    np.save(os.path.join(out, f"t{rank}.npy"), np.array([[r, h[0], o, b] for r, h, o, b in table]))
    dist.destroy_process_group()


def test_peer_exchange_records_world2(tmp_path):
    """The host half of PeerExchange: every rank ends with the same rank-ordered
    table of buffer handles, and inconsistent records are rejected."""
    import torch.multiprocessing as mp
    mp.start_processes(_peer_table_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    t0, t1 = np.load(tmp_path / "t0.npy"), np.load(tmp_path / "t1.npy")
    assert np.array_equal(t0, t1) and t0[:, 0].tolist() == [0, 1] and t0[:, 2].tolist() == [0, 256]
    with pytest.raises(RuntimeError):
        D.peer_table([(0, b"", 0, 1), (0, b"", 0, 1)], 0, 2)
    with pytest.raises(RuntimeError):
        D.peer_table([(0, b"", 0, 1), (1, b"", 0, 2)], 0, 2)
