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
