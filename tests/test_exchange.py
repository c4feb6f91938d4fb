"""Peer-memory gradient exchange (include/mpf.h mpf_exchange_*).

Alg. 2's gradient sum over the images of a global batch sharded over
ranks: every rank's backward pushes its buckets into every rank's exchange buffer, the SGD
kernel sums the slots in rank order and applies theta -= lr/B * sum.

On one GPU, ranks are simulated without any kernel waiting on a concurrently running one:
- in one process, two nets (rank 0 and 1) whose "peer" buffers are plain device pointers;
  both backwards are enqueued before either SGD, on one stream;
- in two processes sharing cuda:0 through CUDA IPC, each rank synchronises and meets the
  other at a host barrier between its push and its SGD.
The references are plain per-rank gradients summed in rank order with torch on the device.
"""
import os
import socket

import numpy as np
import pytest

import mpf_synth as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LR = 0.01


def _nets(cfg, n, count):
    from paper_1302_1690_b200.net import MPFNet
    params = S.init_params(cfg).astype(np.float32)
    nets = []
    for _ in range(count):
        net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=n)
        net.set_params(params)
        nets.append(net)
    return nets


def _shards(cfg, step, world, per):
    out = []
    for r in range(world):
        idx = [step * world * per + r * per + i for i in range(per)]
        im, lb = S.make_batch(cfg, idx)
        out.append((torch.tensor(im, device="cuda"), torch.tensor(lb, device="cuda")))
    return out


def _reference(cfg, steps, world, per):
    """theta after `steps` SGD steps on the rank-order sum of per-rank gradients."""
    (net,) = _nets(cfg, per, 1)
    scale = 1.0 / (world * per)
    for t in range(steps):
        gs = []
        for im, lb in _shards(cfg, t, world, per):
            net.train_step(im, lb)
            gs.append(net.grads.clone())
            net.grads.zero_()
        s = gs[0]
        for g in gs[1:]:
            s = s + g
        net.params -= (LR * scale) * s
    torch.cuda.synchronize()
    return net.params.cpu().numpy()


def _exchange_buffers(nets, world):
    nbytes = nets[0].exchange_bytes(world)
    bufs = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
    return bufs


@pytest.mark.parametrize("push_in_backward", [True, False])
def test_exchange_two_ranks_one_process(push_in_backward):
    cfg = S.CONFIGS["cfg2"]
    world, per, steps = 2, 2, 3
    nets = _nets(cfg, per, world)
    bufs = _exchange_buffers(nets, world)
    for r, net in enumerate(nets):
        net.attach_exchange(r, world, [b.data_ptr() for b in bufs], push_in_backward)
    for t in range(steps):  # epochs 1..3: both slot parities, flags overtaken by later epochs
        for (im, lb), net in zip(_shards(cfg, t, world, per), nets):
            net.train_step(im, lb)
            if not push_in_backward:
                net.exchange_push()
        for net in nets:
            net.sgd_step(LR, 1.0 / (world * per))
    for net in nets:
        net.check()
    p0, p1 = nets[0].params.cpu().numpy(), nets[1].params.cpu().numpy()
    assert np.array_equal(p0, p1), "ranks must hold bitwise identical parameters"
    assert not nets[0].grads.any() and not nets[1].grads.any()
    ref = _reference(cfg, steps, world, per)
    # same sums in the same order; the kernel may contract p - step * s into one FMA
    assert np.max(np.abs(p0 - ref)) <= 1e-6 * max(1.0, np.max(np.abs(ref)))


def test_exchange_three_ranks_scalar_path():
    """cfg1 (898 parameters: buckets and slots not multiples of 4 floats, the push kernel's
    scalar path) with three ranks of one image each, two steps."""
    cfg = S.CONFIGS["cfg1"]
    world, per, steps = 3, 1, 2
    nets = _nets(cfg, per, world)
    bufs = _exchange_buffers(nets, world)
    for r, net in enumerate(nets):
        net.attach_exchange(r, world, [b.data_ptr() for b in bufs])
    for t in range(steps):
        for (im, lb), net in zip(_shards(cfg, t, world, per), nets):
            net.train_step(im, lb)
        for net in nets:
            net.sgd_step(LR, 1.0 / (world * per))
    for net in nets:
        net.check()
    ps = [net.params.cpu().numpy() for net in nets]
    assert np.array_equal(ps[0], ps[1]) and np.array_equal(ps[0], ps[2])
    ref = _reference(cfg, steps, world, per)
    assert np.max(np.abs(ps[0] - ref)) <= 1e-6 * max(1.0, np.max(np.abs(ref)))


def test_exchange_world1_equals_local_sgd():
    """At world 1 the exchange SGD is the local SGD: bitwise the same parameters."""
    cfg = S.CONFIGS["cfg2"]
    a, b = _nets(cfg, 2, 2)
    buf = _exchange_buffers([a], 1)[0]
    a.attach_exchange(0, 1, [buf.data_ptr()])
    for t in range(2):
        (im, lb), = _shards(cfg, t, 1, 2)
        for net in (a, b):
            net.train_step(im, lb)
            net.sgd_step(LR, 0.5)
    a.check()
    assert np.array_equal(a.params.cpu().numpy(), b.params.cpu().numpy())
    a.detach_exchange()
    (im, lb), = _shards(cfg, 5, 1, 2)
    for net in (a, b):  # detached: back to the local update
        net.train_step(im, lb)
        net.sgd_step(LR, 0.5)
    assert np.array_equal(a.params.cpu().numpy(), b.params.cpu().numpy())


def test_exchange_missing_rank_times_out_and_is_reported():
    """A rank that never pushes: the SGD gives up after its bounded wait, theta unchanged,
    mpf_check raises MPF_ERR_INTERNAL (no hang)."""
    from paper_1302_1690_b200 import _lib as L
    cfg = S.CONFIGS["cfg1"]
    nets = _nets(cfg, 1, 2)
    bufs = _exchange_buffers(nets, 2)
    nets[0].attach_exchange(0, 2, [b.data_ptr() for b in bufs])
    (im, lb), _ = _shards(cfg, 0, 2, 1)
    nets[0].train_step(im, lb)
    before = nets[0].params.clone()
    nets[0].sgd_step(LR, 0.5)
    with pytest.raises(L.MpfError) as e:
        nets[0].check()
    assert e.value.status == L.MPF_ERR_INTERNAL and "rank 1" in str(e.value)
    assert torch.equal(nets[0].params, before)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, steps, per, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1302_1690_b200.dist import PeerExchange
    cfg = S.CONFIGS["cfg2"]
    (net,) = _nets(cfg, per, 1)
    ex = PeerExchange(net)
    for t in range(steps):
        im, lb = _shards(cfg, t, world, per)[rank]
        net.train_step(im, lb)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's pushes are complete before any SGD starts waiting
        net.sgd_step(LR, 1.0 / (world * per))
        torch.cuda.synchronize()
        dist.barrier()
    net.check()
    np.save(out_path + f".{rank}.npy", net.params.cpu().numpy())
    ex.close()
    dist.destroy_process_group()


def test_exchange_two_processes_ipc(tmp_path):
    import torch.multiprocessing as mp
    world, per, steps = 2, 2, 2
    out = str(tmp_path / "params")
    mp.start_processes(_ipc_worker, args=(world, _free_port(), steps, per, out), nprocs=world, join=True,
                       start_method="spawn")
    p0, p1 = np.load(out + ".0.npy"), np.load(out + ".1.npy")
    assert np.array_equal(p0, p1)
    ref = _reference(S.CONFIGS["cfg2"], steps, world, per)
    assert np.max(np.abs(p0 - ref)) <= 1e-6 * max(1.0, np.max(np.abs(ref)))
