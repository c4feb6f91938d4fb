"""Data-parallel host logic.

Images are independent units: rank r of N takes the contiguous slice
[r*B/N, (r+1)*B/N) of every global batch of B images and generates its own images
from per-image seeds, so no input crosses ranks.  The only exchange is the sum of
the flat fp32 gradient (Alg. 2's sum over fragments, extended
over images and ranks).  Two exchanges implement it:
- PeerExchange (default in bench.py): the library's backward pushes every gradient bucket
  into every rank's exchange buffer over NVLink P2P as soon as it is final, and the SGD
  kernel sums the ranks' slots (rank order) before applying the same
  ``theta -= lr/B * g`` — the collective fused into the backward's tail and
  the optimizer;
- BucketAllReduce / allreduce_grads: NCCL ``all_reduce(SUM)`` per bucket on a tensor that
  aliases the bound gradient buffer, then ``mpf_sgd_step(lr, 1/B)`` (the baseline).
"""
from __future__ import annotations

from typing import List

import numpy as np


def shard(global_batch: int, world: int, rank: int) -> range:
    """Positions (within one global batch) of the images rank `rank` owns."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} is not divisible by {world} ranks")
    per = global_batch // world
    return range(rank * per, (rank + 1) * per)


def batch_indices(step: int, global_batch: int, world: int, rank: int) -> List[int]:
    """Dataset image indices of this rank for SGD step `step`."""
    return [step * global_batch + i for i in shard(global_batch, world, rank)]


def allreduce_grads(grads, group=None) -> None:
    """Sum the flat gradient over ranks in place (no-op on a single rank)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)


def grad_buckets(layers, w_offset, n_params):
    """The gradient buckets one backward reports through mpf_net_set_grad_hook, in order:
    (layer, offset, count) for every conv/FC layer from the last hidden one down to the
    first; each covers the W / b entries of its layer and of every higher layer not yet
    reported (the softmax FC goes with the last hidden layer), so together they tile
    [0, n_params) exactly once."""
    out, end = [], n_params
    convs = [l for l, ly in enumerate(layers) if ly.kind != 1]  # 1 = POOL
    for l in reversed(convs[:-1]):
        out.append((l, int(w_offset[l]), end - int(w_offset[l])))
        end = int(w_offset[l])
    return out


class BucketAllReduce:
    """Data-parallel gradient exchange overlapped with the backward: installed as the net's
    gradient-ready hook, it starts one all-reduce(SUM) per bucket on the stream that
    produced it (async, so the backward below keeps running), and wait() makes the current
    stream wait for all of them before the SGD step.  Same sum as allreduce_grads (the
    buckets tile the buffer).  On a CPU tensor (gloo tests) stream_ptr is ignored."""

    def __init__(self, grads, group=None):
        self.grads = grads
        self.group = group
        self.works = []
        self.calls = []

    def __call__(self, layer, offset, count, stream_ptr=None):
        import torch
        import torch.distributed as dist
        self.calls.append((layer, offset, count))
        view = self.grads[offset:offset + count]
        if self.grads.is_cuda and stream_ptr is not None:
            with torch.cuda.stream(torch.cuda.ExternalStream(stream_ptr, device=self.grads.device)):
                self.works.append(dist.all_reduce(view, op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        else:
            self.works.append(dist.all_reduce(view, op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def wait(self):
        for w in self.works:
            w.wait()
        self.works.clear()


def peer_table(records, rank: int, world: int):
    """Validate the all-gathered exchange records [(rank, handle bytes, offset, bytes), ...] of
    PeerExchange: one per rank, in rank order, equal buffer sizes.  Returns them sorted."""
    recs = sorted(records, key=lambda r: r[0])
    if [r[0] for r in recs] != list(range(world)):
        raise RuntimeError(f"exchange records do not cover ranks 0..{world - 1}: {[r[0] for r in records]}")
    sizes = {r[3] for r in recs}
    if len(sizes) != 1:
        raise RuntimeError(f"ranks disagree on the exchange buffer size: {sorted(sizes)}")
    if not 0 <= rank < world:
        raise ValueError("bad rank")
    return recs


class PeerExchange:
    """Peer-memory gradient exchange for `net` across the ranks of `group` (include/mpf.h
    mpf_exchange_*): allocates this rank's zero-filled exchange buffer, exports it through CUDA
    IPC, all-gathers the handles (a collective, so no rank attaches before every buffer is
    zeroed), maps the peers' buffers and attaches.  From then on the backward pushes every
    gradient bucket into every rank's buffer as it completes and net.sgd_step sums the ranks'
    slots inside the SGD kernel — no separate all-reduce.  The arithmetic (Alg. 2's sum
    extended over ranks) is all in the library's kernels; this class only
    moves handles."""

    def __init__(self, net, group=None, push_in_backward: bool = True):
        import ctypes
        import torch
        import torch.distributed as dist
        from . import _lib as L
        self.net, self.lib = net, L.lib()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        nbytes = net.exchange_bytes(self.world)
        raw = torch.zeros(nbytes + 256, dtype=torch.uint8, device=net.device)
        shift = (-raw.data_ptr()) % 256
        self._raw, self.buf = raw, raw[shift:shift + nbytes]
        torch.cuda.synchronize(net.device)  # zero-filled before any peer can see it
        handle = (ctypes.c_char * 64)()
        off = ctypes.c_uint64()
        err = ""
        if self.lib.mpf_ipc_export(ctypes.c_void_p(self.buf.data_ptr()), handle, ctypes.byref(off)) != L.MPF_OK:
            err = f"rank {self.rank}: mpf_ipc_export failed: " + self.lib.mpf_last_error().decode(errors="replace")
        recs = [None] * self.world
        dist.all_gather_object(recs, (self.rank, bytes(handle), int(off.value), nbytes, err), group=group)
        bad = [r[4] for r in recs if r[4]]
        if bad:  # every rank raises (no rank is left waiting in a collective)
            raise RuntimeError("PeerExchange: " + "; ".join(bad))
        recs = peer_table([r[:4] for r in recs], self.rank, self.world)
        self.opened = []
        self.group = group
        ptrs, err = [], ""
        for r, h, o, _ in recs:
            if r == self.rank:
                ptrs.append(self.buf.data_ptr())
                continue
            p = ctypes.c_void_p()
            hb = (ctypes.c_char * 64).from_buffer_copy(h)
            st = self.lib.mpf_ipc_open(hb, ctypes.c_uint64(o), ctypes.byref(p))
            if st != L.MPF_OK:
                err = f"rank {self.rank}: mpf_ipc_open of rank {r}'s buffer failed: " + \
                    self.lib.mpf_last_error().decode(errors="replace")
                break
            self.opened.append((p.value, o))
            ptrs.append(p.value)
        # attach only if every rank mapped every buffer (else nobody attaches: the caller
        # falls back to another exchange)
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)
        bad = [e for e in errs if e]
        if bad:
            for p, o in self.opened:
                self.lib.mpf_ipc_close(ctypes.c_void_p(p), ctypes.c_uint64(o))
            self.opened = []
            raise RuntimeError("PeerExchange: " + "; ".join(bad))
        net.attach_exchange(self.rank, self.world, ptrs, push_in_backward)

    def close(self) -> None:
        """Detach and unmap (collective: waits until every rank is done with every buffer)."""
        import ctypes
        import torch
        import torch.distributed as dist
        from . import _lib as L
        torch.cuda.synchronize(self.net.device)
        dist.barrier(group=self.group)
        self.net.detach_exchange()
        for p, o in self.opened:
            L.check(self.lib.mpf_ipc_close(ctypes.c_void_p(p), ctypes.c_uint64(o)), "mpf_ipc_close")
        self.opened = []
        dist.barrier(group=self.group)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a host scalar over ranks (device timing rule: max over ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_sum_scalar(value: float, device=None, group=None) -> float:
    """Sum of a host scalar over ranks in fp64 (the full-batch loss of L-BFGS)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def lbfgs_iteration(ops, alpha0: float, beta: float, c: float, max_backtracks: int) -> dict:
    """One full-batch L-BFGS iteration (reading R21) driven
    from the host over `ops`, whose evaluate() returns the loss summed over ALL ranks after
    summing the gradient buffer over them (dist.allreduce_grads), so every rank sees the same
    gradient and loss and takes the same decisions; the vector work stays in ops' kernels.

    ops: .have_g, .L, .n_pairs, evaluate() -> L, set_gradient(), direction() -> (gtd, fallback),
         trial(alpha), accept() -> stored (bool), reject().
    The first step length and every accept / backtrack decision come from the library
    (mpf_line_search_first / mpf_line_search_decide: the rule mpf_lbfgs_step applies).
    """
    import ctypes
    from . import _lib as Lb
    lib = Lb.lib()
    if not ops.have_g:
        ops.L = ops.evaluate()
        ops.set_gradient()
    L0 = ops.L
    gtd, fallback = ops.direction()
    if not (np.isfinite(L0) and np.isfinite(gtd)):
        raise FloatingPointError("L-BFGS: non-finite loss or direction")
    a = ctypes.c_double()
    Lb.check(lib.mpf_line_search_first(float(alpha0), int(ops.n_pairs), ctypes.byref(a)), "mpf_line_search_first")
    alpha = a.value
    L, evals, accepted = L0, 0, False
    decision, nxt = ctypes.c_int32(), ctypes.c_double()
    while True:
        ops.trial(alpha)
        L = ops.evaluate()
        evals += 1
        Lb.check(lib.mpf_line_search_decide(float(L0), float(gtd), float(c), float(beta), float(alpha), float(L),
                                            evals, int(max_backtracks), ctypes.byref(decision), ctypes.byref(nxt)),
                 "mpf_line_search_decide")
        if decision.value != 0:
            accepted = decision.value == 1
            break
        alpha = nxt.value
    if accepted:
        ops.accept()
        ops.L = L
    else:
        ops.reject()
        L = L0
    return {"loss0": L0, "loss": L, "alpha": alpha if accepted else 0.0, "accepted": accepted, "evals": evals,
            "fallback": bool(fallback), "pairs": ops.n_pairs}
