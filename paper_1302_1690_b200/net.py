"""Thin Python wrapper over the libmpf C ABI (marshalling only).

PyTorch provides device memory and streams; every step of the training path runs
in libmpf's CUDA kernels.  There is no CPU path: constructing an ``MPFNet`` without
a CUDA device, or without the built library, raises.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> Optional[ctypes.c_void_p]:
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def mirror_pad(images: torch.Tensor, patch: int, stream=None) -> torch.Tensor:
    """Same-size-output input: images [n, c, H, W] (cuda float32) mirror-padded
    by floor((P-1)/2) before and the rest of P-1 after each axis (mpf_mirror_pad), so that
    a net created for (H+P-1) x (W+P-1) images predicts exactly H x W pixels."""
    from . import _lib as L
    if images.dtype != torch.float32 or not images.is_cuda or not images.is_contiguous():
        raise ValueError("images must be a contiguous cuda float32 tensor")
    n, c, H, W = images.shape
    pt = (patch - 1) // 2
    out = torch.empty((n, c, H + patch - 1, W + patch - 1), dtype=torch.float32, device=images.device)
    L.check(L.lib().mpf_mirror_pad(_ptr(images), n * c, H, W, pt, pt, H + patch - 1, W + patch - 1, _ptr(out),
                                   _stream_ptr(stream)), "mpf_mirror_pad")
    return out


@dataclass
class Geometry:
    n_layers: int
    n_levels: int
    classes: int
    stride: int
    n_fragments: int
    out_rows: int
    out_cols: int
    padded_rows: int
    padded_cols: int
    frag_rows: int
    frag_cols: int
    n_params: int
    frag: list
    rows: list
    cols: list
    chans: list
    w_offset: list
    b_offset: list


def layers_to_c(layers) -> "ctypes.Array":
    arr = (L.MpfLayer * len(layers))()
    for i, ly in enumerate(layers):
        arr[i].kind, arr[i].k, arr[i].n_out, arr[i].act = int(ly.kind), int(ly.k), int(ly.n_out), int(ly.act)
    return arr


class MPFNet:
    """One network bound to PyTorch-allocated device buffers.

    layers: sequence with .kind/.k/.n_out/.act (mpf_synth.Layer); patch = P.
    """

    def __init__(self, layers: Sequence, patch: int, image_rows: int, image_cols: int, max_images: int,
                 in_channels: int = 1, precision: str = "tf32", device: Optional[torch.device] = None,
                 debug_keep: bool = False, flags: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("MPFNet needs a CUDA device (there is no CPU fallback)")
        self.lib = L.lib()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        cfg = L.MpfConfig(in_channels, patch, image_rows, image_cols, max_images,
                          L.MPF_PREC_TF32 if precision == "tf32" else L.MPF_PREC_FP32, int(flags),
                          1 if debug_keep else 0)
        self.layers = tuple(layers)
        self.patch = patch
        self.in_channels = in_channels
        self.image_rows, self.image_cols = image_rows, image_cols
        self.max_images = max_images
        h = ctypes.c_void_p()
        L.check(self.lib.mpf_net_create(ctypes.byref(cfg), layers_to_c(self.layers), len(self.layers),
                                        ctypes.byref(h)), "mpf_net_create")
        self.h = h
        g = L.MpfGeometry()
        L.check(self.lib.mpf_net_geometry(self.h, ctypes.byref(g)), "mpf_net_geometry")
        nl = g.n_layers
        self.geom = Geometry(g.n_layers, g.n_levels, g.classes, g.stride, g.n_fragments, g.out_rows, g.out_cols,
                             g.padded_rows, g.padded_cols, g.frag_rows, g.frag_cols, g.n_params,
                             list(g.frag[:nl + 1]), list(g.rows[:nl + 1]), list(g.cols[:nl + 1]),
                             list(g.chans[:nl + 1]), list(g.w_offset[:nl]), list(g.b_offset[:nl]))
        pb, gb, tb, sb = (ctypes.c_uint64() for _ in range(4))
        L.check(self.lib.mpf_net_memory(self.h, max_images, ctypes.byref(pb), ctypes.byref(gb), ctypes.byref(tb),
                                        ctypes.byref(sb)), "mpf_net_memory")
        self.bytes = dict(params=pb.value, grads=gb.value, tape=tb.value, scratch=sb.value)
        with torch.cuda.device(self.device):
            self.params = torch.zeros(self.geom.n_params, dtype=torch.float32, device=self.device)
            self.grads = torch.zeros(self.geom.n_params, dtype=torch.float32, device=self.device)
            self.tape = torch.empty(tb.value, dtype=torch.uint8, device=self.device)
            self.scratch = torch.empty(sb.value, dtype=torch.uint8, device=self.device)
        L.check(self.lib.mpf_net_bind(self.h, _ptr(self.params), _ptr(self.grads), _ptr(self.tape),
                                      _ptr(self.scratch), max_images), "mpf_net_bind")
        self._images = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.mpf_net_destroy(h)
            except Exception:
                pass
            self.h = None

    def set_grad_hook(self, fn) -> None:
        """fn(layer, offset, count, stream_ptr) is called during every backward as soon as the
        gradient entries [offset, offset + count) are final in the order of the CUDA stream
        stream_ptr (mpf_net_set_grad_hook; the data-parallel bucketed all-reduce of
        dist.BucketAllReduce).  None removes it."""
        if fn is None:
            self._hook = None
            L.check(self.lib.mpf_net_set_grad_hook(self.h, L.GRAD_READY_FN(), None), "mpf_net_set_grad_hook")
            return

        def _cb(user, layer, offset, count, stream):
            fn(int(layer), int(offset), int(count), stream)
        self._hook = L.GRAD_READY_FN(_cb)  # kept alive as long as the library may call it
        L.check(self.lib.mpf_net_set_grad_hook(self.h, self._hook, None), "mpf_net_set_grad_hook")

    def set_flags(self, flags: int) -> None:
        """Kernel-selection flags (MPF_FLAG_*, include/mpf.h); 0 = the measured defaults."""
        L.check(self.lib.mpf_net_set_flags(self.h, int(flags)), "mpf_net_set_flags")

    # ------------------------------------------------------------------ parameters
    def set_params(self, flat) -> None:
        t = torch.as_tensor(np.asarray(flat, np.float32) if not torch.is_tensor(flat) else flat)
        if t.numel() != self.geom.n_params:
            raise ValueError(f"expected {self.geom.n_params} parameters, got {t.numel()}")
        self.params.copy_(t.reshape(-1).to(self.device, torch.float32))

    def get_params(self) -> torch.Tensor:
        return self.params.clone()

    def save(self, path: str, step: int = 0) -> None:
        """Checkpoint the parameters with the architecture echo (checkpoint.py)."""
        from .checkpoint import save_checkpoint
        save_checkpoint(path, self.layers, self.patch, self.in_channels, self.params.cpu().numpy(), step)

    def load(self, path: str) -> int:
        """Resume from a checkpoint of the same architecture; returns its step counter."""
        from .checkpoint import load_checkpoint
        ck = load_checkpoint(path, self.layers, self.patch, self.in_channels, self.geom.n_params)
        self.set_params(ck["params"])
        return ck["step"]

    def zero_grads(self) -> None:
        self.grads.zero_()

    # ------------------------------------------------------------------ the path
    def forward(self, images: torch.Tensor, want_probs: bool = False, stream=None) -> Optional[torch.Tensor]:
        """images: cuda float32 [n, in_channels, H, W] (kept alive until backward)."""
        if images.dtype != torch.float32 or not images.is_cuda or not images.is_contiguous():
            raise ValueError("images must be a contiguous cuda float32 tensor")
        n = images.shape[0]
        probs = None
        if want_probs:
            g = self.geom
            probs = torch.empty((n * g.n_fragments, g.frag_rows, g.frag_cols, g.classes), dtype=torch.float32,
                                device=self.device)
        L.check(self.lib.mpf_forward_image(self.h, _ptr(images), n, _ptr(probs), _stream_ptr(stream)),
                "mpf_forward_image")
        self._images = images
        return probs

    def backward(self, labels: torch.Tensor, class_w=None, stream=None) -> torch.Tensor:
        """labels: cuda uint8 [n, out_rows, out_cols] (255 = ignore); returns per-image losses [n]."""
        if labels.dtype != torch.uint8 or not labels.is_cuda or not labels.is_contiguous():
            raise ValueError("labels must be a contiguous cuda uint8 tensor")
        n = labels.shape[0]
        loss = torch.empty(n, dtype=torch.float32, device=self.device)
        cw = None
        if class_w is not None:
            arr = (ctypes.c_float * self.geom.classes)(*[float(v) for v in class_w])
            cw = arr
        L.check(self.lib.mpf_backward_image(self.h, _ptr(labels), cw, _ptr(loss), _stream_ptr(stream)),
                "mpf_backward_image")
        return loss

    def train_step(self, images: torch.Tensor, labels: torch.Tensor, class_w=None, stream=None) -> torch.Tensor:
        """Forward + backward in one C call (mpf_train_step).  Gradients are added; returns
        losses [n]."""
        if images.dtype != torch.float32 or not images.is_cuda or not images.is_contiguous():
            raise ValueError("images must be a contiguous cuda float32 tensor")
        if labels.dtype != torch.uint8 or not labels.is_cuda or not labels.is_contiguous():
            raise ValueError("labels must be a contiguous cuda uint8 tensor")
        n = images.shape[0]
        loss = torch.empty(n, dtype=torch.float32, device=self.device)
        cw = None
        if class_w is not None:
            cw = (ctypes.c_float * self.geom.classes)(*[float(v) for v in class_w])
        L.check(self.lib.mpf_train_step(self.h, _ptr(images), n, _ptr(labels), cw, _ptr(loss), _stream_ptr(stream)),
                "mpf_train_step")
        self._images = images
        return loss

    def sgd_step(self, lr: float, grad_scale: float = 1.0, stream=None) -> None:
        L.check(self.lib.mpf_sgd_step(self.h, float(lr), float(grad_scale), _stream_ptr(stream)), "mpf_sgd_step")

    def train_step_host(self, h_images: torch.Tensor, h_labels: torch.Tensor, h_loss: torch.Tensor,
                        apply_sgd: bool = True, lr: float = 0.01, grad_scale: float = 1.0, class_w=None,
                        stream=None) -> None:
        """Host (pinned) buffers in, loss copied back to h_loss; async on `stream`."""
        n = h_images.shape[0]
        cw = None
        if class_w is not None:
            cw = (ctypes.c_float * self.geom.classes)(*[float(v) for v in class_w])
        L.check(self.lib.mpf_train_step_host(self.h, _ptr(h_images), _ptr(h_labels), n, cw, _ptr(h_loss),
                                             1 if apply_sgd else 0, float(lr), float(grad_scale),
                                             _stream_ptr(stream)), "mpf_train_step_host")

    def fragments_to_pixels(self, frag: torch.Tensor, n: int, channels: int, stream=None) -> torch.Tensor:
        g = self.geom
        out = torch.empty((n, channels, g.out_rows, g.out_cols), dtype=torch.float32, device=self.device)
        L.check(self.lib.mpf_fragments_to_pixels(self.h, _ptr(frag), _ptr(out), n, channels, _stream_ptr(stream)),
                "mpf_fragments_to_pixels")
        return out

    def armijo_step(self, images: torch.Tensor, labels: torch.Tensor, alpha0: float = 0.01, beta: float = 0.5,
                    c: float = 1e-4, max_backtracks: int = 10, class_w=None, grad_scale: float = None,
                    stream=None) -> dict:
        """One Armijo-safeguarded step on a batch (mpf_armijo_step; it zeroes the gradient buffer
        before its gradient pass and again at the end); grad_scale defaults to 1/n."""
        n = images.shape[0]
        cw = None
        if class_w is not None:
            cw = (ctypes.c_float * self.geom.classes)(*[float(v) for v in class_w])
        out = (ctypes.c_float * 5)()
        gs = 1.0 / n if grad_scale is None else float(grad_scale)
        L.check(self.lib.mpf_armijo_step(self.h, _ptr(images), n, _ptr(labels), cw, float(alpha0), float(beta),
                                         float(c), int(max_backtracks), gs, out, _stream_ptr(stream)),
                "mpf_armijo_step")
        return {"loss0": out[0], "loss": out[1], "alpha": out[2], "accepted": bool(out[3]), "evals": int(out[4])}

    def predict(self, images: torch.Tensor, stream=None) -> torch.Tensor:
        """Per-pixel softmax probabilities [n, classes, out_rows, out_cols] of whole images
        (forward with the softmax output, then the fragment -> pixel reassembly)."""
        probs = self.forward(images, want_probs=True, stream=stream)
        return self.fragments_to_pixels(probs, images.shape[0], self.geom.classes, stream=stream)

    def class_weights_auto(self, labels: torch.Tensor, stream=None):
        """Inverse-frequency class weights w_c = N / (C n_c) of a batch of label maps
        [n, out_rows, out_cols] (uint8, 255 ignored) and the per-class counts."""
        C = self.geom.classes
        w = (ctypes.c_float * C)()
        cnt = (ctypes.c_uint64 * C)()
        L.check(self.lib.mpf_class_weights_auto(self.h, _ptr(labels), int(labels.shape[0]), w, cnt,
                                                _stream_ptr(stream)), "mpf_class_weights_auto")
        return [float(v) for v in w], [int(v) for v in cnt]

    def debug_tape(self, layer: int, what: int, n: int) -> torch.Tensor:
        g = self.geom
        shape = (n * g.frag[layer + 1], g.rows[layer + 1], g.cols[layer + 1], g.chans[layer + 1])
        dt = torch.uint8 if what == L.MPF_TAPE_ARGMAX else torch.float32
        out = torch.empty(shape, dtype=dt, device=self.device)
        L.check(self.lib.mpf_debug_tape(self.h, layer, what, _ptr(out), _stream_ptr(None)), "mpf_debug_tape")
        return out

    def profile_begin(self, max_launches: int = 100000) -> None:
        L.check(self.lib.mpf_profile_begin(self.h, max_launches), "mpf_profile_begin")

    def profile_end(self) -> list:
        """Per (kernel, layer): launches, total_ms, algorithmic flops/bytes per launch."""
        cap = 512
        arr = (L.MpfKernelStat * cap)()
        n = ctypes.c_int32()
        L.check(self.lib.mpf_profile_end(self.h, arr, cap, ctypes.byref(n)), "mpf_profile_end")
        return [dict(name=arr[i].name.decode(), layer=arr[i].layer, launches=arr[i].launches,
                     total_ms=arr[i].total_ms, flops=arr[i].flops, bytes=arr[i].bytes) for i in range(n.value)]

    def check(self, stream=None) -> None:
        L.check(self.lib.mpf_check(self.h, _stream_ptr(stream)), "mpf_check")

    # ---- data-parallel gradient exchange over peer memory (include/mpf.h mpf_exchange_*;
    # dist.PeerExchange sets it up across processes)
    def exchange_bytes(self, world: int) -> int:
        b = ctypes.c_uint64()
        L.check(self.lib.mpf_exchange_bytes(self.h, int(world), ctypes.byref(b)), "mpf_exchange_bytes")
        return int(b.value)

    def attach_exchange(self, rank: int, world: int, buf_ptrs, push_in_backward: bool = True) -> None:
        """buf_ptrs[r]: device address of rank r's zero-filled exchange buffer as seen from
        this process (buf_ptrs[rank] = this rank's own buffer)."""
        arr = (ctypes.c_void_p * world)(*[int(p) for p in buf_ptrs])
        L.check(self.lib.mpf_exchange_attach(self.h, int(rank), int(world), arr, 1 if push_in_backward else 0),
                "mpf_exchange_attach")

    def exchange_push(self, stream=None) -> None:
        L.check(self.lib.mpf_exchange_push(self.h, _stream_ptr(stream)), "mpf_exchange_push")

    def detach_exchange(self) -> None:
        L.check(self.lib.mpf_exchange_detach(self.h), "mpf_exchange_detach")


class Lbfgs:
    """Full-batch L-BFGS on an MPFNet's parameters (mpf_lbfgs_*, reading R21).

    step(): one iteration on one GPU inside libmpf (mpf_lbfgs_step).
    step_allreduce(): the same iteration over a data-parallel group: each rank evaluates its
    shard, the gradient buffer and the loss are summed over ranks, and the host loop of
    dist.lbfgs_iteration drives the same primitives on every rank."""

    def __init__(self, net: "MPFNet", memory: int = 10):
        self.net = net
        self.lib = net.lib
        self.memory = memory
        nb = ctypes.c_uint64()
        L.check(self.lib.mpf_lbfgs_state_bytes(net.h, int(memory), ctypes.byref(nb)), "mpf_lbfgs_state_bytes")
        # device state allocated by PyTorch and lent to the library (like the net's buffers)
        self.state = torch.empty(nb.value, dtype=torch.uint8, device=net.device)
        h = ctypes.c_void_p()
        L.check(self.lib.mpf_lbfgs_create(net.h, int(memory), _ptr(self.state), nb.value, ctypes.byref(h)),
                "mpf_lbfgs_create")
        self.h = h
        self.have_g, self.L, self.n_pairs = False, 0.0, 0
        self._ctx = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.mpf_lbfgs_destroy(h)
            except Exception:
                pass
            self.h = None

    def reset(self) -> None:
        L.check(self.lib.mpf_lbfgs_reset(self.h), "mpf_lbfgs_reset")
        self.have_g, self.n_pairs = False, 0

    def step(self, images: torch.Tensor, labels: torch.Tensor, alpha0: float = 1.0, beta: float = 0.5,
             c: float = 1e-4, max_backtracks: int = 10, class_w=None, grad_scale: float = None,
             stream=None) -> dict:
        """One iteration over the whole batch `images` (the training set); grad_scale defaults to 1/n."""
        n = images.shape[0]
        cw = None
        if class_w is not None:
            cw = (ctypes.c_float * self.net.geom.classes)(*[float(v) for v in class_w])
        out = (ctypes.c_float * 7)()
        gs = 1.0 / n if grad_scale is None else float(grad_scale)
        L.check(self.lib.mpf_lbfgs_step(self.h, _ptr(images), n, _ptr(labels), cw, float(alpha0), float(beta),
                                        float(c), int(max_backtracks), gs, out, _stream_ptr(stream)),
                "mpf_lbfgs_step")
        self.n_pairs = int(out[6])
        return {"loss0": out[0], "loss": out[1], "alpha": out[2], "accepted": bool(out[3]), "evals": int(out[4]),
                "fallback": bool(out[5]), "pairs": int(out[6])}

    # ---------------------------------------------------------------- primitives (dist.lbfgs_iteration ops)
    def evaluate(self) -> float:
        from . import dist as D
        images, labels, class_w, gs, group = self._ctx
        self.net.zero_grads()
        loss = self.net.train_step(images, labels, class_w=class_w)
        D.allreduce_grads(self.net.grads, group)
        return D.all_sum_scalar(float(loss.double().sum().item()) * gs, device=self.net.device, group=group)

    def set_gradient(self) -> None:
        L.check(self.lib.mpf_lbfgs_set_gradient(self.h, float(self._ctx[3]), _stream_ptr(None)),
                "mpf_lbfgs_set_gradient")
        self.have_g = True

    def direction(self):
        gtd, fb = ctypes.c_double(), ctypes.c_int32()
        L.check(self.lib.mpf_lbfgs_direction(self.h, ctypes.byref(gtd), ctypes.byref(fb), _stream_ptr(None)),
                "mpf_lbfgs_direction")
        return gtd.value, bool(fb.value)

    def trial(self, alpha: float) -> None:
        L.check(self.lib.mpf_lbfgs_trial(self.h, float(alpha), _stream_ptr(None)), "mpf_lbfgs_trial")

    def accept(self) -> bool:
        stored = ctypes.c_int32()
        L.check(self.lib.mpf_lbfgs_accept(self.h, float(self._ctx[3]), ctypes.byref(stored), _stream_ptr(None)),
                "mpf_lbfgs_accept")
        if stored.value:
            self.n_pairs = min(self.n_pairs + 1, self.memory)
        return bool(stored.value)

    def reject(self) -> None:
        L.check(self.lib.mpf_lbfgs_reject(self.h, _stream_ptr(None)), "mpf_lbfgs_reject")
        self.n_pairs = 0

    def step_allreduce(self, images: torch.Tensor, labels: torch.Tensor, global_images: int, alpha0: float = 1.0,
                       beta: float = 0.5, c: float = 1e-4, max_backtracks: int = 10, class_w=None,
                       group=None) -> dict:
        """One iteration whose full batch is the union of every rank's `images`
        (global_images in total; grad_scale = 1 / global_images).  Runs on the current stream."""
        from . import dist as D
        self._ctx = (images, labels, class_w, 1.0 / global_images, group)
        try:
            return D.lbfgs_iteration(self, alpha0, beta, c, max_backtracks)
        finally:
            self._ctx = None
