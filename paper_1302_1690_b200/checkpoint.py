"""Checkpoint / resume of a network's parameters (the flat canonical-order buffer,
SPEC.md:295; a model file echoes the architecture next to the weights).

One ``.npz`` per checkpoint: ``params`` (float32, canonical order: per layer W[C_out][C_in][k][k]
then b), the architecture echo (``layers`` as rows of (kind, k, n_out, act), ``patch``,
``in_channels``), the step counter and a format version.  Loading checks the echo against the
network it is loaded into, so weights never land in a net of another shape.  Host-side only:
no device work, so it runs (and is tested) without a GPU.
"""
from __future__ import annotations

import os
from typing import Optional, Sequence

import numpy as np

FORMAT = "mpf-checkpoint"
VERSION = 1


def _layer_rows(layers: Sequence) -> np.ndarray:
    return np.array([[int(ly.kind), int(ly.k), int(ly.n_out), int(ly.act)] for ly in layers], dtype=np.int32)


def save_checkpoint(path: str, layers: Sequence, patch: int, in_channels: int, params, step: int = 0) -> None:
    """Write params (any array-like of n_params floats) with the architecture echo; atomic
    (written to a temporary file, then renamed)."""
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float32).reshape(-1))
    tmp = path + ".tmp.npz"
    np.savez(tmp, format=np.array(FORMAT), version=np.int32(VERSION), layers=_layer_rows(layers),
             patch=np.int32(patch), in_channels=np.int32(in_channels), step=np.int64(step), params=p)
    os.replace(tmp, path)


def load_checkpoint(path: str, layers: Optional[Sequence] = None, patch: Optional[int] = None,
                    in_channels: Optional[int] = None, n_params: Optional[int] = None) -> dict:
    """Read a checkpoint; when the expected architecture is given, a mismatch raises ValueError."""
    with np.load(path, allow_pickle=False) as z:
        if str(z["format"]) != FORMAT:
            raise ValueError(f"{path}: not an {FORMAT} file")
        if int(z["version"]) != VERSION:
            raise ValueError(f"{path}: checkpoint version {int(z['version'])}, expected {VERSION}")
        out = dict(layers=z["layers"].copy(), patch=int(z["patch"]), in_channels=int(z["in_channels"]),
                   step=int(z["step"]), params=z["params"].copy())
    if layers is not None and not np.array_equal(out["layers"], _layer_rows(layers)):
        raise ValueError(f"{path}: layer list differs from the network's")
    if patch is not None and out["patch"] != int(patch):
        raise ValueError(f"{path}: patch {out['patch']}, network {patch}")
    if in_channels is not None and out["in_channels"] != int(in_channels):
        raise ValueError(f"{path}: in_channels {out['in_channels']}, network {in_channels}")
    if n_params is not None and out["params"].size != int(n_params):
        raise ValueError(f"{path}: {out['params'].size} parameters, network {n_params}")
    return out
