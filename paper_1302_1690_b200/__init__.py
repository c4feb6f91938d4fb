"""paper_1302_1690_b200 — B200-native whole-image MPCNN training with MaxPoolingFragment layers.

The product is the C-ABI library ``lib/libmpf.so`` (include/mpf.h) built from the
sm_100a CUDA sources in ``csrc/``; this package holds its build script and a thin
ctypes binding.  Nothing here imports the oracle.
"""
from ._lib import (MPF_CONV, MPF_FC, MPF_IDENTITY, MPF_LOGISTIC, MPF_POOL, MPF_PREC_FP32, MPF_PREC_TF32,  # noqa: F401
                   MPF_TANH, MPF_TAPE_ARGMAX, MPF_TAPE_VALUE, EXPORTS, LIB_PATH, MpfError)

__all__ = ["MPFNet", "EXPORTS", "LIB_PATH", "MpfError"]


def __getattr__(name):
    if name == "MPFNet":
        from .net import MPFNet
        return MPFNet
    raise AttributeError(name)
