"""ctypes binding of libmpf (include/mpf.h).  Argument marshalling only.

Every function here has the name of the C entry point it wraps.  There is no
fallback: if libmpf.so is missing or fails to load, importing raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libmpf.so")

MPF_OK, MPF_ERR_ARG, MPF_ERR_CONFIG, MPF_ERR_DATA, MPF_ERR_INTERNAL, MPF_ERR_CUDA, MPF_ERR_STATE = range(7)
MPF_CONV, MPF_POOL, MPF_FC = 0, 1, 2
MPF_TANH, MPF_IDENTITY, MPF_LOGISTIC = 0, 1, 2
MPF_PREC_TF32, MPF_PREC_FP32 = 0, 1
MPF_TAPE_VALUE, MPF_TAPE_ARGMAX = 0, 1
MPF_MAX_LAYERS = 24
# kernel-selection flags (mpf_config.flags / mpf_net_set_flags; include/mpf.h)
MPF_FLAG_SERIAL = 1 << 0
MPF_FLAG_TC_SINGLE = 1 << 1
MPF_FLAG_TC_PAIR = 1 << 2
MPF_FLAG_NTAP_ON = 1 << 3
MPF_FLAG_NTAP_OFF = 1 << 4
MPF_FLAG_NTAP_NO_MC = 1 << 5
MPF_FLAG_WGRAD_M128 = 1 << 6
MPF_FLAG_ROLE_TIMERS = 1 << 7
MPF_FLAG_FUSE_FIRST_POOL = 1 << 8
MPF_FLAG_HEAD_LOGITS_OFF = 1 << 9
MPF_FLAG_HEAD_LOGITS_ON = 1 << 10
MPF_FLAG_MPF_BWD_BLOCK = 1 << 11
MPF_FLAG_MPF_BWD_SCATTER = 1 << 12

# every symbol include/mpf.h declares
EXPORTS = ("mpf_version", "mpf_last_error", "mpf_net_create", "mpf_net_destroy", "mpf_net_geometry",
           "mpf_net_set_flags", "mpf_net_set_grad_hook",
           "mpf_net_memory", "mpf_net_bind", "mpf_forward_image", "mpf_backward_image", "mpf_sgd_step",
           "mpf_train_step", "mpf_train_step_host", "mpf_fragments_to_pixels", "mpf_mirror_pad", "mpf_class_weights_auto", "mpf_armijo_step",
           "mpf_lbfgs_state_bytes", "mpf_lbfgs_create", "mpf_lbfgs_destroy", "mpf_lbfgs_reset", "mpf_lbfgs_set_gradient", "mpf_lbfgs_direction",
           "mpf_lbfgs_trial", "mpf_lbfgs_accept", "mpf_lbfgs_reject", "mpf_lbfgs_step",
           "mpf_debug_tape", "mpf_check", "mpf_profile_begin",
           "mpf_profile_end", "mpf_exchange_bytes", "mpf_exchange_attach", "mpf_exchange_push",
           "mpf_exchange_sgd_step", "mpf_exchange_detach", "mpf_ipc_export", "mpf_ipc_open", "mpf_ipc_close",
           "mpf_line_search_first", "mpf_line_search_decide")


# void (*mpf_grad_ready_fn)(void* user, int32_t layer, int64_t offset, int64_t count, void* stream)
GRAD_READY_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_void_p)


class MpfLayer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("k", ctypes.c_int32), ("n_out", ctypes.c_int32), ("act", ctypes.c_int32)]


class MpfConfig(ctypes.Structure):
    _fields_ = [("in_channels", ctypes.c_int32), ("patch", ctypes.c_int32), ("image_rows", ctypes.c_int32),
                ("image_cols", ctypes.c_int32), ("max_images", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("debug_keep", ctypes.c_int32)]


_L1 = MPF_MAX_LAYERS + 1


class MpfGeometry(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("n_levels", ctypes.c_int32), ("classes", ctypes.c_int32),
                ("stride", ctypes.c_int32), ("n_fragments", ctypes.c_int32), ("out_rows", ctypes.c_int32),
                ("out_cols", ctypes.c_int32), ("padded_rows", ctypes.c_int32), ("padded_cols", ctypes.c_int32),
                ("frag_rows", ctypes.c_int32), ("frag_cols", ctypes.c_int32), ("n_params", ctypes.c_int64),
                ("frag", ctypes.c_int32 * _L1), ("rows", ctypes.c_int32 * _L1), ("cols", ctypes.c_int32 * _L1),
                ("chans", ctypes.c_int32 * _L1), ("w_offset", ctypes.c_int64 * MPF_MAX_LAYERS),
                ("b_offset", ctypes.c_int64 * MPF_MAX_LAYERS)]


class MpfKernelStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 40), ("layer", ctypes.c_int32), ("launches", ctypes.c_int32),
                ("total_ms", ctypes.c_double), ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libmpf.so not found at {path}: build it with `python -m paper_1302_1690_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i32, u64p = ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint64)
    st = ctypes.c_int
    lib.mpf_version.restype = i32
    lib.mpf_version.argtypes = []
    lib.mpf_last_error.restype = ctypes.c_char_p
    lib.mpf_last_error.argtypes = []
    lib.mpf_net_create.restype = st
    lib.mpf_net_create.argtypes = [ctypes.POINTER(MpfConfig), ctypes.POINTER(MpfLayer), i32, ctypes.POINTER(vp)]
    lib.mpf_net_destroy.restype = None
    lib.mpf_net_destroy.argtypes = [vp]
    lib.mpf_net_geometry.restype = st
    lib.mpf_net_geometry.argtypes = [vp, ctypes.POINTER(MpfGeometry)]
    lib.mpf_net_set_flags.restype = st
    lib.mpf_net_set_flags.argtypes = [vp, ctypes.c_uint32]
    lib.mpf_net_set_grad_hook.restype = st
    lib.mpf_net_set_grad_hook.argtypes = [vp, GRAD_READY_FN, vp]
    lib.mpf_net_memory.restype = st
    lib.mpf_net_memory.argtypes = [vp, i32, u64p, u64p, u64p, u64p]
    lib.mpf_net_bind.restype = st
    lib.mpf_net_bind.argtypes = [vp, vp, vp, vp, vp, i32]
    lib.mpf_forward_image.restype = st
    lib.mpf_forward_image.argtypes = [vp, vp, i32, vp, vp]
    lib.mpf_backward_image.restype = st
    lib.mpf_backward_image.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_float), vp, vp]
    lib.mpf_sgd_step.restype = st
    lib.mpf_sgd_step.argtypes = [vp, ctypes.c_float, ctypes.c_float, vp]
    lib.mpf_train_step.restype = st
    lib.mpf_train_step.argtypes = [vp, vp, i32, vp, ctypes.POINTER(ctypes.c_float), vp, vp]
    lib.mpf_train_step_host.restype = st
    lib.mpf_train_step_host.argtypes = [vp, vp, vp, i32, ctypes.POINTER(ctypes.c_float), vp, i32, ctypes.c_float,
                                        ctypes.c_float, vp]
    lib.mpf_fragments_to_pixels.restype = st
    lib.mpf_fragments_to_pixels.argtypes = [vp, vp, vp, i32, i32, vp]
    lib.mpf_armijo_step.restype = st
    lib.mpf_armijo_step.argtypes = [vp, vp, i32, vp, ctypes.POINTER(ctypes.c_float), ctypes.c_float, ctypes.c_float,
                                    ctypes.c_float, i32, ctypes.c_float, ctypes.POINTER(ctypes.c_float), vp]
    lib.mpf_lbfgs_state_bytes.restype = st
    lib.mpf_lbfgs_state_bytes.argtypes = [vp, i32, u64p]
    lib.mpf_lbfgs_create.restype = st
    lib.mpf_lbfgs_create.argtypes = [vp, i32, vp, ctypes.c_uint64, ctypes.POINTER(vp)]
    lib.mpf_lbfgs_destroy.restype = None
    lib.mpf_lbfgs_destroy.argtypes = [vp]
    lib.mpf_lbfgs_reset.restype = st
    lib.mpf_lbfgs_reset.argtypes = [vp]
    lib.mpf_lbfgs_set_gradient.restype = st
    lib.mpf_lbfgs_set_gradient.argtypes = [vp, ctypes.c_float, vp]
    lib.mpf_lbfgs_direction.restype = st
    lib.mpf_lbfgs_direction.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32), vp]
    lib.mpf_lbfgs_trial.restype = st
    lib.mpf_lbfgs_trial.argtypes = [vp, ctypes.c_double, vp]
    lib.mpf_lbfgs_accept.restype = st
    lib.mpf_lbfgs_accept.argtypes = [vp, ctypes.c_float, ctypes.POINTER(i32), vp]
    lib.mpf_lbfgs_reject.restype = st
    lib.mpf_lbfgs_reject.argtypes = [vp, vp]
    lib.mpf_lbfgs_step.restype = st
    lib.mpf_lbfgs_step.argtypes = [vp, vp, i32, vp, ctypes.POINTER(ctypes.c_float), ctypes.c_float, ctypes.c_float,
                                   ctypes.c_float, i32, ctypes.c_float, ctypes.POINTER(ctypes.c_float), vp]
    lib.mpf_mirror_pad.restype = st
    lib.mpf_mirror_pad.argtypes = [vp, i32, i32, i32, i32, i32, i32, i32, vp, vp]
    lib.mpf_class_weights_auto.restype = st
    lib.mpf_class_weights_auto.argtypes = [vp, vp, i32, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_uint64),
                                           vp]
    lib.mpf_debug_tape.restype = st
    lib.mpf_debug_tape.argtypes = [vp, i32, i32, vp, vp]
    lib.mpf_check.restype = st
    lib.mpf_check.argtypes = [vp, vp]
    lib.mpf_profile_begin.restype = st
    lib.mpf_profile_begin.argtypes = [vp, i32]
    lib.mpf_profile_end.restype = st
    lib.mpf_profile_end.argtypes = [vp, ctypes.POINTER(MpfKernelStat), i32, ctypes.POINTER(i32)]
    lib.mpf_exchange_bytes.restype = st
    lib.mpf_exchange_bytes.argtypes = [vp, i32, u64p]
    lib.mpf_exchange_attach.restype = st
    lib.mpf_exchange_attach.argtypes = [vp, i32, i32, ctypes.POINTER(vp), i32]
    lib.mpf_exchange_push.restype = st
    lib.mpf_exchange_push.argtypes = [vp, vp]
    lib.mpf_exchange_sgd_step.restype = st
    lib.mpf_exchange_sgd_step.argtypes = [vp, ctypes.c_float, ctypes.c_float, vp]
    lib.mpf_exchange_detach.restype = st
    lib.mpf_exchange_detach.argtypes = [vp]
    lib.mpf_ipc_export.restype = st
    lib.mpf_ipc_export.argtypes = [vp, vp, u64p]
    lib.mpf_ipc_open.restype = st
    lib.mpf_ipc_open.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(vp)]
    lib.mpf_ipc_close.restype = st
    lib.mpf_ipc_close.argtypes = [vp, ctypes.c_uint64]
    dbl, dblp = ctypes.c_double, ctypes.POINTER(ctypes.c_double)
    lib.mpf_line_search_first.restype = st
    lib.mpf_line_search_first.argtypes = [dbl, i32, dblp]
    lib.mpf_line_search_decide.restype = st
    lib.mpf_line_search_decide.argtypes = [dbl, dbl, dbl, dbl, dbl, dbl, i32, i32, ctypes.POINTER(i32), dblp]
    return lib


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


class MpfError(RuntimeError):
    def __init__(self, status, where):
        msg = lib().mpf_last_error().decode(errors="replace")
        super().__init__(f"{where} failed with status {status}: {msg}")
        self.status = status


def check(status, where):
    if status != MPF_OK:
        raise MpfError(status, where)
