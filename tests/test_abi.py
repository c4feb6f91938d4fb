"""C-ABI: the library loads without a GPU, exports every symbol include/mpf.h declares,
and its host-side geometry planner (validate_arch + plan_geometry) matches the closed
forms (no device calls)."""
import ctypes
import os
import re

import pytest

import mpf_synth as S
from paper_1302_1690_b200 import _lib as L
from paper_1302_1690_b200.net import layers_to_c

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "mpf.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mpf_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = L.lib()
    declared = _header_functions()
    assert set(declared) == set(L.EXPORTS), (declared, L.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.mpf_version() == 1


def _create(cfg_name=None, layers=None, P=None, H=None, W=None, n=1, expect=L.MPF_OK):
    lib = L.lib()
    if cfg_name:
        c = S.CONFIGS[cfg_name]
        layers, P, H, W = c.layers, c.P, c.H, c.W
    cfg = L.MpfConfig(1, P, H, W, n, L.MPF_PREC_TF32, 0, 0)
    h = ctypes.c_void_p()
    st = lib.mpf_net_create(ctypes.byref(cfg), layers_to_c(layers), len(layers), ctypes.byref(h))
    assert st == expect, lib.mpf_last_error()
    if st != L.MPF_OK:
        return None, None
    g = L.MpfGeometry()
    assert lib.mpf_net_geometry(h, ctypes.byref(g)) == L.MPF_OK
    return h, g


# closed forms: F = prod k^2, O = H - P + 1, H' = P - 1 + S ceil(O / S)
@pytest.mark.parametrize("name,F,O,Hp,npar", [("cfg1", 16, 19, 33, 898), ("cfg2", 64, 85, 131, 70622),
                                              ("cfg3", 64, 469, 515, 70622), ("cfg4", 256, 931, 1037, 548885),
                                              ("cfg5", 729, 685, 785, 79754)])
def test_geometry_closed_forms(name, F, O, Hp, npar):
    h, g = _create(name, n=8)
    c = S.CONFIGS[name]
    assert g.n_fragments == F
    assert g.out_rows == g.out_cols == O == c.H - c.P + 1
    assert g.padded_rows == Hp
    S_ = g.stride
    assert g.padded_rows == c.P - 1 + S_ * ((O + S_ - 1) // S_)
    assert g.frag_rows * S_ >= O > (g.frag_rows - 1) * S_
    assert g.n_params == npar == S.n_params(c.layers)
    # parameter offsets follow the canonical order
    off = 0
    for l, ly in enumerate(c.layers):
        if ly.kind == S.POOL:
            assert g.w_offset[l] == -1
            continue
        assert g.w_offset[l] == off
        off += ly.n_out * g.chans[l] * ly.k * ly.k
        assert g.b_offset[l] == off
        off += ly.n_out
    # memory query works without a device
    pb, gb, tb, sb = (ctypes.c_uint64() for _ in range(4))
    assert L.lib().mpf_net_memory(h, 8, ctypes.byref(pb), ctypes.byref(gb), ctypes.byref(tb), ctypes.byref(sb)) == 0
    assert pb.value == 4 * npar and tb.value > 0 and sb.value > 0
    L.lib().mpf_net_destroy(h)


def test_uniform_fragment_chain():
    # every level's fragments have equal size: n = k m + k - 1 before each pool
    for name in S.CONFIGS:
        c = S.CONFIGS[name]
        h, g = _create(name)
        for l, ly in enumerate(c.layers):
            if ly.kind == S.POOL:
                n_in = g.rows[l]
                assert (n_in - ly.k + 1) % ly.k == 0
                assert g.rows[l + 1] == (n_in - ly.k + 1) // ly.k
                assert g.frag[l + 1] == g.frag[l] * ly.k * ly.k
        L.lib().mpf_net_destroy(h)


def test_rejects_inexact_geometry_and_bad_heads():
    c = S.CONFIGS["cfg4"]
    _create(layers=c.layers, P=96, H=1024, W=1024, expect=L.MPF_ERR_CONFIG)   # R1
    c5 = S.CONFIGS["cfg5"]
    _create(layers=c5.layers, P=90, H=768, W=768, expect=L.MPF_ERR_CONFIG)
    # last layer must be a linear 1x1 FC
    bad = c.layers[:-1] + (S.F(1, 5, S.TANH),)
    _create(layers=bad, P=94, H=200, W=200, expect=L.MPF_ERR_CONFIG)
    # image smaller than the patch
    _create(layers=c.layers, P=94, H=90, W=200, expect=L.MPF_ERR_CONFIG)


def test_bind_requires_alignment_and_state():
    h, g = _create("cfg1")
    lib = L.lib()
    # forward before bind -> MPF_ERR_STATE, no device touched
    st = lib.mpf_forward_image(h, ctypes.c_void_p(256), 1, None, None)
    assert st == L.MPF_ERR_STATE
    st = lib.mpf_net_bind(h, ctypes.c_void_p(256), ctypes.c_void_p(512), ctypes.c_void_p(300),
                          ctypes.c_void_p(1024), 1)
    assert st == L.MPF_ERR_ARG  # tape not 256-aligned
    lib.mpf_net_destroy(h)


def test_product_does_not_import_oracle():
    # the product package must not reference the oracle (task rule: no CPU fallback)
    pkg = os.path.join(ROOT, "paper_1302_1690_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "o1_patch" not in txt, f


def test_kernel_selection_flags_are_validated():
    """mpf_config.flags / mpf_net_set_flags (host only): unknown bits and contradictory
    pairs are argument errors, at create and later; valid flags are accepted."""
    lib = L.lib()
    c = S.CONFIGS["cfg2"]
    for bad in (1 << 20, L.MPF_FLAG_NTAP_ON | L.MPF_FLAG_NTAP_OFF, L.MPF_FLAG_TC_PAIR | L.MPF_FLAG_TC_SINGLE,
                L.MPF_FLAG_HEAD_LOGITS_ON | L.MPF_FLAG_HEAD_LOGITS_OFF):
        cfg = L.MpfConfig(1, c.P, c.H, c.W, 1, L.MPF_PREC_TF32, bad, 0)
        h = ctypes.c_void_p()
        assert lib.mpf_net_create(ctypes.byref(cfg), layers_to_c(c.layers), len(c.layers), ctypes.byref(h)) == L.MPF_ERR_ARG
    h, _ = _create("cfg2")
    assert lib.mpf_net_set_flags(h, L.MPF_FLAG_SERIAL | L.MPF_FLAG_NTAP_OFF | L.MPF_FLAG_WGRAD_M128) == L.MPF_OK
    assert lib.mpf_net_set_flags(h, 1 << 30) == L.MPF_ERR_ARG
    assert lib.mpf_net_set_flags(h, 0) == L.MPF_OK
    lib.mpf_net_destroy(h)


def test_line_search_rule_host_only():
    """mpf_line_search_first / _decide (the backtracking rule of mpf_lbfgs_step, PAPER.md:251,
    reading R21) on the host: Armijo acceptance L <= L0 + c alpha g'd, backtracking by beta,
    giving up after max_backtracks + 1 trials, non-finite losses never accepted."""
    lib = L.lib()
    a = ctypes.c_double()
    assert lib.mpf_line_search_first(0.25, 0, ctypes.byref(a)) == 0 and a.value == 0.25
    assert lib.mpf_line_search_first(0.25, 3, ctypes.byref(a)) == 0 and a.value == 1.0

    def decide(L0, gtd, alpha, Lt, trials, maxb=2, c=0.1, beta=0.5):
        d, n = ctypes.c_int32(), ctypes.c_double()
        st = lib.mpf_line_search_decide(L0, gtd, c, beta, alpha, Lt, trials, maxb, ctypes.byref(d), ctypes.byref(n))
        return st, d.value, n.value
    # L0 = 1, g'd = -2, alpha = 1, c = 0.1: threshold 0.8
    assert decide(1.0, -2.0, 1.0, 0.8, 1) == (0, 1, 1.0)       # equality accepts
    assert decide(1.0, -2.0, 1.0, 0.80001, 1) == (0, 0, 0.5)   # backtrack to beta * alpha
    assert decide(1.0, -2.0, 0.25, 0.99, 3) == (0, -1, 0.25)   # third trial with max_backtracks 2: give up
    assert decide(1.0, -2.0, 0.5, 0.95, 2)[1] == 0             # second trial: one more allowed
    assert decide(1.0, -2.0, 1.0, float("nan"), 1)[1] == 0     # NaN never accepted
    assert decide(1.0, -2.0, 1.0, float("-inf"), 1)[1] == 0    # nor -inf
    assert decide(1.0, -2.0, 1.0, 0.5, 1, beta=1.0)[0] == L.MPF_ERR_ARG
    assert decide(1.0, -2.0, 1.0, 0.5, 0)[0] == L.MPF_ERR_ARG
