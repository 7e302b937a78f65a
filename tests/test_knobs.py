"""paper_2605_17613_b200/knobs.py (the knob selection bench.py uses) equals
the compiled reference's intra_throughput / optimize_intra
(oracle/_ref, analytics.cpp:45-82, :130-150) on a grid of configurations,
including the measured B200 constants."""
import ctypes as C

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import knobs as K


def _ref():
    r = T.ref()
    if r is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    r.ref_intra_throughput.restype = C.c_double
    r.ref_intra_throughput.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_double)]
    r.ref_optimize_intra.restype = C.c_double
    r.ref_optimize_intra.argtypes = [C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    return r


def _tab(table):
    xs = np.array(sorted(table), np.int32)
    gs = np.array([table[x] for x in xs], np.float64)
    return xs.size, T.ptr(xs, C.c_int), T.ptr(gs, C.c_double), (xs, gs)


# measured B200 constants (round 1/2): decode-step HBM rate, pinned H2D, c of int4 KIVI
B200 = K.Hardware(hbm_bandwidth=5.79e12, interconnect_bandwidth=55.5e9, gpu_mem=179_000_000_000)
W8B, KV32K = 15_010_000_000, 4_294_967_296


def test_expected_gamma_nearest_tie_smaller():
    t = {4: 0.9, 8: 0.8, 16: 0.6}
    assert K.expected_gamma(t, 8) == 0.8
    assert K.expected_gamma(t, 6) == 0.9       # tie 4 vs 8 -> smaller
    assert K.expected_gamma(t, 7) == 0.8
    assert K.expected_gamma(t, 1) == 0.9 and K.expected_gamma(t, 99) == 0.6


def test_intra_throughput_equals_reference():
    r = _ref()
    rng = np.random.default_rng(0)
    table = {2: 0.95, 6: 0.86, 16: 0.72, 30: 0.70, 47: 0.45, 64: 0.38}
    n, xp, gp, keep = _tab(table)
    checked = 0
    for _ in range(400):
        batch = int(rng.integers(1, 65))
        b_c = int(rng.integers(0, batch + 1))
        x = int(rng.integers(1, 65))
        l = int(rng.integers(1, 9))
        c = float(rng.choice([0.266, 0.141, 0.2, 0.5]))
        hw = K.Hardware(float(rng.uniform(1e12, 8e12)), float(rng.uniform(1e10, 1e11)),
                        int(rng.integers(40, 200)) * 1_000_000_000)
        w = int(rng.integers(1, 150)) * 1_000_000_000
        kv = int(rng.integers(1, 20)) * 500_000_000
        want = r.ref_intra_throughput(b_c, x, c, l, hw.hbm_bandwidth, hw.interconnect_bandwidth, hw.gpu_mem,
                                      w, kv, batch, n, xp, gp)
        got = K.intra_throughput(b_c, x, c, l, hw, w, kv, batch, table)
        if want == -1.0:
            assert got is None
        else:
            assert got is not None and got == want, (b_c, x, c, l, got, want)
            checked += 1
    assert checked > 50


@pytest.mark.parametrize("batch,kv,c", [(16, KV32K, 0.266), (48, KV32K, 0.266), (64, KV32K, 0.141),
                                        (4, 4 * KV32K, 0.2)])
def test_optimize_intra_equals_reference(batch, kv, c):
    r = _ref()
    table = {2: 0.95, 6: 0.86, 16: 0.72, 30: 0.70, 47: 0.45, 64: 0.38}
    n, xp, gp, keep = _tab(table)
    bc, x, l = C.c_int(), C.c_int(), C.c_int()
    want = r.ref_optimize_intra(c, 64, 8, B200.hbm_bandwidth, B200.interconnect_bandwidth, B200.gpu_mem, W8B, kv,
                                batch, n, xp, gp, C.byref(bc), C.byref(x), C.byref(l))
    got = K.optimize_intra(B200, W8B, kv, batch, table, c)
    assert want > 0 and got is not None
    assert got == (want, bc.value, x.value, l.value)


def test_composed_accept_length_matches_reference():
    """knobs.composed_accept_length == the compiled reference's
    composed_accept_length (analytics.cpp:413-422) with gamma(x) tabulated at x."""
    r = _ref()
    r.ref_composed_accept_length.restype = C.c_double
    r.ref_composed_accept_length.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double]
    for x, c, d_e, g, ge in [(8, 0.27, 1, 0.5, 0.9), (6, 0.27, 3, 0.872, 0.25), (47, 0.14, 4, 0.42, 0.0),
                             (16, 0.2, 2, 0.7, 1.0)]:
        want = r.ref_composed_accept_length(x, c, d_e, g, ge)
        assert want >= 0
        assert abs(K.composed_accept_length(x, g, d_e, ge) - want) <= 1e-12 * max(1.0, want)
    with pytest.raises(ValueError):
        K.composed_accept_length(6, 0.8, 3, 1.5)
