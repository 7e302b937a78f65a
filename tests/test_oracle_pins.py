"""CPU: pin the oracle and the product's host algorithms to the reference.

Golden vectors come from the reference's own tests (cited per test); where
the compiled reference (oracle/_ref, built from /root/reference by
`make -C oracle ref`) is present the restatements are also compared with it
on seeded inputs.  The committed fixtures in tests/golden/ carry the same
vectors for machines without /root/reference."""
import ctypes as C
import math
import json
import os

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import accept, drop_indices, reload_span

GOLD = json.load(open(os.path.join(T.GOLDEN, "reference_vectors.json")))


# ---- accept rule: test_specloop.cpp:86-115 --------------------------------
@pytest.mark.parametrize("case", GOLD["accept"])
def test_accept_golden(case):
    r = accept(case["drafted"], case["preds"])
    assert r.accepted == case["accepted"]
    assert r.bonus_used == case["bonus"]
    assert (r.first_mismatch or 0) == case["first_mismatch"]
    # the C oracle restates the same rule
    o = T.oracle()
    d = np.array(case["drafted"], np.int32)
    p = np.array(case["preds"], np.int32)
    out = np.zeros(d.size + 1, np.int32)
    fm, bonus = C.c_int(), C.c_int()
    n = o.vco_accept(T.ptr(d, C.c_int32), T.ptr(p, C.c_int32), d.size, T.ptr(out, C.c_int32),
                     C.byref(fm), C.byref(bonus))
    assert out[:n].tolist() == case["accepted"] and fm.value == case["first_mismatch"]


def test_accept_length_contract():
    import paper_2605_17613_b200 as vc
    with pytest.raises(vc.ContractError):
        accept([1, 2], [1, 2])


# ---- drop-index generation: compressor.cpp:114-177, test_compressor.cpp:43-69
def test_drop_counts_golden():
    d = drop_indices("drop-uniform", 4, 8, 100, 0.25, seed=1)
    assert d.shape == (4, 8, 75)
    assert all((np.diff(h) > 0).all() for l in d for h in l)
    w = drop_indices("drop-window", 2, 4, 100, 0.25, seed=0, sink_tokens=4)
    assert (w[0, 0] == np.arange(4, 79)).all()


def test_drop_uniform_100k():
    d = drop_indices("drop-uniform", 2, 4, 100000, 0.25, seed=7)
    assert d.shape == (2, 4, 75000)


def test_drop_rejects_sub_token_ratio():
    import paper_2605_17613_b200 as vc
    with pytest.raises(vc.ConfigError):
        drop_indices("drop-uniform", 1, 1, 10, 0.01)


@pytest.mark.parametrize("tokens,ratio,seed", [(100, 0.25, 1), (4096, 0.2, 9), (777, 0.5, 123)])
def test_drop_uniform_matches_fixture_and_oracle(tokens, ratio, seed):
    got = drop_indices("drop-uniform", 2, 3, tokens, ratio, seed=seed)
    o = T.oracle()
    drop = tokens - int(math.floor(ratio * tokens + 0.5))
    want = np.zeros((2, 3, drop), np.int64)
    assert o.vco_drop_indices(0, 2, 3, tokens, ratio, seed, 0, T.ptr(want, C.c_int64)) == drop
    np.testing.assert_array_equal(got, want)
    key = f"{tokens}_{ratio}_{seed}"
    fx = GOLD["drop_uniform_digest"][key]
    assert int(np.bitwise_xor.reduce(got.reshape(-1) * 2654435761 % (1 << 61))) == fx


def test_drop_uniform_matches_reference_library():
    r = T.ref()
    if r is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    for tokens, ratio, seed in [(100, 0.25, 1), (4096, 0.2, 9), (32768, 0.3, 2)]:
        drop = tokens - int(math.floor(ratio * tokens + 0.5))
        want = np.zeros((2, 3, drop), np.int64)
        pay, bs = C.c_int64(), C.c_int()
        n = r.ref_compress(0, 2, 3, tokens, 256, ratio, 4, seed, 0, T.ptr(want, C.c_int64),
                           C.byref(pay), C.byref(bs))
        assert n == drop
        np.testing.assert_array_equal(drop_indices("drop-uniform", 2, 3, tokens, ratio, seed=seed), want)


# ---- reload_span: test_scheduler.cpp:50-66 -----------------------------------
def test_reload_span_golden():
    it, w = reload_span(4000000000, 5e10, 0.037)
    assert abs(it - 2.162162162) < 1e-8 and w == 3
    it, w = reload_span(1850000000, 5e10, 0.037)
    assert abs(it - 1.0) < 1e-12 and w == 1
    it, w = reload_span(185000000, 5e10, 0.037)
    assert abs(it - 0.1) < 1e-9 and w == 1


# ---- mt19937_64 restatement ----------------------------------------------------
def test_mt64_first_outputs():
    """std::mt19937_64 default-seed 10000th output is 9981545732273789042 (ISO C++)."""
    o = T.oracle()

    class MT(C.Structure):
        _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]

    s = MT()
    o.vco_mt64_seed(C.byref(s), C.c_uint64(5489))
    o.vco_mt64_next.argtypes = [C.POINTER(MT)]
    for _ in range(9999):
        o.vco_mt64_next(C.byref(s))
    assert o.vco_mt64_next(C.byref(s)) == 9981545732273789042


# ---- speculative protocol over the reference's random oracles ---------------
def test_protocol_lossless_reference_oracles():
    """specloop.cpp run_speculative == autoregress over random_table_oracle pairs
    (test_specloop.cpp:130-148), restated by the C oracle's accept."""
    r = T.ref()
    if r is None:
        pytest.skip("oracle/_ref not built")
    for seed in range(8):
        def nxt(sd, pre):
            a = np.array(pre, np.int32)
            return r.ref_random_table_next(4, sd, T.ptr(a, C.c_int32), a.size)
        ctx, out = [0, 1], []
        while len(out) < 32:
            dr = []
            for _ in range(5):
                dr.append(nxt(seed * 2 + 1, ctx + dr))
            preds = [nxt(seed * 2 + 2, ctx + dr[:k]) for k in range(6)]
            acc = accept(dr, preds).accepted
            out += acc
            ctx += acc
        ctx2, ar = [0, 1], []
        for _ in range(32):
            t = nxt(seed * 2 + 2, ctx2)
            ar.append(t)
            ctx2.append(t)
        assert out[:32] == ar


# ---- size law / quant metadata: test_compressor.cpp:71-79 ---------------------
def test_quant_size_law_reference():
    r = T.ref()
    if r is None:
        pytest.skip("oracle/_ref not built")
    pay, bs = C.c_int64(), C.c_int()
    r.ref_compress(2, 4, 8, 100, 128, 0.0, 4, 0, 0, None, C.byref(pay), C.byref(bs))
    assert bs.value == 4 and pay.value == 4 * 8 * 100 * 128 // 4
