"""CPU: the swap scheduler libvericache ships (speckv_host.cpp) reproduces the
reference's scheduler bit-for-bit:
  * the 100k-iteration safety soak digest of acceptance_test.cpp:412-517
    (ba3edc09c927c03c, committed in tests/golden/reference_vectors.json from
    the compiled reference) and a second seed;
  * Algorithm 1's candidate order (test_scheduler.cpp:77-95), the waiting
    outcome (:97-110), bit-exact release (:127-166), cadence (:206-232)."""
import ctypes as C
import json
import os
import subprocess

import numpy as np
import pytest

import vc_testlib as T

BUILD = os.path.join(T.ROOT, "tests", "_build")
SO = os.path.join(BUILD, "libsched_checks.so")


@pytest.fixture(scope="module")
def sc():
    os.makedirs(BUILD, exist_ok=True)
    src = [os.path.join(T.ROOT, "tests", "cpp", "sched_checks.cpp"),
           os.path.join(T.ROOT, "paper_2605_17613_b200", "csrc", "speckv_host.cpp")]
    if not os.path.exists(SO) or any(os.path.getmtime(s) > os.path.getmtime(SO) for s in src):
        subprocess.check_call(["g++", "-std=c++20", "-O2", "-fPIC", "-shared",
                               "-I" + os.path.join(T.ROOT, "include"), "-o", SO] + src)
    lib = C.CDLL(SO)
    lib.sc_soak.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                            C.POINTER(C.c_int64)]
    return lib


GOLD = json.load(open(os.path.join(T.GOLDEN, "reference_vectors.json")))


@pytest.mark.parametrize("key", ["99_100000", "7_20000"])
def test_soak_digest_matches_reference(sc, key):
    seed, iters = map(int, key.split("_"))
    d, em, cpl = C.c_uint64(), C.c_double(), C.c_int64()
    assert sc.sc_soak(seed, iters, C.byref(d), C.byref(em), C.byref(cpl)) == 0
    want = GOLD["soak"][key]
    assert f"{d.value:016x}" == want["digest"]
    assert em.value == want["emitted"] and cpl.value == want["completed"]


def test_soak_digest_live_reference(sc):
    r = T.ref()
    if r is None:
        pytest.skip("oracle/_ref not built")
    for seed in (3, 11):
        a, b = C.c_uint64(), C.c_uint64()
        e1, e2, c1, c2 = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        assert sc.sc_soak(seed, 5000, C.byref(a), C.byref(e1), C.byref(c1)) == 0
        assert r.ref_soak(seed, 5000, C.byref(b), C.byref(e2), C.byref(c2)) == 0
        assert a.value == b.value and e1.value == e2.value and c1.value == c2.value


def test_admit_search_order(sc):
    ex = (C.c_int * 64)()
    vw = C.c_int()
    n = sc.sc_admit_probe(ex, 64, C.byref(vw))
    assert list(ex[:n]) == [25, 24, 26, 23, 27, 22] and vw.value == 22


def test_admit_waiting_outcome(sc):
    assert sc.sc_admit_waiting() == 15


def test_release_bit_exact(sc):
    assert sc.sc_release_exact() == 0


def test_cadence_x_drafts_then_verify(sc):
    x, iters = 3, 40
    v = (C.c_int * iters)()
    d = (C.c_int * iters)()
    sc.sc_cadence(x, iters, v, d)
    ver = np.array(v[:])
    idx = np.nonzero(ver)[0]
    assert len(idx) >= 5
    assert (np.diff(idx) == x + 1).all()
