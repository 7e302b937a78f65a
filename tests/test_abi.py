"""CPU: libvericache.so loads without a GPU, exports every symbol
include/vc_api.h declares, and its host-only entry points (accept, drop
indices, reload_span, update) behave like the reference's (error codes
included: ConfigError -> 1, ContractError -> 2)."""
import ctypes as C
import os
import re

import numpy as np

import vc_testlib as T
from paper_2605_17613_b200 import _lib


def _declared(header):
    txt = open(os.path.join(T.ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vc_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    lib = _lib.load()
    names = _declared("vc_api.h")
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_cpp_api_symbols_exported():
    """The speckv:: drop-in C++ API (include/speckv_b200.hpp) is in the .so."""
    out = os.popen(f"nm -DC {_lib.LIB_PATH}").read()
    for sym in ["speckv::accept(", "speckv::run_speculative(", "speckv::compress(",
                "speckv::update(", "speckv::SpecScheduler::execution_step(",
                "speckv::ReserveRings::admit(", "speckv::reload_span("]:
        assert sym in out, sym


def test_error_codes():
    lib = _lib.load()
    d = np.zeros(2, np.int32)
    out = np.zeros(3, np.int32)
    n, fm, b = C.c_int(), C.c_int(), C.c_int()
    # verify with an empty draft is a ContractError in the reference (specloop.cpp:26)
    assert lib.vc_drop_indices(0, 1, 1, 10, 0.01, 0, 0, None) == -1  # ConfigError
    it, w = C.c_double(), C.c_int()
    assert lib.vc_reload_span(0, 5e10, 0.037, C.byref(it), C.byref(w)) == 2  # ContractError
    assert b"reload_span" in lib.vc_last_error()
    assert lib.vc_accept(T.ptr(d, C.c_int32), T.ptr(d, C.c_int32), 2, T.ptr(out, C.c_int32),
                         C.byref(n), C.byref(fm), C.byref(b)) == 0


def test_update_window_matches_reference_semantics():
    """update(): oldest non-sink positions beyond sink+window (compressor.cpp:208-243;
    test_compressor.cpp:110-150)."""
    lib = _lib.load()
    tokens = np.array([12, 20, 5], np.int64)
    begin = np.array([0, 12, 32], np.int64)
    end = begin + tokens
    already = np.array([0, 3, 0], np.int64)
    cap = 32
    out = np.zeros((3, 2, cap), np.int64)
    nn = np.zeros(3, np.int64)
    rc = lib.vc_update_window(2, 4, 2, 3, T.ptr(tokens, C.c_int64), T.ptr(begin, C.c_int64),
                              T.ptr(end, C.c_int64), T.ptr(already, C.c_int64),
                              T.ptr(out, C.c_int64), cap, T.ptr(nn, C.c_int64))
    assert rc == 0
    assert nn.tolist() == [6, 11, 0]
    assert out[0, 0, :6].tolist() == [2, 3, 4, 5, 6, 7]
    assert out[1, 1, :11].tolist() == list(range(5, 16))
    # offsets must partition the token axis
    bad = begin.copy()
    bad[1] = 13
    assert lib.vc_update_window(2, 4, 2, 3, T.ptr(tokens, C.c_int64), T.ptr(bad, C.c_int64),
                                T.ptr(end, C.c_int64), T.ptr(already, C.c_int64),
                                T.ptr(out, C.c_int64), cap, T.ptr(nn, C.c_int64)) == 2
