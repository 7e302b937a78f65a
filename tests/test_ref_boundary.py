"""The drop-in claim, end to end: the UNMODIFIED reference protocol code --
speckv::run_speculative / speckv::autoregress compiled from
/root/reference/proj/src/specloop.cpp into oracle/_ref/libspeckv_ref.so
(oracle/Makefile `ref`) -- drives the B200 engine through TokenOracle
callbacks into the C-ABI (vc_draft_step / vc_verify / vc_accept_commit /
vc_decode_step).  Its output must equal the engine's own full-KV greedy
decode (losslessness, acceptance_test.cpp:55-79 C1) for the quant tier, the
host tier and the drop tier compressed by the reference's own drop-uniform
indices (vc_compress_spec).

GpuOracles mirrors include/speckv_gpu_oracle.hpp (the C++ adapter) in Python:
the reference's oracles are stateless functions of the prefix, the engine is
stateful, so each call checks the prefix against the request's committed
tokens and open draft round (SURVEY.md §8(b) "C-ABI adapters")."""
import ctypes as C

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine

CB = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_int32), C.c_int64)


def _ref():
    r = T.ref()
    if r is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    r.ref_run_speculative.restype = C.c_int
    r.ref_run_speculative.argtypes = [CB, C.c_void_p, CB, C.c_void_p, C.POINTER(C.c_int32), C.c_int64,
                                      C.c_int64, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int]
    r.ref_autoregress.restype = C.c_int
    r.ref_autoregress.argtypes = [CB, C.c_void_p, C.POINTER(C.c_int32), C.c_int64, C.c_int64,
                                  C.POINTER(C.c_int32)]
    return r


class GpuOracles:
    """Drafter / verifier TokenOracles over one engine slot."""

    def __init__(self, e: Engine, slot: int, stage: int = -1):
        self.e, self.slot, self.stage = e, slot, stage
        self.base = -1
        self.emitted, self.drafts, self.preds = [], [], []
        self.rounds = []
        self.error = None
        self.calls = {"draft": 0, "verify_pass": 0, "decode": 0}
        self.draft_cb = CB(self._wrap(self._draft))
        self.verify_cb = CB(self._wrap(self._verify))

    def _wrap(self, fn):
        def cb(_ctx, p, n):
            if self.error is not None:
                return 0
            try:
                return fn([p[i] for i in range(n)])
            except Exception as ex:  # surfaced by the test after the reference loop returns
                self.error = ex
                return 0
        return cb

    def _bind(self, p):
        if self.base < 0:
            assert p and p[-1] == self.e.state(self.slot)["pending"], "prompt tail is not the pending token"
            self.base = len(p)

    def _is(self, p, k):
        if len(p) != self.base + len(self.emitted) + k:
            return False
        return p[self.base:] == self.emitted + self.drafts[:k]

    def _draft(self, p):
        self._bind(p)
        assert self._is(p, len(self.drafts)), "drafter prefix is not the request's state"
        t = int(self.e.draft([self.slot])[0])
        self.drafts.append(t)
        self.calls["draft"] += 1
        return t

    def _verify(self, p):
        self._bind(p)
        if not self.drafts:  # autoregress: one full-KV decode step
            assert self._is(p, 0)
            t = int(self.e.decode_step([self.slot])[0])
            self.emitted.append(t)
            self.calls["decode"] += 1
            return t
        k = len(p) - (self.base + len(self.emitted))
        assert 0 <= k <= len(self.drafts) and self._is(p, k), "verifier prefix outside the open round"
        if not self.preds:
            assert k == 0, "verify must start at k = 0 (specloop.cpp:30-33)"
            if self.stage >= 0:
                x = self.e.swap_begin(self.slot, self.stage)
                while not self.e.swap_poll(x):
                    pass
            self.preds = [int(t) for t in self.e.verify([self.slot], [self.stage] if self.stage >= 0 else None)]
            self.calls["verify_pass"] += 1
        t = self.preds[k]
        if k == len(self.drafts):  # last prediction of the round: commit it
            out = self.e.accept_commit(self.slot, self.preds, self.stage)
            self.emitted += out
            self.rounds.append(len(out))
            self.drafts, self.preds = [], []
        return t


def _engines(bits=4, tier=0, drop=0.0, n_ctx=1500, K=40, x=8):
    w = T.tiny_weights(TINY, seed=7, std=0.02)
    full = Engine(TINY, max_slots=1, max_ctx=n_ctx + K + 64, max_x=1, quant_bits=0)
    spec = Engine(TINY, max_slots=1, max_ctx=n_ctx + K + 64, max_x=x, quant_bits=bits, full_tier=tier,
                  n_stage=1, drop_ratio=drop)
    for e in (full, spec):
        e.load_weights(w)
        e.add_synthetic(0, n_ctx, 17, seed=1)
    return full, spec


@pytest.mark.gpu
@pytest.mark.parametrize("x,bits,tier,drop", [(1, 4, 0, 0.0), (5, 4, 0, 0.0), (8, 2, 0, 0.0), (6, 4, 1, 0.0),
                                              (4, 0, 0, 0.3)])
def test_reference_run_speculative_drives_engine(cuda, x, bits, tier, drop):
    r = _ref()
    K = 40
    full, spec = _engines(bits, tier, drop, K=K, x=x)
    if drop:
        # the reference's own drop-uniform indices (seed 5) pick the kept set
        meta = spec.compress_spec(0, "drop-uniform", ratio=drop, seed=5)
        dropped = np.zeros((1,), np.int64)
        n_drop = r.ref_compress(0, TINY.layers, TINY.n_kv, 1500, 4 * TINY.d_head, drop, 4, 5, 0, None,
                                T.ptr(dropped, C.c_int64), C.byref(C.c_int()))
        assert meta["retained_tokens"] == 1500 - n_drop
    else:
        spec.compress(0)
    prompt = np.array([17], np.int32)
    # reference autoregress over the full-KV engine
    fo = GpuOracles(full, 0)
    base = np.zeros(K, np.int32)
    assert r.ref_autoregress(fo.verify_cb, None, T.ptr(prompt, C.c_int32), 1, K, T.ptr(base, C.c_int32)) == 0, \
        r.ref_last_error()
    assert fo.error is None, fo.error
    assert fo.calls["decode"] == K
    # reference run_speculative over the compressed-KV drafter + full-KV verifier
    so = GpuOracles(spec, 0, stage=0 if tier else -1)
    out = np.zeros(K + x + 1, np.int32)
    rounds = np.zeros(4096, np.int32)
    nr = r.ref_run_speculative(so.draft_cb, None, so.verify_cb, None, T.ptr(prompt, C.c_int32), 1, K, x,
                               T.ptr(out, C.c_int32), T.ptr(rounds, C.c_int32), rounds.size)
    assert nr > 0, r.ref_last_error()
    assert so.error is None, so.error
    assert out[:K].tolist() == base.tolist(), "reference loop over the GPU engine is not lossless"
    # one verify pass per round, x drafts per round; the reference's accept
    # counts equal the engine's committed rounds
    assert so.calls["verify_pass"] == nr and so.calls["draft"] == nr * x
    assert rounds[:nr].tolist() == so.rounds  # accepted.size() per round (specloop.cpp:71)
    # the engine's committed history is the reference's output (the adapter
    # commits the last round inside run_speculative; advisor finding r1)
    assert spec.history(0)[:K] == base.tolist()
    full.close()
    spec.close()


@pytest.mark.gpu
def test_compress_spec_reference_drop_indices(cuda):
    """vc_compress_spec(drop-uniform / drop-window) keeps exactly the
    complement of the reference's dropped indices, per (layer, head)."""
    r = _ref()
    n_ctx = 3000
    e = Engine(TINY, max_slots=1, max_ctx=n_ctx + 64, max_x=4, quant_bits=0, drop_ratio=0.4)
    e.add_synthetic(0, n_ctx, 17, seed=1)
    for kind, kid, ratio, seed, sink in [("drop-uniform", 0, 0.25, 9, 0), ("drop-window", 1, 0.4, 0, 4)]:
        meta = e.compress_spec(0, kind, ratio=ratio, seed=seed, sink_tokens=sink)
        retained = int(np.floor(ratio * n_ctx + 0.5))
        drop = n_ctx - retained
        out = np.zeros((TINY.layers, TINY.n_kv, drop), np.int64)
        pb, bs = C.c_int64(), C.c_int()
        assert r.ref_compress(kid, TINY.layers, TINY.n_kv, n_ctx, 4 * TINY.d_head, ratio, 4, seed, sink,
                              T.ptr(out, C.c_int64), C.byref(pb), C.byref(bs)) == drop
        assert meta["retained_tokens"] == retained and meta["payload_bytes"] == pb.value
        for l in range(TINY.layers):
            for h in range(TINY.n_kv):
                kept = e.drop_kept(l, h)
                assert np.array_equal(np.setdiff1d(np.arange(n_ctx), out[l, h]), kept), (kind, l, h)
                # the drop tier holds exactly those rows of the full KV
                kk, _ = e.kv_read(3, 0, l, h, 0, 5)
                fk, _ = e.kv_read(0, 0, l, h, int(kept[0]), 1)
                np.testing.assert_array_equal(kk[0], fk[0])
    e.close()


@pytest.mark.gpu
def test_compress_spec_rejects_mismatched_tier(cuda):
    from paper_2605_17613_b200 import _lib
    e = Engine(TINY, max_slots=1, max_ctx=512, max_x=4, quant_bits=4)
    e.add_synthetic(0, 300, 17, seed=1)
    with pytest.raises(_lib.ContractError):
        e.compress_spec(0, "quant-uniform", bits=2)
    with pytest.raises(_lib.ContractError):
        e.compress_spec(0, "drop-uniform", ratio=0.5)
    assert e.compress_spec(0, "quant-uniform", bits=4)["bit_scheme"] == 4
    e.close()
