"""Head-sharded tensor parallelism (BASELINE.json configs[4]).

CPU: the weight sharding covers the full model exactly.
GPU (one device, two in-process ranks over the loopback collective, one host
thread each): the TP=2 forward matches the unsharded model within the logit
tolerance, both ranks compute bit-identical logits, and speculative decoding
over the sharded compressed tiers is lossless against the sharded full-KV
decode (the all-gather + rank-order sum keeps the combine batch-invariant).
The NCCL path (one process per GPU, vc_engine_attach_nccl) runs the same
engine code; with one GPU it is exercised as a one-rank NCCL group (all-gather
captured in the CUDA graph), which must be bit-identical to the fused
residual epilogue.  A multi-GPU TP run needs >= 2 GPUs."""
import threading

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine, TpLoopback, tp_shard

N_CTX = 1500
TP = 2


@pytest.fixture(scope="module")
def weights():
    return T.tiny_weights(TINY, seed=9, std=0.02)


def test_tp_shard_partitions_the_model(weights):
    d, nq, nkv, F = TINY.d_head, TINY.n_q, TINY.n_kv, TINY.ffn
    shards = [tp_shard(weights, TINY, TP, r) for r in range(TP)]
    for layer in range(TINY.layers):
        full = np.asarray(weights["wqkv"][layer]).reshape((nq + 2 * nkv) * d, -1)
        ql, kl = nq // TP * d, nkv // TP * d
        q = np.concatenate([s["wqkv"][layer][:ql] for s in shards])
        k = np.concatenate([s["wqkv"][layer][ql:ql + kl] for s in shards])
        v = np.concatenate([s["wqkv"][layer][ql + kl:] for s in shards])
        assert np.array_equal(np.concatenate([q, k, v]), full)
        assert np.array_equal(np.concatenate([s["wo"][layer] for s in shards], axis=1),
                              np.asarray(weights["wo"][layer]).reshape(TINY.hidden, nq * d))
        assert np.array_equal(np.concatenate([s["wgate"][layer] for s in shards]),
                              np.asarray(weights["wgate"][layer]).reshape(F, -1))
        assert np.array_equal(np.concatenate([s["wdown"][layer] for s in shards], axis=1),
                              np.asarray(weights["wdown"][layer]).reshape(TINY.hidden, F))


def _ranks(weights, kv, **kw):
    group = TpLoopback(TP)
    engines = []
    for r in range(TP):
        e = Engine(TINY, max_slots=2, max_ctx=N_CTX + 200, max_x=8, max_verify=2, tp_size=TP, tp_rank=r, **kw)
        e.attach_loopback(group)
        e.load_weights(weights)
        lo, hi = r * TINY.n_kv // TP, (r + 1) * TINY.n_kv // TP
        for s in range(2):
            e.add_kv(s, kv[0][:, lo:hi], kv[1][:, lo:hi], first_token=17)
        engines.append(e)
    return group, engines


def _parallel(fn, engines):
    out = [None] * len(engines)
    err = []

    def run(i):
        try:
            out[i] = fn(engines[i])
        except Exception as ex:  # surface in the main thread
            err.append(ex)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(engines))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not err, err
    return out


@pytest.mark.gpu
def test_tp2_forward_matches_unsharded(cuda, weights):
    kv = T.synthetic_kv(TINY.layers, TINY.n_kv, N_CTX, TINY.d_head, seed=4)
    full = Engine(TINY, max_slots=1, max_ctx=N_CTX + 200, max_x=8, quant_bits=0)
    full.load_weights(weights)
    full.add_kv(0, kv[0], kv[1], first_token=17)
    _, ref = full.step([(0, 0, [17], -1)], want_logits=True)
    full.close()
    group, ranks = _ranks(weights, kv, quant_bits=0)
    res = _parallel(lambda e: e.step([(0, 0, [17], -1)], want_logits=True)[1], ranks)
    assert np.array_equal(res[0].view(np.uint32), res[1].view(np.uint32)), "ranks disagree"
    err = np.abs(res[0] - ref).max()
    assert err <= 3e-2 * np.abs(ref).max() + 1e-3, err
    for e in ranks:
        e.close()
    group.close()


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [4, 2])
def test_tp2_speculative_lossless(cuda, weights, bits):
    kv = T.synthetic_kv(TINY.layers, TINY.n_kv, N_CTX, TINY.d_head, seed=6)
    group, ranks = _ranks(weights, kv, quant_bits=bits)

    def run(e):
        base, _ = e.autoregress([0], 24)
        e.compress(1)
        spec, rounds, _ = e.run_speculative([1], 24, 4)
        return base, spec

    (b0, s0), (b1, s1) = _parallel(run, ranks)
    assert np.array_equal(b0, b1) and np.array_equal(s0, s1), "ranks disagree"
    np.testing.assert_array_equal(s0, b0)
    for e in ranks:
        e.close()
    group.close()


@pytest.mark.gpu
def test_nccl_one_rank_collective_bit_identical(cuda, weights):
    """The NCCL collective path on real hardware: a one-rank NCCL group runs
    the TP residual path (all-gather inside the CUDA graph + rank-order sum),
    which must be bit-identical to the fused residual epilogue, and lossless."""
    from paper_2605_17613_b200 import _lib, nccl_unique_id
    try:
        uid = nccl_unique_id()
    except _lib.VcError:
        pytest.skip("libnccl.so.2 not available")
    kv = T.synthetic_kv(TINY.layers, TINY.n_kv, N_CTX, TINY.d_head, seed=8)
    outs = []
    for with_nccl in (False, True):
        e = Engine(TINY, max_slots=2, max_ctx=N_CTX + 200, max_x=8, max_verify=2, quant_bits=4)
        if with_nccl:
            e.attach_nccl(uid)
        e.load_weights(weights)
        for s in range(2):
            e.add_kv(s, kv[0], kv[1], first_token=17)
        _, logits = e.step([(0, 0, [17], -1)], want_logits=True)
        base, _ = e.autoregress([0], 16)
        e.compress(1)
        spec, _, _ = e.run_speculative([1], 16, 4)
        outs.append((logits, base, spec))
        e.close()
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[1][2], outs[1][1])
