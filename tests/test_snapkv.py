"""SnapKV token scores for the drop-topk compressor (BASELINE.json configs[2];
PAPER.md:590, :645 name SnapKV among the paper's droppers), on the GPU.

The reference drops by a seeded RNG (compressor.cpp:114-171) and has no
attention scores, so the score itself is pinned by a float64 numpy
restatement of SnapKV (Li et al., 2024) over the engine's own observation
query and keys:
  score[t] = max_{|j-t| <= pool/2} sum_{r in group} softmax_j(q_r . k_j / sqrt(d)),
  the last `recent` positions always kept;
then the kept set must be exactly the oracle's top-k of the GPU scores
(oracle/vc_oracle.c vco_topk_kept, ties -> lower position), and drafting over
the SnapKV-compacted tier must stay lossless."""
import ctypes as C

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine, _lib

N_CTX = 1800
RATIO = 0.25


@pytest.fixture(scope="module")
def weights():
    return T.tiny_weights(TINY, seed=7, std=0.02)


def _snap_ref(q_bf16, k_bf16, n_rep, pool, recent):
    """float64 SnapKV scores of one kv head: q [n_rep][d], k [T][d] (bf16 bits)."""
    q = T.bf16_to_f32(q_bf16).astype(np.float64)
    k = T.bf16_to_f32(k_bf16).astype(np.float64)
    logits = q @ k.T / np.sqrt(k.shape[1])
    p = np.exp(logits - logits.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    a = p.sum(axis=0)
    Tn = a.size
    pad = np.concatenate([np.full(pool // 2, -np.inf), a, np.full(pool // 2, -np.inf)])
    pooled = np.max(np.stack([pad[i:i + Tn] for i in range(pool)]), axis=0)
    pooled[Tn - recent:] = np.inf
    return pooled


@pytest.mark.gpu
@pytest.mark.parametrize("pool,recent", [(7, 32), (1, 0)])
def test_snapkv_scores_and_kept_sets(cuda, weights, pool, recent):
    e = Engine(TINY, max_slots=1, max_ctx=N_CTX + 200, max_x=16, quant_bits=0, drop_ratio=RATIO,
               drop_score="snapkv", snap_pool=pool, snap_recent=recent)
    e.load_weights(weights)
    e.add_synthetic(0, N_CTX, 17, seed=3)
    st0 = e.state(0)
    e.compress(0)
    st1 = e.state(0)
    assert st1["committed"] == st0["committed"] and st1["pending"] == st0["pending"]  # nothing committed
    k = int(np.floor(RATIO * N_CTX + 0.5))
    R = TINY.n_q // TINY.n_kv
    o = T.oracle()
    for layer in range(TINY.layers):
        q = e.obs_query(layer)
        for head in range(TINY.n_kv):
            kf, vf = e.kv_read(0, 0, layer, head, 0, N_CTX)
            got = e.drop_scores(layer, head, N_CTX)
            ref = _snap_ref(q[head * R:(head + 1) * R], kf, R, pool, recent)
            fin = np.isfinite(ref)
            assert np.array_equal(np.isinf(got), ~fin)
            scale = ref[fin].max()
            assert np.abs(got[fin] - ref[fin]).max() <= 2e-5 * scale + 1e-9, "SnapKV scores differ from float64"
            kp = np.zeros(k, np.int32)
            o.vco_topk_kept(T.ptr(np.ascontiguousarray(got), C.c_float), N_CTX, k, T.ptr(kp, C.c_int32))
            kept = e.drop_kept(layer, head)
            assert np.array_equal(kept, kp), "kept set is not the top-k of the scores"
            assert np.all(np.isin(np.arange(N_CTX - recent, N_CTX), kept))  # the recent window is kept
            kd, vd = e.kv_read(3, 0, layer, head, 0, k)
            assert np.array_equal(kd, kf[kp]) and np.array_equal(vd, vf[kp])
    e.close()


@pytest.mark.gpu
def test_snapkv_observation_query_is_the_pending_tokens(cuda, weights):
    """The observation query equals the q the first real decode step computes."""
    e = Engine(TINY, max_slots=1, max_ctx=N_CTX + 200, max_x=16, quant_bits=0, drop_ratio=RATIO,
               drop_score="snapkv")
    e.load_weights(weights)
    e.add_synthetic(0, N_CTX, 17, seed=3)
    e.compress(0)
    q0 = [e.obs_query(l).copy() for l in range(TINY.layers)]
    e.compress(0)  # a second compress recomputes the same observation (deterministic forward)
    for l in range(TINY.layers):
        np.testing.assert_array_equal(e.obs_query(l), q0[l])
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("x", [4, 12])
def test_snapkv_drafting_lossless(cuda, weights, x):
    e = Engine(TINY, max_slots=4, max_ctx=N_CTX + 200, max_x=16, quant_bits=0, drop_ratio=RATIO,
               drop_score="snapkv", max_verify=2)
    e.load_weights(weights)
    for s, first in enumerate([17, 17, 301, 301]):
        e.add_synthetic(s, N_CTX, first, seed=1 + s // 2)
    base, _ = e.autoregress([0, 2], 40)
    e.compress(1)
    e.compress(3)
    spec, rounds, _ = e.run_speculative([1, 3], 40, x)
    np.testing.assert_array_equal(spec, base)
    e.close()


def test_snapkv_config_errors():
    with pytest.raises(_lib.ContractError):  # needs the HBM full tier
        Engine(TINY, max_ctx=600, quant_bits=0, drop_ratio=0.2, drop_score="snapkv", full_tier=1, n_stage=2)
    with pytest.raises(ValueError):
        Engine(TINY, max_ctx=600, quant_bits=0, drop_ratio=0.2, drop_score="attention")
