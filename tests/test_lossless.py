"""The losslessness invariant on the GPU: VeriCache output tokens are
IDENTICAL to the same engine's full-KV greedy decode (bit-exact logits via
batch-invariant kernels), for lock-step rounds and for the swap-scheduled
staggered loop, with the full KV resident (tier 0) or streamed from the
pinned host pool (tier 1).  Mirrors the reference's property tests
(proj/tests/test_specloop.cpp:117-149, acceptance_test.cpp:55-79) with the
model as both oracles."""
import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine

pytestmark = pytest.mark.gpu

N_CTX = 2000
K = 40


@pytest.fixture(scope="module")
def weights():
    return T.tiny_weights(TINY, seed=7, std=0.02)


def _engine(weights, **kw):
    e = Engine(TINY, max_ctx=N_CTX + 400, max_x=16, **kw)
    e.load_weights(weights)
    return e


@pytest.mark.parametrize("x", [1, 4, 8, 16])
@pytest.mark.parametrize("bits", [4, 2])
def test_lockstep_matches_full_kv_decode(cuda, weights, x, bits):
    e = _engine(weights, max_slots=4, quant_bits=bits, max_verify=2)
    for s, first in enumerate([17, 17, 301, 301]):
        e.add_synthetic(s, N_CTX, first, seed=1 + (s // 2))
    base, _ = e.autoregress([0, 2], K)
    e.compress(1)
    e.compress(3)
    spec, rounds, _ = e.run_speculative([1, 3], K, x)
    np.testing.assert_array_equal(spec, base)
    for r in rounds:  # every round emits 1..x+1 tokens (specloop.cpp:37-56)
        assert all(1 <= n <= x + 1 for n in r)
    e.close()


def test_scheduled_tier0_matches_full_kv_decode(cuda, weights):
    e = _engine(weights, max_slots=8, quant_bits=4, max_verify=4)
    n = 4
    for s in range(n):
        e.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
        e.add_synthetic(n + s, N_CTX, 17 + s, seed=1 + s)
    base, _ = e.autoregress(list(range(n)), K)
    for s in range(n, 2 * n):
        e.compress(s)
    out, st = e.run_scheduled(list(range(n, 2 * n)), K, x=6, window=16)
    np.testing.assert_array_equal(out, base)
    assert st["verifies"] > 0 and st["tokens"] == n * K
    e.close()


def test_scheduled_tier1_host_pool_matches(cuda, weights):
    """Full KV in pinned host memory, streamed per verify into staging slots."""
    ref = _engine(weights, max_slots=3, quant_bits=0)
    for s in range(3):
        ref.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
    base, _ = ref.autoregress([0, 1, 2], K)
    ref.close()
    e = _engine(weights, max_slots=3, quant_bits=4, full_tier=1, n_stage=2, max_verify=2)
    for s in range(3):
        e.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
        e.compress(s)
    out, st = e.run_scheduled([0, 1, 2], K, x=8, window=32, link_bandwidth=0.0)
    np.testing.assert_array_equal(out, base)
    assert st["h2d_bytes"] > 0
    e.close()


def test_manual_round_protocol(cuda, weights):
    """draft x -> verify -> accept_commit, the reference loop by hand."""
    e = _engine(weights, max_slots=2, quant_bits=4)
    e.add_synthetic(0, N_CTX, 5, seed=3)
    e.add_synthetic(1, N_CTX, 5, seed=3)
    base, _ = e.autoregress([0], 12)
    e.compress(1)
    out = []
    while len(out) < 12:
        for _ in range(3):
            e.draft([1])
        st = e.state(1)
        assert st["draft_len"] == 3
        preds = e.verify([1])
        assert preds.size == 4
        out += e.accept_commit(1, preds)
        assert e.state(1)["draft_len"] == 0
    assert out[:12] == base[0].tolist()
