"""Two-level composition (composed_accept_length,
/root/reference/proj/src/analytics.cpp:413-422) on the GPU engine.

  * A multi-row draft pass (the next draft input plus auxiliary proposals,
    causal in the compressed tail) gives each row exactly what sequential
    single-row draft passes give (batch-invariant kernels), so a confirmed
    proposal saves a pass without changing any draft token.
  * The composed loop is lossless: its output equals full-KV greedy decode.
  * depth 1 (no auxiliary rows) reproduces plain run_speculative."""
import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine

pytestmark = pytest.mark.gpu
N_CTX = 1500


@pytest.fixture(scope="module")
def weights():
    return T.tiny_weights(TINY, seed=7, std=0.02)


def _engine(weights, depth=3, bits=4, slots=4):
    e = Engine(TINY, max_slots=slots, max_ctx=N_CTX + 400, max_x=24, quant_bits=bits, max_verify=slots,
               draft_depth=depth)
    e.load_weights(weights)
    return e


@pytest.mark.parametrize("bits", [4, 2])
def test_multi_row_draft_equals_sequential(cuda, weights, bits):
    e = _engine(weights, bits=bits)
    for s in (0, 1):
        e.add_synthetic(s, N_CTX, 17, seed=3)
        e.compress(s)
    seq = []
    tok = 17
    for _ in range(3):  # three sequential single-row passes on slot 0
        tok = int(e.draft([0])[0])
        seq.append(tok)
    # one pass on slot 1 carrying [input, d1, d2] as rows (the "proposals" are right)
    out = e.step([(1, 1, [17, seq[0], seq[1]], -1)])
    assert out.tolist() == seq
    e.close()


@pytest.mark.parametrize("depth,ngram", [(1, 2), (3, 2), (4, 1)])
def test_composed_loop_lossless(cuda, weights, depth, ngram):
    e = _engine(weights, depth=max(depth, 1))
    n, K = 2, 48
    for s in range(n):
        e.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
        e.add_synthetic(n + s, N_CTX, 17 + s, seed=1 + s)
    base, _ = e.autoregress(list(range(n)), K)
    for s in range(n, 2 * n):
        e.compress(s)
    out, st = e.run_speculative_composed(list(range(n, 2 * n)), K, x=4, ngram=ngram, depth=depth)
    np.testing.assert_array_equal(out, base)
    assert st["tokens"] == n * K and st["verifies"] > 0
    if depth == 1:
        assert st["aux_proposed"] == 0
    assert st["aux_accepted"] <= st["aux_proposed"]
    print(f"MEASURED composed depth={depth} ngram={ngram}: accepted/verify {st['mean_accept']:.2f}, "
          f"drafted/round {st['drafted'] / max(st['verifies'], 1):.2f}, aux {st['aux_accepted']}/{st['aux_proposed']}")
    e.close()


def test_composed_depth1_equals_plain(cuda, weights):
    e = _engine(weights, depth=1)
    for s in range(2):
        e.add_synthetic(s, N_CTX, 17, seed=1)
        e.compress(s)
    a, _ = e.run_speculative_composed([0], 32, x=5, ngram=2, depth=1)
    b, rounds, _ = e.run_speculative([1], 32, 5)
    np.testing.assert_array_equal(a, b)
    e.close()


@pytest.mark.parametrize("tier,ring,depth", [(0, 0, 3), (1, 0, 3), (1, 3, 4)])
def test_composed_scheduled_lossless(cuda, weights, tier, ring, depth):
    """Composition inside the swap-scheduled loop (vc_run_scheduled with
    ngram/depth): proposals ride the drafting rows of the staggered loop, for
    the HBM tier, the staged host tier and the chunk-ring host tier."""
    n, K = 3, 40
    ref = Engine(TINY, max_slots=n, max_ctx=N_CTX + 200, max_x=1, quant_bits=0)
    ref.load_weights(weights)
    for s in range(n):
        ref.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
    base, _ = ref.autoregress(list(range(n)), K)
    ref.close()
    if tier == 1:
        e = Engine(TINY, max_slots=n, max_ctx=N_CTX + 400, max_x=24, quant_bits=4, full_tier=1,
                   n_stage=0 if ring else 3, ring_chunks=ring, max_verify=4, draft_depth=depth)
    else:
        e = Engine(TINY, max_slots=n, max_ctx=N_CTX + 400, max_x=24, quant_bits=4, max_verify=4, draft_depth=depth)
    e.load_weights(weights)
    for s in range(n):
        e.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
        e.compress(s)
    out, st = e.run_scheduled(list(range(n)), K, x=8, window=32, ngram=1, depth=depth)
    np.testing.assert_array_equal(out, base)
    assert st["aux_accepted"] <= st["aux_proposed"]
    assert st["drafted_tokens"] >= st["verifies"]
    print(f"MEASURED scheduled composition tier={tier} ring={ring}: accepted/verify {st['mean_accept']:.2f}, "
          f"aux {st['aux_accepted']}/{st['aux_proposed']}")
    e.close()
