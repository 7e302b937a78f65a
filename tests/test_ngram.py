"""The drafter composed with n-gram (prompt-lookup) drafts (BASELINE.json
configs[4]; Appendix C): output identical to full-KV greedy
decode whatever mix of n-gram and compressed-KV drafts a round uses, and
n-gram rounds actually occur once the output repeats."""
import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine, _lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def weights():
    return T.tiny_weights(TINY, seed=7, std=0.02)


@pytest.mark.parametrize("ngram,x", [(1, 4), (2, 8), (3, 6)])
def test_ngram_composition_lossless(cuda, weights, ngram, x):
    e = Engine(TINY, max_slots=4, max_ctx=2000 + 300, max_x=8, quant_bits=4, max_verify=2)
    e.load_weights(weights)
    for s, first in enumerate([17, 17, 301, 301]):
        e.add_synthetic(s, 2000, first, seed=1 + s // 2)
    base, _ = e.autoregress([0, 2], 120)
    e.compress(1)
    e.compress(3)
    spec, rounds, ng_rounds, _ = e.run_speculative_ngram([1, 3], 120, x, ngram=ngram)
    np.testing.assert_array_equal(spec, base)
    for r in rounds:
        assert all(1 <= n <= x + 1 for n in r)
    # greedy output of the small random-init model repeats 1- and 2-grams
    # within 120 tokens, so those lookups hit (3-grams need longer runs)
    if ngram <= 2:
        assert sum(ng_rounds) > 0
    e.close()


def test_ngram_must_be_positive(cuda, weights):
    e = Engine(TINY, max_slots=1, max_ctx=600, max_x=4, quant_bits=4)
    e.load_weights(weights)
    e.add_synthetic(0, 300, 5, seed=1)
    e.compress(0)
    with pytest.raises(_lib.ConfigError):
        e.run_speculative_ngram([0], 8, 4, ngram=0)
    e.close()
