"""Config 1 (BASELINE.json configs[0]): tiny Llama-style model, 4K context,
int4 compressor, x=8, batch 1.  The GPU forward matches the CPU oracle's
logits within the stated bound, and greedy tokens match the oracle except at
documented near-tie positions.

Logit tolerance: both sides round activations to
bf16 at the same points; accumulation order differs (fp32 tensor-core tiles
vs fp64), which flips occasional bf16 roundings:
    max|logit - logit_ref| <= 3e-2 * max|logit_ref| + 1e-3.
Near tie: the oracle's top-2 gap at that position is below 2x that bound;
after a near-tie flip the two greedy continuations legitimately diverge."""
import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine

pytestmark = pytest.mark.gpu

N_CTX = 4096
REL, ABS = 3e-2, 1e-3


def _bound(ref):
    return REL * np.abs(ref).max() + ABS


def _report(name, got, want):
    err = float(np.abs(got - want).max())
    print(f"MEASURED {name}: max_abs {err:.3e} rel {err / float(np.abs(want).max()):.3e} bound {_bound(want):.3e}")
    return err


@pytest.fixture(scope="module")
def setup(cuda):
    w = T.tiny_weights(TINY, seed=7, std=0.02)
    k, v = T.synthetic_kv(TINY.layers, TINY.n_kv, N_CTX, TINY.d_head, seed=1)
    e = Engine(TINY, max_slots=4, max_ctx=N_CTX + 256, max_x=16, quant_bits=4)
    e.load_weights(w)
    om = T.OracleModel(TINY, w, cap=N_CTX + 256)
    yield e, om, w, k, v
    e.close()


def _oracle_state(om, k, v):
    return om.new_kv(T.bf16_to_f32(k), T.bf16_to_f32(v))


def test_decode_logits(setup):
    e, om, w, k, v = setup
    e.add_kv(0, k, v, first_token=17)
    st = _oracle_state(om, k, v)
    want = om.forward(st, [17])
    got_tok, got = e.step([(0, 0, [17], -1)], want_logits=True)
    err = _report("tiny decode logits vs oracle", got, want)
    assert err <= _bound(want), (err, _bound(want))
    assert got_tok[0] == np.argmax(got[0])


def test_verify_window_logits(setup):
    """Verify pass (x+1 rows, causal inside the window) vs the oracle."""
    e, om, w, k, v = setup
    e.add_kv(1, k, v, first_token=17)
    st = _oracle_state(om, k, v)
    toks = [17, 3, 99, 1024, 5, 6, 7, 8, 9]
    want = om.forward(st, toks)
    _, got = e.step([(1, 2, toks, -1)], want_logits=True)
    assert _report("tiny verify logits vs oracle", got, want) <= _bound(want)


def test_draft_logits(setup):
    """Draft pass over the compressed cache vs the oracle on the dequantised cache."""
    e, om, w, k, v = setup
    e.add_kv(2, k, v, first_token=17)
    e.compress(2)
    G = 128
    kq = np.zeros((TINY.layers, TINY.n_kv, N_CTX, TINY.d_head), np.float32)
    vq = np.zeros_like(kq)
    for l in range(TINY.layers):
        for h in range(TINY.n_kv):
            ck, sk, zk = T.quant_oracle(k[l, h], G, 4, "rows")
            cv, sv, zv = T.quant_oracle(v[l, h], TINY.d_head, 4, "cols")
            kq[l, h] = ck * np.repeat(T.f16_bits_to_f32(sk), G, 0) + np.repeat(T.f16_bits_to_f32(zk), G, 0)
            vq[l, h] = cv * T.f16_bits_to_f32(sv) + T.f16_bits_to_f32(zv)
    st = om.new_kv(kq, vq)
    want = om.forward(st, [17])
    _, got = e.step([(2, 1, [17], -1)], want_logits=True)
    assert _report("tiny draft logits vs oracle", got, want) <= _bound(want)


def test_greedy_tokens_vs_oracle(setup):
    e, om, w, k, v = setup
    K = 24
    e.add_kv(3, k, v, first_token=17)
    got, _ = e.autoregress([3], K)
    st = _oracle_state(om, k, v)
    tok = 17
    for i in range(K):
        lg = om.forward(st, [tok])[0]
        want = int(np.argmax(lg))
        if got[0, i] != want:
            top2 = np.sort(lg)[-2:]
            assert top2[1] - top2[0] < 2 * _bound(lg), f"non-tie mismatch at {i}"
            break  # documented near-tie: continuations legitimately diverge
        tok = want
