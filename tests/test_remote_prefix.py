"""Remote prefix caching (BASELINE.json configs[3]).

The reference simulates the pipeline (remote_prefix,
/root/reference/proj/src/sim.cpp:510-665): a request's compressed payload
arrives first and drafting starts on it, the full KV is prefetched in
parallel, each cycle verifies once both are resident, and force_baseline
loads the full KV and decodes.  Here the payloads are real (a stored prefix
in pinned host memory streamed over the copy engine) and the checks are the
path's invariants:
  * the emitted tokens equal the full-KV baseline arm and plain greedy decode
    over the same prefix (losslessness, per request, different prompt tails);
  * every request's compressed payload lands before its full KV (the link
    order), and the stats account for every token and transfer;
  * arrivals spread in time change nothing in the tokens."""
import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine, _lib

N_CTX = 2000
K = 40
FIRST = [17, 301, 999, 5]


@pytest.fixture(scope="module")
def weights():
    return T.tiny_weights(TINY, seed=7, std=0.02)


def _engine(weights, bits, **kw):
    e = Engine(TINY, max_slots=len(FIRST) + 1, max_ctx=N_CTX + K + 64, max_x=16, quant_bits=bits,
               max_verify=2, **kw)
    e.load_weights(weights)
    return e


def _greedy(weights):
    e = _engine(weights, 4)
    for s, f in enumerate(FIRST):
        e.add_synthetic(s, N_CTX, f, seed=3)
    out, _ = e.autoregress(list(range(len(FIRST))), K)
    e.close()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [4, 2])
def test_remote_prefix_lossless_vs_baseline_and_greedy(cuda, weights, bits):
    ref = _greedy(weights)
    e = _engine(weights, bits)
    e.add_synthetic(0, N_CTX, 0, seed=3)       # the storage node's prefix
    e.compress(0)
    e.prefix_store(0)
    slots = list(range(1, len(FIRST) + 1))
    base, sb = e.run_remote_prefix(slots, K, 0, FIRST, baseline=True)
    spec, ss = e.run_remote_prefix(slots, K, 6, FIRST)
    np.testing.assert_array_equal(base, ref)
    np.testing.assert_array_equal(spec, ref)
    n = len(FIRST)
    assert sb["tokens"] == ss["tokens"] == n * K
    assert sb["verifies"] == 0 and ss["verifies"] > 0
    assert 0 <= ss["mean_accept"] <= 6
    # VeriCache moves the compressed payload and the full KV; the baseline only the full KV
    full_b = 2 * TINY.layers * TINY.n_kv * N_CTX * TINY.d_head * 2
    assert sb["h2d_bytes"] == pytest.approx(n * full_b)
    assert ss["h2d_bytes"] > n * full_b
    assert 0 < ss["compressed_ready_ms_mean"] <= ss["full_ready_ms_mean"]
    assert ss["makespan_ms"] > 0 and ss["ttft_ms_max"] >= ss["ttft_ms_mean"] > 0
    # the loop releases and reloads its slots: a second run is identical
    spec2, s2 = e.run_remote_prefix(slots, K, 4, FIRST, link_queue=1, payload_order=1)
    np.testing.assert_array_equal(spec2, ref)
    # every compressed payload first: all requests can draft before any full KV lands
    assert s2["compressed_ready_ms_mean"] <= ss["compressed_ready_ms_mean"] + 50.0
    e.close()


@pytest.mark.gpu
def test_remote_prefix_staggered_arrivals(cuda, weights):
    ref = _greedy(weights)
    e = _engine(weights, 4)
    e.add_synthetic(0, N_CTX, 0, seed=3)
    e.compress(0)
    e.prefix_store(0)
    slots = list(range(1, len(FIRST) + 1))
    spec, st = e.run_remote_prefix(slots, K, 8, FIRST, arrival_gap_ms=20.0)
    np.testing.assert_array_equal(spec, ref)
    assert st["wall_ms"] >= 20.0 * (len(FIRST) - 1)
    e.close()


@pytest.mark.gpu
def test_remote_prefix_contract_and_config_errors(cuda, weights):
    e = _engine(weights, 4)
    with pytest.raises(_lib.ContractError):      # nothing stored yet
        e.run_remote_prefix([1], K, 4, [17])
    e.add_synthetic(0, N_CTX, 0, seed=3)
    with pytest.raises(_lib.ContractError):      # not compressed
        e.prefix_store(0)
    e.compress(0)
    e.prefix_store(0)
    with pytest.raises(_lib.ConfigError):
        e.run_remote_prefix([1], K, 17, [17])     # x > max_x
    with pytest.raises(_lib.ConfigError):
        e.run_remote_prefix([1], 10 ** 6, 4, [17])  # beyond max_ctx
    e.add_synthetic(2, 100, 17, seed=3)
    with pytest.raises(_lib.ContractError):      # slot holds another request
        e.prefix_load(2, 0, 17)
    e.release(2)
    assert e.prefix_load(2, 0, 17) > 0
    e.close()
    f = Engine(TINY, max_slots=2, max_ctx=N_CTX + 200, max_x=8, quant_bits=0)
    f.load_weights(weights)
    f.add_synthetic(0, N_CTX, 0, seed=3)
    with pytest.raises(_lib.ConfigError):        # needs the quantising compressor
        f.prefix_store(0)
    f.close()
