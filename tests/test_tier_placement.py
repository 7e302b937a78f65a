"""Per-request tier placement (the reference's B_c knob) and the capacity-
capped full-KV baseline, on the GPU with the tiny model.

  * intra_throughput (/root/reference/proj/src/analytics.cpp:45-82): B_c of
    the B requests keep their full KV offloaded to the host tier, the other
    B_g = B - B_c keep it resident in HBM; every request drafts on its
    compressed KV.  vc_run_scheduled's n_resident = B_g.  Output must stay
    identical to full-KV greedy decode for both kinds of request.
  * baseline_full_kv (sim.cpp:418-494): FIFO admission while a full-KV slot
    is free (vc_run_decode_fifo); every request's tokens equal its own
    unbatched greedy decode, at most max_slots are resident at once, requests
    that can never fit are counted as unserved (:438-440)."""
import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine, _lib

N_CTX = 1800
K = 36


@pytest.fixture(scope="module")
def weights():
    return T.tiny_weights(TINY, seed=7, std=0.02)


def _base(weights, n, K=K, ctx=N_CTX):
    ref = Engine(TINY, max_slots=n, max_ctx=ctx + K + 64, max_x=1, quant_bits=0)
    ref.load_weights(weights)
    for s in range(n):
        ref.add_synthetic(s, ctx, 17 + s, seed=1 + s)
    base, _ = ref.autoregress(list(range(n)), K)
    ref.close()
    return base


@pytest.mark.gpu
@pytest.mark.parametrize("n,n_res,n_stage,x,x_res", [(6, 3, 4, 8, 3), (5, 5, 5, 6, 2), (4, 1, 3, 8, 0)])
def test_mixed_tier_lossless(cuda, weights, n, n_res, n_stage, x, x_res):
    base = _base(weights, n)
    e = Engine(TINY, max_slots=n, max_ctx=N_CTX + 400, max_x=16, quant_bits=4, full_tier=1, n_stage=n_stage,
               max_verify=n_stage + 2, resident_slots=n_res)
    e.load_weights(weights)
    for s in range(n):
        e.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
        e.compress(s)
    out, st = e.run_scheduled(list(range(n)), K, x=x, window=32, x_resident=x_res)
    np.testing.assert_array_equal(out, base)
    assert st["tokens"] == n * K
    assert st["resident_verifies"] > 0
    if n_res < n:
        assert st["verifies"] > st["resident_verifies"] and st["h2d_bytes"] > 0
    # residents' rounds are x_res (or x) long: accepted per verify <= that
    assert st["resident_accept"] <= (x_res or x)
    assert 0 < st["throughput"] and 0 < st["p50_latency_s"] <= st["p99_latency_s"]
    assert st["peak_hbm_bytes"] > 0
    e.close()


def test_mixed_tier_config_errors():
    """Rejected at engine creation, before any device allocation."""
    with pytest.raises(_lib.ContractError):  # 3 residents + 1 rotating slot > 3 stages
        Engine(TINY, max_slots=4, max_ctx=600, max_x=8, quant_bits=4, full_tier=1, n_stage=3, resident_slots=3)
    with pytest.raises(_lib.ContractError):
        Engine(TINY, max_slots=4, max_ctx=600, max_x=8, quant_bits=4, full_tier=1, n_stage=6, resident_slots=5)
    with pytest.raises(_lib.ContractError):  # placement is a host-tier notion
        Engine(TINY, max_slots=4, max_ctx=600, max_x=8, quant_bits=4, full_tier=0, resident_slots=2)


@pytest.mark.gpu
def test_resident_slots_have_no_host_copy(cuda, weights):
    e = Engine(TINY, max_slots=3, max_ctx=600, max_x=8, quant_bits=4, full_tier=1, n_stage=3, resident_slots=2)
    e.load_weights(weights)
    for s in range(3):
        e.add_synthetic(s, 300, 17, seed=1 + s)
        e.compress(s)
    with pytest.raises(_lib.ContractError):
        e.swap_begin(0, 2)   # a resident slot is never reloaded
    with pytest.raises(_lib.ContractError):
        e.swap_begin(2, 0)   # staging slot 0 belongs to resident slot 0
    x = e.swap_begin(2, 2)
    while not e.swap_poll(x):
        pass
    # resident slot 1's full KV sits in staging slot 1, offloaded slot 2's in the host pool
    k, _ = T.synthetic_kv(TINY.layers, TINY.n_kv, 300, TINY.d_head, seed=2)
    sk, _ = e.kv_read(1, 1, 1, 1, 0, 300)
    np.testing.assert_array_equal(sk, k[1, 1])
    k3, _ = T.synthetic_kv(TINY.layers, TINY.n_kv, 300, TINY.d_head, seed=3)
    hk, _ = e.kv_read(2, 2, 0, 1, 0, 300)
    np.testing.assert_array_equal(hk, k3[0, 1])
    e.close()


@pytest.mark.gpu
def test_fifo_baseline_capacity_capped(cuda, weights):
    n, slots = 5, 2
    base = _base(weights, n, K=12)
    e = Engine(TINY, max_slots=slots, max_ctx=N_CTX + 64, max_x=1, quant_bits=0)
    e.load_weights(weights)
    reqs = [(N_CTX, 17 + i, 1 + i, 0.0) for i in range(n)]
    reqs.append((N_CTX + 10_000, 5, 9, 0.0))  # never fits a slot
    out, m = e.run_decode_fifo(reqs, 12)
    np.testing.assert_array_equal(out[:n], base)
    assert m["completed"] == n and m["unserved"] == 1
    assert m["max_batch"] == slots and m["tokens"] == n * 12
    assert m["iterations"] == 3 * 12  # 2 + 2 + 1 requests, 12 steps each
    assert m["throughput"] > 0 and m["p50_latency_s"] <= m["p99_latency_s"]
    assert m["full_batch_throughput"] > 0
    e.close()


@pytest.mark.gpu
def test_fifo_baseline_arrivals(cuda, weights):
    """A request arriving later than the clock waits (sim.cpp:447-452)."""
    e = Engine(TINY, max_slots=2, max_ctx=N_CTX + 64, max_x=1, quant_bits=0)
    e.load_weights(weights)
    out, m = e.run_decode_fifo([(N_CTX, 17, 1, 0.0), (N_CTX, 18, 2, 1e6)], 4)
    assert m["completed"] == 2 and m["max_batch"] == 1
    base = _base(weights, 2, K=4)
    np.testing.assert_array_equal(out, base)
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("tier,resident,ring", [(0, 0, 0), (1, 1, 0), (1, 0, 0), (1, 0, 2), (1, 1, 3)])
def test_scheduled_loop_with_arrivals(cuda, weights, tier, resident, ring):
    """Requests arriving during the run take the slots finished ones free
    (simulate_staggered's arrivals, sim.cpp:227-302); every request, initial
    or arrived, emits exactly its own full-KV greedy decode."""
    n, n_arr, K = 3, 4, 24
    reqs = [(N_CTX - 100 * i, 17 + i, 1 + i) for i in range(n + n_arr)]
    ref = Engine(TINY, max_slots=n + n_arr, max_ctx=N_CTX + K + 64, max_x=1, quant_bits=0)
    ref.load_weights(weights)
    for i, (ctx, tok, seed) in enumerate(reqs):
        ref.add_synthetic(i, ctx, tok, seed=seed)
    base, _ = ref.autoregress(list(range(n + n_arr)), K)
    ref.close()
    # ring > 0: the chunk ring (packed host pool); admissions of arrivals
    # pack and store through the admission chunks while streams are in flight
    kw = (dict(full_tier=1, n_stage=resident + (0 if ring else 2), resident_slots=resident, ring_chunks=ring)
          if tier else {})
    e = Engine(TINY, max_slots=n, max_ctx=N_CTX + 400, max_x=16, quant_bits=4, max_verify=4, **kw)
    e.load_weights(weights)
    for i in range(n):
        e.add_synthetic(i, reqs[i][0], reqs[i][1], seed=reqs[i][2])
        e.compress(i)
    arrivals = [(reqs[n + j][0], reqs[n + j][1], reqs[n + j][2], 5.0 * j) for j in range(n_arr)]
    out, st = e.run_scheduled(list(range(n)), K, x=6, window=32, arrivals=arrivals)
    np.testing.assert_array_equal(out, base)
    assert st["tokens"] == (n + n_arr) * K
    assert 0 < st["p50_latency_s"] <= st["p99_latency_s"]
    e.close()


@pytest.mark.gpu
def test_host_pool_setup_is_race_free(cuda):
    """Consecutive admissions of large requests into the host tier: each
    request's synthesis reuses the scratch staging slot while the previous
    request's host-pool copy (D2H stream) may still read it -- the host pool
    must hold exactly each request's own KV (compared with the HBM tier's copy
    of the same synthetic prefixes, rows at the end of the last slices)."""
    from paper_2605_17613_b200 import ModelShape
    s = ModelShape(vocab=512, hidden=512, layers=4, n_q=32, n_kv=8, d_head=128, ffn=512)
    ctx, n = 32768, 3
    h = Engine(s, max_slots=n, max_ctx=ctx + 64, max_x=8, quant_bits=4, full_tier=1, n_stage=2)
    f = Engine(s, max_slots=n, max_ctx=ctx + 64, max_x=8, quant_bits=0)
    for i in range(n):
        h.add_synthetic(i, ctx, 17, seed=11 + i)
        h.compress(i)
        f.add_synthetic(i, ctx, 17, seed=11 + i)
    for i in range(n):
        for layer, head in [(0, 0), (s.layers - 1, s.n_kv - 1)]:
            hk, hv = h.kv_read(2, i, layer, head, ctx - 64, 64)
            fk, fv = f.kv_read(0, i, layer, head, ctx - 64, 64)
            np.testing.assert_array_equal(hk, fk)
            np.testing.assert_array_equal(hv, fv)
    h.close()
    f.close()
