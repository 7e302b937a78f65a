"""Drop-topk compressor (BASELINE.json configs[2]: score-based token dropping,
top-k retention per layer/head) against the CPU oracle, and losslessness of
drafting over the compacted tier.

Reference semantics (/root/reference/proj/src/compressor.cpp):
  * retained = llround(ratio * T), error when < 1            (:152-158)
  * every head of a layer keeps the same count (shape law)   (:83-86)
  * token-dropping and quantising compressors are exclusive  (:245-254)
The reference drops by a seeded RNG and has no score numerics:
the kept set of the score-based kernel is pinned by oracle/vc_oracle.c
(vco_key_scores + vco_topk_kept), bit-exact -- "parity unpinned by the
reference" as DESIGN.md states."""
import ctypes as C
import math

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine, _lib

N_CTX = 2000
RATIO = 0.2


def _oracle_kept(keys_bf16, k, w):
    """keys [T][d] bf16 bits -> (scores fp32, kept int32 ascending)."""
    o = T.oracle()
    Tn, d = keys_bf16.shape
    sc = np.zeros(Tn, np.float32)
    o.vco_key_scores(T.ptr(np.ascontiguousarray(keys_bf16), C.c_uint16), Tn, d, T.ptr(w, C.c_float),
                     T.ptr(sc, C.c_float))
    kept = np.zeros(k, np.int32)
    o.vco_topk_kept(T.ptr(sc, C.c_float), Tn, k, T.ptr(kept, C.c_int32))
    return sc, kept


def test_mode_exclusivity_and_ratio_are_config_errors():
    """No GPU needed: rejected before any device allocation."""
    with pytest.raises(_lib.ConfigError):
        Engine(TINY, max_ctx=256, quant_bits=4, drop_ratio=0.2)
    with pytest.raises(_lib.ConfigError):
        Engine(TINY, max_ctx=256, quant_bits=0, drop_ratio=1.5)


@pytest.mark.gpu
@pytest.mark.parametrize("Tn,k", [(3000, 1), (3000, 600), (3000, 3000), (4097, 819),
                                  (32768, 6554), (131072, 26214)])  # configs[2]: 128K, c = 0.2
def test_key_scores_and_topk_bit_exact(cuda, Tn, k):
    torch = cuda
    rng = np.random.default_rng(Tn + k)
    rows, d = 3, 64
    keys = T.f32_to_bf16(rng.standard_normal((rows, Tn, d)).astype(np.float32))
    keys[1, 100:400] = keys[1, 0]          # ties: equal scores, lower position wins
    keys[2, :] = keys[2, 7]                # a row of all-equal scores
    if Tn > 10000:                         # long rows: ties straddling the k-th score
        keys[0, Tn // 2: Tn // 2 + 5000] = keys[0, 3]
    w = rng.uniform(0.5, 1.5, d).astype(np.float32)
    lib = _lib.load()
    kd = torch.from_numpy(keys.view(np.int16)).cuda()
    wd = torch.from_numpy(w).cuda()
    sd = torch.zeros((rows, Tn), dtype=torch.float32, device="cuda")
    kept = torch.zeros((rows, k), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert lib.vc_key_scores(kd.data_ptr(), rows, Tn, d, wd.data_ptr(), sd.data_ptr(), st) == 0
    assert lib.vc_topk_select(sd.data_ptr(), rows, Tn, k, kept.data_ptr(), st) == 0
    torch.cuda.synchronize()
    for r in range(rows):
        sc, kp = _oracle_kept(keys[r], k, w)
        assert np.array_equal(sd[r].cpu().numpy().view(np.uint32), sc.view(np.uint32)), "scores differ"
        assert np.array_equal(kept[r].cpu().numpy(), kp), f"kept set differs (row {r})"
    assert lib.vc_topk_select(sd.data_ptr(), rows, Tn, Tn + 1, kept.data_ptr(), st) == _lib.VC_ERR_CONFIG


@pytest.fixture(scope="module")
def weights():
    return T.tiny_weights(TINY, seed=7, std=0.02)


@pytest.mark.gpu
@pytest.mark.parametrize("tier", [0, 1])
def test_compress_keeps_oracle_topk_per_head(cuda, weights, tier):
    e = Engine(TINY, max_slots=2, max_ctx=N_CTX + 200, max_x=16, quant_bits=0, drop_ratio=RATIO,
               full_tier=tier, n_stage=2)
    e.load_weights(weights)
    e.add_synthetic(0, N_CTX, 17, seed=3)
    meta = e.compress(0)
    k = int(math.floor(RATIO * N_CTX + 0.5))
    assert meta["retained_tokens"] == k and meta["bit_scheme"] == 16
    assert meta["payload_bytes"] == k * TINY.layers * TINY.n_kv * TINY.d_head * 4  # size law over kept tokens
    w = np.ones(TINY.d_head, np.float32)
    for layer in range(TINY.layers):
        for head in range(TINY.n_kv):
            kf, vf = e.kv_read(2 if tier else 0, 0, layer, head, 0, N_CTX)
            _, kp = _oracle_kept(kf, k, w)
            got = e.drop_kept(layer, head)
            assert got.size == k  # equal count per head (shape law)
            assert np.array_equal(got, kp)
            kd, vd = e.kv_read(3, 0, layer, head, 0, k)  # compacted rows, position order
            assert np.array_equal(kd, kf[kp]) and np.array_equal(vd, vf[kp])
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("x", [4, 8])
def test_drop_lockstep_lossless(cuda, weights, x):
    e = Engine(TINY, max_slots=4, max_ctx=N_CTX + 200, max_x=16, quant_bits=0, drop_ratio=RATIO,
               max_verify=2)
    e.load_weights(weights)
    for s, first in enumerate([17, 17, 301, 301]):
        e.add_synthetic(s, N_CTX, first, seed=1 + s // 2)
    base, _ = e.autoregress([0, 2], 40)
    e.compress(1)
    e.compress(3)
    spec, rounds, _ = e.run_speculative([1, 3], 40, x)
    np.testing.assert_array_equal(spec, base)
    for r in rounds:
        assert all(1 <= n <= x + 1 for n in r)
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("tier", [0, 1])
def test_drop_scheduled_lossless(cuda, weights, tier):
    ref = Engine(TINY, max_slots=3, max_ctx=N_CTX + 200, max_x=1, quant_bits=0)
    ref.load_weights(weights)
    for s in range(3):
        ref.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
    base, _ = ref.autoregress([0, 1, 2], 40)
    ref.close()
    e = Engine(TINY, max_slots=3, max_ctx=N_CTX + 200, max_x=16, quant_bits=0, drop_ratio=RATIO,
               full_tier=tier, n_stage=2, max_verify=2)
    e.load_weights(weights)
    for s in range(3):
        e.add_synthetic(s, N_CTX, 17 + s, seed=1 + s)
        e.compress(s)
    out, st = e.run_scheduled([0, 1, 2], 40, x=8, window=32)
    np.testing.assert_array_equal(out, base)
    assert st["verifies"] > 0
    e.close()


@pytest.mark.gpu
def test_drop_online_window_lossless_and_bounded(cuda, weights):
    """Online mode (speckv::update, compressor.cpp:208-243): tokens accepted
    after compress live in a sliding window; the tier stays bounded, holds the
    exact K/V of the latest tokens, and decoding stays lossless."""
    W, K = 32, 200
    e = Engine(TINY, max_slots=2, max_ctx=N_CTX + K + 64, max_x=8, quant_bits=0, drop_ratio=RATIO,
               drop_window=W)
    e.load_weights(weights)
    for s in range(2):
        e.add_synthetic(s, N_CTX, 17, seed=3)
    base, _ = e.autoregress([0], K)
    e.compress(1)
    spec, _, _ = e.run_speculative([1], K, 6)
    np.testing.assert_array_equal(spec, base)
    st = e.state(1)
    k = int(math.floor(RATIO * N_CTX + 0.5))
    assert st["drop_base"] == k
    n_win = st["drop_len"] - st["drop_base"]
    assert W <= n_win < 2 * W + 8  # bounded although ~K tokens were appended
    for layer in range(TINY.layers):
        for head in range(TINY.n_kv):
            kd, vd = e.kv_read(3, 1, layer, head, k, n_win)
            kf, vf = e.kv_read(0, 1, layer, head, st["committed"] - n_win, n_win)
            assert np.array_equal(kd, kf) and np.array_equal(vd, vf)
    e.close()


def test_drop_window_needs_drop_compressor():
    with pytest.raises(_lib.ConfigError):
        Engine(TINY, max_ctx=256, quant_bits=4, drop_window=16)
