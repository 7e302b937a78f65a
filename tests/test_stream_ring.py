"""Layer-chunked host tier (ring_chunks > 0), on the GPU.

The reference books a verify reload as bytes over S_r lookahead windows
(/root/reference/proj/src/scheduler.cpp:15-23, :96-163) and charges the
verify the request's full-KV bytes (:366).  The B200 engine streams that
reload one layer per chunk into a ring of a few one-layer chunks and runs the
verify forward range by range as layers land (Engine::stream_*), so staging
HBM is a few layers instead of whole requests.  Batch invariance makes the
range-by-range verify bit-identical to the whole-window verify:
  * predictions and emitted tokens equal the staged (whole-request) verify
    round after round, with the ring smaller than the model's layer count
    (chunks recycled inside one verify) and two streams in flight;
  * the swap-scheduled loop over the ring emits exactly full-KV greedy decode;
  * an aborted stream gives its chunks back;
  * over the drop-topk tier the host pool keeps only the dropped rows and a
    reload moves (1 - c) of the prefix (analytics.cpp:77-78), the rest
    rebuilt from the drop tier."""
import ctypes as C
import dataclasses
import time

import numpy as np
import pytest

import vc_testlib as T
from paper_2605_17613_b200 import TINY, Engine, _lib

TINY6 = dataclasses.replace(TINY, layers=6)
CTX = (1000, 1300)


@pytest.fixture(scope="module")
def w6():
    return T.tiny_weights(TINY6, seed=11, std=0.02)


def _engine(w, ring, **kw):
    if ring:
        e = Engine(TINY6, max_slots=kw.get("slots", 2), max_ctx=2000, max_x=8, quant_bits=4, full_tier=1,
                   n_stage=0, ring_chunks=ring, max_streams=2, max_verify=4, host_pack=kw.get("pack", True))
    else:
        e = Engine(TINY6, max_slots=kw.get("slots", 2), max_ctx=2000, max_x=8, quant_bits=4, full_tier=1,
                   n_stage=3, max_verify=4)
    e.load_weights(w)
    return e


def _until(fn, timeout=30.0):
    t0 = time.time()
    while True:
        r = fn()
        if r is not None:
            return r
        assert time.time() - t0 < timeout, "streamed verify did not finish"


@pytest.mark.gpu
# pack: True (every block packed), False (raw pool), 6 (at most 5 packed
# blocks: the rest of each request, and every row accepted later, raw)
@pytest.mark.parametrize("ring,pack", [(2, True), (3, False), (8, True), (3, 6)])
def test_streamed_verify_equals_staged_verify(cuda, w6, ring, pack):
    a, b = _engine(w6, 0), _engine(w6, ring, pack=pack)
    for e in (a, b):
        for s, n in enumerate(CTX):
            e.add_synthetic(s, n, 17 + s, seed=1 + s)
            e.compress(s)
    x = 5
    for rnd in range(5):
        for _ in range(x):
            da, db = a.draft([0, 1]), b.draft([0, 1])
            np.testing.assert_array_equal(da, db)
        # staged arm: whole-request reloads into two staging slots
        xs = [a.swap_begin(s, s + 1) for s in (0, 1)]
        for xf in xs:
            _until(lambda: True if a.swap_poll(xf) else None)
        pa = a.verify([0, 1], [1, 2])
        # ring arm: both streams in flight, advanced alternately
        sids = [b.stream_begin(s) for s in (0, 1)]
        got = [None, None]

        def step():
            for i, sid in enumerate(sids):
                if got[i] is None:
                    got[i] = b.stream_advance(sid, x)
            return got if all(g is not None for g in got) else None
        _until(step)
        np.testing.assert_array_equal(np.concatenate(got), pa, err_msg=f"round {rnd}: predictions differ")
        for s in (0, 1):
            ea = a.accept_commit(s, pa[s * (x + 1):(s + 1) * (x + 1)], s + 1)
            eb = b.stream_accept(s, sids[s]).tolist()
            assert ea == eb
    for s in (0, 1):
        assert a.history(s) == b.history(s)
        sa, sb = a.state(s), b.state(s)
        assert (sa["committed"], sa["n_groups"], sa["tail_committed"]) == (sb["committed"], sb["n_groups"],
                                                                           sb["tail_committed"])
    # the compressed tier rebuilt from the streamed window rows equals the staged one
    for layer in (0, 5):
        ra, rb = a.compressed_read(1, layer, 1), b.compressed_read(1, layer, 1)
        for k in ra:
            np.testing.assert_array_equal(ra[k], rb[k], err_msg=f"compressed tier {k} differs (layer {layer})")
    a.close()
    b.close()


@pytest.mark.gpu
def test_stream_ring_scheduled_lossless(cuda, w6):
    n, K = 4, 40
    ref = Engine(TINY6, max_slots=n, max_ctx=2000, max_x=1, quant_bits=0)
    ref.load_weights(w6)
    for s in range(n):
        ref.add_synthetic(s, 900 + 150 * s, 17 + s, seed=1 + s)
    base, _ = ref.autoregress(list(range(n)), K)
    ref.close()
    e = _engine(w6, 3, slots=n)
    for s in range(n):
        e.add_synthetic(s, 900 + 150 * s, 17 + s, seed=1 + s)
        e.compress(s)
    out, st = e.run_scheduled(list(range(n)), K, x=6, window=32)
    np.testing.assert_array_equal(out, base)
    assert st["verifies"] > 0 and st["h2d_bytes"] > 0
    layer_bytes = 2 * TINY6.n_kv * 2048 * TINY6.d_head * 2  # K and V of one layer at cap 2048
    # the ring + 2 admission chunks, and the landing chunks the packed blocks arrive in
    assert st["staging_bytes"] == e.staging_bytes() == (3 + 2 + 3) * layer_bytes
    # packed host pool: a reload moves ~0.76 of the raw bytes
    per_token = 2 * TINY6.layers * TINY6.n_kv * TINY6.d_head * 2
    raw = (900 + 150 * 1.5) * per_token  # mean prefix
    assert st["h2d_bytes"] <= 0.80 * raw * st["verifies"] * 1.1
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("n_rows", [1, 100, 128, 300])
def test_pack_roundtrip_bit_exact(cuda, d, n_rows):
    """The host pool's lossless packing (vc_pack.cu) restores every bf16 bit:
    normal values, outlier channels (x1000), a few zeros / subnormals / tiny
    values (escapes), partial last blocks.  (A channel holding inf or NaN
    escapes every other value of the block: overflow, stored raw.)"""
    torch = cuda
    rng = np.random.default_rng(n_rows + d)
    slices = 3
    x = rng.standard_normal((slices, n_rows, d)).astype(np.float32)
    x[:, :, 5] *= 1000.0  # an outlier channel
    x[0, : min(3, n_rows), 7] = 0.0
    x[1, 0, 9] = 1e-39  # subnormal
    x[1, 0, 10] = 1e-30  # far below the channel's maximum
    bits = T.f32_to_bf16(x)
    src = torch.from_numpy(bits.view(np.int16).copy()).cuda()
    nb = (n_rows + 127) // 128
    out = torch.zeros((slices, nb * 128, d), dtype=torch.int16, device="cuda")
    ovf = C.c_int(-1)
    lib = _lib.load()
    assert lib.vc_pack_roundtrip(src.data_ptr(), n_rows, slices, d, out.data_ptr(), C.byref(ovf),
                                 torch.cuda.current_stream().cuda_stream) == 0
    assert ovf.value == 0
    got = out.cpu().numpy().view(np.uint16)[:, :n_rows]
    np.testing.assert_array_equal(got, bits)


@pytest.mark.gpu
def test_pack_overflow_is_reported(cuda):
    """A block with more escapes than the format holds (here: one channel
    whose values are all zero but one) reports overflow: the engine stores it
    raw.  (An all-zero channel packs: its exponent base is 0.)"""
    torch = cuda
    x = np.random.default_rng(0).standard_normal((1, 128, 128)).astype(np.float32)
    x[0, 1:, 3] = 0.0
    src = torch.from_numpy(T.f32_to_bf16(x).view(np.int16).copy()).cuda()
    out = torch.zeros_like(src)
    ovf = C.c_int(0)
    lib = _lib.load()
    assert lib.vc_pack_roundtrip(src.data_ptr(), 128, 1, 128, out.data_ptr(), C.byref(ovf),
                                 torch.cuda.current_stream().cuda_stream) == 0
    assert ovf.value == 1  # 1 + block 0


@pytest.mark.gpu
def test_pack_secondary_overflow_is_reported(cuda):
    """A block whose exponents spread evenly over 13 binades below each
    channel's maximum puts most values outside the 2-bit codes (offsets 1-3):
    the secondary stream (0.28 of the values) overflows with no escape at all,
    and the block is reported (stored raw).  Its neighbour block packs."""
    torch = cuda
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 256, 128)).astype(np.float32)
    expo = (np.arange(128)[:, None] + np.arange(128)[None, :]) % 13  # offsets 0..12 in every channel
    x[0, :128] = np.sign(x[0, :128]) * (1.0 + rng.random((128, 128))) * 2.0 ** (-expo)
    bits = T.f32_to_bf16(x)
    src = torch.from_numpy(bits.view(np.int16).copy()).cuda()
    out = torch.zeros_like(src)
    ovf = C.c_int(0)
    lib = _lib.load()
    assert lib.vc_pack_roundtrip(src.data_ptr(), 256, 1, 128, out.data_ptr(), C.byref(ovf),
                                 torch.cuda.current_stream().cuda_stream) == 0
    assert ovf.value == 1  # 1 + block 0; block 1 (Gaussian) packs
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint16)[:, 128:], bits[:, 128:])


@pytest.mark.gpu
def test_stream_abort_releases_the_ring(cuda, w6):
    b = _engine(w6, 2)
    for s, n in enumerate(CTX):
        b.add_synthetic(s, n, 17 + s, seed=1 + s)
        b.compress(s)
    sid = b.stream_begin(0)
    b.stream_abort(sid)  # nothing drafted: never advanced
    for _ in range(3):
        b.draft([0])
    sid = b.stream_begin(0)
    p = _until(lambda: b.stream_advance(sid, 3))
    em = b.stream_accept(0, sid)
    assert 1 <= em.size <= 4 and em[-1] == p[em.size - 1]
    with pytest.raises(_lib.ContractError):
        b.swap_begin(1, 0)  # no rotating staging slots in ring mode
    b.close()


def test_stream_ring_config_errors():
    """Rejected at engine creation, before any device allocation."""
    with pytest.raises(_lib.ContractError):  # a staging mode of the host tier only
        Engine(TINY6, max_slots=2, max_ctx=600, max_x=8, quant_bits=4, full_tier=0, ring_chunks=4)
    with pytest.raises(_lib.ContractError):  # at least two chunks
        Engine(TINY6, max_slots=2, max_ctx=600, max_x=8, quant_bits=4, full_tier=1, n_stage=0, ring_chunks=1)
    with pytest.raises(_lib.ContractError):  # the drop tier only offline (no sliding window over appended rows)
        Engine(TINY6, max_slots=2, max_ctx=600, max_x=8, quant_bits=0, drop_ratio=0.2, drop_window=64, full_tier=1,
               n_stage=0, ring_chunks=4)
    with pytest.raises(_lib.ContractError):  # resident slots still need their stages
        Engine(TINY6, max_slots=3, max_ctx=600, max_x=8, quant_bits=4, full_tier=1, n_stage=1, resident_slots=2,
               ring_chunks=4)


def _drop_engine(w, ring, slots=2):
    if ring:
        e = Engine(TINY6, max_slots=slots, max_ctx=2000, max_x=8, quant_bits=0, drop_ratio=0.25, full_tier=1,
                   n_stage=0, ring_chunks=ring, max_streams=2, max_verify=4)
    else:
        e = Engine(TINY6, max_slots=slots, max_ctx=2000, max_x=8, quant_bits=0, drop_ratio=0.25, max_verify=4)
    e.load_weights(w)
    return e


@pytest.mark.gpu
@pytest.mark.parametrize("ring", [2, 4])
def test_drop_tier_stream_reloads_only_dropped_rows(cuda, w6, ring):
    """Drop tier over the chunk ring: the host pool keeps only the dropped
    rows, a streamed verify reloads (1 - c) of the full KV and rebuilds the
    kept rows (and the rows accepted since compress) from the drop tier --
    predictions and tokens equal the HBM-resident drop tier's, round by round."""
    a, b = _drop_engine(w6, 0), _drop_engine(w6, ring)
    for e in (a, b):
        for s, n in enumerate(CTX):
            e.add_synthetic(s, n, 17 + s, seed=1 + s)
            e.compress(s)
    for layer in (0, 5):  # the same kept sets
        np.testing.assert_array_equal(a.drop_kept(layer, 1), b.drop_kept(layer, 1))
    x = 5
    for rnd in range(5):
        for _ in range(x):
            np.testing.assert_array_equal(a.draft([0, 1]), b.draft([0, 1]))
        pa = a.verify([0, 1])
        sids = [b.stream_begin(s) for s in (0, 1)]
        got = [None, None]

        def step():
            for i, sid in enumerate(sids):
                if got[i] is None:
                    got[i] = b.stream_advance(sid, x)
            return got if all(g is not None for g in got) else None
        _until(step)
        np.testing.assert_array_equal(np.concatenate(got), pa, err_msg=f"round {rnd}: predictions differ")
        for s in (0, 1):
            assert a.accept_commit(s, pa[s * (x + 1):(s + 1) * (x + 1)]) == b.stream_accept(s, sids[s]).tolist()
    for s in (0, 1):
        assert a.history(s) == b.history(s)
        assert a.state(s)["drop_len"] == b.state(s)["drop_len"]
    a.close()
    b.close()


@pytest.mark.gpu
def test_drop_tier_ring_scheduled_lossless(cuda, w6):
    n, K = 4, 40
    ctx = [900 + 150 * s for s in range(n)]
    ref = Engine(TINY6, max_slots=n, max_ctx=2000, max_x=1, quant_bits=0)
    ref.load_weights(w6)
    for s in range(n):
        ref.add_synthetic(s, ctx[s], 17 + s, seed=1 + s)
    base, _ = ref.autoregress(list(range(n)), K)
    ref.close()
    e = _drop_engine(w6, 3, slots=n)
    for s in range(n):
        e.add_synthetic(s, ctx[s], 17 + s, seed=1 + s)
        e.compress(s)
    out, st = e.run_scheduled(list(range(n)), K, x=6, window=32)
    np.testing.assert_array_equal(out, base)
    # every reload moved (1 - c) of the prefix: the dropped rows only
    per_token = 2 * TINY6.layers * TINY6.n_kv * TINY6.d_head * 2
    full = sum(ctx) / n * per_token
    assert 0 < st["h2d_bytes"] <= 0.76 * full * st["verifies"]
    e.close()


@pytest.mark.gpu
def test_host_tier_wide_windows_lossless(cuda):
    """The host tier at its operating point, scaled down in depth only: 8
    KV heads of 128 channels over 32K keys, 48-row verify windows streamed
    through the ring (3 row blocks x 8 heads x 16 chunks, several items per
    CTA with the softmax groups' column split changing from item to item),
    the packed host pool -- the emitted tokens equal full-KV greedy decode."""
    s = dataclasses.replace(TINY, vocab=512, hidden=1024, layers=2, n_q=32, n_kv=8, d_head=128, ffn=1024)
    w = T.tiny_weights(s, seed=5, std=0.02)
    n, K, ctx = 6, 96, [32000 - 700 * i for i in range(6)]
    ref = Engine(s, max_slots=n, max_ctx=32800, max_x=1, quant_bits=0)
    ref.load_weights(w)
    for i in range(n):
        ref.add_synthetic(i, ctx[i], 5 + i, seed=1 + i)
    base, _ = ref.autoregress(list(range(n)), K)
    ref.close()
    e = Engine(s, max_slots=n, max_ctx=32800, max_x=47, quant_bits=4, full_tier=1, n_stage=0, ring_chunks=4,
               max_verify=4)
    e.load_weights(w)
    for i in range(n):
        e.add_synthetic(i, ctx[i], 5 + i, seed=1 + i)
        e.compress(i)
    out, st = e.run_scheduled(list(range(n)), K, x=47, window=256)
    np.testing.assert_array_equal(out, base)
    assert st["verifies"] > 0
    e.close()
