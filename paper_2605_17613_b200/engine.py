"""Python host mirror of the reference interface for the decode-loop path.

Thin numpy/ctypes layer over include/vc_api.h, with the reference's names
and argument meanings so parity tests read like /root/reference/proj/tests:

  Engine.compress(slot)            speckv::compress, quant-uniform (compressor.cpp:130-178)
  Engine.draft(slots)              one TokenOracle::next per drafting request (specloop.cpp:11-22)
  Engine.verify(slots)             speckv::verify: x+1 predictions (specloop.cpp:24-35)
  accept(drafted, predictions)     speckv::accept (specloop.cpp:37-56)
  Engine.run_speculative(...)      speckv::run_speculative (specloop.cpp:58-79)
  Engine.autoregress(...)          speckv::autoregress over the full KV (specloop.cpp:81-92)
  Engine.run_scheduled(...)        simulate_staggered's loop on real kernels (sim.cpp:182-307)
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class ModelShape:
    vocab: int
    hidden: int
    layers: int
    n_q: int
    n_kv: int
    d_head: int
    ffn: int
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5

    @property
    def kv_bytes_per_token(self) -> int:
        return self.layers * self.n_kv * self.d_head * 2 * 2


# BASELINE.json configs[0] (tiny) and configs[1] (Llama-3-8B shape).  The
# tiny model's FFN and vocabulary are not fixed by the reference; these are
# the values DESIGN.md documents.
TINY = ModelShape(vocab=2048, hidden=512, layers=2, n_q=8, n_kv=2, d_head=64, ffn=1536)
LLAMA3_8B = ModelShape(vocab=128256, hidden=4096, layers=32, n_q=32, n_kv=8, d_head=128, ffn=14336)
LLAMA3_70B = ModelShape(vocab=128256, hidden=8192, layers=80, n_q=64, n_kv=8, d_head=128, ffn=28672)


@dataclass
class SpecRoundResult:
    drafted: list
    predictions: list
    accepted: list
    bonus_used: bool
    first_mismatch: int | None


def accept(drafted, predictions) -> SpecRoundResult:
    """speckv::accept through the C-ABI (vc_accept)."""
    lib = _lib.load()
    d = np.ascontiguousarray(drafted, dtype=np.int32)
    p = np.ascontiguousarray(predictions, dtype=np.int32)
    if p.size != d.size + 1:
        raise _lib.ContractError(2, "accept: |predictions| must equal |drafted| + 1")
    out = np.zeros(d.size + 1, np.int32)
    n, fm, bonus = C.c_int(), C.c_int(), C.c_int()
    check(lib.vc_accept(_ptr(d, C.c_int32), _ptr(p, C.c_int32), d.size, _ptr(out, C.c_int32),
                        C.byref(n), C.byref(fm), C.byref(bonus)))
    return SpecRoundResult(d.tolist(), p.tolist(), out[: n.value].tolist(), bool(bonus.value),
                           fm.value or None)


def drop_indices(kind: str, layers: int, heads: int, tokens: int, ratio: float, seed: int = 0,
                 sink_tokens: int = 0) -> np.ndarray:
    """Dropped positions [layers][heads][drop] of drop-uniform / drop-window."""
    lib = _lib.load()
    k = {"drop-uniform": 0, "drop-window": 1}[kind]
    retained = int(math.floor(ratio * tokens + 0.5))
    drop = max(tokens - retained, 0)
    out = np.zeros((layers, heads, max(drop, 1)), np.int64)
    rc = lib.vc_drop_indices(k, layers, heads, tokens, ratio, seed, sink_tokens, _ptr(out, C.c_int64))
    if rc < 0:
        check(-rc)
    return out[:, :, :rc]


def reload_span(bytes_: int, bandwidth: float, iteration_time: float):
    lib = _lib.load()
    it, w = C.c_double(), C.c_int()
    check(lib.vc_reload_span(int(bytes_), bandwidth, iteration_time, C.byref(it), C.byref(w)))
    return it.value, w.value


class Engine:
    """One serving instance on one GPU (vc_engine)."""

    def __init__(self, model: ModelShape, *, max_slots=1, max_ctx=4096, max_x=16, quant_bits=4,
                 full_tier=0, n_stage=2, max_verify=2, use_graphs=True, device=0, drop_ratio=0.0,
                 tp_size=1, tp_rank=0, drop_window=0, resident_slots=0, draft_depth=1,
                 ring_chunks=0, max_streams=2, drop_score="norm", snap_pool=7, snap_recent=32, host_pack=True):
        """quant_bits > 0: quant-uniform compressor (KIVI int4/int2);
        drop_ratio in (0, 1): drop-topk compressor keeping llround(c*T) tokens per
        (layer, head) -- the two are exclusive (compressor.cpp:245-254).
        tp_size > 1: this engine is rank tp_rank of a head-sharded tensor-parallel
        group (`model` is the full model; attach_nccl / attach_loopback before stepping).
        drop_window > 0 (drop-topk only): online mode -- tokens accepted after
        compress stay in a sliding window of the latest drop_window..2*drop_window.
        resident_slots > 0 (full_tier 1): per-request placement -- slots
        [0, resident_slots) keep their full KV resident in HBM (the reference's
        B_g), the pinned host pool holds the other slots only (B_c).
        ring_chunks > 0 (full_tier 1): reloads stream layer by layer into a ring
        of one-layer chunks and each verify runs range by range as its layers
        land (stream_*); n_stage then holds only the resident slots.
        drop_score (drop-topk): "norm" = L1 norm of the post-RoPE key; "snapkv" =
        SnapKV observation-window attention (the pending token's query over the
        full KV, summed over the GQA group, max-pooled over snap_pool positions,
        the last snap_recent positions always kept).
        host_pack (ring_chunks > 0, quantised tier): the host pool's 128-token
        blocks are stored losslessly packed (~0.76 of the link bytes per reload)."""
        if drop_score not in ("norm", "snapkv"):
            raise ValueError("drop_score is 'norm' or 'snapkv'")
        self.lib = _lib.load()
        self.model = model
        self.max_x = max_x
        md = _lib.ModelDesc(model.vocab, model.hidden, model.layers, model.n_q, model.n_kv,
                            model.d_head, model.ffn, model.rope_theta, model.rms_eps)
        rt = _lib.RuntimeDesc(max_slots, max_ctx, max_x, quant_bits, full_tier, n_stage,
                              max_verify, int(use_graphs), float(drop_ratio), int(tp_size), int(tp_rank),
                              int(drop_window), int(resident_slots), int(draft_depth),
                              int(ring_chunks), int(max_streams), 1 if drop_score == "snapkv" else 0,
                              int(snap_pool), int(snap_recent),
                              (int(host_pack) if not isinstance(host_pack, bool) else (1 if host_pack else -1)))
        self.tp_size, self.tp_rank = int(tp_size), int(tp_rank)
        h = C.c_void_p()
        check(self.lib.vc_engine_create(C.byref(md), C.byref(rt), device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.vc_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- weights ----------------------------------------------------------------
    def init_weights(self, seed: int = 0, std: float = 0.02, resid_std: float = 0.0,
                     q_std: float = 0.0):
        """Random init; resid_std > 0 scales o_proj/down_proj (GPT-2: std/sqrt(2L)),
        q_std > 0 the Q projection (attention temperature)."""
        if resid_std > 0 or q_std > 0:
            check(self.lib.vc_engine_init_weights_scaled(self.h, seed, std, resid_std, q_std))
        else:
            check(self.lib.vc_engine_init_weights(self.h, seed, std))

    def load_weights(self, w: dict):
        """w: logical bf16-bit arrays (uint16) as oracle/vc_oracle.h documents
        (the FULL model; a tensor-parallel rank takes its shard, tp_shard)."""
        if self.tp_size > 1:
            w = tp_shard(w, self.model, self.tp_size, self.tp_rank)
        L = self.model.layers
        keep = []

        def arr(a):
            a = np.ascontiguousarray(a, dtype=np.uint16)
            keep.append(a)
            return _ptr(a, C.c_uint16)

        def lst(name):
            ptrs = (_lib.PU16 * L)(*[arr(w[name][i]) for i in range(L)])
            keep.append(ptrs)
            return ptrs

        check(self.lib.vc_engine_load_weights(
            self.h, arr(w["embed"]), lst("attn_norm"), lst("wqkv"), lst("wo"), lst("mlp_norm"),
            lst("wgate"), lst("wup"), lst("wdown"), arr(w["final_norm"]), arr(w["lm_head"])))

    # ---- tensor parallelism -----------------------------------------------------
    def attach_nccl(self, unique_id: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        check(self.lib.vc_engine_attach_nccl(self.h, buf))

    def attach_loopback(self, group: "TpLoopback"):
        check(self.lib.vc_engine_attach_loopback(self.h, group.h))

    def collective_bench(self, rows, reps=20) -> float:
        """us per o_proj/down_proj combine (all-gather + rank-order sum) of `rows` rows."""
        us = C.c_double()
        check(self.lib.vc_tp_collective_bench(self.h, rows, reps, C.byref(us)))
        return us.value

    def stats(self):
        n, b = C.c_uint64(), C.c_uint64()
        check(self.lib.vc_engine_stats(self.h, C.byref(n), C.byref(b)))
        return {"kernel_launches": n.value, "weight_bytes": b.value}

    # ---- requests ---------------------------------------------------------------
    def add_synthetic(self, slot, n_ctx, first_token, seed=1, outlier_channels=4, outlier_scale=10.0):
        check(self.lib.vc_request_add_synthetic(self.h, slot, n_ctx, first_token, seed,
                                                outlier_channels, outlier_scale))

    def add_kv(self, slot, k: np.ndarray, v: np.ndarray, first_token: int):
        """k, v: uint16 bf16 bits [layers][n_kv][n_ctx][d]."""
        k = np.ascontiguousarray(k, np.uint16)
        v = np.ascontiguousarray(v, np.uint16)
        check(self.lib.vc_request_add_kv(self.h, slot, k.shape[2], first_token, _ptr(k, C.c_uint16),
                                         _ptr(v, C.c_uint16)))

    def prefill(self, slot, prompt):
        p = np.ascontiguousarray(prompt, np.int32)
        check(self.lib.vc_request_prefill(self.h, slot, _ptr(p, C.c_int32), p.size))

    def release(self, slot):
        check(self.lib.vc_request_release(self.h, slot))

    def state(self, slot) -> dict:
        s = _lib.SeqState()
        check(self.lib.vc_request_state(self.h, slot, C.byref(s)))
        return {f: getattr(s, f) for f, _ in s._fields_}

    def history(self, slot) -> list:
        cap = 1 << 16
        out = np.zeros(cap, np.int32)
        n = C.c_int()
        check(self.lib.vc_request_history(self.h, slot, _ptr(out, C.c_int32), cap, C.byref(n)))
        return out[: n.value].tolist()

    # ---- compressor -------------------------------------------------------------
    def compress(self, slot) -> dict:
        m = _lib.CompressedMeta()
        check(self.lib.vc_compress(self.h, slot, C.byref(m)))
        return {f: getattr(m, f) for f, _ in m._fields_}

    COMPRESSOR_KINDS = {"drop-uniform": 0, "drop-window": 1, "quant-uniform": 2, "drop-topk": 3}

    def compress_spec(self, slot, kind: str, ratio: float = 0.0, seed: int = 0, bits: int = 4,
                      sink_tokens: int = 0, window: int = 8) -> dict:
        """speckv::compress(spec, shape, ratio, seed) on this engine's GPU tier
        (vc_compress_spec): drop-uniform / drop-window drop the reference's own
        indices for `seed`; drop-topk keeps the top scores; quant-uniform needs
        bits == the engine's quant_bits."""
        cs = _lib.CompressorSpec(self.COMPRESSOR_KINDS[kind], 0, bits, window, sink_tokens)
        m = _lib.CompressedMeta()
        check(self.lib.vc_compress_spec(self.h, slot, C.byref(cs), float(ratio), seed, C.byref(m)))
        return {f: getattr(m, f) for f, _ in m._fields_}

    def drop_scores(self, layer, head, n):
        """Scores of the last drop-topk compress for one (layer, kv head): n floats."""
        out = np.zeros(n, np.float32)
        check(self.lib.vc_drop_scores(self.h, layer, head, _ptr(out, C.c_float), n))
        return out

    def obs_query(self, layer):
        """SnapKV observation query of a layer: [n_q][d_head] bf16 bits (post-RoPE)."""
        out = np.zeros((self.model.n_q, self.model.d_head), np.uint16)
        check(self.lib.vc_obs_query(self.h, layer, _ptr(out, C.c_uint16)))
        return out

    def drop_kept(self, layer, head):
        """Kept positions (ascending) of one (layer, head) from the last drop-topk compress."""
        n = C.c_int()
        check(self.lib.vc_drop_kept(self.h, layer, head, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.int32)
        check(self.lib.vc_drop_kept(self.h, layer, head, _ptr(out, C.c_int32), out.size, C.byref(n)))
        return out[: n.value]

    def compressed_geometry(self):
        g, w, t, mg = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(self.lib.vc_compressed_geometry(self.h, C.byref(g), C.byref(w), C.byref(t), C.byref(mg)))
        return g.value, w.value, t.value, mg.value

    def compressed_read(self, slot, layer, head):
        G, words, tail_cap, max_groups = self.compressed_geometry()
        d = self.model.d_head
        kc = np.zeros(words * max_groups, np.uint32)
        vc = np.zeros_like(kc)
        ksz = np.zeros(max_groups * d, np.uint32)
        vsz = np.zeros(max_groups * G, np.uint32)
        kt = np.zeros(tail_cap * d, np.uint16)
        vt = np.zeros_like(kt)
        check(self.lib.vc_compressed_read(self.h, slot, layer, head, _ptr(kc, C.c_uint32),
                                          _ptr(ksz, C.c_uint32), _ptr(vc, C.c_uint32),
                                          _ptr(vsz, C.c_uint32), _ptr(kt, C.c_uint16),
                                          _ptr(vt, C.c_uint16)))
        return dict(kc=kc, vc=vc, ksz=ksz, vsz=vsz, ktail=kt.reshape(tail_cap, d),
                    vtail=vt.reshape(tail_cap, d))

    # ---- steps ------------------------------------------------------------------
    def step(self, items, want_logits=False):
        """items: list of (slot, mode, tokens, stage); mode 0 decode, 1 draft, 2 verify."""
        arr = (_lib.StepItem * len(items))()
        keep = []
        rows = 0
        for i, (slot, mode, toks, stage) in enumerate(items):
            t = np.ascontiguousarray(toks, np.int32)
            keep.append(t)
            arr[i] = _lib.StepItem(slot, mode, t.size, stage, _ptr(t, C.c_int32))
            rows += t.size
        out = np.zeros(rows, np.int32)
        logits = np.zeros((rows, self.model.vocab), np.float32) if want_logits else None
        check(self.lib.vc_step(self.h, arr, len(items), _ptr(out, C.c_int32),
                               _ptr(logits, C.c_float) if want_logits else None))
        return (out, logits) if want_logits else out

    def decode_step(self, slots):
        s = np.ascontiguousarray(slots, np.int32)
        out = np.zeros(s.size, np.int32)
        check(self.lib.vc_decode_step(self.h, _ptr(s, C.c_int), s.size, _ptr(out, C.c_int32)))
        return out

    def draft(self, slots):
        s = np.ascontiguousarray(slots, np.int32)
        out = np.zeros(s.size, np.int32)
        check(self.lib.vc_draft_step(self.h, _ptr(s, C.c_int), s.size, _ptr(out, C.c_int32)))
        return out

    def verify(self, slots, stages=None):
        s = np.ascontiguousarray(slots, np.int32)
        total = sum(self.state(int(x))["draft_len"] + 1 for x in s)
        out = np.zeros(total, np.int32)
        st = np.ascontiguousarray(stages, np.int32) if stages is not None else None
        check(self.lib.vc_verify(self.h, _ptr(s, C.c_int), s.size,
                                 _ptr(st, C.c_int) if st is not None else None, _ptr(out, C.c_int32)))
        return out

    def accept_commit(self, slot, preds, stage=-1):
        p = np.ascontiguousarray(preds, np.int32)
        out = np.zeros(p.size, np.int32)
        n = C.c_int()
        check(self.lib.vc_accept_commit(self.h, slot, _ptr(p, C.c_int32), stage, _ptr(out, C.c_int32),
                                        C.byref(n)))
        return out[: n.value].tolist()

    def swap_begin(self, slot, stage) -> int:
        x = C.c_uint64()
        check(self.lib.vc_swap_begin(self.h, slot, stage, C.byref(x)))
        return x.value

    def swap_poll(self, xfer) -> bool:
        d = C.c_int()
        check(self.lib.vc_swap_poll(self.h, xfer, C.byref(d)))
        return bool(d.value)

    # ---- loops ------------------------------------------------------------------
    def autoregress(self, slots, K):
        """Full-KV greedy decode of K tokens per slot -> (tokens [n][K], ms)."""
        s = np.ascontiguousarray(slots, np.int32)
        out = np.zeros((s.size, K), np.int32)
        ms = C.c_double()
        check(self.lib.vc_run_decode(self.h, _ptr(s, C.c_int), s.size, K, _ptr(out, C.c_int32),
                                     C.byref(ms)))
        return out, ms.value

    def run_speculative(self, slots, K, x, max_rounds=4096):
        s = np.ascontiguousarray(slots, np.int32)
        out = np.zeros((s.size, K), np.int32)
        rounds = np.zeros((s.size, max_rounds), np.int32)
        nr = np.zeros(s.size, np.int32)
        ms = C.c_double()
        check(self.lib.vc_run_speculative(self.h, _ptr(s, C.c_int), s.size, K, x, _ptr(out, C.c_int32),
                                          _ptr(rounds, C.c_int32), max_rounds, _ptr(nr, C.c_int),
                                          C.byref(ms)))
        return out, [rounds[i, : nr[i]].tolist() for i in range(s.size)], ms.value

    def run_speculative_ngram(self, slots, K, x, ngram=3, max_rounds=4096):
        """run_speculative with the drafter composed with n-gram (prompt-lookup)
        drafts -> (tokens [n][K], emitted per round, n-gram rounds per slot, ms)."""
        s = np.ascontiguousarray(slots, np.int32)
        out = np.zeros((s.size, K), np.int32)
        rounds = np.zeros((s.size, max_rounds), np.int32)
        nr = np.zeros(s.size, np.int32)
        ng = np.zeros(s.size, np.int32)
        ms = C.c_double()
        check(self.lib.vc_run_speculative_ngram(self.h, _ptr(s, C.c_int), s.size, K, x, ngram,
                                                _ptr(out, C.c_int32), _ptr(rounds, C.c_int32), max_rounds,
                                                _ptr(nr, C.c_int), _ptr(ng, C.c_int), C.byref(ms)))
        return out, [rounds[i, : nr[i]].tolist() for i in range(s.size)], ng.tolist(), ms.value

    def run_speculative_composed(self, slots, K, x, ngram=2, depth=2):
        """Two-level composition: x outer compressed-KV draft
        passes per round, each carrying up to depth-1 prompt-lookup proposals the
        compressed model may confirm -> (tokens [n][K], stats dict)."""
        s = np.ascontiguousarray(slots, np.int32)
        out = np.zeros((s.size, K), np.int32)
        st = _lib.ComposeStats()
        check(self.lib.vc_run_speculative_composed(self.h, _ptr(s, C.c_int), s.size, K, x, ngram, depth,
                                                   _ptr(out, C.c_int32), C.byref(st)))
        return out, {f: getattr(st, f) for f, _ in st._fields_}

    def timing(self, reset=False):
        ms, n = C.c_double(), C.c_int64()
        check(self.lib.vc_engine_timing(self.h, C.byref(ms), C.byref(n), int(reset)))
        return ms.value, n.value

    def kernel_bench(self, kind, slots, reps=5):
        s = np.ascontiguousarray(slots, np.int32)
        ms, b = C.c_double(), C.c_double()
        check(self.lib.vc_kernel_bench(self.h, kind, _ptr(s, C.c_int), s.size, reps, C.byref(ms),
                                       C.byref(b)))
        return ms.value, b.value

    def run_scheduled(self, slots, K, x, window, iteration_time=0.0, link_bandwidth=0.0,
                      hbm_capacity=0, warmup_iterations=0, timed_iterations=0, x_resident=0, arrivals=None,
                      ngram=0, depth=0):
        """Requests in the engine's resident slots (resident_slots, the
        reference's B_g; analytics.cpp:45-82) verify against their HBM-resident
        full KV with x_resident-token rounds; the others are reloaded per verify.
        arrivals = [(n_ctx, first_token, seed, arrival_ms)]: requests that arrive
        during the run and take the slots finished requests free (out gains a
        row per arrival).  ngram >= 1, depth >= 2: two-level composition -- every
        drafting row carries up to depth-1 prompt-lookup proposals (engine
        draft_depth >= depth)."""
        s = np.ascontiguousarray(slots, np.int32)
        arr = arrivals or []
        out = np.zeros((s.size + len(arr), K), np.int32)
        ad = (_lib.RequestDesc * max(len(arr), 1))(*[_lib.RequestDesc(int(a), int(b), int(c), float(d))
                                                     for a, b, c, d in arr])
        sd = _lib.SchedDesc(x, window, iteration_time, link_bandwidth, hbm_capacity, K,
                            warmup_iterations, timed_iterations, x_resident,
                            ad if arr else None, len(arr), int(ngram), int(depth))
        st = _lib.SchedStats()
        check(self.lib.vc_run_scheduled(self.h, _ptr(s, C.c_int), s.size, C.byref(sd),
                                        _ptr(out, C.c_int32), C.byref(st)))
        return out, {f: getattr(st, f) for f, _ in st._fields_}

    # ---- layer-chunked host tier (ring_chunks > 0) --------------------------------
    def stream_begin(self, slot) -> int:
        """Start streaming slot's committed full KV layer by layer (returns an id)."""
        i = C.c_int()
        check(self.lib.vc_stream_begin(self.h, slot, C.byref(i)))
        return i.value

    def stream_advance(self, sid, x):
        """Run the verify over the layers landed so far (the open round must be
        complete) -> the x+1 predictions once every layer ran, else None."""
        done = C.c_int()
        preds = np.zeros(x + 1, np.int32)
        check(self.lib.vc_stream_advance(self.h, sid, C.byref(done), _ptr(preds, C.c_int32)))
        return preds if done.value else None

    def stream_accept(self, slot, sid):
        """Accept + commit from the finished streamed verify -> emitted tokens."""
        out = np.zeros(self.max_x + 2, np.int32)
        n = C.c_int()
        check(self.lib.vc_stream_accept(self.h, slot, sid, _ptr(out, C.c_int32), C.byref(n)))
        return out[:n.value]

    def stream_abort(self, sid):
        check(self.lib.vc_stream_abort(self.h, sid))

    def staging_bytes(self) -> int:
        b = C.c_int64()
        check(self.lib.vc_engine_staging_bytes(self.h, C.byref(b)))
        return b.value

    def run_decode_fifo(self, requests, K):
        """baseline_full_kv (sim.cpp:418-494): requests = [(n_ctx, first_token,
        seed, arrival_ms)], admitted FIFO while a full-KV slot is free ->
        (tokens [n][K], SimMetrics dict)."""
        n = len(requests)
        arr = (_lib.RequestDesc * n)(*[_lib.RequestDesc(int(a), int(b), int(c), float(d)) for a, b, c, d in requests])
        out = np.zeros((n, K), np.int32)
        m = _lib.LoopMetrics()
        check(self.lib.vc_run_decode_fifo(self.h, arr, n, K, _ptr(out, C.c_int32), C.byref(m)))
        return out, {f: getattr(m, f) for f, _ in m._fields_}

    # ---- remote prefix (configs[3]) --------------------------------------------
    def prefix_store(self, slot):
        """Snapshot slot's compressed prefix (full KV + compressed payload) into
        the pinned host store -- the storage node of remote_prefix (sim.cpp:510)."""
        check(self.lib.vc_prefix_store(self.h, slot))

    def prefix_load(self, slot, what, first_token) -> int:
        """Stream the stored prefix into `slot` on the copy stream: what 0 = the
        compressed payload, 1 = the full KV.  Returns a transfer id (swap_poll)."""
        x = C.c_uint64()
        check(self.lib.vc_prefix_load(self.h, slot, what, first_token, C.byref(x)))
        return x.value

    def run_remote_prefix(self, slots, K, x, first_tokens, baseline=False, link_queue=2,
                          arrival_gap_ms=0.0, payload_order=0):
        """Requests over the stored prefix: (tokens [n][K], stats dict)."""
        s = np.ascontiguousarray(slots, np.int32)
        ft = np.ascontiguousarray(first_tokens, np.int32)
        if ft.size != s.size:
            raise ValueError("one first token per request")
        out = np.zeros((s.size, K), np.int32)
        rd = _lib.RemoteDesc(x, K, int(bool(baseline)), link_queue, arrival_gap_ms,
                             _ptr(ft, C.c_int32), payload_order)
        st = _lib.RemoteStats()
        check(self.lib.vc_run_remote_prefix(self.h, _ptr(s, C.c_int), s.size, C.byref(rd),
                                            _ptr(out, C.c_int32), C.byref(st)))
        return out, {f: getattr(st, f) for f, _ in st._fields_}

    # ---- probes -----------------------------------------------------------------
    def kv_read(self, pool, slot, layer, head, pos, n):
        """pool 0 full (HBM), 1 staging, 2 host, 3 drop tier; returns bf16 bits k, v [n][d]."""
        d = self.model.d_head
        k = np.zeros((n, d), np.uint16)
        v = np.zeros_like(k)
        check(self.lib.vc_kv_read(self.h, pool, slot, layer, head, pos, n, _ptr(k, C.c_uint16),
                                  _ptr(v, C.c_uint16)))
        return k, v

    def attention_probe(self, slot, layer, mode, q_dev_ptr, n_rows, kv_len):
        out = np.zeros((n_rows, self.model.n_q, self.model.d_head), np.uint16)
        check(self.lib.vc_attention_probe(self.h, slot, layer, mode, C.c_void_p(q_dev_ptr), n_rows,
                                          kv_len, _ptr(out, C.c_uint16)))
        return out


def tp_shard(w: dict, model: ModelShape, tp: int, rank: int) -> dict:
    """Rank `rank`'s shard of full logical weights for head-sharded TP: q/k/v
    rows of its n_q/tp query and n_kv/tp KV heads, the matching o_proj input
    columns, ffn/tp gate/up rows and down_proj input columns; embedding, norms
    and LM head replicated."""
    d, nq, nkv, F = model.d_head, model.n_q, model.n_kv, model.ffn
    ql, kl, fl = nq // tp * d, nkv // tp * d, F // tp
    out = dict(w)

    def qkv(a):
        a = np.asarray(a).reshape((nq + 2 * nkv) * d, -1)
        q = a[rank * ql:(rank + 1) * ql]
        k = a[nq * d + rank * kl:nq * d + (rank + 1) * kl]
        v = a[(nq + nkv) * d + rank * kl:(nq + nkv) * d + (rank + 1) * kl]
        return np.ascontiguousarray(np.concatenate([q, k, v]))

    out["wqkv"] = [qkv(a) for a in w["wqkv"]]
    out["wo"] = [np.ascontiguousarray(np.asarray(a).reshape(model.hidden, nq * d)[:, rank * ql:(rank + 1) * ql])
                 for a in w["wo"]]
    out["wgate"] = [np.ascontiguousarray(np.asarray(a).reshape(F, -1)[rank * fl:(rank + 1) * fl]) for a in w["wgate"]]
    out["wup"] = [np.ascontiguousarray(np.asarray(a).reshape(F, -1)[rank * fl:(rank + 1) * fl]) for a in w["wup"]]
    out["wdown"] = [np.ascontiguousarray(np.asarray(a).reshape(model.hidden, F)[:, rank * fl:(rank + 1) * fl])
                    for a in w["wdown"]]
    return out


class TpLoopback:
    """In-process tensor-parallel group on one device (one host thread per rank)."""

    def __init__(self, size: int):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.vc_tp_loopback_create(size, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.vc_tp_loopback_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    lib = _lib.load()
    buf = (C.c_uint8 * 128)()
    check(lib.vc_nccl_get_unique_id(buf))
    return bytes(buf)
