/*
 * vc_api.h -- C-ABI of the VeriCache B200 decode loop (libvericache.so).
 *
 * The drop-in boundary for the path BASELINE.json's north star names: a
 * compressed KV cache drafts, the full KV verifies, greedy accept/rollback
 * keeps the output identical to full-KV decode.  Plain pointers and sizes,
 * no exceptions, no torch types.  Every entry point returns a status:
 *   VC_OK (0), VC_ERR_CONFIG (1, bad input -- speckv::ConfigError),
 *   VC_ERR_CONTRACT (2, API misuse -- speckv::ContractError),
 *   VC_ERR_CUDA (3, device failure); vc_last_error() has the message.
 * One host thread per engine (the reference is single-threaded per serving
 * instance: /root/reference/SPEC.md:84, :287).  The engine owns every
 * device and pinned buffer; callers own their token/KV arrays.
 *
 * Reference interfaces each group replaces (all under /root/reference/proj):
 *   vc_compress / vc_compressed_*   speckv::compress / decompress
 *                                   (include/speckv/compressor.hpp:70-80,
 *                                    src/compressor.cpp:130-200)
 *   vc_update_window                speckv::update (compressor.hpp:96-98,
 *                                    src/compressor.cpp:208-243)
 *   vc_draft_step                   speckv::draft's TokenOracle::next calls
 *                                   (include/speckv/specloop.hpp:18-22,39;
 *                                    src/specloop.cpp:11-22)
 *   vc_verify                       speckv::verify (specloop.hpp:44-45,
 *                                    src/specloop.cpp:24-35)
 *   vc_accept / vc_accept_commit    speckv::accept (specloop.hpp:49,
 *                                    src/specloop.cpp:37-56) + KV append
 *   vc_run_speculative / vc_run_decode
 *                                   speckv::run_speculative / autoregress
 *                                   (specloop.hpp:53-61, src/specloop.cpp:58-92)
 *   vc_swap_begin / vc_swap_poll    the transfers SpecScheduler::pending_kickoffs
 *                                   asks for and StepEvents::completed_transfers
 *                                   reports (include/speckv/scheduler.hpp:176-
 *                                   180, 219; src/sim.cpp:243-250)
 *   vc_run_scheduled                simulate_staggered's loop with real kernels
 *                                   and copies (src/sim.cpp:182-307)
 *   vc_prefix_store / vc_prefix_load / vc_run_remote_prefix
 *                                   remote_prefix's payload transfers and
 *                                   draft/verify cycles on real copies and
 *                                   kernels (src/sim.cpp:510-665; closed form
 *                                   t_req_remote, src/analytics.cpp:25-35)
 *   vc_run_speculative_ngram        composition with an n-gram drafter
 *                                   (composed_accept_length, analytics.cpp:413-422)
 *   vc_engine_attach_nccl / vc_tp_* no reference counterpart: the simulator
 *                                   models TP only as GPU counts (core.hpp:45-46);
 *                                   BASELINE.json configs[4] (TP=8 over NVLink)
 */
#ifndef VC_API_H
#define VC_API_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { VC_OK = 0, VC_ERR_CONFIG = 1, VC_ERR_CONTRACT = 2, VC_ERR_CUDA = 3 };

typedef struct vc_engine vc_engine;

typedef struct {
  int vocab, hidden, layers, n_q, n_kv, d_head, ffn;
  float rope_theta, rms_eps;
} vc_model_desc;

typedef struct {
  int max_slots;   /* concurrently resident requests */
  int max_ctx;     /* tokens per request (prefix + generated) */
  int max_x;       /* largest draft horizon */
  int quant_bits;  /* 4 or 2 (quant-uniform compressor), 0 = no compressed tier */
  int full_tier;   /* 0 = full KV resident in HBM, 1 = pinned host pool + staging */
  int n_stage;     /* HBM staging slots for tier 1 */
  int max_verify;  /* verify requests per step */
  int use_graphs;  /* capture steps into CUDA graphs */
  double drop_ratio; /* > 0: drop-topk compressor (retained fraction c in (0,1));
                        exclusive with quant_bits (compressor.cpp:245-254) */
  int tp_size;       /* head-sharded tensor parallelism (configs[4]); 0 or 1 = off.
                        vc_model_desc stays the FULL model; this rank holds
                        n_q/tp_size and n_kv/tp_size heads and ffn/tp_size of the MLP */
  int tp_rank;
  int drop_window;   /* drop-topk tier, online mode (speckv::update, compressor.cpp:
                        208-243): tokens accepted after compress are kept in a
                        sliding window of the latest drop_window..2*drop_window; 0 = keep all */
  int resident_slots; /* tier 1 per-request placement (the reference's B_g = B - B_c,
                         analytics.cpp:45-82): slots [0, resident_slots) keep their
                         full KV resident in HBM (staging slot `slot`, no host copy,
                         never reloaded); the pinned host pool holds the other
                         (offloaded) slots only.  n_stage >= resident_slots + 1. */
  int draft_depth;    /* rows one drafting request may carry in a step: 1 + the
                         auxiliary proposals of the two-level composition
                         (vc_run_speculative_composed); 0 or 1 = plain drafting */
  int ring_chunks;    /* tier 1 staging: > 0 streams every offloaded reload layer by
                         layer into a ring of ring_chunks one-layer chunks and runs
                         the verify range by range as layers land (vc_stream_*);
                         staging HBM = (ring_chunks + 2) layers instead of the
                         rotating whole-request slots (n_stage then holds only the
                         resident slots).  0 = whole-request staging slots.       */
  int max_streams;    /* ring_chunks > 0: streamed verifies in flight (0 -> 2) */
  int drop_score;     /* drop-topk token scores: 0 = L1 norm of the post-RoPE key;
                         1 = SnapKV (observation-window attention of the pending
                         token, summed over the GQA group, max-pooled; HBM full tier) */
  int snap_pool;      /* SnapKV max-pool width (0 -> 7) */
  int snap_recent;    /* SnapKV: last positions always kept (< 0 -> 32) */
  int host_pack;      /* ring_chunks > 0, quantised tier: the host pool stores its
                         128-token blocks losslessly packed (per-channel exponent
                         base + 4-bit offsets + sign|mantissa bytes, escapes for
                         outliers; ~0.76 of the bytes on the link).  0 = default (on),
                         1 = on, -1 = off (raw bf16 rows); k >= 2 = on with at most
                         k-1 packed blocks per request (tests the raw-tail path) */
} vc_runtime_desc;

/* Mirrors speckv::CompressedKVMeta (compressor.hpp:56-65).  Quant-uniform:
 * every position is kept, payload_bytes obeys the size law
 * full_bytes * bit_scheme / 16 (compressor.cpp:96-100, codes only);
 * aux_bytes carries the fp16 scales/zeros the size law does not count.
 * Drop-topk: bit_scheme 16, payload = retained * layers * heads * bytes per
 * token per head (the same size law over the kept tokens).                */
typedef struct {
  int bit_scheme;
  int64_t payload_bytes;
  int64_t aux_bytes;
  int64_t full_bytes;
  int n_groups;
  int tail_tokens;
  int64_t retained_tokens; /* drop-topk: kept tokens per (layer, head); quant: all */
} vc_compressed_meta;

typedef struct {
  int live, committed, pending, n_groups, tail_committed, draft_len;
  int drop_base, drop_len; /* drop-topk tier: kept prefix rows, rows in the tier */
} vc_seq_state;

/* mode: 0 decode (full KV), 1 draft (compressed KV), 2 verify (full KV) */
typedef struct {
  int slot, mode, n_tokens, stage;
  const int32_t* tokens;
} vc_step_item;

const char* vc_last_error(void);
int vc_version(void);

/* ---- engine ----------------------------------------------------------- */
int vc_engine_create(const vc_model_desc* model, const vc_runtime_desc* rt, int device,
                     vc_engine** out);
int vc_engine_destroy(vc_engine* e);
int vc_engine_init_weights(vc_engine* e, uint64_t seed, float stddev);
/* Same, with the residual-branch output projections (o_proj, down_proj)
 * drawn with resid_std (GPT-2 style stddev / sqrt(2 * layers)) and the Q
 * projection rows with q_std (attention temperature); <= 0 keeps stddev.   */
int vc_engine_init_weights_scaled(vc_engine* e, uint64_t seed, float stddev, float resid_std,
                                  float q_std);
/* logical layouts, bf16 bits; per-layer arrays have `layers` pointers      */
int vc_engine_load_weights(vc_engine* e, const uint16_t* embed, const uint16_t* const* attn_norm,
                           const uint16_t* const* wqkv, const uint16_t* const* wo,
                           const uint16_t* const* mlp_norm, const uint16_t* const* wgate,
                           const uint16_t* const* wup, const uint16_t* const* wdown,
                           const uint16_t* final_norm, const uint16_t* lm_head);
int vc_engine_stats(vc_engine* e, uint64_t* kernel_launches, uint64_t* weight_bytes);
/* This engine's KV geometry: layers and KV heads (this rank's share under TP). */
int vc_engine_geometry(vc_engine* e, int* layers, int* kv_heads);
/* Device time (CUDA events, H2D of a step's inputs -> D2H of its tokens)
 * summed over steps since the last reset.                                  */
int vc_engine_timing(vc_engine* e, double* device_ms, int64_t* steps, int reset);
/* Isolated timing of one kernel family over every layer for the given
 * requests: kind 0 draft attention, 1 dense attention (one decode row),
 * 2 dense attention of a verify window (max_x+1 rows), 3 drafting over the
 * drop-topk tier (dense kernel, kept + appended tokens).  *bytes = the
 * algorithmic bytes one launch-set moves.           */
int vc_kernel_bench(vc_engine* e, int kind, const int* slots, int n, int reps, double* ms,
                    double* bytes);

/* ---- tensor parallelism (head-sharded, configs[4]) -------------------------
 * The o_proj / down_proj partials of the ranks are combined as an all-gather
 * plus a fixed rank-order sum (batch-invariant, so verify logits still equal
 * decode logits bit for bit).  Collectives: NCCL over NVLink (one process per
 * GPU; rank 0 creates the 128-byte unique id and shares it), or an in-process
 * loopback group (one host thread per rank on one device; steps run eagerly). */
typedef struct vc_tp_group vc_tp_group;
int vc_nccl_get_unique_id(uint8_t* out128);
int vc_engine_attach_nccl(vc_engine* e, const uint8_t* unique_id128);
int vc_tp_loopback_create(int size, vc_tp_group** out);
int vc_tp_loopback_destroy(vc_tp_group* g);
int vc_engine_attach_loopback(vc_engine* e, vc_tp_group* g);
/* Device time (us, CUDA events on the engine stream) of one combine: the
 * all-gather of rows x hidden fp32 partials + the rank-order residual sum,
 * averaged over reps; every rank of the group must call it together.       */
int vc_tp_collective_bench(vc_engine* e, int rows, int reps, double* us);

/* ---- requests ----------------------------------------------------------- */
int vc_request_add_synthetic(vc_engine* e, int slot, int n_ctx, int32_t first_token, uint64_t seed,
                             int outlier_channels, float outlier_scale);
/* k, v: bf16 [layers][n_kv][n_ctx][d_head] */
int vc_request_add_kv(vc_engine* e, int slot, int n_ctx, int32_t first_token, const uint16_t* k,
                      const uint16_t* v);
int vc_request_prefill(vc_engine* e, int slot, const int32_t* prompt, int n);
int vc_request_release(vc_engine* e, int slot);
int vc_request_state(vc_engine* e, int slot, vc_seq_state* out);
/* every token emitted so far (capacity cap); *n receives the count */
int vc_request_history(vc_engine* e, int slot, int32_t* out, int cap, int* n);

/* ---- compressor ---------------------------------------------------------- */
/* Mirrors speckv::CompressorSpec (compressor.hpp:24-41).  kind: 0 drop-uniform,
 * 1 drop-window, 2 quant-uniform (the reference's three), 3 drop-topk (score-
 * based top-k per (layer, head), BASELINE.json configs[2]).  mode: 0 offline
 * (1 online goes through vc_update_window).                                 */
typedef struct {
  int kind;
  int mode;
  int bits;         /* quant-uniform width */
  int window;       /* drop-window: recent tokens kept (online) */
  int sink_tokens;  /* drop-window: leading tokens never dropped */
} vc_compressor_spec;

/* Offline compress of the request's committed prefix with the engine's own
 * tier (quant bits / drop_ratio given at creation).                        */
int vc_compress(vc_engine* e, int slot, vc_compressed_meta* out);
/* speckv::compress(spec, shape, ratio, seed) (compressor.hpp:70-71) on the GPU
 * tier: shape = the request's committed prefix (layers, n_kv, T, 4*d_head);
 * drop-uniform / drop-window drop exactly the reference's indices for `seed`
 * (compressor.cpp:152-177) and keep the rest in the drop tier; drop-topk keeps
 * llround(ratio*T) by score; quant-uniform needs spec.bits == quant_bits.
 * The spec must fit the engine's tier (ContractError otherwise).           */
int vc_compress_spec(vc_engine* e, int slot, const vc_compressor_spec* spec, double ratio,
                     uint64_t seed, vc_compressed_meta* out);
/* Copy one (layer, kv-head) slice of the compressed tier to host:
 * kcodes/vcodes u32 words (fragment order), ksz [groups][d],
 * vsz [groups*128], ktail/vtail bf16 [tail_cap][d].  Any pointer may be NULL. */
int vc_compressed_read(vc_engine* e, int slot, int layer, int head, uint32_t* kcodes,
                       uint32_t* ksz, uint32_t* vcodes, uint32_t* vsz, uint16_t* ktail,
                       uint16_t* vtail);
/* Kept positions (ascending, int32) of one (layer, kv-head) from the most
 * recent drop-topk vc_compress; *n = retained count.  Positions not listed
 * are the reference's dropped_indices (compressor.hpp:57-59).              */
int vc_drop_kept(vc_engine* e, int layer, int head, int32_t* out, int cap, int* n);
int vc_compressed_geometry(vc_engine* e, int* group, int* words_per_group, int* tail_cap,
                           int* max_groups);
/* Drop-index generation of the token-dropping compressors, bit-identical
 * to speckv::compress (compressor.cpp:152-177): kind 0 drop-uniform, 1
 * drop-window; kept positions are the complement.  out [layers][heads][drop]. */
int64_t vc_drop_indices(int kind, int layers, int heads, int64_t tokens, double ratio,
                        uint64_t seed, int sink_tokens, int64_t* out);
/* speckv::update for drop-window online compression, one layer, a batch of
 * requests (compressor.cpp:208-243).  already[i] = drops so far at layer;
 * new drops for request i, head h at out[(i*heads + h)*cap + k].           */
int vc_update_window(int heads, int window, int sink_tokens, int n_req, const int64_t* tokens,
                     const int64_t* req_begin, const int64_t* req_end, const int64_t* already,
                     int64_t* out, int64_t cap, int64_t* n_new);
/* Drop-topk: keep the k highest scores per row (ties -> lower position);
 * scores device [rows][T] fp32, kept device [rows][k] int32 ascending.    */
int vc_topk_select(const float* scores, int rows, int T, int k, int32_t* kept, void* stream);
/* Key-norm scores s_t = sum_c |k_tc| w_c for device bf16 keys [rows][T][d]. */
/* Host-pool packing round trip (device pointers, tests): src bf16 [slices][n_rows][d]
 * is packed per 128-token block (vc_pack.cu) and unpacked into out (same
 * layout, rows padded to whole blocks); *overflow = 1 + the first block with
 * more escapes than the format holds (0 = every block packed).             */
int vc_pack_roundtrip(const uint16_t* src, int n_rows, int n_slices, int d, uint16_t* out, int* overflow,
                      void* stream);
int vc_key_scores(const uint16_t* keys, int rows, int T, int d, const float* w, float* scores,
                  void* stream);

/* Greedy argmax of device fp32 logits [rows][n] into device out[rows]:
 * std::max_element semantics of speckv::greedy_oracle (specloop.cpp:256-263) --
 * ties -> smallest index; NaNs never win; a NaN at index 0, or a row with
 * nothing above -inf, gives index 0.                                        */
int vc_argmax_rows(const float* logits, int rows, int n, int32_t* out, void* stream);

/* ---- steps ---------------------------------------------------------------- */
/* One forward pass over a heterogeneous batch; out_rows receives the greedy
 * token of every input row (item order).  logits (optional) [rows][vocab]. */
int vc_step(vc_engine* e, const vc_step_item* items, int n, int32_t* out_rows, float* logits);
int vc_decode_step(vc_engine* e, const int* slots, int n, int32_t* out_tokens);
int vc_draft_step(vc_engine* e, const int* slots, int n, int32_t* out_tokens);
/* Verify every slot's open draft round; preds receives x_i+1 tokens per
 * slot back to back.  stages: staging slot per request (tier 1) or NULL.  */
int vc_verify(vc_engine* e, const int* slots, int n, const int* stages, int32_t* preds);
/* Greedy accept rule (specloop.cpp:37-56) on host arrays.                  */
int vc_accept(const int32_t* drafted, const int32_t* preds, int x, int32_t* accepted,
              int* n_accepted, int* first_mismatch, int* bonus);
/* Accept + commit exact KV of the accepted prefix + roll the draft window back. */
int vc_accept_commit(vc_engine* e, int slot, const int32_t* preds, int stage, int32_t* emitted,
                     int* n_emitted);

/* ---- host tier ------------------------------------------------------------ */
int vc_swap_begin(vc_engine* e, int slot, int stage, uint64_t* transfer_id);
int vc_swap_poll(vc_engine* e, uint64_t transfer_id, int* done);
/* Layer-chunked host tier (ring_chunks > 0): the reload the reference books
 * over S_r windows (scheduler.cpp:15-23, :96-163) streamed one layer per
 * chunk, with the verify pipelined on the landed layers.
 *   vc_stream_begin    start streaming slot's committed full KV; *id
 *   vc_stream_advance  run the verify over the layers landed since the last
 *                      call (the slot's open round must be complete: it is
 *                      the window scored); *done = 1 once all layers ran and
 *                      the x+1 predictions are in preds (capacity x+1)
 *   vc_stream_accept   accept + commit from the streamed verify (the exact
 *                      window rows it wrote), frees the stream
 *   vc_stream_abort    drop an unfinished stream (waits for its copies)     */
int vc_stream_begin(vc_engine* e, int slot, int* id);
int vc_stream_advance(vc_engine* e, int id, int* done, int32_t* preds);
int vc_stream_accept(vc_engine* e, int slot, int id, int32_t* emitted, int* n_emitted);
int vc_stream_abort(vc_engine* e, int id);
/* HBM bytes of the host tier's staging (rotating slots or the chunk ring). */
int vc_engine_staging_bytes(vc_engine* e, int64_t* bytes);
/* Drop-topk introspection (tests): the scores of the last compress for one
 * (layer, kv head) row (n <= T floats), and the SnapKV observation query of a
 * layer ([n_q][d_head] bf16, post-RoPE).                                    */
int vc_drop_scores(vc_engine* e, int layer, int head, float* out, int n);
int vc_obs_query(vc_engine* e, int layer, uint16_t* out);

/* ---- decode loops ----------------------------------------------------------- */
/* Full-KV greedy decode of K tokens for each slot (the baseline).
 * out [n][K]; *ms = device time of the loop (one CUDA event pair around it). */
int vc_run_decode(vc_engine* e, const int* slots, int n, int K, int32_t* out, double* ms);
/* Lossless speculative loop (lock-step rounds of x drafts + one verify per
 * slot).  out [n][K]; accepted-per-round written to rounds (cap max_rounds
 * per slot, row-major [n][max_rounds]); n_rounds [n].                       */
int vc_run_speculative(vc_engine* e, const int* slots, int n, int K, int x, int32_t* out,
                       int32_t* rounds, int max_rounds, int* n_rounds, double* ms);

/* Same loop with the drafter composed with n-gram (prompt-lookup) drafts
 * (BASELINE.json configs[4] "int4 compressor composed with n-gram speculative
 * drafts"): a request whose emitted history repeats
 * its last `ngram` tokens drafts the continuation that followed (up to x tokens,
 * no draft steps); the others draft over the compressed tier; all verify in
 * one full-KV pass.  ngram_rounds [n] = rounds that used an n-gram draft.     */
int vc_run_speculative_ngram(vc_engine* e, const int* slots, int n, int K, int x, int ngram, int32_t* out,
                             int32_t* rounds, int max_rounds, int* n_rounds, int* ngram_rounds, double* ms);

/* One request of a synthetic workload: prefix length, first input token,
 * prefix-KV seed (vc_request_add_synthetic), arrival time (ms on the loop clock). */
typedef struct {
  int n_ctx;
  int32_t first_token;
  uint64_t seed;
  double arrival_ms;
} vc_request_desc;

/* Two-level composition (composed_accept_length,
 * analytics.cpp:413-422): lock-step rounds of x OUTER draft passes over the
 * compressed KV; at each outer position an auxiliary prompt-lookup drafter
 * (`ngram`-token key over the request's own context) proposes up to depth-1
 * more tokens that ride the same pass as extra rows (needs draft_depth >=
 * depth); proposals the compressed model confirms join the draft window, then
 * one full-KV verify checks it all.  out [n][K].                            */
typedef struct {
  int64_t rounds, verifies, tokens;
  int64_t draft_steps;    /* compressed-model passes */
  int64_t drafted;        /* draft tokens verified (all rounds) */
  int64_t aux_proposed;   /* auxiliary tokens offered to the compressed model */
  int64_t aux_accepted;   /* of those, confirmed by it (gamma_e = accepted / proposed) */
  double mean_accept;     /* accepted drafted tokens per verify */
  double ms;              /* device time of the loop */
} vc_compose_stats;
int vc_run_speculative_composed(vc_engine* e, const int* slots, int n, int K, int x, int ngram, int depth,
                                int32_t* out, vc_compose_stats* stats);

/* Swap-scheduled loop (tier 1): SpecScheduler semantics drive real draft
 * rows, verify rows and H2D reloads (Algorithm 1).     */
typedef struct {
  int x;                    /* draft_length */
  int window;               /* lookahead_window W */
  double iteration_time;    /* planning T_iter (s); <= 0: measure */
  double link_bandwidth;    /* planning BW (B/s); <= 0: measure */
  int64_t hbm_capacity;     /* bytes for weights + resident + in-flight */
  int K;                    /* output tokens per request */
  int64_t warmup_iterations;  /* iterations before the timed window */
  int64_t timed_iterations;   /* length of the timed window; 0 = run to completion */
  /* Per-request tier placement (the reference's B_c knob, intra_throughput /
   * optimize_intra, analytics.cpp:45-82,130-150), tier 1: requests in the
   * engine's resident slots (vc_runtime_desc.resident_slots, B_g) verify
   * against their HBM-resident full KV and are never reloaded; the others
   * (B_c) are reloaded per verify through the rotating staging slots under
   * the swap scheduler.  Every request drafts on its compressed KV.  Residents
   * run x_resident-token rounds (0 = x), verify as soon as a round is
   * drafted, staggered so about B_g / (x_resident + 1) windows verify per
   * iteration.                                                              */
  int x_resident;
  /* Requests arriving during the run (simulate_staggered's arrivals,
   * sim.cpp:227-302): arrival_ms on the loop's host clock; each is admitted
   * FIFO into a slot a finished request freed (synthetic prefix KV written
   * and compressed at admission; a resident slot's request is resident).
   * out then holds n + n_arrivals rows; latencies are completion - arrival. */
  const vc_request_desc* arrivals;
  int n_arrivals;
  /* Two-level composition inside the serving loop (
   * composed_accept_length, analytics.cpp:413-422): with ngram >= 1 and
   * depth >= 2 every drafting row carries up to depth-1 prompt-lookup
   * proposals (`ngram`-token key over the request's own context) as extra
   * rows of the same pass (engine draft_depth >= depth); proposals the
   * compressed model confirms join the window.  One scheduler draft
   * iteration can then append several tokens; the verify checks them all.
   * 0 = plain drafting.                                                     */
  int ngram;
  int depth;
} vc_sched_desc;

typedef struct {
  double wall_ms;           /* device+host time of the loop */
  int64_t tokens;           /* emitted tokens (all requests) */
  int64_t iterations;
  int64_t verifies;
  int64_t late_transfers;
  double h2d_bytes;         /* bytes of the reloads completed in the timed window */
  double h2d_ms;            /* copy-engine busy time of the reloads (timed window) */
  double verify_wait_ms;    /* exposed swap time: sum over iterations of (sessions
                               stalled on a late reload) x iteration wall time */
  double mean_accept;       /* accepted drafted tokens per verify */
  int64_t timed_iterations; /* iterations inside the timed window */
  int64_t timed_tokens;     /* tokens emitted inside the timed window */
  double timed_wall_ms;     /* host wall time of the timed window (e2e) */
  double timed_device_ms;   /* device time of the window: one CUDA event pair on the
                               compute stream around all its steps (gaps included) */
  double timed_rows;        /* activation rows executed in the window */
  double timed_step_device_ms; /* sum over the window's steps of each step's own device time
                                  (event pair around its H2D, graph and D2H): the window's
                                  device time minus the host-planning gaps between steps */
  int64_t resident_verifies;  /* verifies of resident requests (full KV in HBM) */
  double resident_accept;     /* their accepted drafted tokens per verify */
  int64_t timed_resident_tokens; /* tokens the residents emitted inside the timed window */
  int64_t timed_verifies;     /* verify windows executed inside the timed window */
  double timed_verify_rows;   /* their rows (x+1 each); timed_rows - this = drafting rows */
  /* SimMetrics (sim.hpp:52-74) of the whole run on the loop's host clock:
   * throughput = tokens / wall time, warm = first and last 10% of the run's
   * time cut (sim.cpp:103-109), request latency percentiles (completion -
   * start; rank ceil(q n), sim.cpp:92-99), interconnect busy = copy-engine time
   * / wall time, peak HBM = weights + compressed tier + full-KV slots.     */
  double throughput;
  double warm_throughput;
  double p50_latency_s;
  double p99_latency_s;
  double interconnect_busy;
  int64_t peak_hbm_bytes;
  int64_t staging_bytes;    /* HBM of the host tier's staging (vc_engine_staging_bytes) */
  int64_t drafted_tokens;   /* tokens that entered verify windows (composition: > draft iterations) */
  int64_t aux_proposed;     /* composition: auxiliary tokens offered to the compressed model */
  int64_t aux_accepted;     /* of those, confirmed by it (gamma_e = accepted / proposed) */
  double reload_over_full;  /* bytes a reload moves / the full KV it restores (packed host
                               pool ~0.76, drop tier 1-c, raw 1), over the offloaded requests */
} vc_sched_stats;

/* Reference metrics of a loop (SimMetrics, sim.hpp:52-74) on the engine:
 * the clock is the sum of the steps' device times (CUDA events around each
 * step), so time spent outside steps -- admission, host planning -- is not
 * charged, exactly as the reference charges T_iter = bytes / BW per step. */
typedef struct {
  double throughput;        /* tokens / clock */
  double warm_throughput;   /* first and last 10% of the clock cut (sim.cpp:103-109) */
  double p50_latency_s;     /* completion - arrival on that clock (sim.cpp:92-99) */
  double p99_latency_s;
  int64_t tokens;
  int64_t iterations;
  int64_t completed;
  int64_t unserved;         /* requests that can never fit (sim.cpp:438-440) */
  double clock_s;           /* sum of step device times */
  double wall_ms;           /* host wall time of the loop */
  double mean_batch;        /* requests per decode step */
  int max_batch;
  int64_t peak_hbm_bytes;   /* weights + resident full KV at the peak */
  double full_batch_throughput; /* tokens / clock over the steps that ran with every
                                   slot occupied: the capacity-capped steady state */
} vc_loop_metrics;



/* The reference's full-KV baseline (baseline_full_kv, sim.cpp:418-494) on the
 * real engine: requests are admitted FIFO while a full-KV slot is free (the
 * engine's max_slots full-KV slots ARE its HBM capacity: weights + resident +
 * KV <= gpu_mem, sim.cpp:455-461), each decodes K tokens, one per step, and
 * leaves.  Admission (synthesising the prefix KV) is not on the clock.
 * out [n][K].                                                               */
int vc_run_decode_fifo(vc_engine* e, const vc_request_desc* reqs, int n, int K, int32_t* out,
                       vc_loop_metrics* m);

int vc_run_scheduled(vc_engine* e, const int* slots, int n, const vc_sched_desc* sd,
                     int32_t* out, vc_sched_stats* stats);

/* ---- remote prefix caching (BASELINE.json configs[3]) ---------------------
 * The reference simulates this pipeline (remote_prefix, sim.cpp:510-665;
 * closed form t_req_remote, analytics.cpp:25-35).  Here the storage node is
 * pinned host memory holding one shared prefix in both forms:
 *   vc_prefix_store(e, slot)  snapshot slot's committed (compressed) prefix;
 *   vc_prefix_load(e, slot, what, first_token, &id)  stream one form into a
 *     request slot on the copy stream: what 0 = the compressed payload
 *     (drafting can start), 1 = the full KV (verification can start);
 *     completion via vc_swap_poll.
 * vc_run_remote_prefix runs a workload of n requests over that prefix:
 * arrivals, the payload loads (compressed ahead of full on the link), drafting
 * on the compressed KV while the full KV streams, verify once both are
 * resident (the full KV stays cached, verify_cached), accept/rollback.  With
 * baseline = 1 it is the reference's force_baseline arm: load the full KV,
 * then decode. */
typedef struct {
  int x;                        /* draft horizon */
  int K;                        /* output tokens per request */
  int baseline;                 /* 1: full-KV baseline (load full KV, then decode) */
  int link_queue;               /* transfers kept queued on the copy stream (>= 1) */
  double arrival_gap_ms;        /* request i arrives i * gap after the start (0 = burst) */
  const int32_t* first_tokens;  /* [n] each request's first input token (its own prompt suffix) */
  int payload_order;            /* 0: per request (compressed_i, full_i, compressed_i+1, ...);
                                   1: every arrived compressed payload ahead of any full KV */
} vc_remote_desc;

typedef struct {
  double makespan_ms;       /* device time, start -> last token (event pair on the compute stream) */
  double wall_ms;           /* host wall time of the loop */
  int64_t tokens;           /* emitted tokens (all requests, truncated at K) */
  int64_t iterations;       /* forward steps */
  int64_t link_waits;       /* times the loop blocked on the link with nothing to compute */
  int64_t verifies;
  double mean_accept;       /* accepted drafted tokens per verify */
  double ttft_ms_mean;      /* arrival -> first emitted token (host clock) */
  double ttft_ms_max;
  double compressed_ready_ms_mean; /* arrival -> compressed payload resident */
  double full_ready_ms_mean;       /* arrival -> full KV resident */
  double h2d_bytes;         /* bytes of all payload loads */
  double h2d_ms;            /* copy-engine busy time of those loads */
} vc_remote_stats;

int vc_prefix_store(vc_engine* e, int slot);
int vc_prefix_load(vc_engine* e, int slot, int what, int32_t first_token, uint64_t* transfer_id);
int vc_run_remote_prefix(vc_engine* e, const int* slots, int n, const vc_remote_desc* rd, int32_t* out,
                         vc_remote_stats* stats);

/* ---- scheduler ------------------------------------------------------------ */
int vc_reload_span(int64_t bytes, double bandwidth, double iteration_time, double* iterations,
                   int* windows);

/* ---- kernel-level entry points (device pointers) -------------------------- */
/* Quantise one token-major bf16 slice [n_groups*128][d] into the fragment
 * layout (what vc_compress does per (layer, request, kv-head)).            */
int vc_quant_kivi_slice(const uint16_t* k, const uint16_t* v, int n_groups, int d, int bits,
                        uint32_t* kcodes, uint32_t* ksz, uint32_t* vcodes, uint32_t* vsz,
                        void* stream);
/* Attention of q (bf16 [n_rows][n_q][d], device) for one request/layer of
 * the engine's pools.  mode 1 = draft over the compressed tier (n_rows 1),
 * mode 0/2 = dense over the full tier (causal over the last n_rows).
 * out: host bf16 [n_rows][n_q][d].                                          */
int vc_attention_probe(vc_engine* e, int slot, int layer, int mode, const uint16_t* q_dev,
                       int n_rows, int kv_len, uint16_t* out_host);
/* Read n token rows of one (layer, kv-head) slice of a KV pool to host bf16
 * buffers [n][d]: pool 0 = HBM full tier, 1 = staging slots, 2 = host pool,
 * 3 = drop-topk compacted tier. */
int vc_kv_read(vc_engine* e, int pool, int slot, int layer, int head, int pos, int n, uint16_t* k,
               uint16_t* v);
/* ws = X[M][K] . W[N][K]^T via the batch-invariant projection GEMM (device). */
int vc_gemm_probe(const uint16_t* X, int M, int K, const uint16_t* W, int N, float* Y,
                  void* stream);
/* Same with a fused epilogue: epi 0 = fp32 store, 3 = SiLU-gate over
 * interleaved (gate, up) columns into bf16 act [M][N/2] (tiled layout).     */
int vc_gemm_probe_epi(const uint16_t* X, int M, int K, const uint16_t* W, int N, int epi, void* Y,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif
