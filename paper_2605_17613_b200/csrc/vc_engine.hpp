// vc_engine.hpp -- the B200 decode-loop engine behind include/vc_api.h.
//
// Owns the model weights, the three KV tiers and the step executor:
//   * full KV:        bf16 [slot][layer][kv-head][cap][d], resident in HBM
//                     (tier 0) or in a pinned host pool streamed into HBM
//                     staging slots before each verify (tier 1);
//   * compressed KV:  KIVI int4/int2 codes + fp16 scale/zero in mma fragment
//                     order, plus a bf16 tail (residual group + draft window);
//   * activations and split-K workspaces sized for the largest step.
// A step is one forward pass over a heterogeneous batch: drafting rows
// (compressed KV), verify rows (x+1 per request, full KV) and plain decode
// rows (full KV) share every weight read.  Kernels are launched on the
// compute stream and captured into CUDA graphs keyed by the step shape.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "vc_gemm.h"
#include "vc_kernels.h"
#include "vc_tp.h"

namespace vc {

struct ModelDesc {
  int vocab = 0, hidden = 0, layers = 0, n_q = 0, n_kv = 0, d = 0, ffn = 0;
  float rope_theta = 500000.f, eps = 1e-5f;
};

struct EngineConfig {
  ModelDesc model;
  int max_slots = 1;    // concurrently resident requests
  int max_ctx = 4096;   // token capacity per request (prefix + generated)
  int max_x = 16;       // largest draft horizon
  int quant_bits = 4;   // 4 or 2; 0 disables the compressed tier
  double drop_ratio = 0; // > 0: drop-topk compressed tier (retained fraction c), exclusive with quant
  int drop_window = 0;   // > 0: online sliding window over the tokens accepted after compress
  int full_tier = 0;    // 0: full KV in HBM; 1: pinned host pool + staging
  int n_stage = 2;      // HBM staging slots (tier 1)
  // tier 1, per-request placement (the reference's B_g = B - B_c,
  // analytics.cpp:45-82): slots [0, resident_slots) keep their full KV
  // resident in HBM staging slot `slot` and have no host copy; the host pool
  // holds slots [resident_slots, max_slots) only
  int resident_slots = 0;
  // rows a drafting request may carry per step (1 + auxiliary proposals of
  // the two-level composition); sizes the activation and partial buffers
  int draft_depth = 1;
  int max_verify = 2;   // verify requests per step
  int use_graphs = 1;
  // head-sharded tensor parallelism: `model` is this rank's shard (n_q, n_kv,
  // ffn already divided by tp_size); o_proj/down_proj partials are combined
  // through the attached Collective (vc_tp.h)
  int tp_size = 1, tp_rank = 0;
  // tier 1, layer-chunked streaming: > 0 replaces the rotating whole-request
  // staging slots by a ring of ring_chunks one-layer chunks ([kv-head][cap][d]
  // K and V each); a verify runs layer range by layer range as its chunks
  // land (Engine::stream_*), so staging HBM is ring_chunks layers, not
  // n_stage whole requests.  n_stage then holds the resident slots only.
  int ring_chunks = 0;
  int max_streams = 2;  // streamed verifies in flight (saved hidden state + exact window rows each)
  // chunk ring over the quantised tier: store the host pool's 128-token
  // blocks losslessly packed (vc_pack.cu, ~0.76 of the bytes on the link).
  // 0 off, 1 on; k >= 2: on with at most k - 1 packed blocks per request (a
  // test knob for the raw-tail path that only incompressible data reaches)
  int host_pack = 1;
  // drop-topk token scores: 0 = L1 norm of the post-RoPE key; 1 = SnapKV
  // (Li et al., 2024): attention of the observation query (the request's
  // pending token, one decode-shaped forward over the full KV) summed over the
  // GQA group, max-pooled over snap_pool positions, the last snap_recent
  // positions always kept
  int drop_score = 0;
  int snap_pool = 7;
  int snap_recent = 32;
};

enum class RowMode : int { Decode = 0, Draft = 1, Verify = 2 };

// One request's part of a step.
struct StepItem {
  int slot = 0;
  RowMode mode = RowMode::Decode;
  std::vector<int32_t> tokens;  // inputs: 1 (decode/draft) or x+1 (verify)
  int stage = -1;               // staging slot holding this request's full KV (tier 1 verify)
};

struct SeqState {
  bool live = false;
  int committed = 0;      // positions with exact KV in the full tier
  int32_t pending = 0;    // last emitted token (its KV is not computed yet)
  int n_groups = 0;       // quantised groups in the compressed tier
  int tail_committed = 0; // exact tokens in the draft tail (committed - n_groups*G)
  int draft_len = 0;      // drafted tokens of the open round (their KV in the tail)
  int drop_len = 0;       // drop tier: kept prefix tokens + exact tokens appended since
  int drop_base = 0;      // drop tier: rows of the compress-time kept prefix
  int drop_T = 0;         // drop tier: positions the compress covered (kept + dropped)
  int packed_blocks = 0;  // host tier (chunk ring): leading 128-token blocks stored packed, the rest raw
  std::vector<int32_t> drafted;
  std::vector<int32_t> history;  // every emitted token
};

struct StepTiming {
  float ms = 0.f;
};

class Engine {
 public:
  explicit Engine(const EngineConfig& cfg, int device);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const EngineConfig& config() const { return cfg_; }
  const ModelDesc& model() const { return cfg_.model; }

  // ---- tensor parallelism ---------------------------------------------
  void attach_collective(std::unique_ptr<Collective> c);
  // Device time of one o_proj/down_proj combine (all-gather of rows x hidden
  // fp32 partials + the rank-order residual sum), averaged over reps (us).
  double collective_bench(int rows, int reps);

  // ---- weights -------------------------------------------------------
  void init_weights_random(uint64_t seed, float stddev, float resid_std = 0.f, float q_std = 0.f);
  // Logical layouts (see oracle/vc_oracle.h); bf16 bits.
  void load_weights(const uint16_t* embed, const uint16_t* const* attn_norm,
                    const uint16_t* const* wqkv, const uint16_t* const* wo,
                    const uint16_t* const* mlp_norm, const uint16_t* const* wgate,
                    const uint16_t* const* wup, const uint16_t* const* wdown,
                    const uint16_t* final_norm, const uint16_t* lm_head);

  // ---- requests ------------------------------------------------------
  // Synthetic prefix KV (K ~ N(0,1) with outlier channels x10, V ~ N(0,1))
  // for positions [0, n_ctx); `pending` is the first input token.
  void add_request_synthetic(int slot, int n_ctx, int32_t pending, uint64_t seed,
                             int outlier_channels, float outlier_scale);
  // Host-provided prefix KV: k/v bf16 [layer][kv-head][n_ctx][d].
  void add_request_kv(int slot, int n_ctx, int32_t pending, const uint16_t* k, const uint16_t* v);
  // Real prefill: forward the prompt (all but the last token become context).
  void add_request_prefill(int slot, const int32_t* prompt, int n);
  void release(int slot);
  const SeqState& seq(int slot) const { return seqs_.at(slot); }

  // Quantise the committed prefix into the compressed tier (offline compress).
  void compress(int slot);
  // Same with an explicit retained ratio (drop tier, <= drop_ratio) or an
  // explicit kept set kept_host [layers*n_kv][k_host] (ascending positions).
  void compress_as(int slot, double ratio, const int32_t* kept_host, int k_host);

  // ---- steps ---------------------------------------------------------
  // Executes one forward over the items; writes argmax per input row into
  // `out` (rows in item order) and optionally fp32 logits.
  void run_step(const std::vector<StepItem>& items, std::vector<int32_t>& out,
                float* logits_host = nullptr);
  // Commit helpers (state only; kernels launched as needed).
  void commit_decode(int slot, int32_t next);
  void push_draft(int slot, int32_t tok);
  // Roll back an open draft round without verifying it.
  void discard_drafts(int slot);
  // Accept rule over the open round given the verifier's x+1 predictions;
  // commits exact KV, rolls back the draft window.  Returns emitted tokens.
  std::vector<int32_t> accept_commit(int slot, const std::vector<int32_t>& preds, int stage = -1);

  // ---- host tier -----------------------------------------------------
  // Start the H2D reload of slot's committed full KV into staging slot
  // `stage` on the copy stream; returns a transfer id.
  uint64_t swap_begin(int slot, int stage);
  bool swap_done(uint64_t id);
  void swap_wait(uint64_t id);
  // ---- host tier, layer-chunked (ring_chunks > 0) ------------------------
  // A streamed verify of an offloaded slot: its committed full KV streams
  // layer by layer from the host pool into ring chunks on the copy stream
  // (stream_pump issues a chunk as soon as its ring chunk is free); once the
  // round's draft window is complete, stream_advance runs the verify forward
  // over the layers that have landed (hidden state carried between ranges),
  // releasing each chunk as soon as its layer ran.  When the last layer ran,
  // the x+1 predictions are ready (stream_preds) and accept_commit_stream
  // commits from the exact window rows the verify wrote (no staging slot).
  int stream_begin(int slot);
  void stream_pump();
  // 0: in progress; 1: predictions ready.  Requires the slot's open round to
  // be the window the verify scores (fixed by the first call that runs layers).
  int stream_advance(int id);
  std::vector<int32_t> stream_preds(int id) const;
  std::vector<int32_t> accept_commit_stream(int slot, const std::vector<int32_t>& preds, int id);
  void stream_end(int id);  // abandon / free (waits for its copies)
  int streams_active() const { return static_cast<int>(vstreams_.size()); }
  int stream_layers_done(int id) const;
  bool ring_mode() const { return cfg_.full_tier == 1 && cfg_.ring_chunks > 0; }
  // HBM bytes of the host tier's staging: rotating slots, or the chunk ring
  size_t staging_bytes() const;
  // bytes a reload of the slot's committed full KV moves over the link
  // (packed blocks + raw rows, or the drop tier's dropped rows, or raw)
  double reload_bytes(int slot) const;
  // ---- remote prefix (configs[3]) -------------------------------------
  // The storage node's precomputed KV of one shared prefix: slot's committed
  // full KV and its compressed image (quant tier) snapshotted into pinned
  // host memory.  prefix_load() streams one form into a request slot on the
  // copy stream (what 0 = compressed payload -> drafting can start; 1 = full
  // KV -> verification can start) and returns a transfer id (swap_done).
  void prefix_store(int src_slot);
  void prefix_drop();
  int prefix_tokens() const { return pre_T_; }
  double prefix_bytes(int what) const;
  uint64_t prefix_load(int slot, int what, int32_t pending);

  // copy-engine time of the completed H2D reloads (CUDA events on the copy stream)
  double h2d_ms() const { return h2d_ms_; }
  double h2d_bytes() const { return h2d_bytes_; }  // bytes of the completed reloads

  // tier 1 placement: is the slot's full KV resident in HBM (its own stage)?
  int draft_rows_max() const { return cfg_.max_slots * std::max(1, cfg_.draft_depth); }
  bool resident(int slot) const { return cfg_.full_tier == 1 && slot < cfg_.resident_slots; }
  // staging slot used as scratch for offloaded requests (compress, synthesis)
  int scratch_stage() const { return scratch_override_ >= 0 ? scratch_override_ : cfg_.resident_slots; }
  // the serving loop lends a free rotating staging slot for an admission
  void set_scratch_stage(int stage) { scratch_override_ = stage; }

  // ---- raw access for tests ------------------------------------------
  KvPool full_pool() const { return full_; }
  KvPool stage_pool() const { return stage_; }
  QuantPool quant_pool() const { return quant_; }
  KvPool drop_pool() const { return drop_; }
  bool drop_mode() const { return cfg_.drop_ratio > 0.0; }
  // kept positions (ascending) of the last drop-mode compress, row = layer*n_kv+head
  int last_kept_k() const { return last_kept_k_; }
  // the drop-topk scores of the last compress (row = layer*n_kv+head, T floats)
  // and the SnapKV observation query per layer ([n_q][d] bf16, post-RoPE)
  void drop_scores(int layer, int head, float* out, int n) const;
  void obs_query(int layer, uint16_t* out) const;
  const int32_t* last_kept_device() const { return kept_buf_; }
  // host-pool rows of an offloaded slot (nullptr for a resident slot)
  // wait for the commits still copying exact rows into the host pool
  void sync_host_pool() const { check_d2h(); }
  uint16_t* host_pool_k(int slot) const;
  uint16_t* host_pool_v(int slot) const;
  cudaStream_t stream() const { return st_; }
  size_t weight_bytes() const { return weight_bytes_; }
  size_t full_kv_bytes_per_token() const;
  size_t compressed_bytes(int slot) const;
  const float* last_logits_device() const { return logits_; }
  int last_rows() const { return last_M_; }

  // kernel launch counter (every kernel this engine enqueued)
  uint64_t launches() const { return launches_; }

  // Attention of caller-provided q (device, [n_rows][n_q][d]) for one
  // request/layer: mode 1 draft over the compressed tier, else dense.
  void attention_probe(int slot, int layer, int mode, const uint16_t* q_dev, int n_rows,
                       int kv_len, uint16_t* out_host);
  // Device time of run_step (H2D descriptors -> D2H tokens), accumulated.
  double device_ms() const { return device_ms_; }
  int64_t steps() const { return steps_; }
  void reset_timing() { device_ms_ = 0.0; steps_ = 0; }
  // Isolated timing of one kernel family over the given requests (all
  // layers): kind 0 draft attention (+combine), 1 dense attention (+combine).
  // Returns ms per launch-set and the algorithmic bytes it moves.
  void kernel_bench(int kind, const std::vector<int>& slots, int reps, double* ms, double* bytes);

 private:
  struct Weights {
    uint16_t* embed = nullptr;
    std::vector<uint16_t*> attn_norm, wqkv, wo, mlp_norm, wgu, wd;
    uint16_t* final_norm = nullptr;
    uint16_t* lm_head = nullptr;
  };
  void alloc_all();
  void check_d2h() const;
  void set_kv_rows(const std::vector<StepItem>& items, std::vector<RowDest>& rows) const;
  void enqueue_forward(int M, int n_draft, int n_dense1, int n_densev, int max_rows_v,
                       bool want_logits);
  void quantise_groups(int slot, int g0, int ng, const KvPool& src, int src_slot, int origin = 0,
                       int layer0 = 0, int layers = -1);
  // where accept_commit reads the exact rows of the round: a pool slot whose
  // rows are absolute positions minus `origin`
  struct RowSrc {
    KvPool pool;
    int slot;
    int origin;
  };
  std::vector<int32_t> accept_commit_from(int slot, const std::vector<int32_t>& preds, const RowSrc& src,
                                          bool to_host);
  struct VStream {
    int slot = -1, buf = -1;
    int64_t base = 0;          // chunk sequence number of layer 0 (ring chunk of layer l: (base + l) % R)
    int issued = 0;            // layers whose chunk copies are enqueued
    int landed = 0;            // layers whose chunk copies have completed (observed)
    int done = 0;              // layers the verify forward has run
    int committed = 0, origin = 0, x = -1;
    std::vector<int32_t> tokens;  // verify inputs: pending + drafted (fixed at the first range)
    bool final_enqueued = false;
    cudaEvent_t ev_final = nullptr;
    std::vector<int32_t> preds;
  };
  void stream_issue_chunk(VStream& v);
  bool host_pack_on() const { return ring_mode() && !drop_mode() && cfg_.host_pack > 0; }
  // the slot's host rows of layer l (n_kv slices, rows [0, n)): raw chunk
  // `craw` -> host pool, blocks [0, P) packed through chunk `cpk`; and back
  void host_store_layer(int slot, int l, int craw, int cpk, int n, int P);
  void host_load_layer(int slot, int l, int craw, int cpk, int n, int P);
  int* pack_overflow_ = nullptr;              // device: 1 + first block that did not pack (0 = all packed)
  uint8_t* pack_stage_ = nullptr;             // accept-time packing of the window's block: [2][layers*n_kv][PB]
  void stream_range(VStream& v, int a, int b);
  void ring_fill_layer(int slot, int layer, int chunk, bool from_host);
  void compress_drop(int slot, const KvPool& src, int src_slot, double ratio, const int32_t* kept_host,
                     int k_host);

  EngineConfig cfg_;
  int device_ = 0;
  cudaStream_t st_ = nullptr, copy_st_ = nullptr;
  cudaStream_t d2h_st_ = nullptr;  // commit of exact rows back to the host pool
  cudaEvent_t ev_commit_ = nullptr, ev_d2h_ = nullptr;
  Weights w_;
  void* weight_blob_ = nullptr;
  size_t weight_bytes_ = 0;
  float *rope_cos_ = nullptr, *rope_sin_ = nullptr;
  KvPool full_{}, stage_{};
  DenseMaps dense_maps_{};  // tensor maps of the HBM pool the dense kernel reads (tier 0 full, tier 1 stage)
  QuantPool quant_{};
  // drop-topk tier: compacted bf16 K/V of the kept tokens (+ appended exact
  // tokens + the open draft window), read by the dense kernel
  KvPool drop_{};
  DenseMaps drop_maps_{};
  int max_chunks_x_ = 0;
  float* score_buf_ = nullptr;  // [layers*n_kv][T] key scores of the last compress
  int score_T_ = 0;
  float *snap_logits_ = nullptr, *snap_ms_ = nullptr;  // SnapKV scratch (one layer)
  uint16_t* obs_q_ = nullptr;   // [layers][n_q*d] observation query of the last SnapKV compress
  bool capture_q_ = false;      // enqueue_forward copies row 0's q heads into obs_q_ per layer
  float* score_w_ = nullptr;    // [d] per-channel score weights (ones)
  int32_t* kept_buf_ = nullptr; // [layers*n_kv][k] kept positions of the last compress
  int last_kept_k_ = 0;
  int kept_cap_ = 0;            // kept positions per slice kept_buf_ holds
  int scratch_override_ = -1;   // staging slot used as scratch (-1: the first rotating one)
  // offloaded slot whose freshly synthesised full KV still sits in staging
  // slot scratch_stage_used_ (compress() then skips the reload)
  int scratch_slot_ = -1, scratch_stage_used_ = -1;
  uint16_t *host_k_ = nullptr, *host_v_ = nullptr;
  // prefix store (pinned): full K/V [slice][T][d], records [slice][ng][words], tails [slice][tc][d]
  uint16_t *pre_k_ = nullptr, *pre_v_ = nullptr, *pre_kt_ = nullptr, *pre_vt_ = nullptr;
  uint32_t* pre_rec_ = nullptr;
  int pre_T_ = 0, pre_ng_ = 0, pre_tc_ = 0;
  int max_chunks_q_ = 0, max_chunks_d_ = 0, tail_cap_ = 0, Mmax_ = 0;
  int draft_warps_ = 0, draft_min_tasks_ = 4;  // quantised draft-attention work split
  // activations
  float* x_ = nullptr;
  uint16_t *xn_ = nullptr, *qkv_ = nullptr, *attn_ = nullptr, *act_ = nullptr;
  GemmWorkspace gws_{};
  float* ss_part_ = nullptr;  // per-(row, 128-feature tile) sums of squares
  float* logits_ = nullptr;
  int32_t *tok_in_ = nullptr, *tok_out_ = nullptr;
  Partials part_{};
  RowDest* rows_dev_ = nullptr;
  AttnSeq* seqs_dev_ = nullptr;  // [draft | dense1 | densev]
  QuantJob* jobs_dev_ = nullptr;
  // pinned staging of per-step descriptors
  void* h_desc_ = nullptr;
  void* d_hdesc_ = nullptr;     // device view of the mapped h_desc_
  int32_t* d_hout_ = nullptr;   // device view of the mapped h_out_
  size_t desc_bytes_ = 0;
  int32_t* h_out_ = nullptr;
  std::vector<SeqState> seqs_;
  int last_M_ = 0;
  uint64_t launches_ = 0;
  // tensor parallelism: partial projection output and the gathered partials
  std::unique_ptr<Collective> coll_;
  float *tp_y_ = nullptr, *tp_g_ = nullptr;
  // graphs keyed by step shape
  std::map<std::string, cudaGraphExec_t> graphs_;
  std::map<std::string, uint64_t> launches_per_graph_;
  // transfers
  struct Xfer {
    cudaEvent_t start, done;
    double bytes;
  };
  std::map<uint64_t, Xfer> xfers_;
  // layer-chunk ring (ring_mode)
  KvPool ring_{};
  DenseMaps ring_maps_{};
  std::vector<int64_t> ring_owner_;           // chunk sequence number occupying each chunk (-1 free)
  std::vector<cudaEvent_t> ring_start_, ring_done_, ring_free_;
  std::vector<cudaEvent_t> ring_upload_;      // per buf: its last descriptor upload ran
  // per buf mapped descriptor region: tokens[wrows] | rows[wrows] | seqs[layers] | preds[wrows]
  size_t ring_desc_bytes() const {
    return static_cast<size_t>(wrows_) * (4 + sizeof(RowDest) + 4) + cfg_.model.layers * sizeof(AttnSeq);
  }
  int64_t ring_seq_ = 0;                      // next chunk sequence number to hand out
  std::map<int, VStream> vstreams_;
  std::vector<int> vs_order_;                 // stream ids in begin order (the link serves them FIFO)
  int next_vstream_ = 1;
  std::vector<char> vbuf_used_;
  KvPool wbuf_{};                             // [buf][layer][kv-head][tail_cap][d] exact window rows
  // drop tier over the chunk ring: the host pool holds only each slice's
  // dropped rows (compacted); a layer lands in land_[c] and is rebuilt into
  // ring_[c] from the landed rows + the drop tier (expand_dropped on exp_st_)
  KvPool land_{};
  int32_t* kept_all_ = nullptr;               // [slot][layer*n_kv][k] kept positions per request
  std::vector<cudaEvent_t> ring_landed_;
  cudaStream_t exp_st_ = nullptr;
  int32_t* kept_of(int slot) const {
    return kept_all_ + static_cast<size_t>(slot) * cfg_.model.layers * cfg_.model.n_kv * kept_cap_;
  }
  float *xsave_ = nullptr, *sssave_ = nullptr;  // [buf][Wrows][H], [buf][Wrows][H/128]
  int wrows_ = 0;
  AttnSeq* ring_seqs_dev_ = nullptr;          // [layers] per-layer sequence of the range forward
  void* h_ring_ = nullptr;                    // mapped pinned: tokens | rows | seqs | preds
  void* d_hring_ = nullptr;
  double h2d_ms_ = 0.0, h2d_bytes_ = 0.0;
  uint64_t next_xfer_ = 1;
  cudaEvent_t ev_a_ = nullptr, ev_b_ = nullptr;
  double device_ms_ = 0.0;
  int64_t steps_ = 0;
  unsigned long long* attn_trace_ = nullptr;  // VC_ATTN_TRACE diagnostics buffer
};

// Thrown on CUDA failures; vc_api maps it to VC_ERR_CUDA.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ContractViolation : std::logic_error {
  using std::logic_error::logic_error;
};

void check_cuda(cudaError_t e, const char* what);

// Prompt-lookup n-gram proposal: the continuation (<= x tokens) that followed
// the most recent earlier occurrence of the last `ng` tokens of h.
std::vector<int32_t> ngram_proposal(const std::vector<int32_t>& h, int ng, int x);

}  // namespace vc
