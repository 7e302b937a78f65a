// vc_engine.cu -- host side of the B200 decode loop (see vc_engine.hpp).
#include "vc_engine.hpp"
#include "vc_topk.h"

#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <stdexcept>

namespace vc {

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

std::vector<int32_t> ngram_proposal(const std::vector<int32_t>& h, int ng, int x) {
  std::vector<int32_t> out;
  const int n = static_cast<int>(h.size());
  if (ng < 1 || n <= ng) return out;
  for (int j = n - ng - 1; j >= 0; --j) {
    bool hit = true;
    for (int k = 0; k < ng && hit; ++k) hit = h[j + k] == h[n - ng + k];
    if (!hit) continue;
    for (int k = j + ng; k < n && static_cast<int>(out.size()) < x; ++k) out.push_back(h[k]);
    break;
  }
  return out;
}

#define VC_CK(expr) check_cuda((expr), #expr)
#define VC_LAUNCH(expr)           \
  do {                            \
    check_cuda((expr), #expr);    \
    ++launches_;                  \
  } while (0)

namespace {

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
int bucket_rows(int M) {
  if (M <= 64) return (M + 15) / 16 * 16;
  if (M <= 128) return (M + 31) / 32 * 32;
  return (M + 63) / 64 * 64;
}

template <class T>
T* dmalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  check_cuda(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
  // zeroed: tile loads may read past a sequence's last key (masked, but finite)
  check_cuda(cudaMemset(p, 0, n * sizeof(T)), "cudaMemset");
  // the memset runs on the legacy stream, which the engine's non-blocking
  // streams do not order against (a weight upload into a fresh staging
  // buffer raced it): finish it before the buffer is handed out
  check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  return static_cast<T*>(p);
}

// Synthetic prefix KV, bit-identical with tests/oracle_data.py.
// i0: element offset of slice 0 in the request's [slice][pos][c] order (a
// one-layer chunk synthesises its slices with the values of the whole request).
__global__ void synth_kv_kernel(uint16_t* kbase, uint16_t* vbase, int cap, int n_ctx, int d,
                                int n_slices, uint64_t seed, float k_norm, float k_out,
                                int outlier_period, size_t i0) {
  const size_t per = static_cast<size_t>(n_ctx) * d;
  const size_t total = per * n_slices;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t slice = i / per, rem = i % per;
    const int c = static_cast<int>(rem % d);
    auto val = [&](uint64_t s, float k) {
      uint64_t x = (i + i0) + 0x9e3779b97f4a7c15ull;
      x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
      x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
      x = x ^ (x >> 31);
      uint64_t h = s ^ x;
      h += 0x9e3779b97f4a7c15ull;
      h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
      h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
      h = h ^ (h >> 31);
      const int sm = static_cast<int>(h & 0xffff) + static_cast<int>((h >> 16) & 0xffff) +
                     static_cast<int>((h >> 32) & 0xffff) + static_cast<int>((h >> 48) & 0xffff);
      return __bfloat16_as_ushort(__float2bfloat16_rn(__fmul_rn(static_cast<float>(sm - 131070), k)));
    };
    const bool outlier = outlier_period > 0 && (c % outlier_period) == outlier_period - 1;
    const size_t dst = slice * static_cast<size_t>(cap) * d + rem;
    kbase[dst] = val(seed, outlier ? k_out : k_norm);
    vbase[dst] = val(seed ^ 0x5555555555555555ull, k_norm);
  }
}

// Step descriptors and results cross PCIe through mapped pinned memory read /
// written by the SMs, never through the copy engine: the copy engine serves
// the KV reloads, and a descriptor copy queued behind a reload stalls the
// whole step until the reload lands (91 ms steps, tools/ce_probe.py).
struct MappedSeg {
  const uint32_t* src;
  uint32_t* dst;
  int words;
};
struct MappedCopy {
  MappedSeg seg[3];
  int n;
};

__global__ void mapped_copy_kernel(MappedCopy c) {
  for (int s = 0; s < c.n; ++s) {
    const MappedSeg g = c.seg[s];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.words; i += gridDim.x * blockDim.x) g.dst[i] = g.src[i];
  }
}

// A pitched copy issued as several smaller copies of `rows_per_copy` rows.
// The copy engine runs one copy call to completion before it serves another
// stream's copy: a step's tiny input H2D queued behind a 4.29 GB reload
// waited the whole 77 ms (tools/ce_probe.py); behind a one-layer chunk it
// waits microseconds.
cudaError_t copy2d_chunked(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                           cudaMemcpyKind kind, cudaStream_t st, size_t rows_per_copy) {
  for (size_t r = 0; r < height; r += rows_per_copy) {
    const size_t h = std::min(rows_per_copy, height - r);
    const cudaError_t e = cudaMemcpy2DAsync(static_cast<uint8_t*>(dst) + r * dpitch, dpitch,
                                            static_cast<const uint8_t*>(src) + r * spitch, spitch, width, h, kind, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

void Engine::check_d2h() const { check_cuda(cudaStreamSynchronize(d2h_st_), "host pool commit"); }

uint16_t* Engine::host_pool_k(int slot) const {
  if (!host_k_ || resident(slot)) return nullptr;
  const auto& m = cfg_.model;
  return host_k_ + static_cast<size_t>(slot - cfg_.resident_slots) * m.layers * m.n_kv * full_.cap * m.d;
}
uint16_t* Engine::host_pool_v(int slot) const {
  if (!host_v_ || resident(slot)) return nullptr;
  const auto& m = cfg_.model;
  return host_v_ + static_cast<size_t>(slot - cfg_.resident_slots) * m.layers * m.n_kv * full_.cap * m.d;
}

size_t Engine::full_kv_bytes_per_token() const {
  const auto& m = cfg_.model;
  return static_cast<size_t>(m.layers) * m.n_kv * m.d * 2 * 2;
}

Engine::Engine(const EngineConfig& cfg, int device) : cfg_(cfg), device_(device) {
  const auto& m = cfg_.model;
  if (cfg_.resident_slots < 0 || cfg_.resident_slots > cfg_.max_slots)
    throw ContractViolation("resident_slots out of [0, max_slots]");
  if (cfg_.resident_slots > 0 && cfg_.full_tier != 1)
    throw ContractViolation("resident_slots is a placement of the host tier (full_tier 1)");
  if (cfg_.ring_chunks < 0 || (cfg_.ring_chunks > 0 && cfg_.full_tier != 1))
    throw ContractViolation("ring_chunks is a staging mode of the host tier (full_tier 1)");
  if (cfg_.ring_chunks > 0 &&
      (cfg_.ring_chunks < 2 || cfg_.max_streams < 1 || cfg_.tp_size > 1 ||
       (cfg_.quant_bits == 0 && !(cfg_.drop_ratio > 0.0 && cfg_.drop_window == 0 && cfg_.drop_score == 0))))
    throw ContractViolation(
        "ring_chunks: needs >= 2 chunks, max_streams >= 1, no TP, and the quantised tier or the drop-topk tier "
        "(offline, key-norm scores)");
  if (cfg_.full_tier == 1 && cfg_.ring_chunks == 0 &&
      cfg_.resident_slots + (cfg_.resident_slots < cfg_.max_slots ? 1 : 0) > cfg_.n_stage)
    throw ContractViolation("n_stage must hold every resident slot plus one rotating staging slot");
  if (cfg_.ring_chunks > 0 && cfg_.n_stage < cfg_.resident_slots)
    throw ContractViolation("n_stage must hold every resident slot");
  if (m.n_q % m.n_kv != 0 || (m.d != 64 && m.d != 128)) throw ContractViolation("unsupported head geometry");
  if (cfg_.quant_bits != 0 && cfg_.quant_bits != 2 && cfg_.quant_bits != 4)
    throw ContractViolation("quant_bits must be 0, 2 or 4");
  if (cfg_.drop_ratio < 0.0 || cfg_.drop_ratio >= 1.0) throw ContractViolation("drop_ratio must be in [0, 1)");
  if (cfg_.drop_ratio > 0.0 && cfg_.quant_bits != 0)
    throw ContractViolation("token-dropping and quantising compressors are exclusive");  // compressor.cpp:245-254
  if (cfg_.drop_score != 0 && cfg_.drop_score != 1) throw ContractViolation("drop_score must be 0 (key norm) or 1 (SnapKV)");
  if (cfg_.drop_score == 1 && (cfg_.full_tier != 0 || cfg_.snap_pool < 1 || cfg_.snap_recent < 0 ||
                               m.n_q / m.n_kv > 8))
    throw ContractViolation("SnapKV scores need the HBM full tier, snap_pool >= 1, snap_recent >= 0, n_rep <= 8");
  VC_CK(cudaSetDevice(device_));
  VC_CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  VC_CK(cudaStreamCreateWithFlags(&copy_st_, cudaStreamNonBlocking));
  VC_CK(cudaStreamCreateWithFlags(&d2h_st_, cudaStreamNonBlocking));
  VC_CK(cudaEventCreateWithFlags(&ev_commit_, cudaEventDisableTiming));
  VC_CK(cudaEventCreateWithFlags(&ev_d2h_, cudaEventDisableTiming));
  VC_CK(cudaEventCreate(&ev_a_));
  VC_CK(cudaEventCreate(&ev_b_));
  alloc_all();
  seqs_.resize(cfg_.max_slots);
  if (std::getenv("VC_ATTN_TRACE")) attn_trace_ = dmalloc<unsigned long long>(3 * 8192);
}

Engine::~Engine() {
  cudaSetDevice(device_);
  cudaStreamSynchronize(st_);
  cudaStreamSynchronize(copy_st_);
  cudaStreamSynchronize(d2h_st_);
  for (auto& [k, g] : graphs_) cudaGraphExecDestroy(g);
  for (auto& [k, x] : xfers_) {
    cudaEventDestroy(x.start);
    cudaEventDestroy(x.done);
  }
  for (auto& [k, v] : vstreams_)
    if (v.ev_final) cudaEventDestroy(v.ev_final);
  for (auto* evs : {&ring_start_, &ring_done_, &ring_free_, &ring_upload_, &ring_landed_})
    for (cudaEvent_t e : *evs) cudaEventDestroy(e);
  if (exp_st_) cudaStreamDestroy(exp_st_);
  for (void* p : {static_cast<void*>(land_.k), static_cast<void*>(land_.v), static_cast<void*>(kept_all_),
                  static_cast<void*>(pack_overflow_), static_cast<void*>(pack_stage_)})
    if (p) cudaFree(p);
  for (void* p : {static_cast<void*>(ring_.k), static_cast<void*>(ring_.v), static_cast<void*>(wbuf_.k),
                  static_cast<void*>(wbuf_.v), static_cast<void*>(xsave_), static_cast<void*>(sssave_),
                  static_cast<void*>(ring_seqs_dev_)})
    if (p) cudaFree(p);
  if (h_ring_) cudaFreeHost(h_ring_);
  void* ptrs[] = {weight_blob_, rope_cos_, rope_sin_, full_.k, full_.v, stage_.k, stage_.v,
                  quant_.rec, quant_.ktail, quant_.vtail, drop_.k, drop_.v, score_buf_, score_w_, kept_buf_,
                  snap_logits_, snap_ms_, obs_q_, attn_trace_,
                  tp_y_, tp_g_,
                  x_, xn_, qkv_, attn_, act_, gws_.partial, gws_.counters, ss_part_, logits_,
                  tok_in_, tok_out_, part_.o, part_.ml, rows_dev_, seqs_dev_, jobs_dev_};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (host_k_) cudaFreeHost(host_k_);
  if (host_v_) cudaFreeHost(host_v_);
  prefix_drop();
  if (h_desc_) cudaFreeHost(h_desc_);
  if (h_out_) cudaFreeHost(h_out_);
  cudaEventDestroy(ev_a_);
  cudaEventDestroy(ev_b_);
  cudaEventDestroy(ev_commit_);
  cudaEventDestroy(ev_d2h_);
  cudaStreamDestroy(st_);
  cudaStreamDestroy(copy_st_);
  cudaStreamDestroy(d2h_st_);
}

void Engine::attention_probe(int slot, int layer, int mode, const uint16_t* q_dev, int n_rows,
                             int kv_len, uint16_t* out_host) {
  const auto& m = cfg_.model;
  const SeqState& s = seqs_.at(slot);
  if (n_rows < 1 || n_rows > Mmax_) throw ContractViolation("probe: bad n_rows");
  AttnShape as;
  as.layers = m.layers;
  as.n_kv = m.n_kv;
  as.n_rep = m.n_q / m.n_kv;
  as.d = m.d;
  as.q_stride = m.n_q * m.d;
  as.out_stride = m.n_q * m.d;
  as.out_mp = 0;
  as.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(m.d)));
  as.draft_warps = draft_warps_;
  as.draft_min_tasks = draft_min_tasks_;
  AttnSeq a{};
  a.slot = cfg_.full_tier == 1 && mode != 1 ? 0 : slot;
  a.row0 = 0;
  a.n_rows = n_rows;
  a.kv_len = kv_len;
  a.n_groups = s.n_groups;
  a.tail_len = s.tail_committed;
  a.part0 = 0;
  AttnSeq* h = reinterpret_cast<AttnSeq*>(h_desc_);
  *h = a;
  VC_CK(cudaMemcpyAsync(seqs_dev_, h, sizeof(AttnSeq), cudaMemcpyHostToDevice, st_));
  if (mode == 1) {
    if (n_rows != 1) throw ContractViolation("probe: draft mode takes one row");
    VC_LAUNCH(draft_attention_quant(as, quant_, layer, q_dev, seqs_dev_, 1, max_chunks_q_,
                                    cfg_.quant_bits, part_, st_));
    VC_LAUNCH(attention_combine(as, seqs_dev_, 1, max_chunks_q_, 1, 0, part_, attn_, st_));
  } else {
    const KvPool pool = cfg_.full_tier == 0 ? full_ : stage_;
    DenseMaps maps = dense_maps_;
    if (!make_q_map(&maps, q_dev, m.d, m.n_q, n_rows, m.n_q * m.d, m.n_q / m.n_kv))
      throw ContractViolation("probe: cannot encode the query tensor map");
    VC_LAUNCH(dense_attention(as, pool, maps, layer, seqs_dev_, 1, max_chunks_d_, n_rows, part_, st_));
    VC_LAUNCH(attention_combine(as, seqs_dev_, 1, max_chunks_d_, n_rows, 1, part_, attn_, st_));
  }
  VC_CK(cudaMemcpyAsync(out_host, attn_, static_cast<size_t>(n_rows) * m.n_q * m.d * 2,
                        cudaMemcpyDeviceToHost, st_));
  VC_CK(cudaStreamSynchronize(st_));
}

void Engine::alloc_all() {
  const auto& m = cfg_.model;
  const int L = m.layers, H = m.hidden, F = m.ffn, V = m.vocab, d = m.d;
  const int qkv_n = (m.n_q + 2 * m.n_kv) * d;
  // ---- weights: one blob, 256-B aligned tensors --------------------------
  std::vector<size_t> sizes;
  auto add = [&](size_t elems) { sizes.push_back(round_up(elems * 2, 256)); };
  add(static_cast<size_t>(V) * H);
  for (int l = 0; l < L; ++l) {
    add(H);
    add(static_cast<size_t>(qkv_n) * H);
    add(static_cast<size_t>(H) * m.n_q * d);
    add(H);
    add(static_cast<size_t>(2) * F * H);
    add(static_cast<size_t>(H) * F);
  }
  add(H);
  add(static_cast<size_t>(V) * H);
  size_t total = 0;
  for (size_t s : sizes) total += s;
  weight_bytes_ = total;
  VC_CK(cudaMalloc(&weight_blob_, total));
  uint8_t* p = static_cast<uint8_t*>(weight_blob_);
  size_t idx = 0;
  auto take = [&]() {
    uint16_t* r = reinterpret_cast<uint16_t*>(p);
    p += sizes[idx++];
    return r;
  };
  w_.embed = take();
  for (int l = 0; l < L; ++l) {
    w_.attn_norm.push_back(take());
    w_.wqkv.push_back(take());
    w_.wo.push_back(take());
    w_.mlp_norm.push_back(take());
    w_.wgu.push_back(take());
    w_.wd.push_back(take());
  }
  w_.final_norm = take();
  w_.lm_head = take();

  // ---- rope tables (double math, rounded once; same formula as the oracle)
  const int cap = static_cast<int>(round_up(cfg_.max_ctx + cfg_.max_x + 2, VC_QGROUP));
  {
    const int half = d / 2;
    std::vector<float> c(static_cast<size_t>(cap) * half), s(c.size());
    for (int pos = 0; pos < cap; ++pos)
      for (int i = 0; i < half; ++i) {
        const double inv = std::pow(static_cast<double>(m.rope_theta), -2.0 * i / d);
        const double a = static_cast<double>(pos) * inv;
        c[static_cast<size_t>(pos) * half + i] = static_cast<float>(std::cos(a));
        s[static_cast<size_t>(pos) * half + i] = static_cast<float>(std::sin(a));
      }
    rope_cos_ = dmalloc<float>(c.size());
    rope_sin_ = dmalloc<float>(s.size());
    VC_CK(cudaMemcpyAsync(rope_cos_, c.data(), c.size() * 4, cudaMemcpyHostToDevice, st_));
    VC_CK(cudaMemcpyAsync(rope_sin_, s.data(), s.size() * 4, cudaMemcpyHostToDevice, st_));
    VC_CK(cudaStreamSynchronize(st_));
  }
  // ---- KV tiers ------------------------------------------------------------
  const size_t slices = static_cast<size_t>(cfg_.max_slots) * L * m.n_kv;
  const size_t slice_elems = static_cast<size_t>(cap) * d;
  if (cfg_.full_tier == 0) {
    full_.cap = cap;
    full_.k = dmalloc<uint16_t>(slices * slice_elems);
    full_.v = dmalloc<uint16_t>(slices * slice_elems);
  } else {
    full_.cap = cap;  // geometry of the host pool
    // the host pool holds the offloaded slots only (resident slots live in HBM)
    const size_t host_slices = static_cast<size_t>(cfg_.max_slots - cfg_.resident_slots) * L * m.n_kv;
    const size_t bytes = host_slices * slice_elems * 2;
    if (bytes > 0) {
      VC_CK(cudaHostAlloc(reinterpret_cast<void**>(&host_k_), bytes, cudaHostAllocDefault));
      VC_CK(cudaHostAlloc(reinterpret_cast<void**>(&host_v_), bytes, cudaHostAllocDefault));
    }
    const size_t st_slices = static_cast<size_t>(cfg_.n_stage) * L * m.n_kv;
    stage_.cap = cap;
    stage_.k = dmalloc<uint16_t>(st_slices * slice_elems);
    stage_.v = dmalloc<uint16_t>(st_slices * slice_elems);
    if (ring_mode()) {
      // ring_chunks one-layer chunks for streamed verifies + 2 admission chunks
      const int nch = cfg_.ring_chunks + 2;
      ring_.cap = cap;
      ring_.k = dmalloc<uint16_t>(static_cast<size_t>(nch) * m.n_kv * slice_elems);
      ring_.v = dmalloc<uint16_t>(static_cast<size_t>(nch) * m.n_kv * slice_elems);
      ring_owner_.assign(nch, -1);
      for (int i = 0; i < nch; ++i) {
        cudaEvent_t a, b, c;
        VC_CK(cudaEventCreate(&a));
        VC_CK(cudaEventCreate(&b));
        VC_CK(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
        ring_start_.push_back(a);
        ring_done_.push_back(b);
        ring_free_.push_back(c);
      }
    }
  }
  tail_cap_ = static_cast<int>(round_up(VC_QGROUP + cfg_.max_x + 2, 8));
  if (cfg_.quant_bits > 0) {
    const int capq = cfg_.max_ctx / VC_QGROUP * VC_QGROUP;
    quant_.cap = capq;
    quant_.tail_cap = tail_cap_;
    quant_.rec = dmalloc<uint32_t>(slices * (capq / VC_QGROUP) * quant_record_words(d, cfg_.quant_bits));
    quant_.ktail = dmalloc<uint16_t>(slices * tail_cap_ * d);
    quant_.vtail = dmalloc<uint16_t>(slices * tail_cap_ * d);
    // draft partial slots per (sequence, head): a warp takes >= draft_min_tasks_
    // groups, so at most ceil(groups / min) + 1 warps touch one head
    const int capg = capq / VC_QGROUP;
    draft_min_tasks_ = std::max(4, (capg + 479) / 480);
    max_chunks_q_ = (capg + draft_min_tasks_ - 1) / draft_min_tasks_ + 1;
    draft_warps_ = draft_quant_warps(d, cfg_.quant_bits, m.n_q / m.n_kv);

    if (draft_warps_ <= 0) throw ContractViolation("no draft-attention kernel for this head shape");
  }
  if (drop_mode()) {
    // kept tokens + up to kDropAppend exact appended tokens + the draft window
    const int kDropAppend = cfg_.drop_window > 0 ? 2 * cfg_.drop_window + cfg_.max_x + 2 : 4096;
    const int kmax = static_cast<int>(std::ceil(cfg_.drop_ratio * cfg_.max_ctx)) + 1;
    drop_.cap = static_cast<int>(round_up(static_cast<size_t>(kmax) + kDropAppend + cfg_.max_x + 2, 128));
    drop_.k = dmalloc<uint16_t>(slices * static_cast<size_t>(drop_.cap) * d);
    drop_.v = dmalloc<uint16_t>(slices * static_cast<size_t>(drop_.cap) * d);
    max_chunks_x_ = (drop_.cap + VC_DENSE_CHUNK - 1) / VC_DENSE_CHUNK;
    score_buf_ = dmalloc<float>(static_cast<size_t>(L) * m.n_kv * cap);
    kept_buf_ = dmalloc<int32_t>(static_cast<size_t>(L) * m.n_kv * kmax);
    kept_cap_ = kmax;
    score_w_ = dmalloc<float>(d);
    std::vector<float> ones(d, 1.0f);  // score = L1 norm of the (post-RoPE) key
    VC_CK(cudaMemcpy(score_w_, ones.data(), d * 4, cudaMemcpyHostToDevice));
    if (cfg_.drop_score == 1) {
      snap_logits_ = dmalloc<float>(static_cast<size_t>(m.n_q) * cap);
      snap_ms_ = dmalloc<float>(static_cast<size_t>(m.n_q) * 2);
      obs_q_ = dmalloc<uint16_t>(static_cast<size_t>(L) * m.n_q * d);
    }
  }
  max_chunks_d_ = (cap + VC_DENSE_CHUNK - 1) / VC_DENSE_CHUNK;
  // ---- activations ---------------------------------------------------------
  Mmax_ = static_cast<int>(round_up(draft_rows_max() + cfg_.max_verify * (cfg_.max_x + 1), 64));
  x_ = dmalloc<float>(static_cast<size_t>(Mmax_) * H);
  // tiled GEMM inputs carry 128 rows of slack (the last NT block may overrun Mp)
  xn_ = dmalloc<uint16_t>(static_cast<size_t>(Mmax_ + 128) * (H > F ? H : F));
  qkv_ = dmalloc<uint16_t>(static_cast<size_t>(Mmax_) * qkv_n);
  attn_ = dmalloc<uint16_t>(static_cast<size_t>(Mmax_ + 128) * m.n_q * d);
  // TMA tensor maps of the dense attention path (K/V pool of each tier + the q heads)
  {
    const KvPool& dp = cfg_.full_tier == 0 ? full_ : stage_;
    const size_t dslices = cfg_.full_tier == 0 ? slices : static_cast<size_t>(cfg_.n_stage) * L * m.n_kv;
    if ((dslices > 0 && !make_kv_maps(&dense_maps_, dp, dslices, d)) ||
        !make_q_map(&dense_maps_, qkv_, d, m.n_q + 2 * m.n_kv, Mmax_, qkv_n, m.n_q / m.n_kv))
      throw ContractViolation("dense attention: cannot encode TMA tensor maps for this shape");
    if (ring_mode() &&
        (!make_kv_maps(&ring_maps_, ring_, static_cast<size_t>(cfg_.ring_chunks + 2) * m.n_kv, d) ||
         !make_q_map(&ring_maps_, qkv_, d, m.n_q + 2 * m.n_kv, Mmax_, qkv_n, m.n_q / m.n_kv)))
      throw ContractViolation("chunk ring: cannot encode TMA tensor maps for this shape");
    if (drop_mode() && (!make_kv_maps(&drop_maps_, drop_, slices, d) ||
                        !make_q_map(&drop_maps_, qkv_, d, m.n_q + 2 * m.n_kv, Mmax_, qkv_n, m.n_q / m.n_kv)))
      throw ContractViolation("drop tier: cannot encode TMA tensor maps for this shape");
  }
  act_ = dmalloc<uint16_t>(static_cast<size_t>(Mmax_ + 128) * F);
  {
    size_t pf = 0;
    for (int mm : {16, 32, 64, 128}) {
      pf = std::max(pf, gemm_partial_floats(mm, qkv_n, H));
      pf = std::max(pf, gemm_partial_floats(mm, H, m.n_q * d));
      pf = std::max(pf, gemm_partial_floats(mm, 2 * F, H));
      pf = std::max(pf, gemm_partial_floats(mm, H, F));
      pf = std::max(pf, gemm_partial_floats(mm, V, H));
    }
    gws_.partial_floats = pf;
    gws_.partial = dmalloc<float>(pf);
    gws_.n_counters = std::max(std::max(qkv_n, H), std::max(2 * F, V)) / 128 + 1;
    gws_.counters = dmalloc<int>(gws_.n_counters);
  }
  ss_part_ = dmalloc<float>(static_cast<size_t>(Mmax_) * (H / 128));
  if (cfg_.tp_size > 1) {
    tp_y_ = dmalloc<float>(static_cast<size_t>(Mmax_) * H);
    tp_g_ = dmalloc<float>(static_cast<size_t>(cfg_.tp_size) * Mmax_ * H);
  }
  logits_ = dmalloc<float>(static_cast<size_t>(Mmax_) * V);
  tok_in_ = dmalloc<int32_t>(Mmax_);
  tok_out_ = dmalloc<int32_t>(Mmax_);
  const size_t prow_draft =
      static_cast<size_t>(draft_rows_max() + 4) *
      (drop_mode() ? max_chunks_x_ : draft_parts_per_seq(max_chunks_q_, tail_cap_));
  const size_t prow_dense = static_cast<size_t>(Mmax_) * max_chunks_d_;
  const size_t prow = (prow_draft + prow_dense) * m.n_q;
  part_.o = dmalloc<float>(prow * d);
  part_.ml = dmalloc<float>(prow * 2);
  rows_dev_ = dmalloc<RowDest>(Mmax_);
  const int n_seq_max = 2 * (draft_rows_max() + 4) + cfg_.max_verify + 4;
  seqs_dev_ = dmalloc<AttnSeq>(n_seq_max);
  jobs_dev_ = dmalloc<QuantJob>(static_cast<size_t>(L) * m.n_kv);
  desc_bytes_ = Mmax_ * sizeof(int32_t) + Mmax_ * sizeof(RowDest) + n_seq_max * sizeof(AttnSeq) +
                static_cast<size_t>(L) * m.n_kv * sizeof(QuantJob);
  VC_CK(cudaHostAlloc(&h_desc_, desc_bytes_, cudaHostAllocMapped));
  VC_CK(cudaHostAlloc(reinterpret_cast<void**>(&h_out_), Mmax_ * sizeof(int32_t), cudaHostAllocMapped));
  VC_CK(cudaHostGetDevicePointer(&d_hdesc_, h_desc_, 0));
  VC_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_hout_), h_out_, 0));
  if (ring_mode()) {  // streamed-verify state: exact window rows, carried hidden state, descriptors
    const int nb = cfg_.max_streams;
    wrows_ = bucket_rows(cfg_.max_x + 1);
    wbuf_.cap = tail_cap_;
    wbuf_.k = dmalloc<uint16_t>(static_cast<size_t>(nb) * L * m.n_kv * tail_cap_ * d);
    wbuf_.v = dmalloc<uint16_t>(static_cast<size_t>(nb) * L * m.n_kv * tail_cap_ * d);
    xsave_ = dmalloc<float>(static_cast<size_t>(nb) * wrows_ * H);
    sssave_ = dmalloc<float>(static_cast<size_t>(nb) * wrows_ * (H / 128));
    ring_seqs_dev_ = dmalloc<AttnSeq>(L);
    VC_CK(cudaHostAlloc(&h_ring_, static_cast<size_t>(nb) * ring_desc_bytes(), cudaHostAllocMapped));
    VC_CK(cudaHostGetDevicePointer(&d_hring_, h_ring_, 0));
    vbuf_used_.assign(nb, 0);
    for (int i = 0; i < nb; ++i) {
      cudaEvent_t e;
      VC_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ring_upload_.push_back(e);
    }
    if (host_pack_on()) {
      pack_overflow_ = dmalloc<int>(1);
      pack_stage_ = dmalloc<uint8_t>(4 * static_cast<size_t>(L) * m.n_kv * packed_block_bytes(d));
    }
    if (drop_mode() || host_pack_on()) {
      const size_t chunk = static_cast<size_t>(m.n_kv) * ring_.cap * d;
      land_.cap = ring_.cap;
      land_.k = dmalloc<uint16_t>(static_cast<size_t>(cfg_.ring_chunks) * chunk);
      land_.v = dmalloc<uint16_t>(static_cast<size_t>(cfg_.ring_chunks) * chunk);
    }
    if (drop_mode()) {
      kept_all_ = dmalloc<int32_t>(static_cast<size_t>(cfg_.max_slots) * L * m.n_kv * kept_cap_);
    }
    if (drop_mode() || host_pack_on()) {
      for (int i = 0; i < cfg_.ring_chunks; ++i) {
        cudaEvent_t e;
        VC_CK(cudaEventCreate(&e));
        ring_landed_.push_back(e);
      }
      VC_CK(cudaStreamCreateWithFlags(&exp_st_, cudaStreamNonBlocking));
    }
  }
}

void Engine::attach_collective(std::unique_ptr<Collective> c) {
  // tp_size 1 with a collective runs the TP residual path over a one-rank
  // group (bit-identical to the fused epilogue; exercises the collective)
  if (!tp_y_) {
    const size_t n = static_cast<size_t>(Mmax_) * cfg_.model.hidden;
    tp_y_ = dmalloc<float>(n);
    tp_g_ = dmalloc<float>(static_cast<size_t>(cfg_.tp_size) * n);
  }
  coll_ = std::move(c);
  for (auto& [k, g] : graphs_) cudaGraphExecDestroy(g);  // captured without the collective
  graphs_.clear();
  launches_per_graph_.clear();
}

double Engine::collective_bench(int rows, int reps) {
  if (!coll_) throw ContractViolation("collective_bench: no collective attached");
  if (rows < 1 || rows > Mmax_ || reps < 1) throw ContractViolation("collective_bench: bad rows/reps");
  const int H = cfg_.model.hidden;
  float total = 0.f;
  for (int r = 0; r <= reps; ++r) {  // r = 0 is warm-up
    VC_CK(cudaEventRecord(ev_a_, st_));
    coll_->all_gather(tp_y_, tp_g_, static_cast<size_t>(rows) * H, st_);
    VC_LAUNCH(tp_residual(x_, tp_g_, cfg_.tp_size, rows, H, ss_part_, st_));
    VC_CK(cudaEventRecord(ev_b_, st_));
    VC_CK(cudaEventSynchronize(ev_b_));
    float ms = 0.f;
    VC_CK(cudaEventElapsedTime(&ms, ev_a_, ev_b_));
    if (r > 0) total += ms;
  }
  return 1e3 * total / reps;
}

// ---------------------------------------------------------------- weights
void Engine::init_weights_random(uint64_t seed, float stddev, float resid_std, float q_std) {
  const auto& m = cfg_.model;
  const int L = m.layers, H = m.hidden, F = m.ffn, V = m.vocab, d = m.d;
  const int qkv_n = (m.n_q + 2 * m.n_kv) * d;
  const float k = static_cast<float>(stddev / (65536.0 * std::sqrt(1.0 / 3.0)));
  // residual-branch outputs (o_proj, down_proj) may use a smaller std
  // (GPT-2 style std / sqrt(2 L)); resid_std <= 0 keeps stddev
  const float kr = resid_std > 0.f ? static_cast<float>(resid_std / (65536.0 * std::sqrt(1.0 / 3.0))) : k;
  uint64_t off = 0;
  auto fill_k = [&](uint16_t* p, size_t n, float kk) {
    VC_LAUNCH(fill_normal_bf16(p, n, seed, off, kk, st_));
    off += n;
  };
  auto fill = [&](uint16_t* p, size_t n) { fill_k(p, n, k); };
  const uint16_t one = 0x3f80;
  fill(w_.embed, static_cast<size_t>(V) * H);
  for (int l = 0; l < L; ++l) {
    VC_LAUNCH(fill_const_bf16(w_.attn_norm[l], H, one, st_));
    if (q_std > 0.f) {
      // the Q projection rows are the first n_q*d rows = a contiguous prefix
      // of the tiled layout (blocks are n-tile major)
      const float kq = static_cast<float>(q_std / (65536.0 * std::sqrt(1.0 / 3.0)));
      const size_t nq_elems = static_cast<size_t>(m.n_q) * d * H;
      fill_k(w_.wqkv[l], nq_elems, kq);
      fill(w_.wqkv[l] + nq_elems, static_cast<size_t>(qkv_n) * H - nq_elems);
    } else {
      fill(w_.wqkv[l], static_cast<size_t>(qkv_n) * H);
    }
    fill_k(w_.wo[l], static_cast<size_t>(H) * m.n_q * d, kr);
    VC_LAUNCH(fill_const_bf16(w_.mlp_norm[l], H, one, st_));
    fill(w_.wgu[l], static_cast<size_t>(2) * F * H);
    fill_k(w_.wd[l], static_cast<size_t>(H) * F, kr);
  }
  VC_LAUNCH(fill_const_bf16(w_.final_norm, H, one, st_));
  fill(w_.lm_head, static_cast<size_t>(V) * H);
  VC_CK(cudaStreamSynchronize(st_));
}

void Engine::load_weights(const uint16_t* embed, const uint16_t* const* attn_norm,
                          const uint16_t* const* wqkv, const uint16_t* const* wo,
                          const uint16_t* const* mlp_norm, const uint16_t* const* wgate,
                          const uint16_t* const* wup, const uint16_t* const* wdown,
                          const uint16_t* final_norm, const uint16_t* lm_head) {
  const auto& m = cfg_.model;
  const int L = m.layers, H = m.hidden, F = m.ffn, V = m.vocab, d = m.d;
  const int qkv_n = (m.n_q + 2 * m.n_kv) * d;
  // Every upload is stream-ordered on st_: a plain cudaMemcpy from pageable
  // memory may return before its DMA lands, and st_ does not synchronise with
  // the legacy default stream, so the retile kernel could read stale bytes.
  auto up = [&](uint16_t* dst, const uint16_t* src, size_t n) {
    VC_CK(cudaMemcpyAsync(dst, src, n * 2, cudaMemcpyHostToDevice, st_));
  };
  // GEMM weights: logical [N][K] -> staging -> tiled layout (vc_tiled.cuh)
  const size_t max_elems = std::max(std::max(static_cast<size_t>(V) * H, static_cast<size_t>(2) * F * H),
                                    std::max(static_cast<size_t>(qkv_n) * H, static_cast<size_t>(H) * F));
  uint16_t* tmp = dmalloc<uint16_t>(max_elems);
  auto up_tiled = [&](uint16_t* dst, const uint16_t* src, int N, int K) {
    up(tmp, src, static_cast<size_t>(N) * K);
    VC_LAUNCH(retile_weight(tmp, N, K, dst, st_));
  };
  up(w_.embed, embed, static_cast<size_t>(V) * H);
  std::vector<uint16_t> gu(static_cast<size_t>(2) * F * H);
  for (int l = 0; l < L; ++l) {
    up(w_.attn_norm[l], attn_norm[l], H);
    up_tiled(w_.wqkv[l], wqkv[l], qkv_n, H);
    up_tiled(w_.wo[l], wo[l], H, m.n_q * d);
    up(w_.mlp_norm[l], mlp_norm[l], H);
    // interleave gate/up rows: row 2j = gate_j, row 2j+1 = up_j
    for (int j = 0; j < F; ++j) {
      std::memcpy(&gu[static_cast<size_t>(2 * j) * H], wgate[l] + static_cast<size_t>(j) * H, H * 2);
      std::memcpy(&gu[static_cast<size_t>(2 * j + 1) * H], wup[l] + static_cast<size_t>(j) * H, H * 2);
    }
    up_tiled(w_.wgu[l], gu.data(), 2 * F, H);
    up_tiled(w_.wd[l], wdown[l], H, F);
  }
  up(w_.final_norm, final_norm, H);
  up_tiled(w_.lm_head, lm_head, V, H);
  VC_CK(cudaStreamSynchronize(st_));
  cudaFree(tmp);
}

// --------------------------------------------------------------- requests
void Engine::add_request_synthetic(int slot, int n_ctx, int32_t pending, uint64_t seed,
                                   int outlier_channels, float outlier_scale) {
  if (slot < 0 || slot >= cfg_.max_slots) throw ContractViolation("slot out of range");
  if (n_ctx < 0 || n_ctx + cfg_.max_x + 2 > full_.cap) throw ContractViolation("context exceeds capacity");
  const auto& m = cfg_.model;
  const int n_slices = m.layers * m.n_kv;
  const float k_norm = static_cast<float>(1.0 / (65536.0 * std::sqrt(1.0 / 3.0)));
  const float k_out = static_cast<float>(outlier_scale / (65536.0 * std::sqrt(1.0 / 3.0)));
  const int period = outlier_channels > 0 ? m.d / outlier_channels : 0;
  if (ring_mode() && !resident(slot)) {
    // offloaded, chunk ring: synthesise one layer at a time into the two
    // admission chunks and copy each into the host pool (no whole-request
    // staging slot)
    const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
    const size_t pitch = slice_elems * 2;
    const size_t width = static_cast<size_t>(n_ctx) * m.d * 2;
    check_d2h();  // earlier commits into this slot's host rows land first
    auto synth_layer = [&](int l, int c) {
      const size_t total = static_cast<size_t>(n_ctx) * m.d * m.n_kv;
      const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 32));
      synth_kv_kernel<<<grid, 256, 0, st_>>>(ring_.k + static_cast<size_t>(c) * m.n_kv * slice_elems,
                                             ring_.v + static_cast<size_t>(c) * m.n_kv * slice_elems, full_.cap, n_ctx,
                                             m.d, m.n_kv, seed, k_norm, k_out, period,
                                             static_cast<size_t>(l) * m.n_kv * n_ctx * m.d);
      VC_CK(cudaGetLastError());
      ++launches_;
    };
    if (host_pack_on() && n_ctx > 0) {
      // lossless packing: pass 1 finds the blocks every layer packs (a block
      // with too many escapes is stored raw, and so is everything after it),
      // pass 2 stores packed blocks + raw rows
      const int nb = (n_ctx + VC_QGROUP - 1) / VC_QGROUP;
      int P = nb;
      const int ca = cfg_.ring_chunks, cb = cfg_.ring_chunks + 1;
      for (int l = 0; l < m.layers; ++l) {
        synth_layer(l, ca);
        VC_CK(cudaMemsetAsync(pack_overflow_, 0, sizeof(int), st_));
        for (int kv = 0; kv < 2; ++kv)
          VC_CK(pack_blocks((kv ? ring_.v : ring_.k) + static_cast<size_t>(ca) * m.n_kv * slice_elems, slice_elems, 0,
                            n_ctx, nb, m.n_kv, m.d,
                            reinterpret_cast<uint8_t*>((kv ? ring_.v : ring_.k) + static_cast<size_t>(cb) * m.n_kv * slice_elems),
                            pitch, pack_overflow_, st_));
        int f = 0;
        VC_CK(cudaMemcpyAsync(&f, pack_overflow_, sizeof(int), cudaMemcpyDeviceToHost, st_));
        VC_CK(cudaStreamSynchronize(st_));
        if (f > 0) P = std::min(P, f - 1);
      }
      if (cfg_.host_pack >= 2) P = std::min(P, cfg_.host_pack - 1);
      for (int l = 0; l < m.layers; ++l) {
        synth_layer(l, ca);
        host_store_layer(slot, l, ca, cb, n_ctx, P);
      }
      SeqState& s = seqs_[slot];
      s = SeqState{};
      s.live = true;
      s.committed = n_ctx;
      s.pending = pending;
      s.packed_blocks = P;
      scratch_slot_ = -1;
      VC_CK(cudaStreamSynchronize(st_));
      return;
    }
    for (int l = 0; l < m.layers && n_ctx > 0; ++l) {
      const int c = cfg_.ring_chunks + (l & 1);
      uint16_t* kb = ring_.k + static_cast<size_t>(c) * m.n_kv * slice_elems;
      uint16_t* vb = ring_.v + static_cast<size_t>(c) * m.n_kv * slice_elems;
      VC_CK(cudaStreamWaitEvent(st_, ring_free_[c], 0));  // the chunk's previous host copy is done
      const size_t total = static_cast<size_t>(n_ctx) * m.d * m.n_kv;
      const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 32));
      synth_kv_kernel<<<grid, 256, 0, st_>>>(kb, vb, full_.cap, n_ctx, m.d, m.n_kv, seed, k_norm, k_out, period,
                                             static_cast<size_t>(l) * m.n_kv * n_ctx * m.d);
      VC_CK(cudaGetLastError());
      ++launches_;
      VC_CK(cudaEventRecord(ev_commit_, st_));
      VC_CK(cudaStreamWaitEvent(d2h_st_, ev_commit_, 0));
      const size_t o = static_cast<size_t>(l) * m.n_kv * slice_elems;
      VC_CK(cudaMemcpy2DAsync(host_pool_k(slot) + o, pitch, kb, pitch, width, m.n_kv, cudaMemcpyDeviceToHost, d2h_st_));
      VC_CK(cudaMemcpy2DAsync(host_pool_v(slot) + o, pitch, vb, pitch, width, m.n_kv, cudaMemcpyDeviceToHost, d2h_st_));
      VC_CK(cudaEventRecord(ring_free_[c], d2h_st_));
    }
    VC_CK(cudaEventRecord(ev_d2h_, d2h_st_));
    VC_CK(cudaStreamWaitEvent(copy_st_, ev_d2h_, 0));  // later reloads of these rows wait for them
    SeqState& s = seqs_[slot];
    s = SeqState{};
    s.live = true;
    s.committed = n_ctx;
    s.pending = pending;
    scratch_slot_ = -1;
    VC_CK(cudaStreamSynchronize(st_));
    return;
  }
  // tier 1 synthesises into the request's own staging slot (resident) or the
  // scratch staging slot, then D2H into the host pool (offloaded)
  KvPool dst = cfg_.full_tier == 0 ? full_ : stage_;
  const int dslot = cfg_.full_tier == 0 || resident(slot) ? slot : scratch_stage();
  const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
  uint16_t* kb = dst.k + static_cast<size_t>(dslot) * n_slices * slice_elems;
  uint16_t* vb = dst.v + static_cast<size_t>(dslot) * n_slices * slice_elems;
  if (n_ctx > 0) {
    // the staging slot may still be read by an earlier host-pool copy (a
    // previous synthesis or commit on the D2H stream): write it after that
    if (cfg_.full_tier == 1) VC_CK(cudaStreamWaitEvent(st_, ev_d2h_, 0));
    const size_t total = static_cast<size_t>(n_ctx) * m.d * n_slices;
    int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 32));
    synth_kv_kernel<<<grid, 256, 0, st_>>>(kb, vb, full_.cap, n_ctx, m.d, n_slices, seed, k_norm,
                                           k_out, period, 0);
    VC_CK(cudaGetLastError());
    ++launches_;
  }
  SeqState& s = seqs_[slot];
  s = SeqState{};
  s.live = true;
  s.committed = n_ctx;
  s.pending = pending;
  scratch_slot_ = -1;
  if (cfg_.full_tier == 1 && !resident(slot) && n_ctx > 0) {
    scratch_slot_ = slot;
    scratch_stage_used_ = dslot;
    check_d2h();  // earlier commits into this slot's host rows land first
    const size_t pitch = static_cast<size_t>(full_.cap) * m.d * 2;
    const size_t width = static_cast<size_t>(n_ctx) * m.d * 2;
    uint16_t* hk = host_pool_k(slot);
    uint16_t* hv = host_pool_v(slot);
    // the host copy goes on the commit stream (never the compute stream:
    // it would queue behind an in-flight reload); later reloads wait for it
    VC_CK(cudaEventRecord(ev_commit_, st_));
    VC_CK(cudaStreamWaitEvent(d2h_st_, ev_commit_, 0));
    VC_CK(copy2d_chunked(hk, pitch, kb, pitch, width, n_slices, cudaMemcpyDeviceToHost, d2h_st_, m.n_kv));
    VC_CK(copy2d_chunked(hv, pitch, vb, pitch, width, n_slices, cudaMemcpyDeviceToHost, d2h_st_, m.n_kv));
    VC_CK(cudaEventRecord(ev_d2h_, d2h_st_));
    VC_CK(cudaStreamWaitEvent(copy_st_, ev_d2h_, 0));
  }
  VC_CK(cudaStreamSynchronize(st_));
}

void Engine::add_request_kv(int slot, int n_ctx, int32_t pending, const uint16_t* k, const uint16_t* v) {
  if (slot < 0 || slot >= cfg_.max_slots) throw ContractViolation("slot out of range");
  if (n_ctx + cfg_.max_x + 2 > full_.cap) throw ContractViolation("context exceeds capacity");
  const auto& m = cfg_.model;
  const int n_slices = m.layers * m.n_kv;
  const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
  const size_t pitch = slice_elems * 2, spitch = static_cast<size_t>(n_ctx) * m.d * 2;
  if (n_ctx > 0) {
    if (cfg_.full_tier == 0 || resident(slot)) {
      const KvPool& dp = cfg_.full_tier == 0 ? full_ : stage_;
      uint16_t* kb = dp.k + static_cast<size_t>(slot) * n_slices * slice_elems;
      uint16_t* vb = dp.v + static_cast<size_t>(slot) * n_slices * slice_elems;
      VC_CK(cudaMemcpy2DAsync(kb, pitch, k, spitch, spitch, n_slices, cudaMemcpyHostToDevice, st_));
      VC_CK(cudaMemcpy2DAsync(vb, pitch, v, spitch, spitch, n_slices, cudaMemcpyHostToDevice, st_));
    } else {
      check_d2h();  // no commit still writing these host rows
      uint16_t* hk = host_pool_k(slot);
      uint16_t* hv = host_pool_v(slot);
      for (int i = 0; i < n_slices; ++i) {
        std::memcpy(hk + i * slice_elems, k + static_cast<size_t>(i) * n_ctx * m.d, spitch);
        std::memcpy(hv + i * slice_elems, v + static_cast<size_t>(i) * n_ctx * m.d, spitch);
      }
    }
  }
  SeqState& s = seqs_[slot];
  s = SeqState{};
  s.live = true;
  s.committed = n_ctx;
  s.pending = pending;
  VC_CK(cudaStreamSynchronize(st_));
}

void Engine::add_request_prefill(int slot, const int32_t* prompt, int n) {
  if (n < 1) throw ContractViolation("prefill: empty prompt");
  if (cfg_.full_tier != 0) throw ContractViolation("prefill requires the HBM full tier");
  SeqState& s = seqs_[slot];
  s = SeqState{};
  s.live = true;
  s.committed = 0;
  s.pending = prompt[0];
  // feed the prompt through verify-shaped steps of at most max_x+1 rows
  int pos = 0;
  std::vector<int32_t> out;
  while (pos < n - 1) {
    const int len = std::min(n - 1 - pos, cfg_.max_x + 1);
    StepItem it;
    it.slot = slot;
    it.mode = RowMode::Verify;
    it.tokens.assign(prompt + pos, prompt + pos + len);
    run_step({it}, out);
    s.committed += len;
    pos += len;
  }
  s.pending = prompt[n - 1];
}

void Engine::release(int slot) { seqs_.at(slot) = SeqState{}; }

// Quantise groups [g0, g0+ng) of layers [layer0, layer0+layers) of `slot`
// from src: src_slot's slices hold those layers' rows (layers * n_kv slices),
// row r of a slice = absolute position r + origin.
void Engine::quantise_groups(int slot, int g0, int ng, const KvPool& src, int src_slot, int origin,
                             int layer0, int layers) {
  if (ng <= 0) return;
  const auto& m = cfg_.model;
  if (layers < 0) layers = m.layers;
  const int n_slices = layers * m.n_kv;
  QuantJob* jobs = reinterpret_cast<QuantJob*>(static_cast<uint8_t*>(h_desc_) + desc_bytes_ -
                                               static_cast<size_t>(m.layers) * m.n_kv * sizeof(QuantJob));
  const size_t slice_words = static_cast<size_t>(quant_.cap / VC_QGROUP) * quant_record_words(m.d, cfg_.quant_bits);
  for (int i = 0; i < n_slices; ++i) {
    const size_t ss = static_cast<size_t>(src_slot) * n_slices + i;
    const size_t ds = (static_cast<size_t>(slot) * m.layers + layer0) * m.n_kv + i;
    QuantJob j;
    // token 0 of group 0 (may lie before the source rows: only groups >= g0 are read)
    j.k = src.k + ss * static_cast<size_t>(src.cap) * m.d - static_cast<ptrdiff_t>(origin) * m.d;
    j.v = src.v + ss * static_cast<size_t>(src.cap) * m.d - static_cast<ptrdiff_t>(origin) * m.d;
    j.rec = quant_.rec + ds * slice_words;
    j.g0 = g0;
    j.ng = ng;
    jobs[i] = j;
  }
  // the kernel reads the job table straight from mapped pinned memory (no copy engine)
  const QuantJob* jobs_mapped = reinterpret_cast<const QuantJob*>(
      static_cast<const uint8_t*>(d_hdesc_) + (reinterpret_cast<uint8_t*>(jobs) - static_cast<uint8_t*>(h_desc_)));
  VC_LAUNCH(quant_kivi(jobs_mapped, n_slices, ng, m.d, cfg_.quant_bits, st_));
  // the pinned job table is reused by the next call: wait for the copy
  VC_CK(cudaStreamSynchronize(st_));
}

void Engine::compress(int slot) { compress_as(slot, cfg_.drop_ratio, nullptr, 0); }

void Engine::compress_as(int slot, double ratio, const int32_t* kept_host, int k_host) {
  if (cfg_.quant_bits == 0 && !drop_mode()) throw ContractViolation("compress: compressed tier disabled");
  SeqState& s = seqs_.at(slot);
  const auto& m = cfg_.model;
  KvPool src = full_;
  int src_slot = slot;
  if (resident(slot)) {  // the full KV is already in its own staging slot
    src = stage_;
    src_slot = slot;
  } else if (cfg_.full_tier == 1 && scratch_slot_ == slot) {
    // just synthesised: the full KV is still in the scratch staging slot
    src = stage_;
    src_slot = scratch_stage_used_;
  } else if (ring_mode() && drop_mode()) {
    // chunk ring over the drop tier: one layer at a time through the two
    // admission chunks -- score + top-k (or the given kept set), kept rows
    // into the drop tier, and the DROPPED rows compacted back into the host
    // pool: a verify then reloads only (1 - c) of the full KV
    // (analytics.cpp:77-78 charges exactly that) and rebuilds the rest from
    // the drop tier (expand_dropped)
    if (s.drop_T > 0) throw ContractViolation("compress: the host pool already holds only the dropped rows");
    const int T = s.committed;
    const long long k = kept_host ? k_host : std::llround(ratio * static_cast<double>(T));
    if (k < 1) throw ContractViolation("compress: drop ratio retains < 1 token");
    if (k > kept_cap_ || k + cfg_.max_x + 2 > drop_.cap)
      throw ContractViolation("compress: drop tier capacity exceeded (ratio above the engine's drop_ratio)");
    const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
    const size_t pitch = slice_elems * 2;
    const int ca = cfg_.ring_chunks, cb = cfg_.ring_chunks + 1;  // full rows / compacted dropped rows
    uint16_t* kb = ring_.k + static_cast<size_t>(cb) * m.n_kv * slice_elems;
    uint16_t* vb = ring_.v + static_cast<size_t>(cb) * m.n_kv * slice_elems;
    check_d2h();
    VC_CK(cudaStreamSynchronize(st_));
    int32_t* kept = kept_of(slot);
    for (int l = 0; l < m.layers; ++l) {
      const size_t o = static_cast<size_t>(l) * m.n_kv * slice_elems;
      int32_t* kl = kept + static_cast<size_t>(l) * m.n_kv * k;
      VC_CK(cudaMemcpy2DAsync(ring_.k + static_cast<size_t>(ca) * m.n_kv * slice_elems, pitch, host_pool_k(slot) + o,
                              pitch, static_cast<size_t>(T) * m.d * 2, m.n_kv, cudaMemcpyHostToDevice, st_));
      VC_CK(cudaMemcpy2DAsync(ring_.v + static_cast<size_t>(ca) * m.n_kv * slice_elems, pitch, host_pool_v(slot) + o,
                              pitch, static_cast<size_t>(T) * m.d * 2, m.n_kv, cudaMemcpyHostToDevice, st_));
      if (kept_host) {
        VC_CK(cudaMemcpyAsync(kl, kept_host + static_cast<size_t>(l) * m.n_kv * k,
                              static_cast<size_t>(m.n_kv) * k * sizeof(int32_t), cudaMemcpyHostToDevice, st_));
      } else {
        float* sc = score_buf_ + static_cast<size_t>(l) * m.n_kv * T;
        VC_LAUNCH(key_scores(ring_.k + static_cast<size_t>(ca) * m.n_kv * slice_elems, m.n_kv, T, m.d, slice_elems,
                             score_w_, sc, st_));
        VC_LAUNCH(topk_select(sc, m.n_kv, T, static_cast<int>(k), kl, st_));
      }
      VC_LAUNCH(gather_kept(ring_, ca, kl, static_cast<int>(k), drop_, slot * m.layers + l, m.n_kv, m.d, st_));
      VC_LAUNCH(compact_dropped(ring_, ca, kl, static_cast<int>(k), T, ring_, cb, m.n_kv, m.d, st_));
      const size_t w = static_cast<size_t>(T - k) * m.d * 2;
      if (w > 0) {
        VC_CK(cudaMemcpy2DAsync(host_pool_k(slot) + o, pitch, kb, pitch, w, m.n_kv, cudaMemcpyDeviceToHost, st_));
        VC_CK(cudaMemcpy2DAsync(host_pool_v(slot) + o, pitch, vb, pitch, w, m.n_kv, cudaMemcpyDeviceToHost, st_));
      }
      VC_CK(cudaStreamSynchronize(st_));  // the admission chunks are reused by the next layer
    }
    VC_CK(cudaMemcpyAsync(kept_buf_, kept, static_cast<size_t>(m.layers) * m.n_kv * k * sizeof(int32_t),
                          cudaMemcpyDeviceToDevice, st_));
    score_T_ = T;
    last_kept_k_ = static_cast<int>(k);
    s.drop_len = static_cast<int>(k);
    s.drop_base = static_cast<int>(k);
    s.drop_T = T;
    s.n_groups = 0;
    s.tail_committed = 0;
    s.draft_len = 0;
    s.drafted.clear();
    VC_CK(cudaStreamSynchronize(st_));
    return;
  } else if (ring_mode()) {
    // chunk ring: stream the prefix one layer at a time through the two
    // admission chunks and quantise each layer as it lands
    const int ng = std::min(s.committed / VC_QGROUP, quant_.cap / VC_QGROUP);
    const int tc = s.committed - ng * VC_QGROUP;
    if (tc > tail_cap_ - cfg_.max_x - 1) throw ContractViolation("tail overflow");
    const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
    const size_t pitch = slice_elems * 2;
    const size_t width = static_cast<size_t>(s.committed) * m.d * 2;
    check_d2h();  // commits still writing these host rows land first
    for (int l = 0; l < m.layers; ++l) {
      const int c = cfg_.ring_chunks + (l & 1);
      uint16_t* kb = ring_.k + static_cast<size_t>(c) * m.n_kv * slice_elems;
      uint16_t* vb = ring_.v + static_cast<size_t>(c) * m.n_kv * slice_elems;
      VC_CK(cudaStreamWaitEvent(st_, ring_free_[c], 0));
      const size_t o = static_cast<size_t>(l) * m.n_kv * slice_elems;
      if (s.packed_blocks > 0) {
        VC_CK(cudaStreamSynchronize(st_));  // the other admission chunk is the unpack scratch
        host_load_layer(slot, l, c, cfg_.ring_chunks + ((l + 1) & 1), s.committed, s.packed_blocks);
      } else if (width > 0) {
        VC_CK(cudaMemcpy2DAsync(kb, pitch, host_pool_k(slot) + o, pitch, width, m.n_kv, cudaMemcpyHostToDevice, st_));
        VC_CK(cudaMemcpy2DAsync(vb, pitch, host_pool_v(slot) + o, pitch, width, m.n_kv, cudaMemcpyHostToDevice, st_));
      }
      quantise_groups(slot, 0, ng, ring_, c, 0, l, 1);
      VC_LAUNCH(tail_refill(ring_, c, ng * VC_QGROUP, tc, quant_, slot * m.layers + l, 1, m.n_kv, m.d, st_));
    }
    s.n_groups = ng;
    s.tail_committed = tc;
    s.draft_len = 0;
    s.drafted.clear();
    VC_CK(cudaStreamSynchronize(st_));
    return;
  } else if (cfg_.full_tier == 1) {
    // stream the prefix through the scratch staging slot
    uint64_t id = swap_begin(slot, scratch_stage());
    swap_wait(id);
    src = stage_;
    src_slot = scratch_stage();
  }
  if (drop_mode()) {
    compress_drop(slot, src, src_slot, ratio, kept_host, k_host);
    return;
  }
  const int ng = std::min(s.committed / VC_QGROUP, quant_.cap / VC_QGROUP);
  quantise_groups(slot, 0, ng, src, src_slot);
  s.n_groups = ng;
  s.tail_committed = s.committed - ng * VC_QGROUP;
  if (s.tail_committed > tail_cap_ - cfg_.max_x - 1) throw ContractViolation("tail overflow");
  VC_LAUNCH(tail_refill(src, src_slot, ng * VC_QGROUP, s.tail_committed, quant_, slot, m.layers,
                        m.n_kv, m.d, st_));
  s.draft_len = 0;
  s.drafted.clear();
  VC_CK(cudaStreamSynchronize(st_));
}

// Drop-topk compress: per (layer, kv head) keep k = llround(c * T) tokens with
// the highest key scores (ties -> lower position), compacted in position
// order into the drop tier.  Count rule and error of speckv::compress
// (/root/reference/proj/src/compressor.cpp:152-158); equal count per head
// within a layer (the shape law, :83-86) by construction.
void Engine::compress_drop(int slot, const KvPool& src, int src_slot, double ratio, const int32_t* kept_host,
                           int k_host) {
  SeqState& s = seqs_.at(slot);
  const auto& m = cfg_.model;
  const int n_slices = m.layers * m.n_kv;
  const int T = s.committed;
  const long long k = kept_host ? k_host : std::llround(ratio * static_cast<double>(T));
  if (k < 1) throw ContractViolation("compress: drop ratio retains < 1 token");
  if (k > kept_cap_ || k + cfg_.max_x + 2 > drop_.cap)
    throw ContractViolation("compress: drop tier capacity exceeded (ratio above the engine's drop_ratio)");
  if (kept_host) {
    // the kept set is given (drop-uniform / drop-window: the reference's own
    // drop indices, complemented on the host): [slice][k] ascending positions
    VC_CK(cudaMemcpyAsync(kept_buf_, kept_host, static_cast<size_t>(n_slices) * k * sizeof(int32_t),
                          cudaMemcpyHostToDevice, st_));
  } else {
    const uint16_t* keys = src.k + static_cast<size_t>(src_slot) * n_slices * src.cap * m.d;
    const size_t pitch = static_cast<size_t>(src.cap) * m.d;
    if (cfg_.drop_score == 1) {
      // SnapKV: the observation query is the pending token's (the prompt's
      // last token) -- one decode-shaped forward over the full KV, its q heads
      // captured per layer; nothing is committed (its K/V row at position T is
      // rewritten with the same values by the request's first real step)
      if (T + 1 > full_.cap) throw ContractViolation("compress: no room for the observation row");
      std::vector<int32_t> out;
      StepItem it;
      it.slot = slot;
      it.mode = RowMode::Decode;
      it.tokens = {s.pending};
      capture_q_ = true;
      try {
        run_step({it}, out);
      } catch (...) {
        capture_q_ = false;
        throw;
      }
      capture_q_ = false;
      const float sl2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(m.d)));
      for (int l = 0; l < m.layers; ++l)
        VC_LAUNCH(snap_scores(keys + static_cast<size_t>(l) * m.n_kv * pitch, pitch, m.n_kv, T, m.d, m.n_q / m.n_kv,
                              obs_q_ + static_cast<size_t>(l) * m.n_q * m.d, sl2, cfg_.snap_pool, cfg_.snap_recent,
                              snap_logits_, snap_ms_, score_buf_ + static_cast<size_t>(l) * m.n_kv * T, st_));
    } else {
      VC_LAUNCH(key_scores(keys, n_slices, T, m.d, pitch, score_w_, score_buf_, st_));
    }
    score_T_ = T;
    VC_LAUNCH(topk_select(score_buf_, n_slices, T, static_cast<int>(k), kept_buf_, st_));
  }
  VC_LAUNCH(gather_kept(src, src_slot, kept_buf_, static_cast<int>(k), drop_, slot, n_slices, m.d, st_));
  last_kept_k_ = static_cast<int>(k);
  s.drop_len = static_cast<int>(k);
  s.drop_base = static_cast<int>(k);
  s.drop_T = T;
  s.n_groups = 0;
  s.tail_committed = 0;
  s.draft_len = 0;
  s.drafted.clear();
  VC_CK(cudaStreamSynchronize(st_));
}

void Engine::drop_scores(int layer, int head, float* out, int n) const {
  const auto& m = cfg_.model;
  if (!score_buf_ || layer < 0 || layer >= m.layers || head < 0 || head >= m.n_kv || n > score_T_)
    throw ContractViolation("drop_scores: no drop-topk compress or row out of range");
  check_cuda(cudaMemcpy(out, score_buf_ + (static_cast<size_t>(layer) * m.n_kv + head) * score_T_,
                        static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost), "drop_scores");
}

void Engine::obs_query(int layer, uint16_t* out) const {
  const auto& m = cfg_.model;
  if (!obs_q_ || layer < 0 || layer >= m.layers) throw ContractViolation("obs_query: no SnapKV engine");
  check_cuda(cudaMemcpy(out, obs_q_ + static_cast<size_t>(layer) * m.n_q * m.d, static_cast<size_t>(m.n_q) * m.d * 2,
                        cudaMemcpyDeviceToHost), "obs_query");
}

size_t Engine::compressed_bytes(int slot) const {
  const SeqState& s = seqs_.at(slot);
  const auto& m = cfg_.model;
  if (drop_mode()) return static_cast<size_t>(s.drop_len) * m.layers * m.n_kv * m.d * 2 * 2;
  const size_t per_group = static_cast<size_t>(VC_QGROUP) * m.d * cfg_.quant_bits / 8 * 2  // K+V codes
                           + static_cast<size_t>(m.d) * 4 + VC_QGROUP * 4;                  // scales
  return per_group * s.n_groups * m.layers * m.n_kv;
}

// ------------------------------------------------------------------ steps
void Engine::enqueue_forward(int M, int n_draft, int n_dense1, int n_densev, int max_rows_v,
                             bool /*want_logits*/) {
  const auto& m = cfg_.model;
  const int L = m.layers, H = m.hidden, F = m.ffn, V = m.vocab, d = m.d;
  const int qkv_n = (m.n_q + 2 * m.n_kv) * d;
  AttnShape as;
  as.layers = L;
  as.n_kv = m.n_kv;
  as.n_rep = m.n_q / m.n_kv;
  as.d = d;
  as.q_stride = qkv_n;
  as.out_stride = m.n_q * d;
  as.out_mp = M;  // attention output feeds o_proj in the tiled layout
  as.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d)));
  as.draft_warps = draft_warps_;
  as.draft_min_tasks = draft_min_tasks_;
  const KvPool dense_v_pool = cfg_.full_tier == 0 ? full_ : stage_;
  // VC_TRACE=1 (eager engines only): checksum every stage's output buffer
  static const bool tracing = std::getenv("VC_TRACE") != nullptr;
  auto trace = [&](const char* name, const void* p, size_t bytes) {
    if (!tracing || cfg_.use_graphs) return;
    VC_CK(cudaStreamSynchronize(st_));
    std::vector<uint8_t> h(bytes);
    VC_CK(cudaMemcpy(h.data(), p, bytes, cudaMemcpyDeviceToHost));
    uint64_t x = 0xcbf29ce484222325ull;
    for (uint8_t c : h) x = (x ^ c) * 0x100000001b3ull;
    std::fprintf(stderr, "TRACE %s %016llx\n", name, static_cast<unsigned long long>(x));
  };
  GemmEpilogue eq;
  eq.kind = Epi::Qkv;
  eq.out_bf16 = qkv_;
  eq.rows = rows_dev_;
  eq.rope_cos = rope_cos_;
  eq.rope_sin = rope_sin_;
  eq.n_q = m.n_q;
  eq.n_kv = m.n_kv;
  eq.d = d;
  eq.layers = L;
  eq.full = full_;
  eq.stage = stage_;
  eq.drop = drop_;
  eq.draft = quant_;
  GemmEpilogue er;
  er.kind = Epi::Residual;
  er.x = x_;
  er.ss_part = ss_part_;
  GemmEpilogue es;
  es.kind = Epi::Silu;
  es.out_bf16 = act_;
  GemmEpilogue ef;
  ef.kind = Epi::StoreF32;
  ef.out_f32 = logits_;
  // VC_SKIP (diagnostics only, wrong results): bit 0 skips attention + combine,
  // bit 1 skips rms_apply, bit 2 the combine, bits 3-6 the qkv / o / gate-up /
  // down GEMMs -- to attribute a step's in-graph time
  static const int skip = [] {
    const char* v = std::getenv("VC_SKIP");
    return v ? std::atoi(v) : 0;
  }();
  unsigned long long* attn_trace = attn_trace_;
  VC_LAUNCH(embed_norm(tok_in_, M, M, w_.embed, H, w_.attn_norm[0], m.eps, x_, xn_, st_));
  trace("embed.x", x_, static_cast<size_t>(M) * H * 4);
  trace("w.gu0", w_.wgu[0], static_cast<size_t>(2) * F * H * 2);
  trace("w.qkv0", w_.wqkv[0], static_cast<size_t>(qkv_n) * H * 2);
  // RMSNorm fused into the projection that consumes it (GemmNormIn): the qkv
  // GEMM of layers >= 1 and every gate/up GEMM build their bf16 activation
  // tiles from the residual stream and its per-tile sums of squares (bit-
  // identical to rms_apply; 2 fewer launches per layer).  VC_FUSE_NORM=0
  // restores the separate rms_apply launches.
  static const bool fuse_norm = [] {
    const char* v = std::getenv("VC_FUSE_NORM");
    return !(v && v[0] == '0');
  }();
  auto norm_in = [&](const uint16_t* w) {
    GemmNormIn n;
    n.x = x_;
    n.ss = ss_part_;
    n.w = w;
    n.eps = m.eps;
    return n;
  };
  for (int l = 0; l < L; ++l) {
    eq.layer = l;
    if (skip & 8) {
    } else if (fuse_norm && l > 0) {
      const GemmNormIn nq = norm_in(w_.attn_norm[l]);
      VC_LAUNCH(gemm(nullptr, M, M, H, w_.wqkv[l], qkv_n, eq, gws_, st_, &nq));
    } else {
      VC_LAUNCH(gemm(xn_, M, M, H, w_.wqkv[l], qkv_n, eq, gws_, st_));
    }
    trace("qkv", qkv_, static_cast<size_t>(M) * qkv_n * 2);
    if (capture_q_) {  // SnapKV observation query: row 0's q heads of this layer
      MappedCopy mc{};
      mc.seg[0] = {reinterpret_cast<const uint32_t*>(qkv_),
                   reinterpret_cast<uint32_t*>(obs_q_ + static_cast<size_t>(l) * m.n_q * d), m.n_q * d / 2};
      mc.n = 1;
      mapped_copy_kernel<<<4, 256, 0, st_>>>(mc);
      VC_CK(cudaGetLastError());
      ++launches_;
    }
    // the step's attention kernels, then ONE combine over all their partials
    CombineSets cs;
    auto add_set = [&](const AttnSeq* sq, int n, int max_chunks, int mode, int rows) {
      CombineSet& c = cs.set[cs.n_sets++];
      c.seqs = sq;
      c.n = n;
      c.max_chunks = max_chunks;
      c.mode = mode;
      c.rows = rows;
    };
    if (attn_trace && l == 5) VC_CK(cudaMemsetAsync(attn_trace, 0, 3 * 8192 * 8, st_));
    if (skip & 1) {
    } else if (n_draft > 0 && drop_mode()) {
      VC_LAUNCH(dense_attention(as, drop_, drop_maps_, l, seqs_dev_, n_draft, max_chunks_x_, 1, part_, st_));
      add_set(seqs_dev_, n_draft, max_chunks_x_, 1, 1);
    } else if (n_draft > 0) {
      AttnShape tx = as;
      if (l == 5) tx.trace = attn_trace;
      VC_LAUNCH(draft_attention_quant(tx, quant_, l, qkv_, seqs_dev_, n_draft, max_chunks_q_,
                                      cfg_.quant_bits, part_, st_));
      add_set(seqs_dev_, n_draft, max_chunks_q_, 0, 1);
    }
    if (n_dense1 > 0 && !(skip & 1)) {
      VC_LAUNCH(dense_attention(as, full_, dense_maps_, l, seqs_dev_ + n_draft, n_dense1, max_chunks_d_, 1, part_, st_));
      add_set(seqs_dev_ + n_draft, n_dense1, max_chunks_d_, 1, 1);
    }
    if (n_densev > 0 && !(skip & 1)) {
      const AttnSeq* sv = seqs_dev_ + n_draft + n_dense1;
      VC_LAUNCH(dense_attention(as, dense_v_pool, dense_maps_, l, sv, n_densev, max_chunks_d_, max_rows_v, part_, st_));
      add_set(sv, n_densev, max_chunks_d_, 1, max_rows_v);
    }
    if (cs.n_sets > 0 && !(skip & 4)) VC_LAUNCH(attention_combine_sets(as, cs, part_, attn_, st_));
    // residual projection: fused residual epilogue, or (tensor parallel) the
    // rank's partial -> all-gather -> fixed rank-order sum + residual (vc_tp.h);
    // then the next RMSNorm.  (r1: fusing the RMSNorm into the residual
    // epilogue -- tile finishers spin until every tile's ss_part is in -- was
    // bit-identical but 3% slower per step than this launch.)
    auto residual_gemm = [&](const uint16_t* Xt, int Kd, const uint16_t* Wt, const uint16_t* norm_w, bool norm_next) {
      if (!coll_) {
        if (!(skip & (Kd == H ? 16 : 64))) VC_LAUNCH(gemm(Xt, M, M, Kd, Wt, H, er, gws_, st_));
      } else {
        GemmEpilogue ey;
        ey.kind = Epi::StoreF32;
        ey.out_f32 = tp_y_;
        VC_LAUNCH(gemm(Xt, M, M, Kd, Wt, H, ey, gws_, st_));
        coll_->all_gather(tp_y_, tp_g_, static_cast<size_t>(M) * H, st_);
        VC_LAUNCH(tp_residual(x_, tp_g_, cfg_.tp_size, M, H, ss_part_, st_));
      }
      if (!(skip & 2) && norm_next) VC_LAUNCH(rms_apply(x_, ss_part_, M, M, H, norm_w, m.eps, xn_, st_));
    };
    residual_gemm(attn_, m.n_q * d, w_.wo[l], w_.mlp_norm[l], !fuse_norm);
    trace("attn", attn_, static_cast<size_t>(M) * m.n_q * d * 2);
    trace("x.o", x_, static_cast<size_t>(M) * H * 4);
    trace("ss.o", ss_part_, static_cast<size_t>(M) * (H / 128) * 4);
    trace("xn.o", xn_, static_cast<size_t>(M) * H * 2);
    if (skip & 32) {
    } else if (fuse_norm) {
      const GemmNormIn ng = norm_in(w_.mlp_norm[l]);
      VC_LAUNCH(gemm(nullptr, M, M, H, w_.wgu[l], 2 * F, es, gws_, st_, &ng));
    } else {
      VC_LAUNCH(gemm(xn_, M, M, H, w_.wgu[l], 2 * F, es, gws_, st_));
    }
    trace("act", act_, static_cast<size_t>(M) * F * 2);
    residual_gemm(act_, F, w_.wd[l], l + 1 < L ? w_.attn_norm[l + 1] : w_.final_norm, !fuse_norm || l + 1 == L);
    trace("x.d", x_, static_cast<size_t>(M) * H * 4);
  }
  VC_LAUNCH(gemm(xn_, M, M, H, w_.lm_head, V, ef, gws_, st_));
  trace("logits", logits_, static_cast<size_t>(M) * V * 4);
  VC_LAUNCH(argmax_rows(logits_, M, V, tok_out_, st_));
}

namespace {
int bucket_seqs(int n) { return n == 0 ? 0 : (n + 3) / 4 * 4; }
}  // namespace

void Engine::run_step(const std::vector<StepItem>& items, std::vector<int32_t>& out,
                      float* logits_host) {
  const auto& m = cfg_.model;
  const int n_seq_max = 2 * (draft_rows_max() + 4) + cfg_.max_verify + 4;
  scratch_slot_ = -1;  // a step may write any staging slot
  int32_t* h_tok = static_cast<int32_t*>(h_desc_);
  RowDest* h_rows = reinterpret_cast<RowDest*>(h_tok + Mmax_);
  AttnSeq* h_seqs = reinterpret_cast<AttnSeq*>(h_rows + Mmax_);
  std::vector<AttnSeq> drafts, dense1, densev;
  int M = 0, max_rows_v = 1;
  for (const StepItem& it : items) {
    const SeqState& s = seqs_.at(it.slot);
    if (!s.live) throw ContractViolation("run_step: slot not live");
    const int n = static_cast<int>(it.tokens.size());
    if (n < 1 || M + n > Mmax_) throw ContractViolation("run_step: too many rows");
    AttnSeq a{};
    a.row0 = M;
    a.n_rows = n;
    if (it.mode == RowMode::Draft) {
      // n >= 1 rows over the compressed tier: the next draft input and, for
      // the two-level composition, an auxiliary drafter's proposals after it
      // (row i sees the draft window plus rows 0..i -- the qkv epilogue writes
      // every row's K/V into the tail before attention runs).  Each row is its
      // own draft sequence; rows past the accepted ones are overwritten later.
      if (s.draft_len + n > cfg_.max_x + 1) throw ContractViolation("draft window overflow (rows past max_x)");
      for (int i = 0; i < n; ++i) {
        AttnSeq r = a;
        r.row0 = M + i;
        r.n_rows = 1;
        r.slot = it.slot;
        h_tok[M + i] = it.tokens[i];
        if (drop_mode()) {  // drop tier: dense attention over the compacted kept + appended tokens
          if (s.drop_len + s.draft_len + i + 1 > drop_.cap) throw ContractViolation("drop tier full");
          h_rows[M + i] = RowDest{3, it.slot, s.drop_len + s.draft_len + i, s.committed + s.draft_len + i};
          r.kv_len = s.drop_len + s.draft_len + i + 1;
        } else {
          if (cfg_.quant_bits == 0) throw ContractViolation("draft rows need the compressed tier");
          if (s.tail_committed + s.draft_len + i + 1 > tail_cap_) throw ContractViolation("draft window overflow");
          h_rows[M + i] = RowDest{1, it.slot, s.tail_committed + s.draft_len + i, s.committed + s.draft_len + i};
          r.n_groups = s.n_groups;
          r.tail_len = s.tail_committed + s.draft_len + i + 1;
        }
        drafts.push_back(r);
      }
    } else {
      const bool staged = cfg_.full_tier == 1;
      if (staged && it.mode == RowMode::Decode) throw ContractViolation("decode rows need the HBM full tier");
      if (staged && (it.stage < 0 || it.stage >= cfg_.n_stage)) throw ContractViolation("verify needs a staging slot");
      const int pslot = staged ? it.stage : it.slot;
      if (s.committed + n > full_.cap) throw ContractViolation("context exceeds capacity");
      for (int i = 0; i < n; ++i) {
        h_tok[M + i] = it.tokens[i];
        h_rows[M + i] = RowDest{staged ? 2 : 0, pslot, s.committed + i, s.committed + i};
      }
      a.slot = pslot;
      a.kv_len = s.committed + n;
      if (n == 1 && !staged) {
        dense1.push_back(a);
      } else {
        densev.push_back(a);
        max_rows_v = std::max(max_rows_v, n);
      }
    }
    M += n;
  }
  if (static_cast<int>(drafts.size() + dense1.size() + densev.size()) > n_seq_max)
    throw ContractViolation("run_step: too many sequences");
  // partial-row offsets (units of Hq partial rows)
  int off = 0;
  for (auto& a : drafts) { a.part0 = off; off += drop_mode() ? max_chunks_x_ : draft_parts_per_seq(max_chunks_q_, tail_cap_); }
  for (auto& a : dense1) { a.part0 = off; off += max_chunks_d_ * a.n_rows; }
  for (auto& a : densev) { a.part0 = off; off += max_chunks_d_ * a.n_rows; }
  // Bucket the step shape (padding rows / empty sequences) so a handful of
  // CUDA graphs cover every step; padding never changes a real row's math.
  const int Mb = std::min(bucket_rows(M), Mmax_);
  for (int i = M; i < Mb; ++i) {
    h_tok[i] = 0;
    h_rows[i] = RowDest{-1, 0, 0, 0};
  }
  const int nd = bucket_seqs(static_cast<int>(drafts.size()));
  const int n1 = bucket_seqs(static_cast<int>(dense1.size()));
  const int nv = static_cast<int>(densev.size());
  // verify windows: bucket to multiples of 4 tokens (one 16-row MMA tile at n_rep 4)
  const int mrv = nv ? (max_rows_v + 3) / 4 * 4 : 1;
  int k = 0;
  const AttnSeq empty{};
  for (int i = 0; i < nd; ++i) h_seqs[k++] = i < static_cast<int>(drafts.size()) ? drafts[i] : empty;
  for (int i = 0; i < n1; ++i) h_seqs[k++] = i < static_cast<int>(dense1.size()) ? dense1[i] : empty;
  for (auto& a : densev) h_seqs[k++] = a;
  if (k > n_seq_max) throw ContractViolation("run_step: too many sequences");

  if (cfg_.tp_size > 1 && !coll_) throw ContractViolation("tensor-parallel engine: attach a collective first");
  cudaGraphExec_t exec = nullptr;
  std::string key;
  if (cfg_.use_graphs && !capture_q_ && (!coll_ || coll_->graph_capturable())) {  // capture before the timed window opens
    std::ostringstream ks;
    ks << Mb << ':' << nd << ':' << n1 << ':' << nv << ':' << mrv;
    key = ks.str();
    auto itg = graphs_.find(key);
    if (itg == graphs_.end()) {
      cudaGraph_t g;
      const uint64_t before = launches_;
      VC_CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
      enqueue_forward(Mb, nd, n1, nv, mrv, logits_host != nullptr);
      VC_CK(cudaStreamEndCapture(st_, &g));
      cudaGraphExec_t ge;
      VC_CK(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphDestroy(g);
      launches_per_graph_[key] = launches_ - before;
      itg = graphs_.emplace(key, ge).first;
      launches_ = before;
    }
    exec = itg->second;
  }
  VC_CK(cudaEventRecord(ev_a_, st_));
  {  // descriptors: mapped pinned -> device by the SMs (see mapped_copy_kernel)
    auto dev_of = [&](const void* h) {
      return reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(d_hdesc_) +
                                               (static_cast<const uint8_t*>(h) - static_cast<const uint8_t*>(h_desc_)));
    };
    MappedCopy mc{};
    mc.seg[0] = {dev_of(h_tok), reinterpret_cast<uint32_t*>(tok_in_), Mb};
    mc.seg[1] = {dev_of(h_rows), reinterpret_cast<uint32_t*>(rows_dev_), static_cast<int>(Mb * sizeof(RowDest) / 4)};
    mc.seg[2] = {dev_of(h_seqs), reinterpret_cast<uint32_t*>(seqs_dev_), static_cast<int>(k * sizeof(AttnSeq) / 4)};
    mc.n = 3;
    mapped_copy_kernel<<<8, 256, 0, st_>>>(mc);
    VC_CK(cudaGetLastError());
    ++launches_;
  }
  if (exec) {
    VC_CK(cudaGraphLaunch(exec, st_));
    launches_ += launches_per_graph_[key];
  } else {
    enqueue_forward(Mb, nd, n1, nv, mrv, logits_host != nullptr);
  }
  {  // greedy tokens: device -> mapped pinned by the SMs
    MappedCopy mc{};
    mc.seg[0] = {reinterpret_cast<const uint32_t*>(tok_out_), reinterpret_cast<uint32_t*>(d_hout_), M};
    mc.n = 1;
    mapped_copy_kernel<<<1, 256, 0, st_>>>(mc);
    VC_CK(cudaGetLastError());
    ++launches_;
  }
  if (logits_host)
    VC_CK(cudaMemcpyAsync(logits_host, logits_, static_cast<size_t>(M) * m.vocab * 4,
                          cudaMemcpyDeviceToHost, st_));
  VC_CK(cudaEventRecord(ev_b_, st_));
  VC_CK(cudaStreamSynchronize(st_));
  float ms = 0.f;
  VC_CK(cudaEventElapsedTime(&ms, ev_a_, ev_b_));
  device_ms_ += ms;
  ++steps_;
  static const bool step_log = std::getenv("VC_STEP_LOG") != nullptr;
  if (step_log)
    std::fprintf(stderr, "STEP M=%d Mb=%d drafts=%zu dense1=%zu verify=%zu rows_v=%d ms=%.3f\n", M, Mb,
                 drafts.size(), dense1.size(), densev.size(), max_rows_v, ms);
  out.assign(h_out_, h_out_ + M);
  last_M_ = M;
  if (attn_trace_) {  // diagnostics: layer 5's attention CTA timeline (ns from the first dense/draft start)
    std::vector<unsigned long long> t(3 * 8192);
    VC_CK(cudaMemcpy(t.data(), attn_trace_, t.size() * 8, cudaMemcpyDeviceToHost));
    auto span = [&](size_t off, size_t n, unsigned long long& lo, unsigned long long& hi, int& cnt, double& avg) {
      lo = ~0ull; hi = 0; cnt = 0; avg = 0;
      for (size_t i = 0; i < n; ++i) {
        const unsigned long long a = t[off + 2 * i], b = t[off + 2 * i + 1];
        if (!a || !b) continue;
        lo = std::min(lo, a); hi = std::max(hi, b); ++cnt; avg += static_cast<double>(b - a);
      }
      if (cnt) avg /= cnt;
    };
    unsigned long long dl, dh, ql, qh;
    int dc, qc;
    double da, qa;
    span(0, 4096, dl, dh, dc, da);
    span(8192, 2048, ql, qh, qc, qa);
    const unsigned long long t0 = std::min(dc ? dl : ~0ull, qc ? ql : ~0ull);
    std::fprintf(stderr, "ATTN dense ctas=%d [%.1f, %.1f] us avg %.1f | draft ctas=%d [%.1f, %.1f] us avg %.1f\n", dc,
                 dc ? (dl - t0) / 1e3 : 0.0, dc ? (dh - t0) / 1e3 : 0.0, da / 1e3, qc, qc ? (ql - t0) / 1e3 : 0.0,
                 qc ? (qh - t0) / 1e3 : 0.0, qa / 1e3);
    if (const char* f = std::getenv("VC_ATTN_TRACE_FILE")) {  // raw per-CTA timeline for offline analysis
      if (FILE* fp = std::fopen(f, "wb")) {
        std::fwrite(t.data(), 8, t.size(), fp);
        std::fclose(fp);
      }
    }
    if (qc) {  // the draft grid: the persistent quantised CTAs, then the bf16-tail CTAs (VC_DRAFT_TAIL_LAST)
      const int nq = std::min(draft_warps_ / 4, 2048);
      unsigned long long tl, th, pl, ph;
      int tc, pc;
      double ta, pa;
      span(8192, nq, pl, ph, pc, pa);
      span(8192 + 2 * static_cast<size_t>(nq), 2048 - nq, tl, th, tc, ta);
      unsigned long long pe_lo = ~0ull;  // first quantised CTA to finish
      for (int i = 0; i < nq; ++i)
        if (t[8192 + 2 * i] && t[8192 + 2 * i + 1]) pe_lo = std::min(pe_lo, t[8192 + 2 * i + 1]);
      std::fprintf(stderr, "DRAFT quant ctas=%d [%.1f, %.1f] us, first end %.1f | tail ctas=%d [%.1f, %.1f] avg %.1f\n", pc,
                   pc ? (pl - t0) / 1e3 : 0.0, pc ? (ph - t0) / 1e3 : 0.0, pc ? (pe_lo - t0) / 1e3 : 0.0, tc,
                   tc ? (tl - t0) / 1e3 : 0.0, tc ? (th - t0) / 1e3 : 0.0, ta / 1e3);
    }
  }
}

void Engine::kernel_bench(int kind, const std::vector<int>& slots, int reps, double* ms,
                          double* bytes) {
  // time the kernel alone: no copy of the setup still in flight
  VC_CK(cudaStreamSynchronize(copy_st_));
  check_d2h();
  const auto& m = cfg_.model;
  const int n = static_cast<int>(slots.size());
  AttnShape as;
  as.layers = m.layers;
  as.n_kv = m.n_kv;
  as.n_rep = m.n_q / m.n_kv;
  as.d = m.d;
  as.q_stride = (m.n_q + 2 * m.n_kv) * m.d;
  as.out_stride = m.n_q * m.d;
  as.out_mp = 0;
  as.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(m.d)));
  as.draft_warps = draft_warps_;
  as.draft_min_tasks = draft_min_tasks_;
  AttnSeq* h = reinterpret_cast<AttnSeq*>(static_cast<int32_t*>(h_desc_) + Mmax_) ;
  h = reinterpret_cast<AttnSeq*>(reinterpret_cast<RowDest*>(h) + Mmax_);
  double b = 0.0;
  const double g = VC_QGROUP;
  for (int i = 0; i < n; ++i) {
    const SeqState& s = seqs_.at(slots[i]);
    AttnSeq a{};
    a.slot = slots[i];
    a.n_rows = kind == 2 ? cfg_.max_x + 1 : 1;  // kind 2: a verify window of max_x+1 rows
    a.row0 = i * a.n_rows;
    if ((i + 1) * a.n_rows > Mmax_) throw ContractViolation("kernel_bench: too many rows");
    a.kv_len = kind == 3 ? s.drop_len : s.committed;
    a.n_groups = s.n_groups;
    a.tail_len = s.tail_committed;
    a.part0 = kind == 0 ? i * draft_parts_per_seq(max_chunks_q_, tail_cap_)
                        : i * (kind == 3 ? max_chunks_x_ : max_chunks_d_) * a.n_rows;
    if (kind == 3 && !drop_mode()) throw ContractViolation("kernel_bench: no drop tier");
    h[i] = a;
    // algorithmic bytes per (layer, request, kv-head) -- DESIGN.md §Roofline
    if (kind == 0)
      b += s.n_groups * g * m.d * cfg_.quant_bits / 8.0 * 2  // K + V codes
           + s.n_groups * m.d * 4.0 + s.n_groups * g * 4.0   // K per-channel, V per-token (scale, zero)
           + s.tail_committed * m.d * 2.0 * 2;                // bf16 tail
    else
      b += static_cast<double>(a.kv_len) * m.d * 2 * 2;
  }
  b *= static_cast<double>(m.layers) * m.n_kv;
  VC_CK(cudaMemcpyAsync(seqs_dev_, h, n * sizeof(AttnSeq), cudaMemcpyHostToDevice, st_));
  // time the attention kernel alone (events on the launching stream around
  // each launch); the combine that follows it is launched but not timed
  const int n_ev = m.layers * (reps + 1);
  std::vector<cudaEvent_t> ev(2 * n_ev);
  for (auto& x : ev) VC_CK(cudaEventCreate(&x));
  int k = 0;
  for (int r = 0; r <= reps; ++r)
    for (int l = 0; l < m.layers; ++l, ++k) {
      VC_CK(cudaEventRecord(ev[2 * k], st_));
      if (kind == 0) {
        VC_LAUNCH(draft_attention_quant(as, quant_, l, qkv_, seqs_dev_, n, max_chunks_q_, cfg_.quant_bits, part_, st_));
      } else if (kind == 3) {  // drafting over the drop-topk tier
        VC_LAUNCH(dense_attention(as, drop_, drop_maps_, l, seqs_dev_, n, max_chunks_x_, 1, part_, st_));
      } else {
        const KvPool pool = cfg_.full_tier == 0 ? full_ : stage_;
        VC_LAUNCH(dense_attention(as, pool, dense_maps_, l, seqs_dev_, n, max_chunks_d_, h[0].n_rows, part_, st_));
      }
      VC_CK(cudaEventRecord(ev[2 * k + 1], st_));
      VC_LAUNCH(attention_combine(as, seqs_dev_, n, kind == 0 ? max_chunks_q_ : (kind == 3 ? max_chunks_x_ : max_chunks_d_),
                                  h[0].n_rows, kind == 0 ? 0 : 1,
                                  part_, attn_, st_));
    }
  VC_CK(cudaStreamSynchronize(st_));
  double total = 0.0;
  for (int j = m.layers; j < n_ev; ++j) {  // the first pass is warm-up
    float t = 0.f;
    VC_CK(cudaEventElapsedTime(&t, ev[2 * j], ev[2 * j + 1]));
    total += t;
  }
  for (auto& x : ev) cudaEventDestroy(x);
  *ms = total / reps;  // per launch-set (all layers)
  *bytes = b;
}

void Engine::commit_decode(int slot, int32_t next) {
  SeqState& s = seqs_.at(slot);
  s.committed += 1;
  s.pending = next;
  s.history.push_back(next);
}

void Engine::discard_drafts(int slot) {
  // the draft window's rows (tail / drop tier) are simply overwritten later
  SeqState& s = seqs_.at(slot);
  s.drafted.clear();
  s.draft_len = 0;
}

void Engine::push_draft(int slot, int32_t tok) {
  SeqState& s = seqs_.at(slot);
  s.drafted.push_back(tok);
  s.draft_len += 1;
}

std::vector<int32_t> Engine::accept_commit(int slot, const std::vector<int32_t>& preds, int stage) {
  const bool staged = cfg_.full_tier == 1;
  if (staged && resident(slot) && stage != slot)
    throw ContractViolation("accept: a resident slot verifies in its own staging slot");
  if (staged && !resident(slot) && stage < 0) throw ContractViolation("accept: staged verify needs its stage");
  const RowSrc src{staged ? stage_ : full_, staged ? stage : slot, 0};
  return accept_commit_from(slot, preds, src, staged && !resident(slot));
}

std::vector<int32_t> Engine::accept_commit_from(int slot, const std::vector<int32_t>& preds, const RowSrc& src,
                                                bool to_host) {
  SeqState& s = seqs_.at(slot);
  const int x = static_cast<int>(s.drafted.size());
  if (static_cast<int>(preds.size()) != x + 1) throw ContractViolation("accept: |preds| must be |drafted|+1");
  // accept rule (/root/reference/proj/src/specloop.cpp:37-56)
  int mcount = x;
  for (int k = 0; k < x; ++k)
    if (s.drafted[k] != preds[k]) { mcount = k; break; }
  std::vector<int32_t> emitted(s.drafted.begin(), s.drafted.begin() + mcount);
  emitted.push_back(preds[mcount]);
  const auto& m = cfg_.model;
  const int old = s.committed;
  const int now = old + 1 + mcount;
  if (cfg_.quant_bits > 0 && !drop_mode()) {
    // the bf16 tail holds the residual group + the next draft window; past
    // max_ctx the quantised tier cannot take more groups (same bound as compress)
    const int ng_now = std::min(now / VC_QGROUP, quant_.cap / VC_QGROUP);
    if (now - ng_now * VC_QGROUP > tail_cap_ - cfg_.max_x - 1)
      throw ContractViolation("accept: request exceeds max_ctx (compressed tail overflow)");
  }
  if (src.origin > old) throw ContractViolation("accept: exact rows start after the committed prefix");
  if (to_host) {
    // exact KV of the committed rows back to the host pool
    const int n_slices = m.layers * m.n_kv;
    const size_t dpitch = static_cast<size_t>(full_.cap) * m.d * 2;
    const size_t spitch = static_cast<size_t>(src.pool.cap) * m.d * 2;
    int raw_from = old;  // rows [raw_from, now) go to the host raw
    if (s.packed_blocks > 0 && old < s.packed_blocks * VC_QGROUP) {
      // the window ends inside the packed prefix: re-pack its blocks from the
      // exact rows (the block's earlier rows are in src too: origin is the
      // residual group's start); a block that no longer packs ends the prefix
      const int P = s.packed_blocks;
      const int b0 = old / VC_QGROUP, b1 = std::min(P, (now + VC_QGROUP - 1) / VC_QGROUP);
      if (src.origin > b0 * VC_QGROUP) throw ContractViolation("accept: exact rows do not cover the packed block");
      const int nblk = b1 - b0;
      const size_t PB = packed_block_bytes(m.d);
      VC_CK(cudaStreamWaitEvent(st_, ev_d2h_, 0));  // the staging of the previous commit has left
      VC_CK(cudaMemsetAsync(pack_overflow_, 0, sizeof(int), st_));
      for (int kv = 0; kv < 2; ++kv)
        VC_CK(pack_blocks((kv ? src.pool.v : src.pool.k) + static_cast<size_t>(src.slot) * n_slices * src.pool.cap * m.d,
                          static_cast<size_t>(src.pool.cap) * m.d, b0 * VC_QGROUP - src.origin, now - b0 * VC_QGROUP,
                          nblk, n_slices, m.d, pack_stage_ + kv * static_cast<size_t>(n_slices) * 2 * PB, nblk * PB,
                          pack_overflow_, st_));
      int f = 0;
      VC_CK(cudaMemcpyAsync(&f, pack_overflow_, sizeof(int), cudaMemcpyDeviceToHost, st_));
      VC_CK(cudaStreamSynchronize(st_));
      const int newP = f > 0 ? b0 + f - 1 : P;
      VC_CK(cudaEventRecord(ev_commit_, st_));
      VC_CK(cudaStreamWaitEvent(d2h_st_, ev_commit_, 0));
      if (newP > b0)
        for (int kv = 0; kv < 2; ++kv)
          VC_CK(cudaMemcpy2DAsync(reinterpret_cast<uint8_t*>(kv ? host_pool_v(slot) : host_pool_k(slot)) + b0 * PB,
                                  dpitch, pack_stage_ + kv * static_cast<size_t>(n_slices) * 2 * PB, nblk * PB,
                                  (newP - b0) * PB, n_slices, cudaMemcpyDeviceToHost, d2h_st_));
      s.packed_blocks = newP;
      raw_from = newP * VC_QGROUP;
    }
    const size_t width = static_cast<size_t>(std::max(0, now - raw_from)) * m.d * 2;
    uint16_t* hk = host_pool_k(slot) + static_cast<size_t>(raw_from) * m.d;
    uint16_t* hv = host_pool_v(slot) + static_cast<size_t>(raw_from) * m.d;
    const size_t soff = (static_cast<size_t>(src.slot) * n_slices * src.pool.cap + (raw_from - src.origin)) * m.d;
    // on its own stream: a D2H on the compute stream would queue behind an
    // in-flight 4.29 GB reload in the copy engine and stall the next step for
    // the rest of that reload (measured: 91 ms steps after every offloaded
    // verify).  Later reloads (of this slot, or into this staging slot) wait
    // for it through copy_st_.
    VC_CK(cudaEventRecord(ev_commit_, st_));
    VC_CK(cudaStreamWaitEvent(d2h_st_, ev_commit_, 0));
    if (width > 0) {
      if (raw_from < src.origin) throw ContractViolation("accept: exact rows start after the raw host rows");
      VC_CK(cudaMemcpy2DAsync(hk, dpitch, src.pool.k + soff, spitch, width, n_slices, cudaMemcpyDeviceToHost, d2h_st_));
      VC_CK(cudaMemcpy2DAsync(hv, dpitch, src.pool.v + soff, spitch, width, n_slices, cudaMemcpyDeviceToHost, d2h_st_));
    }
    VC_CK(cudaEventRecord(ev_d2h_, d2h_st_));
    VC_CK(cudaStreamWaitEvent(copy_st_, ev_d2h_, 0));
  }
  if (drop_mode()) {
    // the accepted rows' exact K/V (full tier) are appended to the compacted
    // tier; the draft window's entries beyond them are simply overwritten
    if (s.drop_len + (now - old) + cfg_.max_x + 2 > drop_.cap) throw ContractViolation("drop tier full");
    VC_LAUNCH(copy_rows(src.pool, src.slot, old - src.origin, now - old, drop_, slot, s.drop_len,
                        m.layers * m.n_kv, m.d, st_));
    s.drop_len += now - old;
    // online mode (speckv::update semantics, compressor.cpp:208-243, with the
    // kept prefix as the sink): once 2W tokens have been appended, keep the
    // latest W and drop the older ones -- one non-overlapping row move
    const int W = cfg_.drop_window;
    if (W > 0 && s.drop_len - s.drop_base >= 2 * W) {
      VC_LAUNCH(copy_rows(drop_, slot, s.drop_len - W, W, drop_, slot, s.drop_base, m.layers * m.n_kv, m.d, st_));
      s.drop_len = s.drop_base + W;
    }
  } else if (cfg_.quant_bits > 0 && (s.n_groups > 0 || s.tail_committed > 0 || x > 0)) {
    const int ng_now = std::min(now / VC_QGROUP, quant_.cap / VC_QGROUP);
    if (ng_now > s.n_groups && s.n_groups * VC_QGROUP < src.origin)
      throw ContractViolation("accept: exact rows do not cover the groups to quantise");
    quantise_groups(slot, s.n_groups, ng_now - s.n_groups, src.pool, src.slot, src.origin);
    s.n_groups = ng_now;
    s.tail_committed = now - ng_now * VC_QGROUP;
    VC_LAUNCH(tail_refill(src.pool, src.slot, ng_now * VC_QGROUP - src.origin, s.tail_committed, quant_, slot,
                          m.layers, m.n_kv, m.d, st_));
  }
  s.committed = now;
  s.pending = preds[mcount];
  s.drafted.clear();
  s.draft_len = 0;
  s.history.insert(s.history.end(), emitted.begin(), emitted.end());
  return emitted;
}

// ------------------------------------------------------------ remote prefix
// Remote prefix caching (BASELINE.json configs[3]; the reference's simulated
// remote_prefix, /root/reference/proj/src/sim.cpp:510-665).  The storage node
// holds a precomputed prefix in both forms -- `compress` produced the payload
// at storage -- and the engine streams them into request
// slots: the compressed payload first (drafting can start, kCompressedLoaded
// at sim.cpp:588-610), the full KV behind it (the verify prefetch,
// start_cycle at sim.cpp:562-575).  The full KV stays resident after it
// lands (verify_cached).
void Engine::prefix_drop() {
  for (void* p : {static_cast<void*>(pre_k_), static_cast<void*>(pre_v_), static_cast<void*>(pre_kt_),
                  static_cast<void*>(pre_vt_), static_cast<void*>(pre_rec_)})
    if (p) cudaFreeHost(p);
  pre_k_ = pre_v_ = pre_kt_ = pre_vt_ = nullptr;
  pre_rec_ = nullptr;
  pre_T_ = pre_ng_ = pre_tc_ = 0;
}

double Engine::prefix_bytes(int what) const {
  const auto& m = cfg_.model;
  const double n_slices = static_cast<double>(m.layers) * m.n_kv;
  if (what == 1) return 2.0 * n_slices * pre_T_ * m.d * 2;
  return n_slices * (static_cast<double>(pre_ng_) * quant_record_words(m.d, cfg_.quant_bits) * 4 +
                     2.0 * pre_tc_ * m.d * 2);
}

void Engine::prefix_store(int src_slot) {
  if (cfg_.full_tier != 0) throw ContractViolation("remote prefix: needs the HBM full tier (full_tier 0)");
  if (cfg_.quant_bits == 0) throw ContractViolation("remote prefix: needs the quantised compressed tier");
  const SeqState& s = seqs_.at(src_slot);
  if (!s.live || s.committed < 1) throw ContractViolation("prefix_store: slot holds no prefix");
  if (s.n_groups * VC_QGROUP + s.tail_committed != s.committed || s.draft_len != 0)
    throw ContractViolation("prefix_store: compress the prefix first (no open draft round)");
  prefix_drop();
  const auto& m = cfg_.model;
  const int n_slices = m.layers * m.n_kv;
  pre_T_ = s.committed;
  pre_ng_ = s.n_groups;
  pre_tc_ = s.tail_committed;
  const size_t full_w = static_cast<size_t>(pre_T_) * m.d * 2;
  const size_t words = quant_record_words(m.d, cfg_.quant_bits);
  const size_t rec_w = static_cast<size_t>(pre_ng_) * words * 4;
  const size_t tail_w = static_cast<size_t>(pre_tc_) * m.d * 2;
  auto halloc = [&](size_t bytes) {
    void* p = nullptr;
    VC_CK(cudaHostAlloc(&p, std::max<size_t>(bytes, 256), cudaHostAllocDefault));
    return p;
  };
  pre_k_ = static_cast<uint16_t*>(halloc(full_w * n_slices));
  pre_v_ = static_cast<uint16_t*>(halloc(full_w * n_slices));
  pre_rec_ = static_cast<uint32_t*>(halloc(rec_w * n_slices));
  pre_kt_ = static_cast<uint16_t*>(halloc(tail_w * n_slices));
  pre_vt_ = static_cast<uint16_t*>(halloc(tail_w * n_slices));
  const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
  const size_t base = static_cast<size_t>(src_slot) * n_slices;
  VC_CK(cudaMemcpy2DAsync(pre_k_, full_w, full_.k + base * slice_elems, slice_elems * 2, full_w, n_slices,
                          cudaMemcpyDeviceToHost, st_));
  VC_CK(cudaMemcpy2DAsync(pre_v_, full_w, full_.v + base * slice_elems, slice_elems * 2, full_w, n_slices,
                          cudaMemcpyDeviceToHost, st_));
  const size_t slice_words = static_cast<size_t>(quant_.cap / VC_QGROUP) * words;
  if (rec_w)
    VC_CK(cudaMemcpy2DAsync(pre_rec_, rec_w, quant_.rec + base * slice_words, slice_words * 4, rec_w, n_slices,
                            cudaMemcpyDeviceToHost, st_));
  const size_t tpitch = static_cast<size_t>(tail_cap_) * m.d * 2;
  if (tail_w) {
    VC_CK(cudaMemcpy2DAsync(pre_kt_, tail_w, quant_.ktail + base * tail_cap_ * m.d, tpitch, tail_w, n_slices,
                            cudaMemcpyDeviceToHost, st_));
    VC_CK(cudaMemcpy2DAsync(pre_vt_, tail_w, quant_.vtail + base * tail_cap_ * m.d, tpitch, tail_w, n_slices,
                            cudaMemcpyDeviceToHost, st_));
  }
  VC_CK(cudaStreamSynchronize(st_));
}

uint64_t Engine::prefix_load(int slot, int what, int32_t pending) {
  if (pre_T_ == 0) throw ContractViolation("prefix_load: no prefix stored");
  if (slot < 0 || slot >= cfg_.max_slots) throw ContractViolation("slot out of range");
  if (what != 0 && what != 1) throw ContractViolation("prefix_load: what is 0 (compressed) or 1 (full)");
  if (pre_T_ + cfg_.max_x + 2 > full_.cap) throw ContractViolation("prefix exceeds the slot capacity");
  {
    const SeqState& s0 = seqs_.at(slot);
    // a slot is opened by its first load; the other form may follow (the full
    // KV lands while the request drafts), but nothing may overwrite a slot
    // that has moved past the prefix or a compressed tier being drafted on
    if (s0.live && (s0.committed != pre_T_ || (what == 0 && !s0.drafted.empty())))
      throw ContractViolation("prefix_load: slot holds another request (release it first)");
  }
  const auto& m = cfg_.model;
  const int n_slices = m.layers * m.n_kv;
  const size_t base = static_cast<size_t>(slot) * n_slices;
  // the slot may still be read by an in-flight step on the compute stream
  cudaEvent_t ready;
  VC_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  VC_CK(cudaEventRecord(ready, st_));
  VC_CK(cudaStreamWaitEvent(copy_st_, ready, 0));
  cudaEventDestroy(ready);
  Xfer x{};
  x.bytes = prefix_bytes(what);
  VC_CK(cudaEventCreate(&x.start));
  VC_CK(cudaEventCreate(&x.done));
  VC_CK(cudaEventRecord(x.start, copy_st_));
  if (what == 1) {
    const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
    const size_t w = static_cast<size_t>(pre_T_) * m.d * 2;
    VC_CK(copy2d_chunked(full_.k + base * slice_elems, slice_elems * 2, pre_k_, w, w, n_slices,
                         cudaMemcpyHostToDevice, copy_st_, m.n_kv));
    VC_CK(copy2d_chunked(full_.v + base * slice_elems, slice_elems * 2, pre_v_, w, w, n_slices,
                         cudaMemcpyHostToDevice, copy_st_, m.n_kv));
  } else {
    const size_t words = quant_record_words(m.d, cfg_.quant_bits);
    const size_t slice_words = static_cast<size_t>(quant_.cap / VC_QGROUP) * words;
    const size_t rec_w = static_cast<size_t>(pre_ng_) * words * 4;
    if (rec_w)
      VC_CK(copy2d_chunked(quant_.rec + base * slice_words, slice_words * 4, pre_rec_, rec_w, rec_w, n_slices,
                           cudaMemcpyHostToDevice, copy_st_, m.n_kv));
    const size_t tail_w = static_cast<size_t>(pre_tc_) * m.d * 2;
    const size_t tpitch = static_cast<size_t>(tail_cap_) * m.d * 2;
    if (tail_w) {
      VC_CK(cudaMemcpy2DAsync(quant_.ktail + base * tail_cap_ * m.d, tpitch, pre_kt_, tail_w, tail_w, n_slices,
                              cudaMemcpyHostToDevice, copy_st_));
      VC_CK(cudaMemcpy2DAsync(quant_.vtail + base * tail_cap_ * m.d, tpitch, pre_vt_, tail_w, tail_w, n_slices,
                              cudaMemcpyHostToDevice, copy_st_));
    }
  }
  VC_CK(cudaEventRecord(x.done, copy_st_));
  const uint64_t id = next_xfer_++;
  xfers_[id] = x;
  // request state: the first load of a slot opens it; the compressed form
  // carries the quant-tier geometry
  SeqState& s = seqs_[slot];
  if (!s.live) {
    s = SeqState{};
    s.live = true;
    s.committed = pre_T_;
    s.pending = pending;
  }
  if (what == 0) {
    s.n_groups = pre_ng_;
    s.tail_committed = pre_tc_;
  }
  return id;
}

// ------------------------------------------------------------- host tier
uint64_t Engine::swap_begin(int slot, int stage) {
  if (cfg_.full_tier != 1) throw ContractViolation("swap: host tier disabled");
  if (ring_mode()) throw ContractViolation("swap: the chunk-ring engine streams verifies (stream_begin)");
  if (resident(slot)) throw ContractViolation("swap: the slot's full KV is resident (no host copy)");
  scratch_slot_ = -1;
  if (stage < cfg_.resident_slots || stage >= cfg_.n_stage)
    throw ContractViolation("swap: bad staging slot (resident slots own theirs)");
  const SeqState& s = seqs_.at(slot);
  const auto& m = cfg_.model;
  const int n_slices = m.layers * m.n_kv;
  const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
  const size_t pitch = slice_elems * 2;
  const size_t width = static_cast<size_t>(s.committed) * m.d * 2;
  uint16_t* dk = stage_.k + static_cast<size_t>(stage) * n_slices * slice_elems;
  uint16_t* dv = stage_.v + static_cast<size_t>(stage) * n_slices * slice_elems;
  const uint16_t* hk = host_pool_k(slot);
  const uint16_t* hv = host_pool_v(slot);
  // the stage may still be read by an in-flight step on the compute stream
  cudaEvent_t ready;
  VC_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  VC_CK(cudaEventRecord(ready, st_));
  VC_CK(cudaStreamWaitEvent(copy_st_, ready, 0));
  cudaEventDestroy(ready);
  Xfer x{};
  x.bytes = 2.0 * static_cast<double>(width) * n_slices;
  VC_CK(cudaEventCreate(&x.start));
  VC_CK(cudaEventCreate(&x.done));
  VC_CK(cudaEventRecord(x.start, copy_st_));
  if (width > 0) {  // one layer (n_kv slices) of K, then of V, per copy
    for (int l = 0; l < m.layers; ++l) {
      const size_t o = static_cast<size_t>(l) * m.n_kv * slice_elems;
      VC_CK(cudaMemcpy2DAsync(dk + o, pitch, hk + o, pitch, width, m.n_kv, cudaMemcpyHostToDevice, copy_st_));
      VC_CK(cudaMemcpy2DAsync(dv + o, pitch, hv + o, pitch, width, m.n_kv, cudaMemcpyHostToDevice, copy_st_));
    }
  }
  VC_CK(cudaEventRecord(x.done, copy_st_));
  const uint64_t id = next_xfer_++;
  xfers_[id] = x;
  return id;
}

bool Engine::swap_done(uint64_t id) {
  auto it = xfers_.find(id);
  if (it == xfers_.end()) return true;
  cudaError_t e = cudaEventQuery(it->second.done);
  if (e == cudaErrorNotReady) return false;
  check_cuda(e, "swap_done");
  // order later compute after the copy
  VC_CK(cudaStreamWaitEvent(st_, it->second.done, 0));
  float ms = 0.f;
  VC_CK(cudaEventElapsedTime(&ms, it->second.start, it->second.done));
  h2d_ms_ += ms;
  h2d_bytes_ += it->second.bytes;
  cudaEventDestroy(it->second.start);
  cudaEventDestroy(it->second.done);
  xfers_.erase(it);
  return true;
}

void Engine::swap_wait(uint64_t id) {
  auto it = xfers_.find(id);
  if (it == xfers_.end()) return;
  VC_CK(cudaEventSynchronize(it->second.done));
  swap_done(id);
}

// --------------------------------------------- host tier, layer-chunked ring
// The verify of an offloaded request reads its full KV one layer at a time,
// so the reload is streamed in one-layer chunks (n_kv slices of K and of V,
// 134 MB at 32K for Llama-3-8B) into a ring of ring_chunks chunks, and the
// verify forward runs over each range of layers that has landed, its hidden
// state carried in xsave_/sssave_ between ranges.  A chunk is released as
// soon as the range that read it is enqueued (the next copy into it waits on
// ring_free_ on the copy stream), so staging HBM is ring_chunks layers
// instead of whole requests, the link streams back to back, and the verify
// finishes one chunk after the last layer lands.  The reference books the
// reload as bytes over S_r windows (scheduler.cpp:15-23, :96-163); here the
// same booking drives chunk copies.  Batch invariance makes the range-by-range
// forward bit-identical to a whole-window verify (same GEMM split per (N, K),
// same 2048-key attention chunks, rows independent).
// Host pool layout of a packed slot (per slice region of cap*d*2 bytes):
// blocks [0, P) packed back to back at b * PB bytes, rows [128 P, ...) raw at
// their natural row offset (128 P rows * d * 2 bytes >= P * PB: no overlap).
void Engine::host_store_layer(int slot, int l, int craw, int cpk, int n, int P) {
  const auto& m = cfg_.model;
  const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
  const size_t pitch = slice_elems * 2;
  const size_t o = static_cast<size_t>(l) * m.n_kv * slice_elems;
  const size_t PB = packed_block_bytes(m.d);
  const int r0 = std::min(n, P * VC_QGROUP);
  for (int kv = 0; kv < 2; ++kv) {
    uint16_t* raw = (kv ? ring_.v : ring_.k) + static_cast<size_t>(craw) * m.n_kv * slice_elems;
    uint8_t* pk = reinterpret_cast<uint8_t*>((kv ? ring_.v : ring_.k) + static_cast<size_t>(cpk) * m.n_kv * slice_elems);
    if (P > 0) VC_CK(pack_blocks(raw, slice_elems, 0, n, P, m.n_kv, m.d, pk, pitch, pack_overflow_, st_));
  }
  VC_CK(cudaEventRecord(ev_commit_, st_));
  VC_CK(cudaStreamWaitEvent(d2h_st_, ev_commit_, 0));
  for (int kv = 0; kv < 2; ++kv) {
    uint16_t* host = (kv ? host_pool_v(slot) : host_pool_k(slot)) + o;
    uint16_t* raw = (kv ? ring_.v : ring_.k) + static_cast<size_t>(craw) * m.n_kv * slice_elems;
    uint8_t* pk = reinterpret_cast<uint8_t*>((kv ? ring_.v : ring_.k) + static_cast<size_t>(cpk) * m.n_kv * slice_elems);
    if (P > 0)
      VC_CK(cudaMemcpy2DAsync(host, pitch, pk, pitch, P * PB, m.n_kv, cudaMemcpyDeviceToHost, d2h_st_));
    if (n > r0)
      VC_CK(cudaMemcpy2DAsync(host + static_cast<size_t>(r0) * m.d, pitch, raw + static_cast<size_t>(r0) * m.d, pitch,
                              static_cast<size_t>(n - r0) * m.d * 2, m.n_kv, cudaMemcpyDeviceToHost, d2h_st_));
  }
  VC_CK(cudaStreamSynchronize(d2h_st_));  // both chunks are reused by the next layer
}

void Engine::host_load_layer(int slot, int l, int craw, int cpk, int n, int P) {
  const auto& m = cfg_.model;
  const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
  const size_t pitch = slice_elems * 2;
  const size_t o = static_cast<size_t>(l) * m.n_kv * slice_elems;
  const size_t PB = packed_block_bytes(m.d);
  const int r0 = std::min(n, P * VC_QGROUP);
  for (int kv = 0; kv < 2; ++kv) {
    const uint16_t* host = (kv ? host_pool_v(slot) : host_pool_k(slot)) + o;
    uint16_t* raw = (kv ? ring_.v : ring_.k) + static_cast<size_t>(craw) * m.n_kv * slice_elems;
    uint8_t* pk = reinterpret_cast<uint8_t*>((kv ? ring_.v : ring_.k) + static_cast<size_t>(cpk) * m.n_kv * slice_elems);
    if (P > 0) {
      VC_CK(cudaMemcpy2DAsync(pk, pitch, host, pitch, P * PB, m.n_kv, cudaMemcpyHostToDevice, st_));
      VC_CK(unpack_blocks(pk, pitch, P, m.n_kv, m.d, raw, slice_elems, st_));
    }
    if (n > r0)
      VC_CK(cudaMemcpy2DAsync(raw + static_cast<size_t>(r0) * m.d, pitch, host + static_cast<size_t>(r0) * m.d, pitch,
                              static_cast<size_t>(n - r0) * m.d * 2, m.n_kv, cudaMemcpyHostToDevice, st_));
  }
}

double Engine::reload_bytes(int slot) const {
  const auto& m = cfg_.model;
  const SeqState& s = seqs_.at(slot);
  const double slices = 2.0 * m.layers * m.n_kv;  // K and V
  if (ring_mode() && drop_mode()) return slices * (s.drop_T - s.drop_base) * m.d * 2.0;
  const int r0 = std::min(s.committed, s.packed_blocks * VC_QGROUP);
  return slices * (static_cast<double>(s.packed_blocks) * packed_block_bytes(m.d) +
                   static_cast<double>(s.committed - r0) * m.d * 2.0);
}

size_t Engine::staging_bytes() const {
  const auto& m = cfg_.model;
  const size_t slab = static_cast<size_t>(m.n_kv) * full_.cap * m.d * 2 * 2;  // one layer, K and V
  if (cfg_.full_tier != 1) return 0;
  const size_t rot = ring_mode() ? 0 : static_cast<size_t>(cfg_.n_stage - cfg_.resident_slots) * m.layers * slab;
  return rot + (ring_mode() ? static_cast<size_t>(cfg_.ring_chunks + 2 + (land_.k ? cfg_.ring_chunks : 0)) * slab : 0);
}

int Engine::stream_begin(int slot) {
  if (!ring_mode()) throw ContractViolation("stream: the engine has no chunk ring (ring_chunks 0)");
  if (resident(slot)) throw ContractViolation("stream: the slot's full KV is resident (no host copy)");
  const SeqState& s = seqs_.at(slot);
  if (!s.live) throw ContractViolation("stream: slot not live");
  for (const auto& [id, v] : vstreams_)
    if (v.slot == slot) throw ContractViolation("stream: the slot already has a streamed verify");
  int buf = -1;
  for (int i = 0; i < cfg_.max_streams; ++i)
    if (!vbuf_used_[i]) { buf = i; break; }
  if (buf < 0) throw ContractViolation("stream: max_streams streamed verifies already in flight");
  vbuf_used_[buf] = 1;
  VStream v;
  v.slot = slot;
  v.buf = buf;
  v.base = ring_seq_;
  ring_seq_ += cfg_.model.layers;
  v.committed = s.committed;
  // the exact rows accept needs: the residual group + window (quantised
  // tier), or only the window (drop tier: accepted rows are appended there)
  v.origin = drop_mode() ? s.committed : s.n_groups * VC_QGROUP;
  if (drop_mode() && s.drop_T == 0) throw ContractViolation("stream: compress the request first");
  VC_CK(cudaEventCreateWithFlags(&v.ev_final, cudaEventDisableTiming));
  if (drop_mode()) {  // the rebuild reads drop-tier rows the compute stream appended
    VC_CK(cudaEventRecord(ev_commit_, st_));
    VC_CK(cudaStreamWaitEvent(exp_st_, ev_commit_, 0));
  }
  const int id = next_vstream_++;
  vstreams_[id] = std::move(v);
  vs_order_.push_back(id);
  stream_pump();
  return id;
}

void Engine::stream_issue_chunk(VStream& v) {
  const auto& m = cfg_.model;
  const int R = cfg_.ring_chunks;
  const int l = v.issued;
  const int c = static_cast<int>((v.base + l) % R);
  ring_owner_[c] = v.base + l;
  const size_t slice_elems = static_cast<size_t>(full_.cap) * m.d;
  const size_t pitch = slice_elems * 2;
  const size_t width = static_cast<size_t>(v.committed) * m.d * 2;
  const size_t o = static_cast<size_t>(l) * m.n_kv * slice_elems;
  uint16_t* dk = ring_.k + static_cast<size_t>(c) * m.n_kv * slice_elems;
  uint16_t* dv = ring_.v + static_cast<size_t>(c) * m.n_kv * slice_elems;
  // the chunk's previous layer has been read by its verify range
  VC_CK(cudaStreamWaitEvent(copy_st_, ring_free_[c], 0));
  VC_CK(cudaEventRecord(ring_start_[c], copy_st_));
  if (drop_mode()) {
    // only the dropped rows cross the link; the rebuild (position order,
    // kept rows and rows accepted since compress from the drop tier) runs on
    // its own stream as soon as they land
    const SeqState& s = seqs_.at(v.slot);
    const int T = s.drop_T, k = s.drop_base;
    const size_t w = static_cast<size_t>(T - k) * m.d * 2;
    uint16_t* lk = land_.k + static_cast<size_t>(c) * m.n_kv * slice_elems;
    uint16_t* lv = land_.v + static_cast<size_t>(c) * m.n_kv * slice_elems;
    if (w > 0) {
      VC_CK(cudaMemcpy2DAsync(lk, pitch, host_pool_k(v.slot) + o, pitch, w, m.n_kv, cudaMemcpyHostToDevice, copy_st_));
      VC_CK(cudaMemcpy2DAsync(lv, pitch, host_pool_v(v.slot) + o, pitch, w, m.n_kv, cudaMemcpyHostToDevice, copy_st_));
    }
    VC_CK(cudaEventRecord(ring_landed_[c], copy_st_));
    VC_CK(cudaStreamWaitEvent(exp_st_, ring_landed_[c], 0));
    VC_CK(expand_dropped(land_, c, drop_, v.slot * m.layers + l, kept_of(v.slot) + static_cast<size_t>(l) * m.n_kv * k,
                         k, T, v.committed, ring_, c, m.n_kv, m.d, exp_st_));
    ++launches_;
    VC_CK(cudaEventRecord(ring_done_[c], exp_st_));
  } else if (seqs_.at(v.slot).packed_blocks > 0) {
    // packed blocks land in land_[c] and are unpacked into the chunk on the
    // rebuild stream; the raw tail rows go straight into the chunk
    const int P = seqs_.at(v.slot).packed_blocks;
    const int r0 = std::min(v.committed, P * VC_QGROUP);
    const size_t PB = packed_block_bytes(m.d);
    for (int kv = 0; kv < 2; ++kv) {
      const uint16_t* host = (kv ? host_pool_v(v.slot) : host_pool_k(v.slot)) + o;
      uint8_t* lp = reinterpret_cast<uint8_t*>((kv ? land_.v : land_.k) + static_cast<size_t>(c) * m.n_kv * slice_elems);
      uint16_t* dst = kv ? dv : dk;
      VC_CK(cudaMemcpy2DAsync(lp, pitch, host, pitch, P * PB, m.n_kv, cudaMemcpyHostToDevice, copy_st_));
      if (v.committed > r0)
        VC_CK(cudaMemcpy2DAsync(dst + static_cast<size_t>(r0) * m.d, pitch, host + static_cast<size_t>(r0) * m.d, pitch,
                                static_cast<size_t>(v.committed - r0) * m.d * 2, m.n_kv, cudaMemcpyHostToDevice,
                                copy_st_));
    }
    VC_CK(cudaEventRecord(ring_landed_[c], copy_st_));
    VC_CK(cudaStreamWaitEvent(exp_st_, ring_landed_[c], 0));
    for (int kv = 0; kv < 2; ++kv)
      VC_CK(unpack_blocks(reinterpret_cast<const uint8_t*>((kv ? land_.v : land_.k) +
                                                          static_cast<size_t>(c) * m.n_kv * slice_elems),
                          pitch, P, m.n_kv, m.d, kv ? dv : dk, slice_elems, exp_st_));
    launches_ += 2;
    VC_CK(cudaEventRecord(ring_done_[c], exp_st_));
  } else {
    if (width > 0) {
      VC_CK(cudaMemcpy2DAsync(dk, pitch, host_pool_k(v.slot) + o, pitch, width, m.n_kv, cudaMemcpyHostToDevice, copy_st_));
      VC_CK(cudaMemcpy2DAsync(dv, pitch, host_pool_v(v.slot) + o, pitch, width, m.n_kv, cudaMemcpyHostToDevice, copy_st_));
    }
    VC_CK(cudaEventRecord(ring_done_[c], copy_st_));
  }
  ++v.issued;
}

void Engine::stream_pump() {
  // the link serves streams in begin order; a chunk is issued once the ring
  // chunk it maps to has been released by the range that read its previous layer
  const int R = cfg_.ring_chunks;
  for (int id : vs_order_) {
    VStream& v = vstreams_.at(id);
    while (v.issued < cfg_.model.layers && ring_owner_[(v.base + v.issued) % R] < 0) stream_issue_chunk(v);
    if (v.issued < cfg_.model.layers) break;
  }
}

int Engine::stream_layers_done(int id) const { return vstreams_.at(id).done; }

int Engine::stream_advance(int id) {
  VStream& v = vstreams_.at(id);
  const auto& m = cfg_.model;
  const int R = cfg_.ring_chunks;
  if (v.final_enqueued) {
    const cudaError_t e = cudaEventQuery(v.ev_final);
    if (e == cudaErrorNotReady) return 0;
    check_cuda(e, "stream_advance");
    if (v.preds.empty()) {
      const int32_t* p = reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(h_ring_) +
                                                          v.buf * ring_desc_bytes() + ring_desc_bytes() -
                                                          static_cast<size_t>(wrows_) * 4);
      v.preds.assign(p, p + v.x + 1);
    }
    return 1;
  }
  // chunks that have landed, in layer order
  while (v.landed < v.issued) {
    const int c = static_cast<int>((v.base + v.landed) % R);
    const cudaError_t e = cudaEventQuery(ring_done_[c]);
    if (e == cudaErrorNotReady) break;
    check_cuda(e, "stream chunk");
    float ms = 0.f;
    const SeqState& s = seqs_.at(v.slot);
    const bool rebuilt = drop_mode() || s.packed_blocks > 0;  // the link time ends when the rows landed
    VC_CK(cudaEventElapsedTime(&ms, ring_start_[c], rebuilt ? ring_landed_[c] : ring_done_[c]));
    h2d_ms_ += ms;
    if (drop_mode()) {
      h2d_bytes_ += 2.0 * static_cast<double>(s.drop_T - s.drop_base) * m.d * 2 * m.n_kv;
    } else {
      const int r0 = std::min(v.committed, s.packed_blocks * VC_QGROUP);
      h2d_bytes_ += 2.0 * m.n_kv *
                    (static_cast<double>(s.packed_blocks) * packed_block_bytes(m.d) +
                     static_cast<double>(v.committed - r0) * m.d * 2);
    }
    ++v.landed;
  }
  if (v.landed > v.done) {
    if (v.x < 0) {  // the first range fixes the window the verify scores
      const SeqState& s = seqs_.at(v.slot);
      if (s.committed != v.committed) throw ContractViolation("stream: the request committed during its reload");
      if (s.drafted.empty()) throw ContractViolation("stream: no drafted tokens to verify");
      if (static_cast<int>(s.drafted.size()) + 1 > wrows_) throw ContractViolation("stream: window exceeds max_x");
      v.x = static_cast<int>(s.drafted.size());
      v.tokens.assign(1, s.pending);
      v.tokens.insert(v.tokens.end(), s.drafted.begin(), s.drafted.end());
    }
    stream_range(v, v.done, v.landed);
    v.done = v.landed;
    stream_pump();
  }
  return 0;
}

std::vector<int32_t> Engine::stream_preds(int id) const {
  const VStream& v = vstreams_.at(id);
  if (v.preds.empty()) throw ContractViolation("stream: predictions not ready (stream_advance until 1)");
  return v.preds;
}

std::vector<int32_t> Engine::accept_commit_stream(int slot, const std::vector<int32_t>& preds, int id) {
  VStream& v = vstreams_.at(id);
  if (v.slot != slot) throw ContractViolation("stream: slot mismatch");
  if (v.preds.empty()) throw ContractViolation("stream: verify not finished");
  const SeqState& s = seqs_.at(slot);
  if (static_cast<int>(s.drafted.size()) != v.x || s.pending != v.tokens[0] ||
      !std::equal(s.drafted.begin(), s.drafted.end(), v.tokens.begin() + 1))
    throw ContractViolation("stream: the open round is not the window the verify scored");
  const RowSrc src{wbuf_, v.buf, v.origin};
  auto em = accept_commit_from(slot, preds, src, !drop_mode());
  stream_end(id);
  return em;
}

void Engine::stream_end(int id) {
  auto it = vstreams_.find(id);
  if (it == vstreams_.end()) return;
  VStream& v = it->second;
  const int R = cfg_.ring_chunks;
  const bool finished = v.final_enqueued && cudaEventQuery(v.ev_final) == cudaSuccess;
  if (!finished) {
    // abandoned mid-stream: its copies land and its ranges run first, then
    // the chunks it still holds go back to the ring
    VC_CK(cudaStreamSynchronize(copy_st_));
    if (exp_st_) VC_CK(cudaStreamSynchronize(exp_st_));
    VC_CK(cudaStreamSynchronize(st_));
    for (int l = v.done; l < v.issued; ++l) {
      const int c = static_cast<int>((v.base + l) % R);
      if (ring_owner_[c] == v.base + l) ring_owner_[c] = -1;
    }
  }
  if (v.ev_final) cudaEventDestroy(v.ev_final);
  vbuf_used_[v.buf] = 0;
  vs_order_.erase(std::find(vs_order_.begin(), vs_order_.end(), id));
  vstreams_.erase(it);
  stream_pump();
}

// The verify forward of a streamed window over layers [a, b): the same
// kernels as enqueue_forward's verify set, reading layer l's K/V from its ring
// chunk (dense attention over the ring with one layer per chunk), with the
// window's exact K/V rows [origin, committed + x + 1) of each layer copied to
// the stream's window buffer for accept_commit_stream.
void Engine::stream_range(VStream& v, int a, int b) {
  const auto& m = cfg_.model;
  const int L = m.layers, H = m.hidden, F = m.ffn, V = m.vocab, d = m.d;
  const int qkv_n = (m.n_q + 2 * m.n_kv) * d;
  const int R = cfg_.ring_chunks;
  const int n = v.x + 1;
  const int M = bucket_rows(n);
  const int mrv = (n + 3) / 4 * 4;
  const size_t slice_elems = static_cast<size_t>(full_.cap) * d;
  // descriptors: this buf's mapped region (its previous upload has run)
  VC_CK(cudaEventSynchronize(ring_upload_[v.buf]));
  uint8_t* hb = static_cast<uint8_t*>(h_ring_) + v.buf * ring_desc_bytes();
  const uint8_t* db = static_cast<const uint8_t*>(d_hring_) + v.buf * ring_desc_bytes();
  int32_t* h_tok = reinterpret_cast<int32_t*>(hb);
  RowDest* h_rows = reinterpret_cast<RowDest*>(hb + static_cast<size_t>(wrows_) * 4);
  AttnSeq* h_seqs = reinterpret_cast<AttnSeq*>(hb + static_cast<size_t>(wrows_) * (4 + sizeof(RowDest)));
  const int32_t* d_preds = reinterpret_cast<const int32_t*>(db + ring_desc_bytes() - static_cast<size_t>(wrows_) * 4);
  const int c0 = static_cast<int>(v.base % R);
  for (int i = 0; i < M; ++i) {
    h_tok[i] = i < n ? v.tokens[i] : 0;
    h_rows[i] = i < n ? RowDest{4, c0, v.committed + i, v.committed + i} : RowDest{-1, 0, 0, 0};
  }
  for (int l = a; l < b; ++l) {
    AttnSeq q{};
    q.slot = static_cast<int>((v.base + l) % R);
    q.row0 = 0;
    q.n_rows = n;
    q.kv_len = v.committed + n;
    q.part0 = 0;
    h_seqs[l] = q;
  }
  {
    auto dev = [&](const void* h) {
      return reinterpret_cast<const uint32_t*>(db + (static_cast<const uint8_t*>(h) - hb));
    };
    MappedCopy mc{};
    mc.seg[0] = {dev(h_tok), reinterpret_cast<uint32_t*>(tok_in_), M};
    mc.seg[1] = {dev(h_rows), reinterpret_cast<uint32_t*>(rows_dev_), static_cast<int>(M * sizeof(RowDest) / 4)};
    mc.seg[2] = {dev(h_seqs), reinterpret_cast<uint32_t*>(ring_seqs_dev_), static_cast<int>(L * sizeof(AttnSeq) / 4)};
    mc.n = 3;
    mapped_copy_kernel<<<8, 256, 0, st_>>>(mc);
    VC_CK(cudaGetLastError());
    ++launches_;
    VC_CK(cudaEventRecord(ring_upload_[v.buf], st_));
  }
  AttnShape as;
  as.layers = 1;  // one layer per ring chunk: slice = chunk * n_kv + head
  as.n_kv = m.n_kv;
  as.n_rep = m.n_q / m.n_kv;
  as.d = d;
  as.q_stride = qkv_n;
  as.out_stride = m.n_q * d;
  as.out_mp = M;
  as.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d)));
  as.draft_warps = draft_warps_;
  as.draft_min_tasks = draft_min_tasks_;
  float* xs = xsave_ + static_cast<size_t>(v.buf) * wrows_ * H;
  float* sss = sssave_ + static_cast<size_t>(v.buf) * wrows_ * (H / 128);
  if (a == 0) {
    VC_LAUNCH(embed_norm(tok_in_, M, M, w_.embed, H, w_.attn_norm[0], m.eps, x_, xn_, st_));
  } else {  // resume: the residual stream and its per-tile sums of squares after layer a-1
    // (SM copies: a copy-engine D2D would queue behind the chunk reloads)
    MappedCopy mc{};
    mc.seg[0] = {reinterpret_cast<const uint32_t*>(xs), reinterpret_cast<uint32_t*>(x_), M * H};
    mc.seg[1] = {reinterpret_cast<const uint32_t*>(sss), reinterpret_cast<uint32_t*>(ss_part_), M * (H / 128)};
    mc.n = 2;
    mapped_copy_kernel<<<64, 256, 0, st_>>>(mc);
    VC_CK(cudaGetLastError());
    ++launches_;
    VC_LAUNCH(rms_apply(x_, ss_part_, M, M, H, w_.attn_norm[a], m.eps, xn_, st_));
  }
  GemmEpilogue eq;
  eq.kind = Epi::Qkv;
  eq.out_bf16 = qkv_;
  eq.rows = rows_dev_;
  eq.rope_cos = rope_cos_;
  eq.rope_sin = rope_sin_;
  eq.n_q = m.n_q;
  eq.n_kv = m.n_kv;
  eq.d = d;
  eq.layers = L;
  eq.ring = ring_;
  eq.ring_n = R;
  GemmEpilogue er;
  er.kind = Epi::Residual;
  er.x = x_;
  er.ss_part = ss_part_;
  GemmEpilogue es;
  es.kind = Epi::Silu;
  es.out_bf16 = act_;
  for (int l = a; l < b; ++l) {
    const int c = static_cast<int>((v.base + l) % R);
    eq.layer = l;
    VC_LAUNCH(gemm(xn_, M, M, H, w_.wqkv[l], qkv_n, eq, gws_, st_));
    // the window's exact rows of this layer (written just now by the qkv
    // epilogue) and the residual group before them -> the window buffer
    VC_LAUNCH(copy_rows(ring_, c, v.origin, v.committed + n - v.origin, wbuf_, v.buf * L + l, 0, m.n_kv, d, st_));
    VC_LAUNCH(dense_attention(as, ring_, ring_maps_, 0, ring_seqs_dev_ + l, 1, max_chunks_d_, mrv, part_, st_));
    VC_LAUNCH(attention_combine(as, ring_seqs_dev_ + l, 1, max_chunks_d_, mrv, 1, part_, attn_, st_));
    VC_LAUNCH(gemm(attn_, M, M, m.n_q * d, w_.wo[l], H, er, gws_, st_));
    VC_LAUNCH(rms_apply(x_, ss_part_, M, M, H, w_.mlp_norm[l], m.eps, xn_, st_));
    VC_LAUNCH(gemm(xn_, M, M, H, w_.wgu[l], 2 * F, es, gws_, st_));
    VC_LAUNCH(gemm(act_, M, M, F, w_.wd[l], H, er, gws_, st_));
    VC_LAUNCH(rms_apply(x_, ss_part_, M, M, H, l + 1 < L ? w_.attn_norm[l + 1] : w_.final_norm, m.eps, xn_, st_));
  }
  // the range has read its chunks: release them to the link
  for (int l = a; l < b; ++l) {
    const int c = static_cast<int>((v.base + l) % R);
    VC_CK(cudaEventRecord(ring_free_[c], st_));
    ring_owner_[c] = -1;
  }
  if (b < L) {
    MappedCopy mc{};
    mc.seg[0] = {reinterpret_cast<const uint32_t*>(x_), reinterpret_cast<uint32_t*>(xs), M * H};
    mc.seg[1] = {reinterpret_cast<const uint32_t*>(ss_part_), reinterpret_cast<uint32_t*>(sss), M * (H / 128)};
    mc.n = 2;
    mapped_copy_kernel<<<64, 256, 0, st_>>>(mc);
    VC_CK(cudaGetLastError());
    ++launches_;
  } else {
    GemmEpilogue ef;
    ef.kind = Epi::StoreF32;
    ef.out_f32 = logits_;
    VC_LAUNCH(gemm(xn_, M, M, H, w_.lm_head, V, ef, gws_, st_));
    VC_LAUNCH(argmax_rows(logits_, M, V, tok_out_, st_));
    MappedCopy mc{};
    mc.seg[0] = {reinterpret_cast<const uint32_t*>(tok_out_), const_cast<uint32_t*>(reinterpret_cast<const uint32_t*>(d_preds)), n};
    mc.n = 1;
    mapped_copy_kernel<<<1, 256, 0, st_>>>(mc);
    VC_CK(cudaGetLastError());
    ++launches_;
    VC_CK(cudaEventRecord(v.ev_final, st_));
    v.final_enqueued = true;
  }
  (void)slice_elems;
}

}  // namespace vc
