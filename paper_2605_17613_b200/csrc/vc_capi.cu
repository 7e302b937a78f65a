// vc_capi.cu -- extern "C" boundary (include/vc_api.h).  Thin: validates,
// forwards to the engine / host algorithms, maps exceptions to status codes.
#include <algorithm>
#include <vector>
#include <chrono>
#include <cstring>
#include <string>

#include "speckv_b200.hpp"
#include "vc_api.h"
#include "vc_engine.hpp"
#include "vc_topk.h"
#include "vc_tp.h"

#include <memory>

struct vc_engine {
  vc::Engine* impl;
};

int vc_run_scheduled_impl(vc::Engine& en, const int* slots, int n, const vc_sched_desc& sd,
                          int32_t* out, vc_sched_stats* stats);
int vc_run_remote_prefix_impl(vc::Engine& en, const int* slots, int n, const vc_remote_desc& rd,
                              int32_t* out, vc_remote_stats* stats);
int vc_run_decode_fifo_impl(vc::Engine& en, const vc_request_desc* reqs, int n, int K, int32_t* out,
                            vc_loop_metrics* m);

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return VC_OK;
  } catch (const speckv::ConfigError& e) {
    g_err = e.what();
    return VC_ERR_CONFIG;
  } catch (const speckv::ContractError& e) {
    g_err = e.what();
    return VC_ERR_CONTRACT;
  } catch (const vc::ContractViolation& e) {
    g_err = e.what();
    return VC_ERR_CONTRACT;
  } catch (const vc::CudaError& e) {
    g_err = e.what();
    return VC_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VC_ERR_CONTRACT;
  }
}

vc::Engine& E(vc_engine* e) {
  if (e == nullptr || e->impl == nullptr) throw vc::ContractViolation("null engine");
  return *e->impl;
}


}  // namespace

extern "C" {

const char* vc_last_error(void) { return g_err.c_str(); }
int vc_version(void) { return 1; }

int vc_engine_create(const vc_model_desc* model, const vc_runtime_desc* rt, int device,
                     vc_engine** out) {
  return guard([&] {
    if (!model || !rt || !out) throw vc::ContractViolation("vc_engine_create: null argument");
    vc::EngineConfig c;
    c.model.vocab = model->vocab;
    c.model.hidden = model->hidden;
    c.model.layers = model->layers;
    c.model.n_q = model->n_q;
    c.model.n_kv = model->n_kv;
    c.model.d = model->d_head;
    c.model.ffn = model->ffn;
    c.model.rope_theta = model->rope_theta;
    c.model.eps = model->rms_eps;
    if (c.model.vocab < 2 || c.model.hidden < 64 || c.model.layers < 1 || c.model.ffn < 64 ||
        c.model.hidden % 64 != 0 || c.model.ffn % 64 != 0)
      throw speckv::ConfigError("model: unsupported shape (hidden, ffn must be multiples of 64)");
    c.max_slots = rt->max_slots;
    c.max_ctx = rt->max_ctx;
    c.max_x = rt->max_x;
    c.quant_bits = rt->quant_bits;
    c.full_tier = rt->full_tier;
    c.n_stage = rt->n_stage;
    c.max_verify = rt->max_verify;
    c.use_graphs = rt->use_graphs;
    c.drop_ratio = rt->drop_ratio;
    c.drop_window = rt->drop_window;
    c.resident_slots = rt->resident_slots;
    c.draft_depth = rt->draft_depth > 1 ? rt->draft_depth : 1;
    c.ring_chunks = rt->ring_chunks;
    c.max_streams = rt->max_streams > 0 ? rt->max_streams : 2;
    c.drop_score = rt->drop_score;
    c.snap_pool = rt->snap_pool > 0 ? rt->snap_pool : 7;
    c.snap_recent = rt->snap_recent >= 0 ? rt->snap_recent : 32;
    c.host_pack = rt->host_pack < 0 ? 0 : (rt->host_pack >= 2 ? rt->host_pack : 1);
    if (c.drop_window < 0 || (c.drop_window > 0 && c.drop_ratio <= 0.0))
      throw speckv::ConfigError("compressor: drop_window needs the drop-topk compressor");
    c.tp_size = rt->tp_size > 1 ? rt->tp_size : 1;
    c.tp_rank = c.tp_size > 1 ? rt->tp_rank : 0;
    if (c.tp_size > 1) {  // this rank's shard of the heads and of the MLP
      const int T = c.tp_size;
      if (c.tp_rank < 0 || c.tp_rank >= T) throw speckv::ConfigError("tensor parallel: rank out of range");
      if (c.model.n_kv % T || c.model.n_q % T || c.model.ffn % (64 * T))
        throw speckv::ConfigError("tensor parallel: n_kv, n_q and ffn/64 must divide by tp_size");
      c.model.n_q /= T;
      c.model.n_kv /= T;
      c.model.ffn /= T;
    }
    if (c.drop_ratio < 0.0 || c.drop_ratio >= 1.0)
      throw speckv::ConfigError("compressor: drop ratio must be in (0, 1)");
    if (c.drop_ratio > 0.0 && c.quant_bits != 0)  // speckv::check_mode_exclusivity (compressor.cpp:245-254)
      throw speckv::ConfigError("compressor: token dropping and quantization are mutually exclusive");
    if (c.max_slots < 1 || c.max_ctx < 1 || c.max_x < 1 || c.max_verify < 1)
      throw speckv::ConfigError("runtime: sizes must be >= 1");
    auto* h = new vc_engine{nullptr};
    try {
      h->impl = new vc::Engine(c, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

struct vc_tp_group {
  std::shared_ptr<vc::LoopbackGroup> g;
};

int vc_nccl_get_unique_id(uint8_t* out128) {
  return guard([&] {
    if (!out128) throw vc::ContractViolation("nccl id: null buffer");
    if (!vc::nccl_unique_id(out128)) throw vc::ContractViolation("libnccl.so.2 not found");
  });
}

int vc_engine_attach_nccl(vc_engine* e, const uint8_t* id) {
  return guard([&] {
    vc::Engine& en = E(e);
    en.attach_collective(vc::make_nccl(id, en.config().tp_rank, en.config().tp_size));
  });
}

int vc_engine_geometry(vc_engine* e, int* layers, int* kv_heads) {
  return guard([&] {
    const auto& m = E(e).model();
    if (layers) *layers = m.layers;
    if (kv_heads) *kv_heads = m.n_kv;
  });
}

int vc_tp_collective_bench(vc_engine* e, int rows, int reps, double* us) {
  return guard([&] {
    const double v = E(e).collective_bench(rows, reps);
    if (us) *us = v;
  });
}

int vc_tp_loopback_create(int size, vc_tp_group** out) {
  return guard([&] {
    if (!out) throw vc::ContractViolation("loopback: null out");
    *out = new vc_tp_group{vc::make_loopback_group(size)};
  });
}

int vc_tp_loopback_destroy(vc_tp_group* g) {
  return guard([&] { delete g; });
}

int vc_engine_attach_loopback(vc_engine* e, vc_tp_group* g) {
  return guard([&] {
    if (!g) throw vc::ContractViolation("loopback: null group");
    vc::Engine& en = E(e);
    en.attach_collective(vc::make_loopback(g->g, en.config().tp_rank));
  });
}

int vc_engine_destroy(vc_engine* e) {
  return guard([&] {
    if (!e) return;
    delete e->impl;
    delete e;
  });
}

int vc_engine_init_weights(vc_engine* e, uint64_t seed, float stddev) {
  return guard([&] { E(e).init_weights_random(seed, stddev); });
}

int vc_engine_init_weights_scaled(vc_engine* e, uint64_t seed, float stddev, float resid_std,
                                  float q_std) {
  return guard([&] { E(e).init_weights_random(seed, stddev, resid_std, q_std); });
}

int vc_engine_load_weights(vc_engine* e, const uint16_t* embed, const uint16_t* const* attn_norm,
                           const uint16_t* const* wqkv, const uint16_t* const* wo,
                           const uint16_t* const* mlp_norm, const uint16_t* const* wgate,
                           const uint16_t* const* wup, const uint16_t* const* wdown,
                           const uint16_t* final_norm, const uint16_t* lm_head) {
  return guard([&] {
    E(e).load_weights(embed, attn_norm, wqkv, wo, mlp_norm, wgate, wup, wdown, final_norm, lm_head);
  });
}

int vc_engine_stats(vc_engine* e, uint64_t* launches, uint64_t* weight_bytes) {
  return guard([&] {
    if (launches) *launches = E(e).launches();
    if (weight_bytes) *weight_bytes = E(e).weight_bytes();
  });
}

int vc_engine_timing(vc_engine* e, double* device_ms, int64_t* steps, int reset) {
  return guard([&] {
    vc::Engine& en = E(e);
    if (device_ms) *device_ms = en.device_ms();
    if (steps) *steps = en.steps();
    if (reset) en.reset_timing();
  });
}

int vc_kernel_bench(vc_engine* e, int kind, const int* slots, int n, int reps, double* ms,
                    double* bytes) {
  return guard([&] {
    if (reps < 1 || n < 1) throw speckv::ConfigError("kernel_bench: reps and n must be >= 1");
    E(e).kernel_bench(kind, std::vector<int>(slots, slots + n), reps, ms, bytes);
  });
}

int vc_request_add_synthetic(vc_engine* e, int slot, int n_ctx, int32_t first_token, uint64_t seed,
                             int outlier_channels, float outlier_scale) {
  return guard([&] { E(e).add_request_synthetic(slot, n_ctx, first_token, seed, outlier_channels, outlier_scale); });
}

int vc_request_add_kv(vc_engine* e, int slot, int n_ctx, int32_t first_token, const uint16_t* k,
                      const uint16_t* v) {
  return guard([&] { E(e).add_request_kv(slot, n_ctx, first_token, k, v); });
}

int vc_request_prefill(vc_engine* e, int slot, const int32_t* prompt, int n) {
  return guard([&] { E(e).add_request_prefill(slot, prompt, n); });
}

int vc_request_release(vc_engine* e, int slot) {
  return guard([&] { E(e).release(slot); });
}

int vc_request_state(vc_engine* e, int slot, vc_seq_state* out) {
  return guard([&] {
    const vc::SeqState& s = E(e).seq(slot);
    out->live = s.live;
    out->committed = s.committed;
    out->pending = s.pending;
    out->n_groups = s.n_groups;
    out->tail_committed = s.tail_committed;
    out->draft_len = s.draft_len;
    out->drop_base = s.drop_base;
    out->drop_len = s.drop_len;
  });
}

int vc_request_history(vc_engine* e, int slot, int32_t* out, int cap, int* n) {
  return guard([&] {
    const auto& h = E(e).seq(slot).history;
    *n = static_cast<int>(h.size());
    std::memcpy(out, h.data(), sizeof(int32_t) * std::min<size_t>(h.size(), cap));
  });
}

namespace {
void fill_meta(vc::Engine& en, int slot, vc_compressed_meta* out);
}

int vc_compress(vc_engine* e, int slot, vc_compressed_meta* out) {
  return guard([&] {
    vc::Engine& en = E(e);
    en.compress(slot);
    fill_meta(en, slot, out);
  });
}

// speckv::compress(spec, shape, ratio, seed) (compressor.hpp:70-71) on the
// engine's compressed tier.  The engine's tier is fixed at creation (quant
// bits or a drop tier sized for drop_ratio); the spec must fit it:
//   quant-uniform  spec.bits == quant_bits (KIVI codes of every position);
//   drop-uniform / drop-window  the reference's own drop indices
//     (speckv::compress, compressor.cpp:152-177 -- bit-identical, seeded by
//     `seed`), complemented to kept sets and gathered into the drop tier;
//   drop-topk  keep llround(ratio*T) positions per (layer, head) by score.
int vc_compress_spec(vc_engine* e, int slot, const vc_compressor_spec* cs, double ratio, uint64_t seed,
                     vc_compressed_meta* out) {
  return guard([&] {
    vc::Engine& en = E(e);
    if (!cs) throw vc::ContractViolation("compress: null spec");
    const auto& cfg = en.config();
    const auto& m = en.model();
    if (cs->mode != 0) throw speckv::ConfigError("compress: online mode goes through vc_update_window");
    if (cs->kind == 2) {  // quant-uniform
      if (cs->bits < 1 || cs->bits > 16) throw speckv::ConfigError("compressor.bits out of [1,16]");
      if (cfg.quant_bits == 0 || cs->bits != cfg.quant_bits)
        throw vc::ContractViolation("compress: the engine's quantised tier has another bit width");
      en.compress(slot);
    } else if (cs->kind == 0 || cs->kind == 1 || cs->kind == 3) {
      if (!en.drop_mode()) throw vc::ContractViolation("compress: token-dropping spec on an engine without a drop tier");
      if (!(ratio > 0.0 && ratio < 1.0)) throw speckv::ConfigError("compress: ratio out of (0,1)");
      const int T = en.seq(slot).committed;
      if (cs->kind == 3) {
        en.compress_as(slot, ratio, nullptr, 0);
      } else {
        speckv::CompressorSpec spec;
        spec.kind = cs->kind == 0 ? speckv::CompressorKind::DropUniform : speckv::CompressorKind::DropWindow;
        spec.ratio = ratio;
        spec.window = cs->window > 0 ? cs->window : 8;
        spec.sink_tokens = cs->sink_tokens;
        speckv::KvShape shape{m.layers, m.n_kv, T, static_cast<speckv::Bytes>(m.d) * 2 * 2};
        const speckv::CompressedKVMeta meta = speckv::compress(spec, shape, ratio, seed);
        const int64_t k = meta.retained_tokens(shape, 0);
        std::vector<int32_t> kept(static_cast<size_t>(m.layers) * m.n_kv * k);
        std::vector<uint8_t> dropped(static_cast<size_t>(T));
        for (int l = 0; l < m.layers; ++l)
          for (int h = 0; h < m.n_kv; ++h) {
            std::fill(dropped.begin(), dropped.end(), 0);
            for (int64_t p : meta.dropped_indices[l][h]) dropped[static_cast<size_t>(p)] = 1;
            int32_t* dst = kept.data() + (static_cast<size_t>(l) * m.n_kv + h) * k;
            int64_t j = 0;
            for (int t = 0; t < T; ++t)
              if (!dropped[t]) dst[j++] = t;
            if (j != k) throw vc::ContractViolation("compress: kept count differs from the shape law");
          }
        en.compress_as(slot, ratio, kept.data(), static_cast<int>(k));
      }
    } else {
      throw speckv::ConfigError("compress: unknown compressor kind");
    }
    fill_meta(en, slot, out);
  });
}

namespace {
void fill_meta(vc::Engine& en, int slot, vc_compressed_meta* out) {
    const auto& m = en.model();
    const vc::SeqState& s = en.seq(slot);
    if (en.drop_mode()) {
      const speckv::Bytes bpt = static_cast<speckv::Bytes>(m.d) * 2 * 2;
      if (out) {
        out->bit_scheme = 16;
        out->retained_tokens = s.drop_len;
        out->payload_bytes = static_cast<int64_t>(s.drop_len) * m.layers * m.n_kv * bpt;
        out->full_bytes = static_cast<int64_t>(s.committed) * m.layers * m.n_kv * bpt;
        out->aux_bytes = 0;
        out->n_groups = 0;
        out->tail_tokens = 0;
      }
      return;
    }
    // size law of speckv::compress for quant-uniform (compressor.cpp:144-150)
    speckv::CompressorSpec spec;
    spec.kind = speckv::CompressorKind::QuantUniform;
    spec.bits = en.config().quant_bits;
    speckv::KvShape shape{m.layers, m.n_kv, s.committed, static_cast<speckv::Bytes>(m.d) * 2 * 2};
    speckv::CompressedKVMeta meta = speckv::compress(spec, shape, 0.0, 0);
    if (out) {
      out->bit_scheme = meta.bit_scheme;
      out->payload_bytes = meta.payload_bytes;
      out->full_bytes = shape.full_bytes();
      const int64_t groups = static_cast<int64_t>(s.n_groups) * m.layers * m.n_kv;
      out->aux_bytes = groups * (static_cast<int64_t>(m.d) * 4 + VC_QGROUP * 4);
      out->n_groups = s.n_groups;
      out->tail_tokens = s.tail_committed;
      out->retained_tokens = s.committed;
    }
}
}  // namespace

int vc_drop_kept(vc_engine* e, int layer, int head, int32_t* out, int cap, int* n) {
  return guard([&] {
    vc::Engine& en = E(e);
    const auto& m = en.model();
    if (!en.drop_mode()) throw vc::ContractViolation("drop_kept: no drop-topk tier");
    if (layer < 0 || layer >= m.layers || head < 0 || head >= m.n_kv) throw vc::ContractViolation("drop_kept: bad slice");
    const int k = en.last_kept_k();
    if (n) *n = k;
    if (out && k > 0) {
      if (cap < k) throw vc::ContractViolation("drop_kept: capacity");
      vc::check_cuda(cudaStreamSynchronize(en.stream()), "drop_kept");
      vc::check_cuda(cudaMemcpy(out, en.last_kept_device() + (static_cast<size_t>(layer) * m.n_kv + head) * k,
                                static_cast<size_t>(k) * 4, cudaMemcpyDeviceToHost), "drop_kept");
    }
  });
}

int vc_compressed_geometry(vc_engine* e, int* group, int* words_per_group, int* tail_cap,
                           int* max_groups) {
  return guard([&] {
    vc::Engine& en = E(e);
    const auto q = en.quant_pool();
    if (group) *group = VC_QGROUP;
    if (words_per_group) *words_per_group = static_cast<int>(vc::quant_group_words(en.model().d, en.config().quant_bits));
    if (tail_cap) *tail_cap = q.tail_cap;
    if (max_groups) *max_groups = q.cap / VC_QGROUP;
  });
}

int vc_compressed_read(vc_engine* e, int slot, int layer, int head, uint32_t* kcodes, uint32_t* ksz,
                       uint32_t* vcodes, uint32_t* vsz, uint16_t* ktail, uint16_t* vtail) {
  return guard([&] {
    vc::Engine& en = E(e);
    const auto& m = en.model();
    const auto q = en.quant_pool();
    if (en.config().quant_bits == 0) throw vc::ContractViolation("no compressed tier");
    const size_t slice = (static_cast<size_t>(slot) * m.layers + layer) * m.n_kv + head;
    const int bits = en.config().quant_bits;
    const size_t groups = q.cap / VC_QGROUP;
    const size_t rw = vc::quant_record_words(m.d, bits), uw = vc::quant_unit_words(m.d, bits);
    const size_t ucw = vc::quant_unit_code_words(m.d, bits), gw = vc::quant_group_words(m.d, bits);
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst) vc::check_cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "compressed_read");
    };
    // de-interleave the group records into the flat per-stream layout of the ABI
    std::vector<uint32_t> recs(groups * rw);
    cp(recs.data(), q.rec + slice * groups * rw, recs.size() * 4);
    for (size_t g = 0; g < groups; ++g) {
      const uint32_t* r = recs.data() + g * rw;
      if (ksz) std::copy(r, r + m.d, ksz + g * m.d);
      for (int u = 0; u < VC_QGROUP / VC_QUNIT; ++u) {
        const uint32_t* ur = r + m.d + u * uw;
        if (kcodes) std::copy(ur, ur + ucw, kcodes + g * gw + u * ucw);
        if (vcodes) std::copy(ur + ucw, ur + 2 * ucw, vcodes + g * gw + u * ucw);
        if (vsz) std::copy(ur + 2 * ucw, ur + 2 * ucw + VC_QUNIT, vsz + g * VC_QGROUP + u * VC_QUNIT);
      }
    }
    cp(ktail, q.ktail + slice * q.tail_cap * m.d, static_cast<size_t>(q.tail_cap) * m.d * 2);
    cp(vtail, q.vtail + slice * q.tail_cap * m.d, static_cast<size_t>(q.tail_cap) * m.d * 2);
  });
}

int64_t vc_drop_indices(int kind, int layers, int heads, int64_t tokens, double ratio, uint64_t seed,
                        int sink_tokens, int64_t* out) {
  int64_t drop = -1;
  int rc = guard([&] {
    speckv::CompressorSpec spec;
    spec.kind = kind == 0 ? speckv::CompressorKind::DropUniform : speckv::CompressorKind::DropWindow;
    spec.ratio = ratio;
    spec.sink_tokens = sink_tokens;
    speckv::KvShape shape{layers, heads, tokens, 2};
    auto meta = speckv::compress(spec, shape, ratio, seed);
    drop = meta.dropped_indices.empty() || meta.dropped_indices[0].empty()
               ? 0
               : static_cast<int64_t>(meta.dropped_indices[0][0].size());
    if (out)
      for (int l = 0; l < layers; ++l)
        for (int h = 0; h < heads; ++h)
          std::memcpy(out + (static_cast<size_t>(l) * heads + h) * drop,
                      meta.dropped_indices[l][h].data(), sizeof(int64_t) * drop);
  });
  return rc == VC_OK ? drop : -rc;
}

int vc_update_window(int heads, int window, int sink_tokens, int n_req, const int64_t* tokens,
                     const int64_t* req_begin, const int64_t* req_end, const int64_t* already,
                     int64_t* out, int64_t cap, int64_t* n_new) {
  return guard([&] {
    speckv::CompressorSpec spec;
    spec.kind = speckv::CompressorKind::DropWindow;
    spec.mode = speckv::CompressorMode::Online;
    spec.ratio = 0.5;
    spec.window = window;
    spec.sink_tokens = sink_tokens;
    spec.validate();
    std::vector<speckv::OnlineRequestKv> batch(n_req);
    std::vector<std::pair<int64_t, int64_t>> offs;
    for (int i = 0; i < n_req; ++i) {
      batch[i].shape = speckv::KvShape{1, heads, tokens[i], 2};
      batch[i].dropped_indices.assign(1, std::vector<std::vector<int64_t>>(heads));
      for (int h = 0; h < heads; ++h)
        for (int64_t k = 0; k < already[i]; ++k) batch[i].dropped_indices[0][h].push_back(sink_tokens + k);
      offs.emplace_back(req_begin[i], req_end[i]);
    }
    auto res = speckv::update(spec, 0, batch, offs);
    for (int i = 0; i < n_req; ++i) {
      n_new[i] = static_cast<int64_t>(res[i][0].size());
      for (int h = 0; h < heads; ++h)
        for (int64_t k = 0; k < n_new[i] && k < cap; ++k) out[(static_cast<size_t>(i) * heads + h) * cap + k] = res[i][h][k];
    }
  });
}

int vc_topk_select(const float* scores, int rows, int T, int k, int32_t* kept, void* stream) {
  return guard([&] {
    if (k < 1 || k > T) throw speckv::ConfigError("topk: k out of [1, T]");
    vc::check_cuda(vc::topk_select(scores, rows, T, k, kept, static_cast<cudaStream_t>(stream)), "topk_select");
  });
}

int vc_pack_roundtrip(const uint16_t* src, int n_rows, int n_slices, int d, uint16_t* out, int* overflow,
                      void* stream) {
  return guard([&] {
    auto st = static_cast<cudaStream_t>(stream);
    const int nb = (n_rows + 127) / 128;
    const size_t PB = vc::packed_block_bytes(d);
    uint8_t* buf = nullptr;
    int* ovf = nullptr;
    vc::check_cuda(cudaMalloc(&buf, static_cast<size_t>(n_slices) * nb * PB), "cudaMalloc");
    vc::check_cuda(cudaMalloc(&ovf, sizeof(int)), "cudaMalloc");
    vc::check_cuda(cudaMemsetAsync(ovf, 0, sizeof(int), st), "memset");
    vc::check_cuda(vc::pack_blocks(src, static_cast<size_t>(n_rows) * d, 0, n_rows, nb, n_slices, d, buf, nb * PB, ovf,
                                   st), "pack_blocks");
    vc::check_cuda(vc::unpack_blocks(buf, nb * PB, nb, n_slices, d, out, static_cast<size_t>(nb) * 128 * d, st),
                   "unpack_blocks");
    vc::check_cuda(cudaMemcpyAsync(overflow, ovf, sizeof(int), cudaMemcpyDeviceToHost, st), "copy");
    vc::check_cuda(cudaStreamSynchronize(st), "sync");
    cudaFree(buf);
    cudaFree(ovf);
  });
}

int vc_key_scores(const uint16_t* keys, int rows, int T, int d, const float* w, float* scores,
                  void* stream) {
  return guard([&] {
    vc::check_cuda(vc::key_scores(keys, rows, T, d, static_cast<size_t>(T) * d, w, scores,
                                  static_cast<cudaStream_t>(stream)), "key_scores");
  });
}

int vc_argmax_rows(const float* logits, int rows, int n, int32_t* out, void* stream) {
  return guard([&] {
    if (rows < 1 || n < 1) throw speckv::ConfigError("argmax: empty logits");
    vc::check_cuda(vc::argmax_rows(logits, rows, n, out, static_cast<cudaStream_t>(stream)), "argmax_rows");
  });
}

// ------------------------------------------------------------------ steps
int vc_step(vc_engine* e, const vc_step_item* items, int n, int32_t* out_rows, float* logits) {
  return guard([&] {
    std::vector<vc::StepItem> its(n);
    for (int i = 0; i < n; ++i) {
      its[i].slot = items[i].slot;
      its[i].mode = static_cast<vc::RowMode>(items[i].mode);
      its[i].tokens.assign(items[i].tokens, items[i].tokens + items[i].n_tokens);
      its[i].stage = items[i].stage;
    }
    std::vector<int32_t> out;
    E(e).run_step(its, out, logits);
    std::memcpy(out_rows, out.data(), out.size() * sizeof(int32_t));
  });
}

int vc_decode_step(vc_engine* e, const int* slots, int n, int32_t* out_tokens) {
  return guard([&] {
    vc::Engine& en = E(e);
    std::vector<vc::StepItem> its(n);
    for (int i = 0; i < n; ++i) {
      its[i].slot = slots[i];
      its[i].mode = vc::RowMode::Decode;
      its[i].tokens = {en.seq(slots[i]).pending};
    }
    std::vector<int32_t> out;
    en.run_step(its, out);
    for (int i = 0; i < n; ++i) {
      en.commit_decode(slots[i], out[i]);
      out_tokens[i] = out[i];
    }
  });
}

int vc_draft_step(vc_engine* e, const int* slots, int n, int32_t* out_tokens) {
  return guard([&] {
    vc::Engine& en = E(e);
    std::vector<vc::StepItem> its(n);
    for (int i = 0; i < n; ++i) {
      const vc::SeqState& s = en.seq(slots[i]);
      its[i].slot = slots[i];
      its[i].mode = vc::RowMode::Draft;
      its[i].tokens = {s.drafted.empty() ? s.pending : s.drafted.back()};
    }
    std::vector<int32_t> out;
    en.run_step(its, out);
    for (int i = 0; i < n; ++i) {
      en.push_draft(slots[i], out[i]);
      out_tokens[i] = out[i];
    }
  });
}

int vc_verify(vc_engine* e, const int* slots, int n, const int* stages, int32_t* preds) {
  return guard([&] {
    vc::Engine& en = E(e);
    std::vector<vc::StepItem> its(n);
    for (int i = 0; i < n; ++i) {
      const vc::SeqState& s = en.seq(slots[i]);
      its[i].slot = slots[i];
      its[i].mode = vc::RowMode::Verify;
      its[i].tokens.push_back(s.pending);
      its[i].tokens.insert(its[i].tokens.end(), s.drafted.begin(), s.drafted.end());
      its[i].stage = stages ? stages[i] : -1;
    }
    std::vector<int32_t> out;
    en.run_step(its, out);
    std::memcpy(preds, out.data(), out.size() * sizeof(int32_t));
  });
}

int vc_accept(const int32_t* drafted, const int32_t* preds, int x, int32_t* accepted, int* n_accepted,
              int* first_mismatch, int* bonus) {
  return guard([&] {
    auto r = speckv::accept(std::span<const int32_t>(drafted, x), std::span<const int32_t>(preds, x + 1));
    std::memcpy(accepted, r.accepted.data(), r.accepted.size() * sizeof(int32_t));
    *n_accepted = static_cast<int>(r.accepted.size());
    *first_mismatch = r.first_mismatch.value_or(0);
    *bonus = r.bonus_used ? 1 : 0;
  });
}

int vc_accept_commit(vc_engine* e, int slot, const int32_t* preds, int stage, int32_t* emitted,
                     int* n_emitted) {
  return guard([&] {
    vc::Engine& en = E(e);
    const int x = static_cast<int>(en.seq(slot).drafted.size());
    std::vector<int32_t> p(preds, preds + x + 1);
    auto em = en.accept_commit(slot, p, stage);
    std::memcpy(emitted, em.data(), em.size() * sizeof(int32_t));
    *n_emitted = static_cast<int>(em.size());
  });
}

int vc_swap_begin(vc_engine* e, int slot, int stage, uint64_t* transfer_id) {
  return guard([&] { *transfer_id = E(e).swap_begin(slot, stage); });
}

int vc_swap_poll(vc_engine* e, uint64_t transfer_id, int* done) {
  return guard([&] { *done = E(e).swap_done(transfer_id) ? 1 : 0; });
}

int vc_stream_begin(vc_engine* e, int slot, int* id) {
  return guard([&] { *id = E(e).stream_begin(slot); });
}

int vc_stream_advance(vc_engine* e, int id, int* done, int32_t* preds) {
  return guard([&] {
    vc::Engine& en = E(e);
    en.stream_pump();
    *done = en.stream_advance(id);
    if (*done && preds) {
      const auto p = en.stream_preds(id);
      std::memcpy(preds, p.data(), p.size() * sizeof(int32_t));
    }
  });
}

int vc_stream_accept(vc_engine* e, int slot, int id, int32_t* emitted, int* n_emitted) {
  return guard([&] {
    vc::Engine& en = E(e);
    auto em = en.accept_commit_stream(slot, en.stream_preds(id), id);
    std::memcpy(emitted, em.data(), em.size() * sizeof(int32_t));
    *n_emitted = static_cast<int>(em.size());
  });
}

int vc_stream_abort(vc_engine* e, int id) {
  return guard([&] { E(e).stream_end(id); });
}

int vc_drop_scores(vc_engine* e, int layer, int head, float* out, int n) {
  return guard([&] { E(e).drop_scores(layer, head, out, n); });
}

int vc_obs_query(vc_engine* e, int layer, uint16_t* out) {
  return guard([&] { E(e).obs_query(layer, out); });
}

int vc_engine_staging_bytes(vc_engine* e, int64_t* bytes) {
  return guard([&] { *bytes = static_cast<int64_t>(E(e).staging_bytes()); });
}

// ---------------------------------------------------------- remote prefix
int vc_prefix_store(vc_engine* e, int slot) {
  return guard([&] {
    const auto& c = E(e).config();
    if (c.full_tier != 0) throw speckv::ConfigError("remote prefix: needs the HBM full tier (full_tier 0)");
    if (c.quant_bits == 0) throw speckv::ConfigError("remote prefix: needs the quantising compressor");
    E(e).prefix_store(slot);
  });
}

int vc_prefix_load(vc_engine* e, int slot, int what, int32_t first_token, uint64_t* transfer_id) {
  return guard([&] { *transfer_id = E(e).prefix_load(slot, what, first_token); });
}

int vc_run_remote_prefix(vc_engine* e, const int* slots, int n, const vc_remote_desc* rd, int32_t* out,
                         vc_remote_stats* stats) {
  return guard([&] {
    if (!rd) throw vc::ContractViolation("vc_run_remote_prefix: null descriptor");
    vc_run_remote_prefix_impl(E(e), slots, n, *rd, out, stats);
  });
}

// ------------------------------------------------------------------ loops
int vc_run_decode(vc_engine* e, const int* slots, int n, int K, int32_t* out, double* ms) {
  return guard([&] {
    vc::Engine& en = E(e);
    std::vector<vc::StepItem> its(n);
    std::vector<int32_t> row;
    // *ms: device time of the loop -- one event pair on the compute stream
    cudaEvent_t w0, w1;
    vc::check_cuda(cudaEventCreate(&w0), "event");
    vc::check_cuda(cudaEventCreate(&w1), "event");
    vc::check_cuda(cudaEventRecord(w0, en.stream()), "event");
    for (int k = 0; k < K; ++k) {
      for (int i = 0; i < n; ++i) {
        its[i].slot = slots[i];
        its[i].mode = vc::RowMode::Decode;
        its[i].tokens = {en.seq(slots[i]).pending};
      }
      en.run_step(its, row);
      for (int i = 0; i < n; ++i) {
        en.commit_decode(slots[i], row[i]);
        out[static_cast<size_t>(i) * K + k] = row[i];
      }
    }
    vc::check_cuda(cudaEventRecord(w1, en.stream()), "event");
    vc::check_cuda(cudaEventSynchronize(w1), "event");
    float dms = 0.f;
    vc::check_cuda(cudaEventElapsedTime(&dms, w0, w1), "event");
    cudaEventDestroy(w0);
    cudaEventDestroy(w1);
    if (ms) *ms = dms;
  });
}

namespace {

// Lock-step rounds (speckv::run_speculative, specloop.cpp:58-79).  With
// ngram > 0 the round's drafter is composed: a request whose emitted history
// repeats its last `ngram` tokens takes the n-gram continuation as its draft
// (no draft steps); the others draft x tokens over the compressed tier.  Both
// kinds verify in the same full-KV pass; losslessness is unaffected because
// the verifier alone decides what is emitted.
void speculative_loop(vc::Engine& en, const int* slots, int n, int K, int x, int ngram, int32_t* out,
                      int32_t* rounds, int max_rounds, int* n_rounds, int* ngram_rounds, double* ms) {
  if (x < 1 || x > en.config().max_x) throw speckv::ConfigError("run_speculative: x out of [1, max_x]");
  if (en.config().full_tier != 0) throw vc::ContractViolation("lock-step loop needs the HBM full tier");
  std::vector<int> produced(n, 0), nr(n, 0), ngr(n, 0);
  std::vector<vc::StepItem> its;
  std::vector<int32_t> row;
  cudaEvent_t w0, w1;  // *ms: device time of the loop (one event pair on the compute stream)
  vc::check_cuda(cudaEventCreate(&w0), "event");
  vc::check_cuda(cudaEventCreate(&w1), "event");
  vc::check_cuda(cudaEventRecord(w0, en.stream()), "event");
  for (;;) {
    std::vector<int> act, model;
    for (int i = 0; i < n; ++i)
      if (produced[i] < K) act.push_back(i);
    if (act.empty()) break;
    for (int i : act) {
      const auto prop = vc::ngram_proposal(en.seq(slots[i]).history, ngram, x);
      if (prop.empty()) {
        model.push_back(i);
        continue;
      }
      for (int32_t t : prop) en.push_draft(slots[i], t);  // drafted without a model step
      ++ngr[i];
    }
    for (int j = 0; j < x && !model.empty(); ++j) {  // x draft steps over the compressed tier
      its.assign(model.size(), vc::StepItem{});
      for (size_t a = 0; a < model.size(); ++a) {
        const vc::SeqState& s = en.seq(slots[model[a]]);
        its[a].slot = slots[model[a]];
        its[a].mode = vc::RowMode::Draft;
        its[a].tokens = {s.drafted.empty() ? s.pending : s.drafted.back()};
      }
      en.run_step(its, row);
      for (size_t a = 0; a < model.size(); ++a) en.push_draft(slots[model[a]], row[a]);
    }
    its.assign(act.size(), vc::StepItem{});  // one verify pass over the full KV
    for (size_t a = 0; a < act.size(); ++a) {
      const vc::SeqState& s = en.seq(slots[act[a]]);
      its[a].slot = slots[act[a]];
      its[a].mode = vc::RowMode::Verify;
      its[a].tokens.push_back(s.pending);
      its[a].tokens.insert(its[a].tokens.end(), s.drafted.begin(), s.drafted.end());
    }
    en.run_step(its, row);
    size_t off = 0;
    for (size_t a = 0; a < act.size(); ++a) {
      const int i = act[a];
      const size_t xi = en.seq(slots[i]).drafted.size();
      std::vector<int32_t> p(row.begin() + off, row.begin() + off + xi + 1);
      off += xi + 1;
      auto em = en.accept_commit(slots[i], p);
      if (rounds && nr[i] < max_rounds) rounds[static_cast<size_t>(i) * max_rounds + nr[i]] = static_cast<int32_t>(em.size());
      ++nr[i];
      for (int32_t t : em)
        if (produced[i] < K) out[static_cast<size_t>(i) * K + produced[i]++] = t;  // truncate at K
    }
  }
  vc::check_cuda(cudaEventRecord(w1, en.stream()), "event");
  vc::check_cuda(cudaEventSynchronize(w1), "event");
  float dms = 0.f;
  vc::check_cuda(cudaEventElapsedTime(&dms, w0, w1), "event");
  cudaEventDestroy(w0);
  cudaEventDestroy(w1);
  if (ms) *ms = dms;
  for (int i = 0; i < n; ++i) {
    if (n_rounds) n_rounds[i] = nr[i];
    if (ngram_rounds) ngram_rounds[i] = ngr[i];
  }
}

// Two-level composition (composed_accept_length,
// /root/reference/proj/src/analytics.cpp:413-422): each round makes x OUTER
// draft passes of the target model over the compressed KV; at every outer
// position an auxiliary drafter (prompt lookup over the request's own
// context, `ngram`-token key) proposes up to depth-1 further tokens, which
// ride the same pass as extra rows (engine draft rows, causal in the tail).
// The compressed model keeps its own prediction p0 and each proposal e_j that
// its previous row confirmed (p_{j-1} == e_j), so an outer pass appends
// 1 + (confirmed proposals) tokens.  The full-KV verify then checks the whole
// window; losslessness still rests on the verifier alone.
void composed_loop(vc::Engine& en, const int* slots, int n, int K, int x, int ngram, int depth, int32_t* out,
                   vc_compose_stats* stats) {
  const auto& cfg = en.config();
  if (x < 1 || x > cfg.max_x) throw speckv::ConfigError("composed: x out of [1, max_x]");
  if (ngram < 1 || depth < 1) throw speckv::ConfigError("composed: ngram and depth must be >= 1");
  if (depth > std::max(1, cfg.draft_depth)) throw speckv::ConfigError("composed: depth exceeds the engine's draft_depth");
  if (cfg.full_tier != 0) throw vc::ContractViolation("composed loop needs the HBM full tier");
  vc_compose_stats st{};
  std::vector<int> produced(n, 0);
  std::vector<vc::StepItem> its;
  std::vector<int32_t> row;
  double accepted_sum = 0;
  cudaEvent_t w0, w1;
  vc::check_cuda(cudaEventCreate(&w0), "event");
  vc::check_cuda(cudaEventCreate(&w1), "event");
  vc::check_cuda(cudaEventRecord(w0, en.stream()), "event");
  for (;;) {
    std::vector<int> act;
    for (int i = 0; i < n; ++i)
      if (produced[i] < K) act.push_back(i);
    if (act.empty()) break;
    st.rounds += 1;
    for (int pass = 0; pass < x; ++pass) {  // x outer positions
      std::vector<int> who;
      std::vector<std::vector<int32_t>> props;
      its.clear();
      for (int i : act) {
        const vc::SeqState& s = en.seq(slots[i]);
        const int room = cfg.max_x - static_cast<int>(s.drafted.size());
        if (room < 1) continue;
        std::vector<int32_t> ctx = s.history.empty() ? std::vector<int32_t>{s.pending} : s.history;
        ctx.insert(ctx.end(), s.drafted.begin(), s.drafted.end());
        auto prop = vc::ngram_proposal(ctx, ngram, std::min(depth - 1, room - 1));
        vc::StepItem t;
        t.slot = slots[i];
        t.mode = vc::RowMode::Draft;
        t.tokens = {ctx.back()};
        t.tokens.insert(t.tokens.end(), prop.begin(), prop.end());
        its.push_back(std::move(t));
        who.push_back(i);
        props.push_back(std::move(prop));
      }
      if (its.empty()) break;
      en.run_step(its, row);
      st.draft_steps += 1;
      size_t off = 0;
      for (size_t a = 0; a < who.size(); ++a) {
        const int sl = slots[who[a]];
        const auto& pr = props[a];
        en.push_draft(sl, row[off]);
        int matched = 0;
        for (size_t j = 0; j < pr.size(); ++j) {
          if (row[off + j] != pr[j]) break;  // row j assumed e_{j+1}: valid only if p_j confirmed it
          en.push_draft(sl, row[off + j + 1]);
          ++matched;
        }
        st.aux_proposed += static_cast<int64_t>(pr.size());
        st.aux_accepted += matched;
        off += pr.size() + 1;
      }
    }
    its.assign(act.size(), vc::StepItem{});  // one verify pass over the full KV
    for (size_t a = 0; a < act.size(); ++a) {
      const vc::SeqState& s = en.seq(slots[act[a]]);
      its[a].slot = slots[act[a]];
      its[a].mode = vc::RowMode::Verify;
      its[a].tokens.push_back(s.pending);
      its[a].tokens.insert(its[a].tokens.end(), s.drafted.begin(), s.drafted.end());
    }
    en.run_step(its, row);
    size_t off = 0;
    for (size_t a = 0; a < act.size(); ++a) {
      const int i = act[a];
      const size_t xi = en.seq(slots[i]).drafted.size();
      std::vector<int32_t> p(row.begin() + off, row.begin() + off + xi + 1);
      off += xi + 1;
      st.drafted += static_cast<int64_t>(xi);
      const auto em = en.accept_commit(slots[i], p);
      st.verifies += 1;
      accepted_sum += static_cast<double>(em.size()) - 1;
      for (int32_t t : em)
        if (produced[i] < K) {
          out[static_cast<size_t>(i) * K + produced[i]++] = t;
          st.tokens += 1;
        }
    }
  }
  vc::check_cuda(cudaEventRecord(w1, en.stream()), "event");
  vc::check_cuda(cudaEventSynchronize(w1), "event");
  float dms = 0.f;
  vc::check_cuda(cudaEventElapsedTime(&dms, w0, w1), "event");
  cudaEventDestroy(w0);
  cudaEventDestroy(w1);
  st.ms = dms;
  st.mean_accept = st.verifies ? accepted_sum / static_cast<double>(st.verifies) : 0.0;
  if (stats) *stats = st;
}

}  // namespace

int vc_run_speculative_composed(vc_engine* e, const int* slots, int n, int K, int x, int ngram, int depth,
                                int32_t* out, vc_compose_stats* stats) {
  return guard([&] { composed_loop(E(e), slots, n, K, x, ngram, depth, out, stats); });
}

int vc_run_speculative(vc_engine* e, const int* slots, int n, int K, int x, int32_t* out,
                       int32_t* rounds, int max_rounds, int* n_rounds, double* ms) {
  return guard([&] { speculative_loop(E(e), slots, n, K, x, 0, out, rounds, max_rounds, n_rounds, nullptr, ms); });
}

int vc_run_speculative_ngram(vc_engine* e, const int* slots, int n, int K, int x, int ngram, int32_t* out,
                             int32_t* rounds, int max_rounds, int* n_rounds, int* ngram_rounds, double* ms) {
  return guard([&] {
    if (ngram < 1) throw speckv::ConfigError("run_speculative_ngram: ngram must be >= 1");
    speculative_loop(E(e), slots, n, K, x, ngram, out, rounds, max_rounds, n_rounds, ngram_rounds, ms);
  });
}

int vc_run_scheduled(vc_engine* e, const int* slots, int n, const vc_sched_desc* sd, int32_t* out,
                     vc_sched_stats* stats) {
  return guard([&] {
    if (!sd) throw vc::ContractViolation("vc_run_scheduled: null descriptor");
    vc_run_scheduled_impl(E(e), slots, n, *sd, out, stats);
  });
}

int vc_run_decode_fifo(vc_engine* e, const vc_request_desc* reqs, int n, int K, int32_t* out,
                       vc_loop_metrics* m) {
  return guard([&] { vc_run_decode_fifo_impl(E(e), reqs, n, K, out, m); });
}

int vc_reload_span(int64_t bytes, double bandwidth, double iteration_time, double* iterations,
                   int* windows) {
  return guard([&] {
    auto s = speckv::reload_span(bytes, bandwidth, iteration_time);
    *iterations = s.iterations;
    *windows = s.windows;
  });
}

// ------------------------------------------------------------ kernel level
int vc_quant_kivi_slice(const uint16_t* k, const uint16_t* v, int n_groups, int d, int bits,
                        uint32_t* kcodes, uint32_t* ksz, uint32_t* vcodes, uint32_t* vsz, void* stream) {
  return guard([&] {
    if (n_groups <= 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t rw = vc::quant_record_words(d, bits), uw = vc::quant_unit_words(d, bits);
    const size_t ucw = vc::quant_unit_code_words(d, bits), gw = vc::quant_group_words(d, bits);
    uint32_t* rec = nullptr;
    vc::QuantJob* dj = nullptr;
    vc::check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&rec), n_groups * rw * 4, st), "malloc");
    vc::QuantJob j{k, v, rec, 0, n_groups};
    vc::check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&dj), sizeof(j), st), "malloc");
    vc::check_cuda(cudaMemcpyAsync(dj, &j, sizeof(j), cudaMemcpyHostToDevice, st), "memcpy");
    vc::check_cuda(vc::quant_kivi(dj, 1, n_groups, d, bits, st), "quant_kivi");
    // group records -> the flat per-stream layout of this entry point
    auto cp2d = [&](uint32_t* dst, size_t dpitch, const uint32_t* src, size_t width) {
      if (dst)
        vc::check_cuda(cudaMemcpy2DAsync(dst, dpitch * 4, src, rw * 4, width * 4, n_groups,
                                         cudaMemcpyDeviceToDevice, st), "memcpy2d");
    };
    cp2d(ksz, d, rec, d);
    for (int u = 0; u < VC_QGROUP / VC_QUNIT; ++u) {
      const uint32_t* ur = rec + d + u * uw;
      cp2d(kcodes ? kcodes + u * ucw : nullptr, gw, ur, ucw);
      cp2d(vcodes ? vcodes + u * ucw : nullptr, gw, ur + ucw, ucw);
      cp2d(vsz ? vsz + u * VC_QUNIT : nullptr, VC_QGROUP, ur + 2 * ucw, VC_QUNIT);
    }
    vc::check_cuda(cudaFreeAsync(dj, st), "free");
    vc::check_cuda(cudaFreeAsync(rec, st), "free");
    vc::check_cuda(cudaStreamSynchronize(st), "sync");
  });
}

int vc_kv_read(vc_engine* e, int pool, int slot, int layer, int head, int pos, int n, uint16_t* k,
               uint16_t* v) {
  return guard([&] {
    vc::Engine& en = E(e);
    const auto& m = en.model();
    const vc::KvPool p = pool == 1 ? en.stage_pool() : (pool == 3 ? en.drop_pool() : en.full_pool());
    const size_t slice = (static_cast<size_t>(slot) * m.layers + layer) * m.n_kv + head;
    const size_t off = (slice * p.cap + pos) * m.d;
    const size_t bytes = static_cast<size_t>(n) * m.d * 2;
    if (pool == 2) {
      if (!en.host_pool_k(slot)) throw vc::ContractViolation("no host pool (or the slot is resident)");
      en.sync_host_pool();
      const size_t hoff = ((static_cast<size_t>(layer) * m.n_kv + head) * p.cap + pos) * m.d;
      std::memcpy(k, en.host_pool_k(slot) + hoff, bytes);
      std::memcpy(v, en.host_pool_v(slot) + hoff, bytes);
      return;
    }
    if (!p.k) throw vc::ContractViolation("pool not allocated");
    vc::check_cuda(cudaMemcpy(k, p.k + off, bytes, cudaMemcpyDeviceToHost), "kv_read");
    vc::check_cuda(cudaMemcpy(v, p.v + off, bytes, cudaMemcpyDeviceToHost), "kv_read");
  });
}

int vc_attention_probe(vc_engine* e, int slot, int layer, int mode, const uint16_t* q_dev, int n_rows,
                       int kv_len, uint16_t* out_host) {
  return guard([&] { E(e).attention_probe(slot, layer, mode, q_dev, n_rows, kv_len, out_host); });
}

int vc_gemm_probe(const uint16_t* X, int M, int K, const uint16_t* W, int N, float* Y, void* stream) {
  return vc_gemm_probe_epi(X, M, K, W, N, 0, Y, stream);
}

int vc_gemm_probe_epi(const uint16_t* X, int M, int K, const uint16_t* W, int N, int epi, void* Y,
                      void* stream) {
  return guard([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    vc::GemmWorkspace ws;
    ws.partial_floats = vc::gemm_partial_floats(M > 128 ? 128 : M, N, K);
    ws.n_counters = N / 128 + 1;
    vc::check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&ws.partial), sizeof(float) * ws.partial_floats, st), "malloc");
    vc::check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&ws.counters), sizeof(int) * ws.n_counters, st), "malloc");
    vc::check_cuda(cudaMemsetAsync(ws.counters, 0, sizeof(int) * ws.n_counters, st), "memset");
    vc::GemmEpilogue ep;
    if (epi == 3) {  // SiLU-gate: Y = bf16 act in the tiled layout (Mp = M)
      ep.kind = vc::Epi::Silu;
      ep.out_bf16 = static_cast<uint16_t*>(Y);
    } else {
      ep.kind = vc::Epi::StoreF32;
      ep.out_f32 = static_cast<float*>(Y);
    }
    // logical inputs -> the tiled HBM layouts the GEMM streams
    uint16_t *xt = nullptr, *wt = nullptr;
    const size_t xe = static_cast<size_t>(M + 128) * K, we = static_cast<size_t>(N) * K;
    vc::check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&xt), xe * 2, st), "malloc");
    vc::check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&wt), we * 2, st), "malloc");
    vc::check_cuda(cudaMemsetAsync(xt, 0, xe * 2, st), "memset");
    vc::check_cuda(vc::retile_act(X, M, K, M, xt, st), "retile_act");
    vc::check_cuda(vc::retile_weight(W, N, K, wt, st), "retile_weight");
    vc::check_cuda(vc::gemm(xt, M, M, K, wt, N, ep, ws, st), "gemm");
    vc::check_cuda(cudaFreeAsync(ws.partial, st), "free");
    vc::check_cuda(cudaFreeAsync(ws.counters, st), "free");
    vc::check_cuda(cudaFreeAsync(xt, st), "free");
    vc::check_cuda(cudaFreeAsync(wt, st), "free");
    vc::check_cuda(cudaStreamSynchronize(st), "sync");
  });
}

}  // extern "C"
