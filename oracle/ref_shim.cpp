// ref_shim.cpp -- TEST INFRASTRUCTURE.
//
// extern "C" entry points over the UNMODIFIED reference library compiled
// from /root/reference/proj/src (see oracle/Makefile `ref`).  Python tests
// load oracle/_ref/libspeckv_ref.so through ctypes to (1) pin the CPU
// restatement in vc_oracle.c, (2) produce golden vectors, and (3) let the
// reference's own run_speculative drive this repo's GPU engine through
// TokenOracle callbacks.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "soak_harness.hpp"
#include "speckv/compressor.hpp"
#include "speckv/config.hpp"
#include "speckv/scheduler.hpp"
#include "speckv/specloop.hpp"

namespace {

struct RefNS {
  using SystemConfig = speckv::SystemConfig;
  using GeometricRoundSampler = speckv::GeometricRoundSampler;
  using SpecScheduler = speckv::SpecScheduler;
  using StepEvents = speckv::StepEvents;
  using Request = speckv::Request;
  static speckv::Scenario long_context() { return speckv::Scenario::LongContext; }
  static speckv::AcceptanceModel::Kind per_token_iid() {
    return speckv::AcceptanceModel::Kind::PerTokenIid;
  }
  static speckv::IterationTimeMode fixed_time() { return speckv::IterationTimeMode::Fixed; }
};

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const speckv::ConfigError& e) {
    g_err = e.what();
    return -1;
  } catch (const speckv::ContractError& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -3;
  }
}

using OracleCb = int32_t (*)(void* ctx, const int32_t* prefix, int64_t n);

speckv::TokenOracle wrap(OracleCb cb, void* ctx) {
  speckv::TokenOracle o;
  o.next = [cb, ctx](std::span<const speckv::Token> p) { return cb(ctx, p.data(), (int64_t)p.size()); };
  return o;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_soak(uint64_t seed, int64_t iterations, uint64_t* digest, double* emitted,
             int64_t* completed) {
  return guarded([&] {
    soak::Outcome o = soak::run<RefNS>(seed, iterations);
    *digest = o.digest;
    *emitted = o.emitted;
    *completed = o.completed;
    return 0;
  });
}

// kind: 0 drop-uniform, 1 drop-window, 2 quant-uniform.  out receives
// [layers][heads][drop] when non-null.  Returns drop count (>=0) or <0.
int64_t ref_compress(int kind, int layers, int heads, int64_t tokens, int64_t bpt, double ratio,
                     int bits, uint64_t seed, int sink_tokens, int64_t* out,
                     int64_t* payload_bytes, int* bit_scheme) {
  int64_t result = 0;
  int rc = guarded([&] {
    speckv::CompressorSpec spec;
    spec.kind = kind == 0   ? speckv::CompressorKind::DropUniform
                : kind == 1 ? speckv::CompressorKind::DropWindow
                            : speckv::CompressorKind::QuantUniform;
    spec.ratio = ratio;
    spec.bits = bits;
    spec.sink_tokens = sink_tokens;
    speckv::KvShape shape{layers, heads, tokens, bpt};
    speckv::CompressedKVMeta meta = speckv::compress(spec, shape, ratio, seed);
    *payload_bytes = meta.payload_bytes;
    *bit_scheme = meta.bit_scheme;
    int64_t drop = meta.dropped_indices.empty() || meta.dropped_indices[0].empty()
                       ? 0
                       : (int64_t)meta.dropped_indices[0][0].size();
    if (out) {
      for (int l = 0; l < layers; ++l)
        for (int h = 0; h < heads; ++h)
          std::memcpy(out + ((size_t)l * heads + h) * drop, meta.dropped_indices[l][h].data(),
                      sizeof(int64_t) * drop);
    }
    result = drop;
    return 0;
  });
  return rc < 0 ? rc : result;
}

int ref_accept(const int32_t* drafted, const int32_t* preds, int x, int32_t* out, int* n_out,
               int* first_mismatch, int* bonus) {
  return guarded([&] {
    auto r = speckv::accept(std::span<const int32_t>(drafted, x),
                            std::span<const int32_t>(preds, x + 1));
    std::memcpy(out, r.accepted.data(), sizeof(int32_t) * r.accepted.size());
    *n_out = (int)r.accepted.size();
    *first_mismatch = r.first_mismatch.value_or(0);
    *bonus = r.bonus_used ? 1 : 0;
    return 0;
  });
}

// The reference's run_speculative over caller-supplied oracles.  rounds_out
// receives accepted-per-round (capacity max_rounds).  Returns #rounds or <0.
int ref_run_speculative(OracleCb drafter, void* dctx, OracleCb verifier, void* vctx,
                        const int32_t* prompt, int64_t n_prompt, int64_t K, int x, int32_t* out,
                        int32_t* rounds_out, int max_rounds) {
  int rounds = 0;
  int rc = guarded([&] {
    auto [seq, stats] = speckv::run_speculative(wrap(drafter, dctx), wrap(verifier, vctx),
                                                std::span<const int32_t>(prompt, n_prompt), K, x);
    std::memcpy(out, seq.data(), sizeof(int32_t) * seq.size());
    rounds = stats.rounds();
    for (int i = 0; i < rounds && i < max_rounds; ++i) rounds_out[i] = stats.accepted_per_round[i];
    return 0;
  });
  return rc < 0 ? rc : rounds;
}

int ref_autoregress(OracleCb oracle, void* ctx, const int32_t* prompt, int64_t n_prompt, int64_t K,
                    int32_t* out) {
  return guarded([&] {
    auto seq = speckv::autoregress(wrap(oracle, ctx), std::span<const int32_t>(prompt, n_prompt), K);
    std::memcpy(out, seq.data(), sizeof(int32_t) * seq.size());
    return 0;
  });
}

// random_table_oracle (specloop.cpp:265-273) evaluated on one prefix.
int32_t ref_random_table_next(int vocab, uint64_t seed, const int32_t* prefix, int64_t n) {
  auto o = speckv::random_table_oracle(vocab, seed);
  return o(std::span<const int32_t>(prefix, n));
}

int ref_reload_span(int64_t bytes, double bw, double t_iter, double* iters, int* windows) {
  return guarded([&] {
    auto s = speckv::reload_span(bytes, bw, t_iter);
    *iters = s.iterations;
    *windows = s.windows;
    return 0;
  });
}

// update() for a batch of requests that share one shape (drop-window online).
// already[i] = drops so far at `layer`; out[i][head][k] new drops (capacity
// per request cap).  n_new[i] receives the count.
int ref_update_window(int layers, int heads, int window, int sinks, int layer, int n_req,
                      const int64_t* tokens, const int64_t* already, int64_t* out, int64_t cap,
                      int64_t* n_new) {
  return guarded([&] {
    speckv::CompressorSpec spec;
    spec.kind = speckv::CompressorKind::DropWindow;
    spec.mode = speckv::CompressorMode::Online;
    spec.ratio = 0.5;
    spec.window = window;
    spec.sink_tokens = sinks;
    std::vector<speckv::OnlineRequestKv> batch(n_req);
    std::vector<std::pair<int64_t, int64_t>> offs;
    int64_t cur = 0;
    for (int i = 0; i < n_req; ++i) {
      batch[i].shape = speckv::KvShape{layers, heads, tokens[i], 2};
      batch[i].dropped_indices.assign(layers, std::vector<std::vector<int64_t>>(heads));
      for (int h = 0; h < heads; ++h)
        for (int64_t k = 0; k < already[i]; ++k)
          batch[i].dropped_indices[layer][h].push_back(sinks + k);
      offs.emplace_back(cur, cur + tokens[i]);
      cur += tokens[i];
    }
    auto res = speckv::update(spec, layer, batch, offs);
    for (int i = 0; i < n_req; ++i) {
      n_new[i] = (int64_t)res[i][0].size();
      for (int h = 0; h < heads; ++h)
        for (int64_t k = 0; k < n_new[i] && k < cap; ++k)
          out[((size_t)i * heads + h) * cap + k] = res[i][h][k];
    }
    return 0;
  });
}

}  // extern "C"

// intra_throughput / optimize_intra (analytics.cpp:45-82, :130-150) with a
// tabulated acceptance model {c -> {x_i -> gamma_i}}: pins the measured-
// constant knob selection (paper_2605_17613_b200/knobs.py).  Returns the
// throughput, -1 when infeasible (std::nullopt), or < -1 on error.
#include "speckv/analytics.hpp"
namespace {
speckv::AcceptanceModel tab_model(double c, int n_tab, const int* xs, const double* gs) {
  speckv::AcceptanceModel m;
  m.kind = speckv::AcceptanceModel::Kind::Tabulated;
  for (int i = 0; i < n_tab; ++i) m.table[c][xs[i]] = gs[i];
  return m;
}
speckv::HardwareProfile hw_of(double bw_hbm, double bw_inter, int64_t gpu_mem) {
  speckv::HardwareProfile hw;
  hw.hbm_bandwidth = bw_hbm;
  hw.interconnect_bandwidth = bw_inter;
  hw.gpu_mem = gpu_mem;
  hw.local_gpus = 1;
  return hw;
}
}  // namespace
extern "C" {
double ref_intra_throughput(int b_c, int x, double c, int l, double bw_hbm, double bw_inter, int64_t gpu_mem,
                            int64_t weights, int64_t kv_full, int batch, int n_tab, const int* xs,
                            const double* gs) {
  double out = -1.0;
  int rc = guarded([&] {
    auto v = speckv::intra_throughput(speckv::IntraKnobs{b_c, x, c, l}, hw_of(bw_hbm, bw_inter, gpu_mem), weights,
                                      kv_full, batch, tab_model(c, n_tab, xs, gs));
    out = v ? *v : -1.0;
    return 0;
  });
  return rc < 0 ? -2.0 + rc : out;
}

// Grid: B_c in 0..batch, x in 1..x_max, the single c, l in 1..l_max.
double ref_optimize_intra(double c, int x_max, int l_max, double bw_hbm, double bw_inter, int64_t gpu_mem,
                          int64_t weights, int64_t kv_full, int batch, int n_tab, const int* xs, const double* gs,
                          int* b_c, int* x, int* l) {
  double out = -1.0;
  int rc = guarded([&] {
    speckv::IntraGrids g;
    for (int i = 1; i <= x_max; ++i) g.draft_length.push_back(i);
    g.compression.push_back(c);
    for (int i = 1; i <= l_max; ++i) g.cycles_per_load.push_back(i);
    for (int i = 0; i <= batch; ++i) g.offloaded_count.push_back(i);
    auto best = speckv::optimize_intra(hw_of(bw_hbm, bw_inter, gpu_mem), weights, kv_full, batch,
                                       tab_model(c, n_tab, xs, gs), g);
    if (best) {
      *b_c = best->knobs.offloaded_count;
      *x = best->knobs.draft_length;
      *l = best->knobs.cycles_per_load;
      out = best->throughput;
    }
    return 0;
  });
  return rc < 0 ? -2.0 + rc : out;
}

// composed_accept_length (analytics.cpp:413-422) with gamma(x) tabulated at
// one point and a constant gamma_e: pins knobs.composed_accept_length.
double ref_composed_accept_length(int x, double c, int d_e, double gamma_x, double gamma_e) {
  double out = -1.0;
  int rc = guarded([&] {
    const int xs[1] = {x};
    const double gs[1] = {gamma_x};
    out = speckv::composed_accept_length(x, c, d_e, tab_model(c, 1, xs, gs), [&](int) { return gamma_e; });
    return 0;
  });
  return rc < 0 ? -2.0 + rc : out;
}

}  // extern "C"
