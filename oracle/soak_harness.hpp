// soak_harness.hpp -- TEST INFRASTRUCTURE.
//
// The scheduler safety soak whose digest pins the swap scheduler: a seeded
// arrival stream, transfers delivered on time or 1-4 iterations late, and an
// FNV-1a fold of every step's counters and ring state.  It follows the
// procedure of /root/reference/proj/tests/acceptance_test.cpp:412-517
// (criterion 8) call for call, so the same seed produces the same digest on
// the reference library (oracle/_ref) and on this repo's scheduler.
//
// Written against the speckv:: API names, which both libraries expose; the
// including translation unit picks the implementation.
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <random>

namespace soak {

struct Outcome {
  std::uint64_t digest = 0xcbf29ce484222325ull;
  std::int64_t iterations = 0;
  double emitted = 0.0;
  std::int64_t completed = 0;
};

inline std::uint64_t fold_u64(std::uint64_t h, std::uint64_t v) {
  unsigned char b[8];
  std::memcpy(b, &v, 8);
  for (unsigned char c : b) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

inline std::uint64_t fold_f64(std::uint64_t h, double v) {
  std::uint64_t bits;
  std::memcpy(&bits, &v, 8);
  return fold_u64(h, bits);
}

template <class NS>
Outcome run(std::uint64_t seed, std::int64_t iterations) {
  using Cfg = typename NS::SystemConfig;
  Cfg cfg;
  cfg.scenario = NS::long_context();
  cfg.hardware.hbm_bandwidth = 1.6e12;
  cfg.hardware.interconnect_bandwidth = 5e10;
  cfg.hardware.gpu_mem = 96000000000;
  cfg.hardware.local_gpus = 1;
  cfg.model.weights_bytes = 50000000000;
  cfg.model.kv_bytes_per_token = 40960;
  cfg.acceptance.kind = NS::per_token_iid();
  cfg.acceptance.per_token_prob[0.2] = 0.95;
  cfg.acceptance.per_token_prob[0.25] = 0.97;
  cfg.acceptance.per_token_prob[0.5] = 0.99;
  cfg.acceptance.per_token_prob[1.0] = 1.0;
  cfg.draft_length = 12;
  cfg.lookahead_window = 16;
  cfg.iteration_time_mode = NS::fixed_time();
  cfg.iteration_time = 0.03;
  cfg.batch_size = 16;
  cfg.kv_full_bytes = 2000000000;
  cfg.compression_ratio = 0.25;
  cfg.output_tokens = 60;
  cfg.validate();

  typename NS::GeometricRoundSampler sampler(cfg.acceptance, seed);
  typename NS::SpecScheduler sched(cfg, sampler);
  std::mt19937_64 rng(seed);
  const double ratios[3] = {0.2, 0.25, 0.5};

  Outcome out;
  typename NS::StepEvents ev;
  std::int64_t next_id = 0;
  std::multimap<std::int64_t, std::uint64_t> deliveries;
  for (std::int64_t iter = 0; iter < iterations; ++iter) {
    if (rng() % 8 == 0) {
      typename NS::Request r;
      r.id = next_id++;
      r.arrival = 0.0;
      r.kv_full_bytes = 500000000 + static_cast<std::int64_t>(rng() % 3) * 500000000;
      r.compression_ratio = ratios[rng() % 3];
      r.output_tokens = 20 + static_cast<std::int64_t>(rng() % 40);
      ev.arrivals.push_back(r);
    }
    for (const auto& r : sched.pending_kickoffs()) {
      std::int64_t span = r.verify_iteration - r.span_begin;
      std::int64_t delay = rng() % 6 == 0 ? 1 + static_cast<std::int64_t>(rng() % 4) : 0;
      deliveries.emplace(iter + span + delay, r.id);
    }
    auto range = deliveries.equal_range(iter);
    for (auto it = range.first; it != range.second; ++it) ev.completed_transfers.push_back(it->second);
    deliveries.erase(range.first, range.second);

    auto step = sched.execution_step(ev);
    ev = typename NS::StepEvents{};

    out.emitted += step.tokens_emitted;
    out.completed += static_cast<std::int64_t>(step.completed.size());
    out.digest = fold_u64(out.digest, static_cast<std::uint64_t>(step.verify_count));
    out.digest = fold_u64(out.digest, static_cast<std::uint64_t>(step.drafting_count));
    out.digest = fold_u64(out.digest, static_cast<std::uint64_t>(step.hbm_read_bytes));
    out.digest = fold_f64(out.digest, step.tokens_emitted);
    const auto& rings = sched.rings();
    for (int w = 0; w < rings.window(); ++w) {
      out.digest = fold_f64(out.digest, rings.bw_reserved(w));
      out.digest = fold_u64(out.digest, static_cast<std::uint64_t>(rings.hbm_inflight(w)));
    }
    out.digest = fold_u64(out.digest, static_cast<std::uint64_t>(rings.kv_resident()));
    ++out.iterations;
  }
  return out;
}

}  // namespace soak
