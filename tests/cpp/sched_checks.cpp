// sched_checks.cpp -- TEST INFRASTRUCTURE: drives this repo's swap scheduler
// (paper_2605_17613_b200/csrc/speckv_host.cpp, the code libvericache.so
// ships) through the reference's soak harness and unit scenarios.  Built by
// tests/test_scheduler_parity.py with g++ (CPU only).
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../oracle/soak_harness.hpp"
#include "speckv_b200.hpp"

namespace {
struct NS {
  using SystemConfig = speckv::SystemConfig;
  using GeometricRoundSampler = speckv::GeometricRoundSampler;
  using SpecScheduler = speckv::SpecScheduler;
  using StepEvents = speckv::StepEvents;
  using Request = speckv::Request;
  static speckv::Scenario long_context() { return speckv::Scenario::LongContext; }
  static speckv::AcceptanceModel::Kind per_token_iid() { return speckv::AcceptanceModel::Kind::PerTokenIid; }
  static speckv::IterationTimeMode fixed_time() { return speckv::IterationTimeMode::Fixed; }
};

speckv::SystemConfig sched_cfg(int x, int window) {  // test_scheduler.cpp:14-39 shape
  speckv::SystemConfig c;
  c.scenario = speckv::Scenario::LongContext;
  c.hardware.hbm_bandwidth = 1.6e12;
  c.hardware.interconnect_bandwidth = 5e10;
  c.hardware.gpu_mem = 96000000000;
  c.hardware.local_gpus = 1;
  c.model.weights_bytes = 50000000000;
  c.model.kv_bytes_per_token = 40960;
  c.acceptance.kind = speckv::AcceptanceModel::Kind::PerTokenIid;
  c.acceptance.per_token_prob[0.25] = 0.97;
  c.acceptance.per_token_prob[1.0] = 1.0;
  c.draft_length = x;
  c.lookahead_window = window;
  c.iteration_time_mode = speckv::IterationTimeMode::Fixed;
  c.iteration_time = 0.037;
  c.batch_size = 1;
  c.kv_full_bytes = 1850000000;
  c.compression_ratio = 0.25;
  c.output_tokens = 1000;
  return c;
}
}  // namespace

extern "C" {

int sc_soak(uint64_t seed, int64_t iters, uint64_t* digest, double* emitted, int64_t* completed) {
  try {
    soak::Outcome o = soak::run<NS>(seed, iters);
    *digest = o.digest;
    *emitted = o.emitted;
    *completed = o.completed;
    return 0;
  } catch (...) {
    return 1;
  }
}

// admit() probe order with windows 23..27 saturated (test_scheduler.cpp:77-95)
int sc_admit_probe(int* examined, int cap, int* verify_window) {
  speckv::ReserveRings rings(64, 0.037, 5e10, 96000000000, 50000000000);
  for (int w = 23; w <= 27; ++w)
    if (!rings.admit(100 + w, 1850000000, w)) return -1;
  speckv::AdmitProbe p;
  auto r = rings.admit(1, 1850000000, 25, &p);
  rings.check_invariants();
  *verify_window = r ? r->verify_window : -1;
  for (size_t i = 0; i < p.examined.size() && static_cast<int>(i) < cap; ++i) examined[i] = p.examined[i];
  return static_cast<int>(p.examined.size());
}

// waiting outcome leaves rings unchanged (test_scheduler.cpp:97-110)
int sc_admit_waiting(void) {
  speckv::ReserveRings rings(16, 0.037, 5e10, 50000000000, 50000000000);
  speckv::AdmitProbe p;
  auto r = rings.admit(1, 1850000000, 4, &p);
  if (r) return -1;
  for (int i = 0; i < rings.window(); ++i)
    if (rings.bw_reserved(i) != 0.0 || rings.hbm_inflight(i) != 0) return -2;
  return static_cast<int>(p.examined.size());  // 15
}

// release restores rings bit-exactly (test_scheduler.cpp:127-166)
int sc_release_exact(void) {
  speckv::ReserveRings rings(32, 0.037, 5e10, 96000000000, 50000000000);
  auto a = rings.admit(1, 3000000000, 10);
  auto b = rings.admit(2, 700000000, 10);
  std::vector<double> before;
  for (int i = 0; i < 32; ++i) before.push_back(rings.bw_reserved(i));
  auto c = rings.admit(3, 1234567890, 10);
  rings.release(*c);
  for (int i = 0; i < 32; ++i)
    if (std::memcmp(&before[i], &(const double&)rings.bw_reserved(i), 8) != 0) return -1;
  rings.check_invariants();
  return a && b ? 0 : -2;
}

// single-request cadence: x drafts then a verify every x+1 iterations
// (test_scheduler.cpp:206-232).  Writes per-iteration verify counts.
int sc_cadence(int x, int iters, int* verifies, int* drafts) {
  auto cfg = sched_cfg(x, 16);
  speckv::MeanRoundSampler sampler(cfg.acceptance);
  speckv::SpecScheduler s(cfg, sampler);
  speckv::StepEvents ev;
  speckv::Request r;
  r.id = 0;
  r.kv_full_bytes = 1850000000;
  r.compression_ratio = 0.25;
  r.output_tokens = 1000;
  ev.arrivals.push_back(r);
  for (int i = 0; i < iters; ++i) {
    for (const auto& k : s.pending_kickoffs()) ev.completed_transfers.push_back(k.id);
    auto res = s.execution_step(ev);
    ev = speckv::StepEvents{};
    verifies[i] = res.verify_count;
    drafts[i] = res.drafting_count;
  }
  return 0;
}

}  // extern "C"
