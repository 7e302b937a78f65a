// vc_loops.cu -- the swap-scheduled decode loop (vc_run_scheduled).
//
// simulate_staggered (/root/reference/proj/src/sim.cpp:182-307) with the
// simulated link and HBM replaced by real copies and kernels:
//   1. pending_kickoffs() -> cudaMemcpy2DAsync of the request's committed
//      full KV from the pinned host pool into a free HBM staging slot on the
//      copy stream (tier 1), or nothing (tier 0: full KV already resident);
//   2. completed_transfers <- cudaEventQuery of those copies;
//   3. the iteration is planned on a copy of the scheduler (same state, a
//      recording sampler) to learn which sessions draft and which verify;
//   4. ONE forward pass runs every drafting row and every verify window;
//   5. execution_step() is replayed on the real scheduler with a sampler
//      that returns the measured accept counts in fire_verify order, so the
//      rings, cadence and stalls evolve exactly as Algorithm 1 prescribes.
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <algorithm>
#include <cstdlib>
#include <deque>
#include <map>
#include <set>
#include <thread>

#include "speckv_b200.hpp"
#include "vc_api.h"
#include "vc_engine.hpp"

namespace {

struct RecordingSampler : speckv::RoundSampler {
  std::vector<std::pair<int, double>> calls;
  double accepted_drafted(int drafted, double c) override {
    calls.emplace_back(drafted, c);
    return static_cast<double>(drafted);
  }
};

struct MeasuredSampler : speckv::RoundSampler {
  std::deque<int> accepted;  // accepted drafted tokens, fire_verify order
  double accepted_drafted(int, double) override {
    if (accepted.empty()) throw speckv::ContractError("scheduled loop: verify without a measured result");
    const int a = accepted.front();
    accepted.pop_front();
    return static_cast<double>(a);
  }
};

}  // namespace

int vc_run_scheduled_impl(vc::Engine& en, const int* slots, int n, const vc_sched_desc& sd,
                          int32_t* out, vc_sched_stats* stats) {
  const auto& cfgE = en.config();
  const bool staged = cfgE.full_tier == 1;
  if (sd.x < 1 || sd.x > cfgE.max_x) throw speckv::ConfigError("scheduled: x out of [1, max_x]");
  if (cfgE.quant_bits == 0 && cfgE.drop_ratio <= 0.0) throw vc::ContractViolation("scheduled: needs a compressed tier");
  // per-request tier placement: requests in the engine's resident slots keep
  // their full KV in HBM (B_g), the rest are offloaded (B_c)
  // requests: [0, n) present at the start in `slots`; [n, n + n_arrivals)
  // arrive later (sd.arrivals, host clock) and are admitted FIFO into the
  // slots finished requests free (simulate_staggered's arrivals, sim.cpp:227-302)
  const int n_arr = sd.n_arrivals > 0 ? sd.n_arrivals : 0;
  if (n_arr > 0 && !sd.arrivals) throw vc::ContractViolation("scheduled: null arrivals");
  const int n_total = n + n_arr;
  std::vector<int> slot_of(n_total, -1);
  for (int i = 0; i < n; ++i) slot_of[i] = slots[i];
  std::vector<int> res_idx;
  std::vector<char> is_res(n_total, 0);
  for (int i = 0; i < n; ++i)
    if (en.resident(slots[i])) {
      is_res[i] = 1;
      res_idx.push_back(i);
    }
  const int n_res = static_cast<int>(res_idx.size());
  const int n_off = n - n_res;
  const int x_res = sd.x_resident > 0 ? sd.x_resident : sd.x;
  // two-level composition: prompt-lookup proposals ride each drafting row
  const bool composed = sd.ngram >= 1 && sd.depth >= 2;
  if (composed && sd.depth > std::max(1, cfgE.draft_depth))
    throw speckv::ConfigError("scheduled: depth exceeds the engine's draft_depth");
  if (x_res > cfgE.max_x) throw speckv::ConfigError("scheduled: x_resident out of [1, max_x]");
  const size_t bpt = en.full_kv_bytes_per_token();

  // ---- measure T_iter if not given: one draft step over every request ----
  double t_iter = sd.iteration_time;
  if (t_iter <= 0) {
    std::vector<vc::StepItem> probe(n);
    for (int i = 0; i < n; ++i) {
      probe[i].slot = slots[i];
      probe[i].mode = vc::RowMode::Draft;
      probe[i].tokens = {en.seq(slots[i]).pending};
    }
    std::vector<int32_t> o;
    en.run_step(probe, o);  // warm (graph capture)
    const auto a = std::chrono::steady_clock::now();
    for (int r = 0; r < 3; ++r) en.run_step(probe, o);
    t_iter = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count() / 3;
  }
  double bw = sd.link_bandwidth > 0 ? sd.link_bandwidth : (staged ? 55e9 : 1e15);
  double reload_over_full = 1.0;
  if (staged && en.ring_mode()) {
    // the scheduler books reloads in full-KV bytes (scheduler.cpp:96-163);
    // a packed or drop-tier reload moves fewer: plan with the effective rate
    double raw = 0.0, moved = 0.0;
    for (int i = 0; i < n; ++i)
      if (!en.resident(slots[i])) {
        raw += static_cast<double>(en.seq(slots[i]).committed) * bpt;
        moved += en.reload_bytes(slots[i]);
      }
    if (moved > 0.0 && raw > moved) bw *= raw / moved;
    if (raw > 0.0) reload_over_full = moved / raw;
  }

  // ---- SystemConfig of this serving instance ------------------------------
  speckv::SystemConfig cfg;
  cfg.scenario = speckv::Scenario::LongContext;
  cfg.hardware.hbm_bandwidth = 6.5e12;
  cfg.hardware.interconnect_bandwidth = bw;
  cfg.hardware.local_gpus = 1;
  cfg.model.weights_bytes = static_cast<speckv::Bytes>(en.weight_bytes());
  cfg.model.kv_bytes_per_token = static_cast<speckv::Bytes>(bpt);
  speckv::Bytes kv_max = 0, resident_total = 0, compressed_all = 0;
  std::vector<double> ratio(n_total, 0.0);
  for (int i = 0; i < n; ++i) {
    const auto& s = en.seq(slots[i]);
    const speckv::Bytes kv = static_cast<speckv::Bytes>(s.committed) * bpt;
    kv_max = std::max(kv_max, kv);
    ratio[i] = std::min(1.0, static_cast<double>(en.compressed_bytes(slots[i])) / static_cast<double>(kv));
    compressed_all += static_cast<speckv::Bytes>(en.compressed_bytes(slots[i]));
    if (!is_res[i]) resident_total += static_cast<speckv::Bytes>(std::ceil(ratio[i] * kv));
  }
  // HBM ring capacity: weights + resident compressed caches + one full KV per
  // rotating staging slot, so the ring never books more reloads than we can
  // stage.  Resident requests' full KV is a fixed carve-out outside the ring.
  // chunk ring (ring_chunks > 0): reloads stream layer by layer and each
  // verify runs range by range as its layers land; at most max_streams such
  // verifies are in flight, so the scheduler books that many reloads
  const bool ring = en.ring_mode();
  const int n_stage = staged ? (ring ? cfgE.max_streams : cfgE.n_stage - cfgE.resident_slots)
                             : std::max(1, cfgE.max_verify);
  cfg.hardware.gpu_mem = sd.hbm_capacity > 0
                             ? sd.hbm_capacity
                             : cfg.model.weights_bytes + resident_total + std::max(1, n_stage) * (kv_max + kv_max / 64);
  cfg.acceptance.kind = speckv::AcceptanceModel::Kind::PerTokenIid;
  for (int i = 0; i < n; ++i) cfg.acceptance.per_token_prob[ratio[i]] = 0.99;
  cfg.draft_length = sd.x;
  cfg.lookahead_window = sd.window;
  cfg.iteration_time_mode = speckv::IterationTimeMode::Fixed;
  cfg.iteration_time = t_iter;
  cfg.batch_size = std::max(1, n_off);
  cfg.kv_full_bytes = kv_max;
  int first_off = 0;
  while (first_off < n - 1 && is_res[first_off]) ++first_off;
  cfg.compression_ratio = ratio[first_off];
  cfg.output_tokens = sd.K;
  cfg.validate();

  RecordingSampler rec;
  MeasuredSampler meas;
  speckv::SpecScheduler sched(cfg, meas);
  // VC_EXPEDITE=1 (host tier): verify a drafted round as soon as its reload
  // landed instead of at the booked verify iteration.  Off by default: with
  // x=47 the booked schedule already saturates PCIe (link busy 0.99), and at
  // large x the extra verify steps cost more GPU time than they save.
  static const bool expedite = [] {
    const char* v = std::getenv("VC_EXPEDITE");
    return v && v[0] == '1';
  }();
  // the chunk ring always expedites: a finished streamed verify holds one of
  // the max_streams stream slots, and the next reload cannot start behind it
  sched.set_expedite((expedite || ring) && staged);
  speckv::StepEvents ev;
  for (int i = 0; i < n; ++i) {
    if (is_res[i]) continue;
    speckv::Request r;
    r.id = i;
    r.kv_full_bytes = static_cast<speckv::Bytes>(en.seq(slots[i]).committed) * bpt;
    r.compression_ratio = ratio[i];
    r.output_tokens = sd.K;
    ev.arrivals.push_back(r);
  }

  std::vector<int> produced(n_total, 0);
  std::vector<int> stage_of(n_total, -1);
  std::vector<int> free_stages;
  const int stage_lo = staged ? cfgE.resident_slots : 0;
  for (int s = (staged ? cfgE.n_stage : n_stage) - 1; s >= stage_lo; --s) free_stages.push_back(s);
  // residents verify in their own staging slot (= their slot); first rounds
  // of x_res - (j mod (x_res+1)) drafts stagger their verifies over the
  // x_res + 1 iterations of a round
  std::vector<int> round_x(n_total, 0);
  for (int j = 0; j < n_res; ++j) {
    const int i = res_idx[j];
    stage_of[i] = slots[i];
    round_x[i] = x_res - (j % (x_res + 1));
  }
  int64_t res_verifies = 0;
  double res_accepted = 0;
  int64_t res_tokens_at_window = 0;
  auto res_tokens = [&] {
    int64_t t = 0;
    for (int i : res_idx) t += produced[i];
    return t;
  };
  auto residents_active = [&] {
    for (int i : res_idx)
      if (produced[i] < sd.K) return true;
    return false;
  };
  // reference metrics on the loop's host clock (sim.cpp:80-109)
  std::vector<std::pair<double, double>> emission;  // (seconds, tokens)
  std::vector<double> done_at(n_total, -1.0), t_arr(n_total, 0.0);
  std::deque<int> queue;      // arrived, waiting for a slot
  std::vector<int> free_slots;
  int next_arr = 0;
  std::vector<char> freed(n_total, 0);  // request's slot returned to free_slots
  const double h2d_ms_start = en.h2d_ms();
  struct Xfer {
    uint64_t id;
    speckv::ReservationId res;
    int req;
  };
  std::vector<Xfer> inflight;
  struct VStreamRef {
    int id;
    speckv::ReservationId res;
    int req;
    int64_t verify_iteration;  // the booked verify (the round may end short of x there)
    bool ready;  // predictions in; the scheduler has been told the reload landed
  };
  std::vector<VStreamRef> vstreams;
  // a streamed reload starts once its round has at most `lead` drafts to go
  // (the verify can only run its first layers on a complete window)
  static const int stream_lead = [] {
    const char* v = std::getenv("VC_STREAM_LEAD");
    return v ? std::atoi(v) : 2;
  }();
  std::set<speckv::ReservationId> kicked;  // reloads already started
  constexpr int kLinkQueue = 2;            // copies kept queued on the link ahead of schedule
  static const bool early_kick = [] {
    const char* v = std::getenv("VC_EARLY_KICK");
    return !(v && v[0] == '0');
  }();
  vc_sched_stats st{};
  st.reload_over_full = reload_over_full;
  double accepted_sum = 0;
  const auto t0 = std::chrono::steady_clock::now();
  const std::int64_t guard_iters = 10000 + 20LL * (sd.window + sd.x) + 64LL * sd.K * n_total;
  std::int64_t idle_iters = 0;
  auto last_progress = std::chrono::steady_clock::now();

  int64_t tokens_at_window = 0;
  double rows_in_window = 0;
  auto window_start = t0;
  // the timed window on the device: one event pair on the compute stream around
  // all K steps (host planning gaps included), as bench.py's contract asks
  cudaEvent_t win0 = nullptr, win1 = nullptr;
  vc::check_cuda(cudaEventCreate(&win0), "window event");
  vc::check_cuda(cudaEventCreate(&win1), "window event");
  const bool bounded = sd.timed_iterations > 0;
  // planning iteration time: the reference re-plans every iteration
  // (sim.cpp:238-239); here it tracks the measured wall time of the loop's
  // iterations (EMA), so reload spans are booked in real link seconds
  double t_plan = t_iter;
  const bool adapt = sd.iteration_time <= 0;
  double stall_ms = 0.0, h2d_ms_at_window = 0.0, h2d_bytes_at_window = 0.0;
  auto t_prev = std::chrono::steady_clock::now();
  for (std::int64_t it = 0;
       !sched.idle() || !ev.arrivals.empty() || residents_active() || next_arr < n_arr || !queue.empty(); ++it) {
    // iterations that ran no step (every session waiting on the link) do not
    // count toward the stall guard: a slow device (e.g. under a sanitizer)
    // legitimately spins through many of them
    if (it - idle_iters > guard_iters) throw speckv::ConfigError("scheduled loop stalled");
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - last_progress).count() > 120.0)
      throw speckv::ConfigError("scheduled loop stalled (no step, verify or transfer for 120 s)");
    if (n_arr > 0) {  // arrivals and admissions
      const double now_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      while (next_arr < n_arr && sd.arrivals[next_arr].arrival_ms <= now_ms) {
        t_arr[n + next_arr] = sd.arrivals[next_arr].arrival_ms / 1e3;
        queue.push_back(n + next_arr++);
      }
      for (int r = 0; r < n_total; ++r)  // finished requests give their slot back
        if (slot_of[r] >= 0 && !freed[r] && produced[r] >= sd.K &&
            (is_res[r] || !sched.sessions().count(static_cast<speckv::RequestId>(r)))) {
          freed[r] = 1;
          free_slots.push_back(slot_of[r]);
        }
      while (!queue.empty() && !free_slots.empty()) {
        const int r = queue.front();
        const int slot = free_slots.front();
        const bool res = en.resident(slot);
        int scratch = -1;
        if (staged && !res && !ring) {  // an offloaded admission borrows a free rotating stage
          // (the chunk ring admits through its own two admission chunks)
          if (free_stages.empty()) break;
          scratch = free_stages.back();
          free_stages.pop_back();
          en.set_scratch_stage(scratch);
        }
        queue.pop_front();
        free_slots.erase(free_slots.begin());
        const vc_request_desc& q = sd.arrivals[r - n];
        en.add_request_synthetic(slot, q.n_ctx, q.first_token, q.seed, 4, 10.f);
        en.compress(slot);
        if (scratch >= 0) {
          en.set_scratch_stage(-1);
          free_stages.push_back(scratch);
        }
        slot_of[r] = slot;
        const speckv::Bytes kv = static_cast<speckv::Bytes>(q.n_ctx) * bpt;
        ratio[r] = std::min(1.0, static_cast<double>(en.compressed_bytes(slot)) / static_cast<double>(kv));
        if (res) {
          is_res[r] = 1;
          res_idx.push_back(r);
          stage_of[r] = slot;
          round_x[r] = x_res;
        } else {
          speckv::Request a;
          a.id = r;
          a.kv_full_bytes = kv;
          a.compression_ratio = ratio[r];
          a.output_tokens = sd.K;
          ev.arrivals.push_back(a);
          cfg.acceptance.per_token_prob[ratio[r]] = 0.99;
        }
      }
    }
    if (adapt) sched.set_planning_iteration_time(t_plan);
    if (it == sd.warmup_iterations) {  // open the timed window
      int64_t tk = 0;
      for (int i = 0; i < n_total; ++i) tk += produced[i];
      tokens_at_window = tk;
      res_tokens_at_window = res_tokens();
      en.reset_timing();
      window_start = std::chrono::steady_clock::now();
      vc::check_cuda(cudaEventRecord(win0, en.stream()), "window event");
      stall_ms = 0.0;
      h2d_ms_at_window = en.h2d_ms();
      h2d_bytes_at_window = en.h2d_bytes();
    }
    if (bounded && it == sd.warmup_iterations + sd.timed_iterations) break;
    // 1. kick off transfers.  The reference starts a reload at its span_begin
    // (pending_kickoffs, sim.cpp:243-249).  The copy stream is a FIFO link:
    // here a booked reload (earliest verify first) starts as soon as a staging
    // slot is free and fewer than kLinkQueue copies are queued on the link --
    // the link never idles while a booked reload waits, and a staging slot is
    // taken only about one copy-time before its reload can start, not at
    // booking (which would pin slots for a whole round).  Landing earlier than
    // the reference's schedule is always safe (done_ is checked at verify).
    // VC_EARLY_KICK=0 restores span_begin kickoffs.
    for (const auto& r : sched.pending_kickoffs()) {
      if (r.bytes == 0 || !staged) {  // arrival load (compressed tier resident) / tier 0
        ev.completed_transfers.push_back(r.id);
        continue;
      }
    }
    if (staged) {
      std::vector<speckv::Reservation> want;
      for (const auto& [id, ss] : sched.sessions())
        if (ss.pending && ss.pending->bytes > 0 && !kicked.count(ss.pending->id) &&
            (early_kick || ss.pending->span_begin <= sched.iteration()))
          want.push_back(*ss.pending);
      std::sort(want.begin(), want.end(), [](const speckv::Reservation& a, const speckv::Reservation& b) {
        return a.verify_iteration != b.verify_iteration ? a.verify_iteration < b.verify_iteration : a.id < b.id;
      });
      for (const auto& r : want) {
        if (ring) {
          if (en.streams_active() >= cfgE.max_streams) break;
          const int req = static_cast<int>(r.request_id);
          if (static_cast<int>(en.seq(slot_of[req]).drafted.size()) + stream_lead < sd.x &&
              sched.iteration() + stream_lead < r.verify_iteration)
            continue;
          vstreams.push_back({en.stream_begin(slot_of[req]), r.id, req, r.verify_iteration, false});
          kicked.insert(r.id);
          continue;
        }
        if (free_stages.empty()) break;
        if (early_kick && r.span_begin > sched.iteration() && static_cast<int>(inflight.size()) >= kLinkQueue) break;
        const int req = static_cast<int>(r.request_id);
        const int s = free_stages.back();
        free_stages.pop_back();
        stage_of[req] = s;
        inflight.push_back({en.swap_begin(slot_of[req], s), r.id, req});
        kicked.insert(r.id);
      }
    }
    // 2. completions
    if (ring) {
      en.stream_pump();
      for (auto& v : vstreams) {
        if (v.ready) continue;
        // the verify ranges run once the round's window is final: x drafts, or
        // the booked verify iteration reached (Algorithm 1 stops drafting there)
        if (static_cast<int>(en.seq(slot_of[v.req]).drafted.size()) < sd.x &&
            sched.iteration() < v.verify_iteration)
          continue;
        if (en.stream_advance(v.id) == 1) {
          v.ready = true;
          ev.completed_transfers.push_back(v.res);
        }
      }
    }
    for (size_t i = 0; i < inflight.size();) {
      if (en.swap_done(inflight[i].id)) {
        ev.completed_transfers.push_back(inflight[i].res);
        inflight.erase(inflight.begin() + i);
      } else {
        ++i;
      }
    }
    // 3. plan on a copy
    speckv::SpecScheduler plan = sched;
    rec.calls.clear();
    plan.set_sampler(rec);
    const speckv::StepResult pr = plan.execution_step(ev);
    // 4. one forward pass: drafting rows + verify windows
    std::vector<vc::StepItem> items;
    std::vector<std::vector<int32_t>> props;  // per drafting item: auxiliary proposals (composition)
    // a drafting row: the window's last token, plus (composition) the
    // prompt-lookup continuation of the request's context, bounded by `cap`
    // tokens of window
    // returns false (no row) once a composed window already holds `cap`
    // tokens: the scheduler may still count draft iterations for it
    std::vector<char> drew;  // per scheduler drafting session: a row was added
    auto draft_item = [&](int slot, int cap) {
      const auto& s = en.seq(slot);
      if (composed && static_cast<int>(s.drafted.size()) >= std::min(cap, cfgE.max_x)) {
        drew.push_back(0);
        return;
      }
      drew.push_back(1);
      vc::StepItem t;
      t.slot = slot;
      t.mode = vc::RowMode::Draft;
      t.tokens = {s.drafted.empty() ? s.pending : s.drafted.back()};
      std::vector<int32_t> prop;
      const int room = std::min(cap, cfgE.max_x) - static_cast<int>(s.drafted.size()) - 1;
      if (composed && room > 0) {
        std::vector<int32_t> ctx = s.history.empty() ? std::vector<int32_t>{s.pending} : s.history;
        ctx.insert(ctx.end(), s.drafted.begin(), s.drafted.end());
        prop = vc::ngram_proposal(ctx, sd.ngram, std::min(sd.depth - 1, room));
        t.tokens.insert(t.tokens.end(), prop.begin(), prop.end());
      }
      items.push_back(std::move(t));
      props.push_back(std::move(prop));
    };
    for (speckv::RequestId id : pr.drafted) draft_item(slot_of[id], composed ? sd.x : cfgE.max_x);
    // resident requests: draft their round, then verify against their own
    // HBM-resident full KV (no reload)
    std::vector<int> res_drafting, res_verifying;
    for (int i : res_idx) {
      if (produced[i] >= sd.K) continue;
      const auto& s = en.seq(slot_of[i]);
      if (static_cast<int>(s.drafted.size()) < round_x[i]) {
        draft_item(slot_of[i], round_x[i]);
        res_drafting.push_back(i);
      }
    }
    std::vector<int> verifying, ring_verifying;
    for (const auto& v : pr.verifies) {
      const int req = static_cast<int>(v.request);
      const auto& s = en.seq(slot_of[req]);
      // (composition: confirmed proposals make the window longer than the
      // scheduler's draft iterations)
      if (composed ? static_cast<int>(s.drafted.size()) < v.drafted : static_cast<int>(s.drafted.size()) != v.drafted)
        throw vc::ContractViolation("scheduled loop: draft count diverged from the scheduler");
      if (ring) {  // predictions came from the streamed verify's ranges
        ring_verifying.push_back(req);
        continue;
      }
      vc::StepItem t;
      t.slot = slot_of[req];
      t.mode = vc::RowMode::Verify;
      t.stage = staged ? stage_of[req] : -1;
      t.tokens.push_back(s.pending);
      t.tokens.insert(t.tokens.end(), s.drafted.begin(), s.drafted.end());
      items.push_back(std::move(t));
      verifying.push_back(req);
    }
    for (int i : res_idx) {
      if (produced[i] >= sd.K) continue;
      const auto& s = en.seq(slot_of[i]);
      if (static_cast<int>(s.drafted.size()) >= round_x[i]) {
        vc::StepItem t;
        t.slot = slot_of[i];
        t.mode = vc::RowMode::Verify;
        t.stage = slot_of[i];
        t.tokens.push_back(s.pending);
        t.tokens.insert(t.tokens.end(), s.drafted.begin(), s.drafted.end());
        items.push_back(std::move(t));
        res_verifying.push_back(i);
      }
    }
    std::vector<int32_t> row;
    if (!items.empty() || !pr.verifies.empty() || !ev.completed_transfers.empty())
      last_progress = std::chrono::steady_clock::now();
    if (!items.empty()) {
      en.run_step(items, row);
    } else if (pr.verifies.empty()) {
      ++idle_iters;
      std::this_thread::sleep_for(std::chrono::microseconds(20));  // nothing to run: let the link progress
    }
    if (it >= sd.warmup_iterations) {
      rows_in_window += static_cast<double>(row.size());
      for (const auto& t : items)
        if (t.mode == vc::RowMode::Verify) {
          st.timed_verifies += 1;
          st.timed_verify_rows += static_cast<double>(t.tokens.size());
        }
    }
    const double t_emit = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double emitted_now = 0;
    size_t off = 0;
    // the pass's own prediction, then (composition) each proposal its previous
    // row confirmed: row j assumed proposal j, valid only if p_j matched it
    size_t di = 0, dn = 0;
    auto take_draft = [&](int slot) {
      if (!drew[dn++]) return;
      const auto& pr_ = props[di++];
      en.push_draft(slot, row[off]);
      int matched = 0;
      for (size_t j = 0; j < pr_.size(); ++j) {
        if (row[off + j] != pr_[j]) break;
        en.push_draft(slot, row[off + j + 1]);
        ++matched;
      }
      st.aux_proposed += static_cast<int64_t>(pr_.size());
      st.aux_accepted += matched;
      off += pr_.size() + 1;
    };
    for (speckv::RequestId id : pr.drafted) take_draft(slot_of[id]);
    for (int i : res_drafting) take_draft(slot_of[i]);
    meas.accepted.clear();
    for (int req : verifying) {
      const int x_r = static_cast<int>(en.seq(slot_of[req]).drafted.size());
      std::vector<int32_t> p(row.begin() + off, row.begin() + off + x_r + 1);
      off += x_r + 1;
      st.drafted_tokens += x_r;
      const auto em = en.accept_commit(slot_of[req], p, staged ? stage_of[req] : -1);
      meas.accepted.push_back(static_cast<int>(em.size()) - 1);
      accepted_sum += static_cast<double>(em.size()) - 1;
      for (int32_t t : em)
        if (produced[req] < sd.K) {
          out[static_cast<size_t>(req) * sd.K + produced[req]++] = t;
          emitted_now += 1;
        }
      if (produced[req] >= sd.K && done_at[req] < 0) done_at[req] = t_emit;
      if (staged) {
        free_stages.push_back(stage_of[req]);
        stage_of[req] = -1;
      }
    }
    for (int req : ring_verifying) {
      auto vit = std::find_if(vstreams.begin(), vstreams.end(), [&](const VStreamRef& v) { return v.req == req; });
      if (vit == vstreams.end() || !vit->ready) throw vc::ContractViolation("scheduled loop: verify without a streamed result");
      st.drafted_tokens += static_cast<int64_t>(en.seq(slot_of[req]).drafted.size());
      const auto em = en.accept_commit_stream(slot_of[req], en.stream_preds(vit->id), vit->id);
      vstreams.erase(vit);
      meas.accepted.push_back(static_cast<int>(em.size()) - 1);
      accepted_sum += static_cast<double>(em.size()) - 1;
      for (int32_t t : em)
        if (produced[req] < sd.K) {
          out[static_cast<size_t>(req) * sd.K + produced[req]++] = t;
          emitted_now += 1;
        }
      if (produced[req] >= sd.K && done_at[req] < 0) done_at[req] = t_emit;
      if (it >= sd.warmup_iterations) {
        st.timed_verifies += 1;
        st.timed_verify_rows += static_cast<double>(em.size());  // streamed: rows ran in earlier ranges
      }
    }
    for (int i : res_verifying) {
      const int x_r = static_cast<int>(en.seq(slot_of[i]).drafted.size());
      std::vector<int32_t> p(row.begin() + off, row.begin() + off + x_r + 1);
      off += x_r + 1;
      st.drafted_tokens += x_r;
      const auto em = en.accept_commit(slot_of[i], p, slot_of[i]);
      res_verifies += 1;
      res_accepted += static_cast<double>(em.size()) - 1;
      for (int32_t t : em)
        if (produced[i] < sd.K) {
          out[static_cast<size_t>(i) * sd.K + produced[i]++] = t;
          emitted_now += 1;
        }
      if (produced[i] >= sd.K && done_at[i] < 0) done_at[i] = t_emit;
      round_x[i] = x_res;
    }
    if (emitted_now > 0) emission.emplace_back(t_emit, emitted_now);
    // 5. the real step with measured accept counts
    const speckv::StepResult rr = sched.execution_step(ev);
    if (rr.drafted != pr.drafted || rr.verify_count != pr.verify_count)
      throw vc::ContractViolation("scheduled loop: replay diverged from plan");
    st.verifies += rr.verify_count;
    st.late_transfers += static_cast<int64_t>(rr.late_transfers.size());
    st.iterations += 1;
    const auto t_now = std::chrono::steady_clock::now();
    const double dt = std::chrono::duration<double>(t_now - t_prev).count();
    t_prev = t_now;
    t_plan = 0.8 * t_plan + 0.2 * dt;
    // exposed swap time: a session whose reload is late stalls this iteration
    int stalled = 0, booked = 0, spec = 0;
    for (const auto& [id, ss] : sched.sessions()) {
      stalled += ss.stalled ? 1 : 0;
      spec += ss.mode == speckv::SessionMode::Speculative ? 1 : 0;
      booked += (ss.pending && !kicked.count(ss.pending->id)) ? 1 : 0;
    }
    stall_ms += 1e3 * dt * stalled;
    static const bool sched_log = std::getenv("VC_SCHED_LOG") != nullptr;
    if (sched_log)
      std::fprintf(stderr, "SCHED it=%lld dt=%.2f plan=%.2f spec=%d waiting=%zu stalled=%d booked=%d inflight=%zu free=%zu drafted=%zu verifies=%zu\n",
                   static_cast<long long>(it), dt * 1e3, t_plan * 1e3, spec, sched.waiting_size(), stalled, booked,
                   inflight.size(), free_stages.size(), rr.drafted.size(), rr.verifies.size());
    ev = speckv::StepEvents{};
  }
  const auto t1 = std::chrono::steady_clock::now();
  // a bounded window may end mid-round: land the in-flight reloads and roll
  // the open draft rounds back, so the slots can be scheduled again
  for (const Xfer& x : inflight) en.swap_wait(x.id);
  for (const auto& v : vstreams) en.stream_end(v.id);
  for (int i = 0; i < n_total; ++i)
    if (slot_of[i] >= 0 && !freed[i]) en.discard_drafts(slot_of[i]);
  st.wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  {  // SimMetrics on the host clock (finalize_metrics, sim.cpp:98-109)
    const double end = st.wall_ms / 1e3;
    double total = 0, warm = 0;
    for (const auto& [t, k] : emission) {
      total += k;
      if (t >= 0.1 * end && t <= 0.9 * end) warm += k;
    }
    st.throughput = end > 0 ? total / end : 0.0;
    st.warm_throughput = end > 0 ? warm / (0.8 * end) : 0.0;
    std::vector<double> lat;  // completion - arrival (host clock)
    for (int r = 0; r < n_total; ++r)
      if (done_at[r] >= 0) lat.push_back(done_at[r] - t_arr[r]);
    auto pct = [&](double q) {
      if (lat.empty()) return 0.0;
      std::sort(lat.begin(), lat.end());
      size_t r = static_cast<size_t>(std::ceil(q * static_cast<double>(lat.size())));
      r = std::min(std::max<size_t>(r, 1), lat.size());
      return lat[r - 1];
    };
    st.p50_latency_s = pct(0.5);
    st.p99_latency_s = pct(0.99);
    st.interconnect_busy = end > 0 ? (en.h2d_ms() - h2d_ms_start) / 1e3 / end : 0.0;
    const int64_t slot_bytes = static_cast<int64_t>(en.full_pool().cap) * static_cast<int64_t>(bpt);
    st.peak_hbm_bytes = static_cast<int64_t>(en.weight_bytes()) + compressed_all +
                        (staged ? static_cast<int64_t>(cfgE.resident_slots) * slot_bytes +
                                      static_cast<int64_t>(en.staging_bytes())
                                : static_cast<int64_t>(n) * slot_bytes);
    st.staging_bytes = static_cast<int64_t>(en.staging_bytes());
  }
  st.verifies += res_verifies;  // mean_accept below covers both tiers
  accepted_sum += res_accepted;
  st.resident_verifies = res_verifies;
  st.resident_accept = res_verifies ? res_accepted / static_cast<double>(res_verifies) : 0.0;
  for (int i = 0; i < n_total; ++i) st.tokens += produced[i];
  if (st.iterations > sd.warmup_iterations) {
    st.timed_iterations = st.iterations - sd.warmup_iterations;
    st.timed_tokens = st.tokens - tokens_at_window;
    st.timed_resident_tokens = res_tokens() - res_tokens_at_window;
    st.timed_wall_ms = std::chrono::duration<double, std::milli>(t1 - window_start).count();
    vc::check_cuda(cudaEventRecord(win1, en.stream()), "window event");
    vc::check_cuda(cudaEventSynchronize(win1), "window event");
    float wms = 0.f;
    vc::check_cuda(cudaEventElapsedTime(&wms, win0, win1), "window event");
    st.timed_device_ms = wms;
    st.timed_rows = rows_in_window;
    st.timed_step_device_ms = en.device_ms();  // reset when the window opened
  }
  st.h2d_ms = en.h2d_ms() - h2d_ms_at_window;
  st.h2d_bytes = en.h2d_bytes() - h2d_bytes_at_window;
  st.verify_wait_ms = stall_ms;
  cudaEventDestroy(win0);
  cudaEventDestroy(win1);
  st.mean_accept = st.verifies ? accepted_sum / static_cast<double>(st.verifies) : 0.0;
  if (stats) *stats = st;
  return VC_OK;
}

// ---------------------------------------------------------------------------
// vc_run_remote_prefix: the remote-prefix pipeline on real copies and kernels.
//
// The reference's remote_prefix (/root/reference/proj/src/sim.cpp:510-665)
// runs, per request: arrival -> compressed payload over the link
// (kCompressedLoaded, :588-610) -> a cycle of x drafts on the compressed KV
// while the full KV is prefetched (start_cycle, :562-575) -> verify when both
// are done (:611-619) -> accept (:622-636) -> next cycle; with verify_cached
// the full KV stays resident after its first load.  force_baseline (:605-608)
// loads the full KV and decodes.  Here both "links" are the GPU's copy engine
// (the storage node is pinned host memory on this box), so the two payloads
// share one FIFO, fed in arrival order with at most link_queue transfers
// queued: per request (compressed, then full) by default, so each request
// drafts while its own full KV streams and no later request's payload delays
// an earlier request's first verify; or every compressed payload first.
// One forward pass per iteration runs every drafting row, up to max_verify
// verify windows (oldest ready first) and, in the baseline, every decode row.
int vc_run_remote_prefix_impl(vc::Engine& en, const int* slots, int n, const vc_remote_desc& rd,
                              int32_t* out, vc_remote_stats* stats) {
  const auto& cfgE = en.config();
  const bool base = rd.baseline != 0;
  if (n < 1 || n > cfgE.max_slots) throw speckv::ConfigError("remote prefix: n out of [1, max_slots]");
  if (rd.K < 1) throw speckv::ConfigError("remote prefix: K must be >= 1");
  if (!base && (rd.x < 1 || rd.x > cfgE.max_x)) throw speckv::ConfigError("remote prefix: x out of [1, max_x]");
  if (rd.link_queue < 1) throw speckv::ConfigError("remote prefix: link_queue must be >= 1");
  if (rd.arrival_gap_ms < 0) throw speckv::ConfigError("remote prefix: arrival gap must be >= 0");
  if (rd.payload_order != 0 && rd.payload_order != 1) throw speckv::ConfigError("remote prefix: payload_order is 0 or 1");
  if (en.prefix_tokens() < 1) throw vc::ContractViolation("remote prefix: no prefix stored (vc_prefix_store)");
  if (!rd.first_tokens) throw vc::ContractViolation("remote prefix: null first_tokens");
  if (en.prefix_tokens() + rd.K + cfgE.max_x > cfgE.max_ctx)
    throw speckv::ConfigError("remote prefix: prefix + K + max_x exceeds max_ctx");

  struct Req {
    bool arrived = false, active = false, full = false, done = false;
    bool comp_issued = false, full_issued = false;
    uint64_t comp_id = 0, full_id = 0;
    double t_arr = 0, t_comp = -1, t_full = -1, t_first = -1;
    int produced = 0;
    int64_t ready_seq = -1;  // order in which the request became verifiable
  };
  std::vector<Req> rq(n);
  for (int i = 0; i < n; ++i) en.release(slots[i]);
  const double h2d_ms0 = en.h2d_ms(), h2d_b0 = en.h2d_bytes();
  cudaEvent_t win0 = nullptr, win1 = nullptr;
  vc::check_cuda(cudaEventCreate(&win0), "window event");
  vc::check_cuda(cudaEventCreate(&win1), "window event");
  vc::check_cuda(cudaEventRecord(win0, en.stream()), "window event");
  const auto t0 = std::chrono::steady_clock::now();
  auto now_ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };

  vc_remote_stats st{};
  double accepted_sum = 0;
  int64_t ready_counter = 0;
  std::vector<int32_t> row;
  const int64_t guard_iters = 100000 + 8LL * n * rd.K;
  for (int64_t it = 0;; ++it) {
    if (it > guard_iters) throw speckv::ConfigError("remote prefix loop stalled");
    const double t = now_ms();
    // arrivals (nominal times)
    for (int i = 0; i < n; ++i)
      if (!rq[i].arrived && t >= i * rd.arrival_gap_ms) {
        rq[i].arrived = true;
        rq[i].t_arr = i * rd.arrival_gap_ms;
      }
    // completions
    int inflight = 0;
    for (int i = 0; i < n; ++i) {
      Req& r = rq[i];
      if (r.comp_issued && !r.active) {
        if (en.swap_done(r.comp_id)) { r.active = true; r.t_comp = now_ms(); } else ++inflight;
      }
      if (r.full_issued && !r.full) {
        if (en.swap_done(r.full_id)) { r.full = true; r.t_full = now_ms(); } else ++inflight;
      }
    }
    // feed the link in arrival order: per request (its compressed payload, then
    // its full KV -- the request drafts while its own full KV streams), or
    // every compressed payload ahead of any full KV (payload_order 1)
    while (inflight < rd.link_queue) {
      int pick = -1, what = -1;
      for (int i = 0; i < n && pick < 0; ++i) {
        if (!rq[i].arrived) continue;
        if (!base && !rq[i].comp_issued) { pick = i; what = 0; }
        else if (rd.payload_order == 0 && !rq[i].full_issued) { pick = i; what = 1; }
      }
      for (int i = 0; i < n && pick < 0; ++i)
        if (rq[i].arrived && !rq[i].full_issued) { pick = i; what = 1; }
      if (pick < 0) break;
      const uint64_t id = en.prefix_load(slots[pick], what, rd.first_tokens[pick]);
      if (what == 0) { rq[pick].comp_issued = true; rq[pick].comp_id = id; }
      else { rq[pick].full_issued = true; rq[pick].full_id = id; }
      ++inflight;
    }
    // plan one forward pass
    std::vector<vc::StepItem> items;
    std::vector<int> drafting, verifying, decoding;
    if (base) {
      for (int i = 0; i < n; ++i)
        if (rq[i].full && !rq[i].done) {
          vc::StepItem s;
          s.slot = slots[i];
          s.mode = vc::RowMode::Decode;
          s.tokens = {en.seq(slots[i]).pending};
          items.push_back(std::move(s));
          decoding.push_back(i);
        }
    } else {
      std::vector<int> cand;
      for (int i = 0; i < n; ++i) {
        Req& r = rq[i];
        if (!r.active || r.done) continue;
        const int nd = static_cast<int>(en.seq(slots[i]).drafted.size());
        if (nd == rd.x && r.full) {
          if (r.ready_seq < 0) r.ready_seq = ready_counter++;
          cand.push_back(i);
        }
      }
      std::sort(cand.begin(), cand.end(), [&](int a, int b) { return rq[a].ready_seq < rq[b].ready_seq; });
      if (static_cast<int>(cand.size()) > cfgE.max_verify) cand.resize(cfgE.max_verify);
      verifying = cand;
      for (int i = 0; i < n; ++i) {
        Req& r = rq[i];
        if (!r.active || r.done) continue;
        const auto& s = en.seq(slots[i]);
        if (static_cast<int>(s.drafted.size()) < rd.x) {
          vc::StepItem d;
          d.slot = slots[i];
          d.mode = vc::RowMode::Draft;
          d.tokens = {s.drafted.empty() ? s.pending : s.drafted.back()};
          items.push_back(std::move(d));
          drafting.push_back(i);
        }
      }
      for (int i : verifying) {
        const auto& s = en.seq(slots[i]);
        vc::StepItem v;
        v.slot = slots[i];
        v.mode = vc::RowMode::Verify;
        v.tokens.push_back(s.pending);
        v.tokens.insert(v.tokens.end(), s.drafted.begin(), s.drafted.end());
        items.push_back(std::move(v));
      }
    }
    if (items.empty()) {
      bool all_done = true;
      for (const Req& r : rq) all_done = all_done && r.done;
      if (all_done) break;
      // nothing to compute: block on the oldest in-flight load, or the next arrival
      uint64_t wait_id = 0;  // the earliest-issued (the link is FIFO)
      auto consider = [&](uint64_t id) { if (!wait_id || id < wait_id) wait_id = id; };
      for (const Req& r : rq) {
        if (r.comp_issued && !r.active) consider(r.comp_id);
        if (r.full_issued && !r.full) consider(r.full_id);
      }
      if (wait_id) {
        en.swap_wait(wait_id);
        ++st.link_waits;
      } else {
        std::this_thread::sleep_for(std::chrono::microseconds(100));
      }
      continue;
    }
    en.run_step(items, row);
    st.iterations += 1;
    const double t_out = now_ms();
    auto emit = [&](int i, int32_t tok) {
      Req& r = rq[i];
      if (r.produced < rd.K) {
        out[static_cast<size_t>(i) * rd.K + r.produced++] = tok;
        st.tokens += 1;
        if (r.t_first < 0) r.t_first = t_out;
      }
      if (r.produced >= rd.K) r.done = true;
    };
    size_t off = 0;
    for (int i : decoding) {
      const int32_t tok = row[off++];
      en.commit_decode(slots[i], tok);
      emit(i, tok);
    }
    for (int i : drafting) en.push_draft(slots[i], row[off++]);
    for (int i : verifying) {
      const int x_r = static_cast<int>(en.seq(slots[i]).drafted.size());
      std::vector<int32_t> p(row.begin() + off, row.begin() + off + x_r + 1);
      off += x_r + 1;
      const auto em = en.accept_commit(slots[i], p);
      accepted_sum += static_cast<double>(em.size()) - 1;
      st.verifies += 1;
      rq[i].ready_seq = -1;
      for (int32_t tok : em) emit(i, tok);
    }
  }
  vc::check_cuda(cudaEventRecord(win1, en.stream()), "window event");
  vc::check_cuda(cudaEventSynchronize(win1), "window event");
  float wms = 0.f;
  vc::check_cuda(cudaEventElapsedTime(&wms, win0, win1), "window event");
  cudaEventDestroy(win0);
  cudaEventDestroy(win1);
  st.makespan_ms = wms;
  st.wall_ms = now_ms();
  st.mean_accept = st.verifies ? accepted_sum / static_cast<double>(st.verifies) : 0.0;
  for (const Req& r : rq) {
    const double ttft = r.t_first - r.t_arr;
    st.ttft_ms_mean += ttft / n;
    st.ttft_ms_max = std::max(st.ttft_ms_max, ttft);
    if (!base) st.compressed_ready_ms_mean += (r.t_comp - r.t_arr) / n;
    st.full_ready_ms_mean += (r.t_full - r.t_arr) / n;
  }
  st.h2d_bytes = en.h2d_bytes() - h2d_b0;
  st.h2d_ms = en.h2d_ms() - h2d_ms0;
  if (stats) *stats = st;
  return VC_OK;
}

// ---------------------------------------------------------------------------
// vc_run_decode_fifo: the reference's full-KV baseline (baseline_full_kv,
// /root/reference/proj/src/sim.cpp:418-494) on real kernels.  Requests are
// admitted FIFO (arrival order) while a full-KV slot is free -- the engine's
// max_slots HBM slots are its capacity (weights + resident + KV <= gpu_mem,
// :455-461) -- decode one token per step (:475-486) and leave after K.  The
// clock is the sum of the steps' device times, as the reference's clock is
// the sum of T_iter = (weights + resident) / BW per step (:471); admission
// (writing the request's prefix KV) is free in the reference and is not on
// the clock here either.
int vc_run_decode_fifo_impl(vc::Engine& en, const vc_request_desc* reqs, int n, int K, int32_t* out,
                            vc_loop_metrics* m) {
  const auto& cfgE = en.config();
  if (cfgE.full_tier != 0) throw speckv::ConfigError("fifo decode: needs the HBM full tier");
  if (n < 1 || K < 1) throw speckv::ConfigError("fifo decode: n and K must be >= 1");
  if (!reqs || !out) throw vc::ContractViolation("fifo decode: null workload");
  vc_loop_metrics st{};
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return reqs[a].arrival_ms < reqs[b].arrival_ms; });
  const int cap_tokens = en.full_pool().cap;
  std::deque<int> waiting;
  size_t next = 0;
  std::vector<int> free_slots;
  for (int s = cfgE.max_slots - 1; s >= 0; --s) free_slots.push_back(s);
  struct Active {
    int req, slot, produced;
  };
  std::vector<Active> active;
  std::vector<std::pair<double, double>> emission;
  std::vector<double> latency;
  double clock = 0.0;  // seconds of step device time
  const size_t slot_bytes = static_cast<size_t>(cap_tokens) * en.full_kv_bytes_per_token();
  double batch_sum = 0, full_tokens = 0, full_clock = 0;
  const auto w0 = std::chrono::steady_clock::now();
  std::vector<int32_t> row;
  while (next < order.size() || !waiting.empty() || !active.empty()) {
    while (next < order.size() && reqs[order[next]].arrival_ms <= clock * 1e3 + 1e-9) {
      const int r = order[next++];
      if (reqs[r].n_ctx + K + cfgE.max_x + 2 > cap_tokens) {  // can never fit (sim.cpp:438-440)
        st.unserved += 1;
        continue;
      }
      waiting.push_back(r);
    }
    while (!waiting.empty() && !free_slots.empty()) {  // FIFO admission
      const int r = waiting.front();
      waiting.pop_front();
      const int s = free_slots.back();
      free_slots.pop_back();
      en.add_request_synthetic(s, reqs[r].n_ctx, reqs[r].first_token, reqs[r].seed, 4, 10.f);
      active.push_back({r, s, 0});
    }
    if (active.empty()) {
      if (next < order.size()) {
        clock = std::max(clock, reqs[order[next]].arrival_ms / 1e3);
        continue;
      }
      break;
    }
    st.max_batch = std::max<int>(st.max_batch, static_cast<int>(active.size()));
    st.peak_hbm_bytes = std::max<int64_t>(st.peak_hbm_bytes, static_cast<int64_t>(en.weight_bytes() +
                                                                                  active.size() * slot_bytes));
    std::vector<vc::StepItem> its(active.size());
    for (size_t i = 0; i < active.size(); ++i) {
      its[i].slot = active[i].slot;
      its[i].mode = vc::RowMode::Decode;
      its[i].tokens = {en.seq(active[i].slot).pending};
    }
    const double before = en.device_ms();
    en.run_step(its, row);
    const double dt = (en.device_ms() - before) / 1e3;
    clock += dt;
    if (static_cast<int>(active.size()) == cfgE.max_slots) {
      full_tokens += static_cast<double>(active.size());
      full_clock += dt;
    }
    st.iterations += 1;
    batch_sum += static_cast<double>(active.size());
    std::vector<Active> still;
    for (size_t i = 0; i < active.size(); ++i) {
      Active a = active[i];
      en.commit_decode(a.slot, row[i]);
      out[static_cast<size_t>(a.req) * K + a.produced++] = row[i];
      if (a.produced == K) {
        latency.push_back(clock - reqs[a.req].arrival_ms / 1e3);
        st.completed += 1;
        en.release(a.slot);
        free_slots.push_back(a.slot);
      } else {
        still.push_back(a);
      }
    }
    emission.emplace_back(clock, static_cast<double>(active.size()));
    st.tokens += static_cast<int64_t>(active.size());
    active.swap(still);
  }
  st.clock_s = clock;
  st.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
  st.mean_batch = st.iterations ? batch_sum / static_cast<double>(st.iterations) : 0.0;
  st.throughput = clock > 0 ? static_cast<double>(st.tokens) / clock : 0.0;
  double warm = 0;
  for (const auto& [t, k] : emission)
    if (t >= 0.1 * clock && t <= 0.9 * clock) warm += k;
  st.warm_throughput = clock > 0 ? warm / (0.8 * clock) : 0.0;
  std::sort(latency.begin(), latency.end());
  auto pct = [&](double q) {
    if (latency.empty()) return 0.0;
    size_t r = static_cast<size_t>(std::ceil(q * static_cast<double>(latency.size())));
    r = std::min(std::max<size_t>(r, 1), latency.size());
    return latency[r - 1];
  };
  st.p50_latency_s = pct(0.5);
  st.p99_latency_s = pct(0.99);
  st.full_batch_throughput = full_clock > 0 ? full_tokens / full_clock : 0.0;
  if (m) *m = st;
  return VC_OK;
}
