// speckv_b200.hpp -- the reference's C++ API for the VeriCache decode-loop
// path, re-implemented by libvericache.so (namespace speckv, same names,
// argument meaning and error behaviour), so code written against the
// reference's compressor / specloop / scheduler headers links against this
// library instead.  Only the hot-path surface
// is provided; config JSON I/O, analytics, the simulator and the CLI are out
// of scope.
//
// Reference declarations each block mirrors (paths under /root/reference/proj):
//   errors, domain types ......... include/speckv/core.hpp:13-112
//   SystemConfig (no JSON) ....... include/speckv/config.hpp:20-47
//   compressor ................... include/speckv/compressor.hpp:12-101
//   draft / verify / accept ...... include/speckv/specloop.hpp:14-61, 103-107
//   swap scheduler ............... include/speckv/scheduler.hpp:16-244
#pragma once

#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <optional>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace speckv {

// ============================================================ errors / domain
using Bytes = std::int64_t;
using Seconds = double;
using RequestId = std::int64_t;
using ReservationId = std::uint64_t;
using Token = std::int32_t;
using TokenSeq = std::vector<Token>;

// Bad input; the message names the violated invariant.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// API misuse (programming error).
struct ContractError : std::logic_error {
  using std::logic_error::logic_error;
};

enum class Scenario { LongContext, RemotePrefix };

struct HardwareProfile {
  double hbm_bandwidth = 0.0;
  std::optional<double> interconnect_bandwidth;
  std::optional<double> storage_local_bandwidth;
  std::optional<double> storage_remote_bandwidth;
  Bytes gpu_mem = 0;
  int local_gpus = 0;
  int remote_gpus = 0;
  void validate(Scenario scenario) const;
  bool operator==(const HardwareProfile&) const = default;
};

struct ModelSpec {
  Bytes weights_bytes = 0;
  Bytes kv_bytes_per_token = 0;
  void validate() const;
  bool operator==(const ModelSpec&) const = default;
};

struct Request {
  RequestId id = 0;
  Seconds arrival = 0.0;
  Bytes kv_full_bytes = 0;
  double compression_ratio = 1.0;
  std::int64_t output_tokens = 1;
  bool speculating = true;
  void validate() const;
  bool operator==(const Request&) const = default;
};

struct AcceptanceModel {
  enum class Kind { PerTokenIid, Tabulated };
  Kind kind = Kind::PerTokenIid;
  std::map<double, double> per_token_prob;        // c -> p(c)
  std::map<double, std::map<int, double>> table;  // c -> (x -> gamma)
  void validate() const;
  bool operator==(const AcceptanceModel&) const = default;
};

double expected_gamma(const AcceptanceModel& model, int x, double c);
double implied_per_token_prob(const AcceptanceModel& model, int x, double c);
Bytes kv_full_bytes(const ModelSpec& model, std::int64_t context_tokens);

// ================================================================ compressor
enum class CompressorKind { DropUniform, DropWindow, QuantUniform };
enum class CompressorMode { Offline, Online };

struct CompressorSpec {
  CompressorKind kind = CompressorKind::DropUniform;
  CompressorMode mode = CompressorMode::Offline;
  Scenario scenario = Scenario::LongContext;
  double ratio = 0.25;
  int bits = 4;
  double per_iteration_overhead = 0.0;
  int window = 8;
  int sink_tokens = 0;

  void validate() const;
  bool is_token_dropping() const { return kind != CompressorKind::QuantUniform; }
  double effective_ratio() const;
  bool operator==(const CompressorSpec&) const = default;
};

struct KvShape {
  int layers = 1;
  int heads = 1;
  std::int64_t tokens = 0;
  Bytes bytes_per_token_per_head = 2;
  Bytes full_bytes() const {
    return static_cast<Bytes>(layers) * heads * tokens * bytes_per_token_per_head;
  }
};

struct CompressedKVMeta {
  std::vector<std::vector<std::vector<std::int64_t>>> dropped_indices;  // [layer][head]
  int bit_scheme = 16;
  Bytes payload_bytes = 0;
  std::int64_t retained_tokens(const KvShape& shape, int layer) const;
  void check_invariants(const KvShape& shape) const;
};

CompressedKVMeta compress(const CompressorSpec& spec, const KvShape& shape, double ratio,
                          std::uint64_t seed = 0);

struct DecompressedKV {
  Bytes bytes = 0;
  std::vector<std::int64_t> retained_per_layer;
  bool lossless = false;
};
DecompressedKV decompress(const CompressorSpec& spec, const CompressedKVMeta& meta,
                          const KvShape& shape);

struct OnlineRequestKv {
  KvShape shape;
  std::vector<std::vector<std::vector<std::int64_t>>> dropped_indices;
  std::int64_t dropped_count(int layer) const;
};

std::vector<std::vector<std::vector<std::int64_t>>> update(
    const CompressorSpec& spec, int layer_index, std::span<const OnlineRequestKv> batch,
    const std::vector<std::pair<std::int64_t, std::int64_t>>& req_offsets);

void check_mode_exclusivity(std::span<const CompressorSpec> specs);

// ============================================================ draft / verify
struct TokenOracle {
  std::function<Token(std::span<const Token>)> next;
  Token operator()(std::span<const Token> prefix) const { return next(prefix); }
};

struct SpecRoundResult {
  TokenSeq drafted;
  TokenSeq predictions;
  TokenSeq accepted;
  bool bonus_used = false;
  std::optional<int> first_mismatch;
};

struct SpecRunStats {
  std::vector<int> accepted_per_round;
  int rounds() const { return static_cast<int>(accepted_per_round.size()); }
};

TokenSeq draft(const TokenOracle& drafter, std::span<const Token> prefix, int x);
TokenSeq verify(const TokenOracle& verifier, std::span<const Token> prefix,
                std::span<const Token> drafted);
SpecRoundResult accept(std::span<const Token> drafted, std::span<const Token> predictions);
std::pair<TokenSeq, SpecRunStats> run_speculative(const TokenOracle& drafter,
                                                  const TokenOracle& verifier,
                                                  std::span<const Token> prompt,
                                                  std::int64_t output_tokens, int x);
TokenSeq autoregress(const TokenOracle& oracle, std::span<const Token> prompt,
                     std::int64_t output_tokens);
TokenOracle random_table_oracle(int vocab_size, std::uint64_t seed);

// ============================================================== config
enum class IterationTimeMode { Derived, Fixed };
enum class AcceptanceRealization { SeededDraws, DeterministicMean };

struct SystemConfig {
  HardwareProfile hardware;
  ModelSpec model;
  AcceptanceModel acceptance;
  int draft_length = 1;
  int lookahead_window = 2;
  IterationTimeMode iteration_time_mode = IterationTimeMode::Derived;
  std::optional<double> iteration_time;
  AcceptanceRealization acceptance_realization = AcceptanceRealization::SeededDraws;
  int batch_size = 1;
  Bytes kv_full_bytes = 1;
  double compression_ratio = 1.0;
  std::int64_t output_tokens = 1;
  std::optional<double> decode_time;
  std::optional<double> verify_forward_time;
  bool verify_cached = false;
  Scenario scenario = Scenario::LongContext;
  std::optional<CompressorSpec> compressor;
  void validate() const;
};

// ============================================================ swap scheduler
struct ReloadSpan {
  double iterations = 0.0;
  int windows = 1;
};
ReloadSpan reload_span(Bytes kv_full_bytes, double bandwidth, double iteration_time);

struct Reservation {
  ReservationId id = 0;
  RequestId request_id = 0;
  int verify_window = 0;
  int span_windows = 1;
  std::int64_t verify_iteration = 0;
  std::int64_t span_begin = 0;
  double per_window_bw = 0.0;
  Bytes bytes = 0;
  Bytes transfer_bytes = 0;
};

struct AdmitProbe {
  std::vector<int> examined;
};

class ReserveRings {
 public:
  ReserveRings(int window, double iteration_time, double bandwidth, Bytes hbm_capacity,
               Bytes weights_bytes);
  std::optional<Reservation> admit(RequestId request, Bytes transfer_bytes, int anchor_x,
                                   AdmitProbe* probe = nullptr,
                                   std::optional<Bytes> hbm_bytes = std::nullopt);
  void release(const Reservation& reservation);
  struct Retired {
    std::vector<Reservation> consumed;
  };
  Retired advance();
  void set_iteration_time(double t);
  double iteration_time() const { return t_iter_; }
  double bandwidth() const { return bw_; }
  int window() const { return static_cast<int>(slots_.size()); }
  std::int64_t base_iteration() const { return base_; }
  double bw_reserved(int i) const;
  Bytes hbm_inflight(int i) const;
  Bytes kv_resident() const { return resident_; }
  Bytes hbm_capacity() const { return capacity_; }
  Bytes weights_bytes() const { return weights_; }
  void add_resident(Bytes bytes);
  void remove_resident(Bytes bytes);
  std::size_t live_reservations() const { return live_.size(); }
  void check_invariants() const;

 private:
  struct Slot {  // one lookahead window's ledger
    std::map<ReservationId, std::pair<double, Bytes>> charges;  // id -> (seconds, bytes)
    double seconds = 0.0;
    Bytes bytes = 0;
  };
  bool fits(int first, int last, double seconds, Bytes bytes) const;
  std::deque<Slot> slots_;
  std::map<ReservationId, Reservation> live_;
  double t_iter_, t_cap_, bw_;
  Bytes capacity_, weights_, resident_ = 0;
  std::int64_t base_ = 0;
  ReservationId next_ = 1;
};

enum class SessionMode { Speculative, Waiting, NonSpeculating };

struct SpecSession {
  RequestId id = 0;
  SessionMode mode = SessionMode::Waiting;
  double tokens_emitted = 0.0;
  int drafted_in_round = 0;
  std::optional<Reservation> pending;
  std::optional<Reservation> arrival_load;
  Bytes kv_full_bytes = 0;
  double compression_ratio = 1.0;
  std::int64_t output_tokens = 0;
  bool speculating = true;
  bool loaded = false;
  bool stalled = false;
  Seconds arrival = 0.0;
  Bytes resident_bytes() const;
};

class RoundSampler {
 public:
  virtual ~RoundSampler() = default;
  virtual double accepted_drafted(int drafted, double compression_ratio) = 0;
};

class MeanRoundSampler : public RoundSampler {
 public:
  explicit MeanRoundSampler(const AcceptanceModel& model) : model_(&model) {}
  double accepted_drafted(int drafted, double c) override;

 private:
  const AcceptanceModel* model_;
};

class GeometricRoundSampler : public RoundSampler {
 public:
  GeometricRoundSampler(const AcceptanceModel& model, std::uint64_t seed);
  double accepted_drafted(int drafted, double c) override;

 private:
  const AcceptanceModel* model_;
  std::uint64_t state_;
  std::map<std::pair<int, double>, double> p_cache_;
};

struct StepEvents {
  std::vector<Request> arrivals;
  std::vector<ReservationId> completed_transfers;
};

struct VerifyOutcome {
  RequestId request = 0;
  ReservationId reservation = 0;
  int drafted = 0;
  double emitted = 0.0;
  bool finished = false;
  bool was_late = false;
};

struct StepResult {
  std::vector<Reservation> reload_starts;
  std::vector<VerifyOutcome> verifies;
  std::vector<RequestId> admitted;
  std::vector<RequestId> to_waiting;
  std::vector<RequestId> completed;
  std::vector<ReservationId> late_transfers;
  std::vector<Reservation> consumed;
  std::vector<RequestId> activated;
  int drafting_count = 0;
  int verify_count = 0;
  double tokens_emitted = 0.0;
  Bytes hbm_read_bytes = 0;
  // B200 extension: the sessions that drafted this iteration (id order).
  std::vector<RequestId> drafted;
};

class SpecScheduler {
 public:
  SpecScheduler(const SystemConfig& config, RoundSampler& sampler);
  StepResult execution_step(const StepEvents& events);
  std::vector<Reservation> pending_kickoffs() const;
  const ReserveRings& rings() const { return rings_; }
  std::int64_t iteration() const { return iteration_; }
  const std::map<RequestId, SpecSession>& sessions() const { return sessions_; }
  std::size_t waiting_size() const { return waiting_.size(); }
  bool idle() const;
  void set_planning_iteration_time(double t) { rings_.set_iteration_time(t); }
  int active_batch() const;
  // B200 extension: swap the sampler (the engine plans a step on a copy with
  // a recording sampler, then replays it with measured accept counts).
  void set_sampler(RoundSampler& sampler) { sampler_ = &sampler; }
  // B200 extension: verify a fully drafted round as soon as its reload has
  // landed rather than at the booked verify iteration (default off = the
  // reference's Algorithm 1 exactly; the engine's scheduled loop turns it on).
  void set_expedite(bool on) { expedite_ = on; }

 private:
  void admit_for_verify(SpecSession& s, StepResult& r);
  void admit_for_arrival(SpecSession& s, StepResult& r);
  void verify_now(SpecSession& s, StepResult& r, bool late);
  void activate(SpecSession& s, StepResult& r);

  const SystemConfig* cfg_;
  RoundSampler* sampler_;
  ReserveRings rings_;
  std::int64_t iteration_ = 0;
  std::map<RequestId, SpecSession> sessions_;
  std::deque<RequestId> waiting_;
  std::vector<RequestId> readmit_;
  std::set<ReservationId> done_;
  bool expedite_ = false;
};

}  // namespace speckv
