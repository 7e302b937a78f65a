// speckv_host.cpp -- host half of the drop-in API (include/speckv_b200.hpp):
// compressor metadata, the draft/verify/accept protocol and the swap
// scheduler.  Same semantics as the reference (cited per function) so the
// reference's unit vectors and its 100k-iteration soak digest reproduce
// bit-for-bit (tests/test_scheduler_parity.py); the data plane behind them
// lives in the CUDA kernels.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <random>

#include "speckv_b200.hpp"

namespace speckv {

namespace {

constexpr double kRatioTol = 1e-9;   // ratio keys come from text (core.cpp:14)
constexpr double kBwSlack = 1e-9;    // BW-ring fit tolerance (scheduler.cpp:11)

void need(bool ok, const char* msg) {
  if (!ok) throw ConfigError(msg);
}

std::uint64_t mix64(std::uint64_t x) {  // splitmix64 (util.hpp:30-35)
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <class Map>
typename Map::const_iterator ratio_lookup(const Map& m, double c) {
  auto it = m.lower_bound(c - kRatioTol);
  if (it != m.end() && std::abs(it->first - c) <= kRatioTol) return it;
  return m.end();
}

// sum_{k=1..x} p^k, the expected leading run of a truncated geometric
double leading_run(double p, int x) {
  if (p >= 1.0) return static_cast<double>(x);
  if (p <= 0.0) return 0.0;
  return p * (1.0 - std::pow(p, x)) / (1.0 - p);
}

}  // namespace

// ------------------------------------------------------------------ domain
void HardwareProfile::validate(Scenario scenario) const {  // core.cpp:37-59
  need(hbm_bandwidth > 0, "hbm_bandwidth must be > 0");
  need(gpu_mem > 0, "gpu_mem must be > 0");
  need(local_gpus >= 0 && remote_gpus >= 0, "gpu counts must be >= 0");
  need(local_gpus + remote_gpus >= 1, "local_gpus + remote_gpus must be >= 1");
  for (const auto* v : {&interconnect_bandwidth, &storage_local_bandwidth, &storage_remote_bandwidth})
    if (v->has_value()) need(**v > 0, "link bandwidths must be > 0");
  if (scenario == Scenario::LongContext) {
    need(interconnect_bandwidth.has_value(), "interconnect_bandwidth is required under scenario=long-context");
  } else {
    need(storage_local_bandwidth.has_value(), "storage_local_bandwidth (BW_h) is required under scenario=remote-prefix");
    need(storage_remote_bandwidth.has_value(), "storage_remote_bandwidth (BW_l) is required under scenario=remote-prefix");
    need(*storage_local_bandwidth > *storage_remote_bandwidth,
         "remote-prefix requires storage_local_bandwidth > storage_remote_bandwidth");
  }
}

void ModelSpec::validate() const {
  need(weights_bytes > 0, "weights_bytes must be > 0");
  need(kv_bytes_per_token > 0, "kv_bytes_per_token must be > 0");
}

void Request::validate() const {
  need(kv_full_bytes > 0, "kv_full_bytes must be > 0");
  need(compression_ratio > 0.0 && compression_ratio <= 1.0, "compression_ratio out of (0,1]");
  need(output_tokens >= 1, "output_tokens must be >= 1");
}

void AcceptanceModel::validate() const {  // core.cpp:73-96
  if (kind == Kind::PerTokenIid) {
    need(!per_token_prob.empty(), "per-token-iid acceptance model needs per_token_prob");
    for (const auto& [c, p] : per_token_prob) {
      need(c > 0.0 && c <= 1.0, "per_token_prob key out of (0,1]");
      need(p >= 0.0 && p <= 1.0, "per_token_prob value out of [0,1]");
      if (c == 1.0) need(p == 1.0, "per_token_prob at c=1 must be 1 (no compression)");
    }
    return;
  }
  need(!table.empty(), "tabulated acceptance model needs a table");
  for (const auto& [c, by_x] : table) {
    need(c > 0.0 && c <= 1.0, "tabulated c out of (0,1]");
    double prev = std::numeric_limits<double>::infinity();
    for (const auto& [x, g] : by_x) {
      need(x >= 1, "tabulated x must be >= 1");
      need(g >= 0.0 && g <= 1.0, "tabulated gamma out of [0,1]");
      need(g <= prev, "tabulated gamma must be non-increasing in x for fixed c");
      if (c == 1.0) need(g == 1.0, "tabulated gamma at c=1 must be 1");
      prev = g;
    }
  }
}

double expected_gamma(const AcceptanceModel& model, int x, double c) {  // core.cpp:117-146
  if (x < 1) throw ContractError("expected_gamma: x must be >= 1");
  if (!(c > 0.0 && c <= 1.0)) throw ContractError("expected_gamma: c out of (0,1]");
  if (model.kind == AcceptanceModel::Kind::PerTokenIid) {
    auto it = ratio_lookup(model.per_token_prob, c);
    double p;
    if (it != model.per_token_prob.end()) p = it->second;
    else if (c == 1.0) p = 1.0;
    else throw ConfigError("acceptance model has no per_token_prob entry for this c");
    return leading_run(p, x) / static_cast<double>(x);
  }
  auto grp = ratio_lookup(model.table, c);
  if (grp == model.table.end()) {
    if (c == 1.0) return 1.0;
    throw ConfigError("acceptance table has no entries for this c");
  }
  const auto& by_x = grp->second;
  auto hi = by_x.lower_bound(x);
  if (hi != by_x.end() && hi->first == x) return hi->second;
  if (hi == by_x.begin()) return hi->second;
  if (hi == by_x.end()) return std::prev(hi)->second;
  auto lo = std::prev(hi);
  return (hi->first - x < x - lo->first) ? hi->second : lo->second;  // ties -> smaller x
}

double implied_per_token_prob(const AcceptanceModel& model, int x, double c) {  // core.cpp:148-165
  if (model.kind == AcceptanceModel::Kind::PerTokenIid) {
    auto it = ratio_lookup(model.per_token_prob, c);
    if (it != model.per_token_prob.end()) return it->second;
    if (c == 1.0) return 1.0;
    throw ConfigError("acceptance model has no per_token_prob entry for this c");
  }
  const double target = expected_gamma(model, x, c) * x;
  if (target >= static_cast<double>(x)) return 1.0;
  if (target <= 0.0) return 0.0;
  double lo = 0.0, hi = 1.0;
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    (leading_run(mid, x) < target ? lo : hi) = mid;
  }
  return 0.5 * (lo + hi);
}

Bytes kv_full_bytes(const ModelSpec& model, std::int64_t context_tokens) {
  if (context_tokens < 0) throw ContractError("kv_full_bytes: context_tokens must be >= 0");
  if (context_tokens != 0 && model.kv_bytes_per_token > std::numeric_limits<Bytes>::max() / context_tokens)
    throw ContractError("kv_full_bytes: product overflows 64-bit bytes");
  return model.kv_bytes_per_token * context_tokens;
}

// --------------------------------------------------------------- compressor
void CompressorSpec::validate() const {  // compressor.cpp:38-56
  if (is_token_dropping()) {
    need(ratio > 0.0 && ratio < 1.0, "compressor.ratio out of (0,1)");
  } else {
    need(bits >= 1 && bits <= 16, "compressor.bits out of [1,16]");
  }
  if (mode == CompressorMode::Online) {
    need(per_iteration_overhead >= 0.0, "compressor.per_iteration_overhead must be >= 0");
    need(kind != CompressorKind::QuantUniform, "quant-uniform compressor is offline only");
  }
  if (kind == CompressorKind::DropWindow) {
    need(window >= 1, "compressor.window must be >= 1");
    need(sink_tokens >= 0, "compressor.sink_tokens must be >= 0");
  }
}

double CompressorSpec::effective_ratio() const {
  return kind == CompressorKind::QuantUniform ? bits / 16.0 : ratio;
}

std::int64_t CompressedKVMeta::retained_tokens(const KvShape& shape, int layer) const {
  if (layer < 0 || layer >= shape.layers) throw ContractError("retained_tokens: bad layer");
  if (dropped_indices.empty() || dropped_indices.at(layer).empty()) return shape.tokens;
  return shape.tokens - static_cast<std::int64_t>(dropped_indices[layer].front().size());
}

void CompressedKVMeta::check_invariants(const KvShape& shape) const {  // compressor.cpp:71-101
  if (bit_scheme < 1 || bit_scheme > 16) throw ContractError("bit_scheme out of [1,16]");
  Bytes kept_bytes = 0;
  for (int l = 0; l < shape.layers; ++l) {
    std::size_t per_head = 0;
    if (!dropped_indices.empty() && !dropped_indices.at(l).empty()) {
      const auto& heads = dropped_indices[l];
      if (static_cast<int>(heads.size()) != shape.heads) throw ContractError("dropped_indices head count mismatch");
      per_head = heads.front().size();
      for (const auto& pos : heads) {
        if (pos.size() != per_head) throw ContractError("heads within a layer must drop the same count of tokens");
        for (auto p : pos)
          if (p < 0 || p >= shape.tokens) throw ContractError("dropped position out of range");
      }
    }
    kept_bytes += (shape.tokens - static_cast<std::int64_t>(per_head)) * shape.heads * shape.bytes_per_token_per_head;
  }
  if (kept_bytes * bit_scheme / 16 != payload_bytes)
    throw ContractError("payload_bytes inconsistent with retained tokens and bit_scheme");
}

CompressedKVMeta compress(const CompressorSpec& spec, const KvShape& shape, double ratio,
                          std::uint64_t seed) {  // compressor.cpp:130-178
  CompressedKVMeta meta;
  meta.dropped_indices.assign(shape.layers, std::vector<std::vector<std::int64_t>>(shape.heads));
  auto payload = [&](std::int64_t kept, int bits) {
    return static_cast<Bytes>(shape.layers) * kept * shape.heads * shape.bytes_per_token_per_head * bits / 16;
  };
  if (shape.tokens == 0) {
    meta.bit_scheme = spec.kind == CompressorKind::QuantUniform ? spec.bits : 16;
    meta.payload_bytes = 0;
    return meta;
  }
  if (spec.kind == CompressorKind::QuantUniform) {
    meta.bit_scheme = spec.bits;
    meta.payload_bytes = payload(shape.tokens, spec.bits);
    meta.check_invariants(shape);
    return meta;
  }
  if (!(ratio > 0.0 && ratio < 1.0)) throw ConfigError("compress: ratio out of (0,1)");
  const std::int64_t kept = static_cast<std::int64_t>(std::llround(ratio * shape.tokens));
  if (kept < 1) throw ConfigError("compress: ratio would retain < 1 token/head");
  const std::int64_t drop = shape.tokens - kept;
  meta.bit_scheme = 16;
  std::mt19937_64 rng(mix64(seed));
  std::vector<std::int64_t> perm;
  for (int l = 0; l < shape.layers; ++l)
    for (int h = 0; h < shape.heads; ++h) {
      std::vector<std::int64_t> out(drop);
      if (spec.kind == CompressorKind::DropUniform) {
        // seeded partial Fisher-Yates over [0, tokens), sorted (:114-126)
        perm.resize(shape.tokens);
        std::iota(perm.begin(), perm.end(), 0);
        for (std::int64_t i = 0; i < drop; ++i) {
          const std::int64_t j = i + static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(shape.tokens - i));
          std::swap(perm[i], perm[j]);
        }
        std::copy(perm.begin(), perm.begin() + drop, out.begin());
        std::sort(out.begin(), out.end());
      } else {
        std::iota(out.begin(), out.end(), static_cast<std::int64_t>(spec.sink_tokens));  // oldest non-sink
      }
      meta.dropped_indices[l][h] = std::move(out);
    }
  meta.payload_bytes = payload(kept, 16);
  meta.check_invariants(shape);
  return meta;
}

DecompressedKV decompress(const CompressorSpec& spec, const CompressedKVMeta& meta,
                          const KvShape& shape) {  // compressor.cpp:180-200
  meta.check_invariants(shape);
  DecompressedKV out;
  for (int l = 0; l < shape.layers; ++l) out.retained_per_layer.push_back(meta.retained_tokens(shape, l));
  if (spec.kind == CompressorKind::QuantUniform) {
    out.bytes = meta.payload_bytes * 16 / meta.bit_scheme;
    out.lossless = false;
    return out;
  }
  out.bytes = meta.payload_bytes;
  out.lossless = std::all_of(out.retained_per_layer.begin(), out.retained_per_layer.end(),
                             [&](std::int64_t r) { return r == shape.tokens; });
  return out;
}

std::int64_t OnlineRequestKv::dropped_count(int layer) const {
  if (dropped_indices.empty() || dropped_indices.at(layer).empty()) return 0;
  return static_cast<std::int64_t>(dropped_indices[layer].front().size());
}

std::vector<std::vector<std::vector<std::int64_t>>> update(
    const CompressorSpec& spec, int layer_index, std::span<const OnlineRequestKv> batch,
    const std::vector<std::pair<std::int64_t, std::int64_t>>& req_offsets) {  // compressor.cpp:208-243
  if (spec.mode != CompressorMode::Online) throw ContractError("update: compressor mode is offline; update is unsupported");
  if (req_offsets.size() != batch.size()) throw ContractError("update: req_offsets must have one [begin,end) per request");
  std::int64_t at = 0;
  for (std::size_t i = 0; i < batch.size(); ++i) {
    if (req_offsets[i].first != at || req_offsets[i].second - req_offsets[i].first != batch[i].shape.tokens)
      throw ContractError("update: req_offsets do not partition the batch token axis");
    at = req_offsets[i].second;
  }
  std::vector<std::vector<std::vector<std::int64_t>>> out(batch.size());
  for (std::size_t i = 0; i < batch.size(); ++i) {
    const auto& r = batch[i];
    if (layer_index < 0 || layer_index >= r.shape.layers) throw ContractError("update: layer_index out of range");
    const std::int64_t done = r.dropped_count(layer_index);
    const std::int64_t keep_budget = spec.sink_tokens + spec.window;
    const std::int64_t n = std::max<std::int64_t>(0, r.shape.tokens - done - keep_budget);
    std::vector<std::int64_t> pos(n);
    std::iota(pos.begin(), pos.end(), spec.sink_tokens + done);
    out[i].assign(r.shape.heads, pos);
  }
  return out;
}

void check_mode_exclusivity(std::span<const CompressorSpec> specs) {
  if (specs.empty()) return;
  const bool dropping = specs.front().is_token_dropping();
  for (const auto& s : specs)
    if (s.is_token_dropping() != dropping)
      throw ConfigError("mixing token-dropping and quantization compressors in one run is not allowed");
}

// --------------------------------------------------------- draft / verify
TokenSeq draft(const TokenOracle& drafter, std::span<const Token> prefix, int x) {  // specloop.cpp:11-22
  if (x < 1) throw ContractError("draft: x must be >= 1");
  TokenSeq ctx(prefix.begin(), prefix.end()), out;
  for (int i = 0; i < x; ++i) {
    out.push_back(drafter(ctx));
    ctx.push_back(out.back());
  }
  return out;
}

TokenSeq verify(const TokenOracle& verifier, std::span<const Token> prefix,
                std::span<const Token> drafted) {  // specloop.cpp:24-35
  if (drafted.empty()) throw ContractError("verify: drafted must be non-empty");
  TokenSeq ctx(prefix.begin(), prefix.end()), preds;
  for (std::size_t k = 0; k <= drafted.size(); ++k) {
    preds.push_back(verifier(ctx));
    if (k < drafted.size()) ctx.push_back(drafted[k]);
  }
  return preds;
}

SpecRoundResult accept(std::span<const Token> drafted, std::span<const Token> predictions) {  // specloop.cpp:37-56
  if (predictions.size() != drafted.size() + 1)
    throw ContractError("accept: |predictions| must equal |drafted| + 1");
  SpecRoundResult r;
  r.drafted.assign(drafted.begin(), drafted.end());
  r.predictions.assign(predictions.begin(), predictions.end());
  std::size_t k = 0;
  while (k < drafted.size() && drafted[k] == predictions[k]) ++k;
  r.accepted.assign(drafted.begin(), drafted.begin() + k);
  r.accepted.push_back(predictions[k]);
  if (k < drafted.size()) r.first_mismatch = static_cast<int>(k) + 1;
  else r.bonus_used = true;
  return r;
}

std::pair<TokenSeq, SpecRunStats> run_speculative(const TokenOracle& drafter,
                                                  const TokenOracle& verifier,
                                                  std::span<const Token> prompt,
                                                  std::int64_t output_tokens, int x) {  // specloop.cpp:58-79
  if (output_tokens < 1) throw ContractError("run_speculative: K must be >= 1");
  if (x < 1) throw ContractError("run_speculative: x must be >= 1");
  TokenSeq ctx(prompt.begin(), prompt.end()), out;
  SpecRunStats stats;
  while (static_cast<std::int64_t>(out.size()) < output_tokens) {
    const TokenSeq d = draft(drafter, ctx, x);
    const SpecRoundResult r = accept(d, verify(verifier, ctx, d));
    stats.accepted_per_round.push_back(static_cast<int>(r.accepted.size()));
    out.insert(out.end(), r.accepted.begin(), r.accepted.end());
    ctx.insert(ctx.end(), r.accepted.begin(), r.accepted.end());
  }
  out.resize(output_tokens);
  return {std::move(out), std::move(stats)};
}

TokenSeq autoregress(const TokenOracle& oracle, std::span<const Token> prompt,
                     std::int64_t output_tokens) {
  TokenSeq ctx(prompt.begin(), prompt.end()), out;
  for (std::int64_t i = 0; i < output_tokens; ++i) {
    out.push_back(oracle(ctx));
    ctx.push_back(out.back());
  }
  return out;
}

TokenOracle random_table_oracle(int vocab_size, std::uint64_t seed) {  // specloop.cpp:265-273
  if (vocab_size < 1) throw ContractError("random_table_oracle: vocab_size must be >= 1");
  TokenOracle o;
  o.next = [vocab_size, seed](std::span<const Token> prefix) {
    std::uint64_t h = mix64(seed ^ 0x9e3779b97f4a7c15ull);
    for (Token t : prefix) h = mix64(h ^ static_cast<std::uint64_t>(t + 1));
    return static_cast<Token>(h % static_cast<std::uint64_t>(vocab_size));
  };
  return o;
}

// ------------------------------------------------------------------ config
void SystemConfig::validate() const {  // config.cpp:131-156
  hardware.validate(scenario);
  model.validate();
  acceptance.validate();
  need(draft_length >= 1, "draft_length must be >= 1");
  need(lookahead_window >= 2, "lookahead_window must be >= 2");
  if (iteration_time_mode == IterationTimeMode::Fixed)
    need(iteration_time.has_value() && *iteration_time > 0,
         "iteration_time > 0 is required under iteration_time_mode=fixed");
  need(batch_size >= 1, "batch_size must be >= 1");
  need(kv_full_bytes > 0, "kv_full_bytes must be > 0");
  need(compression_ratio > 0.0 && compression_ratio <= 1.0, "compression_ratio out of (0,1]");
  need(output_tokens >= 1, "output_tokens must be >= 1");
  if (decode_time) need(*decode_time >= 0, "decode_time must be >= 0");
  if (verify_forward_time) need(*verify_forward_time >= 0, "verify_forward_time must be >= 0");
  if (compressor) {
    compressor->validate();
    need(compressor->scenario == scenario, "compressor.scenario must match scenario");
  }
}

// ============================================================ reserve rings
ReloadSpan reload_span(Bytes kv_full_bytes, double bandwidth, double iteration_time) {  // scheduler.cpp:15-23
  if (kv_full_bytes <= 0 || bandwidth <= 0 || iteration_time <= 0)
    throw ContractError("reload_span: inputs must be positive");
  ReloadSpan s;
  s.iterations = static_cast<double>(kv_full_bytes) / (bandwidth * iteration_time);
  s.windows = std::max(1, static_cast<int>(std::ceil(s.iterations)));
  return s;
}

ReserveRings::ReserveRings(int window, double iteration_time, double bandwidth, Bytes hbm_capacity,
                           Bytes weights_bytes)
    : t_iter_(iteration_time), t_cap_(iteration_time), bw_(bandwidth), capacity_(hbm_capacity),
      weights_(weights_bytes) {
  if (window < 2) throw ContractError("ReserveRings: window must be >= 2");
  if (iteration_time <= 0 || bandwidth <= 0)
    throw ContractError("ReserveRings: iteration_time and bandwidth must be positive");
  if (weights_bytes > hbm_capacity) throw ContractError("ReserveRings: weights do not fit in HBM");
  slots_.resize(window);
}

void ReserveRings::set_iteration_time(double t) {
  if (t <= 0) throw ContractError("set_iteration_time: must be positive");
  t_iter_ = t;
  // bookings made under a larger T_iter stay legal until the live set drains
  t_cap_ = live_.empty() ? t : std::max(t_cap_, t);
}

double ReserveRings::bw_reserved(int i) const {
  if (i < 0 || i >= window()) throw ContractError("bw_reserved: window index out of range");
  return slots_[i].seconds;
}

Bytes ReserveRings::hbm_inflight(int i) const {
  if (i < 0 || i >= window()) throw ContractError("hbm_inflight: window index out of range");
  return slots_[i].bytes;
}

void ReserveRings::add_resident(Bytes b) {
  if (b < 0) throw ContractError("add_resident: negative bytes");
  resident_ += b;
}

void ReserveRings::remove_resident(Bytes b) {
  if (b < 0 || b > resident_) throw ContractError("remove_resident: underflow");
  resident_ -= b;
}

bool ReserveRings::fits(int first, int last, double seconds, Bytes bytes) const {
  for (int i = first; i <= last; ++i) {
    if (slots_[i].seconds + seconds > t_iter_ * (1.0 + kBwSlack)) return false;
    if (weights_ + resident_ + slots_[i].bytes + bytes > capacity_) return false;
  }
  return true;
}

std::optional<Reservation> ReserveRings::admit(RequestId request, Bytes transfer_bytes, int anchor_x,
                                               AdmitProbe* probe, std::optional<Bytes> hbm_bytes) {
  // Algorithm 1 (scheduler.cpp:96-163)
  if (anchor_x < 1) throw ContractError("admit: anchor_x must be >= 1");
  const int W = window();
  const int span = reload_span(transfer_bytes, bw_, t_iter_).windows;
  if (span > W - 1) return std::nullopt;
  const Bytes bytes = hbm_bytes.value_or(transfer_bytes);
  const double seconds = static_cast<double>(transfer_bytes) / (bw_ * span);
  const int anchor = std::clamp(anchor_x, span, W - 1);
  auto book = [&](int d) -> std::optional<Reservation> {
    if (probe) probe->examined.push_back(d);
    const int first = d - span + 1;
    if (!fits(first, d, seconds, bytes)) return std::nullopt;
    Reservation r;
    r.id = next_++;
    r.request_id = request;
    r.verify_window = d;
    r.span_windows = span;
    r.verify_iteration = base_ + d;
    r.span_begin = base_ + first;
    r.per_window_bw = seconds;
    r.bytes = bytes;
    r.transfer_bytes = transfer_bytes;
    for (int i = first; i <= d; ++i) {
      slots_[i].charges.emplace(r.id, std::make_pair(seconds, bytes));
      slots_[i].seconds += seconds;  // incremental; equals the id-ordered sum
      slots_[i].bytes += bytes;
    }
    live_.emplace(r.id, r);
    return r;
  };
  // anchor, anchor-1, anchor+1, anchor-2, ... (earlier first at each distance)
  for (int k = 0;; ++k) {
    const int lo = anchor - k, hi = anchor + k;
    const bool lo_ok = lo >= span, hi_ok = hi <= W - 1;
    if (!lo_ok && !hi_ok) break;
    if (lo_ok)
      if (auto r = book(lo)) return r;
    if (k > 0 && hi_ok)
      if (auto r = book(hi)) return r;
  }
  return std::nullopt;
}

void ReserveRings::release(const Reservation& res) {
  auto it = live_.find(res.id);
  if (it == live_.end()) throw ContractError("release: unknown or already-consumed reservation");
  for (std::int64_t abs = std::max(it->second.span_begin, base_); abs <= it->second.verify_iteration; ++abs) {
    Slot& s = slots_[abs - base_];
    s.charges.erase(res.id);
    // canonical id-ordered re-sum keeps release bit-exact
    s.seconds = 0.0;
    s.bytes = 0;
    for (const auto& [id, c] : s.charges) {
      s.seconds += c.first;
      s.bytes += c.second;
    }
  }
  live_.erase(it);
}

ReserveRings::Retired ReserveRings::advance() {
  Retired out;
  for (const auto& [id, c] : slots_.front().charges) {
    auto it = live_.find(id);
    if (it == live_.end()) throw ContractError("advance: ledger entry without live reservation");
    if (it->second.verify_iteration == base_) {
      out.consumed.push_back(it->second);
      live_.erase(it);
    }
  }
  slots_.pop_front();
  slots_.emplace_back();
  ++base_;
  return out;
}

void ReserveRings::check_invariants() const {  // scheduler.cpp:182-221
  std::map<ReservationId, int> seen;
  for (int i = 0; i < window(); ++i) {
    const Slot& s = slots_[i];
    double sec = 0.0;
    Bytes b = 0;
    for (const auto& [id, c] : s.charges) {
      sec += c.first;
      b += c.second;
      ++seen[id];
      auto it = live_.find(id);
      if (it == live_.end()) throw ContractError("ring invariant: entry without reservation");
      const std::int64_t abs = base_ + i;
      if (abs < it->second.span_begin || abs > it->second.verify_iteration)
        throw ContractError("ring invariant: charge outside its reservation span");
    }
    if (sec != s.seconds || b != s.bytes) throw ContractError("ring invariant: cached totals diverged from canonical sums");
    if (s.seconds > t_cap_ * (1.0 + kBwSlack)) throw ContractError("ring invariant: BW ring over-reserved (T[i] > T_iter)");
    if (weights_ + resident_ + s.bytes > capacity_) throw ContractError("ring invariant: HBM ring over capacity");
  }
  for (const auto& [id, r] : live_) {
    const int expect = static_cast<int>(r.verify_iteration - std::max(r.span_begin, base_) + 1);
    auto it = seen.find(id);
    if ((it == seen.end() ? 0 : it->second) != expect)
      throw ContractError("ring invariant: reservation mass leaked or duplicated");
  }
  for (const auto& [id, n] : seen)
    if (!live_.count(id)) throw ContractError("ring invariant: orphaned charge");
}

// ================================================================ sessions
Bytes SpecSession::resident_bytes() const {  // scheduler.cpp:225-229
  if (!speculating) return kv_full_bytes;
  return static_cast<Bytes>(std::ceil(compression_ratio * static_cast<double>(kv_full_bytes)));
}

double MeanRoundSampler::accepted_drafted(int drafted, double c) {
  if (drafted < 1) return 0.0;
  return expected_gamma(*model_, drafted, c) * drafted;
}

GeometricRoundSampler::GeometricRoundSampler(const AcceptanceModel& model, std::uint64_t seed)
    : model_(&model), state_(mix64(seed ^ 0x5bd1e995u)) {}

double GeometricRoundSampler::accepted_drafted(int drafted, double c) {  // scheduler.cpp:239-255
  if (drafted < 1) return 0.0;
  const auto key = std::make_pair(drafted, c);
  auto it = p_cache_.find(key);
  if (it == p_cache_.end()) it = p_cache_.emplace(key, implied_per_token_prob(*model_, drafted, c)).first;
  const double p = it->second;
  state_ = mix64(state_);
  if (p >= 1.0) return drafted;
  if (p <= 0.0) return 0.0;
  // invert one uniform into the leading-success run: P(N >= k) = p^k
  const double u = std::max(static_cast<double>(state_ >> 11) * 0x1.0p-53, 1e-300);
  const double run = std::floor(std::log(u) / std::log(p));
  return std::min(static_cast<double>(drafted), std::max(0.0, run));
}

// =============================================================== scheduler
namespace {
double first_iteration_time(const SystemConfig& c) {
  if (c.iteration_time_mode == IterationTimeMode::Fixed) return *c.iteration_time;
  return static_cast<double>(c.model.weights_bytes) / c.hardware.hbm_bandwidth;
}
double planning_link(const SystemConfig& c) {
  return c.scenario == Scenario::LongContext ? *c.hardware.interconnect_bandwidth
                                             : *c.hardware.storage_local_bandwidth;
}
const SystemConfig& validated(const SystemConfig& c) {
  c.validate();
  return c;
}
}  // namespace

SpecScheduler::SpecScheduler(const SystemConfig& config, RoundSampler& sampler)
    : cfg_(&validated(config)),
      sampler_(&sampler),
      rings_(config.lookahead_window, first_iteration_time(config), planning_link(config),
             config.hardware.gpu_mem, config.model.weights_bytes) {}

bool SpecScheduler::idle() const { return sessions_.empty() && waiting_.empty() && readmit_.empty(); }

int SpecScheduler::active_batch() const {
  int n = 0;
  for (const auto& [id, s] : sessions_) n += s.loaded ? 1 : 0;
  return n;
}

std::vector<Reservation> SpecScheduler::pending_kickoffs() const {
  std::vector<Reservation> out;
  for (const auto& [id, s] : sessions_) {
    if (s.pending && s.pending->span_begin == iteration_) out.push_back(*s.pending);
    if (s.arrival_load && s.arrival_load->span_begin == iteration_) out.push_back(*s.arrival_load);
  }
  return out;
}

void SpecScheduler::admit_for_verify(SpecSession& s, StepResult& r) {  // scheduler.cpp:303-316
  if (auto res = rings_.admit(s.id, s.kv_full_bytes, cfg_->draft_length)) {
    s.mode = SessionMode::Speculative;
    s.pending = *res;
    s.drafted_in_round = 0;
    s.stalled = false;
    r.admitted.push_back(s.id);
  } else {
    s.mode = SessionMode::Waiting;
    waiting_.push_back(s.id);
    r.to_waiting.push_back(s.id);
  }
}

void SpecScheduler::admit_for_arrival(SpecSession& s, StepResult& r) {  // scheduler.cpp:318-343
  const Bytes resident = s.resident_bytes();
  Bytes worst = 0;
  for (int i = 0; i < rings_.window(); ++i) worst = std::max(worst, rings_.hbm_inflight(i));
  std::optional<Reservation> res;
  if (rings_.weights_bytes() + rings_.kv_resident() + resident + worst <= rings_.hbm_capacity())
    res = rings_.admit(s.id, resident, 1, nullptr, Bytes{0});  // earliest feasible slot
  s.mode = SessionMode::Waiting;
  if (res) {
    rings_.add_resident(resident);
    s.arrival_load = *res;
    r.admitted.push_back(s.id);
  } else {
    waiting_.push_back(s.id);
    r.to_waiting.push_back(s.id);
  }
}

void SpecScheduler::verify_now(SpecSession& s, StepResult& r, bool late) {  // scheduler.cpp:345-374
  VerifyOutcome v;
  v.request = s.id;
  v.reservation = s.pending ? s.pending->id : 0;
  v.drafted = s.drafted_in_round;
  v.was_late = late;
  const double kept = sampler_->accepted_drafted(s.drafted_in_round, s.compression_ratio);
  v.emitted = std::min(kept + 1.0, static_cast<double>(s.output_tokens) - s.tokens_emitted);
  s.tokens_emitted += v.emitted;
  s.drafted_in_round = 0;
  s.stalled = false;
  if (s.pending) {
    done_.erase(s.pending->id);
    s.pending.reset();
  }
  v.finished = s.tokens_emitted >= static_cast<double>(s.output_tokens) - 1e-9;
  r.verifies.push_back(v);
  r.verify_count += 1;
  r.tokens_emitted += v.emitted;
  r.hbm_read_bytes += s.kv_full_bytes;
  if (v.finished) {
    rings_.remove_resident(s.resident_bytes());
    r.completed.push_back(s.id);
    sessions_.erase(s.id);
  } else {
    readmit_.push_back(s.id);
  }
}

void SpecScheduler::activate(SpecSession& s, StepResult& r) {
  s.arrival_load.reset();
  s.loaded = true;
  r.activated.push_back(s.id);
  if (s.speculating) readmit_.push_back(s.id);
  else s.mode = SessionMode::NonSpeculating;
}

StepResult SpecScheduler::execution_step(const StepEvents& ev) {  // scheduler.cpp:376-512
  StepResult r;
  done_.insert(ev.completed_transfers.begin(), ev.completed_transfers.end());

  // admissions: last step's verifies, FIFO retries, then arrivals
  std::vector<RequestId> again;
  again.swap(readmit_);
  for (RequestId id : again) {
    auto it = sessions_.find(id);
    if (it != sessions_.end()) admit_for_verify(it->second, r);
  }
  std::deque<RequestId> retry;
  retry.swap(waiting_);
  for (RequestId id : retry) {
    auto it = sessions_.find(id);
    if (it == sessions_.end()) continue;
    SpecSession& s = it->second;
    if (s.loaded) admit_for_verify(s, r);
    else if (!s.arrival_load) admit_for_arrival(s, r);
    else waiting_.push_back(id);  // load still in flight
  }
  for (const Request& q : ev.arrivals) {
    SpecSession s;
    s.id = q.id;
    s.kv_full_bytes = q.kv_full_bytes;
    s.compression_ratio = q.compression_ratio;
    s.output_tokens = q.output_tokens;
    s.speculating = q.speculating;
    s.arrival = q.arrival;
    auto [it, fresh] = sessions_.emplace(q.id, s);
    if (!fresh) throw ContractError("execution_step: duplicate request id");
    admit_for_arrival(it->second, r);
  }
  r.reload_starts = pending_kickoffs();

  // draft / verify / stall, in request-id order
  r.hbm_read_bytes = cfg_->model.weights_bytes;
  std::vector<RequestId> ids;
  for (const auto& [id, s] : sessions_) ids.push_back(id);
  for (RequestId id : ids) {
    auto it = sessions_.find(id);
    if (it == sessions_.end()) continue;
    SpecSession& s = it->second;
    if (!s.speculating && s.loaded) {  // plain decode off the full cache
      const double e = std::min(1.0, static_cast<double>(s.output_tokens) - s.tokens_emitted);
      s.tokens_emitted += e;
      r.tokens_emitted += e;
      r.hbm_read_bytes += s.kv_full_bytes;
      if (s.tokens_emitted >= static_cast<double>(s.output_tokens) - 1e-9) {
        rings_.remove_resident(s.resident_bytes());
        r.completed.push_back(id);
        sessions_.erase(it);
      }
      continue;
    }
    if (s.mode != SessionMode::Speculative || !s.pending) continue;
    const bool arrived = done_.count(s.pending->id) > 0;
    if (s.stalled) {
      if (arrived) verify_now(s, r, true);
      continue;
    }
    if (iteration_ < s.pending->verify_iteration) {
      if (s.drafted_in_round < cfg_->draft_length) {
        s.drafted_in_round += 1;
        r.drafting_count += 1;
        r.hbm_read_bytes += s.resident_bytes();
        r.drafted.push_back(id);
      } else if (expedite_ && arrived) {
        // B200 extension (off by default): the round is fully drafted and its
        // reload has landed -- verify now instead of idling to the booked
        // verify iteration; the ring bookings retire on their own schedule
        verify_now(s, r, false);
      }
      continue;
    }
    if (arrived) {
      verify_now(s, r, false);
    } else {
      r.late_transfers.push_back(s.pending->id);
      s.stalled = true;
    }
  }

  // slide the window; retire arrival loads whose span ended
  for (const Reservation& res : rings_.advance().consumed) {
    r.consumed.push_back(res);
    auto it = sessions_.find(res.request_id);
    if (it == sessions_.end()) continue;
    SpecSession& s = it->second;
    if (!s.arrival_load || s.arrival_load->id != res.id) continue;
    if (done_.count(res.id)) {
      done_.erase(res.id);
      activate(s, r);
    } else {
      r.late_transfers.push_back(res.id);
    }
  }
  for (auto& [id, s] : sessions_) {
    if (!s.loaded && s.arrival_load && s.arrival_load->verify_iteration < iteration_ &&
        done_.count(s.arrival_load->id)) {
      done_.erase(s.arrival_load->id);
      activate(s, r);
    }
  }
  rings_.check_invariants();
  ++iteration_;
  return r;
}

}  // namespace speckv
