// speckv_gpu_oracle.hpp -- the reference's TokenOracle backed by the B200
// engine (header-only, C-ABI only), so the reference's own protocol code
//   speckv::run_speculative(drafter, verifier, prompt, K, x)
//   speckv::autoregress(verifier, prompt, K)
// (/root/reference/proj/include/speckv/specloop.hpp:39-61, src/specloop.cpp:
// 58-92) drives real kernels unchanged.  This is the adapter SURVEY.md §8(b)
// names: the reference's oracles are stateless functions of the whole prefix;
// the engine is stateful, so the adapter compares every prefix with the
// request's committed tokens and open draft round:
//   * drafter(prefix)  prefix == prompt ++ emitted ++ open drafts
//                        -> one draft step over the COMPRESSED KV (vc_draft_step);
//   * verifier(prefix) inside a round: the first call (k = 0) runs ONE verify
//                      pass over the whole window against the FULL KV
//                      (vc_verify, x+1 predictions) and caches it; call k
//                      returns prediction k (specloop.cpp:24-35); the last
//                      call (k = x) commits the round (vc_accept_commit: the
//                      accept rule, exact KV append + rollback);
//                      with no open round: a full-KV decode step
//                      (vc_decode_step), i.e. autoregress.
// It compiles against either the reference headers or include/speckv_b200.hpp
// (both declare speckv::TokenOracle{ std::function next; }).  One adapter per
// (engine, slot); single-threaded like the reference.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "vc_api.h"

namespace speckv::gpu {

// speckv::compress(spec, shape, ratio, seed) (compressor.hpp:70-71) with the
// reference's own types, applied to a request of the GPU engine: the shape is
// the request's committed prefix, the GPU tier receives the data (vc_compress_spec:
// KIVI codes, or the kept rows of the drop tier), and the returned metadata
// is the reference's -- for the dropping kinds the exact dropped_indices the
// reference computes for `seed` (the complement of the tier's kept rows).
// Works with the reference headers or include/speckv_b200.hpp.
template <class Meta, class Spec>
Meta compress(vc_engine* e, int slot, const Spec& spec, double ratio, std::uint64_t seed = 0) {
  vc_compressor_spec cs{};
  const int kind = static_cast<int>(spec.kind);  // DropUniform 0, DropWindow 1, QuantUniform 2
  cs.kind = kind;
  cs.mode = static_cast<int>(spec.mode);
  cs.bits = spec.bits;
  cs.window = spec.window;
  cs.sink_tokens = spec.sink_tokens;
  vc_compressed_meta out{};
  if (vc_compress_spec(e, slot, &cs, ratio, seed, &out) != VC_OK)
    throw std::runtime_error(std::string("vericache: ") + vc_last_error());
  Meta meta;
  meta.bit_scheme = out.bit_scheme;
  meta.payload_bytes = out.payload_bytes;
  vc_seq_state st{};
  vc_request_state(e, slot, &st);
  // one kept list per (layer, head) of the engine's geometry
  std::vector<std::int32_t> kept;
  const bool dropping = kind != 2;
  int layers = 0, heads = 0;
  vc_engine_geometry(e, &layers, &heads);
  meta.dropped_indices.assign(layers, std::vector<std::vector<std::int64_t>>(heads));
  if (dropping) {
    for (int l = 0; l < layers; ++l)
      for (int h = 0; h < heads; ++h) {
        int n = 0;
        vc_drop_kept(e, l, h, nullptr, 0, &n);
        kept.assign(static_cast<size_t>(n), 0);
        vc_drop_kept(e, l, h, kept.data(), n, &n);
        auto& d = meta.dropped_indices[l][h];
        size_t j = 0;
        for (std::int64_t t = 0; t < st.committed; ++t) {
          if (j < kept.size() && kept[j] == t) { ++j; continue; }
          d.push_back(t);
        }
      }
  }
  return meta;
}

class SlotOracles {
 public:
  // stage >= 0: the engine keeps the full KV in the pinned host pool; each
  // verify first streams it into HBM staging slot `stage` (vc_swap_begin).
  SlotOracles(vc_engine* engine, int slot, int stage = -1)
      : st_(std::make_shared<State>(State{engine, slot, stage})) {}

  template <class Oracle>
  Oracle drafter() const {
    auto st = st_;
    return Oracle{[st](std::span<const std::int32_t> p) { return st->draft(p); }};
  }
  template <class Oracle>
  Oracle verifier() const {
    auto st = st_;
    return Oracle{[st](std::span<const std::int32_t> p) { return st->verify(p); }};
  }
  // rounds committed so far and their emitted counts (accepted drafts + 1)
  const std::vector<int>& rounds() const { return st_->rounds; }

 private:
  struct State {
    vc_engine* e;
    int slot, stage;
    long base = -1;                    // prompt length (first prefix seen)
    std::vector<std::int32_t> emitted; // committed output tokens
    std::vector<std::int32_t> drafts;  // open round
    std::vector<std::int32_t> preds;   // cached verify of the open round
    std::vector<int> rounds;

    static void ok(int rc) {
      if (rc != VC_OK) throw std::runtime_error(std::string("vericache: ") + vc_last_error());
    }
    void bind(std::span<const std::int32_t> p) {
      if (base >= 0) return;
      vc_seq_state s;
      ok(vc_request_state(e, slot, &s));
      if (p.empty() || p.back() != s.pending)
        throw std::logic_error("gpu oracle: prompt's last token is not the request's pending token");
      base = static_cast<long>(p.size());
    }
    // does p == prompt ++ emitted ++ drafts[0..k) ?
    bool is(std::span<const std::int32_t> p, size_t k) const {
      if (p.size() != base + emitted.size() + k) return false;
      for (size_t i = 0; i < emitted.size(); ++i)
        if (p[base + i] != emitted[i]) return false;
      for (size_t i = 0; i < k; ++i)
        if (p[base + emitted.size() + i] != drafts[i]) return false;
      return true;
    }
    void commit_round() {  // the caller moved on: apply the cached verify
      std::vector<std::int32_t> out(drafts.size() + 1);
      int n = 0;
      ok(vc_accept_commit(e, slot, preds.data(), stage, out.data(), &n));
      emitted.insert(emitted.end(), out.begin(), out.begin() + n);
      rounds.push_back(n);
      drafts.clear();
      preds.clear();
    }
    std::int32_t draft(std::span<const std::int32_t> p) {
      bind(p);
      if (!is(p, drafts.size())) throw std::logic_error("gpu oracle: drafter prefix is not the request's state");
      std::int32_t t = 0;
      ok(vc_draft_step(e, &slot, 1, &t));
      drafts.push_back(t);
      return t;
    }
    std::int32_t verify(std::span<const std::int32_t> p) {
      bind(p);
      if (drafts.empty()) {  // autoregress: plain full-KV decode
        if (!is(p, 0)) throw std::logic_error("gpu oracle: verifier prefix is not the request's state");
        std::int32_t t = 0;
        ok(vc_decode_step(e, &slot, 1, &t));
        emitted.push_back(t);
        return t;
      }
      const size_t k = p.size() - (base + emitted.size());
      if (k > drafts.size() || !is(p, k)) throw std::logic_error("gpu oracle: verifier prefix outside the open round");
      if (preds.empty()) {
        if (k != 0) throw std::logic_error("gpu oracle: verify must start at k = 0 (specloop.cpp:30-33)");
        if (stage >= 0) {
          std::uint64_t id = 0;
          int done = 0;
          ok(vc_swap_begin(e, slot, stage, &id));
          while (!done) ok(vc_swap_poll(e, id, &done));
        }
        preds.resize(drafts.size() + 1);
        ok(vc_verify(e, &slot, 1, stage >= 0 ? &stage : nullptr, preds.data()));
      }
      const std::int32_t t = preds[k];
      // the round's last prediction (k == x, specloop.cpp:30-33): the accept
      // decision depends only on the cached predictions, so commit now -- the
      // engine's KV, pending token and history match what run_speculative returns
      if (k == drafts.size()) commit_round();
      return t;
    }
  };
  std::shared_ptr<State> st_;
};

}  // namespace speckv::gpu
