// gpu_oracle_run.cpp -- TEST PROGRAM: the reference protocol (speckv::
// run_speculative / autoregress, specloop.cpp:58-92, as exported by
// libvericache.so through include/speckv_b200.hpp) driving the B200 engine
// through include/speckv_gpu_oracle.hpp.  Losslessness (acceptance_test.cpp
// C1, :55-79) with the real model as both oracles:
//   run_speculative(gpu drafter, gpu verifier) == autoregress(gpu full-KV decode)
// Usage: gpu_oracle_run <x> <K> <bits> <tier>    (prints "OK ..." or exits 1)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "speckv_b200.hpp"
#include "speckv_gpu_oracle.hpp"
#include "vc_api.h"

static void ck(int rc) {
  if (rc != VC_OK) {
    std::fprintf(stderr, "vc error %d: %s\n", rc, vc_last_error());
    std::exit(1);
  }
}

int main(int argc, char** argv) {
  const int x = argc > 1 ? std::atoi(argv[1]) : 8;
  const int K = argc > 2 ? std::atoi(argv[2]) : 48;
  const int bits = argc > 3 ? std::atoi(argv[3]) : 4;
  const int tier = argc > 4 ? std::atoi(argv[4]) : 0;
  const int n_ctx = 1500;
  vc_model_desc md{2048, 512, 2, 8, 2, 64, 1536, 500000.f, 1e-5f};  // engine.TINY
  vc_runtime_desc full_rt{1, n_ctx + K + 64, 1, 0, 0, 1, 1, 1};
  vc_runtime_desc spec_rt{1, n_ctx + K + 64, x, bits, tier, 1, 1, 1};
  vc_engine *ef = nullptr, *es = nullptr;
  ck(vc_engine_create(&md, &full_rt, 0, &ef));
  ck(vc_engine_create(&md, &spec_rt, 0, &es));
  for (vc_engine* e : {ef, es}) {
    ck(vc_engine_init_weights(e, 7, 0.02f));
    ck(vc_request_add_synthetic(e, 0, n_ctx, 17, 1, 4, 10.f));
  }
  // the reference signature reaches the GPU tier (speckv::gpu::compress ->
  // vc_compress_spec): quant-uniform at the engine's width, size law checked
  speckv::CompressorSpec cspec;
  cspec.kind = speckv::CompressorKind::QuantUniform;
  cspec.bits = bits;
  const auto meta = speckv::gpu::compress<speckv::CompressedKVMeta>(es, 0, cspec, 0.0, 0);
  const speckv::KvShape shape{2, 2, n_ctx, 2 * 2 * 64};
  meta.check_invariants(shape);
  if (meta.bit_scheme != bits || meta.payload_bytes != shape.full_bytes() * bits / 16) {
    std::fprintf(stderr, "compress meta mismatch\n");
    return 1;
  }

  const std::vector<speckv::Token> prompt = {17};
  speckv::gpu::SlotOracles full(ef, 0);
  speckv::gpu::SlotOracles spec(es, 0, tier ? 0 : -1);
  const speckv::TokenSeq base = speckv::autoregress(full.verifier<speckv::TokenOracle>(), prompt, K);
  auto [out, stats] = speckv::run_speculative(spec.drafter<speckv::TokenOracle>(),
                                              spec.verifier<speckv::TokenOracle>(), prompt, K, x);
  ck(vc_engine_destroy(ef));
  ck(vc_engine_destroy(es));
  if (out != base) {
    std::fprintf(stderr, "MISMATCH x=%d bits=%d tier=%d\n", x, bits, tier);
    for (int i = 0; i < K; ++i)
      if (out[i] != base[i]) {
        std::fprintf(stderr, "  first difference at %d: %d vs %d\n", i, out[i], base[i]);
        break;
      }
    return 1;
  }
  int acc = 0;
  for (int a : stats.accepted_per_round) acc += a;
  std::printf("OK x=%d bits=%d tier=%d K=%d rounds=%d emitted=%d\n", x, bits, tier, K, stats.rounds(), acc);
  return 0;
}
