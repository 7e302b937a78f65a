// vc_tp.h -- head-sharded tensor parallelism (BASELINE.json configs[4]:
// TP=8 with NCCL over NVLink).  Each rank holds n_q/T query heads, n_kv/T KV
// heads (its own KV pools and compressed tiers) and ffn/T of the MLP; the
// o_proj and down_proj outputs are partial sums over the rank's heads / FFN
// slice and are combined across ranks once per projection.
//
// Losslessness needs batch invariance across ranks too: a row's combined
// value must not depend on how many rows the step carries.  A ring/tree
// all-reduce picks its chunking (hence each element's reduction order) by
// message size, so the combine is an ALL-GATHER of the fp32 partials (a pure
// copy) followed by a fixed rank-order sum fused with the residual add
// (tp_residual) -- identical arithmetic for a 16-row decode step and a
// 100-row verify window, and bit-identical on every rank.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <memory>

namespace vc {

struct Collective {
  virtual ~Collective() = default;
  // dst[r * count + i] = (rank r's src)[i] for every rank r, ordered on `st`
  virtual void all_gather(const float* src, float* dst, size_t count, cudaStream_t st) = 0;
  // false for the in-process loopback (host barriers cannot be graph-captured)
  virtual bool graph_capturable() const = 0;
};

// In-process ranks on one device, one host thread per rank (tests, and a
// single-GPU functional check of the sharded model).
class LoopbackGroup;
std::shared_ptr<LoopbackGroup> make_loopback_group(int size);
std::unique_ptr<Collective> make_loopback(const std::shared_ptr<LoopbackGroup>& group, int rank);

// NCCL over NVLink/NVSwitch (libnccl.so.2 resolved at run time); `unique_id`
// is the 128-byte ncclUniqueId rank 0 created and shared.
bool nccl_available();
bool nccl_unique_id(void* out128);
std::unique_ptr<Collective> make_nccl(const void* unique_id, int rank, int size);

// x[m][n] += sum_{r=0..tp-1} gathered[r][m][n]  (rank order), then
// ss_part[m][n/128] = sum over the 128-feature tile of x^2 (fixed tree).
cudaError_t tp_residual(float* x, const float* gathered, int tp, int M, int H, float* ss_part, cudaStream_t st);

}  // namespace vc
