// vc_gemm.h -- batch-invariant projection GEMM with fused split-K fixup and
// fused epilogues, plus the remaining model glue.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "vc_kernels.h"

namespace vc {

// Where a row's freshly computed K/V go (QKV epilogue).
struct RowDest {
  int kind;  // 0: full pool, 2: staging pool, 3: drop pool (slot, pos); 1: draft tail (pos = tail index);
             // 4: layer-chunk ring of a streamed verify (chunk of layer l = (slot + l) % ring_n); -1: none
  int slot;
  int pos;       // position inside the destination (absolute, or tail index for kind 1)
  int rope_pos;  // absolute position (RoPE)
};

enum class Epi : int {
  StoreF32 = 0,  // out_f32[m][n] = y
  Residual = 1,  // x[m][n] += y; ss_part[m][n/128] = sum over the tile of x^2
  Qkv = 2,       // bf16(y) -> RoPE on q/k heads -> qkv[m][n]; K/V heads also scattered to the pools
  Silu = 3,      // (g,u) interleaved columns -> act[m][n/2] = bf16(silu(g) * u)
};

struct GemmEpilogue {
  Epi kind = Epi::StoreF32;
  float* out_f32 = nullptr;
  float* x = nullptr;
  float* ss_part = nullptr;
  uint16_t* out_bf16 = nullptr;
  // Qkv
  const RowDest* rows = nullptr;
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  int n_q = 0, n_kv = 0, d = 0, layer = 0, layers = 0;
  KvPool full{}, stage{}, drop{};
  QuantPool draft{};
  // kind 4 rows: ring of ring_n one-layer chunks, [chunk][kv-head][cap][d]
  KvPool ring{};
  int ring_n = 1;
};

// Fused RMSNorm input (x != nullptr): the GEMM's activation tiles are
// produced in shared memory as bf16(x[m][k] * r_m * w[k]) with
// r_m = rsqrt(sum_t ss[m][t] / H + eps) -- exactly rms_apply's arithmetic, so
// the result is bit-identical to rms_apply followed by the plain GEMM.
struct GemmNormIn {
  const float* x = nullptr;     // [Mp][H] fp32 residual stream
  const float* ss = nullptr;    // [Mp][H/128] per-tile sums of squares
  const uint16_t* w = nullptr;  // [H] bf16 norm weight
  float eps = 0.f;
  int trace = -1;  // VC_GEMM_TRACE builds only: this launch's slot in the phase trace
};

struct GemmWorkspace {
  float* partial = nullptr;   // split partials, fragment order
  int* counters = nullptr;    // one per output tile, self-resetting
  size_t partial_floats = 0;
  int n_counters = 0;
};

// Split count for a weight shape; a function of (N, K) only (batch invariance).
int gemm_splits(int N, int K);
size_t gemm_partial_floats(int M, int N, int K);
int gemm_tiles(int M, int N);
// y = X[M][K] . W[N][K]^T, then the epilogue.  Xt: activations in the tiled
// layout with Mp padded rows; Wt: weights in the tiled layout (vc_tiled.cuh).
// N must be a multiple of 128, K of 64.
cudaError_t gemm(const uint16_t* Xt, int Mp, int M, int K, const uint16_t* Wt, int N,
                 const GemmEpilogue& epi, const GemmWorkspace& ws, cudaStream_t st,
                 const GemmNormIn* norm = nullptr);
// Logical row-major -> tiled layouts (weights at load time, probes).
cudaError_t retile_weight(const uint16_t* src, int N, int K, uint16_t* dst, cudaStream_t st);
cudaError_t retile_act(const uint16_t* src, int M, int K, int Mp, uint16_t* dst, cudaStream_t st);

// x[m][H] fp32 = embed[tok[m]]; xn (tiled, Mp rows) = bf16(rmsnorm(x) * w).
cudaError_t embed_norm(const int32_t* tokens, int M, int Mp, const uint16_t* embed, int H,
                       const uint16_t* norm_w, float eps, float* x, uint16_t* xn, cudaStream_t st);
// xn (tiled) = bf16(x * rsqrt(sum(ss_part[m][:]) / H + eps) * w)
cudaError_t rms_apply(const float* x, const float* ss_part, int M, int Mp, int H,
                      const uint16_t* norm_w, float eps, uint16_t* xn, cudaStream_t st);
// out[m] = argmax_n logits[m][n], ties -> smallest n.
cudaError_t argmax_rows(const float* logits, int M, int N, int32_t* out, cudaStream_t st);
// Synthetic bf16 init shared bit-for-bit with oracle/vc_oracle.c.
cudaError_t fill_normal_bf16(uint16_t* out, size_t n, uint64_t seed, uint64_t offset, float k,
                             cudaStream_t st);
cudaError_t fill_const_bf16(uint16_t* out, size_t n, uint16_t value, cudaStream_t st);
// Copy token rows [src_pos, src_pos+n) of every (layer, head) slice of a
// slot from a full-style pool into the draft tail (tail index 0..n-1).
cudaError_t tail_refill(KvPool src, int src_slot, int src_pos, int n, QuantPool dst, int dst_slot,
                        int layers, int n_kv, int d, cudaStream_t st);
// Drop tier: rows kept[slice][0..k) of every (layer, head) slice of src_slot
// -> positions 0..k of dst_slot (compacted, position order).
cudaError_t gather_kept(KvPool src, int src_slot, const int32_t* kept, int k, KvPool dst, int dst_slot,
                        int n_slices, int d, cudaStream_t st);
// Drop tier over the host tier: the rows of [0, T) NOT in the kept set
// (kept [slice][k] ascending), compacted in position order into dst rows
// [0, T - k); and the inverse -- a chunk rebuilt in position order for
// [0, n) from the landed compact rows, the drop tier's kept rows and the
// drop tier's exact rows appended since compress (rows k + p - T).
cudaError_t compact_dropped(KvPool src, int src_slot, const int32_t* kept, int k, int T, KvPool dst, int dst_slot,
                            int n_slices, int d, cudaStream_t st);
cudaError_t expand_dropped(KvPool land, int land_slot, KvPool drop, int drop_slot, const int32_t* kept, int k, int T,
                           int n, KvPool dst, int dst_slot, int n_slices, int d, cudaStream_t st);
// Lossless packing of 128-token bf16 blocks (vc_pack.cu): per channel an
// exponent base; per value a 2-bit exponent code (offsets 1-3 below the
// base, or 0 = "see the secondary stream") and the sign|mantissa byte; a
// secondary stream of 4-bit offsets (0..14, 15 = escape) for the values
// coded 0, in value order, up to kPackSecNum / kPackSecDen of a block;
// escapes for values more than 14 binades below their channel's maximum.
constexpr int kPackEscCap = 60;
constexpr int kPackSecNum = 7, kPackSecDen = 25;  // secondary capacity: 0.28 of the values
__host__ __device__ constexpr int packed_sec_cap(int d) { return 128 * d * kPackSecNum / kPackSecDen / 8 * 8; }
__host__ __device__ constexpr size_t packed_block_bytes(int d) {
  return (static_cast<size_t>(d) + 128u * d / 4 + 128u * d + 4 + packed_sec_cap(d) / 2 + 4 + 4u * kPackEscCap + 15) /
         16 * 16;
}
// src rows [src_row0 + 128 b, ...) of each slice (slice pitch in elements),
// n_valid rows from src_row0 (the last block may be partial); dst packed
// block b of slice s at dst + s * dst_slice_pitch + b * packed_block_bytes(d)
// (bytes).  *overflow = max(1 + block) over blocks with > kPackEscCap escapes
// or more secondary offsets than packed_sec_cap(d).
cudaError_t pack_blocks(const uint16_t* src, size_t src_slice_pitch, int src_row0, int n_valid, int n_blocks,
                        int n_slices, int d, uint8_t* dst, size_t dst_slice_pitch, int* overflow, cudaStream_t st);
cudaError_t unpack_blocks(const uint8_t* src, size_t src_slice_pitch, int n_blocks, int n_slices, int d, uint16_t* dst,
                          size_t dst_slice_pitch, cudaStream_t st);
// Copy token rows [src_pos, src_pos+n) of every slice to [dst_pos, dst_pos+n).
cudaError_t copy_rows(KvPool src, int src_slot, int src_pos, int n, KvPool dst, int dst_slot, int dst_pos,
                      int n_slices, int d, cudaStream_t st);

}  // namespace vc
