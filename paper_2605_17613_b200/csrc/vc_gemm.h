// vc_gemm.h -- batch-invariant projection GEMM + fused epilogues + model glue.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "vc_kernels.h"

namespace vc {

// Split count for a weight shape; a function of (N, K) only (batch invariance).
int gemm_splits(int N, int K);
// ws[split][M][N] fp32 partial sums of X[M][K] . W[N][K]^T.
cudaError_t gemm_partial(const uint16_t* X, int M, int K, const uint16_t* W, int N, int splits,
                         float* ws, cudaStream_t st);

// Where a row's freshly computed K/V go (kv_store).
struct RowDest {
  int kind;  // 0: full pool, 2: staging pool (slot, pos); 1: draft tail (pos = tail index); -1: none
  int slot;
  int pos;   // absolute position (also the RoPE position for kind 0); see rope_pos
  int rope_pos;
};

// x[m][H] fp32 = embed[tok[m]]; xn = bf16(rmsnorm(x) * w).
cudaError_t embed_norm(const int32_t* tokens, int M, const uint16_t* embed, int H,
                       const uint16_t* norm_w, float eps, float* x, uint16_t* xn, cudaStream_t st);
// qkv[m][:] = bf16(rope(bf16(sum_s ws[s][m][:]))) for q and k heads; v plain.
cudaError_t qkv_epilogue(const float* ws, int splits, int M, int n_q, int n_kv, int d,
                         const RowDest* rows, const float* rope_cos, const float* rope_sin,
                         uint16_t* qkv, cudaStream_t st);
// Scatter every row's K/V heads into the pools.
cudaError_t kv_store(const uint16_t* qkv, int M, int n_q, int n_kv, int d, int layer, int layers,
                     const RowDest* rows, KvPool full, KvPool stage, QuantPool draft,
                     cudaStream_t st);
// x += sum_s ws; xn = bf16(rmsnorm(x) * w)   (w == nullptr: no xn)
cudaError_t residual_norm(const float* ws, int splits, int M, int H, float* x,
                          const uint16_t* norm_w, float eps, uint16_t* xn, cudaStream_t st);
// act[m][j] = bf16(silu(g) * u), (g,u) = interleaved columns (2j, 2j+1).
cudaError_t silu_epilogue(const float* ws, int splits, int M, int F, uint16_t* act,
                          cudaStream_t st);
// logits[m][n] = sum_s ws
cudaError_t sum_epilogue(const float* ws, int splits, int M, int N, float* out, cudaStream_t st);
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

}  // namespace vc
