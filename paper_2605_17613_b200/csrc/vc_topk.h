// vc_topk.h -- drop-topk compressor kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vc {
// scores[r][t] = sum_c |k_rtc| w_c (fixed channel order); row r's keys start
// at keys + r * row_pitch (elements), token-major [T][d].
cudaError_t key_scores(const uint16_t* keys, int rows, int T, int d, size_t row_pitch, const float* w,
                       float* scores, cudaStream_t st);
cudaError_t topk_select(const float* scores, int rows, int T, int k, int32_t* kept,
                        cudaStream_t st);
// SnapKV observation-window scores of one layer (Li et al., 2024): for kv head
// h, scores[h][t] = max over |j - t| <= pool/2 of sum_r softmax_t(q_{hR+r} . k_{h,t}
// / sqrt(d))[j], the last `recent` positions +inf (always kept).  keys: the
// layer's first slice, heads `pitch` elements apart; q: [n_kv * n_rep][d] bf16
// (the observation query, post-RoPE); logits [n_kv*n_rep][T] and ms
// [n_kv*n_rep][2] are scratch.
cudaError_t snap_scores(const uint16_t* keys, size_t pitch, int n_kv, int T, int d, int n_rep, const uint16_t* q,
                        float scale_log2, int pool, int recent, float* logits, float* ms, float* scores,
                        cudaStream_t st);
}  // namespace vc
