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
}  // namespace vc
