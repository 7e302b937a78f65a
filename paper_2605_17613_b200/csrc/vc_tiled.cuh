// vc_tiled.cuh -- HBM layouts the projection GEMM streams with 1-D TMA bulk
// copies.
//
// Weights [N][K] are stored as contiguous 16 KB blocks of 128 rows x 64 k,
// block (n/128, k/64) at ((n/128) * (K/64) + k/64) * 8192 elements; inside a
// block row r holds 64 k values as eight 16-B chunks, chunk c stored at
// c ^ (r & 7) (the XOR swizzle ldmatrix reads bank-conflict free).
// Activations [Mp][K] (Mp = the step's padded row count) are stored k-tile
// major: block (k/64) is Mp rows x 128 B at (k/64) * Mp * 64 elements, same
// chunk swizzle, so rows [m0, m0+NT) of one k-tile are one contiguous copy.
#pragma once
#include <cstddef>
#include <cstdint>

namespace vc {

__host__ __device__ inline size_t wtile_idx(int n, int k, int K) {
  const size_t blk = static_cast<size_t>(n >> 7) * (K >> 6) + (k >> 6);
  const int r = n & 127;
  return blk * 8192 + static_cast<size_t>(r) * 64 + ((((k >> 3) & 7) ^ (r & 7)) << 3) + (k & 7);
}

__host__ __device__ inline size_t atile_idx(int m, int k, int Mp) {
  return (static_cast<size_t>(k >> 6) * Mp + m) * 64 + ((((k >> 3) & 7) ^ (m & 7)) << 3) + (k & 7);
}

}  // namespace vc
