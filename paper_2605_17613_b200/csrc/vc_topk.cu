// vc_topk.cu -- the drop-topk compressor's data plane: per-(layer, head)
// token scores and exact top-k retention (ties -> lower position), emitting
// the kept positions ascending.  Integer radix select over order-preserving
// float keys, then a position-ordered compaction, so the kept set is
// bit-identical with oracle/vc_oracle.c:vco_topk_kept for identical scores.
// The shape law (equal kept count per head within a layer,
// /root/reference/proj/src/compressor.cpp:83-86) holds by construction:
// every row keeps exactly k.
#include "vc_common.cuh"
#include "vc_topk.h"

namespace vc {
namespace {

constexpr int kThreads = 1024;

VC_DEV uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void key_scores_kernel(const uint16_t* keys, int rows, int T, int d, size_t pitch,
                                  const float* w, float* scores) {
  const size_t total = static_cast<size_t>(rows) * T;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint16_t* k = keys + (i / T) * pitch + (i % T) * d;
    float s = 0.f;
    for (int c = 0; c < d; ++c) s = __fmaf_rn(fabsf(bf2f(k[c])), w[c], s);  // channel order
    scores[i] = s;
  }
}

__global__ void __launch_bounds__(kThreads) topk_kernel(const float* scores, int T, int k,
                                                        int32_t* kept) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_prefix, s_mask, s_need;
  __shared__ uint32_t warp_tot[kThreads / 32];
  const float* row = scores + static_cast<size_t>(blockIdx.x) * T;
  int32_t* out = kept + static_cast<size_t>(blockIdx.x) * k;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_mask = 0;
    s_need = static_cast<uint32_t>(k);  // rank (1-based) of the threshold among the largest
  }
  __syncthreads();
  // 4 passes of 8 bits, most significant first: find the k-th largest key
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += kThreads) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix, mask = s_mask;
    for (int t = threadIdx.x; t < T; t += kThreads) {
      const uint32_t key = fkey(row[t]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t need = s_need, acc = 0;
      int b = 255;
      for (; b > 0; --b) {
        if (acc + hist[b] >= need) break;
        acc += hist[b];
      }
      s_need = need - acc;
      s_prefix = prefix | (static_cast<uint32_t>(b) << shift);
      s_mask = mask | (0xffu << shift);
    }
    __syncthreads();
  }
  const uint32_t thr = s_prefix;          // key of the k-th largest score
  const uint32_t take_eq = s_need;        // how many keys == thr to keep (lowest positions)
  // compaction in position order: each thread owns a contiguous segment
  const int seg = (T + kThreads - 1) / kThreads;
  const int t0 = threadIdx.x * seg, t1 = min(T, t0 + seg);
  uint32_t n_gt = 0, n_eq = 0;
  for (int t = t0; t < t1; ++t) {
    const uint32_t key = fkey(row[t]);
    n_gt += key > thr;
    n_eq += key == thr;
  }
  // exclusive block scans of n_eq then of selected counts
  auto block_scan = [&](uint32_t v) -> uint32_t {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = lane < kThreads / 32 ? warp_tot[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < kThreads / 32) warp_tot[lane] = w;
    }
    __syncthreads();
    const uint32_t base = warp > 0 ? warp_tot[warp - 1] : 0u;
    const uint32_t r = base + x - v;
    __syncthreads();
    return r;
  };
  const uint32_t eq_before = block_scan(n_eq);
  const uint32_t eq_take_here =
      eq_before >= take_eq ? 0u : min(n_eq, take_eq - eq_before);
  const uint32_t sel_before = block_scan(n_gt + eq_take_here);
  uint32_t w = sel_before, eq_seen = 0;
  for (int t = t0; t < t1; ++t) {
    const uint32_t key = fkey(row[t]);
    bool take = key > thr;
    if (key == thr) {
      take = eq_seen < eq_take_here;
      ++eq_seen;
    }
    if (take) out[w++] = t;
  }
}

}  // namespace

cudaError_t key_scores(const uint16_t* keys, int rows, int T, int d, size_t row_pitch, const float* w,
                       float* scores, cudaStream_t st) {
  const size_t n = static_cast<size_t>(rows) * T;
  if (n == 0) return cudaSuccess;
  const int grid = static_cast<int>(n / 256 + 1 < 148 * 16 ? n / 256 + 1 : 148 * 16);
  key_scores_kernel<<<grid, 256, 0, st>>>(keys, rows, T, d, row_pitch, w, scores);
  return cudaGetLastError();
}

cudaError_t topk_select(const float* scores, int rows, int T, int k, int32_t* kept,
                        cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (k < 1 || k > T) return cudaErrorInvalidValue;
  topk_kernel<<<rows, kThreads, 0, st>>>(scores, T, k, kept);
  return cudaGetLastError();
}

}  // namespace vc
