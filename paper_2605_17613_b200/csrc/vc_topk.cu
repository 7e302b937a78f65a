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


// ---- SnapKV observation-window scores (Li et al., 2024) --------------------
// logits[h][r][t] = (q_{h*R+r} . k_{h,t}) * scale_log2 over the layer's
// slices; one thread per key position, the group's queries in shared memory.
__global__ void snap_logits_kernel(const uint16_t* keys, size_t pitch, int T, int d, int n_rep,
                                   const uint16_t* q, float scale_log2, float* logits) {
  extern __shared__ float sq[];  // [n_rep][d]
  const int h = blockIdx.y;
  for (int i = threadIdx.x; i < n_rep * d; i += blockDim.x) sq[i] = bf2f(q[static_cast<size_t>(h) * n_rep * d + i]);
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint4* k = reinterpret_cast<const uint4*>(keys + h * pitch + static_cast<size_t>(t) * d);
  float acc[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) acc[r] = 0.f;
  for (int c8 = 0; c8 < d / 8; ++c8) {
    const uint4 w = k[c8];
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float lo = __uint_as_float(u[j] << 16), hi = __uint_as_float(u[j] & 0xffff0000u);
      const int c = c8 * 8 + 2 * j;
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < n_rep) acc[r] = __fmaf_rn(hi, sq[r * d + c + 1], __fmaf_rn(lo, sq[r * d + c], acc[r]));
    }
  }
  for (int r = 0; r < n_rep; ++r) logits[(static_cast<size_t>(h) * n_rep + r) * T + t] = acc[r] * scale_log2;
}

// per (head, rep) row: m = max_t logit, s = sum_t 2^(logit - m)  (fixed block order)
__global__ void __launch_bounds__(1024) snap_norm_kernel(const float* logits, int T, float* ms) {
  __shared__ float red[32];
  const float* row = logits + static_cast<size_t>(blockIdx.x) * T;
  float m = -INFINITY;
  for (int t = threadIdx.x; t < T; t += blockDim.x) m = fmaxf(m, row[t]);
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  m = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int t = threadIdx.x; t < T; t += blockDim.x) sum += exp2f(row[t] - m);
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = 0.f;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) v += red[w];
    ms[blockIdx.x * 2] = m;
    ms[blockIdx.x * 2 + 1] = v;
  }
}

// attention mass of key t summed over the group's queries, max-pooled over
// [t - pool/2, t + pool/2] (SnapKV's clustering), the last `recent` positions
// forced in (score +inf)
__global__ void snap_scores_kernel(const float* logits, const float* ms, int T, int n_rep, int pool, int recent,
                                   float* scores) {
  const int h = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float best = 0.f;
  const int lo = max(0, t - pool / 2), hi = min(T - 1, t + pool / 2);
  for (int j = lo; j <= hi; ++j) {
    float a = 0.f;
    for (int r = 0; r < n_rep; ++r) {
      const int row = h * n_rep + r;
      a += exp2f(logits[static_cast<size_t>(row) * T + j] - ms[row * 2]) / ms[row * 2 + 1];
    }
    best = fmaxf(best, a);
  }
  scores[static_cast<size_t>(h) * T + t] = t >= T - recent ? INFINITY : best;
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

cudaError_t snap_scores(const uint16_t* keys, size_t pitch, int n_kv, int T, int d, int n_rep, const uint16_t* q,
                        float scale_log2, int pool, int recent, float* logits, float* ms, float* scores,
                        cudaStream_t st) {
  if (T <= 0 || n_rep > 8) return cudaErrorInvalidValue;
  snap_logits_kernel<<<dim3((T + 127) / 128, n_kv), 128, static_cast<size_t>(n_rep) * d * 4, st>>>(
      keys, pitch, T, d, n_rep, q, scale_log2, logits);
  snap_norm_kernel<<<n_kv * n_rep, 1024, 0, st>>>(logits, T, ms);
  snap_scores_kernel<<<dim3((T + 255) / 256, n_kv), 256, 0, st>>>(logits, ms, T, n_rep, pool, recent, scores);
  return cudaGetLastError();
}

}  // namespace vc
