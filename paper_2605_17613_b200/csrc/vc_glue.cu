#include <algorithm>
// vc_glue.cu -- model glue outside the GEMM epilogues: embedding + RMSNorm,
// the RMSNorm apply that follows a residual epilogue, greedy argmax, the
// synthetic initialiser and the draft-tail refill.  All reductions run in a
// fixed order so a row's result never depends on the other rows of the batch.
#include "vc_common.cuh"
#include "vc_gemm.h"
#include "vc_tiled.cuh"

namespace vc {
namespace {

constexpr int kNormThreads = 512;

VC_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];  // fixed order
  __syncthreads();
  return t;
}

__global__ void embed_norm_kernel(const int32_t* tokens, int Mp, const uint16_t* embed, int H,
                                  const uint16_t* norm_w, float eps, float* x, uint16_t* xn) {
  __shared__ float red[32];
  const int m = blockIdx.x;
  const uint16_t* e = embed + static_cast<size_t>(tokens[m]) * H;
  float* xr = x + static_cast<size_t>(m) * H;
  float ss = 0.f;
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    const float v = bf2f(e[i]);
    xr[i] = v;
    ss += v * v;
  }
  ss = block_sum(ss, red);
  const float r = rsqrtf(ss / H + eps);
  for (int i = threadIdx.x; i < H; i += blockDim.x)
    xn[atile_idx(m, i, Mp)] = f2bf(__fmul_rn(__fmul_rn(xr[i], r), bf2f(norm_w[i])));
}

// grid (M, H / 1024): every CTA recomputes the row's r from the per-tile
// partial sums (fixed order) and normalises its 1024-wide chunk.
__global__ void rms_apply_kernel(const float* x, const float* ss_part, int H, int Mp,
                                 const uint16_t* w, float eps, uint16_t* xn) {
  pdl_trigger();
  pdl_wait();
  __shared__ float r_s;
  const int m = blockIdx.x;
  const int tiles = H / 128;
  if (threadIdx.x == 0) {
    const float* sp = ss_part + static_cast<size_t>(m) * tiles;
    float s = 0.f;
    for (int t = 0; t < tiles; ++t) s += sp[t];
    r_s = rsqrtf(s / H + eps);
  }
  __syncthreads();
  const float r = r_s;
  const int base = blockIdx.y * 1024;
  for (int i = base + threadIdx.x; i < min(H, base + 1024); i += blockDim.x)
    xn[atile_idx(m, i, Mp)] = f2bf(__fmul_rn(__fmul_rn(x[static_cast<size_t>(m) * H + i], r), bf2f(w[i])));
}

__global__ void argmax_kernel(const float* logits, int N, int32_t* out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sv[32];
  __shared__ int si[32];
  const float* row = logits + static_cast<size_t>(blockIdx.x) * N;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  if ((N & 3) == 0) {  // float4 loads: 4x fewer instructions, more bytes in flight
    const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll 4
    for (int j = threadIdx.x; j < N / 4; j += blockDim.x) {
      const float4 v = r4[j];  // ascending indices per thread: the first max is kept
      if (v.x > best) { best = v.x; bi = 4 * j; }
      if (v.y > best) { best = v.y; bi = 4 * j + 1; }
      if (v.z > best) { best = v.z; bi = 4 * j + 2; }
      if (v.w > best) { best = v.w; bi = 4 * j + 3; }
    }
  } else {
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const float v = row[i];
      if (v > best) { best = v; bi = i; }  // ascending i per thread: first max kept
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // ties -> smaller index (specloop.cpp:260)
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[warp] = best; si[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = sv[0];
    int idx = si[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (sv[w] > b || (sv[w] == b && si[w] < idx)) { b = sv[w]; idx = si[w]; }
    // std::max_element semantics (specloop.cpp:260: `largest < *it` moves on):
    // a NaN at index 0 is never replaced, later NaNs never win, and a row with
    // nothing above -inf keeps index 0
    if (idx == 0x7fffffff || isnan(row[0])) idx = 0;
    out[blockIdx.x] = idx;
  }
}

VC_DEV uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void fill_normal_kernel(uint16_t* out, size_t n, uint64_t seed, uint64_t offset, float k) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = splitmix(seed ^ splitmix(i + offset));
    const int s = static_cast<int>(h & 0xffff) + static_cast<int>((h >> 16) & 0xffff) +
                  static_cast<int>((h >> 32) & 0xffff) + static_cast<int>((h >> 48) & 0xffff);
    out[i] = f2bf(__fmul_rn(static_cast<float>(s - 131070), k));
  }
}

__global__ void fill_const_kernel(uint16_t* out, size_t n, uint16_t v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = v;
}

__global__ void tail_refill_kernel(KvPool src, int src_slot, int src_pos, int n, QuantPool dst,
                                   int dst_slot, int layers, int n_kv, int d) {
  const int sl = blockIdx.x;  // layer * n_kv + head
  const size_t s_slice = static_cast<size_t>(src_slot) * layers * n_kv + sl;
  const size_t d_slice = static_cast<size_t>(dst_slot) * layers * n_kv + sl;
  const uint4* sk = reinterpret_cast<const uint4*>(src.k + (s_slice * src.cap + src_pos) * d);
  const uint4* sv = reinterpret_cast<const uint4*>(src.v + (s_slice * src.cap + src_pos) * d);
  uint4* dk = reinterpret_cast<uint4*>(dst.ktail + d_slice * dst.tail_cap * d);
  uint4* dv = reinterpret_cast<uint4*>(dst.vtail + d_slice * dst.tail_cap * d);
  const int words = n * d / 8;
  for (int i = threadIdx.x; i < words; i += blockDim.x) {
    dk[i] = sk[i];
    dv[i] = sv[i];
  }
}

// one CTA per (slice, 64-row block); 16-byte copies
__global__ void gather_kept_kernel(KvPool src, int src_slot, const int32_t* kept, int k, KvPool dst, int dst_slot,
                                   int n_slices, int d) {
  const int sl = blockIdx.y;
  const size_t s_slice = static_cast<size_t>(src_slot) * n_slices + sl;
  const size_t d_slice = static_cast<size_t>(dst_slot) * n_slices + sl;
  const int vec = d / 8;  // uint4 per row
  const int r0 = blockIdx.x * 64;
  const int32_t* kp = kept + static_cast<size_t>(sl) * k;
  for (int i = threadIdx.x; i < 64 * vec; i += blockDim.x) {
    const int r = r0 + i / vec, c = i % vec;
    if (r >= k) break;
    const size_t so = (s_slice * src.cap + kp[r]) * d, dof = (d_slice * dst.cap + r) * d;
    reinterpret_cast<uint4*>(dst.k + dof)[c] = reinterpret_cast<const uint4*>(src.k + so)[c];
    reinterpret_cast<uint4*>(dst.v + dof)[c] = reinterpret_cast<const uint4*>(src.v + so)[c];
  }
}

// rank of position p among the slice's kept positions (sorted ascending):
// the number of kept positions < p
VC_DEV int kept_rank(const int32_t* kp, int k, int p) {
  int lo = 0, hi = k;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (kp[mid] < p) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// dropped rows of [0, T) (the complement of the kept set) compacted in
// position order: dropped position p -> row p - rank(p)
__global__ void compact_dropped_kernel(KvPool src, int src_slot, const int32_t* kept, int k, int T, KvPool dst,
                                       int dst_slot, int n_slices, int d) {
  const int sl = blockIdx.y;
  const size_t s_slice = static_cast<size_t>(src_slot) * n_slices + sl;
  const size_t d_slice = static_cast<size_t>(dst_slot) * n_slices + sl;
  const int32_t* kp = kept + static_cast<size_t>(sl) * k;
  const int vec = d / 8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T * vec; i += gridDim.x * blockDim.x) {
    const int p = i / vec, c = i % vec;
    const int r = kept_rank(kp, k, p);
    if (r < k && kp[r] == p) continue;  // kept: lives in the drop tier
    const size_t so = (s_slice * src.cap + p) * d, dof = (d_slice * dst.cap + (p - r)) * d;
    reinterpret_cast<uint4*>(dst.k + dof)[c] = reinterpret_cast<const uint4*>(src.k + so)[c];
    reinterpret_cast<uint4*>(dst.v + dof)[c] = reinterpret_cast<const uint4*>(src.v + so)[c];
  }
}

// a full-KV chunk rebuilt in position order for p in [0, n): p < T dropped ->
// landed row p - rank(p); p < T kept -> drop-tier row rank(p); p >= T (exact
// rows accepted since compress) -> drop-tier row k + p - T
__global__ void expand_dropped_kernel(KvPool land, int land_slot, KvPool drop, int drop_slot, const int32_t* kept,
                                      int k, int T, int n, KvPool dst, int dst_slot, int n_slices, int d) {
  const int sl = blockIdx.y;
  const size_t l_slice = static_cast<size_t>(land_slot) * n_slices + sl;
  const size_t r_slice = static_cast<size_t>(drop_slot) * n_slices + sl;
  const size_t d_slice = static_cast<size_t>(dst_slot) * n_slices + sl;
  const int32_t* kp = kept + static_cast<size_t>(sl) * k;
  const int vec = d / 8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * vec; i += gridDim.x * blockDim.x) {
    const int p = i / vec, c = i % vec;
    const uint16_t *sk, *sv;
    if (p >= T) {
      const size_t so = (r_slice * drop.cap + k + (p - T)) * d;
      sk = drop.k + so;
      sv = drop.v + so;
    } else {
      const int r = kept_rank(kp, k, p);
      if (r < k && kp[r] == p) {
        const size_t so = (r_slice * drop.cap + r) * d;
        sk = drop.k + so;
        sv = drop.v + so;
      } else {
        const size_t so = (l_slice * land.cap + (p - r)) * d;
        sk = land.k + so;
        sv = land.v + so;
      }
    }
    const size_t dof = (d_slice * dst.cap + p) * d;
    reinterpret_cast<uint4*>(dst.k + dof)[c] = reinterpret_cast<const uint4*>(sk)[c];
    reinterpret_cast<uint4*>(dst.v + dof)[c] = reinterpret_cast<const uint4*>(sv)[c];
  }
}

__global__ void copy_rows_kernel(KvPool src, int src_slot, int src_pos, int n, KvPool dst, int dst_slot,
                                 int dst_pos, int n_slices, int d) {
  const int sl = blockIdx.x;
  const size_t s_slice = static_cast<size_t>(src_slot) * n_slices + sl;
  const size_t d_slice = static_cast<size_t>(dst_slot) * n_slices + sl;
  const uint4* sk = reinterpret_cast<const uint4*>(src.k + (s_slice * src.cap + src_pos) * d);
  const uint4* sv = reinterpret_cast<const uint4*>(src.v + (s_slice * src.cap + src_pos) * d);
  uint4* dk = reinterpret_cast<uint4*>(dst.k + (d_slice * dst.cap + dst_pos) * d);
  uint4* dv = reinterpret_cast<uint4*>(dst.v + (d_slice * dst.cap + dst_pos) * d);
  const int words = n * d / 8;
  for (int i = threadIdx.x; i < words; i += blockDim.x) {
    dk[i] = sk[i];
    dv[i] = sv[i];
  }
}

int grid_for(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 148 * 16 ? (b == 0 ? 1 : b) : 148 * 16);
}

}  // namespace

cudaError_t embed_norm(const int32_t* tokens, int M, int Mp, const uint16_t* embed, int H,
                       const uint16_t* norm_w, float eps, float* x, uint16_t* xn, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  embed_norm_kernel<<<M, kNormThreads, 0, st>>>(tokens, Mp, embed, H, norm_w, eps, x, xn);
  return cudaGetLastError();
}

cudaError_t rms_apply(const float* x, const float* ss_part, int M, int Mp, int H,
                      const uint16_t* norm_w, float eps, uint16_t* xn, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  return launch_pdl(rms_apply_kernel, dim3(M, (H + 1023) / 1024), dim3(256), 0, st, x, ss_part, H, Mp, norm_w,
                    eps, xn);
}

cudaError_t argmax_rows(const float* logits, int M, int N, int32_t* out, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  return launch_pdl(argmax_kernel, dim3(M), dim3(1024), 0, st, logits, N, out);
}

cudaError_t fill_normal_bf16(uint16_t* out, size_t n, uint64_t seed, uint64_t offset, float k,
                             cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_normal_kernel<<<grid_for(n, 256), 256, 0, st>>>(out, n, seed, offset, k);
  return cudaGetLastError();
}

cudaError_t fill_const_bf16(uint16_t* out, size_t n, uint16_t value, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fill_const_kernel<<<grid_for(n, 256), 256, 0, st>>>(out, n, value);
  return cudaGetLastError();
}

cudaError_t tail_refill(KvPool src, int src_slot, int src_pos, int n, QuantPool dst, int dst_slot,
                        int layers, int n_kv, int d, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  tail_refill_kernel<<<layers * n_kv, 256, 0, st>>>(src, src_slot, src_pos, n, dst, dst_slot, layers, n_kv, d);
  return cudaGetLastError();
}

cudaError_t gather_kept(KvPool src, int src_slot, const int32_t* kept, int k, KvPool dst, int dst_slot,
                        int n_slices, int d, cudaStream_t st) {
  if (k <= 0 || n_slices <= 0) return cudaSuccess;
  gather_kept_kernel<<<dim3((k + 63) / 64, n_slices), 256, 0, st>>>(src, src_slot, kept, k, dst, dst_slot, n_slices, d);
  return cudaGetLastError();
}

cudaError_t compact_dropped(KvPool src, int src_slot, const int32_t* kept, int k, int T, KvPool dst, int dst_slot,
                            int n_slices, int d, cudaStream_t st) {
  if (T <= 0 || n_slices <= 0) return cudaSuccess;
  const size_t work = static_cast<size_t>(T) * (d / 8);
  compact_dropped_kernel<<<dim3(static_cast<unsigned>(std::min<size_t>((work + 255) / 256, 1024)), n_slices), 256, 0,
                           st>>>(src, src_slot, kept, k, T, dst, dst_slot, n_slices, d);
  return cudaGetLastError();
}

cudaError_t expand_dropped(KvPool land, int land_slot, KvPool drop, int drop_slot, const int32_t* kept, int k, int T,
                           int n, KvPool dst, int dst_slot, int n_slices, int d, cudaStream_t st) {
  if (n <= 0 || n_slices <= 0) return cudaSuccess;
  const size_t work = static_cast<size_t>(n) * (d / 8);
  expand_dropped_kernel<<<dim3(static_cast<unsigned>(std::min<size_t>((work + 255) / 256, 1024)), n_slices), 256, 0,
                          st>>>(land, land_slot, drop, drop_slot, kept, k, T, n, dst, dst_slot, n_slices, d);
  return cudaGetLastError();
}

cudaError_t copy_rows(KvPool src, int src_slot, int src_pos, int n, KvPool dst, int dst_slot, int dst_pos,
                      int n_slices, int d, cudaStream_t st) {
  if (n <= 0 || n_slices <= 0) return cudaSuccess;
  copy_rows_kernel<<<n_slices, 256, 0, st>>>(src, src_slot, src_pos, n, dst, dst_slot, dst_pos, n_slices, d);
  return cudaGetLastError();
}

}  // namespace vc
