// vc_glue.cu -- model glue around the projections: embedding + RMSNorm,
// split-sum epilogues (RoPE, residual + RMSNorm, SiLU-gate), KV scatter into
// the pools, greedy argmax, synthetic init.  All reductions run in a fixed
// order so a row's result never depends on the other rows of the batch.
#include "vc_common.cuh"
#include "vc_gemm.h"

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

__global__ void embed_norm_kernel(const int32_t* tokens, const uint16_t* embed, int H,
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
    xn[static_cast<size_t>(m) * H + i] = f2bf(__fmul_rn(__fmul_rn(xr[i], r), bf2f(norm_w[i])));
}

__global__ void residual_norm_kernel(const float* ws, int splits, int M, int H, float* x,
                                     const uint16_t* norm_w, float eps, uint16_t* xn) {
  __shared__ float red[32];
  const int m = blockIdx.x;
  float* xr = x + static_cast<size_t>(m) * H;
  float ss = 0.f;
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += ws[(static_cast<size_t>(s) * M + m) * H + i];
    const float v = xr[i] + acc;
    xr[i] = v;
    ss += v * v;
  }
  if (norm_w == nullptr) return;
  ss = block_sum(ss, red);
  const float r = rsqrtf(ss / H + eps);
  for (int i = threadIdx.x; i < H; i += blockDim.x)
    xn[static_cast<size_t>(m) * H + i] = f2bf(__fmul_rn(__fmul_rn(xr[i], r), bf2f(norm_w[i])));
}

// one CTA per row; thread i handles rotation pairs of one head
__global__ void qkv_epilogue_kernel(const float* ws, int splits, int M, int n_q, int n_kv, int d,
                                    const RowDest* rows, const float* rope_cos,
                                    const float* rope_sin, uint16_t* qkv) {
  const int m = blockIdx.x;
  const int N = (n_q + 2 * n_kv) * d;
  const int half = d / 2;
  const int pos = rows[m].rope_pos;
  uint16_t* out = qkv + static_cast<size_t>(m) * N;
  auto load = [&](int n) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += ws[(static_cast<size_t>(s) * M + m) * N + n];
    return bf2f(f2bf(acc));  // projections round to bf16 before RoPE
  };
  const int n_rot = (n_q + n_kv) * half;  // rotation pairs in q and k heads
  for (int i = threadIdx.x; i < n_rot; i += blockDim.x) {
    const int head = i / half, j = i % half;
    const int a = head * d + j, b = a + half;
    const float x1 = load(a), x2 = load(b);
    const float c = rope_cos[static_cast<size_t>(pos) * half + j];
    const float s = rope_sin[static_cast<size_t>(pos) * half + j];
    out[a] = f2bf(__fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, s)));
    out[b] = f2bf(__fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, s)));
  }
  for (int n = (n_q + n_kv) * d + threadIdx.x; n < N; n += blockDim.x) out[n] = f2bf(load(n));
}

__global__ void kv_store_kernel(const uint16_t* qkv, int n_q, int n_kv, int d, int layer,
                                int layers, const RowDest* rows, KvPool full, KvPool stage,
                                QuantPool draft) {
  const int m = blockIdx.x, h = blockIdx.y;
  const RowDest rd = rows[m];
  if (rd.kind < 0) return;
  const int N = (n_q + 2 * n_kv) * d;
  const uint16_t* k = qkv + static_cast<size_t>(m) * N + static_cast<size_t>(n_q + h) * d;
  const uint16_t* v = qkv + static_cast<size_t>(m) * N + static_cast<size_t>(n_q + n_kv + h) * d;
  const size_t slice = (static_cast<size_t>(rd.slot) * layers + layer) * n_kv + h;
  uint16_t *dk, *dv;
  if (rd.kind == 0 || rd.kind == 2) {
    const KvPool& p = rd.kind == 0 ? full : stage;
    dk = p.k + (slice * p.cap + rd.pos) * d;
    dv = p.v + (slice * p.cap + rd.pos) * d;
  } else {
    dk = draft.ktail + (slice * draft.tail_cap + rd.pos) * d;
    dv = draft.vtail + (slice * draft.tail_cap + rd.pos) * d;
  }
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    reinterpret_cast<uint4*>(dk)[i] = reinterpret_cast<const uint4*>(k)[i];
    reinterpret_cast<uint4*>(dv)[i] = reinterpret_cast<const uint4*>(v)[i];
  }
}

__global__ void silu_kernel(const float* ws, int splits, int M, int F, uint16_t* act) {
  const size_t total = static_cast<size_t>(M) * F;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t m = i / F, j = i % F;
    float g = 0.f, u = 0.f;
    for (int s = 0; s < splits; ++s) {
      const float2 gu = *reinterpret_cast<const float2*>(ws + (static_cast<size_t>(s) * M + m) * 2 * F + 2 * j);
      g += gu.x;
      u += gu.y;
    }
    const float sg = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
    act[i] = f2bf(__fmul_rn(sg, u));
  }
}

__global__ void sum_kernel(const float* ws, int splits, size_t total, float* out) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += ws[static_cast<size_t>(s) * total + i];
    out[i] = acc;
  }
}

__global__ void argmax_kernel(const float* logits, int N, int32_t* out) {
  __shared__ float sv[32];
  __shared__ int si[32];
  const float* row = logits + static_cast<size_t>(blockIdx.x) * N;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float v = row[i];
    if (v > best) { best = v; bi = i; }  // ascending i per thread: first max kept
  }
  // warp then block reduction; ties -> smaller index
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
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

int grid_for(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 148 * 16 ? (b == 0 ? 1 : b) : 148 * 16);
}

}  // namespace

cudaError_t embed_norm(const int32_t* tokens, int M, const uint16_t* embed, int H,
                       const uint16_t* norm_w, float eps, float* x, uint16_t* xn, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  embed_norm_kernel<<<M, kNormThreads, 0, st>>>(tokens, embed, H, norm_w, eps, x, xn);
  return cudaGetLastError();
}

cudaError_t qkv_epilogue(const float* ws, int splits, int M, int n_q, int n_kv, int d,
                         const RowDest* rows, const float* rope_cos, const float* rope_sin,
                         uint16_t* qkv, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  qkv_epilogue_kernel<<<M, 512, 0, st>>>(ws, splits, M, n_q, n_kv, d, rows, rope_cos, rope_sin, qkv);
  return cudaGetLastError();
}

cudaError_t kv_store(const uint16_t* qkv, int M, int n_q, int n_kv, int d, int layer, int layers,
                     const RowDest* rows, KvPool full, KvPool stage, QuantPool draft,
                     cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  kv_store_kernel<<<dim3(M, n_kv), 32, 0, st>>>(qkv, n_q, n_kv, d, layer, layers, rows, full, stage, draft);
  return cudaGetLastError();
}

cudaError_t residual_norm(const float* ws, int splits, int M, int H, float* x,
                          const uint16_t* norm_w, float eps, uint16_t* xn, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  residual_norm_kernel<<<M, kNormThreads, 0, st>>>(ws, splits, M, H, x, norm_w, eps, xn);
  return cudaGetLastError();
}

cudaError_t silu_epilogue(const float* ws, int splits, int M, int F, uint16_t* act,
                          cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  const size_t n = static_cast<size_t>(M) * F;
  silu_kernel<<<grid_for(n, 256), 256, 0, st>>>(ws, splits, M, F, act);
  return cudaGetLastError();
}

cudaError_t sum_epilogue(const float* ws, int splits, int M, int N, float* out, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  const size_t n = static_cast<size_t>(M) * N;
  sum_kernel<<<grid_for(n, 256), 256, 0, st>>>(ws, splits, n, out);
  return cudaGetLastError();
}

cudaError_t argmax_rows(const float* logits, int M, int N, int32_t* out, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  argmax_kernel<<<M, 1024, 0, st>>>(logits, N, out);
  return cudaGetLastError();
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

}  // namespace vc
