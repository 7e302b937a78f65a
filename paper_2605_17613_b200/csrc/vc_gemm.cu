// vc_gemm.cu -- batch-invariant weight-streaming GEMM for the model glue
// (qkv / o / gate-up / down projections and the LM head):
//     ws[split][m][n] = sum_{k in split} X[m][k] * W[n][k]
// followed by fused epilogues that sum the splits in a FIXED order.
//
// Decode and verify differ only in the number of activation rows M (B for a
// draft/decode step, B + x+1 for a step that carries a verify).  For the
// verify logits to equal full-KV decode logits bit-for-bit, the reduction
// order of every output element must not depend on M: the K split and the
// k-tile/k-step order are functions of (N, K) only, activation rows ride the
// MMA N dimension (8 tokens per fragment) and never change the arithmetic of
// another row.  Weight rows are the MMA M dimension (16 per fragment), so a
// 16-row decode batch wastes nothing.
//
// Pipeline: 4-stage cp.async ring of 128x64 weight tiles and NTx64 activation
// tiles (XOR-swizzled 16-B chunks, ldmatrix fragments), mma.sync bf16, fp32
// accumulate.  8 warps x 16 weight rows per CTA.
#include "vc_common.cuh"
#include "vc_gemm.h"

namespace vc {
namespace {

constexpr int kBN = 128;   // weight rows per CTA
constexpr int kBK = 64;    // k per stage (128 B per row)
constexpr int kStages = 4;
constexpr int kThreads = 256;

VC_DEV int swz8(int row, int c) { return c ^ (row & 7); }

template <int NT>
__global__ void __launch_bounds__(kThreads) gemm_kernel(const uint16_t* __restrict__ X, int M, int K,
                                                        const uint16_t* __restrict__ W, int N,
                                                        int k_per_split, float* __restrict__ ws) {
  constexpr int NTF = NT / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sW = smem;                               // [stages][kBN][128 B]
  uint8_t* sX = smem + kStages * kBN * 128;          // [stages][NT][128 B]
  const int n0 = blockIdx.x * kBN;
  const int split = blockIdx.y;
  const int m0 = blockIdx.z * NT;
  const int kbeg = split * k_per_split;
  const int n_tiles = k_per_split / kBK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto load = [&](int t, int stage) {
    const int k0 = kbeg + t * kBK;
    uint8_t* w = sW + stage * kBN * 128;
#pragma unroll
    for (int i = threadIdx.x; i < kBN * 8; i += kThreads) {
      const int r = i >> 3, c = i & 7;
      const int n = n0 + r;
      const bool ok = n < N;
      cp_async16_zfill(w + r * 128 + swz8(r, c) * 16, W + static_cast<size_t>(ok ? n : 0) * K + k0 + c * 8, ok);
    }
    uint8_t* x = sX + stage * NT * 128;
    for (int i = threadIdx.x; i < NT * 8; i += kThreads) {
      const int r = i >> 3, c = i & 7;
      const int m = m0 + r;
      const bool ok = m < M;
      cp_async16_zfill(x + r * 128 + swz8(r, c) * 16, X + static_cast<size_t>(ok ? m : 0) * K + k0 + c * 8, ok);
    }
  };

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < n_tiles) load(s, s);
    cp_async_commit();
  }

  float acc[NTF][4];
#pragma unroll
  for (int f = 0; f < NTF; ++f) acc[f][0] = acc[f][1] = acc[f][2] = acc[f][3] = 0.f;

  for (int t = 0; t < n_tiles; ++t) {
    const int nt = t + kStages - 1;
    if (nt < n_tiles) load(nt, nt % kStages);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncthreads();
    const uint8_t* w = sW + (t % kStages) * kBN * 128;
    const uint8_t* x = sX + (t % kStages) * NT * 128;
#pragma unroll
    for (int ks = 0; ks < kBK / 16; ++ks) {
      uint32_t a[4];
      {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = ks * 2 + (lane >> 4);
        ldmatrix_x4(a[0], a[1], a[2], a[3], w + r * 128 + swz8(r, c) * 16);
      }
#pragma unroll
      for (int f = 0; f < NTF; f += 2) {
        if (f + 1 < NTF) {
          // matrices: (tok f*8.., k lo), (tok f*8.., k hi), (tok (f+1)*8.., k lo), (.., k hi)
          const int r = f * 8 + (lane & 7) + (lane >> 4) * 8;
          const int c = ks * 2 + ((lane >> 3) & 1);
          uint32_t b[4];
          ldmatrix_x4(b[0], b[1], b[2], b[3], x + r * 128 + swz8(r, c) * 16);
          mma_bf16(acc[f], a[0], a[1], a[2], a[3], b[0], b[1]);
          mma_bf16(acc[f + 1], a[0], a[1], a[2], a[3], b[2], b[3]);
        } else {
          const int r = f * 8 + (lane & 7);
          const int c = ks * 2 + ((lane >> 3) & 1);
          uint32_t b[2];
          ldmatrix_x2(b[0], b[1], x + r * 128 + swz8(r, c) * 16);
          mma_bf16(acc[f], a[0], a[1], a[2], a[3], b[0], b[1]);
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  // C fragment: rows = weight rows (features), cols = tokens
  float* out = ws + static_cast<size_t>(split) * M * N;
  const int fa = n0 + warp * 16 + (lane >> 2);
#pragma unroll
  for (int f = 0; f < NTF; ++f) {
    const int tk = m0 + f * 8 + 2 * (lane & 3);
    if (fa < N) {
      if (tk < M) out[static_cast<size_t>(tk) * N + fa] = acc[f][0];
      if (tk + 1 < M) out[static_cast<size_t>(tk + 1) * N + fa] = acc[f][1];
    }
    if (fa + 8 < N) {
      if (tk < M) out[static_cast<size_t>(tk) * N + fa + 8] = acc[f][2];
      if (tk + 1 < M) out[static_cast<size_t>(tk + 1) * N + fa + 8] = acc[f][3];
    }
  }
}

template <int NT>
cudaError_t launch_gemm(const uint16_t* X, int M, int K, const uint16_t* W, int N, int splits,
                        float* ws, cudaStream_t st) {
  const size_t smem = kStages * (kBN + NT) * 128;
  auto kern = gemm_kernel<NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((N + kBN - 1) / kBN, splits, (M + NT - 1) / NT);
  kern<<<grid, kThreads, smem, st>>>(X, M, K, W, N, K / splits, ws);
  return cudaGetLastError();
}

}  // namespace

int gemm_splits(int N, int K) {
  // Fixed per weight shape (never per M): enough CTAs for ~2 waves on 148 SMs.
  const int ctas_n = (N + kBN - 1) / kBN;
  int s = 1;
  while (ctas_n * s < 2 * 148 && (K / (s * 2)) % kBK == 0 && K / (s * 2) >= 512) s *= 2;
  return s;
}

cudaError_t gemm_partial(const uint16_t* X, int M, int K, const uint16_t* W, int N, int splits,
                         float* ws, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  if (K % (splits * kBK) != 0) return cudaErrorInvalidValue;
  if (M <= 16) return launch_gemm<16>(X, M, K, W, N, splits, ws, st);
  if (M <= 32) return launch_gemm<32>(X, M, K, W, N, splits, ws, st);
  if (M <= 64) return launch_gemm<64>(X, M, K, W, N, splits, ws, st);
  return launch_gemm<128>(X, M, K, W, N, splits, ws, st);
}

}  // namespace vc
