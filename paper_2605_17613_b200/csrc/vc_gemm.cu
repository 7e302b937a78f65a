// vc_gemm.cu -- batch-invariant, stream-K, TMA-fed weight-streaming GEMM for
// the model glue (qkv / o / gate-up / down projections, LM head):
//     y[m][n] = sum_k X[m][k] * W[n][k],   then a fused epilogue.
//
// Decode steps are weight-read bound (16 GB of bf16 weights per step against
// a few dozen activation rows), so the kernel is organised around streaming
// W exactly once at full HBM bandwidth:
//   * weights and activations live in HBM pre-tiled (vc_tiled.cuh): one
//     128x64 weight tile is one contiguous, pre-swizzled 16 KB block and the
//     NTx64 activation tile one contiguous block, so a dedicated producer warp
//     moves each pipeline stage with two 1-D TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx) -- no per-thread address math,
//     no __syncthreads in the main loop (full/empty mbarrier ring);
//   * stream-K: a fixed grid of P = min(2 x 148, #k-tiles) CTAs splits the
//     flattened (weight tile, k-tile) list into P equal contiguous ranges --
//     every SM streams the same bytes, no wave-quantisation tail;
//   * a tile whose k-range spans several CTAs is summed by its last-arriving
//     contributor in increasing-k order (self-resetting counters), then the
//     epilogue runs on the 128-feature tile: fp32 store, residual add (+ per
//     tile sum of squares for the next RMSNorm), bf16 + RoPE + KV-pool scatter
//     for qkv, SiLU-gate for gate/up (written in the tiled activation layout).
// Batch invariance (verify logits == decode logits bit-for-bit): the work
// split depends only on (N, K), never on the number of activation rows M;
// activation rows ride the MMA N dimension (8 tokens per fragment), M only
// selects how many fragments exist; M > 128 runs the same schedule per block.
// Math: ldmatrix fragments from the swizzled stages, mma.sync bf16, fp32
// accumulate, 8 consumer warps x 16 weight rows.
#include "vc_common.cuh"
#include "vc_gemm.h"
#include "vc_tiled.cuh"

namespace vc {
namespace {

constexpr int kBN = 128;   // weight rows (output features) per tile
constexpr int kBK = 64;    // k per stage (128 B per row)
constexpr int kConsumers = 256;
constexpr int kThreads = kConsumers + 32;  // + producer warp
constexpr int kCtasPerSm = 2;
constexpr int kSms = 148;
constexpr int kP = kCtasPerSm * kSms;  // stream-K grid upper bound
constexpr int kEpiRows = 16;           // epilogue staging pass (tokens)
constexpr int kLD = kBN + 4;

template <int NT>
struct Cfg {
  static constexpr int kW = kBN * 128;
  static constexpr int kX = NT * 128;
  static constexpr int kStage = kW + kX;
  static constexpr int kStages = NT <= 32 ? 5 : (NT == 64 ? 4 : 3);
  static constexpr int kSmem = kStages * kStage + kEpiRows * kLD * 4;
};

VC_DEV int swz8(int row, int c) { return c ^ (row & 7); }

// P = min(kP, T) so every CTA owns at least one k-tile (a function of N, K).
__host__ __device__ inline long grid_of(long T) { return T < kP ? T : kP; }
// CTA index owning global k-tile g under the split [q*T/P, (q+1)*T/P).
__host__ __device__ inline long owner(long g, long T) { return ((g + 1) * grid_of(T) - 1) / T; }

// Epilogue over one staged pass of 16 tokens x 128 features (sT).
template <Epi E>
__device__ void epilogue_pass(const float* sT, int mbase, int M, int Mp, int n0, int N,
                              const GemmEpilogue& ep) {
  const int tid = threadIdx.x;
  const int t = tid >> 4;          // row of the pass
  const int sub = tid & 15;        // 16 threads per row
  const int m = mbase + t;
  const bool live = m < M;
  const float* row = sT + t * kLD;
  if constexpr (E == Epi::StoreF32) {
    if (live) {
      float4* dst = reinterpret_cast<float4*>(ep.out_f32 + static_cast<size_t>(m) * N + n0 + sub * 8);
      dst[0] = make_float4(row[sub * 8 + 0], row[sub * 8 + 1], row[sub * 8 + 2], row[sub * 8 + 3]);
      dst[1] = make_float4(row[sub * 8 + 4], row[sub * 8 + 5], row[sub * 8 + 6], row[sub * 8 + 7]);
    }
  } else if constexpr (E == Epi::Residual) {
    float sq = 0.f;
    if (live) {
      float4* xp = reinterpret_cast<float4*>(ep.x + static_cast<size_t>(m) * N + n0 + sub * 8);
      float4 a = xp[0], b = xp[1];
      a.x += row[sub * 8 + 0]; a.y += row[sub * 8 + 1]; a.z += row[sub * 8 + 2]; a.w += row[sub * 8 + 3];
      b.x += row[sub * 8 + 4]; b.y += row[sub * 8 + 5]; b.z += row[sub * 8 + 6]; b.w += row[sub * 8 + 7];
      xp[0] = a;
      xp[1] = b;
      sq = ((a.x * a.x + a.y * a.y) + (a.z * a.z + a.w * a.w)) + ((b.x * b.x + b.y * b.y) + (b.z * b.z + b.w * b.w));
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);  // fixed tree
    if (live && sub == 0) ep.ss_part[static_cast<size_t>(m) * (N / kBN) + n0 / kBN] = sq;
  } else if constexpr (E == Epi::Silu) {
    if (live) {
      uint32_t packed[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int p = sub * 4 + i;
        const float g = row[2 * p], u = row[2 * p + 1];
        const float sg = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
        const uint32_t h = f2bf(__fmul_rn(sg, u));
        if (i & 1) packed[i >> 1] |= h << 16; else packed[i >> 1] = h;
      }
      const int k = n0 / 2 + sub * 4;  // 4 consecutive k inside one 16-B chunk
      *reinterpret_cast<uint2*>(ep.out_bf16 + atile_idx(m, k, Mp)) = make_uint2(packed[0], packed[1]);
    }
  } else {  // Qkv: bf16 round, RoPE on q/k heads, scatter k/v to the pools
    if (!live) return;
    const int d = ep.d, half = d / 2;
    const RowDest rd = ep.rows[m];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int pr = sub * 4 + i;                 // rotation pair within the tile
      const int hl = pr / half, jj = pr % half;   // head within tile, pair index
      const int fa = hl * d + jj, fb = fa + half;
      const int head = (n0 + fa) / d;
      float a = bf2f(f2bf(row[fa])), b = bf2f(f2bf(row[fb]));
      if (head < ep.n_q + ep.n_kv) {
        const float c = ep.rope_cos[static_cast<size_t>(rd.rope_pos) * half + jj];
        const float s = ep.rope_sin[static_cast<size_t>(rd.rope_pos) * half + jj];
        const float ra = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s));
        const float rb = __fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s));
        a = ra;
        b = rb;
      }
      const uint16_t ha = f2bf(a), hb = f2bf(b);
      uint16_t* orow = ep.out_bf16 + static_cast<size_t>(m) * N + n0;
      orow[fa] = ha;
      orow[fb] = hb;
      if (head >= ep.n_q && rd.kind >= 0) {
        const bool is_v = head >= ep.n_q + ep.n_kv;
        const int kvh = is_v ? head - ep.n_q - ep.n_kv : head - ep.n_q;
        const size_t slice = (static_cast<size_t>(rd.slot) * ep.layers + ep.layer) * ep.n_kv + kvh;
        uint16_t* dst;
        if (rd.kind == 1) {
          dst = (is_v ? ep.draft.vtail : ep.draft.ktail) + (slice * ep.draft.tail_cap + rd.pos) * d;
        } else {
          const KvPool& p = rd.kind == 0 ? ep.full : (rd.kind == 2 ? ep.stage : ep.drop);
          dst = (is_v ? p.v : p.k) + (slice * p.cap + rd.pos) * d;
        }
        dst[jj] = ha;
        dst[jj + half] = hb;
      }
    }
  }
}

template <int NT, Epi E>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
gemm_tma_kernel(const uint16_t* __restrict__ Xt, int Mp, int M, int K,
                const uint16_t* __restrict__ Wt, int N, int m0, GemmEpilogue ep, GemmWorkspace ws,
                int max_contrib) {
  constexpr int NTF = NT / 8;
  constexpr int ST = Cfg<NT>::kStages;
  constexpr int WB = Cfg<NT>::kW, XB = Cfg<NT>::kX;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sW = smem;                                   // [ST][128 rows][128 B]
  uint8_t* sX = smem + ST * WB;                         // [ST][NT rows][128 B]
  float* sT = reinterpret_cast<float*>(smem + ST * (WB + XB));  // [16][kLD]
  __shared__ __align__(8) uint64_t full[ST], empty[ST];
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = K / kBK;
  const int tiles = N / kBN;
  const long T = static_cast<long>(tiles) * KT;
  const long P = grid_of(T);
  const long p = blockIdx.x;
  const long beg0 = p * T / P, end = (p + 1) * T / P;

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  pdl_trigger();
  if (warp == kConsumers / 32) {  // ---- producer warp: one lane drives the TMA ring
    if (lane == 0) {
      // PDL prologue: the first stages' weight tiles do not depend on the
      // previous kernel -- stream them while it drains, then wait for it
      // before the activation tiles (its output)
      const int pre = static_cast<int>(min(static_cast<long>(ST), end - beg0));
      for (int i = 0; i < pre; ++i) {
        const long g = beg0 + i;
        mbar_expect_tx(&full[i], WB + XB);
        tma_load_1d(sW + i * WB, Wt + (static_cast<size_t>(g / KT) * KT + g % KT) * 8192, WB, &full[i]);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) {
        const int kt = static_cast<int>((beg0 + i) % KT);
        tma_load_1d(sX + i * XB, Xt + (static_cast<size_t>(kt) * Mp + m0) * 64, XB, &full[i]);
      }
      int it = pre;
      for (long g = beg0 + pre; g < end; ++g, ++it) {
        const int st = it % ST;
        if (it >= ST) mbar_wait(&empty[st], ((it / ST) - 1) & 1);
        mbar_expect_tx(&full[st], WB + XB);
        const int tile = static_cast<int>(g / KT), kt = static_cast<int>(g % KT);
        tma_load_1d(sW + st * WB, Wt + (static_cast<size_t>(tile) * KT + kt) * 8192, WB, &full[st]);
        tma_load_1d(sX + st * XB, Xt + (static_cast<size_t>(kt) * Mp + m0) * 64, XB, &full[st]);
      }
    }
    return;
  }

  // ---- consumer warps ------------------------------------------------------
  pdl_wait();  // epilogues read/write buffers the previous kernel touches
  int it = 0;
  long beg = beg0;
  while (beg < end) {
    const int tile = static_cast<int>(beg / KT);
    const int k0 = static_cast<int>(beg % KT);
    const int nk = static_cast<int>(min(static_cast<long>(KT - k0), end - beg));
    const int n0 = tile * kBN;
    beg += nk;
    float acc[NTF][4];
#pragma unroll
    for (int f = 0; f < NTF; ++f) acc[f][0] = acc[f][1] = acc[f][2] = acc[f][3] = 0.f;
    for (int t = 0; t < nk; ++t, ++it) {
      const int st = it % ST;
      mbar_wait(&full[st], (it / ST) & 1);
      const uint8_t* w = sW + st * WB;
      const uint8_t* x = sX + st * XB;
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
          const int r = f * 8 + (lane & 7) + (lane >> 4) * 8;
          const int c = ks * 2 + ((lane >> 3) & 1);
          uint32_t b[4];
          ldmatrix_x4(b[0], b[1], b[2], b[3], x + r * 128 + swz8(r, c) * 16);
          mma_bf16(acc[f], a[0], a[1], a[2], a[3], b[0], b[1]);
          mma_bf16(acc[f + 1], a[0], a[1], a[2], a[3], b[2], b[3]);
        }
      }
      // order this warp's generic-proxy reads of the stage before the producer's
      // next async-proxy (TMA) write into it -- without it the refill can race
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
    }

    // ---- split-K fixup: contributors of this tile, in increasing k ----------
    const long g0 = static_cast<long>(tile) * KT;
    const long q0 = owner(g0, T), q1 = owner(g0 + KT - 1, T);
    const int n_contrib = static_cast<int>(q1 - q0 + 1);
    if (n_contrib > 1) {
      const int c = static_cast<int>(p - q0);
      float4* part = reinterpret_cast<float4*>(ws.partial + (static_cast<size_t>(tile) * max_contrib) * (NT * kBN));
      float4* mine = part + static_cast<size_t>(c) * (NT * kBN / 4) + tid * NTF;
#pragma unroll
      for (int f = 0; f < NTF; ++f) mine[f] = make_float4(acc[f][0], acc[f][1], acc[f][2], acc[f][3]);
      __threadfence();
      named_bar(1, kConsumers);
      if (tid == 0) {
        const int prev = atomicAdd(ws.counters + tile, 1);
        s_last = prev == n_contrib - 1;
        if (s_last) ws.counters[tile] = 0;  // self-reset for the next launch / graph replay
      }
      named_bar(1, kConsumers);
      if (!s_last) continue;
      __threadfence();
#pragma unroll
      for (int f = 0; f < NTF; ++f) {
        float4 s = __ldcg(part + tid * NTF + f);
        for (int cc = 1; cc < n_contrib; ++cc) {
          const float4 v = __ldcg(part + static_cast<size_t>(cc) * (NT * kBN / 4) + tid * NTF + f);
          s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
        acc[f][0] = s.x; acc[f][1] = s.y; acc[f][2] = s.z; acc[f][3] = s.w;
      }
    }
    // ---- epilogue, 16 tokens per staged pass ---------------------------------
    const int fa = warp * 16 + (lane >> 2);
#pragma unroll
    for (int q = 0; q < NT / kEpiRows; ++q) {
#pragma unroll
      for (int ff = 0; ff < 2; ++ff) {
        const int f = 2 * q + ff;
        const int tk = ff * 8 + 2 * (lane & 3);
        sT[tk * kLD + fa] = acc[f][0];
        sT[(tk + 1) * kLD + fa] = acc[f][1];
        sT[tk * kLD + fa + 8] = acc[f][2];
        sT[(tk + 1) * kLD + fa + 8] = acc[f][3];
      }
      named_bar(1, kConsumers);
      if (m0 + q * kEpiRows < M) epilogue_pass<E>(sT, m0 + q * kEpiRows, M, Mp, n0, N, ep);
      named_bar(1, kConsumers);
    }
  }
}

int max_contributors(int N, int K) {
  const long KT = K / kBK, tiles = N / kBN, T = tiles * KT;
  int mx = 1;
  for (long t = 0; t < tiles; ++t) {
    const long n = owner(t * KT + KT - 1, T) - owner(t * KT, T) + 1;
    mx = static_cast<int>(n > mx ? n : mx);
  }
  return mx;
}

template <int NT, Epi E>
cudaError_t launch_nt(const uint16_t* Xt, int Mp, int M, int K, const uint16_t* Wt, int N,
                      const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st) {
  auto kern = gemm_tma_kernel<NT, E>;
  const int smem = Cfg<NT>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int mc = max_contributors(N, K);
  const long T = static_cast<long>(N / kBN) * (K / kBK);
  for (int m0 = 0; m0 < M; m0 += NT) {
    // one launch per NT-row block keeps the schedule independent of M
    e = launch_pdl(kern, dim3(static_cast<unsigned>(grid_of(T))), dim3(kThreads), smem, st, Xt, Mp, M, K, Wt, N,
                   m0, ep, ws, mc);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <Epi E>
cudaError_t launch_e(const uint16_t* Xt, int Mp, int M, int K, const uint16_t* Wt, int N,
                     const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st) {
  if (M <= 16) return launch_nt<16, E>(Xt, Mp, M, K, Wt, N, ep, ws, st);
  if (M <= 32) return launch_nt<32, E>(Xt, Mp, M, K, Wt, N, ep, ws, st);
  if (M <= 64) return launch_nt<64, E>(Xt, Mp, M, K, Wt, N, ep, ws, st);
  return launch_nt<128, E>(Xt, Mp, M, K, Wt, N, ep, ws, st);
}

__global__ void retile_weight_kernel(const uint16_t* src, int N, int K, uint16_t* dst) {
  const size_t total = static_cast<size_t>(N) * K;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i / K), k = static_cast<int>(i % K);
    dst[wtile_idx(n, k, K)] = src[i];
  }
}

__global__ void retile_act_kernel(const uint16_t* src, int M, int K, int Mp, uint16_t* dst) {
  const size_t total = static_cast<size_t>(M) * K;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / K), k = static_cast<int>(i % K);
    dst[atile_idx(m, k, Mp)] = src[i];
  }
}

}  // namespace

int gemm_splits(int, int) { return 1; }

size_t gemm_partial_floats(int M, int N, int K) {
  const int NT = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128;
  return static_cast<size_t>(N / kBN) * max_contributors(N, K) * NT * kBN;
}

int gemm_tiles(int, int N) { return N / kBN; }

cudaError_t gemm(const uint16_t* Xt, int Mp, int M, int K, const uint16_t* Wt, int N,
                 const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  if (N % kBN != 0 || K % kBK != 0 || Mp < M) return cudaErrorInvalidValue;
  switch (ep.kind) {
    case Epi::StoreF32: return launch_e<Epi::StoreF32>(Xt, Mp, M, K, Wt, N, ep, ws, st);
    case Epi::Residual: return launch_e<Epi::Residual>(Xt, Mp, M, K, Wt, N, ep, ws, st);
    case Epi::Qkv: return launch_e<Epi::Qkv>(Xt, Mp, M, K, Wt, N, ep, ws, st);
    case Epi::Silu: return launch_e<Epi::Silu>(Xt, Mp, M, K, Wt, N, ep, ws, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t retile_weight(const uint16_t* src, int N, int K, uint16_t* dst, cudaStream_t st) {
  retile_weight_kernel<<<148 * 8, 256, 0, st>>>(src, N, K, dst);
  return cudaGetLastError();
}

cudaError_t retile_act(const uint16_t* src, int M, int K, int Mp, uint16_t* dst, cudaStream_t st) {
  retile_act_kernel<<<148 * 8, 256, 0, st>>>(src, M, K, Mp, dst);
  return cudaGetLastError();
}

}  // namespace vc
