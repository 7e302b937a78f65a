// vc_gemm.cu -- batch-invariant, stream-K weight-streaming GEMM for the model
// glue (qkv / o / gate-up / down projections, LM head):
//     y[m][n] = sum_k X[m][k] * W[n][k],   then a fused epilogue.
//
// Decode steps are weight-read bound (16 GB of bf16 weights per step against
// a few dozen activation rows), so the kernel is organised around streaming
// W exactly once at full HBM bandwidth:
//   * stream-K: a fixed grid of P = 2 CTAs per SM splits the flattened
//     (128-row weight tile x 64-wide k-tile) work list into P equal,
//     contiguous ranges -- every SM streams the same number of bytes, no
//     wave-quantisation tail;
//   * a tile whose k-range spans several CTAs is summed by its last-arriving
//     contributor in increasing-k order (self-resetting tile counters), then
//     the epilogue runs on the whole 128-feature tile: fp32 store, residual
//     add (+ per-tile sum of squares for the following RMSNorm), bf16 +
//     RoPE + KV-pool scatter for qkv, SiLU-gate for gate/up.
// Batch invariance (verify logits == decode logits bit-for-bit): the work
// split depends only on (N, K, P), never on the number of activation rows M;
// activation rows ride the MMA N dimension (8 tokens per fragment) and M only
// selects how many fragments exist.  M > 128 runs the same schedule once per
// 128-row block.
//
// Mainloop: cp.async (LDGSTS) 3-4 stage ring of 128x64 weight tiles and NTx64
// activation tiles, XOR-swizzled 16-B chunks, ldmatrix fragments, mma.sync
// bf16 with fp32 accumulate; 8 warps x 16 weight rows.
#include "vc_common.cuh"
#include "vc_gemm.h"

namespace vc {
namespace {

constexpr int kBN = 128;   // weight rows (output features) per tile
constexpr int kBK = 64;    // k per stage (128 B per row)
constexpr int kThreads = 256;
constexpr int kCtasPerSm = 2;
constexpr int kSms = 148;
constexpr int kP = kCtasPerSm * kSms;  // fixed stream-K grid

template <int NT>
struct Cfg {
  static constexpr int kStageBytes = (kBN + NT) * 128;
  static constexpr int kStages = (110 * 1024 / kStageBytes) >= 4 ? 4 : 3;
  static constexpr int kSmem = kStages * kStageBytes;
};

VC_DEV int swz8(int row, int c) { return c ^ (row & 7); }

// CTA index owning global k-tile g under the split [q*T/P, (q+1)*T/P).
// P = min(kP, T) so every CTA owns at least one k-tile (a function of N, K).
__host__ __device__ inline long grid_of(long T) { return T < kP ? T : kP; }
__host__ __device__ inline long owner(long g, long T) { return ((g + 1) * grid_of(T) - 1) / T; }

template <int NT, Epi E>
__device__ void epilogue(const float* sT, int m0, int M, int n0, int N, const GemmEpilogue& ep,
                         float* red) {
  constexpr int LD = kBN + 4;
  const int tid = threadIdx.x;
  if constexpr (E == Epi::StoreF32) {
    for (int i = tid; i < NT * kBN; i += kThreads) {
      const int t = i / kBN, j = i % kBN;
      if (m0 + t < M) ep.out_f32[static_cast<size_t>(m0 + t) * N + n0 + j] = sT[t * LD + j];
    }
  } else if constexpr (E == Epi::Residual) {
    // x += y over the tile; per-row sum of squares of the new x (fixed order)
    for (int base = 0; base < NT * kBN; base += kThreads) {
      const int i = base + tid;
      const int t = i / kBN, j = i % kBN;
      float sq = 0.f;
      if (m0 + t < M) {
        float* xp = ep.x + static_cast<size_t>(m0 + t) * N + n0 + j;
        const float v = *xp + sT[t * LD + j];
        *xp = v;
        sq = v * v;
      }
      sq = warp_sum(sq);
      if ((tid & 31) == 0) red[(base / kThreads) * 8 + tid / 32] = sq;  // 2 rows x 4 warps per pass
    }
    __syncthreads();
    for (int t = tid; t < NT; t += kThreads) {
      if (m0 + t >= M) continue;
      const int pass = t / 2, w0 = (t % 2) * 4;
      const float s = ((red[pass * 8 + w0] + red[pass * 8 + w0 + 1]) + red[pass * 8 + w0 + 2]) +
                      red[pass * 8 + w0 + 3];
      ep.ss_part[static_cast<size_t>(m0 + t) * (N / kBN) + n0 / kBN] = s;
    }
  } else if constexpr (E == Epi::Silu) {
    for (int i = tid; i < NT * (kBN / 2); i += kThreads) {
      const int t = i / (kBN / 2), p = i % (kBN / 2);
      if (m0 + t >= M) continue;
      const float g = sT[t * LD + 2 * p], u = sT[t * LD + 2 * p + 1];
      const float sg = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
      ep.out_bf16[static_cast<size_t>(m0 + t) * (N / 2) + n0 / 2 + p] = f2bf(__fmul_rn(sg, u));
    }
  } else {  // Qkv: bf16 round, RoPE on q/k heads, scatter k/v to the pools
    const int d = ep.d, half = d / 2;
    for (int i = tid; i < NT * (kBN / 2); i += kThreads) {
      const int t = i / (kBN / 2), pr = i % (kBN / 2);
      const int m = m0 + t;
      if (m >= M) continue;
      const int hl = pr / half, jj = pr % half;  // head within tile, pair index
      const int fa = hl * d + jj, fb = fa + half;  // tile-local features
      const int head = (n0 + fa) / d;
      float a = bf2f(f2bf(sT[t * LD + fa])), b = bf2f(f2bf(sT[t * LD + fb]));
      const RowDest rd = ep.rows[m];
      if (head < ep.n_q + ep.n_kv) {
        const float c = ep.rope_cos[static_cast<size_t>(rd.rope_pos) * half + jj];
        const float s = ep.rope_sin[static_cast<size_t>(rd.rope_pos) * half + jj];
        const float ra = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s));
        const float rb = __fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s));
        a = ra;
        b = rb;
      }
      const uint16_t ha = f2bf(a), hb = f2bf(b);
      uint16_t* row = ep.out_bf16 + static_cast<size_t>(m) * N + n0;
      row[fa] = ha;
      row[fb] = hb;
      if (head >= ep.n_q && rd.kind >= 0) {
        const bool is_v = head >= ep.n_q + ep.n_kv;
        const int kvh = is_v ? head - ep.n_q - ep.n_kv : head - ep.n_q;
        const size_t slice = (static_cast<size_t>(rd.slot) * ep.layers + ep.layer) * ep.n_kv + kvh;
        uint16_t* dst;
        if (rd.kind == 1) {
          dst = (is_v ? ep.draft.vtail : ep.draft.ktail) + (slice * ep.draft.tail_cap + rd.pos) * d;
        } else {
          const KvPool& p = rd.kind == 0 ? ep.full : ep.stage;
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
gemm_streamk_kernel(const uint16_t* __restrict__ X, int M, int K, const uint16_t* __restrict__ W,
                    int N, int m0, GemmEpilogue ep, GemmWorkspace ws, int max_contrib) {
  constexpr int NTF = NT / 8;
  constexpr int ST = Cfg<NT>::kStages;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sW = smem;                       // [ST][kBN][128 B]
  uint8_t* sX = smem + ST * kBN * 128;      // [ST][NT][128 B]
  __shared__ float red[NT * 4];  // residual epilogue: [row pair][8 warps]
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int KT = K / kBK;
  const int tiles = N / kBN;
  const long T = static_cast<long>(tiles) * KT;
  const long p = blockIdx.x;
  const long P = grid_of(T);
  long beg = p * T / P;
  const long end = (p + 1) * T / P;

  while (beg < end) {
    const int tile = static_cast<int>(beg / KT);
    const int k0 = static_cast<int>(beg % KT);
    const int k1 = static_cast<int>(min(static_cast<long>(KT), k0 + (end - beg)));
    const int nk = k1 - k0;
    const int n0 = tile * kBN;
    beg += nk;

    auto load = [&](int t, int stage) {
      const int kk = (k0 + t) * kBK;
      uint8_t* w = sW + stage * kBN * 128;
#pragma unroll
      for (int i = tid; i < kBN * 8; i += kThreads) {
        const int r = i >> 3, c = i & 7;
        cp_async16(w + r * 128 + swz8(r, c) * 16, W + static_cast<size_t>(n0 + r) * K + kk + c * 8);
      }
      uint8_t* x = sX + stage * NT * 128;
      for (int i = tid; i < NT * 8; i += kThreads) {
        const int r = i >> 3, c = i & 7;
        const int m = m0 + r;
        const bool ok = m < M;
        cp_async16_zfill(x + r * 128 + swz8(r, c) * 16, X + static_cast<size_t>(ok ? m : 0) * K + kk + c * 8, ok);
      }
    };
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
      if (s < nk) load(s, s);
      cp_async_commit();
    }
    float acc[NTF][4];
#pragma unroll
    for (int f = 0; f < NTF; ++f) acc[f][0] = acc[f][1] = acc[f][2] = acc[f][3] = 0.f;
    for (int t = 0; t < nk; ++t) {
      const int nt = t + ST - 1;
      if (nt < nk) load(nt, nt % ST);
      cp_async_commit();
      cp_async_wait<ST - 1>();
      __syncthreads();
      const uint8_t* w = sW + (t % ST) * kBN * 128;
      const uint8_t* x = sX + (t % ST) * NT * 128;
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
      __syncthreads();
    }
    cp_async_wait<0>();

    // ---- split-K fixup: contributors of this tile, in increasing k ----------
    const long g0 = static_cast<long>(tile) * KT;
    const long q0 = owner(g0, T), q1 = owner(g0 + KT - 1, T);
    const int n_contrib = static_cast<int>(q1 - q0 + 1);
    const int tile_id = tile;  // launches of successive row blocks are stream-ordered
    if (n_contrib > 1) {
      const int c = static_cast<int>(p - q0);
      float4* part = reinterpret_cast<float4*>(ws.partial + (static_cast<size_t>(tile_id) * max_contrib) * (NT * kBN));
      float4* mine = part + static_cast<size_t>(c) * (NT * kBN / 4) + tid * NTF;
#pragma unroll
      for (int f = 0; f < NTF; ++f) mine[f] = make_float4(acc[f][0], acc[f][1], acc[f][2], acc[f][3]);
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        const int prev = atomicAdd(ws.counters + tile_id, 1);
        s_last = prev == n_contrib - 1;
        if (s_last) ws.counters[tile_id] = 0;  // self-reset for the next launch / graph replay
      }
      __syncthreads();
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
    // ---- stage the finished tile [NT tokens][128 features] and run the epilogue
    constexpr int LD = kBN + 4;
    float* sT = reinterpret_cast<float*>(smem);
    const int fa = warp * 16 + (lane >> 2);
#pragma unroll
    for (int f = 0; f < NTF; ++f) {
      const int tk = f * 8 + 2 * (lane & 3);
      sT[tk * LD + fa] = acc[f][0];
      sT[(tk + 1) * LD + fa] = acc[f][1];
      sT[tk * LD + fa + 8] = acc[f][2];
      sT[(tk + 1) * LD + fa + 8] = acc[f][3];
    }
    __syncthreads();
    epilogue<NT, E>(sT, m0, M, n0, N, ep, red);
    __syncthreads();
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
cudaError_t launch_nt(const uint16_t* X, int M, int K, const uint16_t* W, int N,
                      const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st) {
  auto kern = gemm_streamk_kernel<NT, E>;
  const int smem = Cfg<NT>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int mc = max_contributors(N, K);
  for (int m0 = 0, blk = 0; m0 < M; m0 += NT, ++blk) {
    // one launch per 128-row block keeps the schedule independent of M
    const long T = static_cast<long>(N / kBN) * (K / kBK);
    kern<<<dim3(static_cast<unsigned>(grid_of(T)), 1), kThreads, smem, st>>>(X, M, K, W, N, m0, ep, ws, mc);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <Epi E>
cudaError_t launch_e(const uint16_t* X, int M, int K, const uint16_t* W, int N,
                     const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st) {
  if (M <= 16) return launch_nt<16, E>(X, M, K, W, N, ep, ws, st);
  if (M <= 32) return launch_nt<32, E>(X, M, K, W, N, ep, ws, st);
  if (M <= 64) return launch_nt<64, E>(X, M, K, W, N, ep, ws, st);
  return launch_nt<128, E>(X, M, K, W, N, ep, ws, st);
}

}  // namespace

int gemm_splits(int, int) { return 1; }

size_t gemm_partial_floats(int M, int N, int K) {
  const int NT = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128;
  return static_cast<size_t>(N / kBN) * max_contributors(N, K) * NT * kBN;
}

int gemm_tiles(int, int N) { return N / kBN; }

cudaError_t gemm(const uint16_t* X, int M, int K, const uint16_t* W, int N, int /*splits*/,
                 const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  if (N % kBN != 0 || K % kBK != 0) return cudaErrorInvalidValue;
  switch (ep.kind) {
    case Epi::StoreF32: return launch_e<Epi::StoreF32>(X, M, K, W, N, ep, ws, st);
    case Epi::Residual: return launch_e<Epi::Residual>(X, M, K, W, N, ep, ws, st);
    case Epi::Qkv: return launch_e<Epi::Qkv>(X, M, K, W, N, ep, ws, st);
    case Epi::Silu: return launch_e<Epi::Silu>(X, M, K, W, N, ep, ws, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace vc
