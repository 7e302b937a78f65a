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
// activation rows ride the UMMA N dimension, M only selects N (16..128);
// M > 128 runs the same schedule per block.  tests/test_gemm.py checks
// that a row's result is bit-identical at every M.
// Math: 5th-gen tensor cores -- one thread issues tcgen05.mma (M = 128
// weight rows, N = the step's token rows, K = 16) from the SW128 smem stages,
// fp32 accumulators in TMEM (double-buffered across a CTA's tiles), 8
// epilogue warps read them with tcgen05.ld.  (r1: the mma.sync version this
// replaces ran a 113-row verify step's projections 2.4x slower.)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vc_common.cuh"
#include "vc_gemm.h"
#include "vc_tiled.cuh"
#include "vc_umma.cuh"

namespace vc {
namespace {

constexpr int kBN = 128;   // weight rows (output features) per tile
constexpr int kBK = 64;    // k per stage (128 B per row)
constexpr int kThreads = 320;  // producer warp + MMA warp + 8 epilogue warps
constexpr int kCtasPerSm = 2;
constexpr int kSms = 148;
#ifndef VC_GEMM_GRID_PER_SM
#define VC_GEMM_GRID_PER_SM kCtasPerSm
#endif
constexpr int kP = VC_GEMM_GRID_PER_SM * kSms;  // stream-K grid upper bound (a function of nothing but the GPU)
constexpr int kEpiRows = 16;           // epilogue staging pass (tokens)
constexpr int kMaxS = 8;               // cluster split-K ranks (portable cluster size)
constexpr int kLD = kBN + 4;
#ifndef VC_FIXUP_UNROLL
#define VC_FIXUP_UNROLL 4       // contributors in flight per loop trip, NT = 16
#endif
#ifndef VC_FIXUP_UNROLL_WIDE
#define VC_FIXUP_UNROLL_WIDE 2  // contributors in flight per loop trip, NT >= 32 (4 float4 each)
#endif
constexpr int kFixUnroll = VC_FIXUP_UNROLL, kFixUnrollWide = VC_FIXUP_UNROLL_WIDE;

#ifdef VC_GEMM_TRACE
// Diagnostics build (-DVC_GEMM_TRACE): per cluster-kernel launch and CTA, the
// global timer at start, after the producer's PDL wait, when the accumulator
// is complete, after the partial exchange and at exit; dumped by
// vc_gemm_trace_dump() (tools/gemm_trace.py).  Production builds compile none of it.
constexpr int kTrLaunches = 512, kTrCtas = 256, kTrPts = 7;
__device__ unsigned long long g_gemm_trace[kTrLaunches * kTrCtas * kTrPts];
int g_gemm_trace_nk[kTrLaunches * 3];  // host: (N, K, S) per launch slot
int g_gemm_trace_next = 0;  // host: next launch slot (one counter for every instantiation)
VC_DEV void gtrace(int id, int pt) {
  if (id >= 0 && id < kTrLaunches && blockIdx.x < kTrCtas)
    g_gemm_trace[(static_cast<size_t>(id) * kTrCtas + blockIdx.x) * kTrPts + pt] = vc_globaltimer();
}
#define VC_GTRACE(pt) gtrace(nin.trace, pt)
#else
#define VC_GTRACE(pt)
#endif

template <int NT>
struct Cfg {
  static constexpr int kW = kBN * 128;
  static constexpr int kX = NT * 128;
  static constexpr int kStage = kW + kX;
  static constexpr int kStages = NT <= 32 ? 5 : (NT == 64 ? 4 : 3);
  static constexpr int kSmem = kStages * kStage + kEpiRows * kLD * 4 + 1024;  // + 1 KB alignment slack
};


// P = min(kP, T) so every CTA owns at least one k-tile (a function of N, K).
__host__ __device__ inline long grid_of(long T) { return T < kP ? T : kP; }
// CTA index owning global k-tile g under the split [q*T/P, (q+1)*T/P).
__host__ __device__ inline long owner(long g, long T) { return ((g + 1) * grid_of(T) - 1) / T; }

// Epilogue operands that do not depend on the accumulator: the residual
// stream slice a Residual thread adds to, and a Qkv thread's row destination
// and RoPE factors.  The cluster kernel's epilogue warps load them while the
// tiles stream (tools/gemm_trace.py, r2: o/down exchange -> exit 2.05 -> 1.5 us;
// the qkv epilogue stays ~2 us, its cost is not these loads).
template <Epi E>
struct EpiPre {
  bool ok = false;
};
template <>
struct EpiPre<Epi::Residual> {
  bool ok = false;
  float4 a, b;
};
template <>
struct EpiPre<Epi::Qkv> {
  bool ok = false;
  RowDest rd;
  float c[4], s[4];
};

template <Epi E>
__device__ void epilogue_load(EpiPre<E>& pre, int m, int M, int n0, int N, const GemmEpilogue& ep, int sub) {
  pre.ok = true;
  if (m >= M) return;
  if constexpr (E == Epi::Residual) {
    const float4* xp = reinterpret_cast<const float4*>(ep.x + static_cast<size_t>(m) * N + n0 + sub * 8);
    pre.a = xp[0];
    pre.b = xp[1];
  } else if constexpr (E == Epi::Qkv) {
    pre.rd = ep.rows[m];
    const int half = ep.d / 2;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int pr = sub * 4 + i, jj = pr % half;
      const int head = (n0 + (pr / half) * ep.d + jj) / ep.d;
      pre.c[i] = pre.s[i] = 0.f;
      if (head < ep.n_q + ep.n_kv) {
        pre.c[i] = ep.rope_cos[static_cast<size_t>(pre.rd.rope_pos) * half + jj];
        pre.s[i] = ep.rope_sin[static_cast<size_t>(pre.rd.rope_pos) * half + jj];
      }
    }
  }
}

// Epilogue over one staged pass of 16 tokens x 128 features (sT); `pre`
// holds the pass's operands if they were loaded early.
template <Epi E>
__device__ void epilogue_pass(const float* sT, int mbase, int M, int Mp, int n0, int N,
                              const GemmEpilogue& ep, int tid, EpiPre<E> pre = EpiPre<E>{}) {
  const int t = tid >> 4;          // row of the pass
  const int sub = tid & 15;        // 16 threads per row
  const int m = mbase + t;
  const bool live = m < M;
  const float* row = sT + t * kLD;
  if (!pre.ok) epilogue_load<E>(pre, m, M, n0, N, ep, sub);
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
      float4 a = pre.a, b = pre.b;
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
    const RowDest rd = pre.rd;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int pr = sub * 4 + i;                 // rotation pair within the tile
      const int hl = pr / half, jj = pr % half;   // head within tile, pair index
      const int fa = hl * d + jj, fb = fa + half;
      const int head = (n0 + fa) / d;
      float a = bf2f(f2bf(row[fa])), b = bf2f(f2bf(row[fb]));
      if (head < ep.n_q + ep.n_kv) {
        const float c = pre.c[i];
        const float s = pre.s[i];
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
        } else if (rd.kind == 4) {
          const size_t rs = static_cast<size_t>((rd.slot + ep.layer) % ep.ring_n) * ep.n_kv + kvh;
          dst = (is_v ? ep.ring.v : ep.ring.k) + (rs * ep.ring.cap + rd.pos) * d;
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

// Warp roles (kThreads = 320): warp 0 TMA producer, warp 1 MMA issuer (one
// thread) + TMEM owner, warps 2..9 epilogue (256 threads; TMEM lane quarter =
// warp & 3, the two warps of a quarter split the token columns).
// D[feature, token] = W[feature, :] . X[token, :] accumulates in TMEM: weight
// rows are the UMMA M (128 lanes), the step's token rows the UMMA N (NT), so a
// decode step (16 rows) and a verify window (100+ rows) run the same
// per-element arithmetic -- fixed k order inside a CTA's range, fixed
// contributor order across CTAs -- whatever the batch (batch invariance).
template <int NT, Epi E>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
gemm_umma_kernel(const uint16_t* __restrict__ Xt, int Mp, int M, int K,
                 const uint16_t* __restrict__ Wt, int N, int m0, GemmEpilogue ep, GemmWorkspace ws,
                 int max_contrib) {
  constexpr int ST = Cfg<NT>::kStages;
  constexpr int WB = Cfg<NT>::kW, XB = Cfg<NT>::kX;
  constexpr uint32_t kAccCols = 2 * NT < 32 ? 32 : 2 * NT;  // two accumulator buffers
  constexpr int kHalf = NT / 2;                             // token columns per epilogue warp
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;                                   // [ST][128 rows][128 B], SW128 K-major
  uint8_t* sX = smem + ST * WB;                         // [ST][NT rows][128 B], SW128 K-major
  float* sT = reinterpret_cast<float*>(smem + ST * (WB + XB));  // [16][kLD]
  __shared__ __align__(8) uint64_t full[ST], empty[ST], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = K / kBK;
  const int tiles = N / kBN;
  const long T = static_cast<long>(tiles) * KT;
  const long P = grid_of(T);
  const long p = blockIdx.x;
  const long beg0 = p * T / P, end = (p + 1) * T / P;

  if (tid == 0) {
    for (int s2 = 0; s2 < ST; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, kAccCols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tmem_base_sh;
  pdl_trigger();

  if (warp == 0) {  // ---- TMA producer: one lane drives the ring
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
  } else if (warp == 1) {  // ---- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kBN, NT, false);  // A = W, B = X, both K-major
      int it = 0, seg = 0;
      for (long beg = beg0; beg < end; ++seg) {
        const int k0 = static_cast<int>(beg % KT);
        const int nk = static_cast<int>(min(static_cast<long>(KT - k0), end - beg));
        beg += nk;
        const int ab = seg & 1;
        if (seg >= 2) mbar_wait(&acc_empty[ab], ((seg >> 1) - 1) & 1);
        tmem_fence_after();
        const uint32_t dacc = tbase + ab * NT;
        for (int t = 0; t < nk; ++t, ++it) {
          const int st = it % ST;
          mbar_wait(&full[st], (it / ST) & 1);
          tmem_fence_after();
          const uint32_t wa = smem_u32(sW + st * WB), xa = smem_u32(sX + st * XB);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            umma_ss(dacc, umma_sdesc_sw128(wa + kk * 32, 16, 1024), umma_sdesc_sw128(xa + kk * 32, 16, 1024), idesc,
                    t > 0 || kk > 0);
          umma_commit(&empty[st]);  // the stage is free once these MMAs have read it
        }
        umma_commit(&acc_full[ab]);
      }
    }
  } else {  // ---- epilogue: split-K fixup + fused epilogue, 256 threads
    pdl_wait();  // epilogues read/write buffers the previous kernel touches
    const int et = tid - 64;                    // 0..255
    const int quarter = warp & 3;
    const int feat = quarter * 32 + lane;       // TMEM lane = output feature within the tile
    const int tok0 = (et >= 128 ? kHalf : 0);   // this warp's token columns [tok0, tok0 + kHalf)
    const uint32_t tlane = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
    int seg = 0;
    for (long beg = beg0; beg < end; ++seg) {
      const int tile = static_cast<int>(beg / KT);
      const int k0 = static_cast<int>(beg % KT);
      const int nk = static_cast<int>(min(static_cast<long>(KT - k0), end - beg));
      const int n0 = tile * kBN;
      beg += nk;
      const int ab = seg & 1;
      mbar_wait(&acc_full[ab], (seg >> 1) & 1);
      tmem_fence_after();
      const uint32_t tacc = tlane + ab * NT + tok0;  // this warp's token columns of the accumulator
      // 8 token columns [c, c+8) of this warp's half from TMEM
      auto ld8 = [&](int c, float* v) {
        uint32_t u[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                     : "r"(tacc + c));
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(u[j]);
      };
      // ---- split-K fixup: contributors of this tile, in increasing k ----------
      const long g0 = static_cast<long>(tile) * KT;
      const long q0 = owner(g0, T), q1 = owner(g0 + KT - 1, T);
      const int n_contrib = static_cast<int>(q1 - q0 + 1);
      // partial layout per contributor: [token / 4][feature][4] floats, so a
      // warp moves 4 tokens of 32 consecutive features as one coalesced
      // 512-B float4 access
      float4* part = reinterpret_cast<float4*>(ws.partial + static_cast<size_t>(tile) * max_contrib * (NT * kBN));
      constexpr int kPart4 = NT * kBN / 4;  // float4 per contributor
      if (n_contrib > 1) {
        const int c = static_cast<int>(p - q0);
        float4* mine = part + static_cast<size_t>(c) * kPart4;
        for (int cc = 0; cc < kHalf; cc += 8) {
          float v[8];
          ld8(cc, v);
          const int t4 = (tok0 + cc) >> 2;
          mine[t4 * kBN + feat] = make_float4(v[0], v[1], v[2], v[3]);
          mine[(t4 + 1) * kBN + feat] = make_float4(v[4], v[5], v[6], v[7]);
        }
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[ab]);  // accumulator free for segment seg+2
        // the barrier orders every epilogue thread's partial stores before
        // thread 0's gpu-scope fence (cumulative), which precedes its atomic;
        // the finisher's fence after the atomic orders the other threads'
        // partial loads (after the second barrier) behind it
        named_bar(1, 256);
        if (et == 0) {
          __threadfence();
          const int prev = atomicAdd(ws.counters + tile, 1);
          s_last = prev == n_contrib - 1;
          if (s_last) {
            ws.counters[tile] = 0;  // self-reset for the next launch / graph replay
            __threadfence();
          }
        }
        named_bar(1, 256);
        if (!s_last) continue;
      }
      // ---- epilogue, 16 tokens per staged pass ---------------------------------
      if constexpr (NT >= 32) {
        // Pass pairs: the two warps of a TMEM lane quarter own token halves
        // [0, kHalf) and [kHalf, NT); pass p stages tokens 16p.. of half 0 and
        // pass p + NT/32 tokens 16p.. of half 1.  Every warp sums all
        // contributors' partials for its 16 tokens of the pair up front, so
        // both halves' loads are in flight together instead of pass after
        // pass (same contributor order per element: bit-identical).
#pragma unroll 1
        for (int pp = 0; pp < NT / 32; ++pp) {
          const int my_tok = tok0 + 16 * pp;  // this warp's 16 tokens of the pair
          float4 acc[4];
          if (m0 + my_tok >= M) {
            // rows past the batch: this warp's pass is skipped (warp-uniform)
          } else if (n_contrib > 1) {
            const float4* src = part + (my_tok >> 2) * kBN + feat;
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] = __ldcg(src + i * kBN);
#pragma unroll kFixUnrollWide
            for (int cc = 1; cc < n_contrib; ++cc) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 x = __ldcg(src + static_cast<size_t>(cc) * kPart4 + i * kBN);
                acc[i].x += x.x; acc[i].y += x.y; acc[i].z += x.z; acc[i].w += x.w;
              }
            }
          } else {
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              float v[8];
              ld8(16 * pp + g * 8, v);
              acc[2 * g] = make_float4(v[0], v[1], v[2], v[3]);
              acc[2 * g + 1] = make_float4(v[4], v[5], v[6], v[7]);
            }
          }
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int qlo = h2 * kHalf + 16 * pp;  // first token of this pass
            if (tok0 == h2 * kHalf) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                sT[(4 * i + 0) * kLD + feat] = acc[i].x;
                sT[(4 * i + 1) * kLD + feat] = acc[i].y;
                sT[(4 * i + 2) * kLD + feat] = acc[i].z;
                sT[(4 * i + 3) * kLD + feat] = acc[i].w;
              }
            }
            named_bar(1, 256);
            if (m0 + qlo < M) epilogue_pass<E>(sT, m0 + qlo, M, Mp, n0, N, ep, et);
            named_bar(1, 256);
          }
        }
      } else
      for (int q = 0; q < NT / kEpiRows; ++q) {
        const int qlo = q * kEpiRows;
        // this warp stages the pass's tokens that lie in its half, 8 at a time
        for (int c8 = 0; c8 < kEpiRows; c8 += 8) {
          const int tok = qlo + c8;
          if (tok < tok0 || tok >= tok0 + kHalf) continue;
          float v[8];
          if (n_contrib > 1) {
            // contributor order 0..n-1 per element (batch invariance); the
            // loads of consecutive contributors are independent, so the
            // unrolled loop keeps several in flight
            const float4* src = part + (tok >> 2) * kBN + feat;
            float4 a = __ldcg(src), b = __ldcg(src + kBN);
#pragma unroll kFixUnroll
            for (int cc = 1; cc < n_contrib; ++cc) {
              const float4 x = __ldcg(src + static_cast<size_t>(cc) * kPart4);
              const float4 y = __ldcg(src + static_cast<size_t>(cc) * kPart4 + kBN);
              a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
              b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
            }
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
          } else {
            ld8(tok - tok0, v);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) sT[(c8 + j) * kLD + feat] = v[j];
        }
        named_bar(1, 256);
        if (m0 + q * kEpiRows < M) epilogue_pass<E>(sT, m0 + q * kEpiRows, M, Mp, n0, N, ep, et);
        named_bar(1, 256);
      }
      if (n_contrib == 1) {
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[ab]);
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, kAccCols);
}

// Cluster split-K for weights with few output tiles (qkv, o_proj, down_proj
// at decode widths): tile t's K range is split over the S CTAs of one thread-
// block cluster (rank r streams k-tiles [r*KT/S, (r+1)*KT/S)), each CTA parks
// its fp32 accumulator in its own shared memory, and after one cluster barrier
// rank r sums tokens [r*NT/S, (r+1)*NT/S) of all S partials over DSMEM in
// rank order 0..S-1 and runs the fused epilogue on them.  Compared with the
// stream-K fixup (partials through L2, a gpu-scope fence + atomic per tile,
// then one finisher reading every partial) the reduction is spread over the
// whole cluster and never leaves the GPC.  S depends only on (N, K): batch
// invariance holds (a token's sum has the same operands in the same order at
// every M).
template <int NT, Epi E>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
gemm_cluster_kernel(const uint16_t* __restrict__ Xt, int Mp, int M, int K,
                    const uint16_t* __restrict__ Wt, int N, int m0, GemmEpilogue ep, int S, GemmNormIn nin) {
  constexpr int ST = Cfg<NT>::kStages;
  constexpr int WB = Cfg<NT>::kW, XB = Cfg<NT>::kX;
  constexpr uint32_t kAccCols = NT < 32 ? 32 : NT;
  constexpr int kHalf = NT / 2;
  static_assert(kBN * NT * 4 <= ST * (WB + XB), "the parked accumulator fits the pipeline stages");
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + ST * WB;
  float* sT = reinterpret_cast<float*>(smem + ST * (WB + XB));  // [16][kLD] epilogue staging
  float* sAcc = reinterpret_cast<float*>(smem);                 // [NT][128] parked partial (reuses the stages)
  __shared__ __align__(8) uint64_t full[ST], empty[ST], acc_full;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float sR[NT];  // fused RMSNorm: per-row scale
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = K / kBK;
  const int rank = static_cast<int>(cluster_rank());
  const int tile = blockIdx.x / S;
  const int k_lo = rank * KT / S, k_hi = (rank + 1) * KT / S;
  const int nk = k_hi - k_lo;
  const bool fused = nin.x != nullptr;  // the 8 epilogue warps write the X half of every stage
  if (tid == 0) VC_GTRACE(0);
  EpiPre<E> pre0;  // epilogue warps: operands of their first pass, loaded early
  if (tid == 0) {
    for (int s2 = 0; s2 < ST; ++s2) {
      mbar_init(&full[s2], fused ? 9 : 1);
      mbar_init(&empty[s2], 1);
    }
    mbar_init(&acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, kAccCols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tmem_base_sh;
  pdl_trigger();

  if (warp == 0) {  // ---- TMA producer
    if (lane == 0) {
      const int pre = min(ST, nk);
      const uint32_t tx = fused ? WB : WB + XB;
      const uint64_t pol = l2_policy_evict_first();  // weights are read once per step
      for (int i = 0; i < pre; ++i) {  // weights do not depend on the previous kernel
        mbar_expect_tx(&full[i], tx);
        tma_load_1d_stream(sW + i * WB, Wt + (static_cast<size_t>(tile) * KT + k_lo + i) * 8192, WB, &full[i], pol);
      }
      pdl_wait();
      VC_GTRACE(1);
      if (!fused)
        for (int i = 0; i < pre; ++i)
          tma_load_1d(sX + i * XB, Xt + (static_cast<size_t>(k_lo + i) * Mp + m0) * 64, XB, &full[i]);
      for (int i = pre; i < nk; ++i) {
        const int st = i % ST;
        mbar_wait(&empty[st], ((i / ST) - 1) & 1);
        mbar_expect_tx(&full[st], tx);
        tma_load_1d_stream(sW + st * WB, Wt + (static_cast<size_t>(tile) * KT + k_lo + i) * 8192, WB, &full[st], pol);
        if (!fused) tma_load_1d(sX + st * XB, Xt + (static_cast<size_t>(k_lo + i) * Mp + m0) * 64, XB, &full[st]);
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kBN, NT, false);
      for (int i = 0; i < nk; ++i) {
        const int st = i % ST;
        mbar_wait(&full[st], (i / ST) & 1);
        tmem_fence_after();
        const uint32_t wa = smem_u32(sW + st * WB), xa = smem_u32(sX + st * XB);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          umma_ss(tbase, umma_sdesc_sw128(wa + kk * 32, 16, 1024), umma_sdesc_sw128(xa + kk * 32, 16, 1024), idesc,
                  i > 0 || kk > 0);
        umma_commit(&empty[st]);
      }
      umma_commit(&acc_full);
    }
  } else {  // ---- park the partial: TMEM -> sAcc[token][feature]
    pdl_wait();  // the epilogue writes buffers the previous kernel may read
    const int et = tid - 64;
    // the first epilogue pass's accumulator-independent operands: in flight
    // while the tiles stream
    epilogue_load<E>(pre0, m0 + rank * NT / S + (et >> 4), M, tile * kBN, N, ep, et & 15);
    if (fused) {
      // ---- fused RMSNorm: the activation half of every stage, in the
      // swizzled layout a bulk copy of rms_apply's tiled output would land
      const int H = K;
      const int tiles = H / kBN;
      // register pipeline: the x / w loads of stage i + kPF are in flight
      // while stage i is converted and stored (a stage's loads alone are an
      // L2 round trip, which would otherwise pace every stage); the first
      // stages' loads go out before the row scales are summed
      constexpr int kCPT = NT * 8 / 256 > 0 ? NT * 8 / 256 : 1;  // 16-B chunks per thread per stage
      constexpr int kPF = kCPT >= 4 ? 1 : (kCPT == 2 ? 2 : 4);   // stages in flight
      struct Chunk {
        float4 a, b;
        uint4 w;
      };
      Chunk buf[kPF][kCPT];
      auto load = [&](int i, Chunk* c) {
        const int k0 = (k_lo + i) * kBK;
#pragma unroll
        for (int j = 0; j < kCPT; ++j) {
          const int e = et + j * 256;
          const int r = e >> 3, cc = e & 7;
          const int m = m0 + r;
          if (e < NT * 8 && m < M) {
            const float4* xp = reinterpret_cast<const float4*>(nin.x + static_cast<size_t>(m) * H + k0 + cc * 8);
            c[j].a = xp[0];
            c[j].b = xp[1];
            c[j].w = *reinterpret_cast<const uint4*>(nin.w + k0 + cc * 8);
          }
        }
      };
#pragma unroll
      for (int p = 0; p < kPF; ++p)
        if (p < nk) load(p, buf[p]);
      if (et < NT) {
        const int m = m0 + et;
        float r = 0.f;
        if (m < M) {
          const float* sp = nin.ss + static_cast<size_t>(m) * tiles;
          float sum = 0.f;
#pragma unroll 8
          for (int t = 0; t < tiles; ++t) sum += sp[t];
          r = rsqrtf(sum / H + nin.eps);
        }
        sR[et] = r;
      }
      named_bar(1, 256);
      for (int i0 = 0; i0 < nk; i0 += kPF) {
#pragma unroll
      for (int p = 0; p < kPF; ++p) {
        const int i = i0 + p;
        if (i >= nk) break;
        const int st = i % ST;
        if (i >= ST) mbar_wait(&empty[st], ((i / ST) - 1) & 1);
        uint8_t* dst = sX + st * XB;
        Chunk* c = buf[p];
#pragma unroll
        for (int j = 0; j < kCPT; ++j) {
          const int e = et + j * 256;
          if (e >= NT * 8) continue;
          const int r = e >> 3, cc = e & 7;
          uint4 o = make_uint4(0u, 0u, 0u, 0u);
          if (m0 + r < M) {
            const float rs = sR[r];
            const float xv[8] = {c[j].a.x, c[j].a.y, c[j].a.z, c[j].a.w, c[j].b.x, c[j].b.y, c[j].b.z, c[j].b.w};
            const uint32_t ww[4] = {c[j].w.x, c[j].w.y, c[j].w.z, c[j].w.w};
            uint32_t pk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float w0 = __uint_as_float(ww[q] << 16), w1 = __uint_as_float(ww[q] & 0xffff0000u);
              const uint32_t lo = f2bf(__fmul_rn(__fmul_rn(xv[2 * q], rs), w0));
              const uint32_t hi = f2bf(__fmul_rn(__fmul_rn(xv[2 * q + 1], rs), w1));
              pk[q] = lo | (hi << 16);
            }
            o = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
          *reinterpret_cast<uint4*>(dst + r * 128 + ((cc ^ (r & 7)) << 4)) = o;
        }
        if (i + kPF < nk) load(i + kPF, c);
        fence_proxy_async();  // generic-proxy stores -> the tensor core's async-proxy reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      }
      }
      // The park below overwrites the stages.  It is already ordered after
      // these stores (store -> full arrive -> MMA -> commit -> acc_full), but
      // racecheck does not follow tcgen05.commit arrivals; a named barrier
      // states the same order in a form it tracks (it costs nothing: every
      // epilogue warp waits on acc_full next anyway).
      named_bar(1, 256);
    }
    const int quarter = warp & 3;
    const int feat = quarter * 32 + lane;
    const int tok0 = et >= 128 ? kHalf : 0;
    const uint32_t tacc = tbase + (static_cast<uint32_t>(quarter * 32) << 16) + tok0;
    mbar_wait(&acc_full, 0);
    if (et == 0) VC_GTRACE(2);
    tmem_fence_after();
    for (int c = 0; c < kHalf; c += 8) {
      uint32_t u[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                   : "r"(tacc + c));
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 8; ++j) sAcc[(tok0 + c + j) * kBN + feat] = __uint_as_float(u[j]);
    }
    tmem_fence_before();
  }
  __syncwarp();
  cluster_sync();  // every rank's partial is parked
  if (tid == 64) VC_GTRACE(3);
  if (warp >= 2) {
    // ---- reduce my tokens over the cluster (rank order), then the epilogue
    const int et = tid - 64;
    const int t_lo = rank * NT / S, t_hi = (rank + 1) * NT / S;
    const int n0 = tile * kBN;
    for (int p0 = t_lo; p0 < t_hi && m0 + p0 < M; p0 += kEpiRows) {
      const int rows = min(kEpiRows, t_hi - p0);
      // rows x 32 float4 per pass; 256 threads
      for (int e = et; e < rows * (kBN / 4); e += 256) {
        const int t = e / (kBN / 4), f4 = e % (kBN / 4);
        const float* src = sAcc + (p0 + t) * kBN + f4 * 4;
        // every rank's partial in flight at once, summed in rank order
        float4 v[kMaxS];
#pragma unroll
        for (int q = 0; q < kMaxS; ++q)
          if (q < S) v[q] = ld_dsmem_f4(dsmem_addr(src, q));
        float4 acc = v[0];
#pragma unroll
        for (int q = 1; q < kMaxS; ++q)
          if (q < S) {
            acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w;
          }
        float* d = sT + t * kLD + f4 * 4;
        d[0] = acc.x; d[1] = acc.y; d[2] = acc.z; d[3] = acc.w;
      }
      named_bar(1, 256);
      if (et == 0 && p0 == t_lo) VC_GTRACE(5);
      epilogue_pass<E>(sT, m0 + p0, min(M, m0 + p0 + rows), Mp, n0, N, ep, et,
                       p0 == t_lo ? pre0 : EpiPre<E>{});
      if (et == 0 && p0 == t_lo) VC_GTRACE(6);
      named_bar(1, 256);
    }
  }
  __syncwarp();
  cluster_sync();  // no rank leaves while another may still read its partial
  if (tid == 64) VC_GTRACE(4);
  if (warp == 1) tmem_dealloc(tbase, kAccCols);
}

// Cluster size for (N, K): S = min(5, stream-K contributors per tile, k-tiles),
// S = 1 for wide weights (gate/up, LM head: one CTA per 128-feature tile, no
// split; r2: mixed step 8.18 -> 8.01 ms vs their stream-K).  Below
// VC_GEMM_CLUSTER_MIN (default 1) the stream-K kernel runs instead.  r2 sweep of a uniform S on
// the mixed x=6 step (in-graph ms): stream-K 8.62, S=3 8.30, 4 8.13, 5 8.06,
// 6 8.26, 8 8.49; S = round(148 / tiles) per shape (qkv 3, o/down 5) 8.11.
// VC_GEMM_CLUSTER=n sets the cap (1 = stream-K everywhere).
int cluster_splits(int N, int K) {
  static const int cap = [] {
    const char* v = std::getenv("VC_GEMM_CLUSTER");
    return v && std::atoi(v) > 0 ? std::atoi(v) : 5;
  }();
  static const int min_s = [] {
    const char* v = std::getenv("VC_GEMM_CLUSTER_MIN");
    return v && std::atoi(v) > 0 ? std::atoi(v) : 1;
  }();
  const int tiles = N / kBN, KT = K / kBK;
  int S = kP / tiles;
  if (S > cap) S = cap;
  if (S > kMaxS) S = kMaxS;
  if (S > KT) S = KT;
  if (S < 1) S = 1;
  return S >= min_s ? S : 0;
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
                      const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st, const GemmNormIn* norm) {
  int S = cluster_splits(N, K);
  if (norm && S < 1) S = std::max(1, std::min(kP / (N / kBN), 8));  // the fused input needs the cluster kernel
  GemmNormIn nin = norm ? *norm : GemmNormIn{};
#ifdef VC_GEMM_TRACE
  nin.trace = g_gemm_trace_next < kTrLaunches ? g_gemm_trace_next++ : -1;
  if (nin.trace >= 0) {  // host-side: a symbol copy is not allowed inside a stream capture
    g_gemm_trace_nk[3 * nin.trace] = N;
    g_gemm_trace_nk[3 * nin.trace + 1] = K;
    g_gemm_trace_nk[3 * nin.trace + 2] = S;
  }
#endif
  if (S >= 1) {
    auto kc = gemm_cluster_kernel<NT, E>;
    const int smem = Cfg<NT>::kSmem;
    cudaError_t e = cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>((N / kBN) * S);
    for (int m0 = 0; m0 < M; m0 += NT) {
      e = launch_pdl_cluster(kc, dim3(grid), dim3(kThreads), smem, st, static_cast<unsigned>(S), Xt, Mp, M, K, Wt,
                             N, m0, ep, S, nin);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  auto kern = gemm_umma_kernel<NT, E>;
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
                     const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st, const GemmNormIn* norm) {
  if (M <= 16) return launch_nt<16, E>(Xt, Mp, M, K, Wt, N, ep, ws, st, norm);
  if (M <= 32) return launch_nt<32, E>(Xt, Mp, M, K, Wt, N, ep, ws, st, norm);
  if (M <= 64) return launch_nt<64, E>(Xt, Mp, M, K, Wt, N, ep, ws, st, norm);
  return launch_nt<128, E>(Xt, Mp, M, K, Wt, N, ep, ws, st, norm);
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
                 const GemmEpilogue& ep, const GemmWorkspace& ws, cudaStream_t st, const GemmNormIn* norm) {
  if (M <= 0) return cudaSuccess;
  if (N % kBN != 0 || K % kBK != 0 || Mp < M) return cudaErrorInvalidValue;
  if (norm && (!norm->x || !norm->ss || !norm->w)) return cudaErrorInvalidValue;
  switch (ep.kind) {
    case Epi::StoreF32: return launch_e<Epi::StoreF32>(Xt, Mp, M, K, Wt, N, ep, ws, st, norm);
    case Epi::Residual: return launch_e<Epi::Residual>(Xt, Mp, M, K, Wt, N, ep, ws, st, norm);
    case Epi::Qkv: return launch_e<Epi::Qkv>(Xt, Mp, M, K, Wt, N, ep, ws, st, norm);
    case Epi::Silu: return launch_e<Epi::Silu>(Xt, Mp, M, K, Wt, N, ep, ws, st, norm);
  }
  return cudaErrorInvalidValue;
}

#ifdef VC_GEMM_TRACE
extern "C" int vc_gemm_trace_dump(const char* path) {
  std::vector<unsigned long long> t(static_cast<size_t>(kTrLaunches) * kTrCtas * kTrPts);
  std::vector<int> nk(g_gemm_trace_nk, g_gemm_trace_nk + kTrLaunches * 3);
  if (cudaMemcpyFromSymbol(t.data(), g_gemm_trace, t.size() * 8) != cudaSuccess) return 1;
  FILE* f = std::fopen(path, "wb");
  if (!f) return 2;
  std::fwrite(nk.data(), 4, nk.size(), f);
  std::fwrite(t.data(), 8, t.size(), f);
  std::fclose(f);
  return 0;
}
#endif

cudaError_t retile_weight(const uint16_t* src, int N, int K, uint16_t* dst, cudaStream_t st) {
  retile_weight_kernel<<<148 * 8, 256, 0, st>>>(src, N, K, dst);
  return cudaGetLastError();
}

cudaError_t retile_act(const uint16_t* src, int M, int K, int Mp, uint16_t* dst, cudaStream_t st) {
  retile_act_kernel<<<148 * 8, 256, 0, st>>>(src, M, K, Mp, dst);
  return cudaGetLastError();
}

}  // namespace vc
