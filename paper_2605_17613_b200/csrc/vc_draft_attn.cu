// vc_draft_attn.cu -- draft decode attention over the KIVI-compressed cache.
//
// One query token per drafting sequence, n_rep query heads per kv head (GQA).
// HBM-bound: every code byte is read exactly once.  Each warp runs its own
// two-stage TMA pipeline: one lane issues 1-D bulk copies
// (cp.async.bulk ... mbarrier::complete_tx) of the next 64-token unit --
// K codes, V codes, V scale/zero, and per group the K scale/zero -- into
// shared memory while the warp computes on the previous unit, so the memory
// system sees ~9 KB in flight per warp without holding registers for it.
// The math runs on legacy mma.sync tensor-core tiles fed from LDS:
//   S^T[tok, head] = Kcodes[tok, ch] . q'^T[ch, head],  q' = q * kscale (per group)
//   O^T[ch, head]  = Vcodes^T[ch, tok] . P'^T[tok, head], P' = P * vscale (per token)
// Dequantisation is folded algebraically into q' / P' and two per-head
// constants (zero points, and the 1024 bias of the lop3 int->fp16 trick), so
// the inner loop is lop3 + mma only.  Codes are stored in mma A-fragment
// order (vc_quant.cu), the P' B-fragments come from the S C-fragments through
// movmatrix.trans, and the online softmax runs on warp shuffles.
// Split-K over 1024-token chunks + one bf16-tail CTA; attention_combine
// merges the partials (LSE) in chunk order.
//
// The reference models this step as a pure HBM read of the compressed cache
// (/root/reference/proj/src/scheduler.cpp:452-457, sim.cpp:254-256).
#include "vc_common.cuh"
#include "vc_kernels.h"

namespace vc {
namespace {

constexpr int kG = VC_QGROUP;
constexpr int kCG = VC_DRAFT_CG;
constexpr int kWarps = 4;
constexpr int kUnit = VC_QUNIT;  // tokens per pipeline unit = one unit record
constexpr float kTau = 8.0f;      // lazy rescale: running max may lag the true max by 2^8

template <int D, int BITS>
struct Geo {
  static constexpr int KS = D / 16;                    // channel k-steps / tiles
  static constexpr int W = (BITS == 4) ? KS : KS / 2;  // u32 per lane per 16-token tile
  static constexpr int CH = W < 4 ? W : 4;
  static constexpr int UMT = kUnit / 16;               // 16-token tiles per unit
  static constexpr int UW = UMT * W * 32;              // u32 of K (or V) codes per unit
  static constexpr int UREC = static_cast<int>(quant_unit_words(D, BITS));
  static constexpr int GREC = static_cast<int>(quant_record_words(D, BITS));
  static_assert(UW == static_cast<int>(quant_unit_code_words(D, BITS)), "unit geometry");
  // stage (u32) mirrors the group record: [ksz D][K codes UW][V codes UW][vsz kUnit];
  // the ksz slot is filled by the first unit of each group only
  static constexpr int OFF_KSZ = 0;
  static constexpr int OFF_K = D;
  static constexpr int OFF_V = D + UW;
  static constexpr int OFF_VSZ = D + 2 * UW;
  static constexpr int STAGE = D + UREC;
  static_assert((STAGE * 4) % 16 == 0 && (D * 4) % 16 == 0, "TMA bulk alignment");
};

template <int D, int NREP>
VC_DEV void write_partial(const AttnShape& s, const AttnSeq& sq, int h, int chunk, float* sm_m,
                          float* sm_l, float* sm_o, Partials part) {
  // sm_m/sm_l: [kWarps][8]; sm_o: [kWarps][8][D]
  const int hq0 = h * NREP;
  const int Hq = s.n_kv * NREP;
  for (int idx = threadIdx.x; idx < NREP * D; idx += blockDim.x) {
    const int n = idx / D, c = idx % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm_m[w * 8 + n]);
    float o = 0.f, l = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float mw = sm_m[w * 8 + n];
      const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      o += f * sm_o[(w * 8 + n) * D + c];
      l += f * sm_l[w * 8 + n];
    }
    const size_t prow = static_cast<size_t>(sq.part0 + chunk) * Hq + hq0 + n;
    part.o[prow * D + c] = o;
    if (c == 0) {
      part.ml[prow * 2] = M;
      part.ml[prow * 2 + 1] = l;
    }
  }
}

template <int D, int BITS, int NREP>
__global__ void __launch_bounds__(128) draft_attn_quant_kernel(AttnShape s, QuantPool pool,
                                                               int layer, const uint16_t* qkv,
                                                               const AttnSeq* seqs, int max_chunks,
                                                               Partials part) {
  static_assert(NREP <= 8, "n_rep > 8 needs two head tiles");
  using GEO = Geo<D, BITS>;
  constexpr int KS = GEO::KS, W = GEO::W, CH = GEO::CH, UMT = GEO::UMT;
  constexpr uint32_t MASK = BITS == 4 ? 0x000f000fu : 0x00030003u;

  extern __shared__ __align__(128) uint32_t dsm[];   // [kWarps][2][STAGE]
  __shared__ float sq_q[NREP * D];                   // scaled q, head-major
  __shared__ __align__(8) uint64_t bars[kWarps][2];
  __shared__ float sm_m[kWarps * 8], sm_l[kWarps * 8];
  float* sm_o = reinterpret_cast<float*>(dsm);       // reused after the pipeline drains

  const AttnSeq sq = seqs[blockIdx.z];
  const int h = blockIdx.y;
  const int chunk = blockIdx.x;
  const bool tail = chunk >= max_chunks;              // bf16 tail chunks follow the quantised ones
  const int t_lo = (chunk - max_chunks) * VC_TAIL_CHUNK;
  const int n_chunks = (sq.n_groups + kCG - 1) / kCG;
  if (tail ? t_lo >= sq.tail_len : chunk >= n_chunks) return;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t slice = (static_cast<size_t>(sq.slot) * s.layers + layer) * s.n_kv + h;

  // q heads h*NREP .. h*NREP+NREP-1 are contiguous in the qkv row.
  const uint16_t* qrow = qkv + static_cast<size_t>(sq.row0) * s.q_stride + static_cast<size_t>(h) * NREP * D;
  for (int i = threadIdx.x; i < NREP * D; i += blockDim.x) sq_q[i] = bf2f(qrow[i]) * s.scale_log2;

  if (tail) {
    __syncthreads();
    // ---- bf16 tail (residual group + draft window), CUDA cores ----------
    constexpr int CPL = D / 32;  // channels per lane
    const uint16_t* kt = pool.ktail + slice * pool.tail_cap * D;
    const uint16_t* vt = pool.vtail + slice * pool.tail_cap * D;
    float m[NREP], l[NREP], o[NREP][CPL];
#pragma unroll
    for (int n = 0; n < NREP; ++n) {
      m[n] = -INFINITY;
      l[n] = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; ++j) o[n][j] = 0.f;
    }
    // this warp's 8 tokens of the 32-token chunk: all loads issued up front
    constexpr int TPW = VC_TAIL_CHUNK / kWarps;
    const int tw = t_lo + warp * TPW;
    const int nt = max(0, min(TPW, sq.tail_len - tw));
    float kv[TPW][CPL], vv[TPW][CPL];
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int t = i < nt ? tw + i : tw;  // clamp; unused when i >= nt
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        kv[i][j] = i < nt ? bf2f(kt[static_cast<size_t>(t) * D + lane * CPL + j]) : 0.f;
        vv[i][j] = i < nt ? bf2f(vt[static_cast<size_t>(t) * D + lane * CPL + j]) : 0.f;
      }
    }
    float dots[TPW][NREP];
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
      for (int n = 0; n < NREP; ++n) {
        float d = 0.f;
#pragma unroll
        for (int j = 0; j < CPL; ++j) d += sq_q[n * D + lane * CPL + j] * kv[i][j];
        dots[i][n] = d;
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)  // all TPW*NREP reductions in flight together
#pragma unroll
      for (int i = 0; i < TPW; ++i)
#pragma unroll
        for (int n = 0; n < NREP; ++n) dots[i][n] += __shfl_xor_sync(0xffffffffu, dots[i][n], off);
#pragma unroll
    for (int n = 0; n < NREP; ++n) {
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < TPW; ++i)
        if (i < nt) mx = fmaxf(mx, dots[i][n]);
      m[n] = mx;
      float ls = 0.f;
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const float p = i < nt ? exp2f(dots[i][n] - mx) : 0.f;
        ls += p;
#pragma unroll
        for (int j = 0; j < CPL; ++j) o[n][j] += p * vv[i][j];
      }
      l[n] = ls;
    }
    if (lane == 0) {
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        sm_m[warp * 8 + n] = n < NREP ? m[n < NREP ? n : 0] : -INFINITY;
        sm_l[warp * 8 + n] = n < NREP ? l[n < NREP ? n : 0] : 0.f;
      }
    }
#pragma unroll
    for (int n = 0; n < NREP; ++n)
#pragma unroll
      for (int j = 0; j < CPL; ++j) sm_o[(warp * 8 + n) * D + lane * CPL + j] = o[n][j];
    __syncthreads();
    write_partial<D, NREP>(s, sq, h, chunk, sm_m, sm_l, sm_o, part);
    return;
  }

  // ---- quantised groups: per-warp TMA pipeline over kUnit-token units --------
  const uint32_t* recs = pool.rec + slice * (static_cast<size_t>(pool.cap / kG) * GEO::GREC);
  uint32_t* stage0 = dsm + static_cast<size_t>(warp) * 2 * GEO::STAGE;
  uint64_t* bar = bars[warp];

  // this warp's groups: chunk*kCG + warp, + kWarps, ... ; kUPG units each
  constexpr int kUPG = kG / kUnit;
  const int g_first = chunk * kCG + warp;
  const int g_end = min((chunk + 1) * kCG, sq.n_groups);
  const int n_mine = g_first < g_end ? (g_end - g_first + kWarps - 1) / kWarps : 0;
  const int n_units = kUPG * n_mine;

  auto issue = [&](int u, int st) {  // lane 0 only: one bulk copy per unit
    const int g = g_first + (u / kUPG) * kWarps;
    const int part = u % kUPG;
    const uint32_t* src = recs + static_cast<size_t>(g) * GEO::GREC;
    uint32_t* dst = stage0 + st * GEO::STAGE;
    if (part == 0) {
      mbar_expect_tx(bar + st, GEO::STAGE * 4);
      tma_load_1d(dst, src, GEO::STAGE * 4, bar + st);
    } else {
      mbar_expect_tx(bar + st, GEO::UREC * 4);
      tma_load_1d(dst + GEO::OFF_K, src + D + part * GEO::UREC, GEO::UREC * 4, bar + st);
    }
  };
  // A-fragment registers of one code word.  int4: one shift + four lop3,
  // pairs 2/3 (k or token +8) arrive as 1024 + 16c -- their B operand carries
  // the matching 1/16.  int2: word holds two k-steps, sub selects one.
  auto unpack = [&](uint32_t w, int sub, uint32_t* a) {
    if constexpr (BITS == 4) {
      const uint32_t w8 = w >> 8;
      a[0] = nib_to_h2(w, 0x000f000fu);
      a[1] = nib_to_h2(w8, 0x000f000fu);
      a[2] = nib_to_h2(w, 0x00f000f0u);
      a[3] = nib_to_h2(w8, 0x00f000f0u);
    } else {
      const int sh = 8 * sub;
#pragma unroll
      for (int j = 0; j < 4; ++j) a[j] = nib_to_h2(w >> (sh + j * BITS), MASK);
    }
  };
  constexpr float kHiScale = BITS == 4 ? 0.0625f : 1.0f;  // B-operand scale of pairs 2/3
  if (lane == 0) {
    mbar_init(bar + 0, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  __syncthreads();  // sq_q and barrier init visible
  if (lane == 0) {
    if (n_units > 0) issue(0, 0);
    if (n_units > 1) issue(1, 1);
  }

  const int hn = lane >> 2;         // head column this lane feeds in B fragments
  const int hc0 = 2 * (lane & 3);   // head columns this lane holds in C fragments
  float mrun0 = -INFINITY, mrun1 = -INFINITY;
  float lsum0 = 0.f, lsum1 = 0.f, corr0 = 0.f, corr1 = 0.f;
  float oacc[KS][4];
#pragma unroll
  for (int ct = 0; ct < KS; ++ct) oacc[ct][0] = oacc[ct][1] = oacc[ct][2] = oacc[ct][3] = 0.f;
  uint32_t b0[KS], b1[KS];
  float bias0 = 0.f, bias1 = 0.f;

  for (int u = 0; u < n_units; ++u) {
    const int st = u & 1;
    mbar_wait(bar + st, (u >> 1) & 1);
    const uint32_t* sb = stage0 + st * GEO::STAGE;
    if (u % kUPG == 0) {
      // new group: q' = q * kscale as fp16 B fragments; per-head constant term
      float bias_part = 0.f;
      const float* qh = sq_q + (hn < NREP ? hn : 0) * D;
      const float qmask = hn < NREP ? 1.f : 0.f;  // padding head columns feed zeros
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const int c0 = k * 16 + 2 * (lane & 3);
#pragma unroll
        for (int hi = 0; hi < 2; ++hi) {  // channels c0,c0+1 then c0+8,c0+9
          const int c = c0 + 8 * hi;
          const uint2 sz = *reinterpret_cast<const uint2*>(sb + GEO::OFF_KSZ + c);
          const float2 sz0 = h2_to_f2(sz.x), sz1 = h2_to_f2(sz.y);  // (scale, zero)
          const float2 q = *reinterpret_cast<const float2*>(qh + c);
          const float q0 = q.x * qmask, q1 = q.y * qmask;
          const float f = hi ? kHiScale : 1.0f;
          const uint32_t bq = pack_h2(q0 * sz0.x * f, q1 * sz1.x * f);
          // zero point and the -1024 fold use the fp16-rounded q' the MMA sees
          const float2 qr = h2_to_f2(bq);
          bias_part += q0 * sz0.y + q1 * sz1.y - 1024.f * (qr.x + qr.y);
          (hi ? b1 : b0)[k] = bq;
        }
      }
      bias_part += __shfl_xor_sync(0xffffffffu, bias_part, 1);
      bias_part += __shfl_xor_sync(0xffffffffu, bias_part, 2);
      bias0 = __shfl_sync(0xffffffffu, bias_part, hc0 * 4);
      bias1 = __shfl_sync(0xffffffffu, bias_part, (hc0 + 1) * 4);
    }

    // S^T tiles of the unit's kUnit tokens
    float sacc[UMT][4];
#pragma unroll
    for (int m = 0; m < UMT; ++m) {
      uint32_t kw[W];
#pragma unroll
      for (int wq = 0; wq < W / CH; ++wq) {
        const uint32_t* p = sb + GEO::OFF_K + (static_cast<size_t>(m * (W / CH) + wq) * 32 + lane) * CH;
        if constexpr (CH == 4) {
          const uint4 v = lds128(p);
          kw[wq * 4 + 0] = v.x; kw[wq * 4 + 1] = v.y; kw[wq * 4 + 2] = v.z; kw[wq * 4 + 3] = v.w;
        } else {
          const uint2 v = lds64(p);
          kw[wq * 2 + 0] = v.x; kw[wq * 2 + 1] = v.y;
        }
      }
      sacc[m][0] = sacc[m][1] = sacc[m][2] = sacc[m][3] = 0.f;
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        uint32_t a[4];
        unpack((BITS == 4) ? kw[k] : kw[k >> 1], k & 1, a);
        mma_f16(sacc[m], a[0], a[1], a[2], a[3], b0[k], b1[k]);
      }
      sacc[m][0] += bias0; sacc[m][1] += bias1; sacc[m][2] += bias0; sacc[m][3] += bias1;
    }

    // online softmax (columns hc0, hc0+1; rows spread over lane>>2 and +8)
    float gm0 = -INFINITY, gm1 = -INFINITY;
#pragma unroll
    for (int m = 0; m < UMT; ++m) {
      gm0 = fmaxf(gm0, fmaxf(sacc[m][0], sacc[m][2]));
      gm1 = fmaxf(gm1, fmaxf(sacc[m][1], sacc[m][3]));
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      gm0 = fmaxf(gm0, __shfl_xor_sync(0xffffffffu, gm0, o));
      gm1 = fmaxf(gm1, __shfl_xor_sync(0xffffffffu, gm1, o));
    }
    // lazy rescale: keep the running max unless a column's max outgrew it by
    // more than kTau (p <= 2^kTau then), so most units skip the O rescale
    if (__any_sync(0xffffffffu, gm0 > mrun0 + kTau || gm1 > mrun1 + kTau)) {
      const float mn0 = fmaxf(mrun0, gm0), mn1 = fmaxf(mrun1, gm1);
      const float al0 = ex2(mrun0 - mn0), al1 = ex2(mrun1 - mn1);
      mrun0 = mn0;
      mrun1 = mn1;
      lsum0 *= al0; lsum1 *= al1; corr0 *= al0; corr1 *= al1;
#pragma unroll
      for (int ct = 0; ct < KS; ++ct) {
        oacc[ct][0] *= al0; oacc[ct][1] *= al1; oacc[ct][2] *= al0; oacc[ct][3] *= al1;
      }
    }
    uint32_t bp0[UMT], bp1[UMT];
#pragma unroll
    for (int m = 0; m < UMT; ++m) {
      const int r = m * 16 + (lane >> 2);
      const uint32_t sz_a = sb[GEO::OFF_VSZ + r], sz_b = sb[GEO::OFF_VSZ + r + 8];
      const float vs_a = h2f(static_cast<uint16_t>(sz_a & 0xffffu)), vz_a = h2f(static_cast<uint16_t>(sz_a >> 16));
      const float vs_b = h2f(static_cast<uint16_t>(sz_b & 0xffffu)), vz_b = h2f(static_cast<uint16_t>(sz_b >> 16));
      const float p0 = ex2(sacc[m][0] - mrun0), p1 = ex2(sacc[m][1] - mrun1);
      const float p2 = ex2(sacc[m][2] - mrun0), p3 = ex2(sacc[m][3] - mrun1);
      lsum0 += p0 + p2;
      lsum1 += p1 + p3;
      const uint32_t pk01 = pack_h2(p0 * vs_a, p1 * vs_a);
      const uint32_t pk23 = pack_h2(p2 * vs_b * kHiScale, p3 * vs_b * kHiScale);  // tokens +8
      const __half2 h01 = *reinterpret_cast<const __half2*>(&pk01);
      const __half2 h23 = *reinterpret_cast<const __half2*>(&pk23);
      corr0 += p0 * vz_a + p2 * vz_b - 1024.f * (__low2float(h01) + __low2float(h23));
      corr1 += p1 * vz_a + p3 * vz_b - 1024.f * (__high2float(h01) + __high2float(h23));
      bp0[m] = movmatrix_trans(pk01);
      bp1[m] = movmatrix_trans(pk23);
    }

    // O^T += Vcodes^T . P'^T
#pragma unroll
    for (int m = 0; m < UMT; ++m) {
      uint32_t vw[W];
#pragma unroll
      for (int wq = 0; wq < W / CH; ++wq) {
        const uint32_t* p = sb + GEO::OFF_V + (static_cast<size_t>(m * (W / CH) + wq) * 32 + lane) * CH;
        if constexpr (CH == 4) {
          const uint4 v = lds128(p);
          vw[wq * 4 + 0] = v.x; vw[wq * 4 + 1] = v.y; vw[wq * 4 + 2] = v.z; vw[wq * 4 + 3] = v.w;
        } else {
          const uint2 v = lds64(p);
          vw[wq * 2 + 0] = v.x; vw[wq * 2 + 1] = v.y;
        }
      }
#pragma unroll
      for (int ct = 0; ct < KS; ++ct) {
        uint32_t a[4];
        unpack((BITS == 4) ? vw[ct] : vw[ct >> 1], ct & 1, a);
        mma_f16(oacc[ct], a[0], a[1], a[2], a[3], bp0[m], bp1[m]);
      }
    }
    fence_proxy_async();  // LDS reads of the stage before the next TMA write into it
    __syncwarp();
    if (lane == 0 && u + 2 < n_units) issue(u + 2, st);
  }

  // reduce the per-lane sums over the 8 lanes sharing a head column
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    lsum0 += __shfl_xor_sync(0xffffffffu, lsum0, o);
    lsum1 += __shfl_xor_sync(0xffffffffu, lsum1, o);
    corr0 += __shfl_xor_sync(0xffffffffu, corr0, o);
    corr1 += __shfl_xor_sync(0xffffffffu, corr1, o);
  }
  __syncthreads();  // all warps done with their stages before sm_o reuses them
  if (lane < 4) {
    sm_m[warp * 8 + hc0] = mrun0;
    sm_m[warp * 8 + hc0 + 1] = mrun1;
    sm_l[warp * 8 + hc0] = lsum0;
    sm_l[warp * 8 + hc0 + 1] = lsum1;
  }
#pragma unroll
  for (int ct = 0; ct < KS; ++ct) {
    const int c = ct * 16 + (lane >> 2);
    sm_o[(warp * 8 + hc0) * D + c] = oacc[ct][0] + corr0;
    sm_o[(warp * 8 + hc0 + 1) * D + c] = oacc[ct][1] + corr1;
    sm_o[(warp * 8 + hc0) * D + c + 8] = oacc[ct][2] + corr0;
    sm_o[(warp * 8 + hc0 + 1) * D + c + 8] = oacc[ct][3] + corr1;
  }
  __syncthreads();
  write_partial<D, NREP>(s, sq, h, chunk, sm_m, sm_l, sm_o, part);
}

template <int D, int BITS, int NREP>
cudaError_t launch_draft(const AttnShape& s, const QuantPool& pool, int layer, const uint16_t* qkv,
                         const AttnSeq* seqs, int n_seq, int max_chunks, Partials part,
                         cudaStream_t st) {
  using GEO = Geo<D, BITS>;
  size_t smem = static_cast<size_t>(kWarps) * 2 * GEO::STAGE * 4;
  const size_t need_o = static_cast<size_t>(kWarps) * 8 * D * 4;  // sm_o reuse
  if (smem < need_o) smem = need_o;
  auto kern = draft_attn_quant_kernel<D, BITS, NREP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(draft_parts_per_seq(max_chunks, pool.tail_cap), s.n_kv, n_seq);
  kern<<<grid, kWarps * 32, smem, st>>>(s, pool, layer, qkv, seqs, max_chunks, part);
  return cudaGetLastError();
}

}  // namespace

cudaError_t draft_attention_quant(const AttnShape& s, const QuantPool& pool, int layer,
                                  const uint16_t* qkv, const AttnSeq* seqs, int n_seq,
                                  int max_chunks, int bits, Partials part, cudaStream_t st) {
  if (n_seq <= 0) return cudaSuccess;
#define VC_DRAFT_CASE(D_, B_, R_)                                                   \
  if (s.d == D_ && bits == B_ && s.n_rep == R_)                                    \
    return launch_draft<D_, B_, R_>(s, pool, layer, qkv, seqs, n_seq, max_chunks, part, st);
  VC_DRAFT_CASE(128, 4, 4)
  VC_DRAFT_CASE(128, 2, 4)
  VC_DRAFT_CASE(128, 4, 8)
  VC_DRAFT_CASE(128, 2, 8)
  VC_DRAFT_CASE(64, 4, 4)
  VC_DRAFT_CASE(64, 2, 4)
#undef VC_DRAFT_CASE
  return cudaErrorInvalidValue;
}

}  // namespace vc
