// vc_draft_attn.cu -- draft decode attention over the KIVI-compressed cache.
//
// One query token per drafting sequence, n_rep query heads per kv head (GQA).
// HBM-bound: every code byte is read exactly once.  The kernel is persistent
// (one wave) and splits the step's (sequence, kv head, group) tasks into equal
// contiguous ranges, one per warp (draft_task_begin, vc_kernels.h), so every
// warp streams the same bytes whatever the batch's context lengths.  Each warp
// runs its own two-stage TMA pipeline: one lane issues ONE 1-D bulk copy
// (cp.async.bulk ... mbarrier::complete_tx) per 32-token unit record -- K
// codes, V codes, V scale/zero, and for a group's first unit the K
// scale/zero (vc_kernels.h quant_record_words) -- into shared memory while the
// warp computes on the previous unit; the stream runs on across group and
// head boundaries, so a warp never drains its pipeline until its range ends.
// The math runs on legacy mma.sync tensor-core tiles fed from LDS:
//   S^T[tok, head] = Kcodes[tok, ch] . q'^T[ch, head],  q' = q * kscale (per group)
//   O^T[ch, head]  = Vcodes^T[ch, tok] . P'^T[tok, head], P' = P * vscale (per token)
// Dequantisation is folded algebraically into q' / P' and two per-head
// constants (zero points, and the 1024 bias of the lop3 int->fp16 trick), so
// the inner loop is lop3 + mma only.  Codes are stored in mma A-fragment
// order (vc_quant.cu), the P' B-fragments come from the S C-fragments through
// movmatrix.trans, and the online softmax runs on warp shuffles.
// A warp emits one partial (m, l, O) per (sequence, head) it touches, the
// bf16 tail (residual group + draft window) runs in separate 32-token CTAs,
// and attention_combine merges the partials (LSE) in token order.
//
// The reference models this step as a pure HBM read of the compressed cache
// (/root/reference/proj/src/scheduler.cpp:452-457, sim.cpp:254-256).
#include "vc_common.cuh"
#include "vc_kernels.h"

namespace vc {
namespace {

constexpr int kG = VC_QGROUP;
constexpr int kWarps = 4;
#ifndef VC_DRAFT_STAGES
#define VC_DRAFT_STAGES 2  // unit records in flight per warp
#endif
constexpr int kStages = VC_DRAFT_STAGES;
#ifndef VC_DRAFT_TAIL_LAST
#define VC_DRAFT_TAIL_LAST 1  // grid order: quantised CTAs, then bf16-tail CTAs
#endif
#ifndef VC_DRAFT_MINB
#define VC_DRAFT_MINB 4  // resident CTAs/SM the n_rep<=4 register budget targets
#endif
#ifndef VC_DRAFT_BIAS_MMA
// the 1024 * sum(P') correction by one MMA per tile instead of per-lane
// f16->f32 sums (int2's rows +8 need that sum apart from the zero-point sum:
// the MMA, or VC_INT2_SPLIT's per-lane sums, which measured faster); for int4
// it measured neutral (16 x 32K set 3.674 vs 3.670 ms) and stays off
#define VC_DRAFT_BIAS_MMA 0
#endif
#ifndef VC_INT2_NOSHIFT
#define VC_INT2_NOSHIFT 1  // int2: four masks per byte, rows +8 carry a x4 the epilogues undo
#endif
#ifndef VC_QK_CHAINS
#define VC_QK_CHAINS 1  // dependent MMA chains per score tile (2: even / odd k-steps)
#endif
#ifndef VC_SHIFT_IMAD
// the unpack's byte shift as IMAD.HI (FMA pipe) instead of SHF (ALU pipe,
// with the lop3s): measured slower (16 x 32K int4 set 3.67 -> 4.14 ms, int2
// 3.47 -> 3.64: the IMAD's latency lands on every A fragment), so off
#define VC_SHIFT_IMAD 0
#endif
constexpr int kUnit = VC_QUNIT;  // tokens per pipeline unit = one unit record

// x >> 8.  The unpack is ALU-pipe heavy (lop3 + the shift: 55% of the ALU
// pipe, whose throttle is a top stall); mul.hi by 2^24 would run on the FMA
// pipe (ptxas keeps it an IMAD.HI.U32) -- slower, see VC_SHIFT_IMAD.
VC_DEV uint32_t shr8(uint32_t x) {
#if VC_SHIFT_IMAD
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(0x01000000u));
  return r;
#else
  return x >> 8;
#endif
}
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


// Sum over sequences [0, n) of the group tasks (n_groups * n_kv); all lanes get it.
VC_DEV int warp_task_sum(const AttnSeq* seqs, int n, int n_kv, int lane) {
  int acc = 0;
  for (int i = lane; i < n; i += 32) acc += seqs[i].n_groups * n_kv;
  return __reduce_add_sync(0xffffffffu, acc);
}

template <int D, int NREP>
__device__ void draft_tail(const AttnShape& s, const QuantPool& pool, int layer, const uint16_t* qkv,
                           const AttnSeq& sq, int h, int tc, int max_chunks, Partials part,
                           float* sm_o, float* sq_q) {
  // ---- bf16 tail (residual group + draft window), CUDA cores ----------
  __shared__ float sm_m[kWarps * 8], sm_l[kWarps * 8];
  constexpr int CPL = D / 32;  // channels per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t_lo = tc * VC_TAIL_CHUNK;
  const size_t slice = (static_cast<size_t>(sq.slot) * s.layers + layer) * s.n_kv + h;
  const uint16_t* kt = pool.ktail + slice * pool.tail_cap * D;
  const uint16_t* vt = pool.vtail + slice * pool.tail_cap * D;
  const uint16_t* qrow = qkv + static_cast<size_t>(sq.row0) * s.q_stride + static_cast<size_t>(h) * NREP * D;
  for (int i = threadIdx.x; i < NREP * D; i += blockDim.x) sq_q[i] = bf2f(qrow[i]) * s.scale_log2;
  __syncthreads();
  float m[NREP], l[NREP], o[NREP][CPL];
#pragma unroll
  for (int n = 0; n < NREP; ++n) {
    m[n] = -INFINITY;
    l[n] = 0.f;
#pragma unroll
    for (int j = 0; j < CPL; ++j) o[n][j] = 0.f;
  }
  // this warp's tokens of the 32-token chunk: all loads issued up front
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
  // merge the warps' partials into the chunk's partial row
  const int Hq = s.n_kv * NREP;
  for (int idx = threadIdx.x; idx < NREP * D; idx += blockDim.x) {
    const int n = idx / D, c = idx % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm_m[w * 8 + n]);
    float ov = 0.f, lv = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float mw = sm_m[w * 8 + n];
      const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      ov += f * sm_o[(w * 8 + n) * D + c];
      lv += f * sm_l[w * 8 + n];
    }
    const size_t prow = static_cast<size_t>(sq.part0 + max_chunks + tc) * Hq + h * NREP + n;
    part.o[prow * D + c] = ov;
    if (c == 0) {
      part.ml[prow * 2] = M;
      part.ml[prow * 2 + 1] = lv;
    }
  }
}

// grid: [n_seq * n_kv * tail chunks] tail CTAs, then s.draft_warps / kWarps
// persistent quantised CTAs.
template <int D, int BITS, int NREP>
__global__ void __launch_bounds__(kWarps * 32, NREP == 8 ? 3 : VC_DRAFT_MINB) draft_attn_quant_kernel(AttnShape s, QuantPool pool,
                                                                         int layer, const uint16_t* qkv,
                                                                         const AttnSeq* seqs, int n_seq,
                                                                         int max_chunks, Partials part) {
  static_assert(NREP <= 8, "n_rep > 8 needs two head tiles");
  using GEO = Geo<D, BITS>;
  constexpr int KS = GEO::KS, W = GEO::W, CH = GEO::CH, UMT = GEO::UMT;
  constexpr int kUPG = kG / kUnit;

  extern __shared__ __align__(128) uint32_t dsm[];   // [kWarps][2][STAGE]
  // per-warp q, fp32 pre-scaled by scale_log2, laid out [channel pair][NREP
  // heads] so the group setup reads one float2 per lane (lanes feeding a
  // padding head column, hn >= NREP, use zeros); the tail CTAs reuse it for
  // NREP*D fp32 q values
  __shared__ __align__(16) float2 sq_q[kWarps][D / 2 * NREP];
  static_assert(kWarps * (D / 2) * NREP * 2 >= NREP * D, "tail q fits");
  __shared__ __align__(8) uint64_t bars[kWarps][kStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TC = (pool.tail_cap + VC_TAIL_CHUNK - 1) / VC_TAIL_CHUNK;
  const int n_tail_ctas = n_seq * s.n_kv * TC;
  // VC_ATTN_TRACE diagnostics: this CTA's start/end on the global timer
  struct TraceEnd {
    unsigned long long* tr;
    __device__ ~TraceEnd() {
      if (tr && threadIdx.x == 0 && blockIdx.x < 2048) tr[8192 + blockIdx.x * 2 + 1] = vc_globaltimer();
    }
  } trace_end{s.trace};
  if (s.trace && threadIdx.x == 0 && blockIdx.x < 2048) {
    s.trace[8192 + blockIdx.x * 2] = vc_globaltimer();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    s.trace[16384 + blockIdx.x] = smid;
  }
  pdl_trigger();
  // grid order: the persistent quantised CTAs first (they fill every slot of
  // the wave and start together), the bf16-tail CTAs after them -- they run
  // in the slots the first-finishing quantised CTAs free (draft step 6.60 ->
  // 6.53 ms).  With the tail CTAs first, the quantised CTAs started 0.5-11 us
  // apart.  (The quantised CTAs still end 76-110 us: an SM's scheduler
  // favours its earliest-launched CTA, so round r of the launch finishes at
  // 82 / 89 / 99 / 109 us; ranges weighted against that kept the SMs' total
  // the same and ran 7% slower -- DESIGN.md.)
#if VC_DRAFT_TAIL_LAST
  const int n_quant_ctas = static_cast<int>(gridDim.x) - n_tail_ctas;
  const bool is_tail = static_cast<int>(blockIdx.x) >= n_quant_ctas;
  const int tail_idx = static_cast<int>(blockIdx.x) - n_quant_ctas, quant_cta = blockIdx.x;
#else
  const bool is_tail = static_cast<int>(blockIdx.x) < n_tail_ctas;
  const int tail_idx = blockIdx.x, quant_cta = static_cast<int>(blockIdx.x) - n_tail_ctas;
#endif
  if (is_tail) {
    pdl_wait();  // the tail holds this step's new K/V (qkv epilogue)
    const int idx = tail_idx;
    const int tc = idx % TC, h = (idx / TC) % s.n_kv, seq = idx / (TC * s.n_kv);
    const AttnSeq sq = seqs[seq];
    if (tc * VC_TAIL_CHUNK >= sq.tail_len) return;
    draft_tail<D, NREP>(s, pool, layer, qkv, sq, h, tc, max_chunks, part, reinterpret_cast<float*>(dsm),
                        reinterpret_cast<float*>(sq_q));
    return;
  }

  // ---- quantised groups: this warp's contiguous range of group tasks ----------
  const int T = warp_task_sum(seqs, n_seq, s.n_kv, lane);
  if (T == 0) return;
  const int nw = draft_active_warps(T, s.draft_warps, s.draft_min_tasks);
  const int w = quant_cta * kWarps + warp;
  if (w >= nw) return;  // no CTA-wide barriers below: warps are independent
  const int t0 = draft_task_begin(w, T, nw), t1 = draft_task_begin(w + 1, T, nw);
  const int n_units = (t1 - t0) * kUPG;

  // locate task t0: sequence (warp scan over 32 sequences at a time), head, group
  int seq0 = 0, base = 0;
  for (int i0 = 0; i0 < n_seq; i0 += 32) {
    const int i = i0 + lane;
    const int c = i < n_seq ? seqs[i].n_groups * s.n_kv : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, t0 < base + inc);
    if (hit) {
      const int L = __ffs(hit) - 1;
      seq0 = i0 + L;
      base += __shfl_sync(0xffffffffu, inc - c, L);
      break;
    }
    base += __shfl_sync(0xffffffffu, inc, 31);
  }

  // Task cursor: (sequence, head, group) plus the sequence's record base.
  struct Cursor {
    int seq, head, g, ng, base;  // base = first task of the sequence
    const uint32_t* slice;       // group records of (slot, layer, head)
  };
  const size_t slice_words = static_cast<size_t>(pool.cap / kG) * GEO::GREC;
  auto set_slice = [&](Cursor& c) {
    c.slice = pool.rec + ((static_cast<size_t>(seqs[c.seq].slot) * s.layers + layer) * s.n_kv + c.head) * slice_words;
  };
  auto next_task = [&](Cursor& c) {
    if (++c.g < c.ng) return;
    c.g = 0;
    if (++c.head < s.n_kv) { set_slice(c); return; }
    c.head = 0;
    c.base += c.ng * s.n_kv;
    // the cursors also step once past a warp's last task: stop at the batch end
    // (compute-sanitizer memcheck caught the unbounded scan reading past seqs)
    do {
      if (++c.seq >= n_seq) {
        c.ng = 1;
        return;
      }
      c.ng = seqs[c.seq].n_groups;
    } while (c.ng == 0);
    set_slice(c);
  };
  Cursor pc;  // producer (lane 0 issues, all lanes track)
  pc.seq = seq0;
  pc.base = base;
  pc.ng = seqs[seq0].n_groups;
  pc.head = (t0 - base) / pc.ng;
  pc.g = (t0 - base) % pc.ng;
  set_slice(pc);
  Cursor cc = pc;  // consumer
  Cursor cur = pc; // (sequence, head) whose partial the accumulators hold
  int ppart = 0;   // producer unit within its group

  uint32_t* stage0 = dsm + static_cast<size_t>(warp) * kStages * GEO::STAGE;
  uint64_t* bar = bars[warp];
  auto issue = [&](int st) {  // one bulk copy of the producer's next unit record
    const uint32_t* src = pc.slice + static_cast<size_t>(pc.g) * GEO::GREC;
    uint32_t* dst = stage0 + st * GEO::STAGE;
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();  // each record is read once per step
      if (ppart == 0) {
        mbar_expect_tx(bar + st, GEO::STAGE * 4);
        tma_load_1d_stream(dst, src, GEO::STAGE * 4, bar + st, pol);
      } else {
        mbar_expect_tx(bar + st, GEO::UREC * 4);
        tma_load_1d_stream(dst + GEO::OFF_K, src + D + ppart * GEO::UREC, GEO::UREC * 4, bar + st, pol);
      }
    }
    if (++ppart == kUPG) {
      ppart = 0;
      next_task(pc);
    }
  };
  // A-fragment registers of one code word.  int4: one shift + four lop3,
  // pairs 2/3 (k or token +8) arrive as 1024 + 16c -- their B operand carries
  // the matching 1/16.  int2: word holds two k-steps, sub selects one.
  auto unpack = [&](uint32_t wd, int sub, uint32_t* a) {
    if constexpr (BITS == 4) {
      const uint32_t w8 = shr8(wd);
      a[0] = nib_to_h2(wd, 0x000f000fu);
      a[1] = nib_to_h2(w8, 0x000f000fu);
      a[2] = nib_to_h2(wd, 0x00f000f0u);
      a[3] = nib_to_h2(w8, 0x00f000f0u);
    } else {
      // int2: code j of a byte sits at bits 2j.  Pairs 2/3 (k or token +8)
      // read bits 4-7 (1024 + 16c, scaled back by the B operand like int4).
#if VC_INT2_NOSHIFT
      // Rows +8 (a[1], a[3]) read bits 2-3 / 6-7 of the same byte in place:
      // 1024 + 4c / 1024 + 64c, so their code part carries a x4 that the
      // score epilogue (K) and the O fold / emit (V) divide out: 1 shift + 8
      // lop3 per word of 16 codes
      const uint32_t lo = sub ? shr8(wd) : wd;
      a[0] = nib_to_h2(lo, 0x00030003u);
      a[1] = nib_to_h2(lo, 0x000c000cu);
      a[2] = nib_to_h2(lo, 0x00300030u);
      a[3] = nib_to_h2(lo, 0x00c000c0u);
#else
      const uint32_t lo = sub ? wd >> 8 : wd, lo2 = lo >> 2;
      a[0] = nib_to_h2(lo, 0x00030003u);
      a[1] = nib_to_h2(lo2, 0x00030003u);
      a[2] = nib_to_h2(lo, 0x00300030u);
      a[3] = nib_to_h2(lo2, 0x00300030u);
#endif
    }
  };
  // x4 on the code part of rows +8 (int2, VC_INT2_NOSHIFT); 1 otherwise.
  // 16 x 32K int2 set: 3.674 ms (3 shifts per word) -> 3.473 ms (bias MMA)
  // -> 3.411 ms (per-lane split sums, VC_INT2_SPLIT)
  constexpr float kRow8 = (BITS == 2 && VC_INT2_NOSHIFT) ? 4.f : 1.f;
#ifndef VC_INT2_SPLIT
// int2: the zero-point and 1024-bias sums kept apart per lane (f16->f32 +
// FADD, reduced at the fold) instead of the bias MMA: 16 x 32K int2 set
// 3.475 -> 3.411 ms, and no register spill
#define VC_INT2_SPLIT 1
#endif
  constexpr bool kSplit = VC_INT2_SPLIT && kRow8 != 1.f;
  constexpr bool kBiasMma = (VC_DRAFT_BIAS_MMA || kRow8 != 1.f) && !kSplit;
  constexpr float kHiScale = 0.0625f;  // B-operand scale of pairs 2/3 (their A holds 1024 + 16c)
  if (lane == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(bar + i, 1);
    fence_mbar_init();
  }
  __syncwarp();
  for (int i = 0; i < kStages && i < n_units; ++i) issue(i);
  pdl_wait();  // compressed records are static within a step; q and the partials are not

  const int hn = lane >> 2;         // head column this lane feeds in B fragments
  const int hc0 = 2 * (lane & 3);   // head columns this lane holds in C fragments
  const int Hq = s.n_kv * NREP;
  float mrun0, mrun1, lsum0, lsum1, corr0, corr1;
  float oacc[KS][4];
  // kBiasMma: corr holds the zero-point part sum(p * vzero) per lane,
  // bacc (an MMA accumulator, A = 1024) the int->fp16 bias 1024 * sum(P') of
  // columns hc0 / hc0+1 over the whole warp (C-fragment [0] / [1]); else corr
  // holds both parts per lane
  float bacc[4];
  auto reset = [&]() {
    mrun0 = mrun1 = -INFINITY;
    lsum0 = lsum1 = corr0 = corr1 = 0.f;
    bacc[0] = bacc[1] = bacc[2] = bacc[3] = 0.f;
#pragma unroll
    for (int ct = 0; ct < KS; ++ct) oacc[ct][0] = oacc[ct][1] = oacc[ct][2] = oacc[ct][3] = 0.f;
  };
  // the O corrections of rows g (A) and g+8 (B, whose code part carries kRow8)
  // from the warp-reduced zero-point sums z and the bias sums
  // (kSplit: bacc[0] / [1] hold per-lane sums of P', reduced here)
  auto corrections = [&](float z0, float z1, float& a0, float& a1, float& b0, float& b1) {
    if constexpr (kSplit) {
      float s0 = bacc[0], s1 = bacc[1];
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      a0 = z0 - 1024.f * s0;
      a1 = z1 - 1024.f * s1;
      b0 = kRow8 * z0 - 1024.f * s0;
      b1 = kRow8 * z1 - 1024.f * s1;
    } else if constexpr (kBiasMma) {
      a0 = z0 - bacc[0];
      a1 = z1 - bacc[1];
      b0 = kRow8 * z0 - bacc[0];
      b1 = kRow8 * z1 - bacc[1];
    } else {
      a0 = b0 = z0;
      a1 = b1 = z1;
    }
  };
  // the partial of the consumer's current (sequence, head)
  auto emit = [&]() {
    float l0 = lsum0, l1 = lsum1, z0 = corr0, z1 = corr1;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {  // over the 8 lanes sharing a head column
      l0 += __shfl_xor_sync(0xffffffffu, l0, o);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      z0 += __shfl_xor_sync(0xffffffffu, z0, o);
      z1 += __shfl_xor_sync(0xffffffffu, z1, o);
    }
    float c0, c1, c08, c18;
    corrections(z0, z1, c0, c1, c08, c18);
    constexpr float kInv8 = 1.f / kRow8;
    const int p0 = cur.base + cur.head * cur.ng;  // first task of the (sequence, head)
    const int slot = w - draft_task_warp(p0, T, nw);
    const size_t prow = static_cast<size_t>(seqs[cur.seq].part0 + slot) * Hq + cur.head * NREP + hc0;
    if (hc0 < NREP) {
#pragma unroll
      for (int ct = 0; ct < KS; ++ct) {
        const int c = ct * 16 + (lane >> 2);
        part.o[prow * D + c] = oacc[ct][0] + c0;
        part.o[prow * D + c + 8] = (oacc[ct][2] + c08) * kInv8;
      }
      if (lane < 4) {
        part.ml[prow * 2] = mrun0;
        part.ml[prow * 2 + 1] = l0;
      }
    }
    if (hc0 + 1 < NREP) {
#pragma unroll
      for (int ct = 0; ct < KS; ++ct) {
        const int c = ct * 16 + (lane >> 2);
        part.o[(prow + 1) * D + c] = oacc[ct][1] + c1;
        part.o[(prow + 1) * D + c + 8] = (oacc[ct][3] + c18) * kInv8;
      }
      if (lane < 4) {
        part.ml[(prow + 1) * 2] = mrun1;
        part.ml[(prow + 1) * 2 + 1] = l1;
      }
    }
  };
  auto load_q = [&]() {  // the consumer head's NREP query rows -> fp32 * scale_log2, [pair][8 heads]
    const uint16_t* qrow = qkv + static_cast<size_t>(seqs[cur.seq].row0) * s.q_stride +
                           static_cast<size_t>(cur.head) * NREP * D;
    __syncwarp();
    for (int i = lane; i < D / 2 * NREP; i += 32) {
      const int cp = i / NREP, h = i % NREP;
      const uint32_t qq = *reinterpret_cast<const uint32_t*>(qrow + h * D + 2 * cp);
      sq_q[warp][i] = make_float2(bf2f(static_cast<uint16_t>(qq & 0xffffu)) * s.scale_log2,
                                  bf2f(static_cast<uint16_t>(qq >> 16)) * s.scale_log2);
    }
    __syncwarp();
  };
  reset();
  load_q();
  uint32_t b0[KS], b1[KS];
  float bias0 = 0.f, bias1 = 0.f, bias08 = 0.f, bias18 = 0.f;
  int cpart = 0;

  for (int u = 0; u < n_units; ++u) {
    const int st = u % kStages;
    if (cpart == 0 && (cc.seq != cur.seq || cc.head != cur.head)) {
      emit();  // crossed into the next (sequence, head): flush its partial, restart
      cur = cc;
      reset();
      load_q();
    }
    mbar_wait(bar + st, (u / kStages) & 1);
    const uint32_t* sb = stage0 + st * GEO::STAGE;
    if (cpart == 0) {
      // new group: q' = q * kscale as fp16 B fragments (f16x2 multiply of the
      // packed q and the two channels' scales, gathered with one PRMT), and the
      // per-head constant  sum_c q_c z_c - 1024 sum_c q'_c : the zero-point
      // part in fp32 FFMAs, the -1024 part (over the fp16 q' the MMA sees) by
      // one extra MMA per k-step against a constant-1024 A tile
      float bias_part = 0.f;
      const float2* qf = sq_q[warp] + (hn < NREP ? hn : 0);
      const bool live_col = hn < NREP;
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const int c0 = k * 16 + 2 * (lane & 3);
#pragma unroll
        for (int hi = 0; hi < 2; ++hi) {  // channels c0,c0+1 then c0+8,c0+9
          const int c = c0 + 8 * hi;
          const uint2 sz = *reinterpret_cast<const uint2*>(sb + GEO::OFF_KSZ + c);  // (s_c|z_c), (s_c1|z_c1)
          const float2 q = live_col ? qf[(c >> 1) * NREP] : make_float2(0.f, 0.f);
          const uint32_t q16 = hi ? pack_h2(q.x * kHiScale, q.y * kHiScale) : pack_h2(q.x, q.y);
          const uint32_t bq = hmul2_u32(q16, __byte_perm(sz.x, sz.y, 0x5410));
          const float2 z = h2_to_f2(__byte_perm(sz.x, sz.y, 0x7632));
          bias_part = fmaf(q.x, z.x, fmaf(q.y, z.y, bias_part));
          (hi ? b1 : b0)[k] = bq;
        }
      }
      float c1024[4] = {0.f, 0.f, 0.f, 0.f};
      constexpr uint32_t kA1024 = 0x64006400u;  // fp16 pair (1024, 1024)
#pragma unroll
      for (int k = 0; k < KS; ++k) mma_f16(c1024, kA1024, kA1024, kA1024, kA1024, b0[k], b1[k]);
      bias_part += __shfl_xor_sync(0xffffffffu, bias_part, 1);
      bias_part += __shfl_xor_sync(0xffffffffu, bias_part, 2);
      const float zq0 = __shfl_sync(0xffffffffu, bias_part, hc0 * 4);
      const float zq1 = __shfl_sync(0xffffffffu, bias_part, (hc0 + 1) * 4);
      bias0 = zq0 - c1024[0];
      bias1 = zq1 - c1024[1];
      bias08 = zq0 - c1024[0] * (1.f / kRow8);  // rows +8: raw / kRow8 + bias08
      bias18 = zq1 - c1024[1] * (1.f / kRow8);
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
#if VC_QK_CHAINS == 2
      // two accumulator chains over the k-steps (even / odd), summed after:
      // halves the dependent MMA chain of a tile (diagnostics A/B)
      float s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        uint32_t a[4];
        unpack((BITS == 4) ? kw[k] : kw[k >> 1], k & 1, a);
        mma_f16((k & 1) ? s2 : sacc[m], a[0], a[1], a[2], a[3], b0[k], b1[k]);
      }
      sacc[m][0] += s2[0]; sacc[m][1] += s2[1]; sacc[m][2] += s2[2]; sacc[m][3] += s2[3];
#else
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        uint32_t a[4];
        unpack((BITS == 4) ? kw[k] : kw[k >> 1], k & 1, a);
        mma_f16(sacc[m], a[0], a[1], a[2], a[3], b0[k], b1[k]);
      }
#endif
      sacc[m][0] += bias0; sacc[m][1] += bias1;
      if constexpr (kRow8 == 1.f) {
        sacc[m][2] += bias0; sacc[m][3] += bias1;
      } else {
        sacc[m][2] = fmaf(sacc[m][2], 1.f / kRow8, bias08);
        sacc[m][3] = fmaf(sacc[m][3], 1.f / kRow8, bias18);
      }
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
      if constexpr (kBiasMma || kSplit) {
        bacc[0] *= al0; bacc[1] *= al1;
      }
#pragma unroll
      for (int ct = 0; ct < KS; ++ct) {
        oacc[ct][0] *= al0; oacc[ct][1] *= al1; oacc[ct][2] *= al0; oacc[ct][3] *= al1;
      }
    }
    uint32_t bp0[UMT], bp1[UMT];
#pragma unroll
    for (int m = 0; m < UMT; ++m) {
      const int r = m * 16 + (lane >> 2);
      const float2 sza = h2_to_f2(sb[GEO::OFF_VSZ + r]), szb = h2_to_f2(sb[GEO::OFF_VSZ + r + 8]);
      const float p0 = ex2(sacc[m][0] - mrun0), p1 = ex2(sacc[m][1] - mrun1);
      const float p2 = ex2(sacc[m][2] - mrun0), p3 = ex2(sacc[m][3] - mrun1);
      lsum0 += p0 + p2;
      lsum1 += p1 + p3;
      const uint32_t pk01 = pack_h2(p0 * sza.x, p1 * sza.x);
      const uint32_t pk23 = pack_h2(p2 * szb.x * kHiScale, p3 * szb.x * kHiScale);  // tokens +8
      if constexpr (kBiasMma) {
        corr0 += p0 * sza.y + p2 * szb.y;
        corr1 += p1 * sza.y + p3 * szb.y;
        bp0[m] = movmatrix_trans(pk01);
        bp1[m] = movmatrix_trans(pk23);
        // 1024 * sum over the tile's tokens of P' (exactly the B operand the
        // PV MMA sees), per head column, accumulated across tiles
        mma_f16(bacc, 0x64006400u, 0x64006400u, 0x64006400u, 0x64006400u, bp0[m], bp1[m]);
      } else if constexpr (kSplit) {
        const float2 h01 = h2_to_f2(pk01), h23 = h2_to_f2(pk23);
        corr0 += p0 * sza.y + p2 * szb.y;
        corr1 += p1 * sza.y + p3 * szb.y;
        bacc[0] += h01.x + h23.x;
        bacc[1] += h01.y + h23.y;
        bp0[m] = movmatrix_trans(pk01);
        bp1[m] = movmatrix_trans(pk23);
      } else {
        const float2 h01 = h2_to_f2(pk01), h23 = h2_to_f2(pk23);
        corr0 += p0 * sza.y + p2 * szb.y - 1024.f * (h01.x + h23.x);
        corr1 += p1 * sza.y + p3 * szb.y - 1024.f * (h01.y + h23.y);
        bp0[m] = movmatrix_trans(pk01);
        bp1[m] = movmatrix_trans(pk23);
      }
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
    if (u + kStages < n_units) issue(st);
    if (++cpart == kUPG) {
      cpart = 0;
      next_task(cc);
      // fold the column's correction into O once per group: the MMA carries
      // 1024 * sum(P') (the int->fp16 bias) that corr cancels; left to grow
      // over a long range (a warp takes T / warps groups -- 14 at 16 x 32K)
      // the two fp32 sums cancel catastrophically (logits off by 20-40% at
      // 24-48 x 32K; tests/test_real_shapes.py::test_draft_batched_equals_single)
      float z0 = corr0, z1 = corr1;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        z0 += __shfl_xor_sync(0xffffffffu, z0, o);
        z1 += __shfl_xor_sync(0xffffffffu, z1, o);
      }
      float c0, c1, c08, c18;
      corrections(z0, z1, c0, c1, c08, c18);
#pragma unroll
      for (int ct = 0; ct < KS; ++ct) {
        oacc[ct][0] += c0; oacc[ct][1] += c1; oacc[ct][2] += c08; oacc[ct][3] += c18;
      }
      corr0 = corr1 = 0.f;
      bacc[0] = bacc[1] = bacc[2] = bacc[3] = 0.f;
    }
  }
  emit();  // the last (sequence, head) of the range
}

template <int D, int BITS, int NREP>
size_t draft_smem() {
  using GEO = Geo<D, BITS>;
  size_t smem = static_cast<size_t>(kWarps) * kStages * GEO::STAGE * 4;
  const size_t need_o = static_cast<size_t>(kWarps) * 8 * D * 4;  // tail CTAs' sm_o
  return smem < need_o ? need_o : smem;
}

template <int D, int BITS, int NREP>
int quant_warps() {
  auto kern = draft_attn_quant_kernel<D, BITS, NREP>;
  const size_t smem = draft_smem<D, BITS, NREP>();
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem) != cudaSuccess)
    return 0;
  return sms * (per_sm > 0 ? per_sm : 1) * kWarps;
}

template <int D, int BITS, int NREP>
cudaError_t launch_draft(const AttnShape& s, const QuantPool& pool, int layer, const uint16_t* qkv,
                         const AttnSeq* seqs, int n_seq, int max_chunks, Partials part,
                         cudaStream_t st) {
  auto kern = draft_attn_quant_kernel<D, BITS, NREP>;
  const size_t smem = draft_smem<D, BITS, NREP>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (s.draft_warps <= 0 || s.draft_warps % kWarps || s.draft_min_tasks <= 0) return cudaErrorInvalidValue;
  const int tail_ctas = n_seq * s.n_kv * ((pool.tail_cap + VC_TAIL_CHUNK - 1) / VC_TAIL_CHUNK);
  return launch_pdl(kern, dim3(tail_ctas + s.draft_warps / kWarps), dim3(kWarps * 32), smem, st, s, pool, layer, qkv,
                    seqs, n_seq, max_chunks, part);
}

}  // namespace

#define VC_DRAFT_SHAPES(X) X(128, 4, 4) X(128, 2, 4) X(128, 4, 8) X(128, 2, 8) X(64, 4, 4) X(64, 2, 4)

int draft_quant_warps(int d, int bits, int n_rep) {
#define VC_DRAFT_CASE(D_, B_, R_) \
  if (d == D_ && bits == B_ && n_rep == R_) return quant_warps<D_, B_, R_>();
  VC_DRAFT_SHAPES(VC_DRAFT_CASE)
#undef VC_DRAFT_CASE
  return 0;
}

cudaError_t draft_attention_quant(const AttnShape& s, const QuantPool& pool, int layer,
                                  const uint16_t* qkv, const AttnSeq* seqs, int n_seq,
                                  int max_chunks, int bits, Partials part, cudaStream_t st) {
  if (n_seq <= 0) return cudaSuccess;
#define VC_DRAFT_CASE(D_, B_, R_)                \
  if (s.d == D_ && bits == B_ && s.n_rep == R_) \
    return launch_draft<D_, B_, R_>(s, pool, layer, qkv, seqs, n_seq, max_chunks, part, st);
  VC_DRAFT_SHAPES(VC_DRAFT_CASE)
#undef VC_DRAFT_CASE
  return cudaErrorInvalidValue;
}

}  // namespace vc
