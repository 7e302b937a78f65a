// vc_dense_attn.cu -- attention_combine: merges the split-K partials (m, l, O)
// of the draft kernel (vc_draft_attn.cu: quantised slots, then the bf16 tail
// chunks) and of the dense kernel (vc_dense_umma.cu: VC_DENSE_CHUNK-key
// absolute chunks) in a fixed order, and writes bf16 attention rows (row-major
// or in the o_proj GEMM's tiled layout).
#include <cstdio>

#include "vc_common.cuh"
#include "vc_kernels.h"
#include "vc_tiled.cuh"

namespace vc {
namespace {

constexpr int kMaxParts = 512;  // chunks per sequence the combine can merge (256K ctx)

#ifdef VC_COMBINE_TRACE
// Diagnostics build: per CTA (blockIdx.x + gridDim.x * blockIdx.z < 4096) of
// every launch, globaltimer at start / after the index math / after the PDL
// wait / after the (m, l) loads / after M, l / at exit.  Read back with
// vc_combine_trace_dump (tools/_trace).
__device__ unsigned long long g_comb_trace[64][4096][6];
__device__ int g_comb_launch;
#define VC_CTRACE(pt)                                                                   \
  do {                                                                                  \
    const int cid = blockIdx.x + gridDim.x * blockIdx.z;                                \
    if (threadIdx.x == 0 && cid < 4096) g_comb_trace[ctr_l & 63][cid][pt] = vc_globaltimer(); \
  } while (0)
#else
#define VC_CTRACE(pt)
#endif

template <int D>
__global__ void combine_kernel(AttnShape s, CombineSets cs, Partials part, uint16_t* out) {
#ifdef VC_COMBINE_TRACE
  const int ctr_l = cs.n_sets >> 8;
  cs.n_sets &= 255;
#endif
  VC_CTRACE(0);
  pdl_trigger();
  // Everything up to the partial-row indices depends only on the step's
  // sequence table (host-written before the step, never by a kernel), so it
  // runs before the PDL wait, overlapping the attention kernel's tail.
  // this block's (set, sequence, query row): set k covers n * rows blocks
  int k = 0, b = blockIdx.x;
  while (k + 1 < cs.n_sets && b >= cs.set[k].n * cs.set[k].rows) {
    b -= cs.set[k].n * cs.set[k].rows;
    ++k;
  }
  const AttnSeq* seqs = cs.set[k].seqs;
  const int n_set = cs.set[k].n, max_chunks = cs.set[k].max_chunks, mode = cs.set[k].mode;
  const int bx = b / cs.set[k].rows, tok = b % cs.set[k].rows;
  const AttnSeq sq = seqs[bx];
  if (tok >= sq.n_rows) return;
  const int hq = blockIdx.z;
  const int Hq = s.n_kv * s.n_rep;
  int n_parts;
  if (mode == 0) {
    // quantised slots of this (sequence, head): the draft warps whose task
    // range touches it (vc_kernels.h draft_task_begin), in token order
    n_parts = 0;
    if (sq.n_groups > 0) {
      int T = 0, base = 0;
      for (int i = threadIdx.x & 31; i < n_set; i += 32) {
        const int c = seqs[i].n_groups * s.n_kv;
        T += c;
        base += i < bx ? c : 0;
      }
      T = __reduce_add_sync(0xffffffffu, T);
      base = __reduce_add_sync(0xffffffffu, base);
      const int nw = draft_active_warps(T, s.draft_warps, s.draft_min_tasks);
      const int p0 = base + (hq / s.n_rep) * sq.n_groups;
      n_parts = draft_task_warp(p0 + sq.n_groups - 1, T, nw) - draft_task_warp(p0, T, nw) + 1;
    }
  } else {
    const int vis = sq.kv_len - sq.n_rows + tok + 1;
    n_parts = (vis + VC_DENSE_CHUNK - 1) / VC_DENSE_CHUNK;
  }
  auto prow_of = [&](int c) -> size_t {
    return mode == 0 ? static_cast<size_t>(sq.part0 + c) * Hq + hq
                     : static_cast<size_t>(sq.part0 + c * sq.n_rows + tok) * Hq + hq;
  };
  // draft mode: the tail-chunk partials are merged after the quantised chunks, in order
  const int n_tail = mode == 0 ? (sq.tail_len + VC_TAIL_CHUNK - 1) / VC_TAIL_CHUNK : 0;
  const int n_all = n_parts + n_tail;
  __shared__ float s_m[kMaxParts], s_lp[kMaxParts];
  __shared__ size_t s_row[kMaxParts];
  for (int c = threadIdx.x; c < n_all; c += blockDim.x)
    s_row[c] = prow_of(c < n_parts ? c : max_chunks + (c - n_parts));
  __syncthreads();
  VC_CTRACE(1);
  pdl_wait();
  VC_CTRACE(2);
#ifdef VC_COMBINE_NOOP
  return;  // diagnostics build: the launch and its PDL boundary without the merge
#endif
  for (int c = threadIdx.x; c < n_all; c += blockDim.x) {  // every (m, l) load in parallel
    const float2 ml = *reinterpret_cast<const float2*>(part.ml + s_row[c] * 2);
    s_m[c] = ml.x;
    s_lp[c] = ml.y;
  }
  __syncthreads();
  VC_CTRACE(3);
  // Every thread (= one channel) merges on its own: M, then the weights, l
  // and O in chunk order.  Short loops instead of a warp-0 reduction and a
  // second barrier: this kernel runs once per layer with cold instruction
  // caches, so its cost is mostly its code footprint (r2 phase trace: the
  // shuffle-tree version spent 2.2 us per CTA computing M and l).
  float M = -INFINITY;
  for (int c = 0; c < n_all; ++c) M = fmaxf(M, s_m[c]);
  VC_CTRACE(4);
  const int c0 = threadIdx.x;  // blockDim.x == D
  float l = 0.f, o = 0.f;
  constexpr int kBatch = 16;  // partial rows in flight per thread
  for (int c = 0; c < n_all; c += kBatch) {
    float v[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) v[j] = c + j < n_all ? part.o[s_row[c + j] * D + c0] : 0.f;
#pragma unroll
    for (int j = 0; j < kBatch; ++j)
      if (c + j < n_all) {
        const float mc = s_m[c + j];
        const float f = mc == -INFINITY ? 0.f : exp2f(mc - M);
        l = fmaf(f, s_lp[c + j], l);
        o = fmaf(f, v[j], o);
      }
  }
  const uint16_t v = f2bf(l > 0.f ? o / l : 0.f);
  if (s.out_mp > 0)
    out[atile_idx(sq.row0 + tok, hq * D + c0, s.out_mp)] = v;
  else
    out[static_cast<size_t>(sq.row0 + tok) * s.out_stride + static_cast<size_t>(hq) * D + c0] = v;
  VC_CTRACE(5);
}

}  // namespace

cudaError_t attention_combine_sets(const AttnShape& s, const CombineSets& cs, Partials part, uint16_t* out,
                                   cudaStream_t st) {
  if (cs.n_sets < 1 || cs.n_sets > 3) return cudaErrorInvalidValue;
  int n = 0;
  for (int k = 0; k < cs.n_sets; ++k) {
    if (cs.set[k].rows < 1) return cudaErrorInvalidValue;
    n += cs.set[k].n * cs.set[k].rows;
  }
  if (n <= 0) return cudaSuccess;
  dim3 grid(n, 1, s.n_kv * s.n_rep);
#ifdef VC_COMBINE_TRACE
  static int launch_no = 0;
  CombineSets ct = cs;
  ct.n_sets |= (launch_no++ & 63) << 8;
  if (s.d == 128) return launch_pdl(combine_kernel<128>, grid, dim3(128), 0, st, s, ct, part, out);
#endif
  if (s.d == 128) return launch_pdl(combine_kernel<128>, grid, dim3(128), 0, st, s, cs, part, out);
  if (s.d == 64) return launch_pdl(combine_kernel<64>, grid, dim3(64), 0, st, s, cs, part, out);
  return cudaErrorInvalidValue;
}

cudaError_t attention_combine(const AttnShape& s, const AttnSeq* seqs, int n_seq, int max_chunks,
                              int max_rows, int mode, Partials part, uint16_t* out,
                              cudaStream_t st) {
  if (n_seq <= 0) return cudaSuccess;
  CombineSets cs;
  cs.set[0].seqs = seqs;
  cs.set[0].n = n_seq;
  cs.set[0].max_chunks = max_chunks;
  cs.set[0].mode = mode;
  cs.set[0].rows = max_rows;
  cs.n_sets = 1;
  return attention_combine_sets(s, cs, part, out, st);
}

#ifdef VC_COMBINE_TRACE
extern "C" int vc_combine_trace_dump(const char* path) {
  static unsigned long long h[64][4096][6];
  if (cudaMemcpyFromSymbol(h, g_comb_trace, sizeof(h)) != cudaSuccess) return 1;
  FILE* f = std::fopen(path, "wb");
  if (!f) return 2;
  std::fwrite(h, 1, sizeof(h), f);
  std::fclose(f);
  return 0;
}
#endif

}  // namespace vc
