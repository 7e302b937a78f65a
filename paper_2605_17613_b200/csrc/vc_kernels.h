// vc_kernels.h -- internal launch interface of the sm_100a kernels (host and
// device visible; no torch types).  The public boundary is include/vc_api.h.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#define VC_QGROUP 128      // tokens per quantised K group (KIVI G)
#define VC_TAIL_CHUNK 32   // bf16-tail tokens per draft-attention tail CTA

// Draft partial slots per sequence: the quantised chunks, then the tail chunks.
inline int draft_parts_per_seq(int max_chunks, int tail_cap) {  // quantised slots + tail chunks
  return max_chunks + (tail_cap + VC_TAIL_CHUNK - 1) / VC_TAIL_CHUNK;
}
#ifndef VC_DENSE_CHUNK
#define VC_DENSE_CHUNK 2048 // keys per dense-attention chunk (absolute positions); r1 sweep: 512 -> 2048 = 1.6x verify, 1.04x decode
#endif

namespace vc {

// ---------------------------------------------------------------- quantiser
// One (layer, request, kv-head) slice: groups [g0, g0+ng) of the bf16 source
// rows (token-major [T][d]) are quantised into the slice's code/scale arrays.
struct QuantJob {
  const uint16_t* k;  // bf16 source rows, token 0 of group 0
  const uint16_t* v;
  uint32_t* rec;      // the slice's group records (quant_record_words each), group 0
  int g0, ng;
};
cudaError_t quant_kivi(const QuantJob* jobs_dev, int n_jobs, int max_groups, int d, int bits,
                       cudaStream_t st);

// u32 words of one quantised group (K or V): G*d*bits/32.
inline constexpr size_t quant_group_words(int d, int bits) {
  return static_cast<size_t>(VC_QGROUP) * d * bits / 32;
}
// Quantised group record, the unit one draft-attention TMA copy streams
// (DESIGN.md "Compressed KV layout"), in u32 words:
//   [ksz: d (scale,zero) fp16 pairs]
//   G/VC_QUNIT unit records: [K codes U*d*bits/32][V codes U*d*bits/32][vsz: U pairs]
// Codes inside a unit record are in mma.sync A-fragment order (vc_quant.cu).
#define VC_QUNIT 32  // tokens per unit record
inline constexpr size_t quant_unit_code_words(int d, int bits) {
  return static_cast<size_t>(VC_QUNIT) * d * bits / 32;
}
inline constexpr size_t quant_unit_words(int d, int bits) {
  return 2 * quant_unit_code_words(d, bits) + VC_QUNIT;
}
inline constexpr size_t quant_record_words(int d, int bits) {
  return static_cast<size_t>(d) + (VC_QGROUP / VC_QUNIT) * quant_unit_words(d, bits);
}

// ------------------------------------------------------------ attention I/O
// Per-sequence descriptor shared by the attention kernels (device array).
struct AttnSeq {
  int slot;      // pool slot of the request
  int row0;      // first activation row of this sequence in the step batch
  int n_rows;    // query tokens (1 for draft/decode, x+1 for verify)
  int kv_len;    // keys visible to the LAST query row (dense pools)
  int n_groups;  // quantised groups (draft pool)
  int tail_len;  // bf16 tail tokens (draft pool)
  int part0;     // first partial-row index of this sequence (combine workspace)
  int pad;
};

struct KvPool {        // bf16 [slot][layer][head][cap][d]
  uint16_t* k;
  uint16_t* v;
  int cap;             // token capacity per slice
};

struct QuantPool {     // per slice: cap/G group records, then the bf16 tail
  uint32_t* rec;       // [slice][cap/G][quant_record_words]
  uint16_t* ktail;     // bf16 [slice][tail_cap][d]
  uint16_t* vtail;
  int cap;             // token capacity of the quantised region (multiple of G)
  int tail_cap;
};

struct AttnShape {
  int layers, n_kv, n_rep, d;
  int q_stride;        // elements per activation row of the qkv buffer
  int out_stride;      // elements per row of the attention output (row-major)
  int out_mp;          // > 0: write the output in the GEMM's tiled layout with Mp rows
  float scale_log2;    // log2(e)/sqrt(d)
  int draft_warps;     // quantised-draft warps launched (persistent, draft_quant_warps)
  int draft_min_tasks; // fewest group tasks a draft warp takes (bounds partials per head)
  // diagnostics (VC_ATTN_TRACE): per-CTA globaltimer at start/end of the draft
  // kernel at [8192 + 2 * cta]; nullptr = off.  (The dense kernel carries no
  // probe: two guarded timer stores there cost it 8% on the decode baseline,
  // r2 A/B 10.60 vs 11.50 ms per 16 x 32K launch set.)
  unsigned long long* trace = nullptr;
};
__device__ __forceinline__ unsigned long long vc_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Draft-attention work split: the T = sum(n_groups * n_kv) group tasks of a
// step, ordered (sequence, kv head, group), are cut into nw contiguous ranges
// of near-equal length, one per warp (stream-K style), so every warp streams
// the same number of bytes whatever the batch's context lengths are.  A warp
// emits one partial per (sequence, head) it touches; its slot is the warp's
// ordinal among the warps touching that head.
__host__ __device__ inline int draft_active_warps(int T, int nw, int min_tasks) {
  const int cap = T / min_tasks;
  return cap < 1 ? 1 : (cap < nw ? cap : nw);
}
__host__ __device__ inline int draft_task_begin(int w, int T, int nw) {
  return static_cast<int>(static_cast<long long>(w) * T / nw);
}
__host__ __device__ inline int draft_task_warp(int t, int T, int nw) {  // warp owning task t
  return static_cast<int>((static_cast<long long>(t + 1) * nw - 1) / T);
}
// warps launched for the quantised draft path (one full wave; 0 = unsupported shape)
int draft_quant_warps(int d, int bits, int n_rep);

// Split-K partials: o [part_rows][d] fp32, ml [part_rows][2] (max in log2
// domain, sum).  A partial row is (sequence part0 + chunk*rows + r).
struct Partials {
  float* o;
  float* ml;
};

cudaError_t draft_attention_quant(const AttnShape& s, const QuantPool& pool, int layer,
                                  const uint16_t* qkv, const AttnSeq* seqs, int n_seq,
                                  int max_chunks, int bits, Partials part, cudaStream_t st);

// TMA tensor maps of the dense path: K and V pools as 2-D [slices*cap, d]
// (128-key x 64-channel boxes) and the query heads of the activation rows as
// 3-D [rows, heads, d] (n_rep heads x 128/n_rep tokens per box), 128B swizzle.
struct DenseMaps {
  CUtensorMap k, v, q;
};
bool make_kv_maps(DenseMaps* m, const KvPool& pool, size_t slices, int d);
bool make_q_map(DenseMaps* m, const uint16_t* qkv, int d, int heads_per_row, int rows, int q_stride, int n_rep);
cudaError_t dense_attention(const AttnShape& s, const KvPool& pool, const DenseMaps& maps, int layer,
                            const AttnSeq* seqs, int n_seq, int max_chunks, int max_rows, Partials part,
                            cudaStream_t st);

// Merge the chunk partials of every (sequence, query token, q head) in chunk
// order into bf16 attention output rows.  mode 0 = draft layout (chunks of
// the quantised pool + one tail partial), 1 = dense layout.
cudaError_t attention_combine(const AttnShape& s, const AttnSeq* seqs, int n_seq, int max_chunks,
                              int max_rows, int mode, Partials part, uint16_t* out,
                              cudaStream_t st);
// Up to three sequence sets of one step (drafting, dense decode, verify
// windows) merged by ONE launch: same per-(sequence, token, head) arithmetic
// and order as attention_combine, one kernel boundary instead of three.
struct CombineSet {
  const AttnSeq* seqs = nullptr;
  int n = 0, max_chunks = 0, mode = 0;
  int rows = 1;  // query rows per sequence the grid covers (max over the set)
};
struct CombineSets {
  CombineSet set[3];
  int n_sets = 0;
};
cudaError_t attention_combine_sets(const AttnShape& s, const CombineSets& cs, Partials part, uint16_t* out,
                                   cudaStream_t st);

}  // namespace vc
