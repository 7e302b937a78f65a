// vc_kernels.h -- internal launch interface of the sm_100a kernels (host and
// device visible; no torch types).  The public boundary is include/vc_api.h.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#define VC_QGROUP 128      // tokens per quantised K group (KIVI G)
#define VC_DRAFT_CG 8      // quantised groups per draft-attention chunk (1024 tokens)
#define VC_TAIL_CHUNK 32   // bf16-tail tokens per draft-attention tail CTA

// Draft partial slots per sequence: the quantised chunks, then the tail chunks.
inline int draft_parts_per_seq(int max_chunks, int tail_cap) {
  return max_chunks + (tail_cap + VC_TAIL_CHUNK - 1) / VC_TAIL_CHUNK;
}
#define VC_DENSE_CHUNK 512 // keys per dense-attention chunk (absolute positions)

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
};

// Split-K partials: o [part_rows][d] fp32, ml [part_rows][2] (max in log2
// domain, sum).  A partial row is (sequence part0 + chunk*rows + r).
struct Partials {
  float* o;
  float* ml;
};

cudaError_t draft_attention_quant(const AttnShape& s, const QuantPool& pool, int layer,
                                  const uint16_t* qkv, const AttnSeq* seqs, int n_seq,
                                  int max_chunks, int bits, Partials part, cudaStream_t st);

cudaError_t dense_attention(const AttnShape& s, const KvPool& pool, int layer, const uint16_t* qkv,
                            const AttnSeq* seqs, int n_seq, int max_chunks, int max_rows,
                            Partials part, cudaStream_t st);

// Merge the chunk partials of every (sequence, query token, q head) in chunk
// order into bf16 attention output rows.  mode 0 = draft layout (chunks of
// the quantised pool + one tail partial), 1 = dense layout.
cudaError_t attention_combine(const AttnShape& s, const AttnSeq* seqs, int n_seq, int max_chunks,
                              int max_rows, int mode, Partials part, uint16_t* out,
                              cudaStream_t st);

}  // namespace vc
