// vc_dense_umma.cu -- attention over a bf16 KV pool on the 5th-gen tensor
// cores: the verify pass (x+1 query tokens per request, causal inside the
// draft window), the full-KV greedy-decode baseline (1 query token), and
// drafting over a token-dropped (compacted) cache.  One kernel serves all
// three so that verify logits are bit-identical to full-KV decode logits (the
// losslessness invariant):
//   * split-K over fixed VC_DENSE_CHUNK-key chunks of ABSOLUTE positions,
//     merged in chunk order by attention_combine;
//   * an item = (sequence, query block of <= 96 (token, rep) rows, kv head,
//     chunk); every per-row decision (causal limit, running max, lazy
//     rescale) depends on that row's scores only, so the arithmetic applied
//     to a row never depends on the other rows of the batch.
//
// Orientation: keys are the MMA M dimension (128 TMEM lanes) and the query
// rows the N dimension (16..96 columns), so the decode/verify row counts
// (4..136) cost N, not a padded M=128, and the softmax spreads over all 128
// threads (one key each) whatever the row count:
//   S^T[key, row] = K[key, :] . Q[row, :]          (SS, both K-major)
//   P^T = 2^(S^T * scale - m[row])  -> shared memory (bf16, MN-major)
//   O^T[ch, row] += V^T[ch, key] . P^T[key, row]    (SS, V^T MN-major)
//   L[., row]    += 1[., key] . P^T[key, row]       (row sums on the MMA)
// Warp roles on one CTA per SM (persistent, items round-robin over CTAs):
//   warp 0  TMA producer (Q block: 3-D map over the qkv rows; K/V tiles:
//           2-D maps over the pool; 128B swizzle; two K/V stages)
//   warp 1  MMA issuer (one thread) and TMEM owner
//   warps 2-5  softmax (thread = key) and epilogue (thread = channel).
// Running max: a row's max is refreshed (exactly, by a warp transpose-reduce)
// only on an item's first tile or when a score exceeds it by more than 2^kTau;
// only rows whose max moved are rescaled (alpha = 1 leaves a row bit-exact).
// The verify charge in the reference is the request's full-KV bytes
// (/root/reference/proj/src/scheduler.cpp:366); verify returns x+1
// predictions (specloop.cpp:24-35).
#include <cudaTypedefs.h>

#include "vc_common.cuh"
#include "vc_kernels.h"
#include "vc_umma.cuh"

namespace vc {
namespace {

constexpr int kTile = 128;            // keys per tile (MMA M)
constexpr int kRows = 80;             // query rows per item (MMA N <= 80: 6 TMEM buffers fit 512 cols)
constexpr int kChunk = VC_DENSE_CHUNK;
#ifndef VC_DENSE_TAU
#define VC_DENSE_TAU 12.0f  // r1: 12 vs 8 = -1.2% per mixed step, 4 = +6%; bf16 P and fp32 sums keep 2^12 exact in range
#endif
constexpr float kTau = VC_DENSE_TAU;  // lazy rescale threshold (log2 units)
// producer(Q,K) | MMA | 2 x 4 softmax warps (two column groups) | producer(V)
constexpr int kSoftGroups = 2;
constexpr int kThreads = 32 * (3 + 4 * kSoftGroups);
constexpr int kWarpV = 2 + 4 * kSoftGroups;
static_assert(kChunk % kTile == 0, "chunks are whole tiles");

struct Item {
  int seq, rb, h, chunk;
  int row0, n_tok, kv_len, slot, part0;
  int k_lo, k_hi, n_tiles;
};

template <int NREP>
VC_DEV bool decode_item(int it, const AttnShape& s, const AttnSeq* seqs, int max_chunks, int row_blocks,
                        Item& I) {
  // row block innermost: the row blocks of one (sequence, head, chunk) run on
  // neighbouring CTAs at the same time, so a long verify window's K/V chunk
  // is fetched from HBM once and re-read from L2 by the other row blocks
  I.rb = it % row_blocks;
  int r = it / row_blocks;
  I.chunk = r % max_chunks;
  r /= max_chunks;
  I.h = r % s.n_kv;
  I.seq = r / s.n_kv;
  const AttnSeq sq = seqs[I.seq];
  const int rows = sq.n_rows * NREP;
  const int row_base = I.rb * kRows;
  if (row_base >= rows) return false;
  I.k_lo = I.chunk * kChunk;
  const int tok_last = min(rows - 1, row_base + kRows - 1) / NREP;
  const int vis_last = sq.kv_len - sq.n_rows + tok_last + 1;
  if (I.k_lo >= vis_last) return false;
  I.k_hi = min(I.k_lo + kChunk, vis_last);
  I.n_tiles = (I.k_hi - I.k_lo + kTile - 1) / kTile;
  I.row0 = sq.row0;
  I.n_tok = sq.n_rows;
  I.kv_len = sq.kv_len;
  I.slot = sq.slot;
  I.part0 = sq.part0;
  return true;
}

VC_DEV void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

VC_DEV bool bar_or(int id, int count, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %1, 0;\n\tbarrier.red.or.pred p, %2, %3, q;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(v)), "r"(id), "r"(count)
      : "memory");
  return r != 0;
}

// Column maxima of a 32-key x 32-column block held one key per lane:
// transpose-reduce so lane j ends with the max of column j (31 shuffles).
VC_DEV float warp_colmax(float* v, int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = lane & off;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const float send = upper ? v[i] : v[i + off];
      const float keep = upper ? v[i + off] : v[i];
      v[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, off));
    }
  }
  return v[0];
}

VC_DEV void st_shared_v4(void* p, const uint32_t* v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(smem_u32(p)), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3])
               : "memory");
}

// SW128 MN-major byte offset of element (k = key row, n = column) in a
// [128 keys x 64-column atoms] operand (atoms 16 KB apart).
VC_DEV uint32_t mn_sw128_off(int k, int n) {
  return (n >> 6) * (kTile * 128) + (k >> 3) * 1024 + (k & 7) * 128 + ((((n & 63) >> 3) ^ (k & 7)) << 4) +
         (n & 7) * 2;
}

template <int D, int NREP>
__global__ void __launch_bounds__(kThreads, 1)
    dense_umma_kernel(const __grid_constant__ DenseMaps maps, AttnShape s, int layer, int pool_cap,
                      const AttnSeq* seqs, int n_seq, int max_chunks, int row_blocks, Partials part) {
  constexpr int ATOMS = D / 64;                 // 128-B swizzle atoms per K/V/Q row
  constexpr int KV_BYTES = kTile * D * 2;       // one K or V tile
  constexpr int KV_ATOM = kTile * 128;          // one atom column of a K/V tile
  constexpr int Q_ATOM = kRows * 128;           // one atom column of the Q block
  constexpr int Q_BYTES = Q_ATOM * ATOMS;
  constexpr int P_BYTES = 2 * KV_ATOM;          // P^T: 128 keys x 2 atoms of 64 columns
  constexpr int KS = D / 16;                    // k-steps of S^T (over channels)
  // TMEM columns: S^T x2 (per tile), O^T x2 and L x2 (per item, so an item's
  // epilogue overlaps the next item's first tiles)
  constexpr uint32_t kColS0 = 0, kColS1 = kRows, kColO = 2 * kRows, kColL = 4 * kRows;
  static_assert(kRows % NREP == 0 && kRows <= 128, "query block");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;                           // [2][KV_BYTES]
  uint8_t* sV = sK + 2 * KV_BYTES;              // [2][KV_BYTES]
  uint8_t* sP = sV + 2 * KV_BYTES;              // [2][P_BYTES]
  uint8_t* sQ = sP + 2 * P_BYTES;               // [Q_BYTES]
  uint8_t* sOnes = sQ + Q_BYTES;                // 128 x 16 bf16 ones, no swizzle (4 KB)
  __shared__ __align__(8) uint64_t q_full, q_empty, k_full[2], v_full[2], k_empty[2], v_empty[2];
  __shared__ __align__(8) uint64_t s_full[2], s_empty[2], p_full[2], o_full[2], o_empty[2];
  __shared__ uint32_t tmem_base_sh;
  // per softmax group: the groups' column ranges move with each item's width,
  // and a group may still run an older item's epilogue while the other starts
  // the next item, so each group keeps its own per-column state
  __shared__ __align__(16) float m_run3[kSoftGroups][2][kRows];
  __shared__ __align__(16) float alpha_g[kSoftGroups][kRows], l_g[kSoftGroups][kRows];
  __shared__ float wmax_g[kSoftGroups][4][kRows];
  __shared__ __align__(16) int lim_g[kSoftGroups][kRows];   // keys < lim_col[row] are visible to the item's row

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = n_seq * row_blocks * s.n_kv * max_chunks;
  pdl_trigger();

  if (threadIdx.x == 0) {
    mbar_init(&q_full, 1);
    mbar_init(&q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 1);
      mbar_init(&p_full[i], 4 * kSoftGroups);
    }
    mbar_init(&o_full[0], 1);
    mbar_init(&o_full[1], 1);
    mbar_init(&o_empty[0], 4 * kSoftGroups);
    mbar_init(&o_empty[1], 4 * kSoftGroups);
    fence_mbar_init();
    tma_prefetch_desc(&maps.q);
    tma_prefetch_desc(&maps.k);
    tma_prefetch_desc(&maps.v);
  }
  for (int i = threadIdx.x; i < 4096 / 16; i += kThreads)  // bf16 1.0 = 0x3F80
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  fence_proxy_async();
  if (warp == 1) tmem_alloc(&tmem_base_sh, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tmem_base_sh;
  // PDL prologue: the first item's K/V tiles lie before this step's new rows
  // (positions < kv_len - n_tok: not written by the qkv epilogue we depend on,
  // nor by anything else in flight), so the producers stream its first two
  // stages while the previous kernel drains, then wait for it
  int first_static = 0;  // K/V tiles of the CTA's first item issued before the wait
  Item I0;
  const bool have0 = n_items > 0 && decode_item<NREP>(blockIdx.x, s, seqs, max_chunks, row_blocks, I0);
  if (have0 && I0.k_hi <= I0.kv_len - I0.n_tok) first_static = I0.n_tiles < 2 ? I0.n_tiles : 2;
  if (warp != 0 && warp != 6) pdl_wait();  // q rows and the window's new K/V come from the qkv epilogue

  // one pool tile (K or V) of item I, tile t, into stage st.  With one row
  // block per window nothing re-reads a tile, so it streams through L2
  // evict-first; wider windows' row blocks re-read it from L2 (normal policy)
  const uint64_t kv_pol = l2_policy_evict_first();
  auto load_kv = [&](const CUtensorMap* map, uint8_t* dst, uint64_t* bar, const Item& I, int t) {
    const int slice_row = static_cast<int>(((static_cast<size_t>(I.slot) * s.layers + layer) * s.n_kv + I.h) *
                                           static_cast<size_t>(pool_cap));
    mbar_expect_tx(bar, KV_BYTES);
    if (row_blocks == 1) {
#pragma unroll
      for (int a = 0; a < ATOMS; ++a)
        tma_load_2d_hint(dst + a * KV_ATOM, map, a * 64, slice_row + I.k_lo + t * kTile, bar, kv_pol);
    } else {
#pragma unroll
      for (int a = 0; a < ATOMS; ++a) tma_load_2d(dst + a * KV_ATOM, map, a * 64, slice_row + I.k_lo + t * kTile, bar);
    }
  };
  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0)
      for (int t = 0; t < first_static; ++t) load_kv(&maps.k, sK + t * KV_BYTES, &k_full[t], I0, t);
    pdl_wait();
    if (lane == 0) {
      int g = 0, n = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        Item I;
        if (!decode_item<NREP>(it, s, seqs, max_chunks, row_blocks, I)) continue;
        if (n >= 1) mbar_wait(&q_empty, (n - 1) & 1);
        mbar_expect_tx(&q_full, Q_BYTES);
#pragma unroll
        for (int a = 0; a < ATOMS; ++a)
          tma_load_3d(sQ + a * Q_ATOM, &maps.q, a * 64, I.h * NREP, I.row0 + I.rb * (kRows / NREP), &q_full);
        for (int t = 0; t < I.n_tiles; ++t, ++g) {
          if (n == 0 && t < first_static) continue;  // issued before the wait
          const int st = g & 1;
          if (g >= 2) mbar_wait(&k_empty[st], ((g >> 1) - 1) & 1);  // S(g-2) done with the stage
          load_kv(&maps.k, sK + st * KV_BYTES, &k_full[st], I, t);
        }
        ++n;
      }
    }
  } else if (warp == kWarpV) {
    // ===================== TMA producer: V (runs behind K by the softmax) =====================
    if (lane == 0)
      for (int t = 0; t < first_static; ++t) load_kv(&maps.v, sV + t * KV_BYTES, &v_full[t], I0, t);
    pdl_wait();
    if (lane == 0) {
      int g = 0, n = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        Item I;
        if (!decode_item<NREP>(it, s, seqs, max_chunks, row_blocks, I)) continue;
        for (int t = 0; t < I.n_tiles; ++t, ++g) {
          if (n == 0 && t < first_static) continue;
          const int st = g & 1;
          if (g >= 2) mbar_wait(&v_empty[st], ((g >> 1) - 1) & 1);  // PV(g-2) done with the stage
          load_kv(&maps.v, sV + st * KV_BYTES, &v_full[st], I, t);
        }
        ++n;
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int g = 0, n = 0;
      int pend = -1, pend_item = 0;
      bool pend_first = false, pend_last = false;
      uint32_t pend_n = 16;
      const uint64_t ones_desc = [&] {  // SWIZZLE_NONE K-major: 8x16B core matrices, LBO 128 (K), SBO 256 (M)
        uint64_t d = static_cast<uint64_t>((smem_u32(sOnes) & 0x3FFFFu) >> 4);
        d |= static_cast<uint64_t>(128 >> 4) << 16;
        d |= static_cast<uint64_t>(256 >> 4) << 32;
        d |= 1ull << 46;
        return d;
      }();
      auto issue_pv = [&]() {
        const int sb = pend & 1;
        const int ob = pend_item & 1;
        if (pend_first && pend_item >= 2) mbar_wait(&o_empty[ob], ((pend_item >> 1) - 1) & 1);
        mbar_wait(&p_full[sb], (pend >> 1) & 1);
        mbar_wait(&v_full[sb], (pend >> 1) & 1);
        tmem_fence_after();
        const uint32_t vbase = smem_u32(sV + sb * KV_BYTES);
        const uint32_t pbase = smem_u32(sP + sb * P_BYTES);
        // A = V^T MN-major, always M = 128 lanes (for d = 64 the upper lanes are ignored)
        const uint32_t idO = umma_idesc_bf16(128, pend_n, true) | (1u << 15);
        const uint32_t idL = umma_idesc_bf16(128, pend_n, true);               // A = ones (K-major)
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk) {
          const uint64_t bp = umma_sdesc_sw128(pbase + kk * 2048, KV_ATOM, 1024);
          const bool acc = !(pend_first && kk == 0);
          umma_ss(tbase + kColO + ob * kRows, umma_sdesc_sw128(vbase + kk * 2048, KV_ATOM, 1024), bp, idO, acc);
          umma_ss(tbase + kColL + ob * kRows, ones_desc, bp, idL, acc);
        }
        umma_commit(&v_empty[sb]);
        umma_commit(&s_empty[sb]);
        if (pend_last) umma_commit(&o_full[ob]);
      };
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        Item I;
        if (!decode_item<NREP>(it, s, seqs, max_chunks, row_blocks, I)) continue;
        const int rows = min(kRows, I.n_tok * NREP - I.rb * kRows);
        const uint32_t npad = static_cast<uint32_t>((rows + 15) & ~15);
        const uint32_t idS = umma_idesc_bf16(kTile, npad, false);
        mbar_wait(&q_full, n & 1);
        tmem_fence_after();
        const uint32_t qbase = smem_u32(sQ);
        for (int t = 0; t < I.n_tiles; ++t, ++g) {
          const int sb = g & 1;
          if (g >= 2) mbar_wait(&s_empty[sb], ((g >> 1) - 1) & 1);
          mbar_wait(&k_full[sb], (g >> 1) & 1);
          tmem_fence_after();
          const uint32_t kbase = smem_u32(sK + sb * KV_BYTES);
#pragma unroll
          for (int kk = 0; kk < KS; ++kk)
            umma_ss(tbase + (sb ? kColS1 : kColS0),
                    umma_sdesc_sw128(kbase + (kk >> 2) * KV_ATOM + (kk & 3) * 32, 16, 1024),
                    umma_sdesc_sw128(qbase + (kk >> 2) * Q_ATOM + (kk & 3) * 32, 16, 1024), idS, kk > 0);
          umma_commit(&s_full[sb]);
          umma_commit(&k_empty[sb]);
          if (t == I.n_tiles - 1) umma_commit(&q_empty);
          if (pend >= 0) issue_pv();
          pend = g;
          pend_item = n;
          pend_first = t == 0;
          pend_last = t == I.n_tiles - 1;
          pend_n = npad;
        }
        ++n;
      }
      if (pend >= 0) issue_pv();
    }
  } else {
    // ===================== softmax (thread = key) + epilogue (thread = channel) =====================
    // two groups of 4 warps: group g owns the query columns [c_lo, c_hi) of
    // every item (16-column granules, group 0 takes the odd one), so a wide
    // verify window's softmax runs on twice the threads; rows are independent,
    // so each group keeps its own barrier and its own lazy-rescale vote
    const int quarter = warp & 3;
    const int grp = (warp - 2) / 4;
    const int gbar = 1 + grp;                             // the group's named barrier
    const int tid = quarter * 32 + lane;                 // key within the tile / channel / row index
    const uint32_t tlane = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
    const int Hq = s.n_kv * NREP;
    float(*m_run2)[kRows] = m_run3[grp];
    float* alpha_sh = alpha_g[grp];
    float* l_sh = l_g[grp];
    float(*wmax)[kRows] = wmax_g[grp];
    int* lim_col = lim_g[grp];
    auto col_range = [&](int npad, int& lo, int& hi) {
      const int half = ((npad >> 4) + 1) >> 1;
      lo = grp == 0 ? 0 : half * 16;
      hi = grp == 0 ? half * 16 : npad;
    };
    // columns [c_lo, c_hi) of a per-item TMEM buffer scaled by alpha_sh (16-column steps)
    auto rescale = [&](uint32_t col0, int c_lo, int c_hi) {
      for (int c = c_lo; c < c_hi; c += 16) {
        uint32_t v[16];
        tmem_ld16(tlane + col0 + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha_sh[c + j]);
        tmem_st16(tlane + col0 + c, v);
      }
    };
    // item ni's (m, l, O) partials: O^T column = query row, lane = channel
    auto epilogue = [&](const Item& I, int ni) {
      const int ob = ni & 1;
      const float* m_run = m_run2[ob];
      const int rows = min(kRows, I.n_tok * NREP - I.rb * kRows);
      const int npad = (rows + 15) & ~15;
      int c_lo, c_hi;
      col_range(npad, c_lo, c_hi);
      mbar_wait(&o_full[ob], (ni >> 1) & 1);
      tmem_fence_after();
      if (quarter == 0) {  // L: every lane holds the same row sums; lane 0's are used
        for (int c = c_lo; c < c_hi; c += 16) {
          uint32_t v[16];
          tmem_ld16(tlane + kColL + ob * kRows + c, v);
          tmem_wait_ld();
          if (lane == 0)
#pragma unroll
            for (int j = 0; j < 16; ++j) l_sh[c + j] = __uint_as_float(v[j]);
        }
      }
      named_bar(gbar, 128);
      for (int c = c_lo; c < c_hi; c += 16) {
        uint32_t v[16];
        tmem_ld16(tlane + kColO + ob * kRows + c, v);
        tmem_wait_ld();
        if (tid < D) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c + j;
            if (col >= rows) break;
            const int r = I.rb * kRows + col;
            const int tok = r / NREP, rep = r % NREP;
            if (I.k_lo >= I.kv_len - I.n_tok + tok + 1) continue;  // row does not see this chunk
            const size_t prow = static_cast<size_t>(I.part0 + I.chunk * I.n_tok + tok) * Hq + I.h * NREP + rep;
            part.o[prow * D + tid] = __uint_as_float(v[j]);
          }
        }
      }
      if (tid >= c_lo && tid < c_hi && tid < rows) {
        const int r = I.rb * kRows + tid;
        const int tok = r / NREP, rep = r % NREP;
        if (I.k_lo < I.kv_len - I.n_tok + tok + 1) {
          const size_t prow = static_cast<size_t>(I.part0 + I.chunk * I.n_tok + tok) * Hq + I.h * NREP + rep;
          part.ml[prow * 2] = m_run[tid];
          part.ml[prow * 2 + 1] = l_sh[tid];
        }
      }
      tmem_fence_before();
      named_bar(gbar, 128);  // l_sh reads done before the next epilogue refills it
      if (lane == 0) mbar_arrive(&o_empty[ob]);
    };
    int g = 0, n = 0;
    Item prev{};
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      Item I;
      if (!decode_item<NREP>(it, s, seqs, max_chunks, row_blocks, I)) continue;
      const int ob = n & 1;
      float* m_run = m_run2[ob];
      const int rows = min(kRows, I.n_tok * NREP - I.rb * kRows);
      const int npad = (rows + 15) & ~15;
      int c_lo, c_hi;
      col_range(npad, c_lo, c_hi);
      // per-row visibility limit (absolute key) inside this chunk; padding rows see nothing
      if (tid >= c_lo && tid < c_hi) {
        const int tok = (I.rb * kRows + tid) / NREP;
        lim_col[tid] = tid < rows ? min(I.k_hi, I.kv_len - I.n_tok + tok + 1) : I.k_lo;
        // padding columns: m = +inf makes every P 0 and keeps them out of the max
        m_run[tid] = tid < rows ? -INFINITY : INFINITY;
      }
      const int tok_first = (I.rb * kRows) / NREP;
      const int lim_min = min(I.k_hi, I.kv_len - I.n_tok + tok_first + 1);   // earliest row's limit
      named_bar(gbar, 128);
      for (int t = 0; t < I.n_tiles; ++t, ++g) {
        const int sb = g & 1;
        const int key0 = I.k_lo + t * kTile;
        const int key = key0 + tid;
        const bool masked_tile = key0 + kTile > lim_min;   // some (row, key) of the tile is invisible
        mbar_wait(&s_full[sb], (g >> 1) & 1);
        tmem_fence_after();
        const uint32_t tS = tlane + (sb ? kColS1 : kColS0);
        uint8_t* pdst = sP + sb * P_BYTES;
        // 16 columns of P from S values v (TMEM already waited on)
        auto p16 = [&](const uint32_t* v, int c, bool track, float& over) {
#pragma unroll
          for (int j8 = 0; j8 < 16; j8 += 8) {
            uint32_t pk[4];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              const int col = c + j8 + j;
              const float2 m = *reinterpret_cast<const float2*>(m_run + col);
              float x0 = __uint_as_float(v[j8 + j]) * s.scale_log2 - m.x;
              float x1 = __uint_as_float(v[j8 + j + 1]) * s.scale_log2 - m.y;
              if (masked_tile) {
                const int2 lm = *reinterpret_cast<const int2*>(lim_col + col);
                if (key >= lm.x) x0 = -INFINITY;
                if (key >= lm.y) x1 = -INFINITY;
              }
              if (track) over = fmaxf(over, fmaxf(x0, x1));
              pk[j >> 1] = pack_bf2(ex2(x0), ex2(x1));
            }
            st_shared_v4(pdst + mn_sw128_off(tid, c + j8), pk);
          }
        };
        // 32 columns per TMEM load + wait where they fit (fewer serialised waits)
        auto write_p = [&](bool track, float& over) {
          int c = c_lo;
          for (; c + 32 <= c_hi; c += 32) {
            uint32_t v[32];
            tmem_ld32(tS + c, v);
            tmem_wait_ld();
            p16(v, c, track, over);
            p16(v + 16, c + 16, track, over);
          }
          if (c < c_hi) {
            uint32_t v[16];
            tmem_ld16(tS + c, v);
            tmem_wait_ld();
            p16(v, c, track, over);
          }
        };
        // optimistic pass: P with the running max; note how far any score overshoots it
        float over = -INFINITY;
        if (t > 0) write_p(true, over);
        const bool refresh = c_hi > c_lo && bar_or(gbar, 128, t == 0 || over > kTau);
        if (refresh) {
          // exact per-row tile max (warp transpose-reduce, then across the 4 warps)
          for (int c = c_lo; c < c_hi; c += 32) {
            uint32_t v[32];
            tmem_ld32(tS + c, v);   // may read past npad: those columns are discarded
            tmem_wait_ld();
            float x[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = min(c + j, kRows - 1);
              x[j] = (c + j < rows && key < lim_col[col]) ? __uint_as_float(v[j]) * s.scale_log2 : -INFINITY;
            }
            const float cm = warp_colmax(x, lane);
            if (c + lane < c_hi) wmax[quarter][c + lane] = cm;
          }
          named_bar(gbar, 128);
          bool grew = false;
          if (tid >= c_lo && tid < c_hi && tid < rows) {
            const float mt = fmaxf(fmaxf(wmax[0][tid], wmax[1][tid]), fmaxf(wmax[2][tid], wmax[3][tid]));
            const float mo = m_run[tid];
            const float mn = fmaxf(mo, mt);
            grew = mn > mo + kTau || (mo == -INFINITY && mn != -INFINITY);
            alpha_sh[tid] = grew ? ex2(mo - mn) : 1.f;
            if (grew) m_run[tid] = mn;
          } else if (tid >= c_lo && tid < c_hi) {
            alpha_sh[tid] = 1.f;
          }
          const bool any_grew = bar_or(gbar, 128, grew && t > 0);
          if (any_grew) {
            // O^T / L hold tiles < t: wait for PV(t-1), scale the columns of the rows that moved
            mbar_wait(&s_empty[(g - 1) & 1], ((g - 1) >> 1) & 1);
            tmem_fence_after();
            rescale(kColO + ob * kRows, c_lo, c_hi);
            rescale(kColL + ob * kRows, c_lo, c_hi);
            tmem_wait_st();
          }
          write_p(false, over);  // P again with the refreshed maxima
        }
        fence_proxy_async();  // P^T st.shared -> visible to the tensor core (async proxy)
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        // the previous item's epilogue runs once this item's first P is out
        if (t == 0 && n > 0) epilogue(prev, n - 1);
      }
      prev = I;
      ++n;
    }
    if (n > 0) epilogue(prev, n - 1);
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

template <int D, int NREP>
cudaError_t launch_umma(const DenseMaps& maps, const AttnShape& s, int layer, int pool_cap, const AttnSeq* seqs,
                        int n_seq, int max_chunks, int max_rows, Partials part, cudaStream_t st) {
  const int row_blocks = (max_rows * NREP + kRows - 1) / kRows;
  const int n_items = n_seq * row_blocks * s.n_kv * max_chunks;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // K, V (2 stages each), P^T (2 buffers), Q block, ones tile, alignment slack
  const size_t smem = 4 * static_cast<size_t>(kTile) * D * 2 + 2 * 2 * kTile * 128 +
                      static_cast<size_t>(kRows) * D * 2 + 4096 + 1024;
  auto kern = dense_umma_kernel<D, NREP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = n_items < sms ? n_items : sms;
  if (grid <= 0) return cudaSuccess;
  return launch_pdl(kern, dim3(grid), dim3(kThreads), smem, st, maps, s, layer, pool_cap, seqs, n_seq, max_chunks,
                    row_blocks, part);
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  return fn;
}

}  // namespace

bool make_kv_maps(DenseMaps* m, const KvPool& pool, size_t slices, int d) {
  auto enc = encoder();
  if (!enc || (d != 64 && d != 128)) return false;
  const size_t rows = slices * static_cast<size_t>(pool.cap);
  if (rows >= (1ull << 31)) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 2};
  cuuint32_t box[2] = {64, kTile};
  cuuint32_t es[2] = {1, 1};
  for (int i = 0; i < 2; ++i) {
    CUresult r = enc(i ? &m->v : &m->k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, i ? pool.v : pool.k, dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
  }
  return true;
}

bool make_q_map(DenseMaps* m, const uint16_t* qkv, int d, int heads_per_row, int rows, int q_stride, int n_rep) {
  auto enc = encoder();
  if (!enc || (d != 64 && d != 128) || kRows % n_rep) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(heads_per_row),
                        static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 2, static_cast<cuuint64_t>(q_stride) * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(n_rep), static_cast<cuuint32_t>(kRows / n_rep)};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(&m->q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(qkv), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t dense_attention(const AttnShape& s, const KvPool& pool, const DenseMaps& maps, int layer,
                            const AttnSeq* seqs, int n_seq, int max_chunks, int max_rows, Partials part,
                            cudaStream_t st) {
  if (n_seq <= 0) return cudaSuccess;
  if (s.d == 128 && s.n_rep == 4) return launch_umma<128, 4>(maps, s, layer, pool.cap, seqs, n_seq, max_chunks, max_rows, part, st);
  if (s.d == 128 && s.n_rep == 8) return launch_umma<128, 8>(maps, s, layer, pool.cap, seqs, n_seq, max_chunks, max_rows, part, st);
  if (s.d == 64 && s.n_rep == 4) return launch_umma<64, 4>(maps, s, layer, pool.cap, seqs, n_seq, max_chunks, max_rows, part, st);
  return cudaErrorInvalidValue;
}

}  // namespace vc
