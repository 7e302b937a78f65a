// vc_dense_attn.cu -- attention over a bf16 KV pool: the verify pass (x+1
// query tokens per request, causal inside the draft window), the full-KV
// greedy-decode baseline (1 query token), and drafting over a token-dropped
// (compacted) cache.  One kernel serves all three so that verify logits are
// bit-identical to full-KV decode logits (the losslessness invariant):
//   * split-K over fixed 256-key chunks of ABSOLUTE positions,
//   * each warp owns one 16-row query tile and walks the chunk's keys in the
//     same 32-key order whatever the number of rows in the batch,
//   * partials are merged in chunk order by attention_combine.
// The row count therefore changes only how many warps a CTA has, never the
// arithmetic applied to a row (batch invariance).
//
// Tiles: K/V 32-key tiles staged by cp.async (3 stages, XOR-swizzled 16-B
// chunks), S = Q K^T and O = P V on mma.sync bf16 (ldmatrix / ldmatrix.trans
// fragments), online softmax in registers.  The verify charge in the
// reference is the request's full-KV bytes (/root/reference/proj/src/
// scheduler.cpp:366); verify returns x+1 predictions (specloop.cpp:24-35).
#include "vc_common.cuh"
#include "vc_kernels.h"
#include "vc_tiled.cuh"

namespace vc {
namespace {

constexpr int kChunk = VC_DENSE_CHUNK;
constexpr int kTile = 32;
constexpr int kStages = 3;
constexpr int kMaxParts = 512;  // chunks per sequence the combine can merge (256K ctx)

template <int D>
VC_DEV int swz(int row, int chunk16) {  // 16-B chunk index within a row
  return chunk16 ^ (row & 7);
}

template <int D, int NREP>
__global__ void __launch_bounds__(256, 2) dense_attn_kernel(AttnShape s, KvPool pool, int layer, const uint16_t* qkv,
                                  const AttnSeq* seqs, int max_chunks, int row_blocks,
                                  Partials part) {
  constexpr int KS = D / 16;       // k-steps over channels
  constexpr int NF = D / 8;        // n8 fragments of O
  constexpr int RB = D * 2;        // bytes per key row
  constexpr int C16 = RB / 16;     // 16-B chunks per key row
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sK = smem;                                  // [kStages][kTile][RB]
  uint8_t* sV = smem + kStages * kTile * RB;

  const AttnSeq sq = seqs[blockIdx.z / row_blocks];
  const int rblk = blockIdx.z % row_blocks;
  const int h = blockIdx.y;
  const int chunk = blockIdx.x;
  const int n_rows = sq.n_rows * NREP;                 // flattened (token, rep) rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int row_base = (rblk * nwarps) * 16;
  if (row_base >= n_rows) return;
  const int k_lo = chunk * kChunk;
  // keys visible to the last row of this CTA: kv_len - n_tok + tok + 1
  const int tok_last = min(n_rows - 1, row_base + nwarps * 16 - 1) / NREP;
  const int vis_last = sq.kv_len - sq.n_rows + tok_last + 1;
  if (k_lo >= vis_last) return;                        // no row of this CTA sees the chunk
  const int k_hi = min(k_lo + kChunk, vis_last);
  const int n_tiles = (k_hi - k_lo + kTile - 1) / kTile;

  const size_t slice = (static_cast<size_t>(sq.slot) * s.layers + layer) * s.n_kv + h;
  const uint16_t* Kg = pool.k + slice * static_cast<size_t>(pool.cap) * D;
  const uint16_t* Vg = pool.v + slice * static_cast<size_t>(pool.cap) * D;

  auto load_tile = [&](int t, int stage) {
    const int key0 = k_lo + t * kTile;
    for (int i = threadIdx.x; i < kTile * C16; i += blockDim.x) {
      const int r = i / C16, c = i % C16;
      const int key = key0 + r;
      const bool ok = key < k_hi;
      const size_t off = static_cast<size_t>(ok ? key : k_lo) * D + c * 8;
      uint8_t* dk = sK + (stage * kTile + r) * RB + swz<D>(r, c) * 16;
      uint8_t* dv = sV + (stage * kTile + r) * RB + swz<D>(r, c) * 16;
      cp_async16_zfill(dk, Kg + off, ok);
      cp_async16_zfill(dv, Vg + off, ok);
    }
  };

  // prologue: start the pipeline before touching Q
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < n_tiles) load_tile(st, st);
    cp_async_commit();
  }

  // This warp's 16 query rows staged in shared memory (swizzled like the K
  // tiles); A fragments are re-read with ldmatrix per k-step, which keeps the
  // register budget for the O accumulators.
  const int r0 = row_base + warp * 16 + (lane >> 2);
  const int r1 = r0 + 8;
  auto qptr = [&](int r) -> const uint16_t* {
    const int tok = r / NREP, rep = r % NREP;
    return qkv + static_cast<size_t>(sq.row0 + tok) * s.q_stride + static_cast<size_t>(h * NREP + rep) * D;
  };
  const bool v0 = r0 < n_rows, v1 = r1 < n_rows;
  uint8_t* sQw = smem + 2 * kStages * kTile * RB + warp * 16 * RB;
  for (int i = lane; i < 16 * C16; i += 32) {
    const int r = i / C16, c = i % C16;
    const int row = row_base + warp * 16 + r;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (row < n_rows) val = *reinterpret_cast<const uint4*>(qptr(row) + c * 8);
    *reinterpret_cast<uint4*>(sQw + r * RB + swz<D>(r, c) * 16) = val;
  }
  __syncwarp();
  // causal limits of this lane's two rows
  const int lim0 = sq.kv_len - sq.n_rows + (v0 ? r0 : 0) / NREP + 1;
  const int lim1 = sq.kv_len - sq.n_rows + (v1 ? r1 : 0) / NREP + 1;
  const bool warp_active = (row_base + warp * 16) < n_rows;

  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[NF][4];
#pragma unroll
  for (int f = 0; f < NF; ++f) o[f][0] = o[f][1] = o[f][2] = o[f][3] = 0.f;

  for (int t = 0; t < n_tiles; ++t) {
    const int nt = t + kStages - 1;
    if (nt < n_tiles) load_tile(nt, nt % kStages);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncthreads();
    const int stage = t % kStages;
    const uint8_t* tk = sK + stage * kTile * RB;
    const uint8_t* tv = sV + stage * kTile * RB;
    const int key0 = k_lo + t * kTile;
    if (warp_active) {
      // ---- S = Q K^T : 16 rows x 32 keys -------------------------------
      float sc[4][4];
#pragma unroll
      for (int nk = 0; nk < 4; ++nk) sc[nk][0] = sc[nk][1] = sc[nk][2] = sc[nk][3] = 0.f;
      // every S element accumulates its k-steps in order 0..KS-1
#pragma unroll
      for (int st = 0; st < KS; ++st) {
        uint32_t a[4];
        {
          const int r = (lane & 7) + ((lane >> 3) & 1) * 8;
          const int c = st * 2 + (lane >> 4);
          ldmatrix_x4(a[0], a[1], a[2], a[3], sQw + r * RB + swz<D>(r, c) * 16);
        }
#pragma unroll
        for (int nk = 0; nk < 4; nk += 2) {
          // x4: (keys nk*8.., ch lo), (.., ch hi), (keys (nk+1)*8.., ch lo), (.., ch hi)
          const int kr = nk * 8 + (lane & 7) + (lane >> 4) * 8;
          const int cc = st * 2 + ((lane >> 3) & 1);
          uint32_t b[4];
          ldmatrix_x4(b[0], b[1], b[2], b[3], tk + kr * RB + swz<D>(kr, cc) * 16);
          mma_bf16(sc[nk], a[0], a[1], a[2], a[3], b[0], b[1]);
          mma_bf16(sc[nk + 1], a[0], a[1], a[2], a[3], b[2], b[3]);
        }
      }
      // scale to log2 domain + causal / range mask
      const bool need_mask = (key0 + kTile > min(lim0, lim1)) || (key0 + kTile > k_hi);
      float tm0 = -INFINITY, tm1 = -INFINITY;
#pragma unroll
      for (int nk = 0; nk < 4; ++nk) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = sc[nk][e] * s.scale_log2;
          if (need_mask) {
            const int key = key0 + nk * 8 + 2 * (lane & 3) + (e & 1);
            const int lim = (e < 2) ? lim0 : lim1;
            if (key >= lim || key >= k_hi) v = -INFINITY;
          }
          sc[nk][e] = v;
        }
        tm0 = fmaxf(tm0, fmaxf(sc[nk][0], sc[nk][1]));
        tm1 = fmaxf(tm1, fmaxf(sc[nk][2], sc[nk][3]));
      }
      tm0 = fmaxf(tm0, __shfl_xor_sync(0xffffffffu, tm0, 1));
      tm0 = fmaxf(tm0, __shfl_xor_sync(0xffffffffu, tm0, 2));
      tm1 = fmaxf(tm1, __shfl_xor_sync(0xffffffffu, tm1, 1));
      tm1 = fmaxf(tm1, __shfl_xor_sync(0xffffffffu, tm1, 2));
      const float mn0 = fmaxf(m0, tm0), mn1 = fmaxf(m1, tm1);
      const float a0 = (mn0 == -INFINITY) ? 1.f : exp2f(m0 - mn0);
      const float a1 = (mn1 == -INFINITY) ? 1.f : exp2f(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      l0 *= a0;
      l1 *= a1;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        o[f][0] *= a0; o[f][1] *= a0; o[f][2] *= a1; o[f][3] *= a1;
      }
      uint32_t pa[2][4];
#pragma unroll
      for (int nk = 0; nk < 4; ++nk) {
        const float p0 = (mn0 == -INFINITY) ? 0.f : exp2f(sc[nk][0] - mn0);
        const float p1 = (mn0 == -INFINITY) ? 0.f : exp2f(sc[nk][1] - mn0);
        const float p2 = (mn1 == -INFINITY) ? 0.f : exp2f(sc[nk][2] - mn1);
        const float p3 = (mn1 == -INFINITY) ? 0.f : exp2f(sc[nk][3] - mn1);
        l0 += p0 + p1;
        l1 += p2 + p3;
        const int kk = nk >> 1, hi = nk & 1;
        pa[kk][hi ? 2 : 0] = pack_bf2(p0, p1);
        pa[kk][hi ? 3 : 1] = pack_bf2(p2, p3);
      }
      // ---- O += P V : 16 rows x D ---------------------------------------
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
        for (int f = 0; f < NF; f += 2) {
          // x4.trans: matrices (keys kk*16+0..7, ch f*8), (keys +8, ch f*8),
          //           (keys 0..7, ch (f+1)*8), (keys +8, ch (f+1)*8)
          const int mi = lane >> 3;
          const int kr = kk * 16 + (mi & 1) * 8 + (lane & 7);
          const int cc = f + (mi >> 1);
          uint32_t b[4];
          ldmatrix_x4_trans(b[0], b[1], b[2], b[3], tv + kr * RB + swz<D>(kr, cc) * 16);
          mma_bf16(o[f], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b[0], b[1]);
          mma_bf16(o[f + 1], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b[2], b[3]);
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  if (!warp_active) return;
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const int Hq = s.n_kv * NREP;
  auto emit = [&](int r, float m, float l, int which, int lim) {
    if (r >= n_rows || k_lo >= lim) return;  // row does not see this chunk
    const int tok = r / NREP, rep = r % NREP;
    const size_t prow = static_cast<size_t>(sq.part0 + chunk * sq.n_rows + tok) * Hq + h * NREP + rep;
    float* dst = part.o + prow * D;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int c = f * 8 + 2 * (lane & 3);
      dst[c] = o[f][which * 2 + 0];
      dst[c + 1] = o[f][which * 2 + 1];
    }
    if ((lane & 3) == 0) {
      part.ml[prow * 2] = m;
      part.ml[prow * 2 + 1] = l;
    }
  };
  emit(r0, m0, l0, 0, lim0);
  emit(r1, m1, l1, 1, lim1);
}

template <int D>
__global__ void combine_kernel(AttnShape s, const AttnSeq* seqs, int max_chunks, int mode,
                               Partials part, uint16_t* out) {
  const AttnSeq sq = seqs[blockIdx.x];
  const int tok = blockIdx.y;
  if (tok >= sq.n_rows) return;
  const int hq = blockIdx.z;
  const int Hq = s.n_kv * s.n_rep;
  int n_parts;
  if (mode == 0) {
    n_parts = (sq.n_groups + VC_DRAFT_CG - 1) / VC_DRAFT_CG;
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
  __shared__ float s_m[kMaxParts], s_f[kMaxParts];
  __shared__ size_t s_row[kMaxParts];
  __shared__ float s_M, s_l;
  for (int c = threadIdx.x; c < n_all; c += blockDim.x) {
    const size_t pr = prow_of(c < n_parts ? c : max_chunks + (c - n_parts));
    s_row[c] = pr;
    s_m[c] = part.ml[pr * 2];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY;
    for (int c = 0; c < n_all; ++c) M = fmaxf(M, s_m[c]);
    float l = 0.f;
    for (int c = 0; c < n_all; ++c) {  // fixed order
      const float f = (s_m[c] == -INFINITY) ? 0.f : exp2f(s_m[c] - M);
      s_f[c] = f;
      l += f * part.ml[s_row[c] * 2 + 1];
    }
    s_M = M;
    s_l = l;
  }
  __syncthreads();
  const float l = s_l;
  for (int c0 = threadIdx.x; c0 < D; c0 += blockDim.x) {
    float o = 0.f;
#pragma unroll 4
    for (int c = 0; c < n_all; ++c) o += s_f[c] * part.o[s_row[c] * D + c0];
    const uint16_t v = f2bf(l > 0.f ? o / l : 0.f);
    if (s.out_mp > 0)
      out[atile_idx(sq.row0 + tok, hq * D + c0, s.out_mp)] = v;
    else
      out[static_cast<size_t>(sq.row0 + tok) * s.out_stride + static_cast<size_t>(hq) * D + c0] = v;
  }
}

template <int D, int NREP>
cudaError_t launch_dense(const AttnShape& s, const KvPool& pool, int layer, const uint16_t* qkv,
                         const AttnSeq* seqs, int n_seq, int max_chunks, int max_rows,
                         Partials part, cudaStream_t st) {
  const int m_tiles = (max_rows * NREP + 15) / 16;
  const int warps = m_tiles < 8 ? m_tiles : 8;
  const int row_blocks = (m_tiles + warps - 1) / warps;
  const size_t smem = 2 * kStages * kTile * D * 2 + static_cast<size_t>(warps) * 16 * D * 2;  // + Q tiles
  auto kern = dense_attn_kernel<D, NREP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(max_chunks, s.n_kv, n_seq * row_blocks);
  kern<<<grid, warps * 32, smem, st>>>(s, pool, layer, qkv, seqs, max_chunks, row_blocks, part);
  return cudaGetLastError();
}

}  // namespace

cudaError_t dense_attention(const AttnShape& s, const KvPool& pool, int layer, const uint16_t* qkv,
                            const AttnSeq* seqs, int n_seq, int max_chunks, int max_rows,
                            Partials part, cudaStream_t st) {
  if (n_seq <= 0) return cudaSuccess;
  if (s.d == 128 && s.n_rep == 4) return launch_dense<128, 4>(s, pool, layer, qkv, seqs, n_seq, max_chunks, max_rows, part, st);
  if (s.d == 128 && s.n_rep == 8) return launch_dense<128, 8>(s, pool, layer, qkv, seqs, n_seq, max_chunks, max_rows, part, st);
  if (s.d == 64 && s.n_rep == 4) return launch_dense<64, 4>(s, pool, layer, qkv, seqs, n_seq, max_chunks, max_rows, part, st);
  return cudaErrorInvalidValue;
}

cudaError_t attention_combine(const AttnShape& s, const AttnSeq* seqs, int n_seq, int max_chunks,
                              int max_rows, int mode, Partials part, uint16_t* out,
                              cudaStream_t st) {
  if (n_seq <= 0) return cudaSuccess;
  dim3 grid(n_seq, max_rows, s.n_kv * s.n_rep);
  if (s.d == 128) combine_kernel<128><<<grid, 128, 0, st>>>(s, seqs, max_chunks, mode, part, out);
  else if (s.d == 64) combine_kernel<64><<<grid, 64, 0, st>>>(s, seqs, max_chunks, mode, part, out);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace vc
