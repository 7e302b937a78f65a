// vc_pack.cu -- lossless packing of the host tier's bf16 KV (chunk ring).
//
// A verify of an offloaded request is bound by the PCIe link (every reload
// moves the request's full KV), so the host pool stores each 128-token block
// of a (layer, kv-head) slice -- K and V separately -- in a lossless packed
// form that moves ~0.71 of the bytes (n = 128 * d values, value v = t*d + c):
//   e_base[c]       the largest bf16 exponent of channel c over the block's tokens
//   code[v]         2 bits: the exponent offset e_base[c] - exponent when it is
//                   1, 2 or 3 (77% of the values of a bell-shaped channel), else
//                   0 = the offset is in the secondary stream
//   sm[v]           8 bits: sign | 7 mantissa bits
//   n_sec, sec[]    4-bit offsets 0..14 of the values coded 0, in value order
//                   (15 = escape), at most packed_sec_cap(d) of them (0.28 n;
//                   0.23-0.24 n is typical, 0.256 the largest of 256 Gaussian
//                   blocks)
//   n_esc, esc[]    values whose exponent lies more than 14 below the channel's
//                   maximum (zeros, denormals, tiny values): (v << 16) | raw bf16
// So a typical value costs 2 + 8 + ~1 bits (the exponent offsets' entropy is
// ~2.5 bits; the previous format spent a flat 4, 0.76 of raw).  K's
// per-channel magnitude structure (outlier channels) is why the exponent base
// is per channel, not per token.  A block with more than kPackEscCap escapes
// or a full secondary stream does not pack (the overflow flag): the engine
// stores it raw.  Each thread owns VPT = d/2 consecutive values of one token
// row; a block-wide scan over the threads' secondary counts places the
// secondary offsets (pack) and finds them again (unpack).  Decoding restores
// the bf16 bits exactly (tests/test_stream_ring.py checks the round trip and
// the streamed verify bit for bit).
#include "vc_common.cuh"
#include "vc_gemm.h"

namespace vc {
namespace {

constexpr int kTok = 128;  // tokens per packed block (= VC_QGROUP)
constexpr int kThreads = 256;

template <int D>
struct PackGeo {
  static constexpr int N = kTok * D;          // values per block
  static constexpr int VPT = N / kThreads;    // values per thread (one token row's d/2 channels)
  static constexpr int SEC = packed_sec_cap(D);
  static constexpr size_t OFF_C2 = D, OFF_SM = D + N / 4, OFF_NS = OFF_SM + N, OFF_SEC = OFF_NS + 4,
                          OFF_NE = OFF_SEC + SEC / 2, OFF_ESC = OFF_NE + 4;
  static_assert(VPT % 16 == 0 && D % VPT == 0 && OFF_NE % 4 == 0, "pack geometry");
  static_assert(OFF_ESC + 4 * kPackEscCap <= packed_block_bytes(D), "pack size");
};

// n consecutive u32 through 16-byte accesses when n % 4 == 0 (a thread's
// segment is 16-byte aligned), else 8-byte ones: one warp instruction moves a
// 512-byte span instead of 32 strided words (the u32 version ran the unpack at
// 80% of L1 throughput)
template <int n>
VC_DEV void ld_words(const uint32_t* p, uint32_t* w) {
  if constexpr (n % 4 == 0) {
#pragma unroll
    for (int i = 0; i < n / 4; ++i) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[i];
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
  } else {
    static_assert(n % 2 == 0, "pairs");
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const uint2 v = reinterpret_cast<const uint2*>(p)[i];
      w[2 * i] = v.x; w[2 * i + 1] = v.y;
    }
  }
}
template <int n>
VC_DEV void st_words(uint32_t* p, const uint32_t* w) {
  if constexpr (n % 4 == 0) {
#pragma unroll
    for (int i = 0; i < n / 4; ++i) reinterpret_cast<uint4*>(p)[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
  } else {
    static_assert(n % 2 == 0, "pairs");
#pragma unroll
    for (int i = 0; i < n / 2; ++i) reinterpret_cast<uint2*>(p)[i] = make_uint2(w[2 * i], w[2 * i + 1]);
  }
}

// exclusive prefix of v over the block's 256 threads (thread order); *total = the sum
VC_DEV int block_scan256(int v, int* ws, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) {
    const int w = ws[i];
    pre += i < warp ? w : 0;
    tot += w;
  }
  __syncthreads();  // ws is reused by the next scan
  *total = tot;
  return pre + x - v;
}

template <int D>
__global__ void __launch_bounds__(kThreads) pack_kernel(const uint16_t* src, size_t src_slice_pitch, int src_row0,
                                                         int n_valid, int n_blocks, uint8_t* dst,
                                                         size_t dst_slice_pitch, int* overflow) {
  using G = PackGeo<D>;
  constexpr int VPT = G::VPT;
  const int b = blockIdx.x, sl = blockIdx.y;
  const uint16_t* s = src + sl * src_slice_pitch + static_cast<size_t>(src_row0 + b * kTok) * D;
  uint8_t* o = dst + sl * dst_slice_pitch + static_cast<size_t>(b) * packed_block_bytes(D);
  const int rows = min(kTok, n_valid - b * kTok);  // valid tokens of this block
  __shared__ uint8_t e_base[D];
  __shared__ uint32_t secw[G::SEC / 8];
  __shared__ int ws[kThreads / 32];
  __shared__ int n_esc;
  if (threadIdx.x == 0) n_esc = 0;
  for (int i = threadIdx.x; i < G::SEC / 8; i += kThreads) secw[i] = 0;
  for (int c = threadIdx.x; c < D; c += kThreads) {
    int m = 0;
    for (int t = 0; t < rows; ++t) m = max(m, (s[static_cast<size_t>(t) * D + c] >> 7) & 0xff);
    e_base[c] = static_cast<uint8_t>(m);
    o[c] = static_cast<uint8_t>(m);
  }
  __syncthreads();
  const int v0 = threadIdx.x * VPT, t = v0 / D, c0 = v0 % D;
  const bool valid = t < rows;
  uint32_t val[VPT / 2];
#pragma unroll
  for (int q = 0; q < VPT / 8; ++q) {
    const uint4 w = valid ? *reinterpret_cast<const uint4*>(s + static_cast<size_t>(t) * D + c0 + 8 * q)
                          : make_uint4(0, 0, 0, 0);
    val[4 * q] = w.x; val[4 * q + 1] = w.y; val[4 * q + 2] = w.z; val[4 * q + 3] = w.w;
  }
  uint32_t code[VPT / 16], smw[VPT / 4];
#pragma unroll
  for (int i = 0; i < VPT / 16; ++i) code[i] = 0;
#pragma unroll
  for (int i = 0; i < VPT / 4; ++i) smw[i] = 0;
  int nsec = 0;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const uint32_t bits = (val[k >> 1] >> (16 * (k & 1))) & 0xffffu;
    const int off = valid ? e_base[c0 + k] - static_cast<int>((bits >> 7) & 0xff) : 1;
    const uint32_t cd = (off >= 1 && off <= 3) ? static_cast<uint32_t>(off) : 0u;
    code[k >> 4] |= cd << (2 * (k & 15));
    nsec += cd == 0;
    smw[k >> 2] |= (((bits >> 8) & 0x80u) | (bits & 0x7fu)) << (8 * (k & 3));
  }
  st_words<VPT / 16>(reinterpret_cast<uint32_t*>(o + G::OFF_C2) + threadIdx.x * (VPT / 16), code);
  st_words<VPT / 4>(reinterpret_cast<uint32_t*>(o + G::OFF_SM) + threadIdx.x * (VPT / 4), smw);
  int total;
  int pos = block_scan256(nsec, ws, &total);
  uint32_t* esc = reinterpret_cast<uint32_t*>(o + G::OFF_ESC);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    if ((code[k >> 4] >> (2 * (k & 15))) & 3u) continue;
    const uint32_t bits = (val[k >> 1] >> (16 * (k & 1))) & 0xffffu;
    const int off = e_base[c0 + k] - static_cast<int>((bits >> 7) & 0xff);
    uint32_t nib = static_cast<uint32_t>(off);
    if (off > 14) {
      nib = 15;
      const int e = atomicAdd(&n_esc, 1);
      if (e < kPackEscCap) esc[e] = (static_cast<uint32_t>(v0 + k) << 16) | bits;
    }
    if (pos < G::SEC) atomicOr(&secw[pos >> 3], nib << (4 * (pos & 7)));
    ++pos;
  }
  __syncthreads();
  uint32_t* osec = reinterpret_cast<uint32_t*>(o + G::OFF_SEC);
  for (int i = threadIdx.x; i < G::SEC / 8; i += kThreads) osec[i] = secw[i];
  if (threadIdx.x == 0) {
    *reinterpret_cast<uint32_t*>(o + G::OFF_NS) = static_cast<uint32_t>(min(total, G::SEC));
    *reinterpret_cast<uint32_t*>(o + G::OFF_NE) = static_cast<uint32_t>(min(n_esc, kPackEscCap));
    if (n_esc > kPackEscCap || total > G::SEC) atomicMax(overflow, b + 1);  // 1 + the block index (0 = none)
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads) unpack_kernel(const uint8_t* src, size_t src_slice_pitch, int n_blocks,
                                                           uint16_t* dst, size_t dst_slice_pitch) {
  using G = PackGeo<D>;
  constexpr int VPT = G::VPT;
  const int b = blockIdx.x, sl = blockIdx.y;
  const uint8_t* in = src + sl * src_slice_pitch + static_cast<size_t>(b) * packed_block_bytes(D);
  uint16_t* d = dst + sl * dst_slice_pitch + static_cast<size_t>(b) * kTok * D;
  __shared__ uint8_t e_base[D];
  __shared__ int ws[kThreads / 32];
  for (int c = threadIdx.x; c < D; c += kThreads) e_base[c] = in[c];
  const int v0 = threadIdx.x * VPT, t = v0 / D, c0 = v0 % D;
  uint32_t code[VPT / 16], smw[VPT / 4];
  ld_words<VPT / 16>(reinterpret_cast<const uint32_t*>(in + G::OFF_C2) + threadIdx.x * (VPT / 16), code);
  int nsec = 0;
#pragma unroll
  for (int i = 0; i < VPT / 16; ++i) nsec += __popc(~(code[i] | (code[i] >> 1)) & 0x55555555u);  // codes equal to 0
  ld_words<VPT / 4>(reinterpret_cast<const uint32_t*>(in + G::OFF_SM) + threadIdx.x * (VPT / 4), smw);
  int total;
  int pos = block_scan256(nsec, ws, &total);  // its barrier also publishes e_base
  const uint8_t* sec = in + G::OFF_SEC;
  uint32_t outw[VPT / 2];
#pragma unroll
  for (int k2 = 0; k2 < VPT / 2; ++k2) {
    uint32_t pair = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = 2 * k2 + j;
      uint32_t off = (code[k >> 4] >> (2 * (k & 15))) & 3u;
      if (off == 0) {
        off = (sec[pos >> 1] >> (4 * (pos & 1))) & 0xfu;  // escapes (15) are overwritten below
        ++pos;
      }
      const uint32_t smj = (smw[k >> 2] >> (8 * (k & 3))) & 0xffu;
      const uint32_t e = (static_cast<uint32_t>(e_base[c0 + k]) - off) & 0xffu;
      pair |= (((smj & 0x80u) << 8) | (e << 7) | (smj & 0x7fu)) << (16 * j);
    }
    outw[k2] = pair;
  }
  st_words<VPT / 2>(reinterpret_cast<uint32_t*>(d + static_cast<size_t>(t) * D + c0), outw);
  __syncthreads();
  const uint32_t ne = *reinterpret_cast<const uint32_t*>(in + G::OFF_NE);
  const uint32_t* esc = reinterpret_cast<const uint32_t*>(in + G::OFF_ESC);
  for (uint32_t i = threadIdx.x; i < ne; i += kThreads) {
    const uint32_t e = esc[i];
    d[e >> 16] = static_cast<uint16_t>(e & 0xffffu);
  }
}

}  // namespace

cudaError_t pack_blocks(const uint16_t* src, size_t src_slice_pitch, int src_row0, int n_valid, int n_blocks,
                        int n_slices, int d, uint8_t* dst, size_t dst_slice_pitch, int* overflow, cudaStream_t st) {
  if (n_blocks <= 0 || n_slices <= 0) return cudaSuccess;
  const dim3 grid(n_blocks, n_slices);
  if (d == 128) pack_kernel<128><<<grid, kThreads, 0, st>>>(src, src_slice_pitch, src_row0, n_valid, n_blocks, dst, dst_slice_pitch, overflow);
  else if (d == 64) pack_kernel<64><<<grid, kThreads, 0, st>>>(src, src_slice_pitch, src_row0, n_valid, n_blocks, dst, dst_slice_pitch, overflow);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t unpack_blocks(const uint8_t* src, size_t src_slice_pitch, int n_blocks, int n_slices, int d, uint16_t* dst,
                          size_t dst_slice_pitch, cudaStream_t st) {
  if (n_blocks <= 0 || n_slices <= 0) return cudaSuccess;
  const dim3 grid(n_blocks, n_slices);
  if (d == 128) unpack_kernel<128><<<grid, kThreads, 0, st>>>(src, src_slice_pitch, n_blocks, dst, dst_slice_pitch);
  else if (d == 64) unpack_kernel<64><<<grid, kThreads, 0, st>>>(src, src_slice_pitch, n_blocks, dst, dst_slice_pitch);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace vc
