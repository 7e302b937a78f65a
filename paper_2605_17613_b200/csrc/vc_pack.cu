// vc_pack.cu -- lossless packing of the host tier's bf16 KV (chunk ring).
//
// A verify of an offloaded request is bound by the PCIe link (every reload
// moves the request's full KV), so the host pool stores each 128-token block
// of a (layer, kv-head) slice -- K and V separately -- in a lossless packed
// form that moves ~0.76 of the bytes:
//   e_base[c]       the largest bf16 exponent of channel c over the block's tokens
//   nib[t][c]       4 bits: e_base[c] - exponent, 0..14 (15 = escape)
//   sm[t][c]        8 bits: sign | 7 mantissa bits
//   n_esc, esc[]    values whose exponent lies more than 14 below the channel's
//                   maximum (zeros, denormals, tiny values): (t*d + c) << 16 | raw bf16
// K's per-channel magnitude structure (outlier channels) is why the exponent
// base is per channel, not per token.  A block with more than kEscCap
// escapes does not pack (the overflow flag): the engine stores it raw.
// Decoding restores the bf16 bits exactly (losslessness of the verify does
// not depend on it: tests/test_stream_ring.py checks the round trip and the
// streamed verify bit for bit).
#include "vc_common.cuh"
#include "vc_gemm.h"

namespace vc {
namespace {

constexpr int kTok = 128;  // tokens per packed block (= VC_QGROUP)

template <int D>
__global__ void pack_kernel(const uint16_t* src, size_t src_slice_pitch, int src_row0, int n_valid, int n_blocks,
                            uint8_t* dst, size_t dst_slice_pitch, int* overflow) {
  constexpr size_t OFF_NIB = D, OFF_SM = D + kTok * D / 2, OFF_NE = D + kTok * D / 2 + kTok * D;
  const int b = blockIdx.x, sl = blockIdx.y;
  const uint16_t* s = src + sl * src_slice_pitch + static_cast<size_t>(src_row0 + b * kTok) * D;
  uint8_t* o = dst + sl * dst_slice_pitch + static_cast<size_t>(b) * packed_block_bytes(D);
  const int rows = min(kTok, n_valid - b * kTok);  // valid tokens of this block
  __shared__ uint8_t e_base[D];
  __shared__ int n_esc;
  if (threadIdx.x == 0) n_esc = 0;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    int m = 0;
    for (int t = 0; t < rows; ++t) m = max(m, (s[static_cast<size_t>(t) * D + c] >> 7) & 0xff);
    e_base[c] = static_cast<uint8_t>(m);
    o[c] = static_cast<uint8_t>(m);
  }
  __syncthreads();
  uint32_t* esc = reinterpret_cast<uint32_t*>(o + OFF_NE + 4);
  for (int pi = threadIdx.x; pi < kTok * D / 2; pi += blockDim.x) {  // one channel pair per step
    const int t = (2 * pi) / D, c = (2 * pi) % D;
    uint32_t nb = 0;
    uint16_t smv = 0;
    if (t < rows) {
      const uint32_t two = *reinterpret_cast<const uint32_t*>(s + static_cast<size_t>(t) * D + c);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t bits = (two >> (16 * j)) & 0xffffu;
        const int off = e_base[c + j] - static_cast<int>((bits >> 7) & 0xff);
        int n = off;
        if (off > 14) {
          n = 15;
          const int k = atomicAdd(&n_esc, 1);
          if (k < kPackEscCap) esc[k] = (static_cast<uint32_t>(t * D + c + j) << 16) | bits;
        }
        nb |= static_cast<uint32_t>(n) << (4 * j);
        smv |= static_cast<uint16_t>(((bits >> 8) & 0x80u) | (bits & 0x7fu)) << (8 * j);
      }
    }
    o[OFF_NIB + pi] = static_cast<uint8_t>(nb);
    *reinterpret_cast<uint16_t*>(o + OFF_SM + 2 * pi) = smv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *reinterpret_cast<uint32_t*>(o + OFF_NE) = static_cast<uint32_t>(min(n_esc, kPackEscCap));
    if (n_esc > kPackEscCap) atomicMax(overflow, b + 1);  // 1 + the block index (0 = none)
  }
}

template <int D>
__global__ void unpack_kernel(const uint8_t* src, size_t src_slice_pitch, int n_blocks, uint16_t* dst,
                              size_t dst_slice_pitch) {
  constexpr size_t OFF_NIB = D, OFF_SM = D + kTok * D / 2, OFF_NE = D + kTok * D / 2 + kTok * D;
  const int b = blockIdx.x, sl = blockIdx.y;
  const uint8_t* in = src + sl * src_slice_pitch + static_cast<size_t>(b) * packed_block_bytes(D);
  uint16_t* d = dst + sl * dst_slice_pitch + static_cast<size_t>(b) * kTok * D;
  __shared__ uint8_t e_base[D];
  for (int c = threadIdx.x; c < D; c += blockDim.x) e_base[c] = in[c];
  __syncthreads();
  // 4 channels (2 nibble bytes, 4 sign|mantissa bytes) per step
  for (int qi = threadIdx.x; qi < kTok * D / 4; qi += blockDim.x) {
    const int t = (4 * qi) / D, c = (4 * qi) % D;
    const uint16_t nb = *reinterpret_cast<const uint16_t*>(in + OFF_NIB + 2 * qi);
    const uint32_t sm = *reinterpret_cast<const uint32_t*>(in + OFF_SM + 4 * qi);
    uint32_t out[2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t n = (nb >> (4 * j)) & 0xfu;
      const uint32_t smj = (sm >> (8 * j)) & 0xffu;
      const uint32_t e = (static_cast<uint32_t>(e_base[c + j]) - n) & 0xffu;  // escapes are overwritten below
      const uint32_t bits = ((smj & 0x80u) << 8) | (e << 7) | (smj & 0x7fu);
      if (j & 1) out[j >> 1] |= bits << 16; else out[j >> 1] = bits;
    }
    *reinterpret_cast<uint2*>(d + static_cast<size_t>(t) * D + c) = make_uint2(out[0], out[1]);
  }
  __syncthreads();
  const uint32_t ne = *reinterpret_cast<const uint32_t*>(in + OFF_NE);
  const uint32_t* esc = reinterpret_cast<const uint32_t*>(in + OFF_NE + 4);
  for (uint32_t i = threadIdx.x; i < ne; i += blockDim.x) {
    const uint32_t e = esc[i];
    d[e >> 16] = static_cast<uint16_t>(e & 0xffffu);
  }
}

}  // namespace

cudaError_t pack_blocks(const uint16_t* src, size_t src_slice_pitch, int src_row0, int n_valid, int n_blocks,
                        int n_slices, int d, uint8_t* dst, size_t dst_slice_pitch, int* overflow, cudaStream_t st) {
  if (n_blocks <= 0 || n_slices <= 0) return cudaSuccess;
  const dim3 grid(n_blocks, n_slices);
  if (d == 128) pack_kernel<128><<<grid, 256, 0, st>>>(src, src_slice_pitch, src_row0, n_valid, n_blocks, dst, dst_slice_pitch, overflow);
  else if (d == 64) pack_kernel<64><<<grid, 256, 0, st>>>(src, src_slice_pitch, src_row0, n_valid, n_blocks, dst, dst_slice_pitch, overflow);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t unpack_blocks(const uint8_t* src, size_t src_slice_pitch, int n_blocks, int n_slices, int d, uint16_t* dst,
                          size_t dst_slice_pitch, cudaStream_t st) {
  if (n_blocks <= 0 || n_slices <= 0) return cudaSuccess;
  const dim3 grid(n_blocks, n_slices);
  if (d == 128) unpack_kernel<128><<<grid, 256, 0, st>>>(src, src_slice_pitch, n_blocks, dst, dst_slice_pitch);
  else if (d == 64) unpack_kernel<64><<<grid, 256, 0, st>>>(src, src_slice_pitch, n_blocks, dst, dst_slice_pitch);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace vc
