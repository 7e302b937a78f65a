// vc_quant.cu -- KIVI-style KV quantiser (the quant-uniform compressor's data
// plane).  K: per-channel asymmetric quantisation over groups of G=128 tokens;
// V: per-token asymmetric quantisation over the head's d channels.  Scale and
// zero are fp16; codes are written directly in the mma.sync A-fragment order
// the draft-attention kernel consumes, so
// the draft path never reshuffles.
//
// Bit-exact with oracle/vc_oracle.c:quant_group (IEEE div/sub, RNE f16,
// round-half-even codes); reference semantics it honours: bit_scheme in
// [1,16] uniform across tokens and layers (/root/reference/proj/src/
// compressor.cpp:42,72), payload size law counts codes only (:96-100).
#include "vc_common.cuh"
#include "vc_kernels.h"

namespace vc {

namespace {

constexpr int kG = VC_QGROUP;  // tokens per K group
// bit offset of fragment pair j (a0a1, a2a3, a4a5, a6a7) inside an int4 word
__device__ constexpr int kNibble[4] = {0, 8, 4, 12};

VC_DEV uint32_t quant_code(float x, float sf, float zf, int qmax) {
  if (sf == 0.0f) return 0u;
  float t = __fdiv_rn(__fsub_rn(x, zf), sf);
  int c = __float2int_rn(t);
  c = c < 0 ? 0 : (c > qmax ? qmax : c);
  return static_cast<uint32_t>(c);
}

// Fragment element (pair j, half e) of an m16n8k16 A tile: row/col offsets.
// a0,a1 (r, k),(r, k+1); a2,a3 (r+8, k),(r+8,k+1); a4,a5 (r, k+8)...; a6,a7 (r+8,k+8)...
VC_DEV void frag_rc(int lane, int j, int e, int& r, int& c) {
  r = (lane >> 2) + ((j & 1) ? 8 : 0);
  c = 2 * (lane & 3) + e + ((j & 2) ? 8 : 0);
}

template <int D, int BITS>
__global__ void __launch_bounds__(128) quant_kivi_kernel(const QuantJob* __restrict__ jobs) {
  const QuantJob job = jobs[blockIdx.y];
  const int g = job.g0 + blockIdx.x;
  if (blockIdx.x >= job.ng) return;
  extern __shared__ __align__(16) uint16_t sm[];
  uint16_t* sk = sm;               // [kG][D]
  uint16_t* sv = sm + kG * D;      // [kG][D]
  float* kscale = reinterpret_cast<float*>(sv + kG * D);  // [D]
  float* kzero = kscale + D;                               // [D]
  float* vscale = kzero + D;                               // [kG]
  float* vzero = vscale + kG;                              // [kG]
  const int tid = threadIdx.x;
  constexpr int QMAX = (1 << BITS) - 1;
  constexpr int UCW = static_cast<int>(quant_unit_code_words(D, BITS));  // codes of one unit
  constexpr int UREC = static_cast<int>(quant_unit_words(D, BITS));
  uint32_t* rec = job.rec + static_cast<size_t>(g) * quant_record_words(D, BITS);

  // 1. stage the group's bf16 K and V rows (contiguous: kG*D elements each)
  const uint4* srck = reinterpret_cast<const uint4*>(job.k + static_cast<size_t>(g) * kG * D);
  const uint4* srcv = reinterpret_cast<const uint4*>(job.v + static_cast<size_t>(g) * kG * D);
  constexpr int NV = kG * D / 8;
  for (int i = tid; i < NV; i += 128) {
    reinterpret_cast<uint4*>(sk)[i] = srck[i];
    reinterpret_cast<uint4*>(sv)[i] = srcv[i];
  }
  __syncthreads();

  // 2. K: per-channel min/max over the group's tokens
  for (int c = tid; c < D; c += 128) {
    float mn = bf2f(sk[c]), mx = mn;
    for (int t = 1; t < kG; ++t) {
      float x = bf2f(sk[t * D + c]);
      mn = fminf(mn, x);
      mx = fmaxf(mx, x);
    }
    mn = __fadd_rn(mn, 0.0f);  // canonical +0
    float sc = __fdiv_rn(__fsub_rn(mx, mn), static_cast<float>(QMAX));
    uint16_t s16 = f2h(sc), z16 = f2h(mn);
    kscale[c] = h2f(s16);
    kzero[c] = h2f(z16);
    rec[c] = static_cast<uint32_t>(s16) | (static_cast<uint32_t>(z16) << 16);
  }
  // 3. V: per-token min/max over the head's channels
  for (int t = tid; t < kG; t += 128) {
    float mn = bf2f(sv[t * D]), mx = mn;
    for (int c = 1; c < D; ++c) {
      float x = bf2f(sv[t * D + c]);
      mn = fminf(mn, x);
      mx = fmaxf(mx, x);
    }
    mn = __fadd_rn(mn, 0.0f);
    float sc = __fdiv_rn(__fsub_rn(mx, mn), static_cast<float>(QMAX));
    uint16_t s16 = f2h(sc), z16 = f2h(mn);
    vscale[t] = h2f(s16);
    vzero[t] = h2f(z16);
    rec[D + (t / VC_QUNIT) * UREC + 2 * UCW + t % VC_QUNIT] =
        static_cast<uint32_t>(s16) | (static_cast<uint32_t>(z16) << 16);
  }
  __syncthreads();

  // 4. pack codes in fragment order.  Per 16-row tile a lane owns W u32s.
  constexpr int KS = D / 16;                   // k-steps (K) / channel tiles (V)
  constexpr int W = (BITS == 4) ? KS : KS / 2; // u32 per lane per 16-row tile
  constexpr int CH = W < 4 ? W : 4;            // u32 per vector load
  constexpr int MT = kG / 16;
  constexpr int TOTAL = MT * W * 32;           // u32 per group (K or V)
  static_assert(TOTAL % UCW == 0, "unit records split the group's code stream");
  for (int idx = tid; idx < TOTAL; idx += 128) {
    // idx = ((m * (W/CH) + w/CH) * 32 + lane) * CH + w%CH
    const int wl = idx % CH;
    const int lane = (idx / CH) % 32;
    const int wq = (idx / (CH * 32)) % (W / CH);
    const int m = idx / (CH * 32 * (W / CH));
    const int w = wq * CH + wl;
    uint32_t kword = 0, vword = 0;
#pragma unroll
    for (int sub = 0; sub < (BITS == 4 ? 1 : 2); ++sub) {
      const int s = (BITS == 4) ? w : 2 * w + sub;  // k-step / channel tile
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, c;
          frag_rc(lane, j, e, r, c);
          // int4: pairs 0,1 sit in the low nibble of bytes 0/1 (and 2/3), pairs
          // 2,3 in the high nibbles, so the consumer unpacks a word with one
          // shift + four lop3 (high nibbles arrive x16, folded into its B operand)
          const int shift = (BITS == 4) ? (kNibble[j] + 16 * e) : (8 * sub + 2 * j + 16 * e);
          // K tile: rows = tokens (m), cols = channels (s)
          const int tk = m * 16 + r, ck = s * 16 + c;
          kword |= quant_code(bf2f(sk[tk * D + ck]), kscale[ck], kzero[ck], QMAX) << shift;
          // V^T tile: rows = channels (s), cols = tokens (m)
          const int cv = s * 16 + r, tv = m * 16 + c;
          vword |= quant_code(bf2f(sv[tv * D + cv]), vscale[tv], vzero[tv], QMAX) << shift;
        }
      }
    }
    // the group's code stream idx is m-tile major, so unit idx / UCW holds it
    uint32_t* urec = rec + D + (idx / UCW) * UREC + idx % UCW;
    urec[0] = kword;
    urec[UCW] = vword;
  }
}

template <int D, int BITS>
cudaError_t launch_quant(const QuantJob* jobs, int n_jobs, int max_groups, cudaStream_t st) {
  const size_t smem = 2 * kG * D * sizeof(uint16_t) + (2 * D + 2 * kG) * sizeof(float);
  auto kern = quant_kivi_kernel<D, BITS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(max_groups, n_jobs);
  kern<<<grid, 128, smem, st>>>(jobs);
  return cudaGetLastError();
}

}  // namespace

cudaError_t quant_kivi(const QuantJob* jobs_dev, int n_jobs, int max_groups, int d, int bits,
                       cudaStream_t st) {
  if (n_jobs <= 0 || max_groups <= 0) return cudaSuccess;
  if (d == 128 && bits == 4) return launch_quant<128, 4>(jobs_dev, n_jobs, max_groups, st);
  if (d == 128 && bits == 2) return launch_quant<128, 2>(jobs_dev, n_jobs, max_groups, st);
  if (d == 64 && bits == 4) return launch_quant<64, 4>(jobs_dev, n_jobs, max_groups, st);
  if (d == 64 && bits == 2) return launch_quant<64, 2>(jobs_dev, n_jobs, max_groups, st);
  return cudaErrorInvalidValue;
}

}  // namespace vc
