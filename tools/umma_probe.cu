// umma_probe.cu -- pins the tcgen05 building blocks the dense attention
// kernel uses, on one CTA:  S = Q K^T (SS, both K-major SW128 tiles loaded by
// 2-D TMA), P = bf16(S * 1/64) written to TMEM with tcgen05.st, O = P V (TS:
// A = P from TMEM, B = V MN-major SW128).  Compares with a CPU reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2605_17613_b200/csrc \
//        tools/umma_probe.cu -o tools/umma_probe && tools/umma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vc_common.cuh"
#include "vc_umma.cuh"

using namespace vc;

constexpr int R = 128, D = 128, NK = 128;

__global__ void probe_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                             const __grid_constant__ CUtensorMap tv, float* S_out, float* O_out, int lbo_mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;              // 2 atoms x 16 KB
  uint8_t* sK = smem + 32768;
  uint8_t* sV = smem + 65536;
  __shared__ __align__(8) uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar_ld, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar_ld, 3 * 32768);
    for (int a = 0; a < 2; ++a) {
      tma_load_2d(sQ + a * 16384, &tq, a * 64, 0, &bar_ld);
      tma_load_2d(sK + a * 16384, &tk, a * 64, 0, &bar_ld);
      tma_load_2d(sV + a * 16384, &tv, a * 64, 0, &bar_ld);
    }
  }
  mbar_wait(&bar_ld, 0);
  // S = Q K^T  (tmem cols 0..127)
  if (threadIdx.x == 0) {
    tmem_fence_after();
    const uint32_t id = umma_idesc_bf16(R, NK, false);
    for (int k = 0; k < D / 16; ++k) {
      const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
      const uint64_t da = umma_sdesc_sw128(smem_u32(sQ) + off, 16, 1024);
      const uint64_t db = umma_sdesc_sw128(smem_u32(sK) + off, 16, 1024);
      umma_ss(tbase, da, db, id, k > 0);
    }
    umma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tmem_fence_after();
  // each thread = one row (lane quarter = warp % 4)
  const int row = (warp & 3) * 32 + lane;
  const uint32_t trow = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  for (int c0 = 0; c0 < NK; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(trow + c0, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) S_out[row * NK + c0 + j] = __uint_as_float(v[j]);
    // P = bf16(S/64) packed two per column into cols 128 + c0/2 ..
    uint32_t p[16];
    for (int j = 0; j < 16; ++j)
      p[j] = pack_bf2(__uint_as_float(v[2 * j]) * 0.015625f, __uint_as_float(v[2 * j + 1]) * 0.015625f);
    tmem_st16(trow + 128 + c0 / 2, p);
  }
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  // O = P V  (tmem cols 256..383), A = P at cols 128.., B = V MN-major
  if (threadIdx.x == 0) {
    tmem_fence_after();
    const uint32_t id = umma_idesc_bf16(R, D, true);
    for (int k = 0; k < NK / 16; ++k) {
      const uint64_t db = umma_sdesc_sw128(smem_u32(sV) + k * 2048, lbo_mode ? 1024 : 16384, lbo_mode ? 16384 : 1024);
      umma_ts(tbase + 256, tbase + 128 + k * 8, db, id, k > 0);
    }
    umma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 1);
  tmem_fence_after();
  for (int c0 = 0; c0 < D; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(trow + 256 + c0, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) O_out[row * D + c0 + j] = __uint_as_float(v[j]);
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

static uint16_t f2bf_host(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fff + ((u >> 16) & 1);
  return static_cast<uint16_t>(u >> 16);
}
static float bf2f_host(uint16_t h) {
  uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main() {
  std::vector<uint16_t> q(R * D), k(NK * D), v(NK * D);
  srand(1);
  auto rnd = [] { return (rand() / (float)RAND_MAX - 0.5f) * 2.f; };
  for (auto& x : q) x = f2bf_host(rnd());
  for (auto& x : k) x = f2bf_host(rnd());
  for (auto& x : v) x = f2bf_host(rnd());
  uint16_t *dq, *dk, *dv;
  float *dS, *dO;
  cudaMalloc(&dq, q.size() * 2);
  cudaMalloc(&dk, k.size() * 2);
  cudaMalloc(&dv, v.size() * 2);
  cudaMalloc(&dS, R * NK * 4);
  cudaMalloc(&dO, R * D * 4);
  cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, k.data(), k.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v.data(), v.size() * 2, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &qr);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  auto mk = [&](CUtensorMap* m, void* p, int rows) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
  };
  CUtensorMap tq, tk, tv;
  mk(&tq, dq, R);
  mk(&tk, dk, NK);
  mk(&tv, dv, NK);
  const int smem = 3 * 32768 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // CPU reference
  std::vector<double> S(R * NK), O(R * D, 0.0);
  std::vector<float> P(R * NK);
  for (int r = 0; r < R; ++r)
    for (int n = 0; n < NK; ++n) {
      double acc = 0;
      for (int c = 0; c < D; ++c) acc += (double)bf2f_host(q[r * D + c]) * bf2f_host(k[n * D + c]);
      S[r * NK + n] = acc;
    }
  for (int mode = 0; mode < 2; ++mode) {
    probe_kernel<<<1, 128, smem>>>(tq, tk, tv, dS, dO, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("kernel error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> gS(R * NK), gO(R * D);
    cudaMemcpy(gS.data(), dS, gS.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(gO.data(), dO, gO.size() * 4, cudaMemcpyDeviceToHost);
    double es = 0;
    for (int i = 0; i < R * NK; ++i) es = fmax(es, fabs(gS[i] - S[i]));
    // O reference from the GPU's own S (rounded like the kernel)
    double eo = 0, omax = 0;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < D; ++c) {
        double acc = 0;
        for (int n = 0; n < NK; ++n) acc += (double)bf2f_host(f2bf_host(gS[r * NK + n] * 0.015625f)) * bf2f_host(v[n * D + c]);
        eo = fmax(eo, fabs(gO[r * D + c] - acc));
        omax = fmax(omax, fabs(acc));
      }
    printf("lbo_mode %d: max|S err| %.3e   max|O err| %.3e (|O|max %.2f)\n", mode, es, eo, omax);
  }
  return 0;
}
