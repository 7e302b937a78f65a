// microbench.cu -- one-off B200 probes that size the design (DESIGN.md
// "Measured constants"): HBM streaming read, legacy mma.sync f16 rate,
// FFMA rate, pinned H2D/D2H over PCIe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void read_kernel(const int4* __restrict__ p, size_t n, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345 && acc.y == 7) *sink = acc;
}

__global__ void mma_kernel(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[0] = s;
}

__global__ void ffma_kernel(float* out, int iters) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 0.001f + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 0.9999f, a[(j + 1) & 7]);
  float s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  // HBM read
  size_t bytes = (size_t)8 << 30;
  int4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  int4* sink; CK(cudaMalloc(&sink, 64));
  for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
    for (int w = 0; w < 2; ++w) read_kernel<<<grid, 512>>>(buf, bytes / 16, sink);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) read_kernel<<<grid, 512>>>(buf, bytes / 16, sink);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("hbm_read grid=%d: %.1f GB/s\n", grid, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  // mma.sync
  float* out; CK(cudaMalloc(&out, 64));
  int iters = 20000;
  mma_kernel<<<148 * 4, 256>>>(out, 100);
  CK(cudaEventRecord(e0));
  mma_kernel<<<148 * 4, 256>>>(out, iters);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
  double flops = 148.0 * 4 * 8 * iters * 4 * 4096.0;
  printf("mma.sync m16n8k16 f16->f32: %.1f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
  ffma_kernel<<<148 * 4, 256>>>(out, 100);
  CK(cudaEventRecord(e0));
  ffma_kernel<<<148 * 4, 256>>>(out, iters);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("ffma: %.1f TFLOP/s\n", 148.0 * 4 * 256 * iters * 8 * 2 / (ms * 1e-3) / 1e12);
  // PCIe
  size_t hb = (size_t)2 << 30;
  void* host; CK(cudaHostAlloc(&host, hb, cudaHostAllocDefault));
  memset(host, 3, hb);
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(e0, s));
    CK(cudaMemcpyAsync(buf, host, hb, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("h2d pinned 2GiB: %.1f GB/s\n", hb / (ms * 1e-3) / 1e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(e0, s));
    CK(cudaMemcpyAsync(host, buf, hb, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("d2h pinned 2GiB: %.1f GB/s\n", hb / (ms * 1e-3) / 1e9);
  }
  // H2D concurrent with a read kernel on another stream
  cudaStream_t s2; CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaEventRecord(e0, s));
  CK(cudaMemcpyAsync((char*)buf + ((size_t)6 << 30), host, hb, cudaMemcpyHostToDevice, s));
  for (int r = 0; r < 20; ++r) read_kernel<<<148 * 8, 512, 0, s2>>>(buf, ((size_t)6 << 30) / 16, sink);
  CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("h2d pinned 2GiB under HBM load: %.1f GB/s\n", hb / (ms * 1e-3) / 1e9);
  CK(cudaDeviceSynchronize());
  int dev; cudaDeviceProp prop; CK(cudaGetDevice(&dev)); CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s sms=%d l2=%d MB smem/block optin=%zu\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin);
  return 0;
}
