// vc_tp.cu -- tensor-parallel collectives and the fixed-order TP residual
// (see vc_tp.h for why the combine is an all-gather + rank-order sum).
#include "vc_tp.h"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "vc_common.cuh"
#include "vc_engine.hpp"

namespace vc {

// ------------------------------------------------------------------ loopback
class LoopbackGroup {
 public:
  explicit LoopbackGroup(int size) : size_(size), src_(size), ready_(size), copied_(size) {}
  int size() const { return size_; }
  // generation barrier over the group's host threads
  void barrier() {
    std::unique_lock<std::mutex> lk(mu_);
    const long g = gen_;
    if (++count_ == size_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen_ != g; });
    }
  }
  std::vector<const float*> src_;
  std::vector<cudaEvent_t> ready_, copied_;

 private:
  int size_;
  std::mutex mu_;
  std::condition_variable cv_;
  int count_ = 0;
  long gen_ = 0;
};

namespace {

class Loopback final : public Collective {
 public:
  Loopback(std::shared_ptr<LoopbackGroup> g, int rank) : g_(std::move(g)), rank_(rank) {
    check_cuda(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming), "loopback event");
    check_cuda(cudaEventCreateWithFlags(&copied_, cudaEventDisableTiming), "loopback event");
  }
  ~Loopback() override {
    cudaEventDestroy(ready_);
    cudaEventDestroy(copied_);
  }
  bool graph_capturable() const override { return false; }
  void all_gather(const float* src, float* dst, size_t count, cudaStream_t st) override {
    LoopbackGroup& g = *g_;
    const int T = g.size();
    // phase 1: publish my source and the event that marks it ready
    check_cuda(cudaEventRecord(ready_, st), "loopback ready");
    g.src_[rank_] = src;
    g.ready_[rank_] = ready_;
    g.barrier();
    for (int p = 0; p < T; ++p) {  // copy every rank's partial, in rank order
      check_cuda(cudaStreamWaitEvent(st, g.ready_[p], 0), "loopback wait");
      check_cuda(cudaMemcpyAsync(dst + static_cast<size_t>(p) * count, g.src_[p], count * sizeof(float),
                                 cudaMemcpyDeviceToDevice, st), "loopback copy");
    }
    // phase 2: nobody may overwrite its source before every peer copied it
    check_cuda(cudaEventRecord(copied_, st), "loopback copied");
    g.copied_[rank_] = copied_;
    g.barrier();
    for (int p = 0; p < T; ++p) check_cuda(cudaStreamWaitEvent(st, g.copied_[p], 0), "loopback wait");
    g.barrier();  // the slots may be republished by the next call
  }

 private:
  std::shared_ptr<LoopbackGroup> g_;
  int rank_;
  cudaEvent_t ready_ = nullptr, copied_ = nullptr;
};

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // reuse an already-loaded libnccl (e.g. torch's) before the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (h) {
      api.h = h;
      api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
      api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  return api.all_gather ? &api : nullptr;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const NcclApi* a = nccl();
    throw CudaError(std::string(what) + ": " + (a && a->error_string ? a->error_string(r) : "nccl error"));
  }
}

class Nccl final : public Collective {
 public:
  Nccl(const void* id, int rank, int size) {
    const NcclApi* a = nccl();
    if (!a) throw ContractViolation("tensor parallelism over NCCL: libnccl.so.2 not found");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(a->comm_init_rank(&comm_, size, uid, rank), "ncclCommInitRank");
  }
  ~Nccl() override {
    if (comm_) nccl()->comm_destroy(comm_);
  }
  bool graph_capturable() const override { return true; }
  void all_gather(const float* src, float* dst, size_t count, cudaStream_t st) override {
    nccl_check(nccl()->all_gather(src, dst, count, ncclFloat32, comm_, st), "ncclAllGather");
  }

 private:
  ncclComm_t comm_ = nullptr;
};

// ------------------------------------------------------------------ residual
// block: 8 rows x 16 threads, one 128-feature tile; thread = 8 features
__global__ void tp_residual_kernel(float* x, const float* g, int tp, int M, int H, float* ss_part) {
  pdl_trigger();
  pdl_wait();
  const int t = threadIdx.x >> 4, sub = threadIdx.x & 15;
  const int m = blockIdx.x * 8 + t;
  const int n0 = blockIdx.y * 128 + sub * 8;
  const bool live = m < M;
  float sq = 0.f;
  if (live) {
    float v[8];
    float4* xp = reinterpret_cast<float4*>(x + static_cast<size_t>(m) * H + n0);
    const float4 a = xp[0], b = xp[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < tp; ++r) {  // rank order
      const float4* gp = reinterpret_cast<const float4*>(g + (static_cast<size_t>(r) * M + m) * H + n0);
      const float4 c = gp[0], d = gp[1];
      s[0] += c.x; s[1] += c.y; s[2] += c.z; s[3] += c.w; s[4] += d.x; s[5] += d.y; s[6] += d.z; s[7] += d.w;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] += s[j];
    xp[0] = make_float4(v[0], v[1], v[2], v[3]);
    xp[1] = make_float4(v[4], v[5], v[6], v[7]);
    sq = ((v[0] * v[0] + v[1] * v[1]) + (v[2] * v[2] + v[3] * v[3])) +
         ((v[4] * v[4] + v[5] * v[5]) + (v[6] * v[6] + v[7] * v[7]));
  }
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);  // fixed tree
  if (live && sub == 0) ss_part[static_cast<size_t>(m) * (H / 128) + blockIdx.y] = sq;
}

}  // namespace

std::shared_ptr<LoopbackGroup> make_loopback_group(int size) {
  if (size < 1) throw ContractViolation("loopback group: size must be >= 1");
  return std::make_shared<LoopbackGroup>(size);
}

std::unique_ptr<Collective> make_loopback(const std::shared_ptr<LoopbackGroup>& group, int rank) {
  if (!group || rank < 0 || rank >= group->size()) throw ContractViolation("loopback: bad rank");
  return std::make_unique<Loopback>(group, rank);
}

bool nccl_available() { return nccl() != nullptr; }

bool nccl_unique_id(void* out128) {
  const NcclApi* a = nccl();
  if (!a) return false;
  ncclUniqueId uid;
  nccl_check(a->get_unique_id(&uid), "ncclGetUniqueId");
  std::memcpy(out128, &uid, sizeof(uid));
  return true;
}

std::unique_ptr<Collective> make_nccl(const void* unique_id, int rank, int size) {
  return std::make_unique<Nccl>(unique_id, rank, size);
}

cudaError_t tp_residual(float* x, const float* gathered, int tp, int M, int H, float* ss_part, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  return launch_pdl(tp_residual_kernel, dim3((M + 7) / 8, H / 128), dim3(128), 0, st, x, gathered, tp, M, H,
                    ss_part);
}

}  // namespace vc
