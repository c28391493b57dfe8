// SPDX-License-Identifier: MIT
// Collectives for sharded decompositions (see comm.cuh).
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.cuh"
#include "runtime.cuh"

namespace rcpg {

// ------------------------------------------------------------------ NCCL
namespace {

// The subset of nccl.h this library uses (NCCL 2.x ABI).
using ncclResult_t = int;
using ncclComm_t = void*;
struct ncclUniqueId {
  char internal[128];
};
constexpr int kNcclSum = 0, kNcclUint8 = 1, kNcclFloat32 = 7, kNcclFloat64 = 8;

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    // prefer an NCCL already loaded into the process (e.g. torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) throw std::runtime_error(std::string("NCCL unavailable: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (p == nullptr) throw std::runtime_error(std::string("NCCL symbol missing: ") + n);
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) throw std::runtime_error(std::string(what) + ": " + nccl().GetErrorString(r));
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm != nullptr) nccl().CommDestroy(comm);
  }
  void allreduce_sum(void* buf, size_t count, CommType t, cudaStream_t st) override {
    const int dt = t == CommType::f64 ? kNcclFloat64 : (t == CommType::f32 ? kNcclFloat32 : kNcclUint8);
    nccl_check(nccl().AllReduce(buf, buf, count, dt, kNcclSum, comm, st), "ncclAllReduce");
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    nccl_check(nccl().AllGather(send, recv, bytes, kNcclUint8, comm, st), "ncclAllGather");
  }
};

}  // namespace

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* id128) {
  auto c = std::make_unique<NcclComm>();
  c->rank = rank;
  c->size = nranks;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  nccl_check(nccl().CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  return c;
}

// -------------------------------------------------------------- loopback
struct LoopbackHub {
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<const void*> ptr;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace {

template <typename T>
__global__ void loopback_sum_kernel(const T* const* src, int n, size_t count, T* out) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < count; e += size_t(gridDim.x) * blockDim.x) {
    T s = src[0][e];
    for (int g = 1; g < n; ++g) s += src[g][e];  // rank order: deterministic
    out[e] = s;
  }
}

struct LoopbackComm final : Comm {
  std::shared_ptr<LoopbackHub> hub;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  void* ptrs_dev = nullptr;
  ~LoopbackComm() override {
    if (tmp) cudaFree(tmp);
    if (ptrs_dev) cudaFree(ptrs_dev);
  }
  void allreduce_sum(void* buf, size_t count, CommType t, cudaStream_t st) override {
    const size_t es = t == CommType::f64 ? 8 : (t == CommType::f32 ? 4 : 1);
    if (t == CommType::bytes) throw std::runtime_error("loopback: byte sums are not defined");
    if (tmp_bytes < count * es) {
      if (tmp) RCPG_CUDA(cudaFree(tmp));
      RCPG_CUDA(cudaMalloc(&tmp, count * es));
      tmp_bytes = count * es;
    }
    if (ptrs_dev == nullptr) RCPG_CUDA(cudaMalloc(&ptrs_dev, sizeof(void*) * size_t(hub->n)));
    RCPG_CUDA(cudaStreamSynchronize(st));
    hub->ptr[size_t(rank)] = buf;
    hub->barrier();  // every rank's input is final
    RCPG_CUDA(cudaMemcpyAsync(ptrs_dev, hub->ptr.data(), sizeof(void*) * size_t(hub->n), cudaMemcpyHostToDevice, st));
    const int blocks = int(std::min<size_t>(1024, (count + 255) / 256));
    if (t == CommType::f64)
      loopback_sum_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double* const*>(ptrs_dev), hub->n, count,
                                                          static_cast<double*>(tmp));
    else
      loopback_sum_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float* const*>(ptrs_dev), hub->n, count,
                                                         static_cast<float*>(tmp));
    RCPG_CUDA(cudaGetLastError());
    RCPG_CUDA(cudaStreamSynchronize(st));
    hub->barrier();  // every rank has read all inputs
    RCPG_CUDA(cudaMemcpyAsync(buf, tmp, count * es, cudaMemcpyDeviceToDevice, st));
    RCPG_CUDA(cudaStreamSynchronize(st));
    hub->barrier();
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    RCPG_CUDA(cudaStreamSynchronize(st));
    hub->ptr[size_t(rank)] = send;
    hub->barrier();
    for (int g = 0; g < hub->n; ++g)
      RCPG_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + size_t(g) * bytes, hub->ptr[size_t(g)], bytes,
                                cudaMemcpyDeviceToDevice, st));
    RCPG_CUDA(cudaStreamSynchronize(st));
    hub->barrier();
  }
};

}  // namespace

std::shared_ptr<LoopbackHub> make_loopback_hub(int nranks) {
  auto h = std::make_shared<LoopbackHub>();
  h->n = nranks;
  h->ptr.assign(size_t(nranks), nullptr);
  return h;
}

std::unique_ptr<Comm> make_loopback_comm(const std::shared_ptr<LoopbackHub>& hub, int rank) {
  auto c = std::make_unique<LoopbackComm>();
  c->hub = hub;
  c->rank = rank;
  c->size = hub->n;
  return c;
}

}  // namespace rcpg
