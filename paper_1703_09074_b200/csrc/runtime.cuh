// SPDX-License-Identifier: MIT
// Runtime plumbing shared by the launchers: kernel-launch accounting,
// device properties, cooperative launches.
#pragma once

#include <atomic>

#include "common.cuh"

namespace rcpg {

// Total kernels this library has launched (exported through
// rcpg_kernel_launches; bench.py reports it as gpu_launches).
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
inline void count_launch(long long n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }

struct DeviceCaps {
  int device = 0;
  int num_sms = 148;
  int max_smem_optin = 227 * 1024;
};

inline const DeviceCaps& device_caps() {
  static thread_local DeviceCaps caps = [] {
    DeviceCaps c;
    RCPG_CUDA(cudaGetDevice(&c.device));
    RCPG_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, c.device));
    RCPG_CUDA(cudaDeviceGetAttribute(&c.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
    return c;
  }();
  return caps;
}

// Largest cooperative grid for `kernel` at `threads` threads and `smem` bytes.
template <typename K>
int max_coop_blocks(K kernel, int threads, size_t smem) {
  // cached: occupancy queries are slow host calls that would leave the GPU idle
  static thread_local struct Entry { const void* k; int threads; size_t smem; int blocks; } cache[16];
  static thread_local int used = 0;
  for (int i = 0; i < used; ++i)
    if (cache[i].k == reinterpret_cast<const void*>(kernel) && cache[i].threads == threads && cache[i].smem == smem)
      return cache[i].blocks;
  int per_sm = 0;
  RCPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  if (per_sm < 1) throw std::runtime_error("cooperative kernel does not fit on an SM");
  const int blocks = per_sm * device_caps().num_sms;
  if (used < 16) cache[used++] = Entry{reinterpret_cast<const void*>(kernel), threads, smem, blocks};
  return blocks;
}

// Opt a kernel into the largest dynamic shared memory the device allows
// (limit minus the kernel's static shared memory); returns that size.
template <typename K>
size_t enable_max_dyn_smem(K kernel) {
  cudaFuncAttributes fa{};
  RCPG_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(kernel)));
  const size_t lim = size_t(device_caps().max_smem_optin) - fa.sharedSizeBytes;
  RCPG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(kernel),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(lim)));
  return lim;
}

template <typename K, typename... Args>
void launch_coop(K kernel, int blocks, int threads, size_t smem, cudaStream_t st, Args... args) {
  void* argv[] = {static_cast<void*>(&args)...};
  RCPG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(blocks), dim3(threads),
                                        argv, smem, st));
  count_launch();
}

}  // namespace rcpg
