// SPDX-License-Identifier: MIT
// Collectives for sharded decompositions: one rank per GPU,
// the tensor split in slabs along its last mode; ranks exchange only small
// partials (I_n x l sketches, J_s x l panels, pivot candidates, pivot rows).
//
//  * NcclComm: NCCL (libnccl.so.2, loaded at run time: the library has no
//    link-time NCCL dependency) on the context's stream; over NVLink /
//    NVSwitch between the GPUs of one node.
//  * LoopbackComm: virtual ranks inside one process (several contexts on one
//    GPU, one host thread each). Used to test the sharded path on a single
//    GPU against the unsharded result; sums are taken in rank order.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>

#include "common.cuh"

namespace rcpg {

enum class CommType { f32, f64, bytes };

struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // in place, element-wise sum over the ranks
  virtual void allreduce_sum(void* buf, size_t count, CommType t, cudaStream_t st) = 0;
  // recv[g * bytes .. (g+1) * bytes) = rank g's send
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
};

// 128-byte NCCL unique id (host only).
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* id128);

// One hub per group of virtual ranks; comms[r] for rank r.
struct LoopbackHub;
std::shared_ptr<LoopbackHub> make_loopback_hub(int nranks);
std::unique_ptr<Comm> make_loopback_comm(const std::shared_ptr<LoopbackHub>& hub, int rank);

// Balanced contiguous split of [0, extent) over nranks: [lo, hi) of `rank`.
inline void slab_range(i64 extent, int nranks, int rank, i64& lo, i64& hi) {
  const i64 base = extent / nranks, rem = extent % nranks;
  lo = rank * base + (rank < rem ? rank : rem);
  hi = lo + base + (rank < rem ? 1 : 0);
}

}  // namespace rcpg
