// SPDX-License-Identifier: MIT
// Shared device/host helpers for the rcpg CUDA library (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace rcpg {

using i64 = std::int64_t;
using u64 = std::uint64_t;

// ---------------------------------------------------------------- errors
struct InvalidArgument : std::invalid_argument {
  explicit InvalidArgument(const std::string& m) : std::invalid_argument(m) {}
};
struct SolverFailure : std::runtime_error {
  int iteration;
  SolverFailure(const std::string& m, int it)
      : std::runtime_error(m + " (iteration " + std::to_string(it) + ")"), iteration(it) {}
};
struct CudaFailure : std::runtime_error {
  cudaError_t code;
  CudaFailure(const std::string& m, cudaError_t c) : std::runtime_error(m), code(c) {}
};

inline void check_arg(bool cond, const std::string& msg) {
  if (!cond) throw InvalidArgument(msg);
}

#define RCPG_CUDA(call)                                                                      \
  do {                                                                                       \
    cudaError_t _e = (call);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      throw ::rcpg::CudaFailure(std::string(#call) + ": " + cudaGetErrorString(_e) + " at " + \
                                    __FILE__ + ":" + std::to_string(__LINE__),               \
                                _e);                                                         \
  } while (0)

#define RCPG_LAUNCHED() RCPG_CUDA(cudaGetLastError())

// --------------------------------------------------------------- traits
template <typename T>
struct Traits;
template <>
struct Traits<float> {
  static constexpr float eps = 1.1920928955078125e-07f;
  static constexpr float realmin = 1.17549435082228750797e-38f;
};
template <>
struct Traits<double> {
  static constexpr double eps = 2.220446049250313080847e-16;
  static constexpr double realmin = 2.2250738585072013830902e-308;
};

__host__ __device__ inline i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

// x - m * u and m * u with separate roundings (no FMA contraction): the
// elimination updates of Eigen's FullPivLU / HouseholderQR in the reference's
// SSE2 build (no -march, so no FMA) and in the oracle (-ffp-contract=off).
// The __*_rn intrinsics are never contracted by nvcc, so these keep the
// GPU's factorizations bit-identical to the oracle's on any input.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <typename T>
__device__ __forceinline__ T sub_mul_rn(T x, T m, T u) { return sub_rn(x, mul_rn(m, u)); }

// ---------------------------------------------------------- warp helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block-wide sum (fixed tree). `scratch` >= 32 doubles.
__device__ inline double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) scratch[0] = r;
  }
  __syncthreads();
  r = scratch[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------- grid barrier
// Sense-free generation barrier for cooperative launches (all CTAs
// co-resident, guaranteed by cudaLaunchCooperativeKernel). count returns to
// 0 after every barrier, so the state can be reused across launches.
struct GridBarrier {
  unsigned int count;
  unsigned int gen;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Flip-bit arrival (the scheme of cooperative_groups' grid sync): CTA 0 adds
// 2^31 - (G - 1), every other CTA adds 1, so the last arrival flips bit 31 and
// the low bits return to their value before the barrier (no reset, any G).
// Waiters spin on the flip: one L2 round trip after the last arrival instead
// of the arrive / reset / generation-bump chain (three dependent atomics).
__device__ inline void grid_sync(GridBarrier* b) {
  __syncthreads();
  const unsigned nblocks = gridDim.x * gridDim.y * gridDim.z;
  if (nblocks == 1) return;
  if (threadIdx.x == 0) {
    const bool master = (blockIdx.x | blockIdx.y | blockIdx.z) == 0;
    const unsigned inc = master ? 0x80000000u - (nblocks - 1) : 1u;
    __threadfence();
    const unsigned old = atomicAdd(&b->count, inc);
    while (((old ^ ld_acquire_u32(&b->count)) & 0x80000000u) == 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

// L2-coherent loads for data produced by other CTAs inside the same launch.
template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
  return __ldcg(p);
}

// ---------------------------------------------------------- tensor views
// Mode-n view of a row-major tensor: element (a, i, b) at a*I*R + i*R + b,
// a over the modes before n (row-major), b over the modes after n.
struct ModeView {
  i64 L = 1, I = 1, R = 1;
};

// Panels (Omega, W = X^T Q, Z = stab(W), KR panels) are stored in the
// "(a, c, b)" layout: row s = a*R + b, column c at a*cols*R + c*R + b. For the
// first mode this is column-major (ld = J); for the last mode row-major.
__host__ __device__ __forceinline__ i64 panel_addr(i64 s, i64 c, i64 R, i64 cols) {
  const i64 a = s / R, b = s - a * R;
  return (a * cols + c) * R + b;
}

// Kolda-Bader column index of the storage position (a, b) of mode n
// (tensor.hpp:14-18): j = colmajor_rank(low digits of a) + L * colmajor_rank(high digits of b).
struct KoldaMap {
  int n_low = 0, n_high = 0;
  i64 low_ext[8];
  i64 high_ext[8];
  i64 L = 1;
  // slab of a sharded tensor: the last high digit is local, the global
  // column rank adds high_last_off times that digit's stride (the last
  // digit's stride does not depend on its own extent)
  i64 high_last_off = 0;
};

__host__ __device__ inline i64 colmajor_rank(i64 rowmajor, const i64* ext, int k) {
  // digits of `rowmajor` in row-major order over ext[0..k) (last fastest);
  // rank with first digit fastest.
  i64 rank = 0, stride = 1;
  i64 digits[8];
  for (int m = k - 1; m >= 0; --m) {
    digits[m] = rowmajor % ext[m];
    rowmajor /= ext[m];
  }
  for (int m = 0; m < k; ++m) {
    rank += digits[m] * stride;
    stride *= ext[m];
  }
  return rank;
}

__host__ __device__ inline i64 kolda_index(const KoldaMap& km, i64 a, i64 b) {
  i64 hi = colmajor_rank(b, km.high_ext, km.n_high);
  if (km.high_last_off != 0) {
    i64 stride = 1;
    for (int m = 0; m + 1 < km.n_high; ++m) stride *= km.high_ext[m];
    hi += km.high_last_off * stride;
  }
  return colmajor_rank(a, km.low_ext, km.n_low) + km.L * hi;
}

// Inverse: Kolda column j -> storage row s = a*R + b.
__host__ __device__ inline i64 kolda_inverse(const KoldaMap& km, i64 j, i64 R) {
  i64 jl = j % km.L, jh = j / km.L;
  // col-major digits (first fastest) -> row-major rank (last fastest)
  i64 a = 0, b = 0;
  {
    i64 digits[8];
    for (int m = 0; m < km.n_low; ++m) {
      digits[m] = jl % km.low_ext[m];
      jl /= km.low_ext[m];
    }
    for (int m = 0; m < km.n_low; ++m) a = a * km.low_ext[m] + digits[m];
  }
  {
    i64 digits[8];
    for (int m = 0; m < km.n_high; ++m) {
      digits[m] = jh % km.high_ext[m];
      jh /= km.high_ext[m];
    }
    for (int m = 0; m < km.n_high; ++m) b = b * km.high_ext[m] + digits[m];
  }
  return a * R + b;
}

}  // namespace rcpg
