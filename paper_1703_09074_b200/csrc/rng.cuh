// SPDX-License-Identifier: MIT
// Counter form of the reference's random streams (random.hpp:16-107).
//
// RandomStream(seed, id) is SplitMix64 started at s0 = derive_seed(seed, id);
// its k-th draw (0-based) is mix64(s0 + (k+1) * gamma) (mod 2^64), so any
// entry of any stream is random-access. normal() pairs draws: normal #e uses
// pair p = e/2 with u1 = ((d_2p >> 11) + 1) 2^-53, u2 = (d_2p+1 >> 11) 2^-53,
// r = sqrt(-2 log u1), theta = (2 pi) u2; even e -> r cos(theta), odd e ->
// r sin(theta) (random.hpp:75-87). uniform_sym #e = 2 (d_e >> 11) 2^-53 - 1.
// SplitMix64 arithmetic is bit-exact; log/sin/cos are CUDA libm (<= 1-2 ulp
// from glibc), the only source of Omega differences.
#pragma once

#include <cstdint>

namespace rcpg {

constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// random.hpp:54-56
__host__ __device__ __forceinline__ std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t salt) {
  return mix64(seed + kGamma * (salt + 1));
}

// random.hpp:48-50
__host__ __device__ __forceinline__ std::uint64_t stream_id(std::uint64_t domain, std::uint64_t k) {
  return (domain << 32) | k;
}

constexpr std::uint64_t kDomainCompress = 1, kDomainInit = 2, kDomainFactors = 3, kDomainNoise = 4;

__device__ __forceinline__ std::uint64_t draw(std::uint64_t s0, std::uint64_t k) {
  return mix64(s0 + (k + 1) * kGamma);
}

// Box-Muller pair p of the stream: (r cos theta, r sin theta).
__device__ __forceinline__ void normal_pair(std::uint64_t s0, std::uint64_t p, double& c, double& s) {
  const std::uint64_t d1 = draw(s0, 2 * p);
  const std::uint64_t d2 = draw(s0, 2 * p + 1);
  const double u1 = static_cast<double>((d1 >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(d2 >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double theta = 6.283185307179586476925286766559 * u2;  // (2.0 * pi) * u2, 2*pi exact in double
  double sn, cs;
  sincos(theta, &sn, &cs);
  c = r * cs;
  s = r * sn;
}

__device__ __forceinline__ double normal_at(std::uint64_t s0, std::uint64_t e) {
  double c, s;
  normal_pair(s0, e >> 1, c, s);
  return (e & 1) ? s : c;
}

__device__ __forceinline__ double uniform_sym_at(std::uint64_t s0, std::uint64_t e) {
  const double u = static_cast<double>(draw(s0, e) >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
}

}  // namespace rcpg
