// SPDX-License-Identifier: MIT
// Omega generated on the host and uploaded (rcpg_set_option "omega_host").
//
// The device generator (passes.cu, rng.cuh) evaluates the reference's
// Box-Muller stream with CUDA's log / sincos, which differ from glibc's in the
// last ulp for ~0.1% of draws (measured: glibc itself is not correctly rounded,
// so no device libm can reproduce it bit for bit). north_star allows the other
// route: this file evaluates RandomStream::normal() (random.hpp:75-87) with the
// host's std::log / std::sqrt / std::sin / std::cos -- the same libm calls, in
// the same order, as the reference -- so the uploaded Omega is bit-identical to
// the reference's fill_gaussian / fill_uniform (random.hpp:90-101), cast to the
// Scalar type as compress.hpp:118-124 does. Entries are random-access through
// the SplitMix64 counter form, so the work splits over host threads.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "common.cuh"
#include "rng.cuh"

namespace rcpg {

namespace {

constexpr double kPi = 3.14159265358979323846;

inline std::uint64_t host_draw(std::uint64_t s0, std::uint64_t k) { return mix64(s0 + (k + 1) * kGamma); }

// RandomStream::normal() pair p: (r cos theta, r sin theta), random.hpp:80-85
inline void host_normal_pair(std::uint64_t s0, std::uint64_t p, double& c, double& s) {
  const double u1 = static_cast<double>((host_draw(s0, 2 * p) >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(host_draw(s0, 2 * p + 1) >> 11) * 0x1.0p-53;
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double theta = 2.0 * kPi * u2;  // kPi == std::numbers::pi
  s = r * std::sin(theta);
  c = r * std::cos(theta);
}

}  // namespace

// Fills the (a, c, b) panel of mode view v (rows s = a R + b, Kolda row j =
// kolda_index(km, a, b)): entry (s, c) = draw #(c Jg + j) of the stream.
// out_kind: 0 float, 1 double, 2 double holding the float-rounded value.
void omega_host_panel(u64 seed, i64 mode, const KoldaMap& km, ModeView v, i64 cols, int distribution, i64 Jg,
                      int out_kind, void* host_out) {
  const u64 s0 = derive_seed(seed, stream_id(kDomainCompress, u64(mode)));
  const i64 J = v.L * v.R;
  if (Jg <= 0) Jg = J;
  auto store = [&](i64 s, i64 c, double x) {
    const i64 a = s / v.R, b = s - a * v.R;
    const i64 at = (a * cols + c) * v.R + b;
    if (out_kind == 0)
      static_cast<float*>(host_out)[at] = static_cast<float>(x);
    else if (out_kind == 1)
      static_cast<double*>(host_out)[at] = x;
    else
      static_cast<double*>(host_out)[at] = double(static_cast<float>(x));
  };
  const unsigned nth = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nth; ++t) {
    pool.emplace_back([&, t] {
      // rows s of this thread: [s_lo, s_hi)
      const i64 s_lo = J * i64(t) / i64(nth), s_hi = J * i64(t + 1) / i64(nth);
      for (i64 c = 0; c < cols; ++c)
        for (i64 s = s_lo; s < s_hi; ++s) {
          const i64 a = s / v.R, b = s - a * v.R;
          const u64 e = u64(c) * u64(Jg) + u64(kolda_index(km, a, b));
          double x;
          if (distribution == 0) {
            double cs, sn;
            host_normal_pair(s0, e >> 1, cs, sn);
            x = (e & 1) ? sn : cs;
          } else {
            x = 2.0 * (static_cast<double>(host_draw(s0, e) >> 11) * 0x1.0p-53) - 1.0;  // uniform_sym
          }
          store(s, c, x);
        }
    });
  }
  for (auto& th : pool) th.join();
}

}  // namespace rcpg
