// Reference-style usage of the drop-in header (mirrors proj/README.md:50-71 and
// test_solve.cpp): builds against include/rcp_b200/rcp.hpp + librcpg.so.
#include <cmath>
#include <cstdio>
#include <random>

#include "rcp_b200/rcp.hpp"

int main() {
  // rank-3 model plus noise, 40 x 36 x 32, row-major like rcp::Tensor
  const rcp::Shape shape{40, 36, 32};
  std::mt19937_64 gen(0x5eed);
  std::normal_distribution<double> nd;
  std::vector<std::vector<double>> A(3);
  for (int m = 0; m < 3; ++m) {
    A[m].resize(size_t(shape[m]) * 3);
    for (auto& v : A[m]) v = nd(gen);
  }
  std::vector<double> x(size_t(40 * 36 * 32));
  for (int i = 0; i < 40; ++i)
    for (int j = 0; j < 36; ++j)
      for (int k = 0; k < 32; ++k) {
        double s = 0;
        for (int r = 0; r < 3; ++r) s += A[0][i + 40 * r] * A[1][j + 36 * r] * A[2][k + 32 * r];
        x[size_t((i * 36 + j) * 32 + k)] = s + 0.01 * nd(gen);
      }
  rcp::Tensor<double> t(shape, x);
  rcp::DecomposeConfig cfg;
  cfg.rank = 3;
  cfg.tol = 1e-10;
  cfg.seed = 7;
  cfg.compress.seed = rcp::derive_seed(7, rcp::stream_id(rcp::StreamDomain::compress));
  auto [model, trace] = rcp::decompose(t, cfg);
  std::printf("iters=%d converged=%d error=%.12f\n", trace.iterations, int(trace.converged),
              trace.final_relative_error);
  if (!(trace.final_relative_error < 0.05)) return 1;
  const double e2 = rcp::relative_error(t, model);
  if (std::abs(e2 - trace.final_relative_error) > 1e-12) return 2;
  // error mapping: std::invalid_argument like the reference (solve.hpp:390-392)
  try {
    rcp::DecomposeConfig bad = cfg;
    bad.compress.target_rank = 4;
    rcp::decompose(t, bad);
    return 3;
  } catch (const std::invalid_argument&) {
  }
  auto comp = rcp::compress(t, cfg.compress.target_rank ? cfg.compress : [] {
    rcp::CompressConfig c;
    c.target_rank = 3;
    return c;
  }());
  std::printf("compressed %lldx%lldx%lld\n", (long long)comp.compressed.extent(0),
              (long long)comp.compressed.extent(1), (long long)comp.compressed.extent(2));
  // projection_residual (compress.hpp:148-164) of that compression
  const double pr = rcp::projection_residual(t, comp);
  std::printf("projection_residual=%.6f\n", pr);
  if (!(pr > 0 && pr < 0.05 * std::sqrt(double(x.size())))) return 4;
  // the BCD solver (solve.hpp:264-376) through the same entry point
  rcp::DecomposeConfig bcd = cfg;
  bcd.method = rcp::SolveMethod::bcd;
  auto [mb, tb] = rcp::decompose(t, bcd);
  std::printf("bcd iters=%d error=%.12f\n", tb.iterations, tb.final_relative_error);
  if (!(tb.final_relative_error < 0.05)) return 5;
  // als_solve (solve.hpp:183-262): the uncompressed ALS equals decompose(randomized=false)
  auto [ma, ta] = rcp::als_solve(t, cfg);
  rcp::DecomposeConfig plain = cfg;
  plain.randomized = false;
  plain.method = rcp::SolveMethod::als;
  auto [mp, tp] = rcp::decompose(t, plain);
  std::printf("als_solve iters=%d error=%.12f\n", ta.iterations, ta.final_relative_error);
  if (ta.iterations != tp.iterations || ta.final_relative_error != tp.final_relative_error) return 7;
  // recover (kruskal.hpp:198-220) of a solve on the compressed tensor through the compress bases
  rcp::DecomposeConfig small = plain;
  small.rank = 3;
  auto [mc, tc] = rcp::decompose(comp.compressed, small);
  auto full = rcp::recover(mc, comp.bases);
  const double rerr = rcp::relative_error(t, full);
  std::printf("recover rows=%lld error=%.6f\n", (long long)full.factors[0].rows(), rerr);
  if (full.factors[0].rows() != t.extent(0) || !(rerr < 0.05)) return 8;
  // validate_bound (diagnostics.hpp:68-86) on this tensor
  const auto rep = rcp::validate_bound(t, 2, 3, 4, 11);
  std::printf("bound=%.6f empirical=%.6f\n", rep.bound, rep.empirical_mean);
  if (!(rep.empirical_mean <= rep.bound)) return 6;
  return 0;
}
