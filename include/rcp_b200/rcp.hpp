// SPDX-License-Identifier: MIT
// Drop-in C++ front end for the B200 rCP path: the reference's `namespace rcp`
// entry points for rcp::decompose / rcp::compress / rcp::relative_error
// (/root/reference/proj/include/rcp/{solve,compress,kruskal}.hpp), same names,
// same argument meaning and exceptions, implemented over the C ABI in
// include/rcpg.h (link with -lrcpg). Eigen is not required: Matrix/Vector are
// minimal column-major stand-ins exposing the members callers use
// (rows, cols, operator(), data, size).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../rcpg.h"

namespace rcp {

using Index = std::int64_t;
using Shape = std::vector<Index>;

template <typename S>
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index r, Index c) : r_(r), c_(c), v_(std::size_t(r * c), S(0)) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  S& operator()(Index i, Index j) { return v_[std::size_t(i + j * r_)]; }
  const S& operator()(Index i, Index j) const { return v_[std::size_t(i + j * r_)]; }
  S* data() { return v_.data(); }
  const S* data() const { return v_.data(); }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<S> v_;
};

template <typename S>
using Vector = std::vector<S>;

// tensor.hpp:19-108 (row-major values, last index fastest)
template <typename S>
class Tensor {
 public:
  Tensor() = default;
  Tensor(Shape shape, std::vector<S> values) : shape_(std::move(shape)), values_(std::move(values)) {}
  Index order() const { return Index(shape_.size()); }
  const Shape& shape() const { return shape_; }
  Index extent(Index m) const { return shape_[std::size_t(m)]; }
  Index size() const { return Index(values_.size()); }
  const std::vector<S>& values() const { return values_; }
  std::vector<S>& values() { return values_; }
  const S* data() const { return values_.data(); }

 private:
  Shape shape_;
  std::vector<S> values_;
};

enum class RandomDistribution { gaussian = RCPG_GAUSSIAN, uniform = RCPG_UNIFORM };
enum class PowerStabilizer { lu = RCPG_STAB_LU, qr = RCPG_STAB_QR };
enum class SolveMethod { als = RCPG_ALS, bcd = RCPG_BCD };
enum class InitMethod { eigenvectors = RCPG_INIT_EIGENVECTORS, random = RCPG_INIT_RANDOM };

// compress.hpp:23-33
struct CompressConfig {
  Index target_rank = 0;
  Index oversampling = 10;
  int power_iterations = 2;
  std::optional<std::vector<Index>> modes;
  RandomDistribution distribution = RandomDistribution::gaussian;
  PowerStabilizer stabilizer = PowerStabilizer::lu;
  std::uint64_t seed = 0;
};

// solve.hpp:22-31
struct DecomposeConfig {
  Index rank = 1;
  SolveMethod method = SolveMethod::als;
  bool randomized = true;
  CompressConfig compress;
  double tol = 1e-5;
  int max_iter = 500;
  std::uint64_t seed = 0;
  InitMethod init = InitMethod::eigenvectors;
};

template <typename S>
struct Kruskal {
  Vector<S> weights;
  std::vector<Matrix<S>> factors;
  Index rank() const { return Index(weights.size()); }
  Index order() const { return Index(factors.size()); }
};

// solve.hpp:35-45
struct FitTrace {
  struct Entry {
    int iteration;
    double fit;
    double seconds;
  };
  std::vector<Entry> entries;
  double final_relative_error = std::numeric_limits<double>::quiet_NaN();
  int iterations = 0;
  bool converged = false;
};

// solve.hpp:48-57
class SolverError : public std::runtime_error {
 public:
  SolverError(const std::string& message, int iteration) : std::runtime_error(message), iteration_(iteration) {}
  int iteration() const { return iteration_; }

 private:
  int iteration_;
};

// types.hpp:60-76
template <typename S>
struct ModeBasis {
  Matrix<S> q;
  bool identity = false;
  Index dim = 0;
  bool rank_warning = false;
};

template <typename S>
struct CompressionResult {
  Tensor<S> compressed;
  std::vector<ModeBasis<S>> bases;
};

namespace detail {

template <typename S>
constexpr rcpg_dtype dtype() {
  static_assert(std::is_same_v<S, float> || std::is_same_v<S, double>, "rcp: float or double");
  return std::is_same_v<S, double> ? RCPG_F64 : RCPG_F32;
}

// One context per thread (rcpg is single-stream per context).
inline rcpg_context* context() {
  struct Holder {
    rcpg_context* ctx = nullptr;
    ~Holder() {
      if (ctx) rcpg_destroy(ctx);
    }
  };
  static thread_local Holder h;
  if (!h.ctx && rcpg_create(0, &h.ctx) != RCPG_OK) throw std::runtime_error("rcp: no usable CUDA device");
  return h.ctx;
}

inline void check(rcpg_context* c, rcpg_status st) {
  if (st == RCPG_OK) return;
  const std::string msg = rcpg_last_error(c);
  if (st == RCPG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == RCPG_SOLVER_ERROR) throw SolverError(msg, rcpg_last_error_iteration(c));
  throw std::runtime_error(msg);
}

struct CCompress {
  rcpg_compress_config c{};
  std::vector<std::int64_t> modes;
  explicit CCompress(const CompressConfig& cfg) {
    c.target_rank = cfg.target_rank;
    c.oversampling = cfg.oversampling;
    c.power_iterations = cfg.power_iterations;
    c.distribution = int32_t(cfg.distribution);
    c.stabilizer = int32_t(cfg.stabilizer);
    c.seed = cfg.seed;
    if (cfg.modes) {
      modes.assign(cfg.modes->begin(), cfg.modes->end());
      c.modes_present = 1;
      c.n_modes = std::int64_t(modes.size());
      c.modes = modes.empty() ? nullptr : modes.data();
    }
  }
};

struct DeviceTensor {
  rcpg_context* c;
  rcpg_tensor* t = nullptr;
  template <typename S>
  DeviceTensor(rcpg_context* ctx, const Tensor<S>& x) : c(ctx) {
    check(c, rcpg_tensor_upload(c, dtype<S>(), int32_t(x.order()), x.shape().data(), x.data(), &t));
  }
  ~DeviceTensor() { rcpg_tensor_free(t); }
};

}  // namespace detail

// solve.hpp:381-398
template <typename S>
std::pair<Kruskal<S>, FitTrace> decompose(const Tensor<S>& t, const DecomposeConfig& cfg) {
  rcpg_context* c = detail::context();
  detail::CCompress cc(cfg.compress);
  rcpg_decompose_config d{};
  d.rank = cfg.rank;
  d.method = int32_t(cfg.method);
  d.randomized = cfg.randomized ? 1 : 0;
  d.compress = cc.c;
  d.tol = cfg.tol;
  d.max_iter = cfg.max_iter;
  d.init = int32_t(cfg.init);
  d.seed = cfg.seed;
  const Index R = cfg.rank > 0 ? cfg.rank : 1;
  Index sum_ext = 0;
  for (Index e : t.shape()) sum_ext += e;
  std::vector<S> w(static_cast<std::size_t>(R)), f(static_cast<std::size_t>(sum_ext * R));
  const int cap = cfg.max_iter > 0 ? cfg.max_iter : 1;
  std::vector<int32_t> it(static_cast<std::size_t>(cap));
  std::vector<double> fit(static_cast<std::size_t>(cap)), sec(static_cast<std::size_t>(cap));
  rcpg_result res{};
  res.weights = w.data();
  res.factors = f.data();
  res.trace_iteration = it.data();
  res.trace_fit = fit.data();
  res.trace_seconds = sec.data();
  res.trace_capacity = cap;
  // the upload is enqueued in front of the decomposition (one synchronization, at the end of the call)
  detail::check(c, rcpg_decompose_host(c, detail::dtype<S>(), int32_t(t.order()), t.shape().data(), t.data(), &d, &res));
  Kruskal<S> model;
  model.weights = w;
  Index off = 0;
  for (Index e : t.shape()) {
    Matrix<S> m(e, R);
    for (Index i = 0; i < e * R; ++i) m.data()[i] = f[std::size_t(off + i)];
    off += e * R;
    model.factors.push_back(std::move(m));
  }
  FitTrace trace;
  for (int i = 0; i < std::min(res.iterations, cap); ++i) trace.entries.push_back({it[size_t(i)], fit[size_t(i)], sec[size_t(i)]});
  trace.iterations = res.iterations;
  trace.converged = res.converged != 0;
  trace.final_relative_error = res.final_relative_error;
  return {std::move(model), trace};
}

// solve.hpp:183-262: CP-ALS on t itself (no compression)
template <typename S>
std::pair<Kruskal<S>, FitTrace> als_solve(const Tensor<S>& t, const DecomposeConfig& cfg) {
  DecomposeConfig d = cfg;
  d.randomized = false;
  d.method = SolveMethod::als;
  return decompose(t, d);
}

// kruskal.hpp:198-220: A_n = Q_n A~_n (identity modes copied), then normalize
template <typename S>
Kruskal<S> recover(const Kruskal<S>& k, const std::vector<ModeBasis<S>>& bases) {
  rcpg_context* c = detail::context();
  const int32_t order = int32_t(k.order());
  if (Index(bases.size()) != k.order()) throw std::invalid_argument("recover: need exactly one basis per mode");
  std::vector<int64_t> sext, dims, cols;
  std::vector<int32_t> ident;
  std::vector<S> f, q;
  for (Index m = 0; m < k.order(); ++m) {
    const auto& fm = k.factors[std::size_t(m)];
    const auto& b = bases[std::size_t(m)];
    sext.push_back(fm.rows());
    f.insert(f.end(), fm.data(), fm.data() + fm.size());
    ident.push_back(b.identity ? 1 : 0);
    dims.push_back(b.identity ? b.dim : b.q.rows());
    cols.push_back(b.identity ? 0 : b.q.cols());
    if (!b.identity) q.insert(q.end(), b.q.data(), b.q.data() + b.q.size());
  }
  if (q.empty()) q.push_back(S(0));
  const Index R = k.rank();
  Index big = 0;
  for (int64_t d : dims) big += d;
  std::vector<S> ow(static_cast<std::size_t>(R)), of(static_cast<std::size_t>(big * R));
  detail::check(c, rcpg_recover(c, detail::dtype<S>(), order, R, sext.data(), k.weights.data(), f.data(),
                                ident.data(), dims.data(), cols.data(), q.data(), ow.data(), of.data()));
  Kruskal<S> out;
  out.weights = ow;
  Index off = 0;
  for (int64_t d : dims) {
    Matrix<S> mtx(d, R);
    for (Index i = 0; i < d * R; ++i) mtx.data()[i] = of[std::size_t(off + i)];
    off += d * R;
    out.factors.push_back(std::move(mtx));
  }
  return out;
}

// compress.hpp:86-146
template <typename S>
CompressionResult<S> compress(const Tensor<S>& t, const CompressConfig& cfg) {
  rcpg_context* c = detail::context();
  detail::CCompress cc(cfg);
  detail::DeviceTensor dt(c, t);
  rcpg_compressed* out = nullptr;
  detail::check(c, rcpg_compress(c, dt.t, &cc.c, &out));
  CompressionResult<S> r;
  const int32_t order = rcpg_compressed_order(out);
  Shape shape(static_cast<std::size_t>(order));
  rcpg_compressed_shape(out, shape.data());
  Index n = 1;
  for (Index e : shape) n *= e;
  std::vector<S> vals(static_cast<std::size_t>(n));
  detail::check(c, rcpg_compressed_download(c, out, vals.data()));
  r.compressed = Tensor<S>(shape, std::move(vals));
  for (int32_t m = 0; m < order; ++m) {
    int32_t ident = 0, rw = 0;
    int64_t dim = 0, cols = 0;
    rcpg_compressed_basis_info(out, m, &ident, &dim, &cols, &rw);
    ModeBasis<S> b;
    b.identity = ident != 0;
    b.dim = dim;
    b.rank_warning = rw != 0;
    if (!b.identity) {
      b.q = Matrix<S>(dim, cols);
      detail::check(c, rcpg_compressed_basis_download(c, out, m, b.q.data()));
    }
    r.bases.push_back(std::move(b));
  }
  rcpg_compressed_free(out);
  return r;
}

// kruskal.hpp:187-194
template <typename S>
S relative_error(const Tensor<S>& x, const Kruskal<S>& k) {
  rcpg_context* c = detail::context();
  std::vector<S> f;
  for (const auto& m : k.factors) f.insert(f.end(), m.data(), m.data() + m.size());
  detail::DeviceTensor dt(c, x);
  double out = 0;
  detail::check(c, rcpg_relative_error(c, dt.t, k.rank(), k.weights.data(), f.data(), &out));
  return S(out);
}

// compress.hpp:148-164
template <typename S>
S projection_residual(const Tensor<S>& t, const CompressionResult<S>& result) {
  if (Index(result.bases.size()) != t.order()) throw std::invalid_argument("projection_residual: need one basis per mode");
  rcpg_context* c = detail::context();
  std::vector<int32_t> ident;
  std::vector<int64_t> cols;
  std::vector<S> q;
  for (const auto& b : result.bases) {
    ident.push_back(b.identity ? 1 : 0);
    cols.push_back(b.identity ? 0 : b.q.cols());
    if (!b.identity) q.insert(q.end(), b.q.data(), b.q.data() + b.q.size());
  }
  detail::DeviceTensor dt(c, t);
  double out = 0;
  detail::check(c, rcpg_projection_residual_bases(c, dt.t, ident.data(), cols.data(), q.data(), &out));
  return S(out);
}

// diagnostics.hpp:23-31
struct BoundReport {
  std::vector<double> tail_energies;
  double bound = 0.0;
  double empirical_mean = std::numeric_limits<double>::quiet_NaN();
  int trials = 0;
  Index k = 0;
  Index p = 0;
};

// diagnostics.hpp:36-62 (tail energies from the eigenvalues of each unfolding's Gram)
template <typename S>
BoundReport theorem_bound(const Tensor<S>& t, Index k, Index p) {
  rcpg_context* c = detail::context();
  detail::DeviceTensor dt(c, t);
  BoundReport r;
  r.k = k;
  r.p = p;
  r.tail_energies.assign(static_cast<std::size_t>(t.order()), 0.0);
  detail::check(c, rcpg_theorem_bound(c, dt.t, k, p, r.tail_energies.data(), &r.bound));
  return r;
}

// diagnostics.hpp:68-86 on a given tensor (the reference draws random_lowrank<double>(shape,
// rank, seed) first; random_lowrank below is that generator)
template <typename S>
BoundReport validate_bound(const Tensor<S>& dense, Index k, Index p, int trials, std::uint64_t seed);

// Library options (include/rcpg.h rcpg_set_option): "fp32_arith", "omega_host", "pass_timing".
inline void set_option(const char* name, std::int64_t value) {
  rcpg_context* c = detail::context();
  detail::check(c, rcpg_set_option(c, name, value));
}

inline const char* method_name(SolveMethod m) { return m == SolveMethod::bcd ? "bcd" : "als"; }

// kruskal.hpp:117-176 (host side; models are small): unit-norm columns (left
// alone within 32 eps of 1), zero columns -> e1 with weight 0, non-negative
// weights, the largest-magnitude entry of each first-factor column
// non-negative (compensated in factor 1), stable sort by weight descending,
// ties by the lexicographically smaller first-factor column. Norms are
// accumulated in double (the documented deviation for float).
template <typename S>
Kruskal<S> normalize(Kruskal<S> k) {
  const Index r = k.rank(), n = k.order();
  if (r < 1 || n < 1) throw std::invalid_argument("normalize: model needs rank >= 1 and order >= 1");
  for (const auto& f : k.factors)
    if (f.cols() != r || f.rows() < 1) throw std::invalid_argument("normalize: factor shape does not match the rank");
  const S window = S(32) * std::numeric_limits<S>::epsilon();
  for (Index j = 0; j < r; ++j) {
    auto& w = k.weights[std::size_t(j)];
    for (Index m = 0; m < n; ++m) {
      auto& f = k.factors[std::size_t(m)];
      double ss = 0.0;
      for (Index i = 0; i < f.rows(); ++i) ss += double(f(i, j)) * double(f(i, j));
      const S nrm = S(std::sqrt(ss));
      if (nrm == S(0)) {
        for (Index i = 0; i < f.rows(); ++i) f(i, j) = S(0);
        f(0, j) = S(1);
        w = S(0);
      } else if (std::abs(nrm - S(1)) > window) {
        for (Index i = 0; i < f.rows(); ++i) f(i, j) /= nrm;
        w *= nrm;
      }
    }
    if (w < S(0)) {
      w = -w;
      for (Index i = 0; i < k.factors[0].rows(); ++i) k.factors[0](i, j) = -k.factors[0](i, j);
    }
    if (n >= 2) {
      auto& lead = k.factors[0];
      Index at = 0;
      for (Index i = 1; i < lead.rows(); ++i)
        if (std::abs(lead(i, j)) > std::abs(lead(at, j))) at = i;
      if (lead(at, j) < S(0)) {
        for (Index i = 0; i < lead.rows(); ++i) lead(i, j) = -lead(i, j);
        for (Index i = 0; i < k.factors[1].rows(); ++i) k.factors[1](i, j) = -k.factors[1](i, j);
      }
    }
  }
  std::vector<Index> ord(static_cast<std::size_t>(r));
  std::iota(ord.begin(), ord.end(), Index(0));
  const auto& lead = k.factors[0];
  std::stable_sort(ord.begin(), ord.end(), [&](Index a, Index b) {
    if (k.weights[std::size_t(a)] != k.weights[std::size_t(b)]) return k.weights[std::size_t(a)] > k.weights[std::size_t(b)];
    for (Index i = 0; i < lead.rows(); ++i)
      if (lead(i, a) != lead(i, b)) return lead(i, a) < lead(i, b);
    return false;
  });
  bool ident = true;
  for (Index j = 0; j < r; ++j) ident = ident && ord[std::size_t(j)] == j;
  if (ident) return k;
  Kruskal<S> out = k;
  for (Index j = 0; j < r; ++j) {
    const Index src = ord[std::size_t(j)];
    out.weights[std::size_t(j)] = k.weights[std::size_t(src)];
    for (Index m = 0; m < n; ++m)
      for (Index i = 0; i < k.factors[std::size_t(m)].rows(); ++i)
        out.factors[std::size_t(m)](i, j) = k.factors[std::size_t(m)](i, src);
  }
  return out;
}

namespace detail {
// Dense model (plus optional add_noise at amplitude SNR `snr` from stream
// (noise_seed, noise)) generated on the device by rcpg_synth, downloaded.
template <typename S>
Tensor<S> synth_dense(const Kruskal<S>& k, double snr, std::uint64_t noise_seed) {
  rcpg_context* c = context();
  Shape shape;
  std::vector<double> w(k.weights.begin(), k.weights.end()), f;
  for (const auto& m : k.factors) {
    shape.push_back(m.rows());
    f.insert(f.end(), m.data(), m.data() + m.size());
  }
  rcpg_tensor* t = nullptr;
  check(c, rcpg_synth(c, dtype<S>(), int32_t(shape.size()), shape.data(), k.rank(), w.data(), f.data(), snr,
                      noise_seed, &t));
  Index n = 1;
  for (Index e : shape) n *= e;
  std::vector<S> v(static_cast<std::size_t>(n));
  const rcpg_status st = rcpg_tensor_download(c, t, v.data());
  rcpg_tensor_free(t);
  check(c, st);
  return Tensor<S>(std::move(shape), std::move(v));
}
}  // namespace detail

// kruskal.hpp:104-110: the dense tensor of the model (computed on the GPU).
template <typename S>
Tensor<S> reconstruct(const Kruskal<S>& k) {
  if (k.rank() < 1 || k.order() < 1) throw std::invalid_argument("reconstruct: empty model");
  return detail::synth_dense(k, 0.0, 0);
}

inline std::uint64_t mix64(std::uint64_t z);
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t salt);

// random.hpp:16-107: SplitMix64 stream with Box-Muller normals (pairs cached).
class RandomStream {
 public:
  RandomStream(std::uint64_t seed, std::uint64_t id) : state_(derive_seed(seed, id)) {}
  std::uint64_t bits() {
    state_ += 0x9e3779b97f4a7c15ULL;
    return mix64(state_);
  }
  double uniform01() { return double(bits() >> 11) * 0x1.0p-53; }
  double normal() {
    if (cached_ok_) {
      cached_ok_ = false;
      return cached_;
    }
    const double u1 = double((bits() >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = uniform01();
    const double rr = std::sqrt(-2.0 * std::log(u1)), th = 2.0 * 3.14159265358979323846 * u2;
    cached_ = rr * std::sin(th);
    cached_ok_ = true;
    return rr * std::cos(th);
  }
  template <typename S>
  void fill_gaussian(Matrix<S>& m) {  // column-major order
    for (Index j = 0; j < m.cols(); ++j)
      for (Index i = 0; i < m.rows(); ++i) m(i, j) = S(normal());
  }

 private:
  std::uint64_t state_;
  double cached_ = 0.0;
  bool cached_ok_ = false;
};

inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// random.hpp:48-56
enum class StreamDomain : std::uint64_t { compress = 1, init = 2, factors = 3, noise = 4, phases = 5, trial = 6 };
inline std::uint64_t stream_id(StreamDomain d, std::uint64_t k = 0) { return (std::uint64_t(d) << 32) | k; }
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t salt) {
  return mix64(seed + 0x9e3779b97f4a7c15ULL * (salt + 1));
}

// synthetic.hpp:21-38: N(0, 1) factors from stream (seed, factors, m), unit
// weights, normalized, reconstructed (on the GPU). With snr > 0 the
// add_noise step (synthetic.hpp:42-58, stream (noise_seed, noise)) is fused
// into the same device pass (the CLI's `synth --snr`).
template <typename S>
std::pair<Tensor<S>, Kruskal<S>> random_lowrank(const Shape& shape, Index rank, std::uint64_t seed, double snr = 0.0,
                                                std::uint64_t noise_seed = 0) {
  if (rank < 1) throw std::invalid_argument("random_lowrank: rank must be at least 1");
  if (shape.empty()) throw std::invalid_argument("random_lowrank: shape must not be empty");
  Kruskal<S> truth;
  truth.weights.assign(static_cast<std::size_t>(rank), S(1));
  for (std::size_t m = 0; m < shape.size(); ++m) {
    if (shape[m] < 1) throw std::invalid_argument("random_lowrank: extents must be positive");
    RandomStream rs(seed, stream_id(StreamDomain::factors, m));
    Matrix<S> f(shape[m], rank);
    rs.fill_gaussian(f);
    truth.factors.push_back(std::move(f));
  }
  truth = normalize(std::move(truth));
  return {detail::synth_dense(truth, snr, noise_seed), truth};
}

template <typename S>
BoundReport validate_bound(const Tensor<S>& dense, Index k, Index p, int trials, std::uint64_t seed) {
  if (trials < 1) throw std::invalid_argument("validate_bound: need at least one trial");
  BoundReport report = theorem_bound(dense, k, p);
  report.trials = trials;
  double sum = 0.0;
  for (int trial = 0; trial < trials; ++trial) {
    CompressConfig cfg;
    cfg.target_rank = k;
    cfg.oversampling = p;
    cfg.power_iterations = 0;
    cfg.seed = derive_seed(seed, stream_id(StreamDomain::trial, static_cast<std::uint64_t>(trial)));
    sum += double(projection_residual(dense, compress(dense, cfg)));
  }
  report.empirical_mean = sum / trials;
  return report;
}

}  // namespace rcp
