// SPDX-License-Identifier: MIT
// ORACLE — TEST INFRASTRUCTURE ONLY (see rcp_oracle.hpp). extern "C" shim so
// the Python tests and bench.py's CPU-baseline leg can drive the C++
// restatement through ctypes. Never loaded by the product path.
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>

#include "rcp_oracle.hpp"

using namespace rcpo;

namespace {

thread_local std::string g_err;
thread_local int g_err_iter = -1;

enum : int { RO_OK = 0, RO_INVALID = 1, RO_SOLVER = 2, RO_OTHER = 3 };

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return RO_OK;
  } catch (const SolverError& e) {
    g_err = e.what();
    g_err_iter = e.iteration();
    return RO_SOLVER;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RO_INVALID;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RO_OTHER;
  }
}

Shape make_shape(int order, const std::int64_t* shape) { return Shape(shape, shape + order); }

template <typename S>
Tensor<S> make_tensor(int order, const std::int64_t* shape, const S* x) {
  Shape s = make_shape(order, shape);
  const Index n = shape_size(s);
  return Tensor<S>(s, std::vector<S>(x, x + n));
}

}  // namespace

extern "C" {

// Mirrors rcp::CompressConfig (compress.hpp:23-33). modes_present = 0 means
// "disengaged" (all modes), 1 means the list (possibly empty) is used.
struct ro_compress_cfg {
  std::int64_t target_rank;
  std::int64_t oversampling;
  std::int32_t power_iterations;
  std::int32_t distribution;
  std::int32_t stabilizer;
  std::int32_t modes_present;
  std::int64_t n_modes;
  const std::int64_t* modes;
  std::uint64_t seed;
};

// Mirrors rcp::DecomposeConfig (solve.hpp:22-31).
struct ro_decompose_cfg {
  std::int64_t rank;
  std::int32_t method;
  std::int32_t randomized;
  ro_compress_cfg compress;
  double tol;
  std::int32_t max_iter;
  std::int32_t init;
  std::uint64_t seed;
};

const char* ro_last_error() { return g_err.c_str(); }
int ro_last_error_iteration() { return g_err_iter; }

std::uint64_t ro_mix64(std::uint64_t z) { return mix64(z); }
std::uint64_t ro_derive_seed(std::uint64_t seed, std::uint64_t salt) { return derive_seed(seed, salt); }
std::uint64_t ro_stream_id(std::uint64_t domain, std::uint64_t k) {
  return (domain << 32) | k;
}

// n sequential RandomStream(seed, id) draws: kind 0 = normal(), 1 = uniform01(),
// 2 = uniform_sym(), 3 = bits() (as double-reinterpreted uint64 in out_bits).
void ro_stream_draws(std::uint64_t seed, std::uint64_t id, int kind, std::int64_t n, double* out,
                     std::uint64_t* out_bits) {
  RandomStream rs(seed, id);
  for (std::int64_t i = 0; i < n; ++i) {
    if (kind == 0) out[i] = rs.normal();
    else if (kind == 1) out[i] = rs.uniform01();
    else if (kind == 2) out[i] = rs.uniform_sym();
    else out_bits[i] = rs.bits();
  }
}

// Omega_n exactly as compress.hpp:118-124 (column-major rows x cols).
void ro_sketch_matrix_d(std::uint64_t seed, std::int64_t mode, std::int64_t rows, std::int64_t cols,
                        int dist, double* out) {
  auto m = sketch_matrix<double>(seed, mode, rows, cols, RandomDistribution(dist));
  std::memcpy(out, m.data(), sizeof(double) * std::size_t(rows * cols));
}
void ro_sketch_matrix_f(std::uint64_t seed, std::int64_t mode, std::int64_t rows, std::int64_t cols,
                        int dist, float* out) {
  auto m = sketch_matrix<float>(seed, mode, rows, cols, RandomDistribution(dist));
  std::memcpy(out, m.data(), sizeof(float) * std::size_t(rows * cols));
}

int ro_unfold_d(int order, const std::int64_t* shape, const double* x, std::int64_t mode, double* out) {
  return guarded([&] {
    auto t = make_tensor(order, shape, x);
    auto m = unfold(t, mode);
    std::memcpy(out, m.data(), sizeof(double) * std::size_t(m.size()));
  });
}

int ro_fold_d(int order, const std::int64_t* shape, const double* m_in, std::int64_t rows,
              std::int64_t cols, std::int64_t mode, double* out) {
  return guarded([&] {
    Matrix<double> m(rows, cols);
    std::memcpy(m.data(), m_in, sizeof(double) * std::size_t(rows * cols));
    auto t = fold(m, mode, make_shape(order, shape));
    std::memcpy(out, t.values.data(), sizeof(double) * t.values.size());
  });
}

int ro_khatri_rao_d(std::int64_t ar, std::int64_t ac, const double* a, std::int64_t br, std::int64_t bc,
                    const double* b, double* out) {
  return guarded([&] {
    Matrix<double> A(ar, ac), B(br, bc);
    std::memcpy(A.data(), a, sizeof(double) * std::size_t(ar * ac));
    std::memcpy(B.data(), b, sizeof(double) * std::size_t(br * bc));
    auto k = khatri_rao(A, B);
    std::memcpy(out, k.data(), sizeof(double) * std::size_t(k.size()));
  });
}

#define RO_MATFN(NAME, S, EXPR)                                                              \
  int NAME(std::int64_t rows, std::int64_t cols, const S* in, S* out, int* rank_warning) {   \
    return guarded([&] {                                                                     \
      Matrix<S> m(rows, cols);                                                               \
      std::memcpy(m.data(), in, sizeof(S) * std::size_t(rows * cols));                       \
      bool rw = false;                                                                       \
      (void)rw;                                                                              \
      Matrix<S> r = EXPR;                                                                    \
      if (rank_warning) *rank_warning = rw ? 1 : 0;                                          \
      std::memcpy(out, r.data(), sizeof(S) * std::size_t(r.size()));                         \
    });                                                                                      \
  }
RO_MATFN(ro_plu_basis_d, double, detail::plu_basis(m))
RO_MATFN(ro_plu_basis_f, float, detail::plu_basis(m))
RO_MATFN(ro_thin_qr_d, double, detail::thin_qr(m, &rw))
RO_MATFN(ro_thin_qr_f, float, detail::thin_qr(m, &rw))
RO_MATFN(ro_pinv_psd_d, double, pinv_psd(m))
RO_MATFN(ro_pinv_psd_f, float, pinv_psd(m))
#undef RO_MATFN

// Symmetric eigendecomposition used by pinv_psd / init_factors.
void ro_sym_eig(int n, const double* a, double* evals, double* vecs) { sym_eig(n, a, evals, vecs); }

}  // extern "C"

namespace {

template <typename S>
CompressConfig to_cc(const ro_compress_cfg& c) {
  CompressConfig cc;
  cc.target_rank = c.target_rank;
  cc.oversampling = c.oversampling;
  cc.power_iterations = c.power_iterations;
  cc.distribution = RandomDistribution(c.distribution);
  cc.stabilizer = PowerStabilizer(c.stabilizer);
  cc.seed = c.seed;
  if (c.modes_present) cc.modes = std::vector<Index>(c.modes, c.modes + c.n_modes);
  return cc;
}

template <typename S>
DecomposeConfig to_dc(const ro_decompose_cfg& c) {
  DecomposeConfig dc;
  dc.rank = c.rank;
  dc.method = SolveMethod(c.method);
  dc.randomized = c.randomized != 0;
  dc.compress = to_cc<S>(c.compress);
  dc.tol = c.tol;
  dc.max_iter = c.max_iter;
  dc.seed = c.seed;
  dc.init = InitMethod(c.init);
  return dc;
}

// out_shape[order], out_compressed (capacity = input size), out_q: column-major
// bases concatenated (capacity = sum I_n * I_n), out_identity[order],
// out_rank_warning[order], out_qcols[order].
template <typename S>
int compress_impl(int order, const std::int64_t* shape, const S* x, const ro_compress_cfg* cfg,
                  std::int64_t* out_shape, S* out_compressed, S* out_q, int* out_identity,
                  int* out_rank_warning, std::int64_t* out_qcols) {
  return guarded([&] {
    auto t = make_tensor(order, shape, x);
    auto r = compress(t, to_cc<S>(*cfg));
    for (int m = 0; m < order; ++m) out_shape[m] = r.compressed.shape[std::size_t(m)];
    std::memcpy(out_compressed, r.compressed.values.data(), sizeof(S) * r.compressed.values.size());
    std::size_t off = 0;
    for (int m = 0; m < order; ++m) {
      const auto& b = r.bases[std::size_t(m)];
      out_identity[m] = b.identity ? 1 : 0;
      out_rank_warning[m] = b.rank_warning ? 1 : 0;
      out_qcols[m] = b.identity ? 0 : b.q.cols();
      if (!b.identity) {
        std::memcpy(out_q + off, b.q.data(), sizeof(S) * std::size_t(b.q.size()));
        off += std::size_t(b.q.size());
      }
    }
  });
}

// out_factors: column-major I_n x R concatenated; trace arrays of capacity max_iter.
template <typename S>
int decompose_impl(int order, const std::int64_t* shape, const S* x, const ro_decompose_cfg* cfg,
                   S* out_weights, S* out_factors, int* trace_it, double* trace_fit,
                   double* trace_sec, int* out_iterations, int* out_converged, double* out_relerr) {
  return guarded([&] {
    auto t = make_tensor(order, shape, x);
    auto [model, trace] = decompose(t, to_dc<S>(*cfg));
    for (Index r = 0; r < model.rank(); ++r) out_weights[r] = model.weights[std::size_t(r)];
    std::size_t off = 0;
    for (const auto& f : model.factors) {
      std::memcpy(out_factors + off, f.data(), sizeof(S) * std::size_t(f.size()));
      off += std::size_t(f.size());
    }
    for (std::size_t i = 0; i < trace.entries.size(); ++i) {
      trace_it[i] = trace.entries[i].iteration;
      trace_fit[i] = trace.entries[i].fit;
      trace_sec[i] = trace.entries[i].seconds;
    }
    *out_iterations = trace.iterations;
    *out_converged = trace.converged ? 1 : 0;
    *out_relerr = trace.final_relative_error;
  });
}

template <typename S>
int projection_residual_impl(int order, const std::int64_t* shape, const S* x, const ro_compress_cfg* cfg,
                             double* out) {
  return guarded([&] {
    auto t = make_tensor(order, shape, x);
    *out = projection_residual(t, compress(t, to_cc<S>(*cfg)));
  });
}

template <typename S>
void read_model(int order, const std::int64_t* shape, std::int64_t rank, const S* w, const S* f,
                Kruskal<S>& k) {
  k.weights.assign(w, w + rank);
  std::size_t off = 0;
  for (int m = 0; m < order; ++m) {
    Matrix<S> a(shape[m], rank);
    std::memcpy(a.data(), f + off, sizeof(S) * std::size_t(a.size()));
    off += std::size_t(a.size());
    k.factors.push_back(std::move(a));
  }
}

template <typename S>
void write_model(const Kruskal<S>& k, S* w, S* f) {
  for (Index r = 0; r < k.rank(); ++r) w[r] = k.weights[std::size_t(r)];
  std::size_t off = 0;
  for (const auto& a : k.factors) {
    std::memcpy(f + off, a.data(), sizeof(S) * std::size_t(a.size()));
    off += std::size_t(a.size());
  }
}

}  // namespace

extern "C" {

int ro_compress_d(int order, const std::int64_t* shape, const double* x, const ro_compress_cfg* cfg,
                  std::int64_t* os, double* oc, double* oq, int* oi, int* orw, std::int64_t* oqc) {
  return compress_impl<double>(order, shape, x, cfg, os, oc, oq, oi, orw, oqc);
}
int ro_compress_f(int order, const std::int64_t* shape, const float* x, const ro_compress_cfg* cfg,
                  std::int64_t* os, float* oc, float* oq, int* oi, int* orw, std::int64_t* oqc) {
  return compress_impl<float>(order, shape, x, cfg, os, oc, oq, oi, orw, oqc);
}
int ro_decompose_d(int order, const std::int64_t* shape, const double* x, const ro_decompose_cfg* cfg,
                   double* w, double* f, int* ti, double* tf, double* ts, int* it, int* conv, double* re) {
  return decompose_impl<double>(order, shape, x, cfg, w, f, ti, tf, ts, it, conv, re);
}
int ro_decompose_f(int order, const std::int64_t* shape, const float* x, const ro_decompose_cfg* cfg,
                   float* w, float* f, int* ti, double* tf, double* ts, int* it, int* conv, double* re) {
  return decompose_impl<float>(order, shape, x, cfg, w, f, ti, tf, ts, it, conv, re);
}
int ro_projection_residual_d(int order, const std::int64_t* shape, const double* x,
                             const ro_compress_cfg* cfg, double* out) {
  return projection_residual_impl<double>(order, shape, x, cfg, out);
}

// theorem_bound / validate_bound (diagnostics.hpp:36-86): tails[order], bound,
// and (trials > 0) the mean projection residual of `trials` q = 0 compressions.
int ro_validate_bound_d(int order, const std::int64_t* shape, const double* x, std::int64_t k, std::int64_t p,
                        int trials, std::uint64_t seed, double* tails, double* bound, double* mean) {
  return guarded([&] {
    auto t = make_tensor(order, shape, x);
    const BoundReport r = trials > 0 ? validate_bound_on(t, k, p, trials, seed) : theorem_bound(t, k, p);
    for (int m = 0; m < order; ++m) tails[m] = r.tail_energies[std::size_t(m)];
    *bound = r.bound;
    *mean = r.empirical_mean;
  });
}

// init_factors (solve.hpp:93-131): out = concatenated column-major I_n x R.
int ro_init_factors_d(int order, const std::int64_t* shape, const double* x, std::int64_t rank,
                      std::uint64_t seed, int method, double* out) {
  return guarded([&] {
    auto t = make_tensor(order, shape, x);
    auto fs = init_factors(t, rank, seed, InitMethod(method));
    std::size_t off = 0;
    for (const auto& f : fs) {
      std::memcpy(out + off, f.data(), sizeof(double) * std::size_t(f.size()));
      off += std::size_t(f.size());
    }
  });
}

int ro_normalize_d(int order, const std::int64_t* shape, std::int64_t rank, const double* w,
                   const double* f, double* ow, double* of) {
  return guarded([&] {
    Kruskal<double> k;
    read_model(order, shape, rank, w, f, k);
    write_model(normalize(k), ow, of);
  });
}

int ro_reconstruct_d(int order, const std::int64_t* shape, std::int64_t rank, const double* w,
                     const double* f, double* out) {
  return guarded([&] {
    Kruskal<double> k;
    read_model(order, shape, rank, w, f, k);
    auto t = reconstruct(k);
    std::memcpy(out, t.values.data(), sizeof(double) * t.values.size());
  });
}

int ro_relative_error_d(int order, const std::int64_t* shape, const double* x, std::int64_t rank,
                        const double* w, const double* f, double* out) {
  return guarded([&] {
    Kruskal<double> k;
    read_model(order, shape, rank, w, f, k);
    *out = relative_error(make_tensor(order, shape, x), k);
  });
}
int ro_relative_error_f(int order, const std::int64_t* shape, const float* x, std::int64_t rank,
                        const float* w, const float* f, double* out) {
  return guarded([&] {
    Kruskal<float> k;
    read_model(order, shape, rank, w, f, k);
    *out = relative_error(make_tensor(order, shape, x), k);
  });
}

int ro_fit_d(int order, const std::int64_t* shape, const double* x, std::int64_t rank, const double* w,
             const double* f, double* out) {
  return guarded([&] {
    Kruskal<double> k;
    read_model(order, shape, rank, w, f, k);
    *out = fit(make_tensor(order, shape, x), k);
  });
}

// random_lowrank (synthetic.hpp:21-38), optionally followed by add_noise
// (synthetic.hpp:42-58) when snr > 0 (noise seed = noise_seed).
int ro_random_lowrank_d(int order, const std::int64_t* shape, std::int64_t rank, std::uint64_t seed,
                        double snr, std::uint64_t noise_seed, double* out_tensor, double* out_w,
                        double* out_f) {
  return guarded([&] {
    auto [t, truth] = random_lowrank<double>(make_shape(order, shape), rank, seed);
    if (snr > 0) t = add_noise(t, snr, noise_seed);
    std::memcpy(out_tensor, t.values.data(), sizeof(double) * t.values.size());
    if (out_w) write_model(truth, out_w, out_f);
  });
}

int ro_add_noise_d(int order, const std::int64_t* shape, const double* x, double snr, std::uint64_t seed,
                   double* out) {
  return guarded([&] {
    auto t = add_noise(make_tensor(order, shape, x), snr, seed);
    std::memcpy(out, t.values.data(), sizeof(double) * t.values.size());
  });
}

// Synthetic ground truth for configs C2-C5 (kind 2..5), noise added with
// add_noise semantics (snr = amplitude ratio, noise stream (seed, noise)).
// Double-precision construction; out is cast to the requested type.
}  // extern "C"
namespace {
template <typename S>
int synth_impl(int kind, int order, const std::int64_t* shape, std::int64_t rank, std::uint64_t seed,
               double snr, S* out, S* out_w, S* out_f) {
  return guarded([&] {
    const Shape s = make_shape(order, shape);
    Kruskal<double> k = synth_model<double>(kind, s, rank, seed);
    Tensor<double> t = reconstruct(k);
    Tensor<S> ts(s);
    for (Index i = 0; i < t.size(); ++i) ts.values[std::size_t(i)] = S(t.values[std::size_t(i)]);
    if (snr > 0) ts = add_noise(ts, snr, seed);
    std::memcpy(out, ts.values.data(), sizeof(S) * ts.values.size());
    if (out_w) {
      Kruskal<S> ks;
      ks.weights.resize(k.weights.size());
      for (std::size_t r = 0; r < k.weights.size(); ++r) ks.weights[r] = S(k.weights[r]);
      for (const auto& f : k.factors) {
        Matrix<S> g(f.rows(), f.cols());
        for (Index i = 0; i < f.size(); ++i) g.v[std::size_t(i)] = S(f.v[std::size_t(i)]);
        ks.factors.push_back(std::move(g));
      }
      write_model(ks, out_w, out_f);
    }
  });
}
}  // namespace

extern "C" {

int ro_synth_d(int kind, int order, const std::int64_t* shape, std::int64_t rank, std::uint64_t seed,
               double snr, double* out, double* out_w, double* out_f) {
  return synth_impl<double>(kind, order, shape, rank, seed, snr, out, out_w, out_f);
}
int ro_synth_f(int kind, int order, const std::int64_t* shape, std::int64_t rank, std::uint64_t seed,
               double snr, float* out, float* out_w, float* out_f) {
  return synth_impl<float>(kind, order, shape, rank, seed, snr, out, out_w, out_f);
}

}  // extern "C"
