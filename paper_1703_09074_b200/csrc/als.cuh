// SPDX-License-Identifier: MIT
// CP-ALS on the (compressed) tensor, solve.hpp:62-262, and the Kruskal-model
// kernels of kruskal.hpp (normalize, recover, relative_error).
#pragma once

#include "common.cuh"

namespace rcpg {

constexpr int kMaxOrder = 8;
constexpr int kMaxRank = 128;

// Device-side ALS control block (one per solve).
struct AlsState {
  int it;          // next iteration (1-based)
  int done;
  int converged;
  int error_it;    // > 0 (or 0 for input errors): SolverError iteration
  int pivots_fallback;  // number of pinv_psd calls that needed the eigen path
  int pad;
  double prev_fit;
  double nx2;      // ||B||^2 (double)
  unsigned long long t0;  // globaltimer at solver start (ns)
};

template <typename T>
struct FactorSet {
  T* f[kMaxOrder];     // factor m: extent[m] x rank, column-major
  T* gram[kMaxOrder];  // R x R (Scalar-rounded), column-major
  i64 extent[kMaxOrder];
  int order;
  int rank;
};

// Materializes the Khatri-Rao panel K[a, r, b] = prod_{k != m} A_k[i_k, r]
// (khatri_rao_all_but, kruskal.hpp:52-64) in the (a, c, b) panel layout of
// mode m of `shape`, so MTTKRP = sketch(B, view_m, K, rank).
template <typename T>
void kr_panel(const FactorSet<T>& fs, const i64* shape, int mode, T* out, cudaStream_t st,
              const int* skip = nullptr);

// init_factors (solve.hpp:93-131) for modes >= 1, each from its Gram matrix
// G = B_(m) B_(m)^T (extent x extent, T, column-major), one CTA per mode:
// leading eigenvectors, sign-canonicalized, padded from the init stream.
// Writes each factor and its Gram; work[q] >= init_work_doubles(n[q]).
template <typename T>
struct InitBatch {
  const T* G[kMaxOrder];
  int n[kMaxOrder];
  int mode[kMaxOrder];
  T* F[kMaxOrder];
  T* gram[kMaxOrder];
  double* work[kMaxOrder];
};
template <typename T>
void init_factors_from_grams(const InitBatch<T>& b, int count, int rank, u64 seed, int method, cudaStream_t st);
// doubles of `work` one mode of extent n needs
size_t init_work_doubles(int n);

// theorem_bound (diagnostics.hpp:36-62): per mode q, the tail energy
// sum_{j >= k} sigma_j^2 of the unfolding from the eigenvalues of its Gram
// G[q] (n[q] x n[q], fp64, n <= 2048); work[q] >= init_work_doubles(n[q]).
struct TailBatch {
  const double* G[kMaxOrder];
  int n[kMaxOrder];
  double* work[kMaxOrder];
};
void gram_tails(const TailBatch& b, int count, int k, double* out, cudaStream_t st);
template <typename T>
void zero_factor(T* factor, i64 extent, int rank, T* gram_out, cudaStream_t st);

// One ALS mode update (solve.hpp:207-230) plus, for the last mode, the fit /
// stopping test (solve.hpp:232-254). W = MTTKRP result (extent x rank).
template <typename T>
void als_update(const FactorSet<T>& fs, int mode, const T* W, T* weights, double tol, int max_iter,
                double* trace_fit, double* trace_sec, AlsState* state, double* work, cudaStream_t st);

void als_start(AlsState* state, double* nx2_src, cudaStream_t st);
template <typename T>
void als_prepare(AlsState* state, double* nx2_src, T* factor0, i64 extent0, int rank, T* gram0, T* weights, T wval,
                 cudaStream_t st);
template <typename T>
void fill_ones(T* p, int n, cudaStream_t st);

// The whole ALS iteration loop as one cooperative kernel (when the mode
// extents and rank fit its shared-memory plan; see als_loop_supported).
template <typename T>
bool als_loop_supported(const i64* shape, int order, int rank);
template <typename T>
void als_loop(const T* B, const i64* shape, int order, const FactorSet<T>& fs, T* weights, double tol, int max_iter,
              double* trace_fit, double* trace_sec, AlsState* state, double* part, i64 part_elems, GridBarrier* bar,
              cudaStream_t st, unsigned long long* prof = nullptr);

// normalize (kruskal.hpp:117-176) in place; `tmp` >= sum extents * rank + rank elements.
template <typename T>
void normalize_model(const FactorSet<T>& fs, T* weights, T* tmp, cudaStream_t st);

// out = Q (dim x l) * A (l x rank), column-major (recover, kruskal.hpp:198-220).
template <typename T>
void small_gemm(const T* Q, i64 dim, i64 l, const T* A, int rank, T* out, cudaStream_t st);
template <typename T>
struct SmallGemmBatch {
  const T* Q[kMaxOrder];
  const T* A[kMaxOrder];
  T* out[kMaxOrder];
  i64 dim[kMaxOrder], l[kMaxOrder];
};
template <typename T>
void small_gemm_batch(const SmallGemmBatch<T>& b, int count, int rank, cudaStream_t st);

// Sum of squares (double) and count of non-finite entries of a device array.
template <typename T>
void norm_and_finite(const T* x, i64 n, double* out2 /* [2]: sumsq, nonfinite */, double* scratch,
                     int num_sms, cudaStream_t st, const double* cond = nullptr);
// flag <- count of CTAs that saw a non-finite entry of y (zeroed first)
template <typename T>
void nonfinite_flag(const T* y, i64 n, double* flag, cudaStream_t st);

// ||X - model||^2 and ||X||^2 (double), streamed over X (relative_error,
// kruskal.hpp:187-194, accumulated in double). out2 = {resid2, x2}.
template <typename T>
void residual_norms(const T* X, const i64* shape, int order, const FactorSet<T>& fs, const T* weights,
                    double* out2, double* scratch, int num_sms, cudaStream_t st);
size_t residual_scratch_doubles(int num_sms, i64 last_extent, int rank);


// Dense reconstruction of a model given in double + add_noise (synthetic data).
template <typename T>
void synth_tensor(const i64* shape, int order, int rank, const double* w_dev, const double* const* f_dev,
                  double snr, u64 noise_seed, T* out, double* scratch, int num_sms, cudaStream_t st);

}  // namespace rcpg
