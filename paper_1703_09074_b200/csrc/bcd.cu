// SPDX-License-Identifier: MIT
// Block coordinate descent over rank-one components (bcd_solve,
// /root/reference/proj/include/rcp/solve.hpp:264-376): the paper's solver for
// its tables, run on the compressed tensor by decompose(method = bcd).
//
// One cooperative launch runs the whole solver. Every CTA executes the same
// control flow and makes the same decisions: every scalar it branches on
// (norms, the component fit, the overall fit) is either reduced from per-CTA
// partials in CTA order after a grid barrier, or computed identically by every
// CTA from identical data. Work split:
//   * squared norms and the elementwise residual / leave-one-out / deflation
//     updates: contiguous element ranges per CTA;
//   * the mode-m products w = Y_(m) z (kron_column_all_but, solve.hpp:150-163):
//     positions (a, b) of the (L, I, R) mode view split over CTAs, every thread
//     owning output rows i, fp64 partials per CTA reduced in CTA order;
//   * the short column updates (col = w / s, norms, lambda): redundantly on
//     every CTA from the reduced w, CTA 0 writing the factor column.
// Scalar roundings follow the reference (Scalar vectors, products rounded at
// every step, no FMA contraction: mul_rn / add_rn); reductions accumulate in
// fp64 and are rounded once (the documented deviation the oracle shares).
#include <cuda_runtime.h>

#include <algorithm>

#include "als.cuh"
#include "bcd.cuh"
#include "runtime.cuh"

namespace rcpg {

namespace {

constexpr int kBcdThreads = 256;

struct BcdShape {
  i64 e[kMaxOrder];
  int n;
};

BcdShape make_bcd_shape(const i64* shape, int order) {
  BcdShape s{};
  s.n = order;
  for (int m = 0; m < order; ++m) s.e[m] = shape[m];
  return s;
}
constexpr int kBcdCap = 200;  // inner iterations per component visit (solve.hpp:277)
constexpr int kZBatch = 256;  // positions whose Kronecker entries are formed per smem batch

template <typename T>
struct BcdArgs {
  const T* X;
  T* res;   // residual
  T* loo;   // leave-one-out residual (the y of the refinement sweeps)
  BcdShape sh;
  i64 S;
  FactorSet<T> fs;
  T* weights;
  double tol;
  int max_iter;
  double* trace_fit;
  double* trace_sec;
  AlsState* st;
  double* part;  // [2][G][max_ext + 1]
  i64 part_stride;
  GridBarrier* bar;
};

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Deterministic block sum (fixed tree); the result is valid in every thread.
__device__ double block_sum_all(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];
  __syncthreads();
  return s;
}

template <typename T>
class Bcd {
 public:
  __device__ Bcd(const BcdArgs<T>& p, double* smem) : p_(p) {
    G_ = int(gridDim.x);
    g_ = int(blockIdx.x);
    N_ = p.sh.n;
    R_ = p.fs.rank;
    red_ = smem;              // [32]
    zb_ = smem + 32;          // [kZBatch] Kronecker entries of a position batch (as double)
    col_ = reinterpret_cast<T*>(zb_ + kZBatch);  // this component's columns, all modes (sum of extents)
    i64 off = 0;
    for (int m = 0; m < N_; ++m) {
      coff_[m] = int(off);
      off += p.sh.e[m];
    }
    phase_ = 0;
    chunk_ = ceil_div(p.S, i64(G_));
    e0_ = std::min(p.S, i64(g_) * chunk_);
    e1_ = std::min(p.S, e0_ + chunk_);
  }

  __device__ void run() {
    const T norm_b2 = T(sumsq(p_.X));
    int total = 0;
    bool error = false;
    // deflation pass (solve.hpp:335-345): res = X, then X - reconstruct(partial)
    for (i64 e = e0_ + threadIdx.x; e < e1_; e += blockDim.x) p_.res[e] = p_.X[e];
    grid_sync(p_.bar);
    for (int r = 0; r < R_ && total < p_.max_iter && !error; ++r) {
      update_component(r, p_.res, total, error);
      if (error) break;
      deflate(r);
    }
    bool converged = false;
    if (!error) {
      T prev_overall = sub_rn(T(1), T(sumsq(p_.res)) / norm_b2);
      while (total < p_.max_iter && !error) {
        for (int r = 0; r < R_ && total < p_.max_iter && !error; ++r) {
          // leave-one-out residual, update, new residual (solve.hpp:351-356)
          component_axpy(r, p_.res, p_.loo, +1);
          grid_sync(p_.bar);
          update_component(r, p_.loo, total, error);
          if (error) break;
          component_axpy(r, p_.loo, p_.res, -1);
          grid_sync(p_.bar);
        }
        if (error) break;
        const T overall = sub_rn(T(1), T(sumsq(p_.res)) / norm_b2);
        if (!isfinite(double(overall))) {
          error = true;
          if (g_ == 0 && threadIdx.x == 0) p_.st->error_it = total;
          break;
        }
        if (fabs(double(sub_rn(overall, prev_overall))) < p_.tol) {
          converged = true;
          break;
        }
        prev_overall = overall;
      }
    }
    if (g_ == 0 && threadIdx.x == 0) {
      p_.st->it = total + 1;
      p_.st->converged = converged ? 1 : 0;
      p_.st->done = 1;
    }
  }

 private:
  // sum of squares of x (fp64), reduced in CTA order: identical on every CTA
  __device__ double sumsq(const T* x) {
    double acc = 0.0;
    for (i64 e = e0_ + threadIdx.x; e < e1_; e += blockDim.x) {
      const double v = double(x[e]);
      acc += v * v;
    }
    acc = block_sum_all(acc, red_);
    double* pb = p_.part + i64(phase_) * G_ * p_.part_stride;
    if (threadIdx.x == 0) pb[i64(g_) * p_.part_stride] = acc;
    grid_sync(p_.bar);
    double s = 0.0;
    for (int q = 0; q < G_; ++q) s += ldcg(&pb[i64(q) * p_.part_stride]);
    phase_ ^= 1;
    return s;
  }

  // ||column r of factor m||^2 from the smem copy (fp64, fixed tree)
  __device__ double col_sq(int m) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < int(p_.sh.e[m]); i += blockDim.x) {
      const double v = double(col_[coff_[m] + i]);
      acc += v * v;
    }
    return block_sum_all(acc, red_);
  }

  // z at Kolda position (a, b) of mode m: prod over k != m of A_k[i_k, r], highest mode first (Scalar)
  __device__ T kron_at(int m, i64 a, i64 b) const {
    i64 idx[kMaxOrder];
    for (int k = N_ - 1; k > m; --k) {
      idx[k] = b % p_.sh.e[k];
      b /= p_.sh.e[k];
    }
    for (int k = m - 1; k >= 0; --k) {
      idx[k] = a % p_.sh.e[k];
      a /= p_.sh.e[k];
    }
    T z = T(1);
    for (int k = N_ - 1; k >= 0; --k)
      if (k != m) z = mul_rn(z, col_[coff_[k] + int(idx[k])]);
    return z;
  }

  // w[i] = sum_{a,b} y[a, i, b] z(a, b) (fp64, CTA partials reduced in CTA order), into wout (every CTA)
  __device__ void mode_product(const T* y, int m, double* wout) {
    const int rows_per_thread = int(ceil_div(p_.sh.e[m], i64(blockDim.x)));
    if (rows_per_thread <= 1)
      mode_product_k<1>(y, m, wout);
    else if (rows_per_thread <= 4)
      mode_product_k<4>(y, m, wout);
    else if (rows_per_thread <= 16)
      mode_product_k<16>(y, m, wout);
    else
      mode_product_k<48>(y, m, wout);
  }

  template <int K>  // output rows per thread: i = threadIdx.x + k * blockDim.x, k < K
  __device__ void mode_product_k(const T* y, int m, double* wout) {
    i64 L = 1, Rr = 1;
    for (int k = 0; k < m; ++k) L *= p_.sh.e[k];
    for (int k = m + 1; k < N_; ++k) Rr *= p_.sh.e[k];
    const int I = int(p_.sh.e[m]);
    const i64 J = L * Rr;
    const i64 pc = ceil_div(J, i64(G_));
    const i64 p0 = std::min(J, i64(g_) * pc), p1 = std::min(J, p0 + pc);
    double* pb = p_.part + i64(phase_) * G_ * p_.part_stride + i64(g_) * p_.part_stride;
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.0;
    for (i64 pbat = p0; pbat < p1; pbat += kZBatch) {
      const int np = int(std::min<i64>(kZBatch, p1 - pbat));
      __syncthreads();
      for (int q = threadIdx.x; q < np; q += blockDim.x) {
        const i64 pos = pbat + q, a = pos / Rr, b = pos - a * Rr;
        zb_[q] = double(kron_at(m, a, b));
      }
      __syncthreads();
      for (int q = 0; q < np; ++q) {
        const i64 pos = pbat + q, a = pos / Rr, b = pos - a * Rr;
        const double z = zb_[q];
        const T* yr = y + a * i64(I) * Rr + b;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int i = threadIdx.x + k * blockDim.x;
          if (i < I) acc[k] += double(ldcg(&yr[i64(i) * Rr])) * z;  // y was written by other CTAs
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      if (i < I) pb[i] = acc[k];
    }
    grid_sync(p_.bar);
    const double* pb0 = p_.part + i64(phase_) * G_ * p_.part_stride;
    for (int i = threadIdx.x; i < I; i += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < G_; ++q) s += ldcg(&pb0[i64(q) * p_.part_stride + i]);
      wout[i] = s;
    }
    phase_ ^= 1;
    __syncthreads();
  }

  // solve.hpp:286-330
  __device__ void update_component(int r, const T* y, int& total, bool& error) {
    const T norm_y2 = T(sumsq(y));
    if (norm_y2 == T(0)) {
      if (g_ == 0) {
        const T* f0 = p_.fs.f[0] + i64(r) * p_.sh.e[0];
        double acc = 0.0;
        for (int i = threadIdx.x; i < int(p_.sh.e[0]); i += blockDim.x) acc += double(f0[i]) * double(f0[i]);
        acc = block_sum_all(acc, red_);
        if (threadIdx.x == 0) p_.weights[r] = T(0);
        if (acc == 0.0)
          for (int i = threadIdx.x; i < int(p_.sh.e[0]); i += blockDim.x) p_.fs.f[0][i64(r) * p_.sh.e[0] + i] = T(i == 0);
      }
      grid_sync(p_.bar);
      return;
    }
    // this component's columns into shared memory (identical copies on every CTA)
    for (int m = 0; m < N_; ++m)
      for (int i = threadIdx.x; i < int(p_.sh.e[m]); i += blockDim.x)
        col_[coff_[m] + i] = ldcg(&p_.fs.f[m][i64(r) * p_.sh.e[m] + i]);
    __syncthreads();
    double* w = reinterpret_cast<double*>(col_ + coff_[N_ - 1] + p_.sh.e[N_ - 1] + 1) + 1;  // after the columns
    w = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(w) + 15) & ~uintptr_t(15));
    T prev = T(0);
    const int cap = min(kBcdCap, p_.max_iter - total);
    T lambda_r = T(0);
    for (int j = 1; j <= cap; ++j) {
      ++total;
      T w_dot_c = T(0);
      for (int mode = 0; mode < N_; ++mode) {
        T sc = T(1);
        for (int m = 0; m < N_; ++m) {
          if (m == mode) continue;
          const double c = sqrt(col_sq(m));  // col.squaredNorm() via the oracle's col_norm^2
          sc = mul_rn(sc, T(c * c));
        }
        mode_product(y, mode, w);
        const int I = int(p_.sh.e[mode]);
        T* col = col_ + coff_[mode];
        for (int i = threadIdx.x; i < I; i += blockDim.x) col[i] = sc > T(0) ? T(w[i]) / sc : T(0);
        __syncthreads();
        const T nrm = T(sqrt(col_sq(mode)));
        if (nrm > T(0))
          for (int i = threadIdx.x; i < I; i += blockDim.x) col[i] = col[i] / nrm;
        __syncthreads();
        if (mode == N_ - 1) {
          lambda_r = nrm;
          double d = 0.0;
          for (int i = threadIdx.x; i < I; i += blockDim.x) d += double(col[i]) * double(T(w[i]));
          w_dot_c = T(block_sum_all(d, red_));
        }
        if (g_ == 0)
          for (int i = threadIdx.x; i < I; i += blockDim.x) p_.fs.f[mode][i64(r) * I + i] = col[i];
      }
      if (g_ == 0 && threadIdx.x == 0) p_.weights[r] = lambda_r;
      // comp_fit = 1 - (norm_y2 + lambda^2 - 2 lambda w.c) / norm_y2, Scalar, left to right
      const T t1 = mul_rn(lambda_r, lambda_r);
      const T t2 = mul_rn(mul_rn(T(2), lambda_r), w_dot_c);
      const T comp_fit = sub_rn(T(1), sub_rn(add_rn(norm_y2, t1), t2) / norm_y2);
      if (!isfinite(double(comp_fit))) {
        if (g_ == 0 && threadIdx.x == 0) p_.st->error_it = total;
        error = true;
        break;
      }
      if (g_ == 0 && threadIdx.x == 0 && total - 1 < p_.max_iter) {
        p_.trace_fit[total - 1] = double(comp_fit);
        p_.trace_sec[total - 1] = double(gtimer_ns() - p_.st->t0) * 1e-9;
      }
      if (j >= 2 && fabs(double(sub_rn(comp_fit, prev))) < p_.tol) break;
      prev = comp_fit;
    }
    grid_sync(p_.bar);  // CTA 0's factor columns and weight visible everywhere
  }

  // res = X - reconstruct(components 0..r) (the oracle's reconstruct: per element
  // p_c = w_c prod_{m = N-2..0} A_m, s = sum_c p_c A_{N-1}, all fp64, rounded once)
  __device__ void deflate(int r) {
    const i64 E = p_.sh.e[N_ - 1];
    for (i64 e = e0_ + threadIdx.x; e < e1_; e += blockDim.x) {
      const i64 pi = e / E, il = e - pi * E;
      double s = 0.0;
      for (int c = 0; c <= r; ++c) {
        double pc = double(ldcg(&p_.weights[c]));
        i64 rem = pi;
        for (int m = N_ - 2; m >= 0; --m) {
          const i64 im = rem % p_.sh.e[m];
          rem /= p_.sh.e[m];
          pc = __dmul_rn(pc, double(ldcg(&p_.fs.f[m][im + i64(c) * p_.sh.e[m]])));
        }
        s = __dadd_rn(s, __dmul_rn(pc, double(ldcg(&p_.fs.f[N_ - 1][il + i64(c) * E]))));
      }
      p_.res[e] = sub_rn(p_.X[e], T(s));
    }
    grid_sync(p_.bar);
  }

  // out = in + sign * component_tensor(r) (solve.hpp:165-175: A0(i, r) * (w_r * z_j), Scalar)
  __device__ void component_axpy(int r, const T* in, T* out, int sign) {
    const T wr = ldcg(&p_.weights[r]);
    for (i64 e = e0_ + threadIdx.x; e < e1_; e += blockDim.x) {
      // digits, last mode fastest
      i64 rem = e, idx[kMaxOrder];
      for (int m = N_ - 1; m >= 0; --m) {
        idx[m] = rem % p_.sh.e[m];
        rem /= p_.sh.e[m];
      }
      T z = T(1);
      for (int m = N_ - 1; m >= 1; --m) z = mul_rn(z, ldcg(&p_.fs.f[m][idx[m] + i64(r) * p_.sh.e[m]]));
      const T c = mul_rn(ldcg(&p_.fs.f[0][idx[0] + i64(r) * p_.sh.e[0]]), mul_rn(wr, z));
      out[e] = sign > 0 ? add_rn(in[e], c) : sub_rn(in[e], c);
    }
  }

  BcdArgs<T> p_;
  int G_, g_, N_, R_, phase_;
  int coff_[kMaxOrder];
  i64 chunk_, e0_, e1_;
  double* red_;
  double* zb_;
  T* col_;
};

template <typename T>
__global__ void __launch_bounds__(kBcdThreads) bcd_kernel(BcdArgs<T> p) {
  extern __shared__ __align__(16) double bcd_smem[];
  Bcd<T> solver(p, bcd_smem);
  solver.run();
}

}  // namespace

bool bcd_supported(const i64* shape, int order, int rank) {
  (void)rank;
  i64 sum = 0;
  for (int m = 0; m < order; ++m) {
    if (shape[m] > 48 * kBcdThreads) return false;
    sum += shape[m];
  }
  return (32 + kZBatch) * 8 + sum * 8 + 2 * 12288 * 8 + 64 <= 200 * 1024;
}

template <typename T>
void bcd_solve(const T* X, T* res, T* loo, const i64* shape, int order, const FactorSet<T>& fs, T* weights,
               double tol, int max_iter, double* trace_fit, double* trace_sec, AlsState* state, double* part,
               i64 part_elems, GridBarrier* bar, cudaStream_t st) {
  i64 S = 1, sum = 0, maxe = 1;
  for (int m = 0; m < order; ++m) {
    S *= shape[m];
    sum += shape[m];
    maxe = std::max(maxe, shape[m]);
  }
  const size_t smem = size_t(32 + kZBatch) * 8 + size_t(sum) * sizeof(T) + size_t(maxe) * 8 + 64;
  static const size_t lim = enable_max_dyn_smem(bcd_kernel<T>);
  if (smem > lim) throw std::runtime_error("bcd: shared-memory plan too large");
  const int maxc = max_coop_blocks(bcd_kernel<T>, kBcdThreads, smem);
  const i64 stride = maxe + 1;
  int G = int(std::min<i64>({i64(maxc), i64(device_caps().num_sms), std::max<i64>(1, ceil_div(S, 4096)),
                             part_elems / (2 * stride)}));
  G = std::max(G, 1);
  BcdArgs<T> a{X, res, loo, make_bcd_shape(shape, order), S, fs, weights, tol, max_iter, trace_fit, trace_sec, state,
               part, stride, bar};
  launch_coop(bcd_kernel<T>, G, kBcdThreads, smem, st, a);
}

template void bcd_solve<float>(const float*, float*, float*, const i64*, int, const FactorSet<float>&, float*, double,
                               int, double*, double*, AlsState*, double*, i64, GridBarrier*, cudaStream_t);
template void bcd_solve<double>(const double*, double*, double*, const i64*, int, const FactorSet<double>&, double*,
                                double, int, double*, double*, AlsState*, double*, i64, GridBarrier*, cudaStream_t);

}  // namespace rcpg
