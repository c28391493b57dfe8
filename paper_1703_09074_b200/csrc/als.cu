// SPDX-License-Identifier: MIT
// CP-ALS kernels (solve.hpp:62-262) and Kruskal-model kernels
// (kruskal.hpp:52-220). The MTTKRP itself is a streamed `sketch` pass over
// the tensor against a materialized Khatri-Rao panel (kr_panel); the R x R
// algebra of one mode update (Gram Hadamard, pinv_psd, normalization, Gram,
// fit, stopping test) runs in one CTA so a whole ALS iteration is a handful
// of launches with no host round trip; each launch first checks the
// device-side `done` flag so the host can enqueue iterations ahead.
#include <cooperative_groups.h>

#include <cfloat>
#include <type_traits>

#include "als.cuh"
#include "passes.cuh"
#include "rng.cuh"
#include "runtime.cuh"

namespace rcpg {

namespace {

constexpr int kSmallThreads = 1024;
constexpr int kEigSmemMax = 96;   // Jacobi in shared memory up to 96 x 96
constexpr int kAlsSmemRank = 64;  // ALS R x R algebra in shared memory up to R = 64

struct ShapeArg {
  i64 e[kMaxOrder];
  int n;
};

ShapeArg make_shape(const i64* shape, int order) {
  ShapeArg s{};
  s.n = order;
  for (int m = 0; m < order; ++m) s.e[m] = shape[m];
  return s;
}

// ------------------------------------------------------------ KR panel
template <typename T>
__global__ void kr_panel_kernel(FactorSet<T> fs, ShapeArg sh, int mode, i64 J, i64 Rr, T* out, const int* skip) {
  if (skip != nullptr && *skip) return;
  const int rank = fs.rank;
  const i64 total = J * rank;
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const i64 s = e / rank;
    const int r = int(e - s * rank);
    const i64 a0 = s / Rr, b0 = s - a0 * Rr;
    i64 a = a0, b = b0;
    i64 idx[kMaxOrder];
    for (int k = sh.n - 1; k > mode; --k) {
      idx[k] = b % sh.e[k];
      b /= sh.e[k];
    }
    for (int k = mode - 1; k >= 0; --k) {
      idx[k] = a % sh.e[k];
      a /= sh.e[k];
    }
    T v = T(1);
    for (int k = sh.n - 1; k >= 0; --k) {  // highest mode first (kruskal.hpp:58-62)
      if (k == mode) continue;
      v *= fs.f[k][idx[k] + i64(r) * fs.extent[k]];
    }
    out[(a0 * rank + r) * Rr + b0] = v;
  }
}

// --------------------------------------------------------- block helpers
// Total order on doubles for rank computations: NaN sorts as +inf, so ranks
// stay a permutation even on non-finite data (the input check that rejects
// such data is raised after the device work, see api.cu Deferred).
__device__ __forceinline__ double order_key(double x) { return isnan(x) ? INFINITY : x; }
__device__ double block_reduce_sum(double v) {
  __shared__ double scratch[33];
  return block_sum(v, scratch);
}

// Jacobi rotation (c, s) that annihilates a_pq: tan(phi) = t, the smaller root
// of t^2 + 2 theta t - 1 = 0 with theta = (a_qq - a_pp) / (2 a_pq) (the
// oracle's symmetric Jacobi), in half-angle form so the chain of long-latency
// fp64 operations is two reciprocal square roots instead of two square roots
// and three divisions: with d = a_qq - a_pp, b = 2 a_pq, h = sqrt(d^2 + b^2):
// c^2 = (1 + |d| / h) / 2 and 2 s c = sign(theta) |b| / h. The round waits
// on this chain, so its latency is the Jacobi's critical path.
__device__ __forceinline__ void jacobi_rotation(double app, double aqq, double apq, double& c, double& s) {
  const double d = aqq - app, b = 2.0 * apq;
  const double h2 = d * d + b * b;
  if (h2 > 1e-290 && h2 < 1e290) {
    const double r = rsqrt(h2);  // 1 / h
    const double c2 = fma(0.5 * fabs(d), r, 0.5);
    const double ic = rsqrt(c2);
    const bool pos = d == 0.0 || ((d > 0.0) == (b > 0.0));  // theta >= 0
    c = c2 * ic;
    s = (pos ? 0.5 : -0.5) * fabs(b) * r * ic;
  } else {  // d^2 + b^2 under- or overflows: the scale-free form
    const double theta = d / b;
    const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
    c = 1.0 / sqrt(t * t + 1.0);
    s = t * c;
  }
}

// Parallel cyclic Jacobi (round-robin pairs) on a symmetric n x n matrix in
// global memory A (destroyed; diagonal -> eigenvalues), V <- eigenvectors.
// On exit evals[0..n) ascending, order[0..n) the column of V for each.
// A, V: n x n with leading dimension ld (odd ld keeps the row-wise rotations,
// which stride by ld, off a single shared-memory bank)
__device__ void jacobi_eig(double* A, double* V, int n, int ld, double* evals, int* order) {
  __shared__ double cs_c[kMaxRank * 8], cs_s[kMaxRank * 8];
  __shared__ int pp[kMaxRank * 8], pq[kMaxRank * 8];
  __shared__ int s_stop;
  const int tid = threadIdx.x, nt = blockDim.x;
  // SelfAdjointEigenSolver (solve.hpp:65, 110) reads the lower triangle only:
  // mirror it, so an input that is symmetric only up to rounding (a tensor-core
  // Gram) is treated exactly like the reference treats it.
  for (int e = tid; e < n * n; e += nt) {
    const int i = e % n, j = e / n;
    if (i < j) A[i + j * ld] = A[j + i * ld];
  }
  for (int e = tid; e < n * n; e += nt) V[(e % n) + (e / n) * ld] = (e % n == e / n) ? 1.0 : 0.0;
  __syncthreads();
  const int m = n + (n & 1);  // players (one dummy when n is odd)
  const int npairs = m / 2;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const int nwp = npairs < nw ? npairs : nw;  // warps that own a pair
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, dg = 0.0;
    for (int e = tid; e < n * n; e += nt) {
      const double x = A[(e % n) + (e / n) * ld];
      if (e % n == e / n)
        dg += x * x;
      else
        off += x * x;
    }
    off = block_reduce_sum(off);
    dg = block_reduce_sum(dg);
    if (tid == 0) s_stop = (off <= 1e-30 * dg) || off == 0.0;
    __syncthreads();
    if (s_stop) break;
    // One round = m / 2 disjoint rotations. The warp that owns pair q computes
    // its rotation itself (no staging barrier) from columns i, j, which no other
    // warp touches before the barrier, and rotates those columns; after the
    // barrier it rotates rows i, j of A and columns i, j of V. Only the warps that own a pair take part (named barrier 1);
    // the others wait at the sweep's closing barrier.
    if (wid < nwp) {
      for (int round = 0; round < m - 1; ++round) {
        // lane u computes the rotation of this warp's u-th pair (all of the
        // warp's pairs in one pass; at most 32 of them for n <= 2048)
        int pi = 0, pj = n;
        double pc = 1.0, ps = 0.0;
        {
          const int q = wid + lane * nwp;
          if (q < npairs) {
            int i, j;
            if (q == 0) {
              i = m - 1;
              j = round;
            } else {
              i = round + q;
              if (i >= m - 1) i -= m - 1;
              j = round + m - 1 - q;
              if (j >= m - 1) j -= m - 1;
            }
            if (i > j) {
              const int t = i;
              i = j;
              j = t;
            }
            pi = i;
            pj = j;
            if (j < n) {
              const double apq = A[i + j * ld];
              if (apq != 0.0) jacobi_rotation(A[i + i * ld], A[j + j * ld], apq, pc, ps);
            }
            pp[q] = i;
            pq[q] = j;
            cs_c[q] = pc;
            cs_s[q] = ps;
          }
        }
        __syncwarp();  // every rotation is formed before a lane overwrites its entries
        // columns: A <- A J
        for (int u = 0; wid + u * nwp < npairs; ++u) {
          const int i = __shfl_sync(0xffffffffu, pi, u), j = __shfl_sync(0xffffffffu, pj, u);
          const double c = __shfl_sync(0xffffffffu, pc, u), s = __shfl_sync(0xffffffffu, ps, u);
          if (j >= n) continue;
          for (int k = lane; k < n; k += 32) {
            const double akp = A[k + i * ld], akq = A[k + j * ld];
            A[k + i * ld] = c * akp - s * akq;
            A[k + j * ld] = s * akp + c * akq;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(nwp * 32) : "memory");
        // rows: A <- J^T A, and V <- V J
        for (int q = wid; q < npairs; q += nwp) {
          const int i = pp[q], j = pq[q];
          if (j >= n) continue;
          const double c = cs_c[q], s = cs_s[q];
          for (int k = lane; k < n; k += 32) {
            const double apk = A[i + k * ld], aqk = A[j + k * ld];
            A[i + k * ld] = c * apk - s * aqk;
            A[j + k * ld] = s * apk + c * aqk;
            const double vkp = V[k + i * ld], vkq = V[k + j * ld];
            V[k + i * ld] = c * vkp - s * vkq;
            V[k + j * ld] = s * vkp + c * vkq;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(nwp * 32) : "memory");
      }
    }
    __syncthreads();
  }
  // ascending, stable by index
  for (int i = tid; i < n; i += nt) {
    const double di = order_key(A[i + i * ld]);
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = order_key(A[j + j * ld]);
      if (dj < di || (dj == di && j < i)) ++rank;
    }
    evals[rank] = A[i + i * ld];
    order[rank] = i;
  }
  __syncthreads();
}

// ------------------------------------------------------------- init
template <typename T>
__device__ void init_from_gram_body(const T* G, int n, int R, int mode, u64 seed, int method, T* F, T* gram,
                                    double* work) {
  const int tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const bool in_smem = n <= kEigSmemMax;  // A and V resident in shared memory
  const int ld = n | 1;                   // odd leading dimension (bank spread)
  double* A = in_smem ? reinterpret_cast<double*>(smem_raw) : work;
  double* V = A + i64(n) * ld;
  double* ev = work + 2 * i64(n) * ld;
  int* ord = reinterpret_cast<int*>(ev + n);
  double* col = ev + 2 * n;  // [n] padding scratch
  __shared__ int s_filled;
  for (i64 e = tid; e < i64(n) * R; e += nt) F[e] = T(0);
  __syncthreads();
  int filled = 0;
  if (method == 0) {
    for (i64 e = tid; e < i64(n) * n; e += nt) A[(e % n) + (e / n) * ld] = double(G[e]);
    __syncthreads();
    jacobi_eig(A, V, n, ld, ev, ord);
    filled = R < n ? R : n;
    for (i64 e = tid; e < i64(n) * filled; e += nt) {
      const int i = int(e % n), j = int(e / n);
      F[i + i64(j) * n] = T(V[i + i64(ord[n - 1 - j]) * ld]);
    }
    __syncthreads();
    // canonicalize_column_signs (solve.hpp:77-84): first max |entry| >= 0
    for (int j = tid; j < R; j += nt) {
      int at = 0;
      T best = fabs(F[i64(j) * n]);
      for (int i = 1; i < n; ++i) {
        const T x = fabs(F[i + i64(j) * n]);
        if (x > best) {
          best = x;
          at = i;
        }
      }
      if (F[at + i64(j) * n] < T(0))
        for (int i = 0; i < n; ++i) F[i + i64(j) * n] = -F[i + i64(j) * n];
    }
    __syncthreads();
  }
  if (tid == 0) s_filled = filled;
  __syncthreads();
  // padding columns from stream (seed, init << 32 | mode), solve.hpp:117-127
  if (tid == 0 && filled < R) {
    const u64 s0 = derive_seed(seed, stream_id(kDomainInit, u64(mode)));
    u64 e = 0;
    for (int j = filled; j < R; ++j) {
      double nr = 0.0;
      for (int i = 0; i < n; ++i) {
        const T x = T(normal_at(s0, e++));
        col[i] = double(x);
        nr += double(x) * double(x);
      }
      nr = sqrt(nr);
      if (filled > 0 && filled < n) {
        // col -= F(:, :j) (F(:, :j)^T col)
        double proj[kMaxRank];
        for (int c = 0; c < j; ++c) {
          double s = 0.0;
          for (int i = 0; i < n; ++i) s += double(F[i + i64(c) * n]) * col[i];
          proj[c] = s;
        }
        double raw_nr = nr;
        double nrm2 = 0.0;
        double newc[1];  // placeholder to keep scope
        (void)newc;
        for (int i = 0; i < n; ++i) {
          double s = 0.0;
          for (int c = 0; c < j; ++c) s += double(F[i + i64(c) * n]) * proj[c];
          const T v = T(col[i] - s);
          nrm2 += double(v) * double(v);
          // stash the projected value in A (scratch) to keep `col` (raw) intact
          A[i] = double(v);
        }
        const double nrm = sqrt(nrm2);
        for (int i = 0; i < n; ++i)
          F[i + i64(j) * n] = (T(nrm) > T(1e-8)) ? T(A[i] / nrm) : (raw_nr > 0 ? T(col[i] / raw_nr) : T(col[i]));
      } else {
        for (int i = 0; i < n; ++i) F[i + i64(j) * n] = nr > 0 ? T(col[i] / nr) : T(col[i]);
      }
    }
  }
  __syncthreads();
  // Gram F^T F
  for (int e = tid; e < R * R; e += nt) {
    const int a = e % R, b = e / R;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += double(F[i + i64(a) * n]) * double(F[i + i64(b) * n]);
    gram[e] = T(s);
  }
}

// Every initialized mode in one launch, one CTA per mode (the eigenproblems
// are independent and each is latency bound on one SM).
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) init_from_gram_kernel(InitBatch<T> b, int R, u64 seed, int method) {
  const int q = blockIdx.x;
  init_from_gram_body<T>(b.G[q], b.n[q], R, b.mode[q], seed, method, b.F[q], b.gram[q], b.work[q]);
}

template <typename T>
__global__ void zero_factor_kernel(T* F, i64 n, int R, T* gram) {
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < n * R; e += i64(gridDim.x) * blockDim.x) F[e] = T(0);
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < i64(R) * R; e += i64(gridDim.x) * blockDim.x)
    gram[e] = T(0);
}

// --------------------------------------------------------------- ALS
// One mode update (solve.hpp:207-230) and, for the last mode, the fit and
// stopping test (solve.hpp:232-254), executed by one CTA with everything in
// shared memory. W (I x R, column-major) is the MTTKRP. `work` holds
// 3 R^2 + 4 R + I R doubles.
//
// pinv_psd(V) (solve.hpp:62-73) drops eigenvalues <= R eps lambda_max. V is
// inverted by Gauss-Jordan (SPD, no pivoting); if every pivot is positive and
// 1 / ||V^-1||_F > R eps ||V||_F (which bounds lambda_min from below and
// lambda_max from above) no eigenvalue can fall under the cutoff, so
// pinv(V) = V^-1. Otherwise the exact eigen path runs (cyclic Jacobi).
__device__ unsigned long long* g_als_prof = nullptr;
#define ALS_STAMP(slot)                                                              \
  do {                                                                               \
    if (g_als_prof && threadIdx.x == 0 && blockIdx.x == 0) {                         \
      unsigned long long _t;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                          \
      g_als_prof[slot] += _t - _tlast;                                               \
      _tlast = _t;                                                                   \
    }                                                                                \
  } while (0)

// Gauss-Jordan inverse of an R x R matrix in place (A column-major, smem),
// with the entries in registers: thread (warp w, lane l) holds (i, j),
// i = w + k * warps, j = l + 32 m. Step k needs row k (published by its
// owner into a double-buffered shared row after its update in step k - 1)
// and the own row's column-k entry (a shuffle from lane k % 32): one barrier
// per pivot. Same arithmetic, in the same order, as the shared-memory
// ping-pong version (bitwise identical). *ok = 0 if a pivot is not > 0.
// `scratch` (2 * 32 * KC doubles of dynamic shared memory) holds the row
// buffers: static shared memory here would shrink the dynamic budget of the
// ALS loop kernel that inlines this (and push it to a smaller MTTKRP batch).
template <int KR, int KC>
__device__ void gj_inverse_regs(double* A, int R, int* ok, double* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  double (*rowbuf)[32 * KC] = reinterpret_cast<double (*)[32 * KC]>(scratch);
  double v[KR][KC];
#pragma unroll
  for (int q = 0; q < KR; ++q)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int i = wid + q * nw, j = lane + 32 * m;
      v[q][m] = (i < R && j < R) ? A[i + j * R] : 0.0;
    }
  if (wid == 0)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[0][lane + 32 * m] = v[0][m];
  __syncthreads();
  int bad = 0;
  // pivot k = q * nw + w: the slot q of the pivot row (and of the next one,
  // q or q + 1) is a compile-time index, so v stays in registers (a runtime
  // slot index made the compiler keep v on the stack: ~1.2 us per step)
#pragma unroll
  for (int q0 = 0; q0 < KR; ++q0) {
    for (int w = 0; w < nw; ++w) {
      const int k = q0 * nw + w;
      if (k >= R) break;
      const double* rk = rowbuf[k & 1];
      const double p = rk[k];
      double rkj[KC];
#pragma unroll
      for (int m = 0; m < KC; ++m) rkj[m] = rk[lane + 32 * m];
      const int mk = k >> 5, lk = k & 31;
      double aik[KR];
#pragma unroll
      for (int q = 0; q < KR; ++q) {
        double x = v[q][0];
#pragma unroll
        for (int m = 1; m < KC; ++m) x = (m == mk) ? v[q][m] : x;
        aik[q] = __shfl_sync(0xffffffffu, x, lk);
      }
      bad |= !(p > 0.0);
      const double ip = 1.0 / p;
      // the general update on every entry (one FMA: v - aik akj), then the
      // column-k entries (-aik / p, lane lk) and row k (akj, its pivot 1 / p)
      // overwritten: the values of the branchy per-entry form, a quarter of
      // the instructions
      double akj[KC];
#pragma unroll
      for (int m = 0; m < KC; ++m) akj[m] = rkj[m] * ip;
#pragma unroll
      for (int m = 0; m < KC; ++m)
#pragma unroll
        for (int q = 0; q < KR; ++q) v[q][m] = fma(-aik[q], akj[m], v[q][m]);
      if (lane == lk)
#pragma unroll
        for (int m = 0; m < KC; ++m)
          if (m == mk)
#pragma unroll
            for (int q = 0; q < KR; ++q) v[q][m] = -aik[q] * ip;
      if (wid == w)
#pragma unroll
        for (int m = 0; m < KC; ++m) v[q0][m] = (lane + 32 * m == k) ? ip : akj[m];
      // publish row k + 1: warp w + 1, slot q0 -- or warp 0, slot q0 + 1
      if (k + 1 < R) {
        double* dst = rowbuf[(k + 1) & 1];
        if (w + 1 < nw) {
          if (wid == w + 1)
#pragma unroll
            for (int m = 0; m < KC; ++m) dst[lane + 32 * m] = v[q0][m];
        } else if (q0 + 1 < KR) {
          if (wid == 0)
#pragma unroll
            for (int m = 0; m < KC; ++m) dst[lane + 32 * m] = v[q0 + 1 < KR ? q0 + 1 : q0][m];
        }
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int q = 0; q < KR; ++q)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int i = wid + q * nw, j = lane + 32 * m;
      if (i < R && j < R) A[i + j * R] = v[q][m];
    }
  if (tid == 0 && bad) *ok = 0;
  __syncthreads();
}

// part 0: the whole mode update. part 1: only V and pinv(V) (steps 1-2), written
// to pm_io (R x R doubles) -- they depend only on the other modes' Grams, so the
// loop kernel computes them on one CTA while the others run the MTTKRP.
// part 2: steps 3-6 with pinv(V) read from pm_io.
template <typename T, typename WT>
__device__ void als_mode_update(const FactorSet<T>& fs, int mode, const WT* W, T* weights, double tol,
                                int max_iter, double* trace_fit, double* trace_sec, AlsState* st, double* work,
                                int part = 0, double* pm_io = nullptr) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int R = fs.rank, N = fs.order;
  const int I = int(fs.extent[mode]);
  T* F = fs.f[mode];
  double* V = work;          // R x R
  double* A = V + R * R;     // R x R: Gauss-Jordan in place -> V^{-1}
  double* X = A + R * R;     // R x R: eigenvectors (fallback)
  double* ev = X + R * R;    // R
  int* ord = reinterpret_cast<int*>(ev + R);
  const int ldf = I | 1;     // odd leading dimension: column-strided reads spread over the banks
  double* Fs = ev + 2 * R;   // I x R new factor (double, smem, leading dimension ldf)
  double* nr = Fs + i64(ldf) * R;  // R column norms
  __shared__ int s_ok;
  unsigned long long _tlast = 0;
  if (g_als_prof && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_tlast));

  const int R2 = R * R;
  const int lane0 = tid & 31, wid0 = tid >> 5, nw0 = nt >> 5;
  double* Pm = A;
  if (part == 2) {
    for (int e0 = tid; e0 < R2; e0 += 8 * nt) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = e0 + u * nt < R2 ? ldcg(&pm_io[e0 + u * nt]) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (e0 + u * nt < R2) A[e0 + u * nt] = v[u];
    }
    __syncthreads();
  } else {
  // 1. V = Hadamard of the other modes' Grams (solve.hpp:209-211): the
  // reference's Scalar product chain, v = 1, then v *= G_k for k ascending
  // (the Grams come from other CTAs in this launch: L2-coherent loads, the
  // chunk's loads issued before any product)
  for (int e0 = 0; e0 < R * R; e0 += 4 * nt) {
    T gk[kMaxOrder][4];
#pragma unroll
    for (int k = 0; k < kMaxOrder; ++k)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * nt + tid;
        gk[k][u] = (k < N && k != mode && e < R * R) ? ldcg(&fs.gram[k][e]) : T(1);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * nt + tid;
      if (e >= R * R) continue;
      T v = T(1);
#pragma unroll
      for (int k = 0; k < kMaxOrder; ++k)
        if (k < N && k != mode) v = mul_rn(v, gk[k][u]);
      V[e] = double(v);
      A[e] = V[e];
    }
  }
  if (tid == 0) s_ok = 1;
  __syncthreads();
  // 2. Gauss-Jordan inverse of the SPD matrix, one barrier per pivot
  // X (R x R, used only by the eigen fallback afterwards) holds the row buffers
  if (R <= 32 && R <= 4 * nw0 && R * R >= 64) {
    gj_inverse_regs<4, 1>(A, R, &s_ok, X);
  } else if (R <= 64 && R <= 8 * nw0 && R * R >= 128) {
    gj_inverse_regs<8, 2>(A, R, &s_ok, X);
  } else {
  // ping-pong between A and X
  double* src = A;
  double* dst = X;
  for (int k = 0; k < R; ++k) {
    // restrict-qualified with the pivot column hoisted: without it every
    // store may alias the next column's loads and the step serializes
    const double* __restrict__ sp = src;
    double* __restrict__ dp = dst;
    const double p = sp[k + k * R];
    const double ip = 1.0 / p;
    const double aik0 = lane0 < R ? sp[lane0 + k * R] : 0.0;
    const double aik1 = lane0 + 32 < R ? sp[lane0 + 32 + k * R] : 0.0;
    for (int j = wid0; j < R; j += nw0) {
      const double akj = sp[k + j * R] * ip;
      const double s0 = lane0 < R ? sp[lane0 + j * R] : 0.0;
      const double s1 = lane0 + 32 < R ? sp[lane0 + 32 + j * R] : 0.0;
      double v0, v1;
      if (j != k) {
        v0 = (lane0 != k) ? s0 - aik0 * akj : akj;
        v1 = (lane0 + 32 != k) ? s1 - aik1 * akj : akj;
      } else {
        v0 = (lane0 != k) ? -aik0 * ip : ip;
        v1 = (lane0 + 32 != k) ? -aik1 * ip : ip;
      }
      if (lane0 < R) dp[lane0 + j * R] = v0;
      if (lane0 + 32 < R) dp[lane0 + 32 + j * R] = v1;
    }
    if (tid == 0 && !(p > 0.0)) s_ok = 0;
    __syncthreads();
    double* t = src;
    src = dst;
    dst = t;
  }
  if (src != A) {
    for (int e = tid; e < R2; e += nt) A[e] = src[e];
    __syncthreads();
  }
  }
  ALS_STAMP(8);
  double fro = 0.0, ifro = 0.0;
  for (int e = tid; e < R2; e += nt) {
    fro += V[e] * V[e];
    ifro += A[e] * A[e];
  }
  fro = sqrt(block_reduce_sum(fro));
  ifro = sqrt(block_reduce_sum(ifro));
  const bool direct = s_ok && isfinite(ifro) && ifro > 0.0 && (1.0 / ifro) > double(R) * double(Traits<T>::eps) * fro;
  if (!direct) {
    for (int e = tid; e < R2; e += nt) A[e] = V[e];
    __syncthreads();
    jacobi_eig(A, X, R, R, ev, ord);
    T lmax = T(0);
    for (int k = 0; k < R; ++k) lmax = T(ev[k]) > lmax ? T(ev[k]) : lmax;
    const T tau = T(R) * Traits<T>::eps * lmax;
    for (int e = tid; e < R2; e += nt) {
      const int a = e % R, b = e / R;
      double s = 0.0;
      for (int k = 0; k < R; ++k) {
        const T lk = T(ev[k]);
        if (lk > tau) {
          const int c = ord[k];
          s += X[a + c * R] * (1.0 / double(lk)) * X[b + c * R];
        }
      }
      V[e] = s;
    }
    Pm = V;
    if (tid == 0) st->pivots_fallback += 1;
    __syncthreads();
  }
  // pinv_psd returns Matrix<Scalar> (solve.hpp:62-73): F = W pinv(V) uses
  // the Scalar-rounded pseudo-inverse
  for (int e = tid; e < R2; e += nt) Pm[e] = double(T(Pm[e]));
  __syncthreads();
  if (part == 1) {
    for (int e = tid; e < R2; e += nt) pm_io[e] = Pm[e];
    return;
  }
  }
  ALS_STAMP(9);
  // 3. F = W pinv(V), rounded to Scalar like the reference's factor.
  // Register tile per thread: rows lane + 32u (u < 4) x 4 consecutive columns,
  // so one smem load of W feeds 4 FMAs; every output is still the chain
  // s = sum_k W[i, k] Pm[k, r] in k order from 0 (same bits as one chain per output).
  {
    const WT* __restrict__ Wr = W;
    const double* __restrict__ Pr = Pm;
    constexpr int TR = 4;
    const int ngrp = (R + TR - 1) / TR;
    for (int item = wid0; item < ngrp * ((I + 127) / 128); item += nw0) {
      const int rg = item % ngrp, ib = (item / ngrp) * 128 + lane0;
      const int r0 = rg * TR;
      double s[4][TR];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < TR; ++j) s[u][j] = 0.0;
      for (int k = 0; k < R; ++k) {
        double pk[TR];
#pragma unroll
        for (int j = 0; j < TR; ++j) pk[j] = r0 + j < R ? Pr[k + (r0 + j) * R] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = ib + 32 * u;
          const double w = i < I ? double(Wr[i + k * I]) : 0.0;
#pragma unroll
          for (int j = 0; j < TR; ++j) s[u][j] += w * pk[j];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < TR; ++j)
          if (ib + 32 * u < I && r0 + j < R) Fs[ib + 32 * u + (r0 + j) * ldf] = double(T(s[u][j]));
    }
  }
  __syncthreads();
  ALS_STAMP(10);
  // 4. column norms; weights from the last mode (solve.hpp:215-229)
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int r = wid; r < R; r += nw) {
    double s = 0.0;
    for (int i = lane; i < I; i += 32) s += Fs[i + r * ldf] * Fs[i + r * ldf];
    s = warp_sum(s);
    if (lane == 0) {
      const T nrm = T(sqrt(s));
      nr[r] = double(nrm);
      if (mode == N - 1) weights[r] = nrm;
    }
  }
  __syncthreads();
  for (int r = wid0; r < R; r += nw0) {
    const T nrm = T(nr[r]);
    for (int i = lane0; i < I; i += 32) {
      const int e = i + r * ldf;
      const T v = nrm > T(0) ? T(Fs[e]) / nrm : T(Fs[e]);
      Fs[e] = double(v);
      F[i + r * I] = v;
    }
  }
  __syncthreads();
  ALS_STAMP(11);
  // 5. Gram of the new factor: 4 x 4 blocks (a-block <= b-block) per thread,
  // 8 loads per i for 16 FMAs; entry (a, b), a <= b, is the chain
  // sum_i F[i, a] F[i, b] in i order (same bits as one chain per pair) and is
  // written to both (a, b) and (b, a)
  {
    const double* __restrict__ Fr = Fs;
    const int nb = (R + 3) / 4, nblk = nb * (nb + 1) / 2;
    for (int q = tid; q < nblk; q += nt) {
      int bb = int((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
      while (bb * (bb + 1) / 2 > q) --bb;
      while ((bb + 1) * (bb + 2) / 2 <= q) ++bb;
      const int ab = q - bb * (bb + 1) / 2;  // ab <= bb
      const int a0 = 4 * ab, b0 = 4 * bb;
      double acc[4][4];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
      int ca[4], cb[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        ca[x] = (a0 + x < R ? a0 + x : a0) * ldf;
        cb[x] = (b0 + x < R ? b0 + x : b0) * ldf;
      }
      for (int i = 0; i < I; ++i) {
        double fa[4], fb[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          fa[x] = Fr[i + ca[x]];
          fb[x] = Fr[i + cb[x]];
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] += fa[x] * fb[y];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int a = a0 + x, b = b0 + y;
          if (a >= R || b >= R || a > b) continue;
          const T g = T(acc[x][y]);
          fs.gram[mode][a + b * R] = g;
          fs.gram[mode][b + a * R] = g;
          V[a + b * R] = double(g);  // this mode's Gram, for the fit
          V[b + a * R] = double(g);
        }
    }
  }
  __syncthreads();
  ALS_STAMP(12);
  if (mode != N - 1) return;
  // 6. fit (solve.hpp:232-254), double accumulation; g = the Scalar
  // Hadamard chain of all Grams (g = 1, g *= G_k for k ascending)
  double m2 = 0.0;
  for (int e = tid; e < R2; e += nt) {
    const int a = e % R, b = e / R;
    T g = T(1);
    for (int k = 0; k < N; ++k) g = mul_rn(g, k == mode ? T(V[e]) : fs.gram[k][e]);
    m2 += nr[a] * double(g) * nr[b];
  }
  m2 = block_reduce_sum(m2);
  double xi = 0.0;
  for (int e = tid; e < I * R; e += nt) xi += double(W[e]) * Fs[(e % I) + (e / I) * ldf] * nr[e / I];
  xi = block_reduce_sum(xi);
  if (tid == 0) {
    const double model2 = m2 > 0.0 ? m2 : 0.0;
    const double nx2 = st->nx2;
    const double fit_now = 1.0 - (nx2 + model2 - 2.0 * xi) / nx2;
    const int it = st->it;
    if (!isfinite(fit_now)) {
      st->error_it = it;
      st->done = 1;
    } else {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      trace_fit[it - 1] = fit_now;
      trace_sec[it - 1] = double(now - st->t0) * 1e-9;
      if (it >= 2 && fabs(fit_now - st->prev_fit) < tol) {
        st->converged = 1;
        st->done = 1;
      }
      st->prev_fit = fit_now;
      if (it >= max_iter) st->done = 1;
      st->it = it + 1;
    }
  }
  __syncthreads();
  ALS_STAMP(13);
}

template <typename T>
__global__ void __launch_bounds__(kSmallThreads)
    als_update_kernel(FactorSet<T> fs, int mode, const T* W, T* weights, double tol, int max_iter,
                      double* trace_fit, double* trace_sec, AlsState* st, double* work) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  work = reinterpret_cast<double*>(smem_raw);
  als_mode_update<T, T>(fs, mode, W, weights, tol, max_iter, trace_fit, trace_sec, st, work);
}

// Whole ALS loop in one cooperative launch (solve.hpp:205-255). Per mode:
//   A. every CTA: MTTKRP partial over its slice of the mode's (a, b)
//      positions, Khatri-Rao rows formed on the fly (no panel);
//   B. CTA 0: fixed-order reduction of the partials, then als_mode_update.
// Two grid barriers per mode; the stop flag is read after the last mode.
constexpr int kAlsThreads = 256;
constexpr int kAlsBatch = 32;   // positions per smem batch
constexpr int kAlsAcc = 32;     // accumulators per thread: I * R <= kAlsAcc * kAlsThreads

template <typename T>
struct AlsLoopArgs {
  const T* B;
  ShapeArg sh;
  FactorSet<T> fs;
  T* weights;
  double tol;
  int max_iter;
  double* trace_fit;
  double* trace_sec;
  AlsState* st;
  double* part;  // [2][G][max I*R]
  double* pm;    // R x R pinv(V) from the last CTA (nullptr: CTA 0 does the whole update)
  i64 part_stride;
  GridBarrier* bar;
  unsigned long long* prof;  // optional [8] ns per phase (CTA 0): A, bar1, B, bar2
  int grid_update;           // split mode: mode update spread over the grid (als_update_grid)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kAlsTiles = 8;  // 16x8 output tiles per warp: ceil(I/16) ceil(R/8) <= 8 warps x kAlsTiles

__host__ __device__ constexpr int als_ld(int n) { return (n + 15) / 16 * 16 + 4; }

template <typename T, int BATCH = kAlsBatch>
__host__ __device__ constexpr i64 als_fib_doubles(i64 I) {  // [2][BATCH][I] raw T, in doubles
  return (2 * BATCH * I * i64(sizeof(T)) + 15) / 16 * 2;
}

template <typename T>
__device__ __forceinline__ void als_cp_elem(T* dst, const T* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 4 : 0));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void als_cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void als_cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void als_dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// The mode update of the loop kernel spread over the whole grid (split mode:
// pinv(V) is already in pm). Every output keeps the operation order of
// als_mode_update, so the factors and Grams carry the same bits:
//  B1  CTA g owns rows i = g, g + G, ...: W(i, :) reduced from the GA MTTKRP
//      partials in a fixed order and rounded to Scalar (solve.hpp:212-213);
//      F(i, :) = W(i, :) pinv(V), the k-ascending chain, rounded to Scalar.
//  --  grid sync
//  B2  every CTA: the R column norms from F (warp per column, lanes striding
//      the rows: identical in every CTA), the weights (last mode); its own rows
//      normalized into the factor; the 4 x 4 Gram blocks spread over the grid,
//      one i-ascending chain per entry (solve.hpp:215-230).
//  --  grid sync
//  B3  last mode: CTA 0 the fit and the stopping test (solve.hpp:232-254),
//      then a grid sync so every CTA reads the same `done`.
// CTA 0's mode update used to serialize B1-B3 on one SM (C5: 45 us per mode step).
template <typename T, typename Sync>
__device__ void als_update_grid(const FactorSet<T>& fs, int mode, const double* part0, i64 pstride, int GA,
                                double* wbuf, double* fraw, const double* pm, T* weights, double tol, int max_iter,
                                double* trace_fit, double* trace_sec, AlsState* st, double* sm, Sync gsync,
                                unsigned long long* prof = nullptr) {
  const int tid = threadIdx.x, nt = blockDim.x, G = gridDim.x, g = blockIdx.x;
  const int R = fs.rank, N = fs.order, I = int(fs.extent[mode]);
  const bool stamp = prof != nullptr && g == 0 && tid == 0;
  unsigned long long ts = 0;
  if (stamp) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
  auto mark = [&](int slot) {
    if (stamp) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      prof[slot] += t - ts;
      ts = t;
    }
  };
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  double* wrow = sm;             // [R] this row of W (Scalar-rounded)
  double* nr = wrow + R;         // [R] column norms (Scalar-rounded)
  double* spm = nr + R;          // [R][R] pinv(V), staged (one L2 round trip, not R)
  double* sfr = spm + R * R;     // [I][R] F before normalization, staged
  double* fn = sfr + I * R;      // [R][I | 1] normalized factor (Gram / fit CTAs); B1's subset sums
  // ---- B1 (partials row-major: partial q's row i is R contiguous doubles)
  const int nsub = nt / R > 0 ? nt / R : 1;  // partial subsets, summed in order
  const int rr = tid % R, sb = tid / R;
  double* red = fn;                          // [nsub][R] subset sums (fn is free here)
  if (g < I) {  // transposed: thread r reads pinv(V)(k, r) at k R + r; 8 loads in flight per thread
    for (int e0 = tid; e0 < R * R; e0 += 8 * nt) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = e0 + u * nt < R * R ? ldcg(pm + e0 + u * nt) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * nt;
        if (e < R * R) spm[(e % R) * R + e / R] = v[u];
      }
    }
  }
  for (int i = g; i < I; i += G) {
    if (sb < nsub) {
      const double* src = part0 + i64(i) * R + rr;
      double s = 0.0;
      for (int q0 = sb; q0 < GA; q0 += 16 * nsub) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int q = q0 + nsub * u;
          v[u] = q < GA ? ldcg(src + i64(q) * pstride) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
      }
      red[sb * R + rr] = s;
    }
    __syncthreads();
    for (int r = tid; r < R; r += nt) {
      double s = 0.0;
      for (int b = 0; b < nsub; ++b) s += red[b * R + r];
      const double w = double(T(s));
      wrow[r] = w;
      wbuf[i + i64(r) * I] = w;
    }
    __syncthreads();
    for (int r = tid; r < R; r += nt) {
      double acc = 0.0;
      for (int k = 0; k < R; ++k) acc += wrow[k] * spm[k * R + r];
      fraw[i + i64(r) * I] = double(T(acc));
    }
    __syncthreads();
  }
  mark(25);
  gsync();
  mark(26);
  // ---- B2
  for (int e0 = tid; e0 < I * R; e0 += 8 * nt) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = e0 + u * nt < I * R ? ldcg(&fraw[e0 + u * nt]) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u * nt < I * R) sfr[e0 + u * nt] = v[u];
  }
  __syncthreads();
  for (int r = wid; r < R; r += nw) {
    double s = 0.0;
    for (int i = lane; i < I; i += 32) {
      const double f = sfr[i + r * I];
      s += f * f;
    }
    s = warp_sum(s);
    if (lane == 0) {
      const T nrm = T(sqrt(s));
      nr[r] = double(nrm);
      if (g == 0 && mode == N - 1) weights[r] = nrm;
    }
  }
  __syncthreads();
  for (int i = g; i < I; i += G)
    for (int r = tid; r < R; r += nt) {
      const T nrm = T(nr[r]);
      const T f = T(sfr[i + r * I]);
      fs.f[mode][i + i64(r) * I] = nrm > T(0) ? f / nrm : f;
    }
  // Gram entries (a <= b) in CTA-contiguous ranges: a warp shares b and walks
  // consecutive a (odd leading dimension: conflict-free), one i-ascending
  // chain per entry -- the per-entry chain of the 4 x 4 register tiles of
  // als_mode_update, so the same bits
  const int ldn = I | 1;
  const int E = R * (R + 1) / 2, gcta = (E + nt - 1) / nt;
  const bool last = mode == N - 1;
  if (g < gcta || (last && g == 0)) {
    for (int e = tid; e < I * R; e += nt) {
      const int i = e % I, r = e / I;
      const T nrm = T(nr[r]);
      const T f = T(sfr[e]);
      fn[i + r * ldn] = double(nrm > T(0) ? f / nrm : f);
    }
    __syncthreads();
    const int e = g * nt + tid;
    if (g < gcta && e < E) {
      int b = int((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (b * (b + 1) / 2 > e) --b;
      while ((b + 1) * (b + 2) / 2 <= e) ++b;
      const int a = e - b * (b + 1) / 2;
      const double* fa = fn + a * ldn;
      const double* fb = fn + b * ldn;
      double acc = 0.0;
      for (int i = 0; i < I; ++i) acc += fa[i] * fb[i];
      const T gv = T(acc);
      fs.gram[mode][a + b * R] = gv;
      fs.gram[mode][b + a * R] = gv;
    }
  }
  mark(27);
  gsync();
  mark(28);
  if (!last) return;
  // ---- B3
  if (g == 0) {
    const int R2 = R * R;
    double m2 = 0.0;
    for (int e0 = 0; e0 < R2; e0 += 4 * nt) {  // every Gram load of the chunk in flight first
      T gk[kMaxOrder][4];
#pragma unroll
      for (int k = 0; k < kMaxOrder; ++k)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * nt + tid;
          gk[k][u] = (k < N && e < R2) ? ldcg(&fs.gram[k][e]) : T(1);
        }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * nt + tid;
        if (e >= R2) continue;
        T gv = T(1);
#pragma unroll
        for (int k = 0; k < kMaxOrder; ++k)
          if (k < N) gv = mul_rn(gv, gk[k][u]);
        m2 += nr[e % R] * double(gv) * nr[e / R];
      }
    }
    m2 = block_reduce_sum(m2);
    double xi = 0.0;
    for (int e0 = tid; e0 < I * R; e0 += 8 * nt) {
      double wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) wv[u] = e0 + u * nt < I * R ? ldcg(&wbuf[e0 + u * nt]) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * nt;
        if (e < I * R) xi += wv[u] * fn[(e % I) + (e / I) * ldn] * nr[e / I];
      }
    }
    xi = block_reduce_sum(xi);
    if (tid == 0) {
      const double model2 = m2 > 0.0 ? m2 : 0.0;
      const double nx2 = st->nx2;
      const double fit_now = 1.0 - (nx2 + model2 - 2.0 * xi) / nx2;
      const int it = st->it;
      if (!isfinite(fit_now)) {
        st->error_it = it;
        st->done = 1;
      } else {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        trace_fit[it - 1] = fit_now;
        trace_sec[it - 1] = double(now - st->t0) * 1e-9;
        if (it >= 2 && fabs(fit_now - st->prev_fit) < tol) {
          st->converged = 1;
          st->done = 1;
        }
        st->prev_fit = fit_now;
        if (it >= max_iter) st->done = 1;
        st->it = it + 1;
      }
    }
  }
  mark(29);
  gsync();
  mark(30);
}

// CLUSTER: the grid is one thread-block cluster (<= 16 CTAs, small compressed
// tensors such as C1 / C2): the hardware cluster barrier replaces the grid
// barrier (release / acquire at cluster scope orders the global-memory partials
// and factors exactly like grid_sync), ~2 us less per barrier, three per mode step.
template <typename T, int BATCH, bool CLUSTER = false>
__global__ void __launch_bounds__(kAlsThreads, CLUSTER ? 1 : 2) als_loop_kernel(AlsLoopArgs<T> p) {
  auto gsync = [&]() {
    if constexpr (CLUSTER) {
      __threadfence();
      cooperative_groups::this_cluster().sync();
    } else {
      grid_sync(p.bar);
    }
  };
  __shared__ int pidx[BATCH * kMaxOrder];
  __shared__ int sfoff[kMaxOrder], sext[kMaxOrder];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int G = gridDim.x, g = blockIdx.x;
  const int N = p.sh.n, R = p.fs.rank;
  int parity = 0;
  for (;;) {
    for (int m = 0; m < N; ++m) {
      const i64 I = p.sh.e[m];
      i64 L = 1, Rr = 1;
      for (int k = 0; k < m; ++k) L *= p.sh.e[k];
      for (int k = m + 1; k < N; ++k) Rr *= p.sh.e[k];
      const i64 J = L * Rr;
      const int nout = int(I) * R;
      unsigned long long tp0 = 0;
      if (p.prof && g == 0 && tid == 0) tp0 = gtimer();
      // the last CTA computes pinv(V) of this mode (it needs only the other
      // modes' Grams) while CTAs 0 .. G-2 run the MTTKRP
      const bool split = p.pm != nullptr && G >= 2;
      const int GA = split ? G - 1 : G;
      if (split && g == G - 1) {
        FactorSet<T> fs = p.fs;
        als_mode_update<T, double>(fs, m, static_cast<const double*>(nullptr), p.weights, p.tol, p.max_iter,
                                   p.trace_fit, p.trace_sec, p.st, sm, 1, p.pm);
      }
      // ---- A: partial MTTKRP over positions [j0, j1): W_part = Fib^T KC on
      //      the FP64 tensor cores (mma.m16n8k4, M = i, N = r, K = positions);
      //      each warp keeps its 16x8 output tiles in registers. Fibers are
      //      gathered with cp.async into a double buffer: batch b+1 lands
      //      while batch b's Khatri-Rao rows are formed and multiplied.
      const int lane = tid & 31, wrp = tid >> 5, nwarp = nt >> 5, gq = lane >> 2, tq = lane & 3;
      const int I16 = (int(I) + 15) / 16, R8 = (R + 7) / 8, NTILE = I16 * R8;
      double acc[kAlsTiles][4];
#pragma unroll
      for (int t = 0; t < kAlsTiles; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0;
      const i64 chunk = ceil_div(J, GA);
      const i64 j0 = g < GA ? g * chunk : J, j1 = j0 + chunk < J ? j0 + chunk : J;
      // padded row strides (== 4 mod 16 doubles): the MMA fragment loads of
      // rows pp = 4 ks + tq hit distinct banks
      const int ldI = als_ld(int(I)), ldR = als_ld(R);
      T* fibT = reinterpret_cast<T*>(sm);                  // [2][BATCH][I], raw T (cp.async)
      double* fibD = sm + als_fib_doubles<T, BATCH>(I);           // [BATCH][ldI], converted once
      double* kc = fibD + BATCH * ldI;                 // [BATCH][ldR]
      T* fsm = reinterpret_cast<T*>(kc + BATCH * ldR); // other modes' factors, row-major (rank fastest)
      // gather: thread tid always handles position pp = tid % BATCH
      auto gather = [&](i64 pb, int buf) {
        const int pp = tid % BATCH;
        const bool ok = pb + pp < j1;
        const unsigned s_ = unsigned(ok ? pb + pp : pb);
        const unsigned a = s_ / unsigned(Rr), b = s_ - a * unsigned(Rr);
        const T* src = p.B + i64(a) * I * Rr + b;
        T* dst = fibT + buf * BATCH * int(I) + pp * int(I);
        for (int i = tid / BATCH; i < int(I); i += nt / BATCH) als_cp_elem(dst + i, src + i64(i) * Rr, ok);
        als_cp_commit();
      };
      // the first batch's fibers are in flight while the factors are staged
      if (j0 < j1) gather(j0, 0);
      {
        __syncthreads();
        if (tid == 0) {
          int off = 0;
          for (int k = 0; k < N; ++k) {
            sfoff[k] = off;
            sext[k] = int(p.sh.e[k]);
            if (k != m) off += int(p.sh.e[k]) * R;
          }
        }
        __syncthreads();
        for (int k = 0; k < N; ++k) {
          if (k == m) continue;
          const int nk = sext[k] * R;
          const T* src = p.fs.f[k];
          const int ek = sext[k];
          // transpose (a warp then reads one row's ranks) with every element's
          // copy in flight at once: one L2 round trip, not one per element
          for (int e = tid; e < nk; e += nt) {
            const int row = e / R, r = e - (e / R) * R;
            als_cp_elem(&fsm[sfoff[k] + e], &src[row + r * ek], true);
          }
        }
        als_cp_commit();
        als_cp_wait<0>();
        __syncthreads();
      }
      const bool stampA = p.prof != nullptr && g == 0 && tid == 0;
      unsigned long long ts = stampA ? gtimer() : 0;
      if (stampA) p.prof[22] += ts - tp0;
      auto stampa = [&](int slot) {
        if (stampA) {
          const unsigned long long t = gtimer();
          p.prof[slot] += t - ts;
          ts = t;
        }
      };
      // fibD rows beyond I and kc rows beyond R stay zero for the whole mode
      // step (the per-batch writes cover [0, I) and [0, R) only), so the MMA
      // fragment loads below need no bounds checks
      for (int e = tid; e < BATCH * (ldI + ldR); e += nt) fibD[e] = 0.0;  // kc follows fibD
      // this warp's tiles: packed (i0 | r0 << 16), the divisions done once
      int toff[kAlsTiles];
#pragma unroll
      for (int t = 0; t < kAlsTiles; ++t) {
        const int tile = wrp + t * nwarp;
        toff[t] = tile < NTILE ? ((16 * (tile % I16) + gq) | ((8 * (tile / I16) + gq) << 16)) : 0;
      }
      // Khatri-Rao rows: thread -> (column kr_r, first position kr_p0), stride kr_ps
      const int kr_ps = nt / R, kr_r = tid % R, kr_p0 = tid / R;
      __syncthreads();
      stampa(16);
      int buf = 0;
      for (i64 pb = j0; pb < j1; pb += BATCH, buf ^= 1) {
        const int np = int(j1 - pb < BATCH ? j1 - pb : BATCH);
        if (pb + BATCH < j1)
          gather(pb + BATCH, buf ^ 1);
        else
          als_cp_commit();  // keep one group per iteration
        stampa(17);
        if (tid < BATCH) {  // multi-index digits of each position, once (32-bit: J < 2^31)
          // stored as smem offsets of the factor rows, slot j = j-th other mode
          // from the highest down (the product order of kruskal.hpp:58-62)
          const unsigned s_ = unsigned(pb) + unsigned(tid);
          unsigned a = s_ / unsigned(Rr), b = s_ - a * unsigned(Rr);
          int j = 0;
          for (int k = N - 1; k > m; --k, ++j) {
            const unsigned ek = unsigned(sext[k]);
            pidx[tid * kMaxOrder + j] = sfoff[k] + int(b % ek) * R;
            b /= ek;
          }
          for (int k = m - 1; k >= 0; --k, ++j) {
            const unsigned ek = unsigned(sext[k]);
            pidx[tid * kMaxOrder + j] = sfoff[k] + int(a % ek) * R;
            a /= ek;
          }
        }
        __syncthreads();
        if (kr_p0 < kr_ps) {
          // four positions at a time: their index and factor loads issued
          // before the products (the per-position chain of dependent shared
          // loads was the longest stall of the MTTKRP); the same product order
          // (fp32 only: in the fp64 kernels the extra registers spill, C2 0.43 -> 0.46 ms)
          if ((sizeof(T) == 4 || CLUSTER) && N <= 4) {  // (one-cluster variant: registers to spare)
            for (int pp0 = kr_p0; pp0 < BATCH; pp0 += 4 * kr_ps) {
              T f[4][3];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int pp = pp0 + u * kr_ps;
                const int* po = pidx + (pp < np ? pp : 0) * kMaxOrder;
#pragma unroll
                for (int j = 0; j < 3; ++j) f[u][j] = j < N - 1 ? fsm[po[j] + kr_r] : T(1);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int pp = pp0 + u * kr_ps;
                if (pp >= BATCH) break;
                T prod = T(1);
#pragma unroll
                for (int j = 0; j < 3; ++j)
                  if (j < N - 1) prod *= f[u][j];
                kc[pp * ldR + kr_r] = pp < np ? double(prod) : 0.0;
              }
            }
          } else {
            for (int pp = kr_p0; pp < BATCH; pp += kr_ps) {
              double v = 0.0;
              if (pp < np) {
                const int* po = pidx + pp * kMaxOrder;
                T prod = T(1);
#pragma unroll
                for (int j = 0; j < kMaxOrder - 1; ++j)
                  if (j < N - 1) prod *= fsm[po[j] + kr_r];
                v = double(prod);
              }
              kc[pp * ldR + kr_r] = v;
            }
          }
        }
        stampa(18);
        als_cp_wait<1>();  // this batch's fibers (own copies) have landed
        {  // each thread converts the elements it copied itself (no barrier needed before)
          const int pp = tid % BATCH;
          const T* src = fibT + buf * BATCH * int(I) + pp * int(I);
          double* dst = fibD + pp * ldI;
#pragma unroll 4
          for (int i = tid / BATCH; i < int(I); i += nt / BATCH) dst[i] = double(src[i]);
        }
        __syncthreads();
        stampa(19);
        const double* fb = fibD;
        if (CLUSTER && NTILE <= nwarp) {
          // (one-cluster variant only: one CTA per SM, registers to spare; the grid
          // variant keeps 128 registers for two CTAs per SM)
          // at most one tile per warp (small compressed tensors: C1 / C2): one
          // accumulator would be a chain of BATCH / 4 dependent DMMAs (3.8 us per
          // batch at C2); four interleaved chains, summed pairwise per batch
          if (wrp < NTILE) {
            const int i0 = toff[0] & 0xffff, r0 = toff[0] >> 16;
            double a4[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a4[u][0] = a4[u][1] = a4[u][2] = a4[u][3] = 0.0;
#pragma unroll 2
            for (int ks4 = 0; ks4 < BATCH / 16; ++ks4) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int pp = 4 * (4 * ks4 + u) + tq;
                als_dmma(a4[u], fb[pp * ldI + i0], fb[pp * ldI + i0 + 8], kc[pp * ldR + r0]);
              }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[0][q] += (a4[0][q] + a4[1][q]) + (a4[2][q] + a4[3][q]);
          }
        } else {
#pragma unroll 2
          for (int ks = 0; ks < BATCH / 4; ++ks) {
            const int pp = 4 * ks + tq;
            const double* frow = fb + pp * ldI;
            const double* krow = kc + pp * ldR;
#pragma unroll
            for (int t = 0; t < kAlsTiles; ++t) {
              if (wrp + t * nwarp < NTILE) {  // zero padding beyond I and R (see above)
                const int i0 = toff[t] & 0xffff, r0 = toff[t] >> 16;
                als_dmma(acc[t], frow[i0], frow[i0 + 8], krow[r0]);
              }
            }
          }
        }
        __syncthreads();  // buffers are refilled next iteration
        stampa(20);
        if (stampA) p.prof[21] += 1;
      }
      als_cp_wait<0>();
      double* pt = p.part + (i64(parity) * G + g) * p.part_stride;
#pragma unroll
      for (int t = 0; t < kAlsTiles; ++t) {
        const int tile = wrp + t * nwarp;
        if (tile < NTILE) {
          const int ib = 16 * (tile % I16) + gq, rb = 8 * (tile / I16) + 2 * tq;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = ib + (q >> 1) * 8, r = rb + (q & 1);
            // the grid update reads each row's R outputs of one partial together
            if (i < I && r < R) pt[p.grid_update && split ? i64(i) * R + r : i + i64(r) * I] = acc[t][q];
          }
        }
      }
      unsigned long long tp1 = 0;
      if (p.prof && g == 0 && tid == 0) {
        tp1 = gtimer();
        p.prof[23] += tp1 - ts;
        p.prof[24] = G;
      }
      gsync();
      unsigned long long tp2 = 0;
      if (p.prof && g == 0 && tid == 0) tp2 = gtimer();
      if (split && p.grid_update) {
        const double* pp0 = p.part + i64(parity) * G * p.part_stride;
        double* Wg = p.part + 2 * i64(G) * p.part_stride;
        double* fraw = p.part + (2 * i64(G) + 2) * p.part_stride;
        FactorSet<T> fs = p.fs;
        als_update_grid<T>(fs, m, pp0, p.part_stride, GA, Wg, fraw, p.pm, p.weights, p.tol, p.max_iter, p.trace_fit,
                           p.trace_sec, p.st, sm, gsync, p.prof);
        parity ^= 1;
        if (p.prof && g == 0 && tid == 0) {
          const unsigned long long tp4 = gtimer();
          p.prof[0] += tp1 - tp0;
          p.prof[1] += tp2 - tp1;
          p.prof[2] += tp4 - tp2;
          p.prof[4] += 1;
        }
        continue;
      }
      // ---- reduction of the partials, spread over all CTAs (fixed CTA
      //      order per output: deterministic), into Wg after the partials
      double* Wg = p.part + 2 * i64(G) * p.part_stride;
      {
        const double* pp0 = p.part + i64(parity) * G * p.part_stride;
        // `sub` threads (a power of two <= 32, within one warp) per output:
        // member l sums partials l, l + sub, ... (16 loads in flight), then a
        // fixed butterfly over the group -- deterministic for a given G
        const int ch = (nout + G - 1) / G;
        const int o1 = min(nout, (g + 1) * ch);
        int sub = 1;
        while (sub < 32 && 2 * sub * ch <= nt) sub *= 2;
        const int gi = tid / sub, l = tid % sub, ng = nt / sub;
        for (int ob = g * ch; ob < o1; ob += ng) {  // uniform trip count: the shuffles see full warps
          const int o = ob + gi;
          const bool on = o < o1;
          double s = 0.0;
          for (int q0 = l; q0 < GA; q0 += 16 * sub) {
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int q = q0 + sub * u;
              v[u] = (on && q < GA) ? ldcg(&pp0[i64(q) * p.part_stride + o]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) s += v[u];
          }
          for (int off = sub / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
          if (on && l == 0) Wg[o] = s;
        }
      }
      gsync();
      // ---- B: mode update on CTA 0
      if (g == 0) {
        double* W = sm;                   // I x R
        double* work = sm + nout;         // 3 R^2 + 4 R
        // the MTTKRP result is a Matrix<Scalar> (solve.hpp:212-213): rounded once
        for (int o = tid; o < nout; o += nt) W[o] = double(T(ldcg(&Wg[o])));
        __syncthreads();
        if (p.prof && tid == 0) {
          g_als_prof = p.prof;
          p.prof[14] += gtimer() - tp2;
        }
        FactorSet<T> fs = p.fs;
        als_mode_update<T, double>(fs, m, W, p.weights, p.tol, p.max_iter, p.trace_fit, p.trace_sec, p.st, work,
                                   split ? 2 : 0, p.pm);
      }
      unsigned long long tp3 = 0;
      if (p.prof && g == 0 && tid == 0) tp3 = gtimer();
      parity ^= 1;
      gsync();
      if (p.prof && g == 0 && tid == 0) {
        const unsigned long long tp4 = gtimer();
        p.prof[0] += tp1 - tp0;
        p.prof[1] += tp2 - tp1;
        p.prof[2] += tp3 - tp2;
        p.prof[3] += tp4 - tp3;
        p.prof[4] += 1;
      }
    }
    if (ldcg(&p.st->done)) break;
  }
}

__global__ void als_start_kernel(AlsState* st, const double* nx2) {
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  st->it = 1;
  st->done = 0;
  st->converged = 0;
  st->error_it = -1;
  st->pivots_fallback = 0;
  st->prev_fit = 0.0;
  st->nx2 = nx2[0];
  st->t0 = now;
}

// ----------------------------------------------------------- normalize
// kruskal.hpp:117-176 on device (one CTA).
template <typename T>
__global__ void __launch_bounds__(kSmallThreads) normalize_kernel(FactorSet<T> fs, T* weights, T* tmp) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int R = fs.rank, N = fs.order;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const T skip = T(32) * Traits<T>::eps;
  __shared__ int s_order[kMaxRank];
  for (int j = wid; j < R; j += nw) {
    for (int m = 0; m < N; ++m) {
      T* f = fs.f[m] + i64(j) * fs.extent[m];
      const i64 n = fs.extent[m];
      double s = 0.0;
      for (i64 i = lane; i < n; i += 32) s += double(f[i]) * double(f[i]);
      s = warp_sum(s);
      const T nrm = T(sqrt(s));
      __syncwarp();
      if (nrm == T(0)) {
        for (i64 i = lane; i < n; i += 32) f[i] = (i == 0) ? T(1) : T(0);
        if (lane == 0) weights[j] = T(0);
      } else if (fabs(nrm - T(1)) > skip) {
        for (i64 i = lane; i < n; i += 32) f[i] = f[i] / nrm;
        if (lane == 0) weights[j] = weights[j] * nrm;
      }
      __syncwarp();
    }
    const bool neg = weights[j] < T(0);
    __syncwarp();
    T* f0 = fs.f[0] + i64(j) * fs.extent[0];
    const i64 n0 = fs.extent[0];
    if (neg) {
      if (lane == 0) weights[j] = -weights[j];
      for (i64 i = lane; i < n0; i += 32) f0[i] = -f0[i];
    }
    __syncwarp();
    if (N >= 2) {
      // first index of the max |entry| of factor 0's column
      T best = T(-1);
      i64 at = 0;
      for (i64 i = lane; i < n0; i += 32) {
        const T x = fabs(f0[i]);
        if (x > best) {
          best = x;
          at = i;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const T ob = __shfl_xor_sync(0xffffffffu, best, o);
        const i64 oa = __shfl_xor_sync(0xffffffffu, at, o);
        if (ob > best || (ob == best && oa < at)) {
          best = ob;
          at = oa;
        }
      }
      const bool flip = f0[at] < T(0);
      __syncwarp();
      if (flip) {
        for (i64 i = lane; i < n0; i += 32) f0[i] = -f0[i];
        T* f1 = fs.f[1] + i64(j) * fs.extent[1];
        for (i64 i = lane; i < fs.extent[1]; i += 32) f1[i] = -f1[i];
      }
    }
  }
  __syncthreads();
  // stable sort: weight descending, ties by lexicographic factor-0 column
  for (int a = tid; a < R; a += nt) {
    int pos = 0;
    const double wa = -order_key(-double(weights[a]));  // NaN -> -inf: last
    const T* ca = fs.f[0] + i64(a) * fs.extent[0];
    for (int b = 0; b < R; ++b) {
      if (b == a) continue;
      const double wb = -order_key(-double(weights[b]));
      bool before;
      if (wb != wa) {
        before = wb > wa;
      } else {
        const T* cb = fs.f[0] + i64(b) * fs.extent[0];
        int cmp = 0;
        for (i64 i = 0; i < fs.extent[0]; ++i) {
          const double xb = order_key(double(cb[i])), xa = order_key(double(ca[i]));
          if (xb != xa) {
            cmp = xb < xa ? -1 : 1;
            break;
          }
        }
        before = cmp < 0 || (cmp == 0 && b < a);
      }
      pos += before ? 1 : 0;
    }
    s_order[pos] = a;
  }
  __syncthreads();
  bool ident = true;
  for (int j = 0; j < R; ++j) ident = ident && (s_order[j] == j);
  if (ident) return;
  // permute columns through tmp
  i64 off = 0;
  for (int m = 0; m < N; ++m) {
    const i64 n = fs.extent[m];
    for (i64 e = tid; e < n * R; e += nt) tmp[off + e] = fs.f[m][e];
    off += n * R;
  }
  for (int j = tid; j < R; j += nt) tmp[off + j] = weights[j];
  __syncthreads();
  off = 0;
  for (int m = 0; m < N; ++m) {
    const i64 n = fs.extent[m];
    for (i64 e = tid; e < n * R; e += nt) {
      const i64 i = e % n;
      const int j = int(e / n);
      fs.f[m][e] = tmp[off + i + i64(s_order[j]) * n];
    }
    off += n * R;
  }
  for (int j = tid; j < R; j += nt) weights[j] = tmp[off + s_order[j]];
}

template <typename T>
__global__ void small_gemm_kernel(const T* Q, i64 dim, i64 l, const T* A, int rank, T* out) {
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < dim * rank; e += i64(gridDim.x) * blockDim.x) {
    const i64 i = e % dim, r = e / dim;
    double s = 0.0;
    for (i64 c = 0; c < l; ++c) s += double(Q[i + c * dim]) * double(A[c + r * l]);
    out[e] = T(s);
  }
}

// ------------------------------------------------------------ reductions
template <typename T>
__global__ void __launch_bounds__(256) norm_finite_kernel(const T* __restrict__ x, i64 n, double* part,
                                                          const double* cond = nullptr) {
  if (cond != nullptr && *cond == 0.0) {  // the caller proved the input finite (sum not needed)
    if (threadIdx.x == 0) {
      part[2 * blockIdx.x] = 0.0;
      part[2 * blockIdx.x + 1] = 0.0;
    }
    return;
  }
  // 16-byte loads, four in flight per thread (a streaming reduction needs many
  // bytes in flight per SM to reach HBM bandwidth); scalar head/tail
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int W = 16 / int(sizeof(T));
  double s = 0.0, bad = 0.0;
  auto acc = [&](T t) {
    const double v = double(t);
    if (isfinite(v))
      s += v * v;
    else
      bad += 1.0;
  };
  const i64 head = i64((16 - (reinterpret_cast<uintptr_t>(x) & 15)) & 15) / i64(sizeof(T));
  const i64 h = head < n ? head : n;
  const i64 nv = (n - h) / W;
  const V* xv = reinterpret_cast<const V*>(x + h);
  const i64 tid = blockIdx.x * i64(blockDim.x) + threadIdx.x, nth = i64(gridDim.x) * blockDim.x;
  if (tid < h) acc(x[tid]);
  i64 e = tid;
  for (; e + 3 * nth < nv; e += 4 * nth) {
    V v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(xv + e + u * nth);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const T* t = reinterpret_cast<const T*>(&v[u]);
#pragma unroll
      for (int w = 0; w < W; ++w) acc(t[w]);
    }
  }
  for (; e < nv; e += nth) {
    const V v = __ldcs(xv + e);
    const T* t = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int w = 0; w < W; ++w) acc(t[w]);
  }
  for (i64 r = h + nv * W + tid; r < n; r += nth) acc(x[r]);
  s = block_reduce_sum(s);
  bad = block_reduce_sum(bad);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s;
    part[2 * blockIdx.x + 1] = bad;
  }
}

// Fixed-order (deterministic) sum of nblocks (a, b) pairs by one CTA.
__global__ void sum_pairs_kernel(const double* part, int nblocks, double* out, const int* skip = nullptr) {
  if (skip != nullptr && *skip) return;
  double a = 0.0, b = 0.0;
  for (int q = threadIdx.x; q < nblocks; q += blockDim.x) {
    a += part[2 * q];
    b += part[2 * q + 1];
  }
  a = block_reduce_sum(a);
  b = block_reduce_sum(b);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

constexpr int kResRows = 16;

// ||X - Xhat||^2 and ||X||^2 streamed over X (row-major prefix x last mode):
// Xhat(p, l) = sum_r coef[p][r] A_last[l][r], coef = lambda_r prod_{m<N-1} A_m.
// Each CTA takes kResRows prefix rows at a time; the 16 X loads per thread
// are independent (memory-level parallelism), A_last is read once per r for
// all 16 rows.
template <typename T>
__global__ void __launch_bounds__(256) residual_kernel(const T* X, ShapeArg sh, FactorSet<T> fs, const T* w,
                                                       double* part, const int* skip = nullptr) {
  if (skip != nullptr && *skip) return;
  __shared__ T coef[kMaxRank][kResRows];
  __shared__ int dig[kResRows][kMaxOrder];
  __shared__ const T* fptr[kMaxOrder];
  __shared__ int ext[kMaxOrder];
  const int R = fs.rank, N = sh.n;
  if (threadIdx.x < kMaxOrder) {
    fptr[threadIdx.x] = threadIdx.x < N ? fs.f[threadIdx.x] : nullptr;
    ext[threadIdx.x] = threadIdx.x < N ? int(sh.e[threadIdx.x]) : 1;
  }
  const i64 last = sh.e[N - 1];
  i64 prefix = 1;
  for (int m = 0; m < N - 1; ++m) prefix *= sh.e[m];
  const T* Al = fs.f[N - 1];
  double acc_r = 0.0, acc_x = 0.0;
  __syncthreads();
  for (i64 p0 = i64(blockIdx.x) * kResRows; p0 < prefix; p0 += i64(gridDim.x) * kResRows) {
    __syncthreads();
    if (threadIdx.x < kResRows) {  // multi-index digits of this row, once
      i64 rem = p0 + threadIdx.x;
      for (int m = N - 2; m >= 0; --m) {
        dig[threadIdx.x][m] = int(rem % ext[m]);
        rem /= ext[m];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kResRows * R; e += blockDim.x) {
      const int q = e % kResRows, r = e / kResRows;
      T v = T(0);
      if (p0 + q < prefix) {
        v = w[r];
        for (int m = N - 2; m >= 0; --m) v *= fptr[m][dig[q][m] + i64(r) * ext[m]];
      }
      coef[r][q] = v;
    }
    __syncthreads();
    const int nrows = int(prefix - p0 < kResRows ? prefix - p0 : kResRows);
    for (i64 il = threadIdx.x; il < last; il += blockDim.x) {
      T xv[kResRows];
#pragma unroll
      for (int q = 0; q < kResRows; ++q) xv[q] = q < nrows ? X[(p0 + q) * last + il] : T(0);
      T xh[kResRows];
#pragma unroll
      for (int q = 0; q < kResRows; ++q) xh[q] = T(0);
      for (int r = 0; r < R; ++r) {
        const T a = Al[il + i64(r) * last];
#pragma unroll
        for (int q = 0; q < kResRows; ++q) xh[q] = fma(coef[r][q], a, xh[q]);
      }
#pragma unroll
      for (int q = 0; q < kResRows; ++q) {
        const double x = double(xv[q]);
        const double d = x - double(xh[q]);
        acc_r += d * d;
        acc_x += x * x;
      }
    }
  }
  acc_r = block_reduce_sum(acc_r);
  acc_x = block_reduce_sum(acc_x);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = acc_r;
    part[2 * blockIdx.x + 1] = acc_x;
  }
}

// fp64 ||X - Xhat||^2 and ||X||^2 with Xhat on the FP64 tensor cores
// (mma.m16n8k4): X viewed as prefix x last (row-major), Xhat(p, l) =
// sum_r coef[p][r] A_last[l][r]. A_last^T stays in smem for the whole
// launch; per block of 64 prefix rows the coefficients are formed once and
// every warp keeps its 16-row A fragments in registers while it walks half
// of the n8 column tiles. X is read straight into the accumulator fragment
// layout (two consecutive doubles per row per thread) and compared in fp64.
// The SIMT residual_kernel is smem bound (one shared load per FMA); here a
// DMMA does 512 FMAs from three register fragments.
constexpr int kRdRows = 64;  // 4 m16 tiles per block step, 8 warps

template <int KS>  // k4 steps: rank <= 4 * KS
__global__ void __launch_bounds__(256) residual_dmma_kernel(const double* __restrict__ X, ShapeArg sh,
                                                            FactorSet<double> fs, const double* __restrict__ w,
                                                            double* part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int dig[kRdRows][kMaxOrder];
  const int R = fs.rank, N = sh.n;
  const int L = int(sh.e[N - 1]);
  const int NT8 = (L + 7) / 8;
  constexpr int ldb = 4 * KS + 1;  // odd: the fragment reads spread over the banks
  double* Bs = reinterpret_cast<double*>(smem_raw);  // [NT8 * 8][ldb] A_last rows (zero padded)
  double* Cs = Bs + i64(NT8) * 8 * ldb;               // [kRdRows][ldb] coefficients
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const double* Al = fs.f[N - 1];
  for (int e = tid; e < NT8 * 8 * 4 * KS; e += blockDim.x) {
    const int l = e / (4 * KS), r = e - l * (4 * KS);
    Bs[l * ldb + r] = (l < L && r < R) ? Al[l + i64(r) * L] : 0.0;
  }
  i64 prefix = 1;
  for (int m = 0; m < N - 1; ++m) prefix *= sh.e[m];
  const int mt = warp & 3, nh = warp >> 2;
  const bool v16 = (L & 1) == 0;
  double acc_r = 0.0, acc_x = 0.0;
  for (i64 p0 = i64(blockIdx.x) * kRdRows; p0 < prefix; p0 += i64(gridDim.x) * kRdRows) {
    __syncthreads();
    if (tid < kRdRows) {
      i64 rem = p0 + tid;
      for (int m = N - 2; m >= 0; --m) {
        dig[tid][m] = int(rem % sh.e[m]);
        rem /= sh.e[m];
      }
    }
    __syncthreads();
    for (int e = tid; e < kRdRows * 4 * KS; e += blockDim.x) {
      const int q = e % kRdRows, r = e / kRdRows;
      double v = 0.0;
      if (p0 + q < prefix && r < R) {
        v = w[r];
        for (int m = N - 2; m >= 0; --m) v *= fs.f[m][dig[q][m] + i64(r) * sh.e[m]];
      }
      Cs[q * ldb + r] = v;
    }
    __syncthreads();
    double a0[KS], a1[KS];
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      a0[s] = Cs[(mt * 16 + g) * ldb + 4 * s + t];
      a1[s] = Cs[(mt * 16 + g + 8) * ldb + 4 * s + t];
    }
    const i64 row0 = p0 + mt * 16 + g, row1 = row0 + 8;
    const bool ok0 = row0 < prefix, ok1 = row1 < prefix;
    const double* x0 = X + row0 * L;
    const double* x1 = X + row1 * L;
    // X of kPf tiles loaded before their MMAs: with the loads interleaved with the
    // (volatile asm) MMAs one HBM latency was exposed per tile (C2: 2.2 TB/s)
    constexpr int kPf = 8;
    for (int nb = nh; nb < NT8; nb += 2 * kPf) {
      double xv[kPf][4];
#pragma unroll
      for (int u = 0; u < kPf; ++u) {
        const int nt = nb + 2 * u;
        const int c = nt * 8 + 2 * t;
        xv[u][0] = xv[u][1] = xv[u][2] = xv[u][3] = 0.0;
        if (nt >= NT8) continue;
        if (v16 && c + 1 < L) {
          if (ok0) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(x0 + c));
            xv[u][0] = v.x;
            xv[u][1] = v.y;
          }
          if (ok1) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(x1 + c));
            xv[u][2] = v.x;
            xv[u][3] = v.y;
          }
        } else {
          if (ok0 && c < L) xv[u][0] = x0[c];
          if (ok0 && c + 1 < L) xv[u][1] = x0[c + 1];
          if (ok1 && c < L) xv[u][2] = x1[c];
          if (ok1 && c + 1 < L) xv[u][3] = x1[c + 1];
        }
      }
#pragma unroll
      for (int u = 0; u < kPf; ++u) {
        const int nt = nb + 2 * u;
        if (nt >= NT8) break;
        const int c = nt * 8 + 2 * t;
        const double x00 = xv[u][0], x01 = xv[u][1], x10 = xv[u][2], x11 = xv[u][3];
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int s = 0; s < KS; ++s) als_dmma(acc, a0[s], a1[s], Bs[(nt * 8 + g) * ldb + 4 * s + t]);
        // acc: (row g, col c), (g, c + 1), (g + 8, c), (g + 8, c + 1); padding is zero on both sides
        const double d00 = x00 - acc[0], d01 = x01 - acc[1], d10 = x10 - acc[2], d11 = x11 - acc[3];
        const bool c0 = c < L, c1 = c + 1 < L;
        acc_r += (ok0 && c0 ? d00 * d00 : 0.0) + (ok0 && c1 ? d01 * d01 : 0.0) + (ok1 && c0 ? d10 * d10 : 0.0) +
                 (ok1 && c1 ? d11 * d11 : 0.0);
        acc_x += (x00 * x00 + x01 * x01) + (x10 * x10 + x11 * x11);
      }
    }
  }
  acc_r = block_reduce_sum(acc_r);
  acc_x = block_reduce_sum(acc_x);
  if (tid == 0) {
    part[2 * blockIdx.x] = acc_r;
    part[2 * blockIdx.x + 1] = acc_x;
  }
}

// ------------------------------------------------------------ synthetic
struct DFactors {
  const double* f[kMaxOrder];
};

template <typename T>
__global__ void synth_reconstruct_kernel(ShapeArg sh, int R, const double* w, DFactors fs, T* out, i64 total) {
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    i64 idx[kMaxOrder];
    i64 rem = e;
    for (int m = sh.n - 1; m >= 0; --m) {
      idx[m] = rem % sh.e[m];
      rem /= sh.e[m];
    }
    double s = 0.0;
    for (int r = 0; r < R; ++r) {
      double p = w[r];
      for (int m = 0; m < sh.n; ++m) p *= fs.f[m][idx[m] + i64(r) * sh.e[m]];
      s += p;
    }
    out[e] = T(s);
  }
}

template <typename T>
__global__ void sum_and_sq_kernel(const T* x, i64 n, double mean, double* part) {
  double s = 0.0, q = 0.0;
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < n; e += i64(gridDim.x) * blockDim.x) {
    const double v = double(x[e]);
    s += v;
    q += (v - mean) * (v - mean);
  }
  s = block_reduce_sum(s);
  q = block_reduce_sum(q);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s;
    part[2 * blockIdx.x + 1] = q;
  }
}

template <typename T>
__global__ void add_noise_kernel(T* x, i64 n, T sigma, u64 s0) {
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < n; e += i64(gridDim.x) * blockDim.x)
    x[e] += sigma * T(normal_at(s0, u64(e)));
}

}  // namespace

// ================================================================ host
template <typename T>
void kr_panel(const FactorSet<T>& fs, const i64* shape, int mode, T* out, cudaStream_t st, const int* skip) {
  const ShapeArg sh = make_shape(shape, fs.order);
  i64 L = 1, Rr = 1;
  for (int m = 0; m < mode; ++m) L *= shape[m];
  for (int m = mode + 1; m < fs.order; ++m) Rr *= shape[m];
  const i64 J = L * Rr;
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(J * fs.rank, 256), 148 * 16)));
  kr_panel_kernel<T><<<blocks, 256, 0, st>>>(fs, sh, mode, J, Rr, out, skip);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
void init_factors_from_grams(const InitBatch<T>& b, int count, int rank, u64 seed, int method, cudaStream_t st) {
  check_arg(rank <= kMaxRank, "init_factors: rank above the supported maximum");
  check_arg(count >= 1 && count <= kMaxOrder, "init_factors: mode count");
  size_t smem = 0;
  for (int q = 0; q < count; ++q)
    if (b.n[q] <= kEigSmemMax) smem = std::max(smem, 2 * size_t(b.n[q]) * size_t(b.n[q] | 1) * sizeof(double));
  static const size_t lim = enable_max_dyn_smem(init_from_gram_kernel<T>);
  (void)lim;
  // 1024 threads: a Jacobi round rotates up to 48 row/column pairs, one warp each
  init_from_gram_kernel<T><<<count, kSmallThreads, smem, st>>>(b, rank, seed, method);
  count_launch();
  RCPG_LAUNCHED();
}

size_t init_work_doubles(int n) { return 2 * size_t(n) * size_t(n | 1) + 4 * size_t(n) + 64; }

namespace {
// Tail energy of one Gram G = X_(m) X_(m)^T (n x n, fp64): the sum of its
// n - k smallest eigenvalues (clamped at 0) = sum_{j >= k} sigma_j^2 of the
// unfolding (diagnostics.hpp:47-58), one CTA per mode.
__global__ void __launch_bounds__(kSmallThreads) gram_tail_kernel(TailBatch b, int k, double* out) {
  const int q = blockIdx.x, n = b.n[q], tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const bool in_smem = n <= kEigSmemMax;
  const int ld = n | 1;
  double* work = b.work[q];
  double* A = in_smem ? reinterpret_cast<double*>(smem_raw) : work;
  double* V = A + i64(n) * ld;
  double* ev = work + 2 * i64(n) * ld;
  int* ord = reinterpret_cast<int*>(ev + n);
  for (i64 e = tid; e < i64(n) * n; e += nt) A[(e % n) + (e / n) * ld] = b.G[q][e];
  __syncthreads();
  jacobi_eig(A, V, n, ld, ev, ord);
  if (tid == 0) {
    double t = 0.0;
    for (int j = 0; j < n - k; ++j) t += ev[j] > 0.0 ? ev[j] : 0.0;  // ascending: the n - k smallest
    out[q] = t;
  }
}
}  // namespace

void gram_tails(const TailBatch& b, int count, int k, double* out, cudaStream_t st) {
  check_arg(count >= 1 && count <= kMaxOrder, "theorem_bound: mode count");
  size_t smem = 0;
  for (int q = 0; q < count; ++q) {
    check_arg(b.n[q] <= 2 * kMaxRank * 8, "theorem_bound: extents up to 2048");
    if (b.n[q] <= kEigSmemMax) smem = std::max(smem, 2 * size_t(b.n[q]) * size_t(b.n[q] | 1) * sizeof(double));
  }
  static const size_t lim = enable_max_dyn_smem(gram_tail_kernel);
  (void)lim;
  gram_tail_kernel<<<count, kSmallThreads, smem, st>>>(b, k, out);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
void zero_factor(T* factor, i64 extent, int rank, T* gram_out, cudaStream_t st) {
  zero_factor_kernel<T><<<64, 256, 0, st>>>(factor, extent, rank, gram_out);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
void als_update(const FactorSet<T>& fs, int mode, const T* W, T* weights, double tol, int max_iter,
                double* trace_fit, double* trace_sec, AlsState* state, double* work, cudaStream_t st) {
  const int R = fs.rank;
  const size_t smem = (3 * size_t(R) * R + 5 * size_t(R) + size_t(fs.extent[mode]) * R) * sizeof(double);
  check_arg(R <= kAlsSmemRank && smem <= 200 * 1024, "als: mode update exceeds the shared-memory plan");
  static const size_t lim = enable_max_dyn_smem(als_update_kernel<T>);
  (void)lim;
  als_update_kernel<T><<<1, kSmallThreads, smem, st>>>(fs, mode, W, weights, tol, max_iter, trace_fit, trace_sec,
                                                        state, work);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
bool als_loop_supported(const i64* shape, int order, int rank) {
  if (rank > kAlsSmemRank) return false;
  i64 S = 1;
  for (int m = 0; m < order; ++m) S *= shape[m];
  if (S >= (i64(1) << 31)) return false;  // 32-bit position arithmetic in the loop kernel
  for (int m = 0; m < order; ++m) {
    if (shape[m] * rank > i64(kAlsAcc) * kAlsThreads) return false;
    i64 fac = 0;
    for (int k = 0; k < order; ++k)
      if (k != m) fac += shape[k] * rank;
    const size_t smA = (size_t(als_fib_doubles<T>(shape[m])) + size_t(kAlsBatch) * (als_ld(int(shape[m])) + als_ld(rank))) * sizeof(double) +
                       size_t(fac) * sizeof(T);
    if (((shape[m] + 15) / 16) * ((rank + 7) / 8) > i64(kAlsTiles) * (kAlsThreads / 32)) return false;
    const size_t smB = (2 * size_t(shape[m]) * rank + 3 * size_t(rank) * rank + 6 * size_t(rank)) * sizeof(double);
    if (std::max(smA, smB) > 180 * 1024) return false;
  }
  return true;
}

template <typename T, int BATCH>
size_t als_loop_smem(const i64* shape, int order, int R) {
  size_t smem = 0;
  for (int m = 0; m < order; ++m) {
    i64 fac = 0;
    for (int k = 0; k < order; ++k)
      if (k != m) fac += shape[k] * R;
    const size_t smA = (size_t(als_fib_doubles<T, BATCH>(shape[m])) +
                        size_t(BATCH) * (als_ld(int(shape[m])) + als_ld(R))) * sizeof(double) +
                       size_t(fac) * sizeof(T);
    const size_t smB = (2 * size_t(shape[m]) * R + 3 * size_t(R) * R + 6 * size_t(R)) * sizeof(double);
    smem = std::max(smem, std::max(smA, smB));
  }
  return smem;
}

template <typename T>
void als_loop(const T* B, const i64* shape, int order, const FactorSet<T>& fs, T* weights, double tol, int max_iter,
              double* trace_fit, double* trace_sec, AlsState* state, double* part, i64 part_elems, GridBarrier* bar,
              cudaStream_t st, unsigned long long* prof) {
  const int R = fs.rank;
  i64 maxJ = 1, S = 1, maxout = 1;
  for (int m = 0; m < order; ++m) S *= shape[m];
  for (int m = 0; m < order; ++m) {
    maxJ = std::max(maxJ, S / shape[m]);
    maxout = std::max(maxout, shape[m] * R);
  }
  AlsLoopArgs<T> a{B, make_shape(shape, order), fs, weights, tol, max_iter, trace_fit, trace_sec, state, part,
                   nullptr, maxout, bar, prof, 1};
  static const bool grid_upd = [] {  // RCPG_ALS_GRIDUPD=0: CTA 0 does the mode update (A/B hook)
    const char* e = std::getenv("RCPG_ALS_GRIDUPD");
    return !(e != nullptr && e[0] == '0');
  }();
  a.grid_update = grid_upd && R >= 8 ? 1 : 0;  // (B1's subset sums fit the smem layout from R = 8)
  // 64-position batches when they fit: half the per-batch latency chains
  static const size_t lim64 = enable_max_dyn_smem(als_loop_kernel<T, 64>);
  static const size_t lim32 = enable_max_dyn_smem(als_loop_kernel<T, 32>);
  (void)lim64;
  (void)lim32;
  auto run = [&](auto kern, size_t smem, int batch) {
    const int maxc = max_coop_blocks(kern, kAlsThreads, smem);
    // pinv(V) of the mode on one extra CTA, concurrently with the MTTKRP (stored after the
    // reduced W); RCPG_ALS_SPLIT=0: CTA 0 does the whole mode update after the MTTKRP (A/B hook)
    const char* sp = std::getenv("RCPG_ALS_SPLIT");
    const bool want_split = !(sp != nullptr && sp[0] == '0') && i64(R) * R <= maxout;
    int G = int(std::max<i64>(1, std::min<i64>(ceil_div(maxJ, batch) + (want_split ? 1 : 0), maxc)));
    // + slots for the reduced W, pinv(V) and the grid update's unnormalized factor
    G = int(std::min<i64>(G, part_elems / (2 * maxout) - 2));
    static const int g_cap = std::getenv("RCPG_ALS_MAXG") ? atoi(std::getenv("RCPG_ALS_MAXG")) : 0;  // A/B hook
    if (g_cap > 0) G = std::min(G, g_cap);
    G = std::max(G, 1);
    const bool split_ok = want_split && G >= 3 && (2 * i64(G) + 3) * maxout <= part_elems;
    a.pm = split_ok ? part + (2 * i64(G) + 1) * maxout : nullptr;
    return G;
  };
  const size_t s64 = als_loop_smem<T, 64>(shape, order, R);
  const bool b64 = s64 <= 180 * 1024;
  const size_t smem = b64 ? s64 : als_loop_smem<T, 32>(shape, order, R);
  const int G = b64 ? run(als_loop_kernel<T, 64>, smem, 64) : run(als_loop_kernel<T, 32>, smem, 32);
  // small grids run as one thread-block cluster (cluster barriers); RCPG_ALS_CLUSTER=0 (A/B) keeps the grid
  static const bool cl_np = [] {
    return cudaFuncSetAttribute(als_loop_kernel<T, 64, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
               cudaSuccess &&
           cudaFuncSetAttribute(als_loop_kernel<T, 32, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
               cudaSuccess;
  }();
  static const bool cl_off = [] {
    const char* e = std::getenv("RCPG_ALS_CLUSTER");
    return e != nullptr && e[0] == '0';
  }();
  if (!cl_off && G >= 2 && G <= (cl_np ? 16 : 8)) {
    auto kern = b64 ? als_loop_kernel<T, 64, true> : als_loop_kernel<T, 32, true>;
    static const size_t l64c = enable_max_dyn_smem(als_loop_kernel<T, 64, true>);
    static const size_t l32c = enable_max_dyn_smem(als_loop_kernel<T, 32, true>);
    if (smem <= (b64 ? l64c : l32c)) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(kAlsThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = G;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters >= 1) {
        RCPG_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
        count_launch();
        return;
      }
      (void)cudaGetLastError();
    }
  }
  if (b64)
    launch_coop(als_loop_kernel<T, 64>, G, kAlsThreads, smem, st, a);
  else
    launch_coop(als_loop_kernel<T, 32>, G, kAlsThreads, smem, st, a);
}

template <typename T>
__global__ void fill_ones_kernel(T* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = T(1);
}

template <typename T>
void fill_ones(T* p, int n, cudaStream_t st) {
  fill_ones_kernel<T><<<1, 128, 0, st>>>(p, n);
  count_launch();
  RCPG_LAUNCHED();
}

void als_start(AlsState* state, double* nx2_src, cudaStream_t st) {
  als_start_kernel<<<1, 1, 0, st>>>(state, nx2_src);
  count_launch();
  RCPG_LAUNCHED();
}

// als_start + zero_factor + the initial weights in one launch (three dependent
// 3 us kernels before): state reset and t0, factor 0 = zeros (solve.hpp:98) with
// its Gram, weights = wval (ones for ALS, solve.hpp:190; zeros for BCD, :281).
template <typename T>
__global__ void als_prepare_kernel(AlsState* st, const double* nx2, T* F, i64 n, int R, T* gram, T* weights, T wval) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    st->it = 1;
    st->done = 0;
    st->converged = 0;
    st->error_it = -1;
    st->pivots_fallback = 0;
    st->prev_fit = 0.0;
    st->nx2 = nx2[0];
    st->t0 = now;
  }
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < R; j += blockDim.x) weights[j] = wval;
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < n * R; e += i64(gridDim.x) * blockDim.x) F[e] = T(0);
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < i64(R) * R; e += i64(gridDim.x) * blockDim.x)
    gram[e] = T(0);
}

template <typename T>
void als_prepare(AlsState* state, double* nx2_src, T* factor0, i64 extent0, int rank, T* gram0, T* weights, T wval,
                 cudaStream_t st) {
  als_prepare_kernel<T><<<64, 256, 0, st>>>(state, nx2_src, factor0, extent0, rank, gram0, weights, wval);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
void normalize_model(const FactorSet<T>& fs, T* weights, T* tmp, cudaStream_t st) {
  normalize_kernel<T><<<1, kSmallThreads, 0, st>>>(fs, weights, tmp);
  count_launch();
  RCPG_LAUNCHED();
}

// recover's A_n = Q_n A~_n of every non-identity mode in one launch
// (blockIdx.y = entry; the per-output sums are small_gemm_kernel's)
template <typename T>
__global__ void small_gemm_batch_kernel(SmallGemmBatch<T> b, int rank) {
  const int q = blockIdx.y;
  const T* Q = b.Q[q];
  const T* A = b.A[q];
  T* out = b.out[q];
  const i64 dim = b.dim[q], l = b.l[q];
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < dim * rank; e += i64(gridDim.x) * blockDim.x) {
    const i64 i = e % dim, r = e / dim;
    double s = 0.0;
    for (i64 c = 0; c < l; ++c) s += double(Q[i + c * dim]) * double(A[c + r * l]);
    out[e] = T(s);
  }
}

template <typename T>
void small_gemm_batch(const SmallGemmBatch<T>& b, int count, int rank, cudaStream_t st) {
  if (count <= 0) return;
  i64 most = 1;
  for (int q = 0; q < count; ++q) most = std::max(most, b.dim[q] * rank);
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(most, 256), 148 * 8)));
  small_gemm_batch_kernel<T><<<dim3(unsigned(blocks), unsigned(count)), 256, 0, st>>>(b, rank);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
void small_gemm(const T* Q, i64 dim, i64 l, const T* A, int rank, T* out, cudaStream_t st) {
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(dim * rank, 256), 148 * 8)));
  small_gemm_kernel<T><<<blocks, 256, 0, st>>>(Q, dim, l, A, rank, out);
  count_launch();
  RCPG_LAUNCHED();
}

// flag (zeroed here) += 1 per CTA that saw a non-finite entry of y
template <typename T>
__global__ void nonfinite_flag_kernel(const T* __restrict__ y, i64 n, double* flag) {
  bool bad = false;
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < n; e += i64(gridDim.x) * blockDim.x)
    bad |= !isfinite(double(y[e]));
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(flag, 1.0);
}

template <typename T>
void nonfinite_flag(const T* y, i64 n, double* flag, cudaStream_t st) {
  RCPG_CUDA(cudaMemsetAsync(flag, 0, sizeof(double), st));
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(n, 256 * 8), 296)));
  nonfinite_flag_kernel<T><<<blocks, 256, 0, st>>>(y, n, flag);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
void norm_and_finite(const T* x, i64 n, double* out2, double* scratch, int num_sms, cudaStream_t st,
                     const double* cond) {
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(n, 256), i64(num_sms) * 4)));
  norm_finite_kernel<T><<<blocks, 256, 0, st>>>(x, n, scratch, cond);
  sum_pairs_kernel<<<1, 256, 0, st>>>(scratch, blocks, out2);
  count_launch(2);
  RCPG_LAUNCHED();
}

template <int KS>
bool launch_residual_dmma(const double* X, const ShapeArg& sh, const FactorSet<double>& fs, const double* w,
                          double* part, int blocks, i64 L, cudaStream_t st) {
  // [NT8 * 8 + kRdRows][4 KS + 1] doubles, the kernel's own layout
  const size_t smem = (size_t(ceil_div(L, 8)) * 8 + kRdRows) * size_t(4 * KS + 1) * sizeof(double);
  static const size_t lim = enable_max_dyn_smem(residual_dmma_kernel<KS>);
  if (smem > lim) return false;
  residual_dmma_kernel<KS><<<blocks, 256, smem, st>>>(X, sh, fs, w, part);
  count_launch();
  RCPG_LAUNCHED();
  return true;
}

size_t residual_scratch_doubles(int num_sms, i64 last_extent, int rank) {
  // per-CTA partial pairs (+ the C^T hi / lo planes of the tensor-core path)
  return size_t(num_sms) * 8 * 2 + 16 + (residual_tc_scratch_floats(last_extent, rank) + 1) / 2 + 16;
}

template <typename T>
void residual_norms(const T* X, const i64* shape, int order, const FactorSet<T>& fs, const T* weights,
                    double* out2, double* scratch, int num_sms, cudaStream_t st) {
  check_arg(fs.rank <= kMaxRank, "relative_error: rank above the supported maximum");
  if constexpr (std::is_same<T, float>::value) {
    if (tc_residual_ok(shape, order, fs.rank)) {  // Xhat on the tensor cores (passes_tc.cu)
      int blocks = 0;
      double* part = scratch;
      float* ct = reinterpret_cast<float*>(scratch + size_t(num_sms) * 2 + 16);
      residual_tc(X, shape, order, fs.f, weights, fs.rank, ct, part, num_sms, blocks, st);
      sum_pairs_kernel<<<1, 256, 0, st>>>(part, blocks, out2);
      count_launch();
      RCPG_LAUNCHED();
      return;
    }
  }
  const ShapeArg sh = make_shape(shape, order);
  i64 prefix = 1;
  for (int m = 0; m < order - 1; ++m) prefix *= shape[m];
  if constexpr (std::is_same<T, double>::value) {
    const i64 L = shape[order - 1];
    const int KS = (fs.rank + 3) / 4;
    if (order >= 2 && KS <= 8 && L >= 8 && std::getenv("RCPG_RESIDUAL_SIMT") == nullptr) {
      const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(prefix, kRdRows), i64(num_sms) * 2)));
      bool done = false;
      if (KS <= 2) done = launch_residual_dmma<2>(X, sh, fs, weights, scratch, blocks, L, st);
      else if (KS <= 3) done = launch_residual_dmma<3>(X, sh, fs, weights, scratch, blocks, L, st);
      else if (KS <= 4) done = launch_residual_dmma<4>(X, sh, fs, weights, scratch, blocks, L, st);
      else if (KS <= 5) done = launch_residual_dmma<5>(X, sh, fs, weights, scratch, blocks, L, st);
      else if (KS <= 6) done = launch_residual_dmma<6>(X, sh, fs, weights, scratch, blocks, L, st);
      else done = launch_residual_dmma<8>(X, sh, fs, weights, scratch, blocks, L, st);
      if (done) {
        sum_pairs_kernel<<<1, 256, 0, st>>>(scratch, blocks, out2);
        count_launch();
        RCPG_LAUNCHED();
        return;
      }
    }
  }
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(prefix, kResRows), i64(num_sms) * 8)));
  residual_kernel<T><<<blocks, 256, 0, st>>>(X, sh, fs, weights, scratch);
  sum_pairs_kernel<<<1, 256, 0, st>>>(scratch, blocks, out2);
  count_launch(2);
  RCPG_LAUNCHED();
}

template <typename T>
void synth_tensor(const i64* shape, int order, int rank, const double* w_dev, const double* const* f_dev, double snr,
                  u64 noise_seed, T* out, double* scratch, int num_sms, cudaStream_t st) {
  const ShapeArg sh = make_shape(shape, order);
  DFactors fs{};
  for (int m = 0; m < order; ++m) fs.f[m] = f_dev[m];
  i64 total = 1;
  for (int m = 0; m < order; ++m) total *= shape[m];
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(total, 256), i64(num_sms) * 8)));
  synth_reconstruct_kernel<T><<<blocks, 256, 0, st>>>(sh, rank, w_dev, fs, out, total);
  count_launch();
  RCPG_LAUNCHED();
  if (!(snr > 0)) return;
  // add_noise (synthetic.hpp:42-58): sigma = sd / snr, sd the sample std.
  double h[2];
  sum_and_sq_kernel<T><<<blocks, 256, 0, st>>>(out, total, 0.0, scratch);
  sum_pairs_kernel<<<1, 256, 0, st>>>(scratch, blocks, scratch + 2 * blocks);
  RCPG_CUDA(cudaMemcpyAsync(h, scratch + 2 * blocks, sizeof(h), cudaMemcpyDeviceToHost, st));
  RCPG_CUDA(cudaStreamSynchronize(st));
  const double mean = h[0] / double(total);
  sum_and_sq_kernel<T><<<blocks, 256, 0, st>>>(out, total, mean, scratch);
  sum_pairs_kernel<<<1, 256, 0, st>>>(scratch, blocks, scratch + 2 * blocks);
  RCPG_CUDA(cudaMemcpyAsync(h, scratch + 2 * blocks, sizeof(h), cudaMemcpyDeviceToHost, st));
  RCPG_CUDA(cudaStreamSynchronize(st));
  const T sd = total > 1 ? T(sqrt(h[1] / double(total - 1))) : T(0);
  const T sigma = sd / T(snr);
  const u64 s0 = derive_seed(noise_seed, stream_id(kDomainNoise, 0));
  add_noise_kernel<T><<<blocks, 256, 0, st>>>(out, total, sigma, s0);
  count_launch(5);
  RCPG_LAUNCHED();
}

#define RCPG_INST(T)                                                                                          \
  template void kr_panel<T>(const FactorSet<T>&, const i64*, int, T*, cudaStream_t, const int*);                          \
  template void init_factors_from_grams<T>(const InitBatch<T>&, int, int, u64, int, cudaStream_t);           \
  template void zero_factor<T>(T*, i64, int, T*, cudaStream_t);                                               \
  template void fill_ones<T>(T*, int, cudaStream_t);                                               \
  template void als_update<T>(const FactorSet<T>&, int, const T*, T*, double, int, double*, double*,          \
                              AlsState*, double*, cudaStream_t);                                              \
  template void normalize_model<T>(const FactorSet<T>&, T*, T*, cudaStream_t);                                \
  template bool als_loop_supported<T>(const i64*, int, int);                                                  \
  template void als_loop<T>(const T*, const i64*, int, const FactorSet<T>&, T*, double, int, double*, double*, \
                            AlsState*, double*, i64, GridBarrier*, cudaStream_t, unsigned long long*);                                \
  template void small_gemm<T>(const T*, i64, i64, const T*, int, T*, cudaStream_t); \
  template void als_prepare<T>(AlsState*, double*, T*, i64, int, T*, T*, T, cudaStream_t); \
  template void small_gemm_batch<T>(const SmallGemmBatch<T>&, int, int, cudaStream_t);                           \
  template void norm_and_finite<T>(const T*, i64, double*, double*, int, cudaStream_t, const double*);       \
  template void nonfinite_flag<T>(const T*, i64, double*, cudaStream_t);                                      \
  template void residual_norms<T>(const T*, const i64*, int, const FactorSet<T>&, const T*, double*, double*, \
                                  int, cudaStream_t);                                                         \
  template void synth_tensor<T>(const i64*, int, int, const double*, const double* const*, double, u64, T*,   \
                                double*, int, cudaStream_t);
RCPG_INST(float)
RCPG_INST(double)
#undef RCPG_INST

}  // namespace rcpg
