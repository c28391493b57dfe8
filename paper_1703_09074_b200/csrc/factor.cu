// SPDX-License-Identifier: MIT
// Tall-skinny factorizations of the power-iteration chain (SURVEY.md §2.2
// K5/K6/K8), restating the reference's Eigen calls:
//   plu_basis  compress.hpp:47-58  = Eigen::FullPivLU (complete pivoting),
//                                   returns P^{-1} L
//   thin_qr    compress.hpp:60-73  = Eigen::HouseholderQR (LAPACK sign
//                                   convention) + householderQ() * I + rank warning
// Parity needs the reference's *basis*, not only its span,
// so both are faithful right-looking algorithms, not CholeskyQR / tournament
// pivoting. They run as one cooperative persistent kernel over the panel in
// its storage layout (rows s = a*R + b, column c at panel_addr(s, c)); every
// CTA owns a contiguous block of rows, keeps the row's Kolda (physical)
// position for the reference's column-major tie-breaking, and the
// grid-wide pivot / reduction steps use a generation barrier. With one CTA
// the barrier degenerates to __syncthreads (small I x l sample matrices).
#include "factor.cuh"
#include "runtime.cuh"

namespace rcpg {

namespace {

constexpr int kFacThreads = 256;

// ----------------------------------------------------------- row keys
__global__ void init_row_keys_kernel(KoldaMap km, i64 J, i64 R, i64* keys) {
  for (i64 s = blockIdx.x * i64(blockDim.x) + threadIdx.x; s < J; s += i64(gridDim.x) * blockDim.x) {
    const i64 a = s / R, b = s - a * R;
    keys[s] = kolda_index(km, a, b);
  }
}

// ---------------------------------------------------------------- LU
template <typename T>
struct Cand {
  T v;       // |value|; -1 = none
  int pcol;  // physical column (tie key 1)
  int c;     // storage column
  i64 prow;  // physical row (tie key 2)
  i64 s;     // storage row
};

template <typename T>
__device__ __forceinline__ bool better(const Cand<T>& a, const Cand<T>& b) {
  if (a.v != b.v) return a.v > b.v;
  if (a.pcol != b.pcol) return a.pcol < b.pcol;
  return a.prow < b.prow;
}

template <typename T>
__device__ Cand<T> shfl_cand(const Cand<T>& x, int off) {
  Cand<T> y;
  y.v = __shfl_xor_sync(0xffffffffu, x.v, off);
  y.pcol = __shfl_xor_sync(0xffffffffu, x.pcol, off);
  y.c = __shfl_xor_sync(0xffffffffu, x.c, off);
  y.prow = __shfl_xor_sync(0xffffffffu, x.prow, off);
  y.s = __shfl_xor_sync(0xffffffffu, x.s, off);
  return y;
}

// Block-wide arg-max with deterministic tie-breaking; result broadcast.
template <typename T>
__device__ Cand<T> block_best(Cand<T> x, Cand<T>* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand<T> y = shfl_cand(x, o);
    if (better(y, x)) x = y;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    Cand<T> y = lane < nw ? scratch[lane] : Cand<T>{T(-1), 0x7fffffff, 0, 0, 0};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Cand<T> z = shfl_cand(y, o);
      if (better(z, y)) y = z;
    }
    if (lane == 0) scratch[32] = y;
  }
  __syncthreads();
  Cand<T> r = scratch[32];
  __syncthreads();
  return r;
}

template <typename T>
struct LuArgs {
  T* A;        // panel J x n (in/out, destroyed)
  T* Z;        // output panel J x r = P^{-1} L
  i64 J, R;
  int n, r;
  i64* phys;   // [J] physical row position (init = Kolda index)
  KoldaMap km;
  Cand<T>* cands;  // [2][gridDim]
  GridBarrier* bar;
  int* info;   // [1] nonzero pivots
};

template <typename T>
__global__ void __launch_bounds__(kFacThreads) plu_kernel(LuArgs<T> p) {
  __shared__ Cand<T> red[33];
  __shared__ int pcol_of[kMaxPanelCols], col_at[kMaxPanelCols];
  __shared__ T U[kMaxPanelCols];
  __shared__ i64 ov_pos[kMaxPanelCols], ov_row[kMaxPanelCols];
  __shared__ int n_ov;
  __shared__ i64 s_u;

  const int G = gridDim.x;
  const i64 chunk = ceil_div(p.J, G);
  const i64 r0 = blockIdx.x * chunk;
  const i64 r1 = r0 + chunk < p.J ? r0 + chunk : p.J;
  const Cand<T> none{T(-1), 0x7fffffff, 0, 0x7fffffffffffffffll, 0};

  for (int c = threadIdx.x; c < p.n; c += blockDim.x) {
    pcol_of[c] = c;
    col_at[c] = c;
  }
  if (threadIdx.x == 0) n_ov = 0;

  // step-0 candidates
  Cand<T> best = none;
  for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
    const i64 ps = p.phys[s];
    for (int c = 0; c < p.n; ++c) {
      const Cand<T> x{T(fabs(p.A[panel_addr(s, c, p.R, p.n)])), c, c, ps, s};
      if (better(x, best)) best = x;
    }
  }
  best = block_best(best, red);
  if (threadIdx.x == 0) p.cands[blockIdx.x] = best;
  grid_sync(p.bar);

  int k0 = p.r;
  for (int k = 0; k < p.r; ++k) {
    const Cand<T>* cb = p.cands + (k & 1) * G;
    Cand<T> g = none;
    for (int q = threadIdx.x; q < G; q += blockDim.x) {
      Cand<T> x;
      x.v = ldcg(&cb[q].v);
      x.pcol = ldcg(&cb[q].pcol);
      x.c = ldcg(&cb[q].c);
      x.prow = ldcg(&cb[q].prow);
      x.s = ldcg(&cb[q].s);
      if (better(x, g)) g = x;
    }
    g = block_best(g, red);
    if (g.v == T(0) || g.v < T(0)) {  // exactly-zero corner (FullPivLU early stop)
      k0 = k;
      break;
    }
    const i64 ss = g.s;
    const int cs = g.c;
    const i64 pr = g.prow;
    const int pc = g.pcol;
    const T piv = ldcg(&p.A[panel_addr(ss, cs, p.R, p.n)]);
    if (threadIdx.x == 0) {
      // the row at physical position k before the swap
      i64 u = -1;
      for (int q = n_ov - 1; q >= 0; --q)
        if (ov_pos[q] == k) {
          u = ov_row[q];
          break;
        }
      if (u < 0) u = kolda_inverse(p.km, k, p.R);
      s_u = u;
      if (pr != k) {
        ov_pos[n_ov] = pr;
        ov_row[n_ov] = u;
        ++n_ov;
      }
      const int colk = col_at[k];
      pcol_of[cs] = k;
      pcol_of[colk] = pc;
      col_at[k] = cs;
      col_at[pc] = colk;
    }
    for (int c = threadIdx.x; c < p.n; c += blockDim.x) U[c] = ldcg(&p.A[panel_addr(ss, c, p.R, p.n)]);
    __syncthreads();
    const i64 u = s_u;
    // physical-position bookkeeping for rows this CTA owns
    if (threadIdx.x == 0) {
      if (ss >= r0 && ss < r1) p.phys[ss] = k;
      if (u != ss && u >= r0 && u < r1) p.phys[u] = pr;
    }
    __syncthreads();

    best = none;
    Cand<T>* out = p.cands + ((k + 1) & 1) * G;
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
      const i64 ps = p.phys[s];
      if (s == ss) {
        p.Z[panel_addr(s, k, p.R, p.r)] = T(1);
        for (int j = k + 1; j < p.r; ++j) p.Z[panel_addr(s, j, p.R, p.r)] = T(0);
        continue;
      }
      if (ps <= k) continue;  // pivoted earlier
      const T m = p.A[panel_addr(s, cs, p.R, p.n)] / piv;
      p.Z[panel_addr(s, k, p.R, p.r)] = m;
      if (k + 1 < p.r) {
        for (int q = k + 1; q < p.n; ++q) {
          const int c = col_at[q];
          const i64 ad = panel_addr(s, c, p.R, p.n);
          const T v = p.A[ad] - m * U[c];
          p.A[ad] = v;
          const Cand<T> x{T(fabs(v)), q, c, ps, s};
          if (better(x, best)) best = x;
        }
      }
    }
    if (k + 1 < p.r) {
      best = block_best(best, red);
      if (threadIdx.x == 0) out[blockIdx.x] = best;
      grid_sync(p.bar);
    }
  }

  if (k0 < p.r) {
    // Remaining L columns are unit vectors at the rows sitting at physical
    // positions k0..r-1 (the corner is exactly zero).
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
      const i64 ps = p.phys[s];
      if (ps < k0) continue;
      for (int j = k0; j < p.r; ++j) p.Z[panel_addr(s, j, p.R, p.r)] = (ps == j) ? T(1) : T(0);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.info = k0;
}

// ---------------------------------------------------------- Householder
template <typename T>
struct QrArgs {
  T* A;        // panel J x n (in/out: essential vectors below the diagonal)
  T* Q;        // output panel J x r
  i64 J, R;
  int n, r;
  const i64* krow;  // [J] Kolda row index
  KoldaMap km;
  double* part;     // [2][G][kMaxPanelCols + 1]
  T* tau;           // [r]
  T* diag;          // [r] R_kk = beta_k
  GridBarrier* bar;
  int* rank_warning;
};

template <typename T>
__global__ void __launch_bounds__(kFacThreads) householder_kernel(QrArgs<T> p) {
  __shared__ double red[33];
  __shared__ double tmp[kMaxPanelCols];
  const int G = gridDim.x;
  const i64 chunk = ceil_div(p.J, G);
  const i64 r0 = blockIdx.x * chunk;
  const i64 r1 = r0 + chunk < p.J ? r0 + chunk : p.J;
  constexpr int PW = kMaxPanelCols + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int phase = 0;

  for (int k = 0; k < p.r; ++k) {
    const i64 sk = kolda_inverse(p.km, k, p.R);
    const bool own_k = (sk >= r0 && sk < r1);
    // 1. tail squared norm of column k
    double acc = 0.0;
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x)
      if (p.krow[s] > k) {
        const double x = double(p.A[panel_addr(s, k, p.R, p.n)]);
        acc += x * x;
      }
    acc = block_sum(acc, red);
    double* pb = p.part + phase * G * PW;
    if (threadIdx.x == 0) pb[blockIdx.x * PW] = acc;
    grid_sync(p.bar);
    double tsq = 0.0;
    for (int q = 0; q < G; ++q) tsq += ldcg(&pb[q * PW]);
    phase ^= 1;
    const T tail_sq = T(tsq);
    const T c0 = ldcg(&p.A[panel_addr(sk, k, p.R, p.n)]);
    T beta, t;
    const bool trivial = !(tail_sq > Traits<T>::realmin);
    if (trivial) {
      t = T(0);
      beta = c0;
    } else {
      beta = sqrt(c0 * c0 + tail_sq);
      if (c0 >= T(0)) beta = -beta;
      t = (beta - c0) / beta;
    }
    const T denom = c0 - beta;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.tau[k] = t;
      p.diag[k] = beta;
    }
    // 2. essential vector (own tail rows) and partial v^T A(:, j)
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x)
      if (p.krow[s] > k) {
        const i64 ad = panel_addr(s, k, p.R, p.n);
        p.A[ad] = trivial ? T(0) : p.A[ad] / denom;
      }
    __syncthreads();
    const int ncol = p.n - k - 1;
    if (ncol <= 0) continue;
    if (trivial) continue;  // tau == 0: H_k = I
    pb = p.part + phase * G * PW;
    for (int jj = wid; jj < ncol; jj += nw) {  // warp per column
      const int j = k + 1 + jj;
      double a2 = 0.0;
      for (i64 s = r0 + lane; s < r1; s += 32)
        if (p.krow[s] > k)
          a2 += double(p.A[panel_addr(s, k, p.R, p.n)]) * double(p.A[panel_addr(s, j, p.R, p.n)]);
      a2 = warp_sum(a2);
      if (lane == 0) pb[blockIdx.x * PW + jj] = a2 + (own_k ? double(p.A[panel_addr(sk, j, p.R, p.n)]) : 0.0);
    }
    grid_sync(p.bar);
    for (int jj = threadIdx.x; jj < ncol; jj += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += ldcg(&pb[q * PW + jj]);
      tmp[jj] = s;
    }
    phase ^= 1;
    __syncthreads();
    // 3. rank-1 update of own rows
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
      const i64 kr = p.krow[s];
      if (kr > k) {
        const T e = p.A[panel_addr(s, k, p.R, p.n)];
        for (int jj = 0; jj < ncol; ++jj) {
          const i64 ad = panel_addr(s, k + 1 + jj, p.R, p.n);
          p.A[ad] -= t * e * T(tmp[jj]);
        }
      } else if (kr == k) {
        for (int jj = 0; jj < ncol; ++jj) {
          const i64 ad = panel_addr(s, k + 1 + jj, p.R, p.n);
          p.A[ad] -= t * T(tmp[jj]);
        }
      }
    }
  }
  // every tau/diag write (block 0) visible before the Q sweep
  grid_sync(p.bar);
  // rank warning (compress.hpp:64-71)
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.rank_warning) {
    T dmax = T(0), dmin = T(INFINITY);
    for (int k = 0; k < p.r; ++k) {
      const T d = fabs(ldcg(&p.diag[k]));
      dmax = d > dmax ? d : dmax;
      dmin = d < dmin ? d : dmin;
    }
    const T tol = T(p.J) * Traits<T>::eps * dmax;
    *p.rank_warning = (dmax == T(0)) || (dmin <= tol);
  }
  // Q = H_0 ... H_{r-1} I(J, r): start from the identity columns.
  for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
    const i64 kr = p.krow[s];
    for (int j = 0; j < p.r; ++j) p.Q[panel_addr(s, j, p.R, p.r)] = (kr == j) ? T(1) : T(0);
  }
  __syncthreads();  // rows are written thread-per-row, read warp-per-column below
  for (int k = p.r - 1; k >= 0; --k) {
    const T t = ldcg(&p.tau[k]);
    if (t == T(0)) continue;  // uniform across CTAs
    const i64 sk = kolda_inverse(p.km, k, p.R);
    const bool own_k = (sk >= r0 && sk < r1);
    const int ncol = p.r - k;  // columns j < k are untouched (exactly unchanged in Eigen too)
    double* pb = p.part + phase * G * PW;
    for (int jj = wid; jj < ncol; jj += nw) {  // warp per column
      const int j = k + jj;
      double a2 = 0.0;
      for (i64 s = r0 + lane; s < r1; s += 32)
        if (p.krow[s] > k)
          a2 += double(p.A[panel_addr(s, k, p.R, p.n)]) * double(p.Q[panel_addr(s, j, p.R, p.r)]);
      a2 = warp_sum(a2);
      if (lane == 0) pb[blockIdx.x * PW + jj] = a2 + (own_k ? double(p.Q[panel_addr(sk, j, p.R, p.r)]) : 0.0);
    }
    grid_sync(p.bar);
    for (int jj = threadIdx.x; jj < ncol; jj += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += ldcg(&pb[q * PW + jj]);
      tmp[jj] = s;
    }
    phase ^= 1;
    __syncthreads();
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
      const i64 kr = p.krow[s];
      if (kr > k) {
        const T e = p.A[panel_addr(s, k, p.R, p.n)];
        for (int jj = 0; jj < ncol; ++jj) p.Q[panel_addr(s, k + jj, p.R, p.r)] -= t * e * T(tmp[jj]);
      } else if (kr == k) {
        for (int jj = 0; jj < ncol; ++jj) p.Q[panel_addr(s, k + jj, p.R, p.r)] -= t * T(tmp[jj]);
      }
    }
    __syncthreads();
  }
}

int pick_grid(i64 J, int n, int maxc) {
  // ~8K panel entries per CTA; single CTA for the small I x l samples.
  const i64 want = ceil_div(J * n, 8192);
  return int(std::max<i64>(1, std::min<i64>(want, maxc)));
}

}  // namespace

void init_row_keys(const KoldaMap& km, i64 J, i64 R, i64* keys, cudaStream_t st) {
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(J, 256), 148 * 8)));
  init_row_keys_kernel<<<blocks, 256, 0, st>>>(km, J, R, keys);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
int plu_basis(T* A, T* Z, i64 J, i64 R, int n, const KoldaMap& km, FactorWork& w, cudaStream_t st) {
  check_arg(n <= kMaxPanelCols, "plu_basis: panel wider than supported");
  const int r = int(std::min<i64>(J, n));
  init_row_keys(km, J, R, w.keys, st);
  const int maxc = max_coop_blocks(plu_kernel<T>, kFacThreads, 0);
  const int G = pick_grid(J, n, maxc);
  LuArgs<T> a{A, Z, J, R, n, r, w.keys, km, reinterpret_cast<Cand<T>*>(w.cands), w.bar, w.info};
  launch_coop(plu_kernel<T>, G, kFacThreads, 0, st, a);
  return r;
}

template <typename T>
int thin_qr(T* A, T* Q, i64 J, i64 R, int n, const KoldaMap& km, FactorWork& w, int* rank_warning_dev,
            cudaStream_t st) {
  check_arg(n <= kMaxPanelCols, "thin_qr: panel wider than supported");
  const int r = int(std::min<i64>(J, n));
  init_row_keys(km, J, R, w.keys, st);
  const int maxc = max_coop_blocks(householder_kernel<T>, kFacThreads, 0);
  const int G = std::min(pick_grid(J, n, maxc), w.max_blocks);
  QrArgs<T> a{A, Q, J, R, n, r, w.keys, km, w.part, reinterpret_cast<T*>(w.tau), reinterpret_cast<T*>(w.diag),
              w.bar, rank_warning_dev};
  launch_coop(householder_kernel<T>, G, kFacThreads, 0, st, a);
  return r;
}

size_t factor_cand_bytes() { return sizeof(Cand<double>); }

template int plu_basis<float>(float*, float*, i64, i64, int, const KoldaMap&, FactorWork&, cudaStream_t);
template int plu_basis<double>(double*, double*, i64, i64, int, const KoldaMap&, FactorWork&, cudaStream_t);
template int thin_qr<float>(float*, float*, i64, i64, int, const KoldaMap&, FactorWork&, int*, cudaStream_t);
template int thin_qr<double>(double*, double*, i64, i64, int, const KoldaMap&, FactorWork&, int*, cudaStream_t);

}  // namespace rcpg
