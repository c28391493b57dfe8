// SPDX-License-Identifier: MIT
// Tall-skinny factorizations of the power-iteration chain (SURVEY.md §2.2
// K5/K6/K8), restating the reference's Eigen calls:
//   plu_basis  compress.hpp:47-58  = Eigen::FullPivLU (complete pivoting),
//                                   returns P^{-1} L
//   thin_qr    compress.hpp:60-73  = Eigen::HouseholderQR (LAPACK sign
//                                   convention) + householderQ() * I + rank warning
// Parity needs the reference's *basis*, not only its span.
//
// FullPivLU, by panel size (plu_basis picks the first that fits):
//  * plu_reg_kernel: rows in registers on one CTA or a cluster of up to 16,
//    integer-pipe pivot search (fp64 panels of <= 32 columns up to 12288 rows);
//  * plu_onchip_kernel: one CTA, rows owned by threads, swaps bookkept (the
//    I x l samples Y and small W);
//  * plu_cluster_kernel: one thread-block cluster of 8-16 CTAs, rows in DSMEM,
//    Eigen's physical row / column swaps (W up to ~3.5 MB);
//  * plu_resident_kernel: the panel resident in the SMs (one CTA per SM, smem +
//    register columns), one grid barrier per pivot (W up to ~40 MB);
//  * plu_coop_kernel: cooperative grid over an HBM/L2 panel, rows handed out in
//    chunks per step, delayed write-back (C3-C5's big W);
//  * plu_basis_dist: the row-sharded panel of the multi-GPU path.
// thin_qr: cqr2_* (CholeskyQR2 in double + the Householder sign
// reconstruction, fp64), householder_cluster_kernel / householder_kernel (the
// faithful Householder order: fp32, or when CholeskyQR2 declines).
#include <cooperative_groups.h>

#include <algorithm>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "factor.cuh"
#include "runtime.cuh"

namespace rcpg {

namespace {

constexpr int kFacThreads = 256;
constexpr int kSmallThreads = 1024;

// Storage offset of panel row s (column stride R): a*cols*R + b.
__device__ __forceinline__ i64 row_base(i64 s, i64 R, i64 J, i64 cols) {
  if (R == J) return s;  // first-mode panels and I x l samples: column-major
  const i64 a = s / R, b = s - a * R;
  return a * cols * R + b;
}

// ----------------------------------------------------------- row keys
__global__ void init_row_keys_kernel(KoldaMap km, i64 J, i64 R, i64* keys) {
  for (i64 s = blockIdx.x * i64(blockDim.x) + threadIdx.x; s < J; s += i64(gridDim.x) * blockDim.x) {
    const i64 a = s / R, b = s - a * R;
    keys[s] = kolda_index(km, a, b);
  }
}

// ------------------------------------------------------------ candidates
template <typename T>
struct __align__(16) Cand {
  T v;       // |value|; -1 = none
  int pcol;  // physical column (tie key 1)
  int c;     // storage column
  i64 prow;  // physical row (tie key 2)
  i64 s;     // storage row
};

template <typename T>
__device__ __forceinline__ Cand<T> load_cand_cg(const Cand<T>* p) {
  static_assert(sizeof(Cand<T>) == 32 || sizeof(Cand<T>) == 24, "candidate layout");
  Cand<T> x;
  if constexpr (sizeof(Cand<T>) == 32) {
    const int4 a = __ldcg(reinterpret_cast<const int4*>(p));
    const int4 b = __ldcg(reinterpret_cast<const int4*>(p) + 1);
    *reinterpret_cast<int4*>(&x) = a;
    *(reinterpret_cast<int4*>(&x) + 1) = b;
  } else {
    x.v = __ldcg(&p->v);
    x.pcol = __ldcg(&p->pcol);
    x.c = __ldcg(&p->c);
    x.prow = __ldcg(&p->prow);
    x.s = __ldcg(&p->s);
  }
  return x;
}

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
    Cand<T> y = lane < nw ? scratch[lane] : Cand<T>{T(-1), 0x7fffffff, 0, 0x7fffffffffffffffll, 0};
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

// ------------------------------------------------ LU, shared-memory CTA
// Eigen FullPivLU verbatim on an I x n column-major panel held in shared
// memory (physical row/column swaps, first maximum in column-major order).
// The pivot key is (|a|, column-major index) so one 64-bit value and one
// 32-bit index move per shuffle.
constexpr int kSmemLuThreads = 256;  // 512 from 128 rows per CTA (plu_basis)

template <typename T>
__device__ __forceinline__ void key_better(T& v, int& idx, T ov, int oidx) {
  if (ov > v || (ov == v && oidx < idx)) {
    v = ov;
    idx = oidx;
  }
}

template <typename T>
__device__ void block_argmax(T& v, int& idx, T* sv, int* si) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) key_better(v, idx, __shfl_xor_sync(0xffffffffu, v, o), __shfl_xor_sync(0xffffffffu, idx, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) {
    sv[wid] = v;
    si[wid] = idx;
  }
  __syncthreads();
  v = lane < nw ? sv[lane] : T(-1);
  idx = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) key_better(v, idx, __shfl_xor_sync(0xffffffffu, v, o), __shfl_xor_sync(0xffffffffu, idx, o));
  __syncthreads();
}

// FullPivLU on a panel held in the distributed shared memory of one thread-
// block cluster (CS = 1..16 CTAs; CS = 1 is a plain shared-memory kernel).
// Rows are kept in physical (Kolda) order -- physical row p is storage row
// kolda_inverse(p) of the (L, n, R) panel -- and CTA r of the cluster owns
// physical rows [r*chunk, (r+1)*chunk). Row swaps move rows between CTAs
// through DSMEM, column swaps are local, so the elimination is Eigen's,
// operation for operation. Two cluster barriers per pivot.
template <typename T, bool CLUSTER, int NT = kSmemLuThreads>
__global__ void __launch_bounds__(NT) plu_cluster_kernel(const T* __restrict__ A, T* __restrict__ Z,
                                                                     int J, int n, int chunk, i64 R, KoldaMap km,
                                                                     int* info) {
  namespace cg = cooperative_groups;
  const int CS = CLUSTER ? int(cg::this_cluster().num_blocks()) : 1;
  const int me = CLUSTER ? int(cg::this_cluster().block_rank()) : 0;
  auto csync = [&]() {
    if constexpr (CLUSTER)
      cg::this_cluster().sync();
    else
      __syncthreads();
  };
  auto remote = [&](auto* ptr, int rank) {
    if constexpr (CLUSTER)
      return cg::this_cluster().map_shared_rank(ptr, rank);
    else
      return ptr;
  };
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* a = reinterpret_cast<T*>(smem_raw);                       // [n][chunk] local rows, column-major
  T* U = a + i64(chunk) * n;                                    // [n] pivot row (old row br)
  T* Tk = U + n;                                                // [n] old row k
  int* perm = reinterpret_cast<int*>(Tk + n);                   // [chunk] original physical index
  __shared__ T cand_v;
  __shared__ int cand_i;
  __shared__ T sv[32];
  __shared__ int si[32];
  __shared__ int s_meta[4];  // perm_br, perm_k
  const int tid = threadIdx.x, nt = blockDim.x;
  const int r = J < n ? J : n;
  const int p0 = me * chunk;
  const int p1 = min(J, p0 + chunk);
  const int rows = p1 > p0 ? p1 - p0 : 0;
  const bool ident = (R == i64(J)) && km.n_low == 0 && km.n_high == 1;
  // load own rows (physical order)
  for (int lp = tid; lp < rows; lp += nt) {
    const int p = p0 + lp;
    perm[lp] = p;
    i64 base;
    if (ident) {
      base = p;
    } else {
      const i64 srow = kolda_inverse(km, p, R);
      const i64 aa = srow / R, bb = srow - aa * R;
      base = aa * n * R + bb;
    }
    for (int j = 0; j < n; ++j) a[lp + j * chunk] = A[base + j * R];
  }
  __syncthreads();
  const int tx = tid & 31, ty = tid >> 5, ny = nt >> 5;
  T bv = T(-1);
  int bi = 0x7fffffff;
  for (int j = ty; j < n; j += ny)
    for (int lp = tx; lp < rows; lp += 32) key_better(bv, bi, T(fabs(a[lp + j * chunk])), j * J + p0 + lp);
  int k0 = r;
  for (int k = 0; k < r; ++k) {
    block_argmax(bv, bi, sv, si);
    if (tid == 0) {
      cand_v = bv;
      cand_i = bi;
    }
    csync();  // B1: candidates published
    if (tid < 32) {  // reduce the cluster's candidates (same order in every CTA)
      T v = T(-1);
      int idx = 0x7fffffff;
      if (tid < CS) {
        v = *remote(&cand_v, tid);
        idx = *remote(&cand_i, tid);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        key_better(v, idx, __shfl_xor_sync(0xffffffffu, v, o), __shfl_xor_sync(0xffffffffu, idx, o));
      if (tid == 0) {
        sv[0] = v;
        si[0] = idx;
      }
    }
    __syncthreads();
    const T gv = sv[0];
    const int gi = si[0];
    if (!(gv > T(0))) {
      k0 = k;
      break;  // uniform across the cluster
    }
    const int br = gi % J, bc = gi / J;
    const int ok_ = k / chunk, obr = br / chunk;
    // old row br -> U (every CTA); old row k -> Tk (owner of br, when swapping)
    {
      const T* rb = remote(a, obr);
      for (int j = tid; j < n; j += nt) U[j] = rb[(br - obr * chunk) + j * chunk];
      if (tid == 0) s_meta[0] = *remote(perm + (br - obr * chunk), obr);
      if (br != k && me == obr) {
        const T* rk = remote(a, ok_);
        for (int j = tid; j < n; j += nt) Tk[j] = rk[(k - ok_ * chunk) + j * chunk];
        if (tid == 0) s_meta[1] = *remote(perm + (k - ok_ * chunk), ok_);
      }
    }
    csync();  // B2: every remote read done before rows are overwritten
    if (br != k) {
      if (me == ok_) {
        for (int j = tid; j < n; j += nt) a[(k - p0) + j * chunk] = U[j];
        if (tid == 0) perm[k - p0] = s_meta[0];
      }
      if (me == obr) {
        for (int j = tid; j < n; j += nt) a[(br - p0) + j * chunk] = Tk[j];
        if (tid == 0) perm[br - p0] = s_meta[1];
      }
    }
    __syncthreads();
    if (bc != k) {  // column swap in the local rows and in U
      for (int lp = tid; lp < rows; lp += nt) {
        const T t = a[lp + k * chunk];
        a[lp + k * chunk] = a[lp + bc * chunk];
        a[lp + bc * chunk] = t;
      }
      if (tid == 0) {
        const T t = U[k];
        U[k] = U[bc];
        U[bc] = t;
      }
    }
    __syncthreads();
    const T piv = U[k];
    // multipliers (col k below the diagonal), then the rank-1 update fused with
    // the next pivot search
    const int lo = max(k + 1, p0) - p0;
    for (int lp = lo + tid; lp < rows; lp += nt) a[lp + k * chunk] = a[lp + k * chunk] / piv;
    __syncthreads();
    bv = T(-1);
    bi = 0x7fffffff;
    if (k < r - 1) {
      for (int j = k + 1 + ty; j < n; j += ny) {
        const T u = U[j];
        for (int lp = lo + tx; lp < rows; lp += 32) {
          const T x = sub_mul_rn(a[lp + j * chunk], a[lp + k * chunk], u);
          a[lp + j * chunk] = x;
          key_better(bv, bi, T(fabs(x)), j * J + p0 + lp);
        }
      }
    }
    __syncthreads();
  }
  // P^{-1} L: physical row p of L goes to original row perm[p]
  for (int lp = tid; lp < rows; lp += nt) {
    const int p = p0 + lp;
    i64 base;
    if (ident) {
      base = perm[lp];
    } else {
      const i64 srow = kolda_inverse(km, perm[lp], R);
      const i64 aa = srow / R, bb = srow - aa * R;
      base = aa * r * R + bb;
    }
    for (int j = 0; j < r; ++j) Z[base + j * R] = (p == j) ? T(1) : (p > j ? a[lp + j * chunk] : T(0));
  }
  if (me == 0 && tid == 0) *info = k0;
  csync();  // keep every CTA's shared memory alive until all remote reads are done
}

// FullPivLU of a panel that fits one CTA's shared memory, without moving data:
// slot i holds the row at Kolda (physical) index i, column-major, each thread
// owning whole rows. Row and column swaps are bookkept (phys/rowat,
// col_at/pcol_of) and the pivot key is (|a|, physical column, physical row) --
// the same pick as Eigen's first maximum in column-major order on the swapped
// matrix (see plu_coop_kernel). The multiplier of row i at step k overwrites
// its entry in the pivot column, the rank-1 update is fused with the next
// pivot search: four block barriers per pivot.
template <typename T>
__global__ void __launch_bounds__(1024) plu_onchip_kernel(const T* __restrict__ A, T* __restrict__ Z, int J, int n,
                                                          i64 R, KoldaMap km, int W, int* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* a = reinterpret_cast<T*>(smem_raw);                   // [n][J]
  // [J] physical row of slot i; 8-byte aligned: it first holds one i64 per row (rbase below)
  int* phys = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(a + i64(J) * n) + 7) & ~uintptr_t(7));
  int* rowat = phys + J;                                   // [J] slot at physical row p
  __shared__ int col_at[kMaxPanelCols];                    // storage column at physical column q
  __shared__ T red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_ss, s_cs, s_stop;
  const int tid = threadIdx.x, nt = blockDim.x;
  // W row lanes x tpr column groups: thread (g, i0) updates rows i0, i0 + W, ...
  // in physical columns k+1+g, k+1+g+tpr, ... (tpr > 1 only when W >= J)
  const int tpr = nt / W, g = tid / W, i0 = tid - g * W;
  const int r = J < n ? J : n;
  const bool ident = (R == i64(J)) && km.n_low == 0 && km.n_high == 1;
  for (int c = tid; c < n; c += nt) col_at[c] = c;
  // panel load, coalesced along columns with many loads in flight per thread;
  // Kolda row bases go through the phys/rowat area (one i64 per row) first
  i64* rbase = reinterpret_cast<i64*>(phys);
  if (!ident) {
    for (int i = tid; i < J; i += nt) {
      const i64 srow = kolda_inverse(km, i, R);
      const i64 aa = srow / R, bb = srow - aa * R;
      rbase[i] = aa * n * R + bb;
    }
    __syncthreads();
  }
  for (int i = tid; i < J; i += nt) {
    const i64 base = ident ? i64(i) : rbase[i];
    int c = 0;
    for (; c + 8 <= n; c += 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = A[base + (c + u) * R];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[i + i64(c + u) * J] = v[u];
    }
    for (; c < n; ++c) a[i + i64(c) * J] = A[base + c * R];
  }
  __syncthreads();
  for (int i = tid; i < J; i += nt) {
    phys[i] = i;
    rowat[i] = i;
  }
  __syncthreads();
  // candidate key: (|a| desc, physical column asc, physical row asc) with the
  // two positions packed as pcol * J + prow (< 2^31 for on-chip panels)
  T bv = T(-1);
  int bi = 0x7fffffff;
  for (int i = i0; i < J; i += W)
    for (int c = g; c < n; c += tpr) key_better(bv, bi, T(fabs(a[i + i64(c) * J])), c * J + i);
  int k0 = r;
  T m_pend = T(0);  // tpr > 1: the multiplier of the previous step, stored one step late
  int c_pend = -1;
  for (int k = 0; k < r; ++k) {
    // one block reduction; warp 0 finishes it and does the bookkeeping
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      key_better(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
    if ((tid & 31) == 0) {
      red_v[tid >> 5] = bv;
      red_i[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid < 32) {
      bv = tid < (nt >> 5) ? red_v[tid] : T(-1);
      bi = tid < (nt >> 5) ? red_i[tid] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        key_better(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
      if (tid == 0) {
        s_stop = !(bv > T(0));
        if (bv > T(0)) {
          const int pc = bi / J, pr = bi - pc * J;
          const int ss = rowat[pr], cs = col_at[pc];
          const int u = rowat[k];  // slot at physical row k moves to the pivot's physical row
          phys[ss] = k;
          rowat[k] = ss;
          phys[u] = pr;
          rowat[pr] = u;
          col_at[pc] = col_at[k];
          col_at[k] = cs;
          s_ss = ss;
          s_cs = cs;
        }
      }
    }
    __syncthreads();
    if (c_pend >= 0) {  // every sibling has read it (two barriers ago)
      a[i0 + i64(c_pend) * J] = m_pend;
      c_pend = -1;
    }
    if (s_stop) {  // exactly-zero corner (FullPivLU early stop)
      k0 = k;
      break;
    }
    // the pivot row is read in place (broadcast): nobody writes it this step
    const int ss = s_ss, cs = s_cs;
    const T* __restrict__ up = a + ss;
    const T piv = up[i64(cs) * J];
    bv = T(-1);
    bi = 0x7fffffff;
    const bool more = k + 1 < r;
    for (int i = i0; i < J; i += W) {
      const int ps = phys[i];
      if (ps <= k) continue;  // pivoted (the pivot row itself has ps == k)
      const T m = a[i + i64(cs) * J] / piv;
      if (tpr == 1) {
        a[i + i64(cs) * J] = m;
      } else if (g == 0) {
        m_pend = m;
        c_pend = cs;
      }
      if (!more) continue;
      T rv = T(-1);
      int rq = 0;
      // 32-bit offsets from per-row / pivot-row base pointers (J * n < 2^31 on
      // this path): no 64-bit address arithmetic per entry
      T* __restrict__ ai = a + i;
#pragma unroll 4
      for (int q = k + 1 + g; q < n; q += tpr) {
        const int co = col_at[q] * J;
        const T x = sub_mul_rn(ai[co], m, up[co]);
        ai[co] = x;
        if (fabs(x) > rv) {
          rv = fabs(x);
          rq = q;
        }
      }
      key_better(bv, bi, rv, rq * J + ps);
    }
  }
  __syncthreads();
  if (c_pend >= 0) a[i0 + i64(c_pend) * J] = m_pend;
  __syncthreads();
  // P^{-1} L: slot i (Kolda row i) at physical row p: multipliers left of p
  // (columns before an early stop), its unit entry at p, zeros right of it
  for (int i = tid; i < J; i += nt) {
    const int p = phys[i];
    i64 base = i;
    if (!ident) {
      const i64 srow = kolda_inverse(km, i, R);
      const i64 aa = srow / R, bb = srow - aa * R;
      base = aa * r * R + bb;
    }
    for (int j = 0; j < r; ++j)
      Z[base + j * R] = (p == j) ? T(1) : (j < p && j < k0 ? a[i + i64(col_at[j]) * J] : T(0));
  }
  if (tid == 0) *info = k0;
}

// FullPivLU with the panel in registers: thread t of CTA q (of a cluster of CS
// CTAs) owns Kolda rows (q*RPT + j)*NT + t, j < RPT, as NC register columns in
// storage order. Columns are bookkept (col_at / pcol_of in shared memory, every
// CTA an identical copy), rows too (phys per row in a register): no data moves
// per pivot. The multiplier of step k is stored straight to Z (column k of
// P^{-1} L), so a column that has been eliminated, and a row that has been
// pivoted, no longer holds anything that is read: the rank-1 update runs over
// all NC columns of every row without a branch or a select, and the candidate
// search masks eliminated columns out.
//
// Candidate search on the integer pipe: for |y| >= 0 the IEEE bit pattern is
// monotone, so each row keeps the max of (high word of |y|) & mask[c] (two ALU
// ops per entry, no fp64 compares); a warp reduces those with redux.sync, and
// only the row(s) that reach the warp's maximum are resolved exactly -- staged
// in shared memory, one column per lane: the low word, then the physical
// column among equal values (Eigen's first maximum in column-major order),
// then the physical row. One barrier (a cluster barrier on a cluster), warp 0
// picks the winner among all warps (DSMEM) and stages (u, mask) per column,
// one block barrier, then the multipliers (the pivot column found by a switch:
// register arrays take compile-time indices only) and the update. Same picks,
// same operations, same bits as plu_onchip_kernel / Eigen (x - m*u rounded
// twice, m = x / pivot). Requires finite panels (compress checks its input).
template <typename T>
struct __align__(16) LuUpk {
  T u;            // pivot row entry (storage column c)
  unsigned mask;  // 0x7fffffff while column c is not eliminated, else 0
  int pcol;       // physical column of storage column c after this pivot's swap
};

template <typename T, int NC, int RPT>
constexpr int lu_reg_max_threads() {
  // registers: the rows plus ~40 for the rest; at most 1024 threads
  constexpr int need = NC * RPT * int(sizeof(T)) / 4 + 40;
  constexpr int t = (65536 / need) / 32 * 32;
  return t > 1024 ? 1024 : t;
}

// high word of |y| (the whole pattern for float) and the low word (0 for float)
template <typename T>
__device__ __forceinline__ unsigned lu_hi(T y) {
  if constexpr (sizeof(T) == 8)
    return unsigned(__double2hiint(y));
  else
    return __float_as_uint(y);
}
template <typename T>
__device__ __forceinline__ unsigned lu_lo(T y) {
  if constexpr (sizeof(T) == 8)
    return unsigned(__double2loint(y));
  else
    return 0u;
}

#ifdef RCPG_LU_REG_PROF
__device__ unsigned long long g_lu_reg_prof[8];
#define LU_REG_STAMP(i)                  \
  do {                                   \
    if (tid == 0 && me == 0) {           \
      const long long t_ = clock64();    \
      prof_acc[i] += t_ - prof_t;        \
      prof_t = t_;                       \
    }                                    \
  } while (0)
#else
#define LU_REG_STAMP(i) \
  do {                  \
  } while (0)
#endif

#define RCPG_LU_CASE(C)                                 \
  case C:                                               \
    if constexpr (C < NC) {                             \
      _Pragma("unroll") for (int j = 0; j < RPT; ++j) { \
        m[j] = x[j][C] / piv;                           \
      }                                                 \
    }                                                   \
    break;

template <typename T, int NC, int RPT, bool CL>
__global__ void __launch_bounds__(lu_reg_max_threads<T, NC, RPT>(), 1)
    plu_reg_kernel(const T* __restrict__ A, T* __restrict__ Z, int J, int n, i64 R, KoldaMap km, int* info) {
  namespace cg = cooperative_groups;
  constexpr int kMaxW = lu_reg_max_threads<T, NC, RPT>() / 32;
  constexpr int kCPL = (NC + 31) / 32;  // columns per lane in the exact resolution
  __shared__ T wrow[2][kMaxW][NC];      // each warp's best row, by pivot parity
  __shared__ T wtmp[kMaxW][NC];         // a tied row being resolved
  __shared__ unsigned wkh[2][kMaxW], wkl[2][kMaxW];
  __shared__ int wki[2][kMaxW];
  __shared__ LuUpk<T> upk[NC];
  __shared__ int col_at[NC], pcol_of[NC];
  __shared__ T s_piv;
  __shared__ int s_pr, s_cs, s_stop;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5, NW = NT >> 5;
  const int me = CL ? int(cg::this_cluster().block_rank()) : 0;
  const int CS = CL ? int(cg::this_cluster().num_blocks()) : 1;
  const int r = J < n ? J : n;
  const bool ident = (R == i64(J)) && km.n_low == 0 && km.n_high == 1;
  for (int c = tid; c < NC; c += NT) {
    col_at[c] = c;
    pcol_of[c] = c;
    upk[c].mask = c < n ? 0x7fffffffu : 0u;
    upk[c].pcol = c;
  }
  T x[RPT][NC];
  int ph[RPT];    // physical row (-1: padding)
  i64 ob[RPT];    // Z offset of the row
  unsigned mh[RPT];  // max over live columns of the high word of |x|
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int slot = (me * RPT + j) * NT + tid;
    ph[j] = slot < J ? slot : -1;
    i64 base = slot;
    ob[j] = slot;
    if (!ident && slot < J) {
      const i64 srow = kolda_inverse(km, slot, R);
      const i64 aa = srow / R, bb = srow - aa * R;
      base = aa * n * R + bb;
      ob[j] = aa * r * R + bb;
    }
    mh[j] = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      x[j][c] = (slot < J && c < n) ? A[base + c * R] : T(0);
      mh[j] = max(mh[j], lu_hi(x[j][c]) & 0x7fffffffu);
    }
  }
  __syncthreads();
  int k0 = r;
#ifdef RCPG_LU_REG_PROF
  long long prof_t = clock64(), prof_acc[6] = {0, 0, 0, 0, 0, 0};
#endif
  for (int k = 0; k < r; ++k) {
    const int par = k & 1;
    LU_REG_STAMP(0);
    // ---- warp: the rows at the warp's largest high word, resolved exactly
    unsigned mt = 0;
#pragma unroll
    for (int j = 0; j < RPT; ++j)
      if (ph[j] >= k) mt = max(mt, mh[j]);  // live rows (phys >= k before this pivot)
    const unsigned hmax = __reduce_max_sync(0xffffffffu, mt);
    unsigned wl = 0;
    int wi = 0x7fffffff;
    {  // (hmax == 0 with live rows: a zero or subnormal corner; every live row is resolved)
      unsigned pend = 0;  // my rows at hmax
#pragma unroll
      for (int j = 0; j < RPT; ++j)
        if (ph[j] >= k && mh[j] == hmax) pend |= 1u << j;
      bool first = true;
      for (unsigned bal = __ballot_sync(0xffffffffu, pend != 0); bal; bal = __ballot_sync(0xffffffffu, pend != 0)) {
        const int src = __ffs(bal) - 1;
        T* dst = first ? &wrow[par][wid][0] : &wtmp[wid][0];
        int prow = 0;
        if (lane == src) {
          const int j = __ffs(pend) - 1;
          pend &= pend - 1;
#pragma unroll
          for (int jj = 0; jj < RPT; ++jj)
            if (jj == j) {
              prow = ph[jj];
#pragma unroll
              for (int c = 0; c < NC; ++c) dst[c] = x[jj][c];
            }
        }
        prow = __shfl_sync(0xffffffffu, prow, src);
        __syncwarp();
        unsigned l = 0;
        int pc = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < kCPL; ++q) {
          const int c = lane + 32 * q;
          if (c < NC) {
            const T v = dst[c];
            const LuUpk<T>& e = upk[c];
            if ((lu_hi(v) & e.mask) == hmax) {
              const unsigned lo = lu_lo(v);
              if (lo > l || (lo == l && e.pcol < pc)) {
                l = lo;
                pc = e.pcol;
              }
            }
          }
        }
        const unsigned L = __reduce_max_sync(0xffffffffu, l);
        const int P = int(__reduce_min_sync(0xffffffffu, unsigned(l == L ? pc : 0x7fffffff)));
        const int I = (P << 16) | prow;
        if (first || L > wl || (L == wl && I < wi)) {
          if (!first) {  // a better tie: it becomes the staged row
#pragma unroll
            for (int q = 0; q < kCPL; ++q) {
              const int c = lane + 32 * q;
              if (c < NC) wrow[par][wid][c] = wtmp[wid][c];
            }
          }
          wl = L;
          wi = I;
        }
        first = false;
        __syncwarp();
      }
    }
    if (lane == 0) {
      wkh[par][wid] = hmax;
      wkl[par][wid] = wl;
      wki[par][wid] = wi;
    }
    LU_REG_STAMP(1);
    if constexpr (CL)
      cg::this_cluster().sync();
    else
      __syncthreads();
    LU_REG_STAMP(2);
    // ---- warp 0: the winner over the cluster's warps, bookkeeping, staging
    if (wid == 0) {
      unsigned gh = 0, gl = 0;
      int gi = 0x7fffffff, ge = 0;
      for (int e = lane; e < CS * NW; e += 32) {
        const int q = e / NW, w = e - q * NW;
        unsigned oh, ol;
        int oi;
        if constexpr (CL) {
          oh = *cg::this_cluster().map_shared_rank(&wkh[par][w], q);
          ol = *cg::this_cluster().map_shared_rank(&wkl[par][w], q);
          oi = *cg::this_cluster().map_shared_rank(&wki[par][w], q);
        } else {
          oh = wkh[par][w];
          ol = wkl[par][w];
          oi = wki[par][w];
        }
        if (oh > gh || (oh == gh && (ol > gl || (ol == gl && oi < gi)))) {
          gh = oh;
          gl = ol;
          gi = oi;
          ge = e;
        }
      }
      const unsigned H = __reduce_max_sync(0xffffffffu, gh);
      const unsigned Lw = __reduce_max_sync(0xffffffffu, gh == H ? gl : 0u);
      const int I = int(__reduce_min_sync(0xffffffffu, unsigned(gh == H && gl == Lw ? gi : 0x7fffffff)));
      const unsigned who = __ballot_sync(0xffffffffu, gh == H && gl == Lw && gi == I);
      const int E = __shfl_sync(0xffffffffu, ge, __ffs(who) - 1);
      const bool stop = H == 0 && Lw == 0;  // the largest remaining |a| is 0
      if (lane == 0) {
        s_stop = stop;
        if (!stop) {
          const int pc = I >> 16, pr = I & 0xffff;
          const int cs = col_at[pc], ck = col_at[k];
          col_at[pc] = ck;
          col_at[k] = cs;
          pcol_of[cs] = k;
          pcol_of[ck] = pc;
          s_pr = pr;
          s_cs = cs;
        }
      }
      __syncwarp();
      if (!stop) {
        const int q = E / NW, w = E - q * NW;
        const T* src = &wrow[par][w][0];
        if constexpr (CL) src = cg::this_cluster().map_shared_rank(src, q);
        const int cs = s_cs;
        for (int c = lane; c < NC; c += 32) {
          const T u = src[c];
          upk[c].u = u;
          upk[c].pcol = pcol_of[c];
          if (c == cs) {
            upk[c].mask = 0u;
            s_piv = u;
          }
        }
      }
    }
    LU_REG_STAMP(3);
    __syncthreads();
    LU_REG_STAMP(4);
    if (s_stop) {
      k0 = k;
      break;
    }
    const int pr = s_pr, cs = s_cs;
    const T piv = s_piv;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int p = ph[j];
      ph[j] = p == pr ? k : (p == k ? pr : p);
    }
    T m[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) m[j] = T(0);
    switch (cs) {
      RCPG_LU_CASE(0)
      RCPG_LU_CASE(1)
      RCPG_LU_CASE(2)
      RCPG_LU_CASE(3)
      RCPG_LU_CASE(4)
      RCPG_LU_CASE(5)
      RCPG_LU_CASE(6)
      RCPG_LU_CASE(7)
      RCPG_LU_CASE(8)
      RCPG_LU_CASE(9)
      RCPG_LU_CASE(10)
      RCPG_LU_CASE(11)
      RCPG_LU_CASE(12)
      RCPG_LU_CASE(13)
      RCPG_LU_CASE(14)
      RCPG_LU_CASE(15)
      RCPG_LU_CASE(16)
      RCPG_LU_CASE(17)
      RCPG_LU_CASE(18)
      RCPG_LU_CASE(19)
      RCPG_LU_CASE(20)
      RCPG_LU_CASE(21)
      RCPG_LU_CASE(22)
      RCPG_LU_CASE(23)
      RCPG_LU_CASE(24)
      RCPG_LU_CASE(25)
      RCPG_LU_CASE(26)
      RCPG_LU_CASE(27)
      RCPG_LU_CASE(28)
      RCPG_LU_CASE(29)
      RCPG_LU_CASE(30)
      RCPG_LU_CASE(31)
      RCPG_LU_CASE(32)
      RCPG_LU_CASE(33)
      RCPG_LU_CASE(34)
      RCPG_LU_CASE(35)
      RCPG_LU_CASE(36)
      RCPG_LU_CASE(37)
      RCPG_LU_CASE(38)
      RCPG_LU_CASE(39)
      RCPG_LU_CASE(40)
      RCPG_LU_CASE(41)
      RCPG_LU_CASE(42)
      RCPG_LU_CASE(43)
      RCPG_LU_CASE(44)
      RCPG_LU_CASE(45)
      RCPG_LU_CASE(46)
      RCPG_LU_CASE(47)
      RCPG_LU_CASE(48)
      RCPG_LU_CASE(49)
      RCPG_LU_CASE(50)
      RCPG_LU_CASE(51)
      RCPG_LU_CASE(52)
      RCPG_LU_CASE(53)
      RCPG_LU_CASE(54)
      RCPG_LU_CASE(55)
      RCPG_LU_CASE(56)
      RCPG_LU_CASE(57)
      RCPG_LU_CASE(58)
      RCPG_LU_CASE(59)
      RCPG_LU_CASE(60)
      RCPG_LU_CASE(61)
      RCPG_LU_CASE(62)
      RCPG_LU_CASE(63)
      RCPG_LU_CASE(64)
      RCPG_LU_CASE(65)
      RCPG_LU_CASE(66)
      RCPG_LU_CASE(67)
      RCPG_LU_CASE(68)
      RCPG_LU_CASE(69)
      RCPG_LU_CASE(70)
      RCPG_LU_CASE(71)
      RCPG_LU_CASE(72)
      RCPG_LU_CASE(73)
      RCPG_LU_CASE(74)
      RCPG_LU_CASE(75)
      RCPG_LU_CASE(76)
      RCPG_LU_CASE(77)
      RCPG_LU_CASE(78)
      RCPG_LU_CASE(79)
      RCPG_LU_CASE(80)
      RCPG_LU_CASE(81)
      RCPG_LU_CASE(82)
      RCPG_LU_CASE(83)
      RCPG_LU_CASE(84)
      RCPG_LU_CASE(85)
      RCPG_LU_CASE(86)
      RCPG_LU_CASE(87)
      RCPG_LU_CASE(88)
      RCPG_LU_CASE(89)
      RCPG_LU_CASE(90)
      RCPG_LU_CASE(91)
      RCPG_LU_CASE(92)
      RCPG_LU_CASE(93)
      RCPG_LU_CASE(94)
      RCPG_LU_CASE(95)
      default:
        break;
    }
#pragma unroll
    for (int j = 0; j < RPT; ++j)
      if (ph[j] > k) Z[ob[j] + i64(k) * R] = m[j];  // column k of P^{-1} L
    LU_REG_STAMP(5);
    if (k + 1 < r) {
#pragma unroll
      for (int j = 0; j < RPT; ++j) mh[j] = 0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const LuUpk<T> e = upk[c];
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          const T y = sub_mul_rn(x[j][c], m[j], e.u);
          x[j][c] = y;
          mh[j] = max(mh[j], lu_hi(y) & e.mask);
        }
      }
    }
  }
#ifdef RCPG_LU_REG_PROF
  if (tid == 0 && me == 0) {
    for (int i = 0; i < 6; ++i) g_lu_reg_prof[i] = prof_acc[i];
    g_lu_reg_prof[6] = k0;
  }
#endif
  // the rest of P^{-1} L: the unit entry at p, zeros right of it (and from an
  // early stop on); the multipliers left of min(p, k0) were stored per step
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int p = ph[j];
    if (p < 0) continue;
    for (int jj = min(p, k0); jj < r; ++jj) Z[ob[j] + i64(jj) * R] = jj == p ? T(1) : T(0);
  }
  if (me == 0 && tid == 0) *info = k0;
  if constexpr (CL) cg::this_cluster().sync();  // remote readers done before exit
}
#undef RCPG_LU_CASE

// -------------------------------------------------- LU, cooperative grid
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
  unsigned long long* prof;  // optional [8]: ns in reduce / bookkeeping / update / barrier (CTA 0)
  int delay;   // 1: store the panel after odd pivots only (see plu_coop_kernel)
  unsigned* ctr;  // [n] per-step chunk counters (zeroed before the launch)
  int chunk_groups;  // row groups (blockDim * V rows) per dynamically scheduled chunk; 0 = static split
};

__device__ __forceinline__ unsigned long long lu_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kLuThreads = 256;
// minimum CTAs per SM of the grid LU: 3 caps it at 85 registers (3 x 256 threads
// per SM): the read-latency-bound sweep gets 50% more bytes in flight. C4's LUs
// 75.6 ms at 1 (255 registers allowed), 54.3 ms at the compiler's default (128
// registers, 2 CTAs), 51.3 ms at 3 (tools/ab_r2.sh)
#ifndef RCPG_LU_MINB
#define RCPG_LU_MINB 3
#endif
// Column batch per load round; a software-pipelined variant (the next batch's
// loads issued before this batch's update: B = 4 / 8, 2 or 3 CTAs per SM) was
// 12-23% slower on every C3-C5 panel (tools/gpu_s3r.sh), not kept.
#ifndef RCPG_LU_B
#define RCPG_LU_B 8
#endif

// V consecutive panel rows per thread (16-byte loads/stores when V > 1): the
// sweep is read-latency bound, so V multiplies the bytes each load keeps in
// flight. Requires J % V == 0, R % V == 0 and 16-byte aligned A and Z.
template <typename T, int V>
struct alignas(sizeof(T) * V) LuVec {
  T x[V];
};

template <typename T, int V>
__device__ __forceinline__ LuVec<T, V> ld_lv(const T* p) {
  return *reinterpret_cast<const LuVec<T, V>*>(p);
}

template <typename T, int V>
__device__ __forceinline__ void st_lv(T* p, const LuVec<T, V>& v) {
  *reinterpret_cast<LuVec<T, V>*>(p) = v;
}

template <typename T, int V>
__global__ void __launch_bounds__(kLuThreads, RCPG_LU_MINB) plu_coop_kernel(LuArgs<T> p) {
  __shared__ Cand<T> red[33];
  __shared__ int pcol_of[kMaxPanelCols], col_at[kMaxPanelCols];
  __shared__ T U[kMaxPanelCols], Uprev[kMaxPanelCols];
  __shared__ T s_pivprev;
  __shared__ int s_cprev;
  __shared__ i64 ov_pos[kMaxPanelCols], ov_row[kMaxPanelCols];
  __shared__ int n_ov;
  __shared__ i64 s_u;
  __shared__ unsigned s_chunk[2];

  const int G = gridDim.x;
  const i64 chunk = ceil_div(p.J, i64(G) * V) * V;
  const i64 r0 = blockIdx.x * chunk;
  const i64 r1 = r0 + chunk < p.J ? r0 + chunk : p.J;
  const Cand<T> none{T(-1), 0x7fffffff, 0, 0x7fffffffffffffffll, 0};
  const i64 R = p.R;
  const bool unit = (p.R == p.J);

  for (int c = threadIdx.x; c < p.n; c += blockDim.x) {
    pcol_of[c] = c;
    col_at[c] = c;
  }
  if (threadIdx.x == 0) n_ov = 0;

  Cand<T> best = none;
  for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
    const i64 ps = p.phys[s];
    const i64 ba = row_base(s, R, p.J, p.n);
    for (int c = 0; c < p.n; ++c) {
      const Cand<T> x{T(fabs(p.A[ba + c * R])), c, c, ps, s};
      if (better(x, best)) best = x;
    }
  }
  best = block_best(best, red);
  if (threadIdx.x == 0) p.cands[blockIdx.x] = best;
  grid_sync(p.bar);

  int k0 = p.r;
  const bool prof = p.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t_a = prof ? lu_timer() : 0;
  for (int k = 0; k < p.r; ++k) {
    const Cand<T>* cb = p.cands + (k & 1) * G;
    Cand<T> g = none;
    for (int q = threadIdx.x; q < G; q += blockDim.x) {
      const Cand<T> x = load_cand_cg(cb + q);
      if (better(x, g)) g = x;
    }
    g = block_best(g, red);
    if (!(g.v > T(0))) {  // exactly-zero corner (FullPivLU early stop)
      k0 = k;
      break;
    }
    const i64 ss = g.s;
    const int cs = g.c;
    const i64 pr = g.prow;
    const int pc = g.pcol;
    const i64 bss = row_base(ss, R, p.J, p.n);
    // Delayed write-back (p.delay): the panel is stored only after odd pivots.
    // On odd k the stored rows hold a^(k-1) and pivot k-1 is re-applied on the
    // fly with the identical expression (bit-identical to storing it), so a
    // pair of pivots costs two reads and one write of the trailing panel.
    const bool pend = p.delay && (k & 1) != 0;
    const bool wr = !p.delay || (k & 1) != 0;
    if (threadIdx.x == 0) {
      i64 u = -1;  // row at physical position k before the swap
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
    {
      // the pivot row at state k (stored as a^(k-1) when pend)
      const T mprev = pend ? ldcg(&p.A[bss + s_cprev * R]) / s_pivprev : T(0);
      for (int c = threadIdx.x; c < p.n; c += blockDim.x) {
        const T st = ldcg(&p.A[bss + c * R]);
        U[c] = pend ? sub_mul_rn(st, mprev, Uprev[c]) : st;
      }
    }
    __syncthreads();
    const T piv = U[cs];
    const i64 u = s_u;
    if (threadIdx.x == 0 && blockIdx.x == 0) {  // read in later steps (after a grid barrier)
      p.phys[ss] = k;
      if (u != ss) p.phys[u] = pr;
    }
    const bool dyn = p.chunk_groups > 0;
    if (threadIdx.x == 0) s_chunk[0] = dyn ? atomicAdd(&p.ctr[k], 1u) : unsigned(blockIdx.x);
    __syncthreads();
    unsigned long long t_b = 0;
    if (prof) {
      t_b = lu_timer();
      p.prof[0] += t_b - t_a;
    }

    best = none;
    Cand<T>* out = p.cands + ((k + 1) & 1) * G;
    const bool more = (k + 1 < p.r);
    const int cprev = s_cprev;
    const T pivprev = s_pivprev;
    // Snake order: odd pivots walk each thread's row groups backwards, so a step
    // starts on the rows the previous step touched last -- still in L2 (up to
    // ~100 MB of the trailing panel per step; all of it once it fits). The
    // candidates are order-independent (total order), so the bits do not change.
    // Rows are handed out in chunks from a per-step counter (the static split left
    // every step waiting ~25% on the slowest CTA: the SMs do not get equal shares
    // of HBM); the next chunk is claimed while this one is swept.
    // With fewer than two chunks per CTA the static split (one range per CTA) is
    // better balanced (chunk_groups = 0).
    const i64 grp = i64(blockDim.x) * V;
    const i64 csz = dyn ? grp * p.chunk_groups : chunk;
    const i64 nchunks = dyn ? ceil_div(p.J, csz) : i64(G);
    for (int ci = 0;; ++ci) {
      const i64 c0 = s_chunk[ci & 1];
      if (c0 >= nchunks) break;
      if (threadIdx.x == 0) s_chunk[(ci + 1) & 1] = dyn ? atomicAdd(&p.ctr[k], 1u) : unsigned(nchunks);
      const i64 cb = (dyn && (k & 1) ? nchunks - 1 - c0 : c0) * csz;
      const i64 cend = cb + csz < p.J ? cb + csz : p.J;
      for (i64 s0 = cb + i64(threadIdx.x) * V; s0 < cend; s0 += grp) {
      i64 ba, bz;
      if (unit) {
        ba = s0;
        bz = s0;
      } else {  // the V rows share one Kolda slice (R % V == 0)
        const i64 aa = s0 / R, bb = s0 - aa * R;
        ba = aa * p.n * R + bb;
        bz = aa * p.r * R + bb;
      }
      constexpr int B = RCPG_LU_B;  // vector loads in flight per thread
      LuVec<T, V> v[B];
      // the rows' physical positions, pivot-column values and the first chunk
      // are independent loads: one memory round trip, not two
      i64 ps[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const i64 se = s0 + e;
        ps[e] = se == ss ? i64(k) : (se == u ? pr : p.phys[se]);
      }
      const LuVec<T, V> pcv = ld_lv<T, V>(p.A + ba + cs * R);
      LuVec<T, V> pvv;
      if (pend) pvv = ld_lv<T, V>(p.A + ba + cprev * R);
#pragma unroll
      for (int u = 0; u < B; ++u)
        if (more && k + 1 + u < p.n) v[u] = ld_lv<T, V>(p.A + ba + col_at[k + 1 + u] * R);
      bool act[V], anyact = false;
      int ispiv = -1;
      LuVec<T, V> zk;
      T m[V], m1[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        // rows pivoted earlier keep their L row (zeros past their step) and
        // their panel values; the pivot row gets its unit entry
        act[e] = ps[e] >= k && s0 + e != ss;
        if (s0 + e == ss) ispiv = e;
        anyact |= act[e];
        // multiplier of the pending pivot k-1, exactly as written to Z then
        m1[e] = pend && act[e] ? pvv.x[e] / pivprev : T(0);
        const T pc = pend ? sub_mul_rn(pcv.x[e], m1[e], Uprev[cs]) : pcv.x[e];
        m[e] = act[e] ? pc / piv : T(0);
        zk.x[e] = s0 + e == ss ? T(1) : m[e];
      }
      if (!anyact && ispiv < 0) continue;  // all pivoted earlier
      st_lv<T, V>(p.Z + bz + k * R, zk);
      if (ispiv >= 0)
        for (int j = k + 1; j < p.r; ++j) p.Z[bz + ispiv + j * R] = T(0);
      if (more && anyact) {
        // each row's first maximum in physical-column order (one float compare
        // per entry), then one full candidate comparison per row: the same
        // pick as comparing every entry (all share the physical row ps)
        T rv[V];
        int rq[V], rc[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
          rv[e] = T(-1);
          rq[e] = 0;
          rc[e] = 0;
        }
        for (int q0 = k + 1; q0 < p.n; q0 += B) {
          if (q0 > k + 1) {
#pragma unroll
            for (int u = 0; u < B; ++u)
              if (q0 + u < p.n) v[u] = ld_lv<T, V>(p.A + ba + col_at[q0 + u] * R);
          }
#pragma unroll
          for (int u = 0; u < B; ++u)
            if (q0 + u < p.n) {
              const int c = col_at[q0 + u];
              const T uc = U[c];
              const T up = pend ? Uprev[c] : T(0);
              LuVec<T, V> x;
#pragma unroll
              for (int e = 0; e < V; ++e) {
                // inactive rows are written back unchanged (same bits)
                const T x1 = pend ? sub_mul_rn(v[u].x[e], m1[e], up) : v[u].x[e];
                x.x[e] = act[e] ? sub_mul_rn(x1, m[e], uc) : v[u].x[e];
                const T ax = fabs(x.x[e]);
                if (act[e] && ax > rv[e]) {
                  rv[e] = ax;
                  rq[e] = q0 + u;
                  rc[e] = c;
                }
              }
              if (wr) st_lv<T, V>(p.A + ba + c * R, x);
            }
        }
#pragma unroll
        for (int e = 0; e < V; ++e)
          if (act[e]) {
            const Cand<T> cd{rv[e], rq[e], rc[e], ps[e], s0 + e};
            if (better(cd, best)) best = cd;
          }
      }
      }
      __syncthreads();  // s_chunk[(ci + 1) & 1] visible; s_chunk[ci & 1] free
    }
    unsigned long long t_c = 0;
    if (prof) {
      t_c = lu_timer();
      p.prof[1] += t_c - t_b;
    }
    if (more) {
      best = block_best(best, red);
      if (threadIdx.x == 0) out[blockIdx.x] = best;
      grid_sync(p.bar);
    }
    // pivot k becomes the pending one of the next step (after every thread of
    // the block is done reading Uprev: the last step has no grid_sync)
    __syncthreads();
    for (int c = threadIdx.x; c < p.n; c += blockDim.x) Uprev[c] = U[c];
    if (threadIdx.x == 0) {
      s_cprev = cs;
      s_pivprev = piv;
    }
    __syncthreads();
    if (prof) {
      t_a = lu_timer();
      p.prof[2] += t_a - t_c;
      p.prof[3] += 1;
    }
  }

  if (k0 < p.r) {
    // the remaining L columns are unit vectors at the rows sitting at
    // physical positions k0..r-1 (the corner is exactly zero)
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
      const i64 ps = p.phys[s];
      if (ps < k0) continue;
      const i64 aa = s / R, bb = s - aa * R;
      const i64 bz = unit ? s : aa * p.r * R + bb;
      for (int j = k0; j < p.r; ++j) p.Z[bz + j * R] = (ps == j) ? T(1) : T(0);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.info = k0;
}

// ------------------------------------------------- LU, panel resident on chip
// The whole panel stays in the SMs for the factorization: CTA b (one per SM)
// owns rows [b*chunk, (b+1)*chunk); storage columns [0, ns) of its rows in
// shared memory, the last RC columns in registers (RPT rows per thread).
// Per pivot: block reduction, then each CTA publishes its best candidate with
// that row's current values (double-buffered by step parity); one grid
// barrier; every CTA picks the winner from the G keys, reads its row and
// applies the bookkeeping of plu_coop_kernel. Same keys, same arithmetic,
// same results as plu_coop_kernel; no panel traffic per pivot.
template <typename T>
struct LuResArgs {
  const T* A;
  T* Z;
  i64 J, R;
  int n, r, ns, chunk;
  const i64* keys;  // [J] Kolda (physical) index of every storage row
  KoldaMap km;
  Cand<T>* pubk;    // [2][G]
  T* pubr;          // [2][G][n]
  GridBarrier* bar;
  int* info;
  unsigned long long* prof;  // optional [8] (CTA 0): ns in reduce+publish / barrier / pick+book / update
};

__host__ __device__ constexpr int lu_res_max_threads(int rc, int rpt) { return rc * rpt == 0 ? 1024 : 640; }
constexpr int kResKeyLoads = 5;  // grids of up to 160 CTAs

// CL: the grid is one thread-block cluster; candidates and the winner's row
// are exchanged through distributed shared memory, one cluster barrier per
// pivot instead of a grid barrier.
template <typename T, int RC, int RPT, bool CL>
__global__ void __launch_bounds__(lu_res_max_threads(RC, RPT), 1) plu_resident_kernel(LuResArgs<T> p) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, nt = blockDim.x, G = gridDim.x, b = blockIdx.x;
  const int n = p.n, ns = p.ns, ldl = p.chunk;
  const i64 R = p.R;
  const i64 r0 = i64(b) * p.chunk;
  const int rows = int(max(i64(0), min(i64(p.chunk), p.J - r0)));
  T* a = reinterpret_cast<T*>(smem_raw);                                             // [ns][ldl]
  i64* physl = reinterpret_cast<i64*>(smem_raw + ((size_t(ns) * ldl * sizeof(T) + 15) & ~size_t(15)));  // [ldl]
  __shared__ int pcol_of[kMaxPanelCols], col_at[kMaxPanelCols];
  __shared__ T U[kMaxPanelCols];
  __shared__ i64 ov_pos[kMaxPanelCols], ov_row[kMaxPanelCols];
  __shared__ int n_ov, red_w[kResKeyLoads];
  __shared__ i64 kinv[kMaxPanelCols];  // Kolda row at physical position k (before any swap)
  __shared__ Cand<T> red[33];
  __shared__ Cand<T> cpub[CL ? 2 : 1];                       // CL: this CTA's candidate per parity
  __shared__ __align__(16) T rpub[CL ? 2 : 1][CL ? kMaxPanelCols : 1];  // CL: its row
  const Cand<T> none{T(-1), 0x7fffffff, 0, 0x7fffffffffffffffll, 0};
  T rg[RPT][RC > 0 ? RC : 1];
  for (int c = tid; c < n; c += nt) {
    pcol_of[c] = c;
    col_at[c] = c;
  }
  if (tid == 0) n_ov = 0;
  for (int q = tid; q < p.r; q += nt) kinv[q] = kolda_inverse(p.km, q, p.R);
  // load own rows, first candidates (all columns, physical order = storage order)
  Cand<T> best = none;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int lr = tid + i * nt;
    if (lr >= rows) continue;
    const i64 s = r0 + lr;
    const i64 ba = row_base(s, R, p.J, n);
    const i64 ps = p.keys[s];
    physl[lr] = ps;
    T rv = T(-1);
    int rq = 0;
    for (int c = 0; c < ns; ++c) {
      const T x = p.A[ba + c * R];
      a[c * ldl + lr] = x;
      if (fabs(x) > rv) {
        rv = fabs(x);
        rq = c;
      }
    }
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      const T x = ns + j < n ? p.A[ba + (ns + j) * R] : T(0);
      rg[i][j] = x;
      if (ns + j < n && fabs(x) > rv) {
        rv = fabs(x);
        rq = ns + j;
      }
    }
    const Cand<T> cd{rv, rq, rq, ps, s};
    if (better(cd, best)) best = cd;
  }
  int k0 = p.r;
  const bool prof = p.prof != nullptr && b == 0 && tid == 0;
  unsigned long long t0 = prof ? lu_timer() : 0, t1 = 0;
  for (int k = 0; k < p.r; ++k) {
    const int par = k & 1;
    // 1. this CTA's best, published with its row's current values
    best = block_best(best, red);
    if (tid == 0) {
      if constexpr (CL)
        cpub[par] = best;
      else
        p.pubk[par * G + b] = best;
    }
    if (best.v > T(0) && best.s >= r0 && best.s < r0 + rows) {
      const int lr = int(best.s - r0);
      if (lr % nt == tid) {
        const int i = lr / nt;
        T* dst = CL ? &rpub[par & (CL ? 1 : 0)][0] : p.pubr + (i64(par) * G + b) * n;
        for (int c = 0; c < ns; ++c) dst[c] = a[c * ldl + lr];
#pragma unroll
        for (int ii = 0; ii < RPT; ++ii)
          if (ii == i) {
#pragma unroll
            for (int j = 0; j < RC; ++j)
              if (ns + j < n) dst[ns + j] = rg[ii][j];
          }
      }
    }
    if (prof) {
      t1 = lu_timer();
      p.prof[0] += t1 - t0;
      t0 = t1;
    }
    if constexpr (CL)
      cg::this_cluster().sync();
    else
      grid_sync(p.bar);
    if (prof) {
      t1 = lu_timer();
      p.prof[1] += t1 - t0;
      t0 = t1;
    }
    // 2. the winner (every CTA, same order), its row, the bookkeeping
    // up to five warps, one key per thread: every key load in flight at once
    if (tid < 32 * kResKeyLoads) {
      Cand<T> g = none;
      if (tid < G) {
        if constexpr (CL)
          g = *cg::this_cluster().map_shared_rank(&cpub[par & (CL ? 1 : 0)], tid);
        else
          g = load_cand_cg(p.pubk + par * G + tid);
      }
      int gw = tid;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const Cand<T> y = shfl_cand(g, o);
        const int yw = __shfl_xor_sync(0xffffffffu, gw, o);
        if (better(y, g)) {
          g = y;
          gw = yw;
        }
      }
      if ((tid & 31) == 0) {
        red[tid >> 5] = g;
        red_w[tid >> 5] = gw;
      }
    }
    __syncthreads();
    // every thread reduces the <= 5 warp winners itself (no second barrier)
    Cand<T> g = red[0];
    int gwin = red_w[0];
    for (int q = 1; q < kResKeyLoads && 32 * q < G; ++q)
      if (better(red[q], g)) {
        g = red[q];
        gwin = red_w[q];
      }
    if (!(g.v > T(0))) {  // exactly-zero corner (FullPivLU early stop)
      k0 = k;
      break;
    }
    const i64 ss = g.s, pr = g.prow;
    const int cs = g.c, pc = g.pcol;
    if constexpr (CL) {
      const T* src = cg::this_cluster().map_shared_rank(&rpub[par & (CL ? 1 : 0)][0], gwin);
      for (int c = tid; c < n; c += nt) U[c] = src[c];
    } else {
      const T* src = p.pubr + (i64(par) * G + gwin) * n;
      for (int c = tid; c < n; c += nt) U[c] = ldcg(src + c);
    }
    if (tid == 0) {
      i64 u = -1;  // row at physical position k before the swap
      for (int q = n_ov - 1; q >= 0; --q)
        if (ov_pos[q] == k) {
          u = ov_row[q];
          break;
        }
      if (u < 0) u = kinv[k];
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
      if (ss >= r0 && ss < r0 + rows) physl[ss - r0] = k;
      if (u != ss && u >= r0 && u < r0 + rows) physl[u - r0] = pr;
    }
    __syncthreads();
    const T piv = U[cs];
    const bool more = k + 1 < p.r;
    if (prof) {
      t1 = lu_timer();
      p.prof[2] += t1 - t0;
      t0 = t1;
    }
    // 3. update own rows, next candidates: 8 columns per batch, every load of
    // a batch before its stores (no smem aliasing chain), all rows together
    best = none;
    bool act[RPT];
    T m[RPT], rv[RPT];
    int rq[RPT], rcol[RPT];
    i64 psr[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int lr = tid + i * nt;
      act[i] = false;
      m[i] = T(0);
      rv[i] = T(-1);
      rq[i] = 0x7fffffff;
      rcol[i] = 0;
      psr[i] = 0;
      if (lr >= rows) continue;
      psr[i] = physl[lr];
      if (psr[i] <= k) continue;  // pivoted (the pivot row itself has ps == k)
      act[i] = true;
      T pcv;
      if (cs < ns) {
        pcv = a[cs * ldl + lr];
      } else {
        pcv = T(0);
#pragma unroll
        for (int j = 0; j < RC; ++j)
          if (cs == ns + j) pcv = rg[i][j];
      }
      m[i] = pcv / piv;
      if (cs < ns) {
        a[cs * ldl + lr] = m[i];
      } else {
#pragma unroll
        for (int j = 0; j < RC; ++j)
          if (cs == ns + j) rg[i][j] = m[i];
      }
    }
    if (more) {
      constexpr int NB = RC * RPT >= 8 ? 4 : 8;
      for (int q0 = k + 1; q0 < n; q0 += NB) {
        int cc[NB];
        T uc[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          cc[u] = q0 + u < n ? col_at[q0 + u] : ns;
          uc[u] = cc[u] < ns ? U[cc[u]] : T(0);
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          if (!act[i]) continue;
          const int lr = tid + i * nt;
          T xv[NB];
#pragma unroll
          for (int u = 0; u < NB; ++u)
            if (cc[u] < ns) xv[u] = a[cc[u] * ldl + lr];
#pragma unroll
          for (int u = 0; u < NB; ++u)
            if (cc[u] < ns) {
              const T x = sub_mul_rn(xv[u], m[i], uc[u]);
              a[cc[u] * ldl + lr] = x;
              if (fabs(x) > rv[i]) {  // columns in physical order: first maximum
                rv[i] = fabs(x);
                rq[i] = q0 + u;
                rcol[i] = cc[u];
              }
            }
        }
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        if (!act[i]) continue;
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          const int c = ns + j;
          if (c >= n) continue;
          const int q = pcol_of[c];
          if (q <= k) continue;
          const T x = sub_mul_rn(rg[i][j], m[i], U[c]);
          rg[i][j] = x;
          const T ax = fabs(x);
          if (ax > rv[i] || (ax == rv[i] && q < rq[i])) {
            rv[i] = ax;
            rq[i] = q;
            rcol[i] = c;
          }
        }
        const Cand<T> cd{rv[i], rq[i], rcol[i], psr[i], r0 + tid + i * nt};
        if (better(cd, best)) best = cd;
      }
    }
    if (prof) {
      t1 = lu_timer();
      p.prof[3] += t1 - t0;
      p.prof[4] += 1;
      t0 = t1;
    }
  }
  __syncthreads();
  // P^{-1} L for own rows: multipliers left of the row's physical position
  // (before an early stop), the unit entry, zeros right of it
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int lr = tid + i * nt;
    if (lr >= rows) continue;
    const i64 s = r0 + lr;
    const i64 pp = physl[lr];
    const i64 bz = row_base(s, R, p.J, p.r);
    for (int j = 0; j < p.r; ++j) {
      T v = T(0);
      if (pp == j) {
        v = T(1);
      } else if (j < pp && j < k0) {
        const int c = col_at[j];
        if (c < ns) {
          v = a[c * ldl + lr];
        } else {
#pragma unroll
          for (int jj = 0; jj < RC; ++jj)
            if (c == ns + jj) v = rg[i][jj];
        }
      }
      p.Z[bz + j * R] = v;
    }
  }
  if (b == 0 && tid == 0) *p.info = k0;
  if constexpr (CL) cg::this_cluster().sync();  // keep this CTA's smem alive for remote readers
}

// ---------------------------------------------------------- Householder
template <typename T>
struct QrArgs {
  T* A;        // panel J x n (in/out: essential vectors below the diagonal)
  T* Q;        // output panel J x r
  i64 J, R;
  int n, r;
  i64* krow;        // [J] Kolda row index (filled by the kernel: every CTA reads only its own rows)
  KoldaMap km;
  double* part;     // [2][G][kMaxPanelCols + 1]
  T* tau;           // [r]
  T* diag;          // [r] R_kk = beta_k
  GridBarrier* bar;
  int* rank_warning;
  const int* skip;  // when non-null and *skip == 0: CholeskyQR2 already produced Q
  double* rowk;     // [kMaxPanelCols] row k before step k's update (FactorWork::rowk)
};

template <typename T>
__global__ void __launch_bounds__(kFacThreads) householder_kernel(QrArgs<T> p) {
  if (p.skip != nullptr && *p.skip == 0) return;
  __shared__ double red[33];
  __shared__ double tmp[kMaxPanelCols];
  const int G = gridDim.x;
  const i64 chunk = ceil_div(p.J, G);
  const i64 r0 = blockIdx.x * chunk;
  const i64 r1 = r0 + chunk < p.J ? r0 + chunk : p.J;
  constexpr int PW = kMaxPanelCols + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const i64 R = p.R;
  int phase = 0;
  // row keys of this CTA's rows (no separate launch: the kernel is a skipped
  // fallback after CholeskyQR2 in the common case)
  for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
    const i64 a = s / R, b = s - a * R;
    p.krow[s] = kolda_index(p.km, a, b);
  }
  __syncthreads();

  for (int k = 0; k < p.r; ++k) {
    const i64 sk = kolda_inverse(p.km, k, p.R);
    const bool own_k = (sk >= r0 && sk < r1);
    const i64 bk = row_base(sk, R, p.J, p.n);
    // 1. tail squared norm of column k
    double acc = 0.0;
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x)
      if (p.krow[s] > k) {
        const double x = double(p.A[row_base(s, R, p.J, p.n) + k * R]);
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
    const T c0 = ldcg(&p.A[bk + k * R]);
    T beta, t;
    const bool trivial = !(tail_sq > Traits<T>::realmin);
    if (trivial) {
      t = T(0);
      beta = c0;
    } else {
      beta = sqrt(add_rn(mul_rn(c0, c0), tail_sq));
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
        const i64 ad = row_base(s, R, p.J, p.n) + k * R;
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
        if (p.krow[s] > k) {
          const i64 b = row_base(s, R, p.J, p.n);
          a2 += double(p.A[b + k * R]) * double(p.A[b + j * R]);
        }
      a2 = warp_sum(a2);
      if (lane == 0) pb[blockIdx.x * PW + jj] = a2;
    }
    if (own_k)  // row k as it is before this step's update (read by every CTA after the barrier)
      for (int jj = threadIdx.x; jj < ncol; jj += blockDim.x) p.rowk[jj] = double(p.A[bk + (k + 1 + jj) * R]);
    grid_sync(p.bar);
    // tmp_j = Scalar(v_tail . A(tail, j)) + A(k, j): the dot product in double,
    // rounded to Scalar, then one Scalar addition (the oracle's thin_qr order)
    for (int jj = threadIdx.x; jj < ncol; jj += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += ldcg(&pb[q * PW + jj]);
      tmp[jj] = double(add_rn(T(s), T(ldcg(&p.rowk[jj]))));
    }
    phase ^= 1;
    __syncthreads();
    // 3. rank-1 update of own rows
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
      const i64 kr = p.krow[s];
      const i64 b = row_base(s, R, p.J, p.n);
      if (kr > k) {
        const T e = p.A[b + k * R];
        const T te = mul_rn(t, e);
        for (int jj = 0; jj < ncol; ++jj) {
          T& x = p.A[b + (k + 1 + jj) * R];
          x = sub_mul_rn(x, te, T(tmp[jj]));
        }
      } else if (kr == k) {
        for (int jj = 0; jj < ncol; ++jj) {
          T& x = p.A[b + (k + 1 + jj) * R];
          x = sub_mul_rn(x, t, T(tmp[jj]));
        }
      }
    }
  }
  grid_sync(p.bar);  // every tau/diag write (block 0) visible before the Q sweep
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
    const i64 b = row_base(s, R, p.J, p.r);
    for (int j = 0; j < p.r; ++j) p.Q[b + j * R] = (kr == j) ? T(1) : T(0);
  }
  __syncthreads();  // rows are written thread-per-row, read warp-per-column below
  for (int k = p.r - 1; k >= 0; --k) {
    const T t = ldcg(&p.tau[k]);
    if (t == T(0)) continue;  // uniform across CTAs
    const i64 sk = kolda_inverse(p.km, k, p.R);
    const bool own_k = (sk >= r0 && sk < r1);
    const i64 bqk = row_base(sk, R, p.J, p.r);
    const int ncol = p.r - k;  // columns j < k are untouched (exactly unchanged in Eigen too)
    double* pb = p.part + phase * G * PW;
    for (int jj = wid; jj < ncol; jj += nw) {
      const int j = k + jj;
      double a2 = 0.0;
      for (i64 s = r0 + lane; s < r1; s += 32)
        if (p.krow[s] > k)
          a2 += double(p.A[row_base(s, R, p.J, p.n) + k * R]) * double(p.Q[row_base(s, R, p.J, p.r) + j * R]);
      a2 = warp_sum(a2);
      if (lane == 0) pb[blockIdx.x * PW + jj] = a2;
    }
    if (own_k)
      for (int jj = threadIdx.x; jj < ncol; jj += blockDim.x) p.rowk[jj] = double(p.Q[bqk + (k + jj) * R]);
    grid_sync(p.bar);
    for (int jj = threadIdx.x; jj < ncol; jj += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += ldcg(&pb[q * PW + jj]);
      tmp[jj] = double(add_rn(T(s), T(ldcg(&p.rowk[jj]))));
    }
    phase ^= 1;
    __syncthreads();
    for (i64 s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
      const i64 kr = p.krow[s];
      const i64 bq = row_base(s, R, p.J, p.r);
      if (kr > k) {
        const T e = p.A[row_base(s, R, p.J, p.n) + k * R];
        const T te = mul_rn(t, e);
        for (int jj = 0; jj < ncol; ++jj) {
          T& x = p.Q[bq + (k + jj) * R];
          x = sub_mul_rn(x, te, T(tmp[jj]));
        }
      } else if (kr == k) {
        for (int jj = 0; jj < ncol; ++jj) {
          T& x = p.Q[bq + (k + jj) * R];
          x = sub_mul_rn(x, t, T(tmp[jj]));
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------- Householder on one cluster
// The faithful thin_qr (compress.hpp:60-73, Eigen's unblocked HouseholderQR in
// the reference's Scalar arithmetic, operation for operation as
// householder_kernel) for panels that fit the distributed shared memory of one
// thread-block cluster: CTA r owns rows [r chunk, (r+1) chunk) of the I x n
// panel (column-major in its smem); the per-column reductions (tail norm, the
// n - k - 1 dot products, in fp64) are partial sums per CTA added in CTA order
// through DSMEM. Two cluster barriers per reflector, one per Q column step,
// instead of householder_kernel's grid barriers. Q (I x r, ld I) is built in
// global memory, each CTA updating its own rows.
constexpr int kHhThreads = 512;

// sum_{q < CS} (value at p in CTA q of the cluster), in rank order, with every
// DSMEM load issued before the first add (a dependent chain of remote loads
// cost ~1.5 us per reduction at 16 CTAs)
__device__ __forceinline__ double cluster_ordered_sum(cooperative_groups::cluster_group& cl, double* p, int CS) {
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = q < CS ? *cl.map_shared_rank(p, q) : 0.0;
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q)
    if (q < CS) s += v[q];
  return s;
}

template <typename T>
__global__ void __launch_bounds__(kHhThreads) householder_cluster_kernel(const T* __restrict__ A, T* __restrict__ Q,
                                                                         int I, int n, int chunk,
                                                                         int* rank_warning) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = int(cl.num_blocks()), me = int(cl.block_rank());
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* part = reinterpret_cast<double*>(smem_raw);   // [2][kMaxPanelCols + 1] partial sums (double-buffered)
  double* rowk = part + 2 * (kMaxPanelCols + 1);        // [2][kMaxPanelCols] row k (owner's copy)
  T* tau = reinterpret_cast<T*>(rowk + 2 * kMaxPanelCols);  // [kMaxPanelCols]
  T* diag = tau + kMaxPanelCols;                        // [kMaxPanelCols]
  T* a = diag + kMaxPanelCols;                          // [n][chunk] own rows
  __shared__ double red[32];
  __shared__ double tmp[kMaxPanelCols];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const int r0 = me * chunk, rows = max(0, min(chunk, I - r0));
  const int r = min(I, n);
  for (int e = tid; e < chunk * n; e += nt) {
    const int i = e % chunk, j = e / chunk;
    a[e] = i < rows ? A[i64(r0 + i) + i64(j) * I] : T(0);
  }
  __syncthreads();
  auto block_sum = [&](double v) {
    v = warp_sum(v);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    if (wid == 0) {
      s = lane < nw ? red[lane] : 0.0;
      s = warp_sum(s);
    }
    return s;  // valid in warp 0
  };
  for (int k = 0; k < r; ++k) {
    const int buf = k & 1;
    double* pb = part + buf * (kMaxPanelCols + 1);
    const int ok = k / chunk, lk = k - ok * chunk;  // owner CTA / local row of row k
    const int i0 = max(0, k + 1 - r0);              // first own row below k
    // 1. tail squared norm of column k (fp64)
    double acc = 0.0;
    for (int i = i0 + tid; i < rows; i += nt) {
      const double x = double(a[i + k * chunk]);
      acc += x * x;
    }
    acc = block_sum(acc);
    if (tid == 0) pb[kMaxPanelCols] = acc;
    cl.sync();
    const double tsq = cluster_ordered_sum(cl, pb + kMaxPanelCols, CS);
    const T tail_sq = T(tsq);
    const T c0 = *cl.map_shared_rank(a + lk + k * chunk, ok);
    T beta, t;
    const bool trivial = !(tail_sq > Traits<T>::realmin);
    if (trivial) {
      t = T(0);
      beta = c0;
    } else {
      beta = sqrt(add_rn(mul_rn(c0, c0), tail_sq));
      if (c0 >= T(0)) beta = -beta;
      t = (beta - c0) / beta;
    }
    const T denom = c0 - beta;
    if (tid == 0) {
      tau[k] = t;
      diag[k] = beta;
    }
    // 2. essential vector of own tail rows
    for (int i = i0 + tid; i < rows; i += nt) a[i + k * chunk] = trivial ? T(0) : a[i + k * chunk] / denom;
    __syncthreads();
    const int ncol = n - k - 1;
    // 3. partial v^T A(:, j) (fp64) and the owner's row k
    if (!trivial && ncol > 0) {
      for (int jj = wid; jj < ncol; jj += nw) {
        const int j = k + 1 + jj;
        double s = 0.0;
        for (int i = i0 + lane; i < rows; i += 32) s += double(a[i + k * chunk]) * double(a[i + j * chunk]);
        s = warp_sum(s);
        if (lane == 0) pb[jj] = s;
      }
      if (me == ok)
        for (int jj = tid; jj < ncol; jj += nt) rowk[buf * kMaxPanelCols + jj] = double(a[lk + (k + 1 + jj) * chunk]);
    }
    cl.sync();
    // 4. tmp_j = Scalar(v . A(:, j)) + A(k, j); rank-1 update of own rows
    if (!trivial && ncol > 0) {
      for (int jj = tid; jj < ncol; jj += nt) {
        const double sum = cluster_ordered_sum(cl, pb + jj, CS);
        tmp[jj] = double(add_rn(T(sum), T(*cl.map_shared_rank(rowk + buf * kMaxPanelCols + jj, ok))));
      }
      __syncthreads();
      // a thread per own row (no index division per entry, conflict-free
      // columns); t * v_i formed once per row -- the same value per entry
      for (int i = max(0, k - r0) + tid; i < rows; i += nt) {
        const T f = r0 + i == k ? t : mul_rn(t, a[i + k * chunk]);
        for (int jj = 0; jj < ncol; ++jj) {
          T& x = a[i + (k + 1 + jj) * chunk];
          x = sub_mul_rn(x, f, T(tmp[jj]));
        }
      }
    }
    if (me == ok && tid == 0) a[lk + k * chunk] = beta;
    __syncthreads();
  }
  if (me == 0 && tid == 0 && rank_warning != nullptr) {
    T dmax = T(0), dmin = T(INFINITY);
    for (int k = 0; k < r; ++k) {
      const T d = fabs(diag[k]);
      dmax = d > dmax ? d : dmax;
      dmin = d < dmin ? d : dmin;
    }
    const T tol = T(I) * Traits<T>::eps * dmax;
    *rank_warning = (dmax == T(0)) || (dmin <= tol);
  }
  // Q = H_0 ... H_{r-1} I(I, r), accumulated backward in shared memory in place
  // of the essential vectors: step k needs vector k and Q columns k..r-1; Q
  // column j > k already sits in slot j (its vector was used at step j), and Q
  // column k -- e_k before the step -- is written into slot k by each row's
  // thread after that row's other columns (the vector entry is read first).
  __syncthreads();
  for (int k = r - 1; k >= 0; --k) {
    const T t = tau[k];
    const int buf = k & 1;
    double* pb = part + buf * (kMaxPanelCols + 1);
    const int ok = k / chunk, lk = k - ok * chunk;
    const int i0 = max(0, k + 1 - r0);
    const int ncol = r - k;  // columns j < k are untouched (exactly unchanged in Eigen too)
    if (t != T(0)) {         // identical on every CTA
      // v . Q(:, j) over the own rows below k (column k: Q = e_k, the sum is 0)
      for (int jj = wid; jj < ncol; jj += nw) {
        double s = 0.0;
        if (jj > 0)
          for (int i = i0 + lane; i < rows; i += 32) s += double(a[i + k * chunk]) * double(a[i + (k + jj) * chunk]);
        s = warp_sum(s);
        if (lane == 0) pb[jj] = s;
      }
      if (me == ok)  // Q(k, k + jj): 1 for jj = 0, else slot k + jj's row k
        for (int jj = tid; jj < ncol; jj += nt) rowk[buf * kMaxPanelCols + jj] = jj == 0 ? 1.0 : double(a[lk + (k + jj) * chunk]);
    }
    cl.sync();  // partials of this step; the other buffer is free (read before the previous barrier)
    if (t != T(0))
      for (int jj = tid; jj < ncol; jj += nt) {
        const double sum = cluster_ordered_sum(cl, pb + jj, CS);
        tmp[jj] = double(add_rn(T(sum), T(*cl.map_shared_rank(rowk + buf * kMaxPanelCols + jj, ok))));
      }
    __syncthreads();
    for (int i = tid; i < rows; i += nt) {
      const int gi = r0 + i;
      const T q0 = gi == k ? T(1) : T(0);  // Q(gi, k) before the step
      if (t == T(0) || gi < k) {
        a[i + k * chunk] = q0;
        continue;
      }
      const T f = gi == k ? t : mul_rn(t, a[i + k * chunk]);
      for (int jj = 1; jj < ncol; ++jj) {
        T& x = a[i + (k + jj) * chunk];
        x = sub_mul_rn(x, f, T(tmp[jj]));
      }
      a[i + k * chunk] = sub_mul_rn(q0, f, T(tmp[0]));
    }
    __syncthreads();
  }
  for (int e = tid; e < rows * r; e += nt) {
    const int i = e % rows, j = e / rows;
    Q[i64(r0 + i) + i64(j) * I] = a[i + j * chunk];
  }
  cl.sync();  // no CTA exits while others may still read its shared memory
}

// -------------------------------------------------------- CholeskyQR2
// One CTA; Y is I x n column-major (I >= n). work >= I*n doubles.
// status: 0 = Q written, 1 = fall back to Householder.
constexpr int kCqrThreads = 512;

template <typename T>
__global__ void __launch_bounds__(kCqrThreads) cqr2_kernel(const T* __restrict__ Y, T* __restrict__ Q, int I, int n,
                                                             double* __restrict__ work, int* status,
                                                             int* rank_warning) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* G = reinterpret_cast<double*>(smem_raw);  // n x n
  double* Rm = G + n * n;                            // n x n upper Cholesky factor
  double* dg = Rm + n * n;                           // [2][n] diagonals of R1, R2
  double* sgn = dg + 2 * n;                          // [n]
  __shared__ int s_fail;
  __shared__ double s_piv;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  if (tid == 0) s_fail = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    // G = V^T V with V = Y (pass 0) or Q1 (pass 1, in work)
    for (int e = wid; e < n * n; e += nw) {
      const int a = e % n, b = e / n;
      if (a > b) continue;
      double s = 0.0;
      if (pass == 0) {
        for (int i = lane; i < I; i += 32) s += double(Y[i + i64(a) * I]) * double(Y[i + i64(b) * I]);
      } else {
        for (int i = lane; i < I; i += 32) s += work[i + i64(a) * I] * work[i + i64(b) * I];
      }
      s = warp_sum(s);
      if (lane == 0) {
        G[a + b * n] = s;
        G[b + a * n] = s;
      }
    }
    __syncthreads();
    // upper Cholesky G = R^T R (R in Rm, column-major upper)
    for (int j = 0; j < n; ++j) {
      if (tid == 0) {
        double d = G[j + j * n];
        for (int k = 0; k < j; ++k) d -= Rm[k + j * n] * Rm[k + j * n];
        if (!(d > 0.0)) s_fail = 1;
        s_piv = d > 0.0 ? sqrt(d) : 1.0;
        Rm[j + j * n] = s_piv;
        dg[pass * n + j] = s_piv;
      }
      __syncthreads();
      const double dj = s_piv;
      for (int c = j + 1 + tid; c < n; c += nt) {
        double s = G[j + c * n];
        for (int k = 0; k < j; ++k) s -= Rm[k + j * n] * Rm[k + c * n];
        Rm[j + c * n] = s / dj;
      }
      __syncthreads();
    }
    if (s_fail) break;
    // Ri = R^{-1} (upper; column-parallel back substitution), stored in G
    for (int j = tid; j < n; j += nt) {
      for (int i = j + 1; i < n; ++i) G[i + j * n] = 0.0;
      G[j + j * n] = 1.0 / Rm[j + j * n];
      for (int i = j - 1; i >= 0; --i) {
        double s = 0.0;
        for (int k = i + 1; k <= j; ++k) s += Rm[i + k * n] * G[k + j * n];
        G[i + j * n] = -s / Rm[i + i * n];
      }
    }
    __syncthreads();
    // V <- V R^{-1}: out (i, j) = sum_{k <= j} V(i, k) Ri(k, j); pass 0 writes
    // Q1 into work, pass 1 keeps Q1 (work) and writes Q2 to the tail half.
    double* dst = pass == 0 ? work : work + i64(I) * n;
    for (i64 e = tid; e < i64(I) * n; e += nt) {
      const int i = int(e % I), j = int(e / I);
      double s = 0.0;
      for (int k = 0; k <= j; ++k)
        s += (pass == 0 ? double(Y[i + i64(k) * I]) : work[i + i64(k) * I]) * G[k + j * n];
      dst[e] = s;
    }
    __syncthreads();
  }
  if (!s_fail) {
    for (i64 e = tid; e < i64(I) * n; e += nt) work[e] = work[e + i64(I) * n];
    __syncthreads();
  }
  if (!s_fail && tid == 0) {
    // conditioning guard: CholeskyQR2 is only used well inside its stable range
    double mx = 0.0, mn = INFINITY;
    for (int j = 0; j < n; ++j) {
      mx = fmax(mx, dg[j]);
      mn = fmin(mn, dg[j]);
    }
    if (!(mn > 0.0) || mx / mn > 1e6) s_fail = 1;
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0) *status = 1;
    return;
  }
  // Householder sign reconstruction on the top n x n block of Q2 (in G).
  for (int e = tid; e < n * n; e += nt) G[e] = work[(e % n) + i64(e / n) * I];
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    // Eigen's Householder leaves the last column of a square panel unreflected
    // (empty tail: tau = 0, beta = c0), so its sign is the opposite one
    if (tid == 0) sgn[k] = (G[k + k * n] > 0.0) != (k == I - 1) ? -1.0 : 1.0;
    __syncthreads();
    const double sk = sgn[k];
    if (sk < 0.0)
      for (int i = tid; i < n; i += nt) G[i + k * n] = -G[i + k * n];
    __syncthreads();
    if (tid == 0) G[k + k * n] -= 1.0;
    __syncthreads();
    const double dkk = G[k + k * n];
    for (int j = k + 1 + (tid >> 5); j < n; j += (nt >> 5))
      for (int i = k + 1 + (tid & 31); i < n; i += 32) G[i + j * n] -= (G[i + k * n] / dkk) * G[k + j * n];
    __syncthreads();
  }
  for (i64 e = tid; e < i64(I) * n; e += nt) Q[e] = T(work[e] * sgn[e / I]);
  if (tid == 0) {
    T dmax = T(0), dmin = T(INFINITY);
    for (int j = 0; j < n; ++j) {
      const T d = T(dg[j] * dg[n + j]);
      dmax = d > dmax ? d : dmax;
      dmin = d < dmin ? d : dmin;
    }
    if (rank_warning) *rank_warning = (dmax == T(0)) || (dmin <= T(I) * Traits<T>::eps * dmax);
    *status = 0;
  }
}

// ------------------------------------------------ CholeskyQR2, all SMs
// Small dense steps shared by the CholeskyQR2 kernels, one CTA, matrices in
// shared memory with an odd leading dimension ld (bank spread):
//   chol_inv_small: upper Cholesky A = R^T R, dg[j] = R(j, j), X = R^{-1}
//     (upper), *fail on breakdown;
//   sign_reconstruct: signs of Eigen's HouseholderQR Q relative to the
//     CholeskyQR Q from the top n x n block (modified LU of Q_top - S).
// Both are latency chains of n dependent steps; each step is one barrier.
//
// chol_inv_small runs symmetric elimination without square roots (A = U^T D U,
// U unit upper) on the augmented matrix [A | I] held in ONE n x n array M:
// the upper triangle (incl. the diagonal) is the A part, the strict lower
// triangle the I part (the I part's diagonal stays 1 until its row is
// pivotal, so it is implicit). Step j, for every row r > j:
//   A part (c >= r): M(r, c) -= (M(j, r) / d_j) * M(j, c)
//   I part (c <= j): M(r, c) -= (M(j, r) / d_j) * (c == j ? 1 : M(j, c))
// with d_j = M(j, j). Row j is never written from step j on, so after the
// last step U(j, c) = M(j, c) / d_j and (U^{-T})(j, c) = M(j, c) (c < j);
// R = D^{1/2} U and R^{-1} = U^{-1} D^{-1/2} then come out of one parallel
// pass. The critical path per step is one reciprocal, two FMAs and one
// barrier (no square root, no division chain); every thread owns the
// entries (r, c) with r = warp (mod warps), c = lane (mod 32).
__device__ __forceinline__ double sq_scale(double m, double rd, double sq) { return (m * rd) * sq; }

__device__ void chol_inv_small(double* A, double* X, int n, int ld, double* dg, int* fail) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  __shared__ double s_rd[kMaxPanelCols];  // 1 / d_j
  // the I part starts as the identity: strict lower triangle = 0 (own entries)
  for (int r = wid; r < n; r += nw)
    for (int c = lane; c < r; c += 32) A[r + c * ld] = 0.0;
  __syncthreads();
  int bad = 0;
  for (int j = 0; j < n; ++j) {
    const double d = A[j + j * ld];
    bad |= !(d > 0.0);
    const double rd = d > 0.0 ? __drcp_rn(d) : 1.0;
    if (tid == 0) s_rd[j] = rd;
    // first owned row below j
    int r = wid + ((j + 1 - wid + nw - 1) / nw) * nw;
    if (r < j + 1) r += nw;
    for (; r < n; r += nw) {
      const double t = A[j + r * ld] * rd;  // U(j, r)
      for (int c = lane; c < n; c += 32) {
        if (c >= r) {
          A[r + c * ld] -= t * A[j + c * ld];
        } else if (c <= j) {
          A[r + c * ld] -= t * (c == j ? 1.0 : A[j + c * ld]);
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0 && bad) *fail = 1;
  // R(j, c) = sqrt(d_j) U(j, c); X = R^{-1}: X(c, j) = (U^{-T})(j, c) / sqrt(d_j)
  for (int j = wid; j < n; j += nw) {
    const double d = A[j + j * ld];
    const double sq = d > 0.0 ? sqrt(d) : 1.0;
    const double rs = 1.0 / sq;
    if (lane == 0) dg[j] = sq;
    for (int c = lane; c < n; c += 32) {
      if (c < j) X[c + j * ld] = A[j + c * ld] * rs;
      else X[c + j * ld] = (c == j) ? rs : 0.0;
    }
  }
  __syncthreads();
  for (int j = wid; j < n; j += nw)
    for (int c = j + 1 + lane; c < n; c += 32) A[j + c * ld] = sq_scale(A[j + c * ld], s_rd[j], dg[j]);
  for (int j = tid; j < n; j += nt) A[j + j * ld] = dg[j];
  __syncthreads();
}

// G: top n x n block of Q2 (ld), destroyed. rows = panel height (square
// panels: Eigen leaves the last column unreflected, opposite sign).
// One barrier per step: the sign flip of column k is folded into the
// multipliers (negation is exact); every thread forms 1 / d_kk itself.
__device__ void sign_reconstruct_smem(double* G, int n, int ld, int rows, double* sgn) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < n; ++k) {
    const double gkk = G[k + k * ld];
    const double sk = (gkk > 0.0) != (k == rows - 1) ? -1.0 : 1.0;
    const double rd = __drcp_rn(sk * gkk - 1.0);
    if (tid == 0) sgn[k] = sk;
    int i = wid + ((k + 1 - wid + nw - 1) / nw) * nw;
    if (i < k + 1) i += nw;
    for (; i < n; i += nw) {  // warp per row, lanes over columns
      const double l = (sk * G[i + k * ld]) * rd;
      for (int j = k + 1 + lane; j < n; j += 32) G[i + j * ld] -= l * G[k + j * ld];
    }
    __syncthreads();
  }
}

// Register-resident versions of the two elimination chains (n <= 32 KC and
// n <= KR * warps): thread (warp w, lane l) keeps the entries (r, c),
// r = w + k * warps, c = l + 32 m, in registers for the whole factorization.
// Step j needs only row j from other threads: its owner publishes it into a
// double-buffered shared row right after updating it in step j - 1, so a
// step is one barrier, one reciprocal and register FMAs (no shared-memory
// round trip per entry).
template <int KR, int KC>
__device__ void chol_inv_regs(double* A, double* X, int n, int ld, double* dg, int* fail) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  __shared__ double rowbuf[2][32 * KC];
  __shared__ double s_d[32 * KC];
  double v[KR][KC];
#pragma unroll
  for (int k = 0; k < KR; ++k)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int r = wid + k * nw, c = lane + 32 * m;
      v[k][m] = (r < n && c < n && c >= r) ? A[r + c * ld] : 0.0;  // I part: identity minus its diagonal
    }
  if (wid == 0)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[0][lane + 32 * m] = v[0][m];
  __syncthreads();
  int bad = 0;
  int nxw = 1 % nw, nxk = 1 / nw;  // owner (warp, slot) of row j + 1, advanced per step (no integer division)
  for (int j = 0; j < n; ++j) {
    const double* rj = rowbuf[j & 1];
    // every shared read of the step is issued before the reciprocal
    const double d = rj[j];
    double tk[KR], aj[KC];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = wid + k * nw;
      tk[k] = (r > j && r < n) ? rj[r] : 0.0;
    }
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int c = lane + 32 * m;
      aj[m] = c == j ? 1.0 : (c < n ? rj[c] : 0.0);
    }
    bad |= !(d > 0.0);
    const double rd = d > 0.0 ? 1.0 / d : 1.0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = wid + k * nw;
      if (r > j && r < n) {
        const double t = tk[k] * rd;  // U(j, r)
#pragma unroll
        for (int m = 0; m < KC; ++m) {
          const int c = lane + 32 * m;
          if (c < n && (c >= r || c <= j)) v[k][m] -= t * aj[m];
        }
      }
    }
    if (j + 1 < n && wid == nxw) {
#pragma unroll
      for (int k = 0; k < KR; ++k)
        if (k == nxk)
#pragma unroll
          for (int m = 0; m < KC; ++m) rowbuf[(j + 1) & 1][lane + 32 * m] = v[k][m];
    }
    if (++nxw == nw) {
      nxw = 0;
      ++nxk;
    }
    if (tid == 0) s_d[j] = d;
    __syncthreads();
  }
  if (tid == 0 && bad) *fail = 1;
  for (int j = tid; j < n; j += blockDim.x) dg[j] = s_d[j] > 0.0 ? sqrt(s_d[j]) : 1.0;
  // R(r, c) = sqrt(d_r) U(r, c) (upper), X = R^{-1}: X(c, r) = (U^{-T})(r, c) / sqrt(d_r)
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int r = wid + k * nw;
    if (r < n) {
      const double dr = s_d[r];
      const double sq = dr > 0.0 ? sqrt(dr) : 1.0, rs = 1.0 / sq, rd = dr > 0.0 ? 1.0 / dr : 1.0;
#pragma unroll
      for (int m = 0; m < KC; ++m) {
        const int c = lane + 32 * m;
        if (c >= n) continue;
        if (c < r) {
          X[c + r * ld] = v[k][m] * rs;
        } else if (c == r) {
          X[r + r * ld] = rs;
          A[r + r * ld] = sq;
        } else {
          X[c + r * ld] = 0.0;
          A[r + c * ld] = (v[k][m] * rd) * sq;
        }
      }
    }
  }
  __syncthreads();
}

template <int KR, int KC>
__device__ void sign_reconstruct_regs(double* G, int n, int ld, int rows, double* sgn) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  __shared__ double rowbuf[2][32 * KC];
  double v[KR][KC];
#pragma unroll
  for (int k = 0; k < KR; ++k)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int r = wid + k * nw, c = lane + 32 * m;
      v[k][m] = (r < n && c < n) ? G[r + c * ld] : 0.0;
    }
  if (wid == 0)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[0][lane + 32 * m] = v[0][m];
  __syncthreads();
  int nxw = 1 % nw, nxk = 1 / nw;  // owner of row k0 + 1
  for (int k0 = 0; k0 < n; ++k0) {
    const double* rk = rowbuf[k0 & 1];
    const double gkk = rk[k0];
    double ak[KC];
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int c = lane + 32 * m;
      ak[m] = c < n ? rk[c] : 0.0;
    }
    const int mk = k0 >> 5, lk = k0 & 31;
    double gik[KR];  // G(r, k0): lane lk of this warp holds it
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      double x = 0.0;
#pragma unroll
      for (int m = 0; m < KC; ++m)
        if (m == mk) x = v[k][m];
      gik[k] = __shfl_sync(0xffffffffu, x, lk);
    }
    const double sk = (gkk > 0.0) != (k0 == rows - 1) ? -1.0 : 1.0;
    const double rd = 1.0 / (sk * gkk - 1.0);
    if (tid == 0) sgn[k0] = sk;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = wid + k * nw;
      if (r > k0 && r < n) {
        const double l = (sk * gik[k]) * rd;
#pragma unroll
        for (int m = 0; m < KC; ++m) {
          const int c = lane + 32 * m;
          if (c > k0 && c < n) v[k][m] -= l * ak[m];
        }
      }
    }
    if (k0 + 1 < n && wid == nxw) {
#pragma unroll
      for (int k = 0; k < KR; ++k)
        if (k == nxk)
#pragma unroll
          for (int m = 0; m < KC; ++m) rowbuf[(k0 + 1) & 1][lane + 32 * m] = v[k][m];
    }
    if (++nxw == nw) {
      nxw = 0;
      ++nxk;
    }
    __syncthreads();
  }
}

__device__ void sign_reconstruct(double* G, int n, int ld, int rows, double* sgn) {
  const int nw = blockDim.x >> 5;
  if (n <= 32 && n <= 4 * nw) sign_reconstruct_regs<4, 1>(G, n, ld, rows, sgn);
  else if (n <= 64 && n <= 8 * nw) sign_reconstruct_regs<8, 2>(G, n, ld, rows, sgn);
  else if (n <= 96 && n <= 12 * nw) sign_reconstruct_regs<12, 3>(G, n, ld, rows, sgn);
  else sign_reconstruct_smem(G, n, ld, rows, sgn);
}

__device__ void chol_inv(double* A, double* X, int n, int ld, double* dg, int* fail) {
  const int nw = blockDim.x >> 5;
  if (n <= 32 && n <= 4 * nw) chol_inv_regs<4, 1>(A, X, n, ld, dg, fail);
  else if (n <= 64 && n <= 8 * nw) chol_inv_regs<8, 2>(A, X, n, ld, dg, fail);
  else if (n <= 96 && n <= 12 * nw) chol_inv_regs<12, 3>(A, X, n, ld, dg, fail);
  else chol_inv_small(A, X, n, ld, dg, fail);
}

// The same CholeskyQR2 + Householder sign reconstruction as cqr2_kernel,
// spread over a cooperative grid: each CTA keeps a contiguous chunk of rows
// of V in shared memory (fp64) for both passes; the Gram is accumulated per
// CTA in 4x4 register blocks of the upper triangle and reduced in fixed CTA
// order (deterministic); CTA 0 factors it (Cholesky, R^{-1}) while the grid
// waits; V <- V R^{-1} is parallel over (row, column). Workspace (doubles):
// part [G][NB(NB+1)/2][16] | Gram n*n | R^{-1} n*n | top n*n | sgn n | dg 2n.
constexpr int kCqrCoopThreads = 256;

template <typename T>
struct CqrCoopArgs {
  const T* Y;
  T* Q;
  int I, n, rows_per;  // rows_per: chunk of rows per CTA
  double* work;
  GridBarrier* bar;
  int* status;
  int* rank_warning;
  unsigned long long* prof;  // optional phase stamps (RCPG_PROFILE_QR)
};

__device__ __forceinline__ void cqr_stamp(unsigned long long* prof, int slot) {
  if (prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    prof[slot] = t;
  }
}

__host__ __device__ inline int cqr_nb(int n) { return (n + 3) / 4; }

template <typename T>
__global__ void __launch_bounds__(kCqrCoopThreads) cqr2_coop_kernel(CqrCoopArgs<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = p.n, NB = cqr_nb(n), n4 = 4 * NB, NP = NB * (NB + 1) / 2;
  const int ld = p.rows_per + 1;                                 // odd column stride: fewer bank conflicts
  double* V = reinterpret_cast<double*>(smem_raw);              // [n4][ld] own rows, column-major
  double* Ri = V + i64(n4) * ld;                                // n x n R^{-1} (upper), or scratch
  __shared__ int s_fail;
  __shared__ double dg_loc[2 * kMaxPanelCols];  // diagonals of R1, R2 (this CTA's copy)
  const int tid = threadIdx.x, nt = blockDim.x;
  const int r0 = blockIdx.x * p.rows_per;
  const int rows = max(0, min(p.rows_per, p.I - r0));
  double* part = p.work;
  double* Gf = part + i64(gridDim.x) * NP * 16;
  double* Rg = Gf + n * n;
  double* top = Rg + n * n;
  double* sgn = top + n * n;
  double* dg = sgn + n;

  for (int e = tid; e < n4 * ld; e += nt) {
    const int i = e % ld, j = e / ld;
    V[e] = (i < rows && j < n) ? double(p.Y[(r0 + i) + i64(j) * p.I]) : 0.0;
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  cqr_stamp(p.prof, 0);

  for (int pass = 0; pass < 2; ++pass) {
    // 1. partial Gram of own rows, 4x4 blocks (A <= B) of the upper triangle
    for (int pb = tid; pb < NP; pb += nt) {
      int B = int((sqrt(8.0 * pb + 1.0) - 1.0) * 0.5);
      while (B * (B + 1) / 2 > pb) --B;
      while ((B + 1) * (B + 2) / 2 <= pb) ++B;
      const int A = pb - B * (B + 1) / 2;
      double acc[4][4] = {};
      const double* va = V + i64(4 * A) * ld;
      const double* vb = V + i64(4 * B) * ld;
      for (int i = 0; i < rows; ++i) {
        double x[4], y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[u] = va[u * ld + i];
          y[u] = vb[u * ld + i];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] += x[u] * y[v];
      }
      double* dst = part + (i64(blockIdx.x) * NP + pb) * 16;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) dst[u * 4 + v] = acc[u][v];
    }
    cqr_stamp(p.prof, 1 + 5 * pass);
    grid_sync(p.bar);
    // 2. reduce the partials in CTA order; scatter into the full symmetric Gram
    for (i64 e = blockIdx.x * i64(nt) + tid; e < i64(NP) * 16; e += i64(gridDim.x) * nt) {
      const int pb = int(e / 16), uv = int(e % 16);
      double s = 0.0;
      for (int q = 0; q < int(gridDim.x); ++q) s += ldcg(&part[(i64(q) * NP + pb) * 16 + uv]);
      int B = int((sqrt(8.0 * pb + 1.0) - 1.0) * 0.5);
      while (B * (B + 1) / 2 > pb) --B;
      while ((B + 1) * (B + 2) / 2 <= pb) ++B;
      const int A = pb - B * (B + 1) / 2;
      const int a = 4 * A + uv / 4, b = 4 * B + uv % 4;
      if (a < n && b < n && a <= b) {
        Gf[a + b * n] = s;
        Gf[b + a * n] = s;
      }
    }
    cqr_stamp(p.prof, 2 + 5 * pass);
    grid_sync(p.bar);
    cqr_stamp(p.prof, 13 + pass);
    // 3. every CTA factors the (identical) Gram itself: upper Cholesky, R^{-1}
    //    (deterministic, so all CTAs agree; no barrier, nobody waits on CTA 0)
    const int ldn = n + 1;
    double* As = Ri;              // n x ldn Gram -> R
    double* Xs = Ri + n * ldn;    // n x ldn R^{-1}
    for (int e = tid; e < n * n; e += nt) As[(e % n) + (e / n) * ldn] = ldcg(&Gf[e]);
    __syncthreads();
    chol_inv(As, Xs, n, ldn, dg_loc + pass * n, &s_fail);
    if (blockIdx.x == 0)
      for (int j = tid; j < n; j += nt) dg[pass * n + j] = dg_loc[pass * n + j];
    cqr_stamp(p.prof, 3 + 5 * pass);
    if (s_fail) {  // Cholesky broke down (same verdict in every CTA): Householder runs instead
      if (blockIdx.x == 0 && tid == 0) *p.status = 1;
      return;
    }
    // 4. V <- V R^{-1} (own rows): out(i, j) = sum_{k <= j} V(i, k) Ri(k, j)
    {
      double* out = Xs + n * ldn;  // [n][ld] staging, then copied back over V
      for (int e = tid; e < n * rows; e += nt) {
        const int i = e % rows, j = e / rows;
        double s = 0.0;
        for (int k = 0; k <= j; ++k) s += V[k * ld + i] * Xs[k + j * ldn];
        out[j * ld + i] = s;
      }
      __syncthreads();
      for (int e = tid; e < n * rows; e += nt) {
        const int i = e % rows, j = e / rows;
        V[j * ld + i] = out[j * ld + i];
      }
      __syncthreads();
    }
    cqr_stamp(p.prof, 4 + 5 * pass);
  }
  // conditioning guard (CholeskyQR2 only well inside its stable range); every
  // CTA evaluates it on its own (identical) diagonals
  {
    __shared__ int s_bad;
    if (tid == 0) {
      double mx = 0.0, mn = INFINITY;
      for (int j = 0; j < n; ++j) {
        mx = fmax(mx, dg_loc[j]);
        mn = fmin(mn, dg_loc[j]);
      }
      s_bad = (!(mn > 0.0) || mx / mn > 1e6) ? 1 : 0;
    }
    __syncthreads();
    if (s_bad) {
      if (blockIdx.x == 0 && tid == 0) *p.status = 1;
      return;
    }
  }
  // rows < n of Q2 -> top (for the sign reconstruction)
  for (int e = tid; e < n * rows; e += nt) {
    const int i = e % rows, j = e / rows;
    if (r0 + i < n) top[(r0 + i) + j * n] = V[j * ld + i];
  }
  grid_sync(p.bar);
  cqr_stamp(p.prof, 11);
  // every CTA reconstructs the Householder signs from the top block itself
  const int ldn = n + 1;
  double* Gs = Ri;
  __shared__ double sg[kMaxPanelCols];
  for (int e = tid; e < n * n; e += nt) Gs[(e % n) + (e / n) * ldn] = ldcg(&top[e]);
  __syncthreads();
  sign_reconstruct(Gs, n, ldn, p.I, sg);
  cqr_stamp(p.prof, 12);
  if (blockIdx.x == 0 && tid == 0) {
    T dmax = T(0), dmin = T(INFINITY);
    for (int j = 0; j < n; ++j) {
      const T d = T(dg[j] * dg[n + j]);
      dmax = d > dmax ? d : dmax;
      dmin = d < dmin ? d : dmin;
    }
    if (p.rank_warning) *p.rank_warning = (dmax == T(0)) || (dmin <= T(p.I) * Traits<T>::eps * dmax);
    *p.status = 0;
  }
  for (int e = tid; e < n * rows; e += nt) {
    const int i = e % rows, j = e / rows;
    p.Q[(r0 + i) + i64(j) * p.I] = T(V[j * ld + i] * sg[j]);
  }
}

// CholeskyQR2 + Householder sign reconstruction with Y resident in shared
// memory (I * n doubles): everything after the load is on-chip.
template <typename T>
__global__ void __launch_bounds__(kCqrThreads) cqr2_smem_kernel(const T* __restrict__ Y, T* __restrict__ Q, int I,
                                                                int n, int* status, int* rank_warning) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* V = reinterpret_cast<double*>(smem_raw);  // I x n
  double* G = V + i64(I) * n;                        // n x n
  double* Rm = G + n * n;                            // n x n upper
  double* dg = Rm + n * n;                           // [2][n]
  double* sgn = dg + 2 * n;                          // [n]
  __shared__ int s_fail;
  __shared__ double s_piv;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < I * n; e += nt) V[e] = double(Y[e]);
  if (tid == 0) s_fail = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    // G = V^T V: warp per (a, b) pair, lanes over rows (conflict-free: a
    // column of V is contiguous; lanes striding a row would all hit one bank)
    for (int pr = wid; pr < n * (n + 1) / 2; pr += nw) {
      int b = int((sqrt(8.0 * pr + 1.0) - 1.0) * 0.5);
      while (b * (b + 1) / 2 > pr) --b;
      while ((b + 1) * (b + 2) / 2 <= pr) ++b;
      const int a = pr - b * (b + 1) / 2;
      const double* va = V + i64(a) * I;
      const double* vb = V + i64(b) * I;
      double s = 0.0;
      for (int i = lane; i < I; i += 32) s += va[i] * vb[i];
      s = warp_sum(s);
      if (lane == 0) {
        G[a + b * n] = s;
        G[b + a * n] = s;
      }
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {  // upper Cholesky G = R^T R
      if (tid == 0) {
        double d = G[j + j * n];
        for (int k = 0; k < j; ++k) d -= Rm[k + j * n] * Rm[k + j * n];
        if (!(d > 0.0)) s_fail = 1;
        s_piv = d > 0.0 ? sqrt(d) : 1.0;
        Rm[j + j * n] = s_piv;
        dg[pass * n + j] = s_piv;
      }
      __syncthreads();
      const double dj = s_piv;
      for (int c = j + 1 + tid; c < n; c += nt) {
        double s = G[j + c * n];
        for (int k = 0; k < j; ++k) s -= Rm[k + j * n] * Rm[k + c * n];
        Rm[j + c * n] = s / dj;
      }
      __syncthreads();
    }
    if (s_fail) break;
    for (int i = tid; i < I; i += nt)  // V <- V R^{-1}, in place, row by row
      for (int j = 0; j < n; ++j) {
        double v = V[i + i64(j) * I];
        for (int k = 0; k < j; ++k) v -= V[i + i64(k) * I] * Rm[k + j * n];
        V[i + i64(j) * I] = v / Rm[j + j * n];
      }
    __syncthreads();
  }
  if (!s_fail && tid == 0) {
    double mx = 0.0, mn = INFINITY;
    for (int j = 0; j < n; ++j) {
      mx = fmax(mx, dg[j]);
      mn = fmin(mn, dg[j]);
    }
    if (!(mn > 0.0) || mx / mn > 1e6) s_fail = 1;
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0) *status = 1;
    return;
  }
  for (int e = tid; e < n * n; e += nt) G[e] = V[(e % n) + i64(e / n) * I];
  __syncthreads();
  for (int k = 0; k < n; ++k) {  // sign reconstruction (modified LU of Q_top - S)
    if (tid == 0) {
      sgn[k] = (G[k + k * n] > 0.0) != (k == I - 1) ? -1.0 : 1.0;  // square panel: see cqr2_kernel
      if (sgn[k] < 0.0)
        for (int i = 0; i < n; ++i) G[i + k * n] = -G[i + k * n];
      G[k + k * n] -= 1.0;
    }
    __syncthreads();
    const double dkk = G[k + k * n];
    for (int j = k + 1 + wid; j < n; j += nw)
      for (int i = k + 1 + lane; i < n; i += 32) G[i + j * n] -= (G[i + k * n] / dkk) * G[k + j * n];
    __syncthreads();
  }
  for (int j = wid; j < n; j += nw)
    for (int i = lane; i < I; i += 32) Q[i + i64(j) * I] = T(V[i + i64(j) * I] * sgn[j]);
  if (tid == 0) {
    T dmax = T(0), dmin = T(INFINITY);
    for (int j = 0; j < n; ++j) {
      const T d = T(dg[j] * dg[n + j]);
      dmax = d > dmax ? d : dmax;
      dmin = d < dmin ? d : dmin;
    }
    if (rank_warning) *rank_warning = (dmax == T(0)) || (dmin <= T(I) * Traits<T>::eps * dmax);
    *status = 0;
  }
}

int pick_grid(i64 J, int n, int maxc) {
  // ~4K panel entries per CTA: the per-step update is latency bound
  const i64 want = ceil_div(J * n, 4096);
  return int(std::max<i64>(1, std::min<i64>(want, maxc)));
}

size_t smem_lu_bytes(i64 I, int n, size_t tsize) { return size_t(I) * n * tsize + size_t(I) * sizeof(int); }

}  // namespace

void init_row_keys(const KoldaMap& km, i64 J, i64 R, i64* keys, cudaStream_t st) {
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(J, 256), 148 * 8)));
  init_row_keys_kernel<<<blocks, 256, 0, st>>>(km, J, R, keys);
  count_launch();
  RCPG_LAUNCHED();
}

// Panel-resident LU (plu_resident_kernel) when the panel fits the SMs'
// shared memory plus RC register columns: the smallest grid that fits, one
// row per thread when possible. Returns false when it does not fit.
template <typename T>
bool plu_resident(T* A, T* Z, i64 J, i64 R, int n, int r, const KoldaMap& km, FactorWork& w, cudaStream_t st) {
  const int nsm = std::min(device_caps().num_sms, 32 * kResKeyLoads);
  if (J < 2 || J > i64(nsm) * 2 * 1024 || nsm > w.max_blocks) return false;
  using K = void (*)(LuResArgs<T>);
  struct V {
    int rc, rpt;
    K k;
  };
  static const V vars[] = {{0, 1, plu_resident_kernel<T, 0, 1, false>}, {4, 1, plu_resident_kernel<T, 4, 1, false>},
                           {8, 1, plu_resident_kernel<T, 8, 1, false>}, {0, 2, plu_resident_kernel<T, 0, 2, false>},
                           {4, 2, plu_resident_kernel<T, 4, 2, false>}, {8, 2, plu_resident_kernel<T, 8, 2, false>}};
  static const struct Lim {
    size_t smem[6];
    int regs[6];
  } lim = [] {
    Lim l{};
    for (int i = 0; i < 6; ++i) {
      l.smem[i] = enable_max_dyn_smem(vars[i].k);
      cudaFuncAttributes fa{};
      RCPG_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(vars[i].k)));
      l.regs[i] = fa.numRegs;
    }
    return l;
  }();
  // Rows per CTA: ~512 when that many CTAs are resident (71680 x 70 fp32 821 -> 715 us,
  // 40000 x 80 fp32 921 -> 834 us), else as few CTAs as fit; fewer rows (256, 128)
  // lose (tools/lu_resident_rows.py). RCPG_LU_RES_ROWS overrides the target (A/B).
  const char* rr = std::getenv("RCPG_LU_RES_ROWS");
  i64 res_rows = rr ? std::max(32, atoi(rr)) : 512;
  if (rr == nullptr && ceil_div(J, res_rows) > nsm) res_rows = 0;
  for (int rpt = 1; rpt <= 2; ++rpt)
    for (i64 G = std::max<i64>({i64(1), ceil_div(J, i64(1024) * rpt), res_rows ? ceil_div(J, res_rows) : 1}); G <= nsm; ++G) {
      const int chunk = int(ceil_div(J, G));
      const int nt = int(ceil_div(ceil_div(i64(chunk), rpt), 32) * 32);
      for (int i = 0; i < 6; ++i) {
        if (vars[i].rpt != rpt) continue;
        const int rc = vars[i].rc;
        const int ns = std::max(0, n - rc);
        if (nt > lu_res_max_threads(rc, rpt) || nt * lim.regs[i] > 65536) continue;
        if (rc > 0 && n - ns > rc) continue;
        const size_t smem = ((size_t(ns) * chunk * sizeof(T) + 15) & ~size_t(15)) + size_t(chunk) * sizeof(i64);
        if (smem > lim.smem[i]) continue;
        if (ceil_div(J, i64(chunk)) != G) continue;  // every CTA owns rows
        init_row_keys(km, J, R, w.keys, st);
        LuResArgs<T> a{A, Z, J, R, n, r, ns, chunk, w.keys, km, reinterpret_cast<Cand<T>*>(w.cands),
                       reinterpret_cast<T*>(w.part), w.bar, w.info, w.prof};
        launch_coop(vars[i].k, int(G), nt, smem, st, a);
        RCPG_LAUNCHED();
        if (w.prof) {
          unsigned long long h[8];
          RCPG_CUDA(cudaMemcpyAsync(h, w.prof, sizeof(h), cudaMemcpyDeviceToHost, st));
          RCPG_CUDA(cudaStreamSynchronize(st));
          if (h[4])
            fprintf(stderr, "[rcpg lu resident] J=%lld n=%d G=%d nt=%d rc=%d rpt=%d: reduce+publish %.2f  barrier %.2f  "
                            "pick+book %.2f  update %.2f us/step\n", (long long)J, n, int(G), nt, rc, rpt,
                    h[0] / 1e3 / h[4], h[1] / 1e3 / h[4], h[2] / 1e3 / h[4], h[3] / 1e3 / h[4]);
        }
        return true;
      }
    }
  return false;
}

// The same resident LU on one thread-block cluster (2..16 CTAs, panel in
// their shared memory): the smallest cluster that holds the panel with one
// row per thread, else two. Returns false when no cluster holds it.
template <typename T>
bool plu_resident_cluster(T* A, T* Z, i64 J, i64 R, int n, int r, const KoldaMap& km, FactorWork& w,
                          cudaStream_t st) {
  using K = void (*)(LuResArgs<T>);
  static const K k1 = plu_resident_kernel<T, 0, 1, true>, k2 = plu_resident_kernel<T, 0, 2, true>;
  static const struct Lim {
    size_t smem1, smem2;
    bool nonportable;
  } lim = [] {
    Lim l{};
    l.smem1 = enable_max_dyn_smem(k1);
    l.smem2 = enable_max_dyn_smem(k2);
    l.nonportable = cudaFuncSetAttribute(k1, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
                    cudaFuncSetAttribute(k2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    return l;
  }();
  const int csmax = lim.nonportable ? 16 : 8;
  for (int rpt = 1; rpt <= 2; ++rpt)
    for (int cs = 2; cs <= csmax; ++cs) {
      const int chunk = int(ceil_div(J, i64(cs)));
      const int nt = int(ceil_div(ceil_div(i64(chunk), rpt), 32) * 32);
      if (nt > 1024 || ceil_div(J, i64(chunk)) != cs) continue;
      const size_t smem = ((size_t(n) * chunk * sizeof(T) + 15) & ~size_t(15)) + size_t(chunk) * sizeof(i64);
      if (smem > (rpt == 1 ? lim.smem1 : lim.smem2)) continue;
      init_row_keys(km, J, R, w.keys, st);
      LuResArgs<T> a{A, Z, J, R, n, r, n, chunk, w.keys, km, nullptr, nullptr, nullptr, w.info, nullptr};
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(nt);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      RCPG_CUDA(cudaLaunchKernelEx(&cfg, rpt == 1 ? k1 : k2, a));
      count_launch();
      return true;
    }
  return false;
}

// Launch plu_reg_kernel<T, NC, RPT, CL> on the smallest CTA count (1, or a
// cluster of 2..16) whose threads hold the panel with RPT rows each.
template <typename T, int NC, int RPT>
bool plu_reg_try(T* A, T* Z, i64 J, i64 R, int n, const KoldaMap& km, FactorWork& w, cudaStream_t st, int force_cs) {
  constexpr int maxt = lu_reg_max_threads<T, NC, RPT>();
  static const bool nonportable = [] {
    return cudaFuncSetAttribute(plu_reg_kernel<T, NC, RPT, true>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                1) == cudaSuccess;
  }();
  const int max_cs = nonportable ? 16 : 8;
  for (int cs = 1; cs <= max_cs; cs *= 2) {
    if (force_cs > 0 && cs != force_cs) continue;
    const i64 per = ceil_div(J, i64(cs) * RPT);
    if (per > maxt) continue;
    const int nt = int(std::max<i64>(32, ceil_div(per, 32) * 32));
    if (cs == 1) {
      plu_reg_kernel<T, NC, RPT, false><<<1, nt, 0, st>>>(A, Z, int(J), n, R, km, w.info);
    } else {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(nt);
      cfg.dynamicSmemBytes = 0;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      RCPG_CUDA(cudaLaunchKernelEx(&cfg, plu_reg_kernel<T, NC, RPT, true>, (const T*)A, Z, int(J), n, R, km,
                                   w.info));
    }
    count_launch();
    RCPG_LAUNCHED();
#ifdef RCPG_LU_REG_PROF
    unsigned long long h[8];
    RCPG_CUDA(cudaMemcpyFromSymbolAsync(h, g_lu_reg_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
    RCPG_CUDA(cudaStreamSynchronize(st));
    const double kk = double(h[6] ? h[6] : 1);
    fprintf(stderr, "[lu reg] J=%lld n=%d cs=%d nt=%d rpt=%d cycles/pivot: update %.0f  reduce+stage %.0f  bar1 %.0f  pick %.0f  bar2 %.0f  mult %.0f\n",
            (long long)J, n, cs, nt, RPT, h[0] / kk, h[1] / kk, h[2] / kk, h[3] / kk, h[4] / kk, h[5] / kk);
#endif
    return true;
  }
  return false;
}

// The register-resident LU for panels it holds (n <= 32 for double; 48 / 80
// for float), one row per thread first, two when one row per thread needs more
// than 16 CTAs. RCPG_LU_REG=0 disables it, RCPG_LU_REG_RPT / _CS force a shape,
// RCPG_LU_PATH=reg takes it for every panel it holds (parity tests).
template <typename T>
bool plu_reg(T* A, T* Z, i64 J, i64 R, int n, const KoldaMap& km, FactorWork& w, cudaStream_t st, bool all) {
  static const int env_mode = [] {
    const char* e = std::getenv("RCPG_LU_REG");
    return e ? atoi(e) : 1;
  }();
  const int mode = all ? 2 : env_mode;
  static const int force_rpt = [] {
    const char* e = std::getenv("RCPG_LU_REG_RPT");
    return e ? atoi(e) : 0;
  }();
  static const int force_cs = [] {
    const char* e = std::getenv("RCPG_LU_REG_CS");
    return e ? atoi(e) : 0;
  }();
  if (mode == 0 || J >= 65536) return false;  // row index in the low 16 bits of the pivot key
  auto go = [&](auto nc_tag) {
    constexpr int NC = decltype(nc_tag)::value;
    if (force_rpt != 2 && plu_reg_try<T, NC, 1>(A, Z, J, R, n, km, w, st, force_cs)) return true;
    if (force_rpt != 1 && plu_reg_try<T, NC, 2>(A, Z, J, R, n, km, w, st, force_cs)) return true;
    return false;
  };
  // where it beats the one-CTA / cluster kernels (tools/gpu_s4c.sh): fp64 up to
  // 32 columns (12000 x 30 161 -> 136 us, 400 x 30 70 -> 67); fp32 only for the
  // 48-column panels of 1024+ rows (3072 x 48 178 -> 162 us), the 70-80 column
  // ones lose (1024 x 70 241 -> 299). RCPG_LU_REG=2 takes every panel it holds.
  if constexpr (sizeof(T) == 8) {
    if (n <= 32) return go(std::integral_constant<int, 32>{});
  } else {
    if (n <= 48 && (J >= 1024 || mode == 2)) return go(std::integral_constant<int, 48>{});
    if (n <= 80 && mode == 2) return go(std::integral_constant<int, 80>{});
  }
  return false;
}

template <typename T>
int plu_basis(T* A, T* Z, i64 J, i64 R, int n, const KoldaMap& km, FactorWork& w, cudaStream_t st) {
  check_arg(n <= kMaxPanelCols, "plu_basis: panel wider than supported");
  const int r = int(std::min<i64>(J, n));
  // one CTA, rows owned by threads, swaps bookkept
  static const size_t oc_lim = enable_max_dyn_smem(plu_onchip_kernel<T>);
  const size_t oc_smem = size_t(J) * n * sizeof(T) + 8 + 2 * size_t(J) * sizeof(int);
  // A/B testing: RCPG_LU_PATH = reg | onchip | rcluster | cluster | resident |
  // coop starts the chain (rows in registers -> one CTA -> one cluster, swaps
  // bookkept -> one cluster, Eigen's physical swaps -> panel resident in the
  // SMs -> grid) further down
  const char* lp = std::getenv("RCPG_LU_PATH");
  const std::string lpath = lp ? lp : "";
  // from ~640 rows an 8-CTA cluster beats one CTA (C2's 900 x 30 W: 156 -> 110 us;
  // its 400 x 30 samples stay faster on one CTA: 69 vs 90 us; tools/ab_r2b.sh)
  static const i64 oc_rows = [] {
    const char* e = std::getenv("RCPG_LU_ONCHIP_ROWS");
    return e ? i64(atoll(e)) : i64(640);
  }();
  if ((lpath.empty() || lpath == "reg") && plu_reg<T>(A, Z, J, R, n, km, w, st, lpath == "reg")) return r;
  if (oc_smem <= oc_lim && J * i64(n) < (i64(1) << 31) && (lpath.empty() || lpath == "onchip") && J < oc_rows) {
    // W row lanes (whole warps) x tpr column groups, at most 1024 threads
    const int W = int(std::min<i64>(1024, ceil_div(J, 32) * 32));
    // column groups per row for short panels: 128 x 48 f32 (C4's samples) 100 -> 76 us
    // with 4, no gain from 400 rows up (tools/gpu_s3ac.sh); RCPG_LU_TPR overrides
    const char* tp = std::getenv("RCPG_LU_TPR");
    const int tpr = tp ? std::max(1, std::min(atoi(tp), 1024 / W)) : (J <= 256 ? std::min(4, 1024 / W) : 1);
    plu_onchip_kernel<T><<<1, W * tpr, oc_smem, st>>>(A, Z, int(J), n, R, km, W, w.info);
    count_launch();
    RCPG_LAUNCHED();
    return r;
  }
  // one thread-block cluster, panel resident, swaps bookkept (A/B only: its
  // fixed per-pivot cost loses to the swap kernel below at these sizes)
  if (lpath == "rcluster" && plu_resident_cluster<T>(A, Z, J, R, n, r, km, w, st)) return r;
  // on-chip paths: one CTA, or one cluster of up to 16 CTAs
  static const size_t lu_lim1 = enable_max_dyn_smem(plu_cluster_kernel<T, false>);
  static const size_t lu_lim = std::min(enable_max_dyn_smem(plu_cluster_kernel<T, true>),
                                        enable_max_dyn_smem(plu_cluster_kernel<T, true, 512>));
  static const bool nonportable = [] {
    return cudaFuncSetAttribute(plu_cluster_kernel<T, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
               cudaSuccess &&
           cudaFuncSetAttribute(plu_cluster_kernel<T, true, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
               cudaSuccess;
  }();
  // When the panel needs a cluster, ~128 rows per CTA (at least 8 CTAs) beat the
  // smallest cluster that fits: 1024 x 70 fp32 (C3's samples) 403 us on 2 CTAs, 290
  // on 4, 250 on 8, 256 on 16; 4096 x 48 fp32 354 / 239 / 195 us on 4 / 8 / 16
  // (tools/lu_cluster_sizes.py, tools/lu_onchip_vs_cluster.py; same bits on every
  // size). RCPG_LU_MINCS overrides the smallest size tried (A/B).
  const char* mcs = std::getenv("RCPG_LU_MINCS");
  const int max_cs = nonportable ? 16 : 8;
  int want_cs = 8;
  while (want_cs < max_cs && J > 128 * i64(want_cs)) want_cs *= 2;
  // a panel the one-CTA kernel declined for size goes straight to the 8-CTA cluster
  const int min_cs = mcs ? std::max(1, atoi(mcs)) : (J >= oc_rows && oc_smem <= oc_lim ? 8 : 1);
  for (int cs = 1; cs <= max_cs && lpath != "coop" && lpath != "resident"; cs *= 2) {
    if (cs < min_cs || (mcs == nullptr && cs > 1 && cs < want_cs)) continue;
    const int chunk = int(ceil_div(J, cs));
    const size_t smem = size_t(chunk) * n * sizeof(T) + 2 * size_t(n) * sizeof(T) + size_t(chunk) * sizeof(int) + 16;
    if (smem > (cs == 1 ? lu_lim1 : lu_lim) - 1024) continue;
    if (cs == 1) {
      plu_cluster_kernel<T, false><<<1, kSmemLuThreads, smem, st>>>(A, Z, int(J), n, chunk, R, km, w.info);
      count_launch();
      RCPG_LAUNCHED();
      return r;
    }
    // 512 threads from 128 rows per CTA (12000 x 30 f64 on 16 CTAs 180 -> 161 us,
    // 10000 x 80 f32 649 -> 534 us), 256 below (900 x 30: 95 vs 98 us); tools/gpu_s3q.sh
    const bool wide = chunk >= 128;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(wide ? 512 : kSmemLuThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (wide)
      RCPG_CUDA(cudaLaunchKernelEx(&cfg, plu_cluster_kernel<T, true, 512>, (const T*)A, Z, int(J), n, chunk, R, km,
                                   w.info));
    else
      RCPG_CUDA(cudaLaunchKernelEx(&cfg, plu_cluster_kernel<T, true>, (const T*)A, Z, int(J), n, chunk, R, km, w.info));
    count_launch();
    return r;
  }
  // panel resident in the SMs (grid of up to one CTA per SM, one grid barrier per pivot)
  if (lpath != "coop" && plu_resident<T>(A, Z, J, R, n, r, km, w, st)) return r;
  init_row_keys(km, J, R, w.keys, st);
  // chunks of 1 row group (blockDim * V rows) per claim; 2 on panels of 4M+ rows
  // (fewer claims on the one counter)
  LuArgs<T> a{A, Z, J, R, n, r, w.keys, km, reinterpret_cast<Cand<T>*>(w.cands), w.bar, w.info, w.prof,
              std::getenv("RCPG_LU_NODELAY") == nullptr ? 1 : 0, w.ctr, 0};
  RCPG_CUDA(cudaMemsetAsync(w.ctr, 0, size_t(n + 1) * sizeof(unsigned), st));
  // about one group of V panel rows per thread; the per-step work is latency bound
  auto run = [&](auto kern, int V) {
    const int maxc = max_coop_blocks(kern, kLuThreads, 0);
    const int G = int(std::max<i64>(1, std::min<i64>({ceil_div(J, i64(kLuThreads) * V), i64(maxc), i64(w.max_blocks)})));
    const i64 cgr = J >= (i64(1) << 22) ? 2 : 1;
    a.chunk_groups = ceil_div(J, i64(kLuThreads) * V * cgr) >= 2 * i64(G) ? int(cgr) : 0;
    launch_coop(kern, G, kLuThreads, 0, st, a);
  };
  constexpr int VV = 16 / int(sizeof(T));
  const bool vec = std::getenv("RCPG_LU_SCALAR") == nullptr && J % VV == 0 && R % VV == 0 &&
                   reinterpret_cast<uintptr_t>(A) % 16 == 0 && reinterpret_cast<uintptr_t>(Z) % 16 == 0;
  if (vec)
    run(plu_coop_kernel<T, VV>, VV);
  else
    run(plu_coop_kernel<T, 1>, 1);
  return r;
}

template <typename T>
int thin_qr(T* A, T* Q, i64 J, i64 R, int n, const KoldaMap& km, FactorWork& w, int* rank_warning_dev,
            cudaStream_t st) {
  check_arg(n <= kMaxPanelCols, "thin_qr: panel wider than supported");
  const int r = int(std::min<i64>(J, n));
  const bool kolda_identity = (km.n_low == 0 && km.n_high == 1);
  const int* skip = nullptr;
  const size_t cq_smem = (2 * size_t(n) * n + 3 * size_t(n)) * sizeof(double);
  static const size_t cq_lim = enable_max_dyn_smem(cqr2_kernel<T>);
  static const size_t cqs_lim = enable_max_dyn_smem(cqr2_smem_kernel<T>);
  const size_t cqs_smem = (size_t(J) * n + 2 * size_t(n) * n + 3 * size_t(n)) * sizeof(double);
  // CholeskyQR2 over all SMs for panels too tall for one SM to factor quickly
  static const size_t cc_lim = enable_max_dyn_smem(cqr2_coop_kernel<T>);
  const int nb4 = 4 * cqr_nb(n);
  const char* qp = std::getenv("RCPG_QR_PATH");  // A/B testing: smem | global | coop | householder
  // faithful: the Householder QR with the reference's operation order only
  const std::string path = w.faithful_qr ? "householder" : (qp ? qp : "");
  bool done = false;
  if (R == J && kolda_identity && J >= n && w.cqr_work != nullptr && path != "smem" && path != "global" &&
      path != "householder" && (path == "coop" || J * n >= 4096)) {
    const int maxc = max_coop_blocks(cqr2_coop_kernel<T>, kCqrCoopThreads, cc_lim);
    // >= 32 rows per CTA; the chunk (plus 2 n x n fp64) must fit in shared memory
    int rows_per = int(std::max<i64>(32, ceil_div(J, i64(std::min(maxc, w.max_blocks)))));
    // V chunk [4 NB][rp + 1] | R, R^{-1} [n][n + 1] each | staging [n][rp + 1]  (doubles)
    auto smem_of = [&](int rp) {
      return (size_t(nb4) * (rp + 1) + 2 * size_t(n) * (n + 1) + size_t(n) * (rp + 1)) * 8;
    };
    const int G = int(ceil_div(J, i64(rows_per)));
    const size_t need = (size_t(G) * (cqr_nb(n) * (cqr_nb(n) + 1) / 2) * 16 + 3 * size_t(n) * n + 3 * size_t(n)) * 8;
    if (smem_of(rows_per) <= cc_lim && G <= maxc && need <= size_t(2) * w.cqr_rows * kMaxPanelCols * 8) {
      static unsigned long long* qprof = nullptr;
      const bool want_prof = std::getenv("RCPG_PROFILE_QR") != nullptr;
      if (want_prof && qprof == nullptr) RCPG_CUDA(cudaMalloc(&qprof, 16 * sizeof(unsigned long long)));
      CqrCoopArgs<T> a{A, Q, int(J), n, rows_per, w.cqr_work, w.bar, w.info + 2, rank_warning_dev,
                       want_prof ? qprof : nullptr};
      launch_coop(cqr2_coop_kernel<T>, G, kCqrCoopThreads, smem_of(rows_per), st, a);
      RCPG_LAUNCHED();
      if (want_prof) {
        unsigned long long h[16];
        RCPG_CUDA(cudaMemcpyAsync(h, qprof, sizeof(h), cudaMemcpyDeviceToHost, st));
        RCPG_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "[rcpg qr] %lldx%d G=%d rows/CTA=%d us:", (long long)J, n, G, rows_per);
        const char* nm[] = {"gram0", "red0", "chol0", "apply0", "-", "gram1", "red1", "chol1", "apply1", "top", "sign",
                            "sync0", "sync1"};
        const int at[] = {1, 2, 3, 4, -1, 6, 7, 8, 9, 11, 12, 13, 14};
        const int from[] = {0, 1, 2, 3, -1, 4, 6, 7, 8, 9, 11, 2, 7};
        for (int q = 0; q < 13; ++q)
          if (at[q] >= 0) fprintf(stderr, " %s %.1f", nm[q], (h[at[q]] - h[from[q]]) * 1e-3);
        fprintf(stderr, "\n");
      }
      skip = w.info + 2;
      done = true;
    }
  }
  if (done) {
  } else if (R == J && kolda_identity && J >= n && cqs_smem <= cqs_lim && path != "global" && path != "householder") {
    cqr2_smem_kernel<T><<<1, kCqrThreads, cqs_smem, st>>>(A, Q, int(J), n, w.info + 2, rank_warning_dev);
    count_launch();
    RCPG_LAUNCHED();
    skip = w.info + 2;
  } else if (R == J && kolda_identity && J >= n && J <= w.cqr_rows && cq_smem <= cq_lim && path != "householder") {
    cqr2_kernel<T><<<1, kCqrThreads, cq_smem, st>>>(A, Q, int(J), n, w.cqr_work, w.info + 2, rank_warning_dev);
    count_launch();
    RCPG_LAUNCHED();
    skip = w.info + 2;  // the Householder kernel below runs only if CholeskyQR2 declined
  }
  // (fp64 keeps householder_kernel below: CholeskyQR2's hand-over to it must give the same bits)
  if (!done && skip == nullptr && R == J && kolda_identity && (w.faithful_qr || path == "cluster_householder")) {
    // one cluster, panel in distributed shared memory (the faithful Householder of the fp32 configs)
    static const size_t hh_lim = enable_max_dyn_smem(householder_cluster_kernel<T>);
    static const bool hh_np = [] {
      return cudaFuncSetAttribute(householder_cluster_kernel<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
             cudaSuccess;
    }();
    const int max_cs = hh_np ? 16 : 8;
    const size_t fixed = (2 * (kMaxPanelCols + 1) + 2 * kMaxPanelCols) * sizeof(double) + 2 * kMaxPanelCols * sizeof(T);
    for (int cs = 1; cs <= max_cs; cs *= 2) {
      const int chunk = int(ceil_div(J, i64(cs)));
      static const int hh_rows = [] {  // rows per CTA targeted (A/B: RCPG_HH_ROWS)
        const char* e = std::getenv("RCPG_HH_ROWS");
        return e ? std::max(16, atoi(e)) : 64;
      }();
      if (cs < max_cs && chunk > hh_rows) continue;  // <= 64 rows per CTA: the largest cluster wins (1024 x 70: 16 CTAs 0.74 ms, 4 CTAs 1.45 ms)
      const size_t smem = fixed + size_t(chunk) * n * sizeof(T);
      if (smem > hh_lim - 1024) continue;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(kHhThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      RCPG_CUDA(cudaLaunchKernelEx(&cfg, householder_cluster_kernel<T>, (const T*)A, Q, int(J), n, chunk,
                                   rank_warning_dev));
      count_launch();
      return r;
    }
  }
  const int maxc = max_coop_blocks(householder_kernel<T>, kFacThreads, 0);
  const int G = std::min(pick_grid(J, n, maxc), w.max_blocks);
  QrArgs<T> a{A,     Q,      J, R, n, r, w.keys, km, w.part, reinterpret_cast<T*>(w.tau), reinterpret_cast<T*>(w.diag),
              w.bar, rank_warning_dev, skip, w.rowk};
  launch_coop(householder_kernel<T>, G, kFacThreads, 0, st, a);
  return r;
}

namespace {

// ------------------------------------- complete-pivoting LU, row-sharded
// the rows of W whose last-mode index lies in this rank's
// slab are local; a row is identified by its global Kolda index (= its
// initial physical position). Per pivot every rank (1) applies the previous
// pivot to its rows and reduces its candidates per CTA, (2) all-gathers the
// candidates, (3) runs the identical choice and bookkeeping (the same total
// order as plu_coop: |value|, then physical column, then physical row), and
// (4) all-reduces the pivot row, which only its owner fills.
constexpr int kDluThreads = 256;

template <typename T>
struct DluState {
  int k0, done, cs, owner, n_ov;
  i64 srow;  // owner-local storage row of the current pivot
  int col_at[kMaxPanelCols];
  i64 ov_pos[kMaxPanelCols], ov_row[kMaxPanelCols];  // position -> global row id (latest wins)
};

template <typename T>
struct DluArgs {
  T* A;
  T* Z;
  i64 J, R;  // local rows, local R of the mode view
  int n, r;
  i64* phys;
  Cand<T>* cand_loc;        // [G]
  const Cand<T>* cand_all;  // [nranks * G]
  T* U;                     // [n]
  DluState<T>* st;
  int rank, G;
  SlabMap sm;
};

__device__ void dlu_locate(const SlabMap& sm, i64 rowid, int& owner, i64& sloc) {
  const i64 row = kolda_inverse(sm.kmg, rowid, sm.Rg);  // a * Rg + b (global)
  const i64 a = row / sm.Rg, bg = row - a * sm.Rg;
  const i64 d = bg % sm.Es, rest = bg / sm.Es;  // last mode is b's fastest digit
  int g = 0;
  while (g + 1 < sm.nranks && d >= sm.hi[g]) ++g;
  owner = g;
  const i64 ext = sm.hi[g] - sm.lo[g];
  sloc = a * ((sm.Rg / sm.Es) * ext) + rest * ext + (d - sm.lo[g]);
}

template <typename T>
__global__ void dlu_init_kernel(DluState<T>* st, int n, int r) {
  if (threadIdx.x == 0) {
    st->k0 = r;
    st->done = 0;
    st->n_ov = 0;
    st->owner = -1;
    st->srow = -1;
    st->cs = 0;
  }
  for (int c = threadIdx.x; c < n; c += blockDim.x) st->col_at[c] = c;
}

// k >= 0: apply pivot k (Z column k) and reduce the candidates for k + 1;
// k == -1: initial scan.
template <typename T>
__global__ void __launch_bounds__(kDluThreads) dlu_update_kernel(DluArgs<T> p, int k) {
  __shared__ Cand<T> red[33];
  __shared__ int col_at[kMaxPanelCols];
  __shared__ T U[kMaxPanelCols];
  const Cand<T> none{T(-1), 0x7fffffff, 0, 0x7fffffffffffffffll, 0};
  const DluState<T>* st = p.st;
  const i64 R = p.R;
  if (k >= 0 && st->done) {
    if (st->k0 == k) {  // exactly-zero corner: unit vectors at positions k0..r-1
      for (i64 s = blockIdx.x * i64(blockDim.x) + threadIdx.x; s < p.J; s += i64(gridDim.x) * blockDim.x) {
        const i64 ps = p.phys[s];
        if (ps < k) continue;
        const i64 a = s / R, b = s - a * R, bz = a * p.r * R + b;
        for (int j = k; j < p.r; ++j) p.Z[bz + j * R] = (ps == j) ? T(1) : T(0);
      }
    }
    if (threadIdx.x == 0) p.cand_loc[blockIdx.x] = none;
    return;
  }
  for (int c = threadIdx.x; c < p.n; c += blockDim.x) {
    col_at[c] = k < 0 ? c : st->col_at[c];
    U[c] = k < 0 ? T(0) : p.U[c];
  }
  __syncthreads();
  const int cs = k < 0 ? 0 : st->cs;
  const T piv = k < 0 ? T(1) : U[cs];
  const bool own_piv = k >= 0 && st->owner == p.rank;
  const i64 srow = st->srow;
  const bool more = (k + 1 < p.r);
  const i64 tag = i64(p.rank) << 40;
  Cand<T> best = none;
  for (i64 s = blockIdx.x * i64(blockDim.x) + threadIdx.x; s < p.J; s += i64(gridDim.x) * blockDim.x) {
    const i64 ps = p.phys[s];
    if (ps < k) continue;  // pivoted earlier
    const i64 a = s / R, b = s - a * R;
    const i64 ba = a * p.n * R + b, bz = a * p.r * R + b;
    if (own_piv && s == srow) {
      p.Z[bz + k * R] = T(1);
      for (int j = k + 1; j < p.r; ++j) p.Z[bz + j * R] = T(0);
      continue;
    }
    T rv = T(-1);
    int rq = 0, rc = 0;
    if (k < 0) {
      for (int c = 0; c < p.n; ++c) {
        const T ax = fabs(p.A[ba + c * R]);
        if (ax > rv) {
          rv = ax;
          rq = c;
          rc = c;
        }
      }
    } else {
      const T m = p.A[ba + cs * R] / piv;
      p.Z[bz + k * R] = m;
      if (!more) continue;
      for (int q = k + 1; q < p.n; ++q) {
        const int c = col_at[q];
        const T x = sub_mul_rn(p.A[ba + c * R], m, U[c]);
        p.A[ba + c * R] = x;
        const T ax = fabs(x);
        if (ax > rv) {
          rv = ax;
          rq = q;
          rc = c;
        }
      }
    }
    const Cand<T> cd{rv, rq, rc, ps, tag | s};
    if (better(cd, best)) best = cd;
  }
  best = block_best(best, red);
  if (threadIdx.x == 0) p.cand_loc[blockIdx.x] = best;
}

template <typename T>
__global__ void __launch_bounds__(kDluThreads) dlu_pick_kernel(DluArgs<T> p, int k, int total) {
  __shared__ Cand<T> red[33];
  DluState<T>* st = p.st;
  if (st->done) {
    for (int c = threadIdx.x; c < p.n; c += blockDim.x) p.U[c] = T(0);
    return;
  }
  const Cand<T> none{T(-1), 0x7fffffff, 0, 0x7fffffffffffffffll, 0};
  Cand<T> g = none;
  for (int q = threadIdx.x; q < total; q += blockDim.x) {
    const Cand<T> x = load_cand_cg(p.cand_all + q);
    if (better(x, g)) g = x;
  }
  g = block_best(g, red);
  if (!(g.v > T(0))) {  // exactly-zero corner (FullPivLU early stop)
    if (threadIdx.x == 0) {
      st->done = 1;
      st->k0 = k;
    }
    for (int c = threadIdx.x; c < p.n; c += blockDim.x) p.U[c] = T(0);
    return;
  }
  const int owner = int(g.s >> 40);
  const i64 sloc = g.s & ((i64(1) << 40) - 1);
  if (threadIdx.x == 0) {
    i64 u = -1;  // global id of the row at physical position k before the swap
    for (int q = st->n_ov - 1; q >= 0; --q)
      if (st->ov_pos[q] == k) {
        u = st->ov_row[q];
        break;
      }
    if (u < 0) u = k;
    if (g.prow != k) {
      st->ov_pos[st->n_ov] = g.prow;
      st->ov_row[st->n_ov] = u;
      st->n_ov += 1;
      int uo;
      i64 uloc;
      dlu_locate(p.sm, u, uo, uloc);
      if (uo == p.rank) p.phys[uloc] = g.prow;
    }
    const int colk = st->col_at[k];
    st->col_at[k] = g.c;
    st->col_at[g.pcol] = colk;
    st->cs = g.c;
    st->owner = owner;
    st->srow = sloc;
    if (owner == p.rank) p.phys[sloc] = k;
  }
  const i64 R = p.R;
  const i64 base = (sloc / R) * p.n * R + (sloc % R);
  for (int c = threadIdx.x; c < p.n; c += blockDim.x) p.U[c] = owner == p.rank ? p.A[base + c * R] : T(0);
}

}  // namespace

size_t dlu_state_bytes() { return sizeof(DluState<double>); }

template <typename T>
int plu_basis_dist(T* A, T* Z, i64 J, i64 R, int n, i64 J_global, const KoldaMap& km, const SlabMap& sm, Comm& comm,
                   const DluWork& w, cudaStream_t st) {
  check_arg(n <= kMaxPanelCols, "plu_basis: panel wider than supported");
  const int r = int(std::min<i64>(J_global, n));
  init_row_keys(km, J, R, w.phys, st);
  DluState<T>* state = reinterpret_cast<DluState<T>*>(w.state);
  dlu_init_kernel<T><<<1, 256, 0, st>>>(state, n, r);
  DluArgs<T> a{A, Z, J, R, n, r, w.phys, reinterpret_cast<Cand<T>*>(w.cand_loc),
               reinterpret_cast<const Cand<T>*>(w.cand_all), reinterpret_cast<T*>(w.U), state, comm.rank, w.G, sm};
  dlu_update_kernel<T><<<w.G, kDluThreads, 0, st>>>(a, -1);
  count_launch(2);
  for (int k = 0; k < r; ++k) {
    comm.allgather(w.cand_loc, w.cand_all, size_t(w.G) * sizeof(Cand<T>), st);
    dlu_pick_kernel<T><<<1, kDluThreads, 0, st>>>(a, k, w.G * comm.size);
    comm.allreduce_sum(w.U, size_t(n), sizeof(T) == 8 ? CommType::f64 : CommType::f32, st);
    dlu_update_kernel<T><<<w.G, kDluThreads, 0, st>>>(a, k);
    count_launch(2);
  }
  RCPG_LAUNCHED();
  return r;
}

template int plu_basis_dist<float>(float*, float*, i64, i64, int, i64, const KoldaMap&, const SlabMap&, Comm&,
                                   const DluWork&, cudaStream_t);
template int plu_basis_dist<double>(double*, double*, i64, i64, int, i64, const KoldaMap&, const SlabMap&, Comm&,
                                    const DluWork&, cudaStream_t);

size_t factor_cand_bytes() { return sizeof(Cand<double>); }

template int plu_basis<float>(float*, float*, i64, i64, int, const KoldaMap&, FactorWork&, cudaStream_t);
template int plu_basis<double>(double*, double*, i64, i64, int, const KoldaMap&, FactorWork&, cudaStream_t);
template int thin_qr<float>(float*, float*, i64, i64, int, const KoldaMap&, FactorWork&, int*, cudaStream_t);
template int thin_qr<double>(double*, double*, i64, i64, int, const KoldaMap&, FactorWork&, int*, cudaStream_t);

}  // namespace rcpg
