// SPDX-License-Identifier: MIT
// Streamed tensor passes over the mode-n view of a row-major tensor.
//
// Every HBM pass of the rCP path contracts the mode-n fibres of the working
// tensor with a thin panel:
//   sketch   Y[i, c]       = sum_{a,b} X[a, i, b] * P[a, c, b]   (Y = X_(n) Omega, X_(n) Z, MTTKRP)
//   project  O[a, c, b]    = sum_i     Q[i, c]    * X[a, i, b]   (W = X_(n)^T Q and B = Q^T X_(n))
// The unfolding X_(n) (tensor.hpp:171-183) is never materialized: the
// panels are indexed by storage position s = a*R + b, so `project` writes
// the folded tensor fold(Q^T X_(n)) (compress.hpp:139-141) directly in its
// row-major layout. Both are register-tiled SIMT GEMMs (256 threads, 16x16
// thread grid, double-buffered shared memory); `sketch` splits K = L*R over
// CTAs and reduces the per-CTA partials in a fixed order (deterministic).
#pragma once

#include "common.cuh"

namespace rcpg {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ core
template <typename T, int BM, int BN, int BK>
struct TileSmem {
  T a[2][BK][BM + 1];
  T b[2][BK][BN + 1];
};

// Loader concept (device):
//   static constexpr bool A_KC, B_KC;      // global A / B contiguous along k?
//   void range(i64& t0, i64& t1) const;    // k tiles of this CTA
//   struct Tile; Tile tile(i64 t) const;
//   T a(const Tile&, int k, int m) const;  // 0 when out of range
//   T b(const Tile&, int k, int n) const;
// Epilogue concept: void operator()(int m, int n, T v) const (m, n local).
template <typename T, int BM, int BN, int BK, bool TXM, class LD, class EP>
__global__ void __launch_bounds__(kThreads) tile_gemm_kernel(LD ld, EP ep) {
  static_assert(BM % 16 == 0 && BN % 16 == 0, "tile shape");
  static_assert((BM * BK) % kThreads == 0 && (BN * BK) % kThreads == 0, "loader shape");
  constexpr int MR = BM / 16, NR = BN / 16;
  constexpr int NA = BM * BK / kThreads, NB = BN * BK / kThreads;
  if (ld.skip != nullptr && *ld.skip) return;  // device-side stop flag (ALS)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<TileSmem<T, BM, BN, BK>*>(smem_raw);

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int mi = TXM ? tx : ty, ni = TXM ? ty : tx;

  T acc[MR][NR];
#pragma unroll
  for (int r = 0; r < MR; ++r)
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[r][c] = T(0);

  i64 t0, t1;
  ld.range(t0, t1);
  T ra[NA], rb[NB];

  auto fetch = [&](i64 t) {
    const auto tl = ld.tile(t);
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int e = tid + q * kThreads;
      const int k = LD::A_KC ? (e % BK) : (e / BM);
      const int m = LD::A_KC ? (e / BK) : (e % BM);
      ra[q] = ld.a(tl, k, m);
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int e = tid + q * kThreads;
      const int k = LD::B_KC ? (e % BK) : (e / BN);
      const int n = LD::B_KC ? (e / BK) : (e % BN);
      rb[q] = ld.b(tl, k, n);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int e = tid + q * kThreads;
      const int k = LD::A_KC ? (e % BK) : (e / BM);
      const int m = LD::A_KC ? (e / BK) : (e % BM);
      sm.a[buf][k][m] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int e = tid + q * kThreads;
      const int k = LD::B_KC ? (e % BK) : (e / BN);
      const int n = LD::B_KC ? (e / BK) : (e % BN);
      sm.b[buf][k][n] = rb[q];
    }
  };

  if (t0 < t1) {
    fetch(t0);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (i64 t = t0; t < t1; ++t) {
      const bool more = (t + 1 < t1);
      if (more) fetch(t + 1);
#pragma unroll 8
      for (int k = 0; k < BK; ++k) {
        T av[MR], bv[NR];
#pragma unroll
        for (int r = 0; r < MR; ++r) av[r] = sm.a[buf][k][mi + 16 * r];
#pragma unroll
        for (int c = 0; c < NR; ++c) bv[c] = sm.b[buf][k][ni + 16 * c];
#pragma unroll
        for (int r = 0; r < MR; ++r)
#pragma unroll
          for (int c = 0; c < NR; ++c) acc[r][c] = fma(av[r], bv[c], acc[r][c]);
      }
      if (more) {
        stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < MR; ++r)
#pragma unroll
    for (int c = 0; c < NR; ++c) ep(mi + 16 * r, ni + 16 * c, acc[r][c]);
}

// ------------------------------------------------------------- sketch
// Y = X_(n) P: partial[split][c][i] over the CTA's k tiles.
// General mode (R > 1): k = (a, b), tiles of BK consecutive b within one a.
template <typename T, int BM, int BN, int BK, typename TX = T, typename TP = T>
struct SketchLoader {
  static constexpr bool A_KC = true, B_KC = true;
  const TX* X;
  const TP* P;
  i64 L, I, R, cols, nbt, tiles_per_split, total;
  const int* skip = nullptr;
  struct Tile {
    i64 a, b0;
  };
  __device__ void range(i64& t0, i64& t1) const {
    t0 = blockIdx.y * tiles_per_split;
    t1 = t0 + tiles_per_split < total ? t0 + tiles_per_split : total;
  }
  __device__ Tile tile(i64 t) const {
    const i64 a = t / nbt;
    return {a, (t - a * nbt) * BK};
  }
  __device__ T a(const Tile& tl, int k, int m) const {
    const i64 i = i64(blockIdx.x) * BM + m, b = tl.b0 + k;
    return (i < I && b < R) ? T(X[(tl.a * I + i) * R + b]) : T(0);
  }
  __device__ T b(const Tile& tl, int k, int n) const {
    const i64 c = i64(blockIdx.z) * BN + n, b = tl.b0 + k;
    return (c < cols && b < R) ? T(P[(tl.a * cols + c) * R + b]) : T(0);
  }
};

// Last mode (R == 1): k = a; X rows contiguous in i, P rows contiguous in c.
template <typename T, int BM, int BN, int BK, typename TX = T, typename TP = T>
struct SketchLastLoader {
  static constexpr bool A_KC = false, B_KC = false;
  const TX* X;
  const TP* P;
  i64 L, I, cols, tiles_per_split, total;
  const int* skip = nullptr;
  struct Tile {
    i64 a0;
  };
  __device__ void range(i64& t0, i64& t1) const {
    t0 = blockIdx.y * tiles_per_split;
    t1 = t0 + tiles_per_split < total ? t0 + tiles_per_split : total;
  }
  __device__ Tile tile(i64 t) const { return {t * BK}; }
  __device__ T a(const Tile& tl, int k, int m) const {
    const i64 i = i64(blockIdx.x) * BM + m, a = tl.a0 + k;
    return (i < I && a < L) ? T(X[a * I + i]) : T(0);
  }
  __device__ T b(const Tile& tl, int k, int n) const {
    const i64 c = i64(blockIdx.z) * BN + n, a = tl.a0 + k;
    return (c < cols && a < L) ? T(P[a * cols + c]) : T(0);
  }
};

template <typename T, int BM, int BN>
struct SketchEpilogue {
  T* part;  // [splits][cols][I]
  i64 I, cols;
  __device__ void operator()(int m, int n, T v) const {
    const i64 i = i64(blockIdx.x) * BM + m, c = i64(blockIdx.z) * BN + n;
    if (i < I && c < cols) part[(i64(blockIdx.y) * cols + c) * I + i] = v;
  }
};

// ------------------------------------------------------------ project
// O[a, c, b] = sum_i Q[i, c] X[a, i, b]; M = b (BM), N = c (BN), K = i.
template <typename T, int BM, int BN, int BK, typename TX = T, typename TP = T>
struct ProjectLoader {
  static constexpr bool A_KC = false, B_KC = true;
  const TX* X;
  const TP* Q;  // column-major I x cols (ld = ldq)
  i64 I, R, cols, ldq, ktiles;
  const int* skip = nullptr;
  struct Tile {
    i64 i0;
  };
  __device__ void range(i64& t0, i64& t1) const {
    t0 = 0;
    t1 = ktiles;
  }
  __device__ Tile tile(i64 t) const { return {t * BK}; }
  __device__ T a(const Tile& tl, int k, int m) const {
    const i64 b = i64(blockIdx.x) * BM + m, i = tl.i0 + k, a = blockIdx.y;
    return (b < R && i < I) ? T(X[(a * I + i) * R + b]) : T(0);
  }
  __device__ T b(const Tile& tl, int k, int n) const {
    const i64 c = i64(blockIdx.z) * BN + n, i = tl.i0 + k;
    return (c < cols && i < I) ? T(Q[i + c * ldq]) : T(0);
  }
};

template <typename T, int BM, int BN, typename TO = T>
struct ProjectEpilogue {
  TO* O;
  i64 R, cols;
  __device__ void operator()(int m, int n, T v) const {
    const i64 b = i64(blockIdx.x) * BM + m, c = i64(blockIdx.z) * BN + n, a = blockIdx.y;
    if (b < R && c < cols) O[(a * cols + c) * R + b] = TO(v);
  }
};

// Last mode (R == 1): O[a, c] = sum_i X[a, i] Q[i, c]; M = a, N = c, K = i.
template <typename T, int BM, int BN, int BK, typename TX = T, typename TP = T>
struct ProjectLastLoader {
  static constexpr bool A_KC = true, B_KC = true;
  const TX* X;
  const TP* Q;
  i64 L, I, cols, ldq, ktiles;
  const int* skip = nullptr;
  i64 tps = 0;  // > 0: split-K, blockIdx.y takes K tiles [y tps, (y + 1) tps)
  struct Tile {
    i64 i0;
  };
  __device__ void range(i64& t0, i64& t1) const {
    t0 = tps > 0 ? blockIdx.y * tps : 0;
    t1 = tps > 0 && t0 + tps < ktiles ? t0 + tps : ktiles;
  }
  __device__ Tile tile(i64 t) const { return {t * BK}; }
  __device__ T a(const Tile& tl, int k, int m) const {
    const i64 a = i64(blockIdx.x) * BM + m, i = tl.i0 + k;
    return (a < L && i < I) ? T(X[a * I + i]) : T(0);
  }
  __device__ T b(const Tile& tl, int k, int n) const {
    const i64 c = i64(blockIdx.z) * BN + n, i = tl.i0 + k;
    return (c < cols && i < I) ? T(Q[i + c * ldq]) : T(0);
  }
};

// split-K partial of the last-mode projection: part[y][a * cols + c]
template <typename T, int BM, int BN>
struct ProjectLastPartEpilogue {
  T* part;
  i64 L, cols;
  __device__ void operator()(int m, int n, T v) const {
    const i64 a = i64(blockIdx.x) * BM + m, c = i64(blockIdx.z) * BN + n;
    if (a < L && c < cols) part[(i64(blockIdx.y) * L + a) * cols + c] = v;
  }
};

template <typename T, int BM, int BN, typename TO = T>
struct ProjectLastEpilogue {
  TO* O;
  i64 L, cols;
  __device__ void operator()(int m, int n, T v) const {
    const i64 a = i64(blockIdx.x) * BM + m, c = i64(blockIdx.z) * BN + n;
    if (a < L && c < cols) O[a * cols + c] = TO(v);
  }
};

// ------------------------------------------------------------ host API
struct PassStats {
  double bytes = 0;  // algorithmic bytes of the pass
  double flops = 0;
};

template <typename T>
void sketch(const T* X, ModeView v, const T* P, i64 cols, T* Y, T* scratch, i64 scratch_elems,
            int num_sms, cudaStream_t st, const int* skip = nullptr);
template <typename T>
i64 sketch_scratch_elems(ModeView v, i64 cols, int num_sms);
// scratch (optional): split-K partials of a last-mode view (R == 1), when the
// plain grid would be small (project_scratch_elems doubles)
template <typename T>
void project(const T* X, ModeView v, const T* Q, i64 ldq, i64 cols, T* O, cudaStream_t st, T* scratch = nullptr,
             i64 scratch_elems = 0);
template <typename T>
i64 project_scratch_elems(ModeView v, i64 cols, int num_sms);

// 128-byte CUtensorMap (opaque here) for an fp64 (d0, d1, d2) view, box {16, b1, 1}, 128B swizzle.
void tensor_map_f64_3d(void* out, const double* base, i64 d0, i64 d1, i64 d2, int b1, i64 pitch = 0);
// fp32 (d0, d1, d2) view, box {16, b1, 1}, 64B swizzle (fp32 X of the fp64-arithmetic passes).
void tensor_map_f32_3d_sw64(void* out, const float* base, i64 d0, i64 d1, i64 d2, int b1, i64 pitch = 0);
// FP64 tensor-core (DMMA) versions for mode views with R > 1 (passes_dmma.cu).
i64 sketch_dmma_splits(ModeView v, i64 cols, int num_sms, i64& tps, i64& total);
void sketch_dmma(const double* X, ModeView v, const double* P, i64 cols, double* part, int num_sms,
                 const int* skip, cudaStream_t st);
void project_dmma(const double* X, ModeView v, const double* Q, i64 ldq, i64 cols, double* O, cudaStream_t st);
// fp32 X with fp64 products and sums (the fp32 configs' faithful passes); false
// when the view does not suit the TMA kernels (the caller takes the SIMT path).
i64 sketch_dmma_f32_splits(ModeView v, i64 cols, int num_sms, i64& tps, i64& total);
bool sketch_dmma_f32(const float* X, ModeView v, const double* P, i64 cols, double* part, int num_sms,
                     const int* skip, cudaStream_t st);
bool project_dmma_f32(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, float* O, cudaStream_t st);
bool project_dmma_f32(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, double* O, cudaStream_t st);
// Mixed passes of the faithful fp32 path: X fp32, panel fp64, fp64 accumulation,
// one rounding of each result to fp32 (Y [I x cols] column-major, O in the
// (a, c, b) layout). scratch: sketch_mixed_scratch_doubles().
i64 sketch_mixed_scratch_doubles(ModeView v, i64 cols, int num_sms);
void sketch_mixed(const float* X, ModeView v, const double* P, i64 cols, float* Y, double* scratch,
                  i64 scratch_doubles, int num_sms, cudaStream_t st, const int* skip = nullptr);
void project_mixed(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, float* O, cudaStream_t st);
// fp64-output versions: a rank's unrounded partial of a sum sharded over ranks
// (all-reduced in fp64, then rounded once with narrow_f64)
void sketch_mixed(const float* X, ModeView v, const double* P, i64 cols, double* Y, double* scratch,
                  i64 scratch_doubles, int num_sms, cudaStream_t st, const int* skip = nullptr);
void project_mixed(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, double* O, cudaStream_t st);
void narrow_f64(const double* src, float* dst, i64 n, cudaStream_t st);
// dst[i] = double(src[i]) (exact)
void widen_f32(const float* src, double* dst, i64 n, cudaStream_t st);

// FP32 tcgen05 (3xTF32, TMEM accumulator) versions for mode views with R > 1
// (passes_tc.cu). RCPG_NO_TC=1 in the environment routes fp32 to the SIMT
// kernels instead (A/B testing only).
bool tc_enabled();
bool tc_sketch_ok(const float* X, const float* P, ModeView v);
bool tc_project_ok(const float* X, const float* Q, ModeView v, i64 ldq);
i64 sketch_tc_splits(ModeView v, i64 cols, int num_sms, i64& tps, i64& total);
// pblk: sketch_tc_panel_floats() of scratch for the K-tile-blocked panel copy
// (nullptr: read the (a, c, b) panel directly). RCPG_TC_PBLK=0|1|2 selects
// direct / blocked raw / blocked hi+lo planes (A/B hook; default 1).
i64 sketch_tc_panel_floats(ModeView v, i64 cols);
void sketch_tc(const float* X, ModeView v, const float* P, i64 cols, float* part, float* pblk, int num_sms,
               const int* skip, cudaStream_t st);
void project_tc(const float* X, ModeView v, const float* Q, i64 ldq, i64 cols, float* O, int num_sms,
                cudaStream_t st);
// ||X - Xhat||^2, ||X||^2 partials per CTA (part[2 * blocks]) with Xhat on tcgen05;
// rank <= 64, last extent % 4 == 0. ct_scratch: residual_tc_scratch_floats().
bool tc_residual_ok(const i64* shape, int order, int rank);
size_t residual_tc_scratch_floats(i64 E, int rank);
void residual_tc(const float* X, const i64* shape, int order, const float* const* factors, const float* weights,
                 int rank, float* ct_scratch, double* part, int num_sms, int& blocks, cudaStream_t st);

// Omega_n written in the panel layout (a, c, b): entry (s, c) is normal /
// uniform_sym number c*J + kolda(s) of stream (seed, (compress << 32) | mode).
template <typename T>
void omega_panel(u64 seed, i64 mode, const KoldaMap& km, ModeView v, i64 cols, int distribution, T* P,
                 cudaStream_t st, i64 J_global = 0);
// Omega generated on the host with the reference's libm (omega_host.cu);
// out_kind 0 float, 1 double, 2 double holding the float-rounded value.
void omega_host_panel(u64 seed, i64 mode, const KoldaMap& km, ModeView v, i64 cols, int distribution, i64 Jg,
                      int out_kind, void* host_out);
// Omega rounded to fp32 (the fp32 configs' Matrix<float> Omega) stored as fp64.
void omega_panel_f32_as_f64(u64 seed, i64 mode, const KoldaMap& km, ModeView v, i64 cols, int distribution,
                            double* P, cudaStream_t st, i64 J_global = 0);

}  // namespace rcpg
