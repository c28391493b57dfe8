// SPDX-License-Identifier: MIT
// FP64 streamed passes on the B200 double-precision tensor cores
// (mma.sync.m16n8k4.f64, DMMA). The fp64 configs (C1/C2) are FP64-pipe
// bound: a pass does 2*S*l flops over S*8 bytes (AI = l/4 flop/B), so at
// l = 30 the ~37 TFLOP/s FP64 peak caps a pass at ~75% of HBM bandwidth.
// SIMT DFMA tiles were shared-memory-bandwidth bound (one LDS per two
// FMAs); a DMMA does 512 FMAs per warp instruction from register fragments.
//
//   sketch  Y[i, c]    = sum_{a,b} X[a, i, b] P[a, c, b]   (K = (a, b), split over CTAs)
//   project O[a, c, b] = sum_i X[a, i, b] Q[i, c]          (K = i, full per CTA)
// (mode views with R > 1; the last mode (R = 1) keeps the SIMT kernels.)
// Operand tiles stream through a multi-stage cp.async pipeline (16-byte
// copies when the row strides are even, 8-byte otherwise; out-of-range
// elements are zero-filled by the copy itself).
//
// The sketch with even R runs TMA-fed (sketch_dmma_tma_kernel): one producer
// warp streams 128B-swizzled K-tiles of X and the panel (16 doubles per row)
// through a 4-stage mbarrier ring and four consumer warps only load
// fragments and issue DMMAs. The cp.async version spends more issue slots on
// address math and copies than on the MMAs; with the copies off the
// consumers four CTAs (16 consumer warps) per SM keep the FP64 pipe ~25%
// busier (tools/microbench/dmma_tma.cu: C2 mode-0 sketch 195 -> 159 us).
#include <cuda.h>  // CUtensorMap (encoded in passes_tc.cu)

#include <cstdlib>

#include "passes.cuh"
#include "runtime.cuh"
#include "tc.cuh"

namespace rcpg {

namespace {

constexpr int kDThreads = 128;  // 4 warps, each a 16-row slab of the CTA tile
constexpr int kDBM = 64;
constexpr int kDBK = 16;  // 16: four CTAs (16 warps) per SM hide the DMMA accumulator latency

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = ok ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = ok ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

template <int BN>
constexpr int stages_for() {
  return BN <= 32 ? 4 : (BN <= 48 ? 3 : 2);
}

// ------------------------------------------------------------- sketch
// smem per stage: A [BM][BK+4] (m rows, k contiguous), B [BN][BK+4].
template <int BN, bool V16>
__global__ void __launch_bounds__(kDThreads) sketch_dmma_kernel(const double* __restrict__ X,
                                                                const double* __restrict__ P, i64 I, i64 R, i64 cols,
                                                                i64 nbt, i64 tiles_per_split, i64 total,
                                                                double* __restrict__ part, const int* skip) {
  if (skip != nullptr && *skip) return;
  constexpr int S = stages_for<BN>();
  constexpr int SA = kDBK + 4;
  constexpr int NT = BN / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);  // [S][BM][SA]
  double* sB = sA + S * kDBM * SA;                    // [S][BN][SA]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const i64 m0 = i64(blockIdx.x) * kDBM;
  const i64 n0 = i64(blockIdx.z) * BN;
  const i64 t0 = blockIdx.y * tiles_per_split;
  const i64 t1 = t0 + tiles_per_split < total ? t0 + tiles_per_split : total;
  const int nk = int(t1 - t0);

  auto load = [&](int stage, i64 tt) {
    const i64 a = tt / nbt, b0 = (tt - a * nbt) * kDBK;
    double* dA = sA + stage * kDBM * SA;
    double* dB = sB + stage * BN * SA;
    constexpr int W = V16 ? 2 : 1;       // doubles per copy
    constexpr int CPR = kDBK / W;        // copies per row
    for (int e = tid; e < kDBM * CPR; e += kDThreads) {
      const int m = e / CPR, k = (e % CPR) * W;
      const i64 i = m0 + m, b = b0 + k;
      const bool ok = (i < I) && (b < R);
      const double* src = X + (ok ? ((a * I + i) * R + b) : 0);
      if (V16) cp_async16(dA + m * SA + k, src, ok); else cp_async8(dA + m * SA + k, src, ok);
    }
    for (int e = tid; e < BN * CPR; e += kDThreads) {
      const int n = e / CPR, k = (e % CPR) * W;
      const i64 c = n0 + n, b = b0 + k;
      const bool ok = (c < cols) && (b < R);
      const double* src = P + (ok ? ((a * cols + c) * R + b) : 0);
      if (V16) cp_async16(dB + n * SA + k, src, ok); else cp_async8(dB + n * SA + k, src, ok);
    }
  };

  double acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;

#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < nk) load(s, t0 + s);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<S - 2>();
    __syncthreads();
    const int pre = kt + S - 1;
    if (pre < nk) load(pre % S, t0 + pre);
    cp_commit();
    const double* cA = sA + (kt % S) * kDBM * SA + (w * 16) * SA;
    const double* cB = sB + (kt % S) * BN * SA;
#pragma unroll
    for (int kk = 0; kk < kDBK; kk += 4) {
      const double a0 = cA[g * SA + kk + t];
      const double a1 = cA[(g + 8) * SA + kk + t];
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[j], a0, a1, cB[(j * 8 + g) * SA + kk + t]);
    }
  }
  cp_wait<0>();
  // partial[split][c][i]
  const i64 r0 = m0 + w * 16 + g;
  double* out = part + i64(blockIdx.y) * cols * I;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const i64 c0 = n0 + j * 8 + 2 * t;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const i64 i = r0 + (q >> 1) * 8, c = c0 + (q & 1);
      if (i < I && c < cols) out[c * I + i] = acc[j][q];
    }
  }
}

// ------------------------------------------------------------ project
// M = b (BM), N = c, K = i. smem per stage: A [BK][BM+8] (k rows, m
// contiguous), B [BN][BK+4].
template <int BN, bool VA16, bool VB16>
__global__ void __launch_bounds__(kDThreads) project_dmma_kernel(const double* __restrict__ X,
                                                                 const double* __restrict__ Q, i64 I, i64 R, i64 cols,
                                                                 i64 ldq, double* __restrict__ O) {
  constexpr int S = stages_for<BN>();
  constexpr int SAm = kDBM + 8;
  constexpr int SB = kDBK + 4;
  constexpr int NT = BN / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);  // [S][BK][SAm]
  double* sB = sA + S * kDBK * SAm;                   // [S][BN][SB]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const i64 b0 = i64(blockIdx.x) * kDBM;
  const i64 a = blockIdx.y;
  const i64 n0 = i64(blockIdx.z) * BN;
  const int nk = int(ceil_div(I, kDBK));
  const double* Xa = X + a * I * R;

  auto load = [&](int stage, int kt) {
    const i64 i0 = i64(kt) * kDBK;
    double* dA = sA + stage * kDBK * SAm;
    double* dB = sB + stage * BN * SB;
    {
      constexpr int W = VA16 ? 2 : 1;
      constexpr int CPR = kDBM / W;
      for (int e = tid; e < kDBK * CPR; e += kDThreads) {
        const int k = e / CPR, m = (e % CPR) * W;
        const i64 i = i0 + k, b = b0 + m;
        const bool ok = (i < I) && (b < R);
        const double* src = Xa + (ok ? (i * R + b) : 0);
        if (VA16) cp_async16(dA + k * SAm + m, src, ok); else cp_async8(dA + k * SAm + m, src, ok);
      }
    }
    {
      constexpr int W = VB16 ? 2 : 1;
      constexpr int CPR = kDBK / W;
      for (int e = tid; e < BN * CPR; e += kDThreads) {
        const int n = e / CPR, k = (e % CPR) * W;
        const i64 c = n0 + n, i = i0 + k;
        const bool ok = (c < cols) && (i < I);
        const double* src = Q + (ok ? (i + c * ldq) : 0);
        if (VB16) cp_async16(dB + n * SB + k, src, ok); else cp_async8(dB + n * SB + k, src, ok);
      }
    }
  };

  double acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < nk) load(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<S - 2>();
    __syncthreads();
    const int pre = kt + S - 1;
    if (pre < nk) load(pre % S, pre);
    cp_commit();
    const double* cA = sA + (kt % S) * kDBK * SAm + w * 16;
    const double* cB = sB + (kt % S) * BN * SB;
#pragma unroll
    for (int kk = 0; kk < kDBK; kk += 4) {
      const double a0 = cA[(kk + t) * SAm + g];
      const double a1 = cA[(kk + t) * SAm + g + 8];
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[j], a0, a1, cB[(j * 8 + g) * SB + kk + t]);
    }
  }
  cp_wait<0>();
  const i64 bb = b0 + w * 16 + g;
  double* Oa = O + a * cols * R;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const i64 c0 = n0 + j * 8 + 2 * t;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const i64 b = bb + (q >> 1) * 8, c = c0 + (q & 1);
      if (b < R && c < cols) Oa[c * R + b] = acc[j][q];
    }
  }
}

// ------------------------------------------------------ sketch, TMA-fed
constexpr int kTmaWM = 4;      // consumer warps, 16 rows each
constexpr int kTmaStages = 4;  // 4 stages: four CTAs per SM at BN = 32

// TX = element type of X in HBM: double (128-byte box rows, 128B swizzle) or
// float (64-byte box rows, 64B swizzle; the fp32 configs' faithful passes,
// converted to fp64 when a fragment is loaded). The panel is always fp64.
template <int BN, typename TX = double>
struct TmaPlan {
  static constexpr int BM = kTmaWM * 16, ABYTES = BM * 16 * int(sizeof(TX)), BBYTES = BN * 128,
                       STAGE = ABYTES + BBYTES;
  static constexpr int SMEM = kTmaStages * STAGE + 1024;  // + 1024 B alignment slack (swizzle atoms)
  static constexpr int THREADS = (kTmaWM + 1) * 32;
};

// element (r, k) of a 128B-swizzled box with 16-double rows
__device__ __forceinline__ int swz16(int r, int k) { return r * 16 + ((((k >> 1) ^ (r & 7))) << 1) + (k & 1); }
// element (r, k) of a 64B-swizzled box with 16-float rows (16-byte chunk k / 4
// XOR bits 7-8 of the row's byte offset): the 8 rows x 4 k of a fragment load
// hit 32 distinct banks
__device__ __forceinline__ int swz16f(int r, int k) { return r * 16 + ((((k >> 2) ^ ((r >> 1) & 3))) << 2) + (k & 3); }
__device__ __forceinline__ double ldsx(const double* A, int r, int k) { return A[swz16(r, k)]; }
__device__ __forceinline__ double ldsx(const float* A, int r, int k) { return double(A[swz16f(r, k)]); }

template <int BN, typename TX>
__global__ void __launch_bounds__(TmaPlan<BN, TX>::THREADS) sketch_dmma_tma_kernel(const __grid_constant__ CUtensorMap mx,
                                                                               const __grid_constant__ CUtensorMap mp,
                                                                               i64 I, i64 cols, i64 nbt, i64 tps,
                                                                               i64 total, double* __restrict__ part,
                                                                               const int* skip) {
  using G = TmaPlan<BN, TX>;
  using namespace tc;
  constexpr int NT = BN / 8, S = kTmaStages;
  if (skip != nullptr && *skip) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const i64 t0 = blockIdx.y * tps;
  const i64 t1 = t0 + tps < total ? t0 + tps : total;
  const int nk = int(t1 - t0);
  const int m0 = blockIdx.x * G::BM, n0 = blockIdx.z * BN;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaWM);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (w == kTmaWM) {  // producer: one thread issues both boxes of a K-tile
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % S;
        if (kt >= S) mbar_wait(&empty[s], uint32_t(((kt / S) - 1) & 1));
        const i64 tt = t0 + kt, a = tt / nbt, b0 = (tt - a * nbt) * 16;
        mbar_arrive_tx(&full[s], G::STAGE);
        unsigned char* st = smem + s * G::STAGE;
        tma_load_3d(st, &mx, int(b0), m0, int(a), &full[s]);
        tma_load_3d(st + G::ABYTES, &mp, int(b0), n0, int(a), &full[s]);
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3, r0 = w * 16 + g;
  double acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % S;
    mbar_wait(&full[s], uint32_t((kt / S) & 1));
    const TX* A = reinterpret_cast<const TX*>(smem + s * G::STAGE);
    const double* B = reinterpret_cast<const double*>(smem + s * G::STAGE + G::ABYTES);
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      const double a0 = ldsx(A, r0, kk + t);
      const double a1 = ldsx(A, r0 + 8, kk + t);
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[j], a0, a1, B[swz16(j * 8 + g, kk + t)]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  // partial[split][c][i]
  const i64 ri = m0 + r0;
  double* out = part + i64(blockIdx.y) * cols * I;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const i64 c0 = n0 + j * 8 + 2 * t;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const i64 i = ri + (q >> 1) * 8, c = c0 + (q & 1);
      if (i < I && c < cols) out[c * I + i] = acc[j][q];
    }
  }
}

// ---------------------------------------------------- project, TMA-fed
// O[a, c, b] = sum_i X[a, i, b] Q[i, c]: M = b (four 16-wide boxes of X per
// stage, one per consumer warp), N = c, K = i (16 per stage), no split.
template <int BN, typename TX, typename TO>
__global__ void __launch_bounds__(TmaPlan<BN, TX>::THREADS) project_dmma_tma_kernel(const __grid_constant__ CUtensorMap mx,
                                                                                const __grid_constant__ CUtensorMap mq,
                                                                                i64 I, i64 R, i64 cols, int a_base,
                                                                                TO* __restrict__ O) {
  using G = TmaPlan<BN, TX>;
  using namespace tc;
  constexpr int NT = BN / 8, S = kTmaStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nk = int(ceil_div(I, i64(16)));
  const int b0 = blockIdx.x * G::BM, n0 = blockIdx.z * BN;
  const int a = a_base + int(blockIdx.y);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaWM);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (w == kTmaWM) {
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % S;
        if (kt >= S) mbar_wait(&empty[s], uint32_t(((kt / S) - 1) & 1));
        mbar_arrive_tx(&full[s], G::STAGE);
        unsigned char* st = smem + s * G::STAGE;
#pragma unroll
        for (int q = 0; q < kTmaWM; ++q)
          tma_load_3d(st + q * 256 * int(sizeof(TX)), &mx, b0 + 16 * q, kt * 16, a, &full[s]);
        tma_load_3d(st + G::ABYTES, &mq, kt * 16, n0, 0, &full[s]);
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  double acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % S;
    mbar_wait(&full[s], uint32_t((kt / S) & 1));
    const TX* A = reinterpret_cast<const TX*>(smem + s * G::STAGE) + w * 256;  // box of this warp's b's
    const double* B = reinterpret_cast<const double*>(smem + s * G::STAGE + G::ABYTES);
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      const double a0 = ldsx(A, kk + t, g);
      const double a1 = ldsx(A, kk + t, g + 8);
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[j], a0, a1, B[swz16(j * 8 + g, kk + t)]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  const i64 bb = b0 + w * 16 + g;
  TO* Oa = O + i64(blockIdx.y) * cols * R;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const i64 c0 = n0 + j * 8 + 2 * t;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const i64 b = bb + (q >> 1) * 8, c = c0 + (q & 1);
      if (b < R && c < cols) Oa[c * R + b] = TO(acc[j][q]);
    }
  }
}

template <int BN, typename TX = double>
int tma_ctas_per_sm() {
  static const int per = [] {
    const size_t lim = enable_max_dyn_smem(sketch_dmma_tma_kernel<BN, TX>);
    if (size_t(TmaPlan<BN, TX>::SMEM) > lim) return 0;
    int n = 0;
    RCPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sketch_dmma_tma_kernel<BN, TX>,
                                                            TmaPlan<BN, TX>::THREADS, TmaPlan<BN, TX>::SMEM));
    return n;
  }();
  return per;
}

int pick_bn8(i64 cols) {
  if (cols <= 16) return 16;
  if (cols <= 32) return 32;
  if (cols <= 48) return 48;
  if (cols <= 64) return 64;
  if (cols <= 72) return 72;  // TMA kernels only (C3's l = 70: 80 wasted 12% of the MMAs);
  return 80;                  // the cp.async kernels run 72 as 80
}

template <int BN, bool V>
void launch_sketch(dim3 grid, const double* X, const double* P, ModeView v, i64 cols, i64 nbt, i64 tps, i64 total,
                   double* part, const int* skip, cudaStream_t st) {
  constexpr int S = stages_for<BN>();
  const size_t smem = size_t(S) * (kDBM + BN) * (kDBK + 4) * sizeof(double);
  static const size_t lim = enable_max_dyn_smem(sketch_dmma_kernel<BN, V>);
  if (smem > lim) throw std::runtime_error("sketch_dmma: smem plan too large");
  sketch_dmma_kernel<BN, V><<<grid, kDThreads, smem, st>>>(X, P, v.I, v.R, cols, nbt, tps, total, part, skip);
  count_launch();
  RCPG_LAUNCHED();
}

template <int BN, bool VA, bool VB>
void launch_project(dim3 grid, const double* X, const double* Q, ModeView v, i64 cols, i64 ldq, double* O,
                    cudaStream_t st) {
  constexpr int S = stages_for<BN>();
  const size_t smem = size_t(S) * (kDBK * (kDBM + 8) + BN * (kDBK + 4)) * sizeof(double);
  static const size_t lim = enable_max_dyn_smem(project_dmma_kernel<BN, VA, VB>);
  if (smem > lim) throw std::runtime_error("project_dmma: smem plan too large");
  project_dmma_kernel<BN, VA, VB><<<grid, kDThreads, smem, st>>>(X, Q, v.I, v.R, cols, ldq, O);
  count_launch();
  RCPG_LAUNCHED();
}

}  // namespace

namespace {
// TMA needs 16-byte row pitches: R even for fp64 X, R % 4 == 0 for fp32 X
template <typename TX>
bool tma_sketch_shape_ok(ModeView v, i64 cols) {
  constexpr i64 kMax = (i64(1) << 31) - 1;
  constexpr i64 vec = 16 / i64(sizeof(TX));
  return v.R % vec == 0 && v.R <= kMax && v.I <= kMax && v.L <= kMax && cols <= kMax &&
         std::getenv("RCPG_DMMA_CPASYNC") == nullptr;
}

template <typename TX>
int tma_per_sm(int bn) {
  switch (bn) {
    case 16: return tma_ctas_per_sm<16, TX>();
    case 32: return tma_ctas_per_sm<32, TX>();
    case 48: return tma_ctas_per_sm<48, TX>();
    case 64: return tma_ctas_per_sm<64, TX>();
    case 72: return tma_ctas_per_sm<72, TX>();
    default: return tma_ctas_per_sm<80, TX>();
  }
}

template <typename TX>
i64 sketch_dmma_splits_t(ModeView v, i64 cols, int num_sms, i64& tps, i64& total) {
  const int bn = pick_bn8(cols);
  total = v.L * ceil_div(v.R, kDBK);
  i64 mt, per_sm;
  if (tma_sketch_shape_ok<TX>(v, cols) && tma_per_sm<TX>(bn) > 0) {
    mt = ceil_div(v.I, i64(kTmaWM * 16));
    per_sm = tma_per_sm<TX>(bn);
  } else {
    // residency from the smem plan, capped by registers: ~80 per thread x 128 threads
    mt = ceil_div(v.I, kDBM);
    const int S = bn <= 32 ? 4 : (bn <= 48 ? 3 : 2);
    const i64 smem = i64(S) * (kDBM + bn) * (kDBK + 4) * 8 + 1024;
    per_sm = std::max<i64>(1, std::min<i64>(6, (227 * 1024) / smem));
  }
  const i64 nt = ceil_div(cols, i64(bn));
  // whole waves of resident CTAs: a grid a few CTAs over a wave boundary
  // leaves most SMs idle for the last wave. From ~2 waves up to ~8, the split
  // count whose grid fills its last wave best (C5's 157 m-tiles at 3 CTAs per
  // SM: 5 splits filled 1.77 waves, 14 fill 4.95)
  const i64 slots = per_sm * i64(num_sms), waves = 2;
  i64 want = std::max<i64>(1, (waves * slots) / (mt * nt));
  want = std::max<i64>(1, std::min<i64>(want, 65535));
  i64 best_tps = std::max<i64>(1, ceil_div(total, want));
  // small views (C2's mode 1: 750 K-tiles over 7 m-tiles): a two-wave plan gives
  // every CTA ~5 K-tiles, mostly pipeline fill, and doubles the partials; one
  // wave of CTAs twice as long is shorter
  static const int short_tps = getenv("RCPG_SKETCH_SHORT_TPS") ? atoi(getenv("RCPG_SKETCH_SHORT_TPS")) : 16;
  if (best_tps < short_tps) {
    want = std::max<i64>(1, std::min<i64>(slots / (mt * nt), 65535));
    best_tps = std::max<i64>(1, ceil_div(total, want));
  }
  double best_fill = -1.0;
  {  // keep the 2-wave plan when its last wave is already >= 90% full or its CTAs
     // are short (more splits only add partial traffic: C2's X Z 0.42 -> 0.44 ms)
    const i64 sp = ceil_div(total, best_tps), ctas = mt * nt * sp;
    if (double(ctas) / double(ceil_div(ctas, slots) * slots) >= 0.9 || best_tps < 64) {
      tps = best_tps;
      return sp;
    }
  }
  for (i64 s = want; s <= std::min<i64>(4 * want, 65535); ++s) {
    const i64 tp = std::max<i64>(1, ceil_div(total, s)), sp = ceil_div(total, tp);
    const i64 ctas = mt * nt * sp;
    const double fill = double(ctas) / double(ceil_div(ctas, slots) * slots);
    if (fill > best_fill + 1e-3) {
      best_fill = fill;
      best_tps = tp;
    }
    if (fill > 0.99) break;
  }
  tps = best_tps;
  return ceil_div(total, tps);
}

void tensor_map_x(void* out, const double* X, ModeView v, int b1) { tensor_map_f64_3d(out, X, v.R, v.I, v.L, b1); }
void tensor_map_x(void* out, const float* X, ModeView v, int b1) { tensor_map_f32_3d_sw64(out, X, v.R, v.I, v.L, b1); }

template <int BN, typename TX>
void launch_sketch_tma(const TX* X, ModeView v, const double* P, i64 cols, i64 tps, i64 total, i64 splits,
                       double* part, const int* skip, cudaStream_t st) {
  using G = TmaPlan<BN, TX>;
  static const size_t lim = enable_max_dyn_smem(sketch_dmma_tma_kernel<BN, TX>);
  if (size_t(G::SMEM) > lim) throw std::runtime_error("sketch_dmma_tma: smem plan too large");
  alignas(64) unsigned char mx[128], mp[128];
  tensor_map_x(mx, X, v, kTmaWM * 16);
  tensor_map_f64_3d(mp, P, v.R, cols, v.L, BN);
  dim3 grid{unsigned(ceil_div(v.I, i64(kTmaWM * 16))), unsigned(splits), unsigned(ceil_div(cols, i64(BN)))};
  sketch_dmma_tma_kernel<BN, TX><<<grid, G::THREADS, G::SMEM, st>>>(
      *reinterpret_cast<const CUtensorMap*>(mx), *reinterpret_cast<const CUtensorMap*>(mp), v.I, cols,
      ceil_div(v.R, kDBK), tps, total, part, skip);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename TX>
bool sketch_tma_dispatch(const TX* X, ModeView v, const double* P, i64 cols, double* part, i64 tps, i64 total,
                         i64 splits, const int* skip, cudaStream_t st) {
  const int BN = pick_bn8(cols);
  const bool aligned = reinterpret_cast<uintptr_t>(X) % 16 == 0 && reinterpret_cast<uintptr_t>(P) % 16 == 0;
  if (!(tma_sketch_shape_ok<TX>(v, cols) && aligned && tma_per_sm<TX>(BN) > 0)) return false;
  switch (BN) {
    case 16: launch_sketch_tma<16, TX>(X, v, P, cols, tps, total, splits, part, skip, st); break;
    case 32: launch_sketch_tma<32, TX>(X, v, P, cols, tps, total, splits, part, skip, st); break;
    case 48: launch_sketch_tma<48, TX>(X, v, P, cols, tps, total, splits, part, skip, st); break;
    case 64: launch_sketch_tma<64, TX>(X, v, P, cols, tps, total, splits, part, skip, st); break;
    case 72: launch_sketch_tma<72, TX>(X, v, P, cols, tps, total, splits, part, skip, st); break;
    default: launch_sketch_tma<80, TX>(X, v, P, cols, tps, total, splits, part, skip, st); break;
  }
  return true;
}

template <int BN, typename TX, typename TO>
void launch_project_tma(const TX* X, ModeView v, const double* Q, i64 ldq, i64 cols, TO* O, cudaStream_t st) {
  using G = TmaPlan<BN, TX>;
  static const size_t lim = enable_max_dyn_smem(project_dmma_tma_kernel<BN, TX, TO>);
  if (size_t(G::SMEM) > lim) throw std::runtime_error("project_dmma_tma: smem plan too large");
  alignas(64) unsigned char mx[128], mq[128];
  tensor_map_x(mx, X, v, 16);
  tensor_map_f64_3d(mq, Q, v.I, cols, 1, BN, ldq);  // Q column-major: i fastest (pitch ldq), c; rows >= I read as 0
  for (i64 a0 = 0; a0 < v.L; a0 += 65535) {
    const i64 na = std::min<i64>(65535, v.L - a0);
    dim3 grid{unsigned(ceil_div(v.R, i64(kTmaWM * 16))), unsigned(na), unsigned(ceil_div(cols, i64(BN)))};
    project_dmma_tma_kernel<BN, TX, TO><<<grid, G::THREADS, G::SMEM, st>>>(
        *reinterpret_cast<const CUtensorMap*>(mx), *reinterpret_cast<const CUtensorMap*>(mq), v.I, v.R, cols,
        int(a0), O + a0 * cols * v.R);
    count_launch();
    RCPG_LAUNCHED();
  }
}

template <typename TX, typename TO>
bool project_tma_dispatch(const TX* X, ModeView v, const double* Q, i64 ldq, i64 cols, TO* O, cudaStream_t st) {
  const int BN = pick_bn8(cols);
  const bool aligned = reinterpret_cast<uintptr_t>(X) % 16 == 0 && reinterpret_cast<uintptr_t>(Q) % 16 == 0;
  if (!(tma_sketch_shape_ok<TX>(v, cols) && ldq % 2 == 0 && ldq >= v.I && aligned)) return false;
  switch (BN) {
    case 16: launch_project_tma<16, TX, TO>(X, v, Q, ldq, cols, O, st); break;
    case 32: launch_project_tma<32, TX, TO>(X, v, Q, ldq, cols, O, st); break;
    case 48: launch_project_tma<48, TX, TO>(X, v, Q, ldq, cols, O, st); break;
    case 64: launch_project_tma<64, TX, TO>(X, v, Q, ldq, cols, O, st); break;
    case 72: launch_project_tma<72, TX, TO>(X, v, Q, ldq, cols, O, st); break;
    default: launch_project_tma<80, TX, TO>(X, v, Q, ldq, cols, O, st); break;
  }
  return true;
}
}  // namespace

i64 sketch_dmma_splits(ModeView v, i64 cols, int num_sms, i64& tps, i64& total) {
  return sketch_dmma_splits_t<double>(v, cols, num_sms, tps, total);
}

void sketch_dmma(const double* X, ModeView v, const double* P, i64 cols, double* part, int num_sms, const int* skip,
                 cudaStream_t st) {
  i64 tps, total;
  const i64 splits = sketch_dmma_splits(v, cols, num_sms, tps, total);
  if (sketch_tma_dispatch<double>(X, v, P, cols, part, tps, total, splits, skip, st)) return;
  const int BN = pick_bn8(cols);
  const i64 nbt = ceil_div(v.R, kDBK);
  dim3 grid{unsigned(ceil_div(v.I, kDBM)), unsigned(splits), unsigned(ceil_div(cols, BN))};
  const bool v16 = (v.R % 2 == 0) && reinterpret_cast<uintptr_t>(X) % 16 == 0 && reinterpret_cast<uintptr_t>(P) % 16 == 0;
#define RCPG_SK(BNV)                                                                              \
  case BNV:                                                                                       \
    if (v16)                                                                                      \
      launch_sketch<BNV, true>(grid, X, P, v, cols, nbt, tps, total, part, skip, st);             \
    else                                                                                          \
      launch_sketch<BNV, false>(grid, X, P, v, cols, nbt, tps, total, part, skip, st);            \
    break;
  switch (BN) {
    RCPG_SK(16)
    RCPG_SK(32)
    RCPG_SK(48)
    RCPG_SK(64)
    default:
      RCPG_SK(80)
  }
#undef RCPG_SK
}

void project_dmma(const double* X, ModeView v, const double* Q, i64 ldq, i64 cols, double* O, cudaStream_t st) {
  if (project_tma_dispatch<double, double>(X, v, Q, ldq, cols, O, st)) return;
  const int BN = pick_bn8(cols);
  // 16-byte copies need 16-byte aligned rows: even strides and aligned bases (a slab's Q + lo may not be)
  const bool va = (v.R % 2 == 0) && reinterpret_cast<uintptr_t>(X) % 16 == 0,
             vb = (ldq % 2 == 0) && reinterpret_cast<uintptr_t>(Q) % 16 == 0;
  for (i64 a0 = 0; a0 < v.L; a0 += 65535) {
    const i64 na = std::min<i64>(65535, v.L - a0);
    dim3 grid{unsigned(ceil_div(v.R, kDBM)), unsigned(na), unsigned(ceil_div(cols, BN))};
    const double* Xa = X + a0 * v.I * v.R;
    double* Oa = O + a0 * cols * v.R;
#define RCPG_PJ(BNV)                                                                                       \
  case BNV:                                                                                                \
    if (va && vb)                                                                                          \
      launch_project<BNV, true, true>(grid, Xa, Q, v, cols, ldq, Oa, st);                                  \
    else if (va)                                                                                           \
      launch_project<BNV, true, false>(grid, Xa, Q, v, cols, ldq, Oa, st);                                 \
    else                                                                                                   \
      launch_project<BNV, false, false>(grid, Xa, Q, v, cols, ldq, Oa, st);                                \
    break;
    switch (BN) {
      RCPG_PJ(16)
      RCPG_PJ(32)
      RCPG_PJ(48)
      RCPG_PJ(64)
      default:
        RCPG_PJ(80)
    }
#undef RCPG_PJ
  }
}

// ------------------------------------------------ fp32 X, fp64 arithmetic
// The fp32 configs' faithful passes: X stays fp32 in HBM, every product and
// sum is fp64 (DMMA), so the Scalar-rounded results equal the oracle's
// double-accumulated GEMMs (the checker's gemm_nn / gemm_tn) except where
// the exact sum lies within fp64 rounding of a float rounding boundary.
i64 sketch_dmma_f32_splits(ModeView v, i64 cols, int num_sms, i64& tps, i64& total) {
  return sketch_dmma_splits_t<float>(v, cols, num_sms, tps, total);
}

bool sketch_dmma_f32(const float* X, ModeView v, const double* P, i64 cols, double* part, int num_sms,
                     const int* skip, cudaStream_t st) {
  i64 tps, total;
  const i64 splits = sketch_dmma_f32_splits(v, cols, num_sms, tps, total);
  return sketch_tma_dispatch<float>(X, v, P, cols, part, tps, total, splits, skip, st);
}

bool project_dmma_f32(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, float* O, cudaStream_t st) {
  return project_tma_dispatch<float, float>(X, v, Q, ldq, cols, O, st);
}

bool project_dmma_f32(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, double* O, cudaStream_t st) {
  return project_tma_dispatch<float, double>(X, v, Q, ldq, cols, O, st);
}

}  // namespace rcpg
