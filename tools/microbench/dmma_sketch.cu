// Variant sweep for the fp64 sketch pass Y[i,c] = sum_{a,b} X[a,i,b] P[a,c,b] on
// the FP64 tensor cores (mma.sync m16n8k4), C2 shapes. CUDA-event timing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_sketch dmma_sketch.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
typedef long long i64;

__device__ __forceinline__ void cp16(double* dst, const double* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// WM = warps along M (16 rows each), WK = warps splitting each k-tile
template <int WM, int WK, int BN, int BK, int S, int ACC, bool NOLOAD = false, bool V128 = false>
__global__ void __launch_bounds__(WM * WK * 32) sk(const double* __restrict__ X, const double* __restrict__ P, i64 I,
                                                   i64 R, i64 cols, i64 nbt, i64 tps, i64 total,
                                                   double* __restrict__ part) {
  constexpr int BM = WM * 16, NTH = WM * WK * 32, SA = V128 ? BK + 8 : BK + 4, NT = BN / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + S * BM * SA;
  double* red = sB;  // reused after the main loop
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wm = w % WM, wk = w / WM;
  const i64 m0 = i64(blockIdx.x) * BM, n0 = i64(blockIdx.z) * BN;
  const i64 t0 = blockIdx.y * tps;
  const i64 t1 = t0 + tps < total ? t0 + tps : total;
  const int nk = int(t1 - t0);
  auto load = [&](int stage, i64 tt) {
    const i64 a = tt / nbt, b0 = (tt - a * nbt) * BK;
    double* dA = sA + stage * BM * SA;
    double* dB = sB + stage * BN * SA;
    constexpr int CPR = BK / 2;
    for (int e = tid; e < BM * CPR; e += NTH) {
      const int m = e / CPR, k = (e % CPR) * 2;
      const i64 i = m0 + m, b = b0 + k;
      const bool ok = (i < I) && (b < R);
      cp16(dA + m * SA + k, X + (ok ? ((a * I + i) * R + b) : 0), ok);
    }
    for (int e = tid; e < BN * CPR; e += NTH) {
      const int n = e / CPR, k = (e % CPR) * 2;
      const i64 c = n0 + n, b = b0 + k;
      const bool ok = (c < cols) && (b < R);
      cp16(dB + n * SA + k, P + (ok ? ((a * cols + c) * R + b) : 0), ok);
    }
  };
  double acc[ACC][NT][4];
#pragma unroll
  for (int s = 0; s < ACC; ++s)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[s][j][0] = acc[s][j][1] = acc[s][j][2] = acc[s][j][3] = 0.0;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < nk) load(s, t0 + s);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 2));
    __syncthreads();
    const int pre = kt + S - 1;
    if (!NOLOAD && pre < nk) load(pre % S, t0 + pre);
    asm volatile("cp.async.commit_group;\n" ::);
    const double* cA = sA + (kt % S) * BM * SA + (wm * 16) * SA;
    const double* cB = sB + (kt % S) * BN * SA;
    if (V128) {
      // k order permuted per 8: step s uses k = 8 (s >> 1) + 2 t + (s & 1), so a thread's two
      // consecutive steps read one 16-byte pair (same permutation on A and B)
#pragma unroll
      for (int k8 = wk * 8, q = 0; k8 < BK; k8 += 8 * WK, ++q) {
        const double2 a0 = *reinterpret_cast<const double2*>(cA + g * SA + k8 + 2 * t);
        const double2 a1 = *reinterpret_cast<const double2*>(cA + (g + 8) * SA + k8 + 2 * t);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const double2 b = *reinterpret_cast<const double2*>(cB + (j * 8 + g) * SA + k8 + 2 * t);
          dmma(acc[(2 * q) % ACC][j], a0.x, a1.x, b.x);
          dmma(acc[(2 * q + 1) % ACC][j], a0.y, a1.y, b.y);
        }
      }
    } else {
#pragma unroll
    for (int kk = wk * 4, q = 0; kk < BK; kk += 4 * WK, ++q) {
      const double a0 = cA[g * SA + kk + t];
      const double a1 = cA[(g + 8) * SA + kk + t];
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[q % ACC][j], a0, a1, cB[(j * 8 + g) * SA + kk + t]);
    }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
  for (int s = 1; s < ACC; ++s)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[0][j][q] += acc[s][j][q];
  if (WK > 1) {
    __syncthreads();
    // warps wk > 0 park their tiles in smem, warp-group 0 adds them in order
    if (wk > 0)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) red[((wk - 1) * WM * 32 + wm * 32 + lane) * (NT * 4) + j * 4 + q] = acc[0][j][q];
    __syncthreads();
    if (wk > 0) return;
    for (int s = 1; s < WK; ++s)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[0][j][q] += red[((s - 1) * WM * 32 + wm * 32 + lane) * (NT * 4) + j * 4 + q];
  }
  const i64 r0 = m0 + wm * 16 + g;
  double* out = part + i64(blockIdx.y) * cols * I;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const i64 c0 = n0 + j * 8 + 2 * t;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const i64 i = r0 + (q >> 1) * 8, c = c0 + (q & 1);
      if (i < I && c < cols) out[c * I + i] = acc[0][j][q];
    }
  }
}

template <int WM, int WK, int BN, int BK, int S, int ACC, bool NOLOAD = false, bool V128 = false>
void run(const char* name, const double* X, const double* P, i64 L, i64 I, i64 R, i64 cols, double* part, int waves,
         int per_sm_force) {
  constexpr int BM = WM * 16;
  constexpr int NT = BN / 8;
  const size_t smem = std::max<size_t>(size_t(S) * (BM + BN) * (BK + 8) * 8,
                                       size_t(S) * BM * (BK + 8) * 8 + size_t(WK - 1) * WM * 32 * NT * 4 * 8);
  auto k = sk<WM, WK, BN, BK, S, ACC, NOLOAD, V128>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, WM * WK * 32, smem);
  const i64 mt = (I + BM - 1) / BM, nt = (cols + BN - 1) / BN, nbt = (R + BK - 1) / BK, total = L * nbt;
  const i64 slots = i64(per_sm) * 148;
  i64 want = std::max<i64>(1, (waves * slots) / (mt * nt));
  const i64 tps = std::max<i64>(1, (total + want - 1) / want), splits = (total + tps - 1) / tps;
  dim3 grid{unsigned(mt), unsigned(splits), unsigned(nt)};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<grid, WM * WK * 32, smem>>>(X, P, I, R, cols, nbt, tps, total, part);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) k<<<grid, WM * WK * 32, smem>>>(X, P, I, R, cols, nbt, tps, total, part);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1e3 * ms / reps;
  const double fl = 2.0 * L * I * R * cols;
  fflush(stdout);
  printf("%-34s L=%lld I=%lld R=%lld: %7.1f us  %5.1f TF  %6.0f GB/s  occ=%d/SM splits=%lld err=%s\n", name, L, I, R, us,
         fl / us * 1e-6, L * I * R * 8.0 / us * 1e-3, per_sm, splits, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const i64 N = 400 * 160000;
  double *X, *P, *part;
  if (cudaMalloc(&X, N * 8) || cudaMalloc(&P, 160000 * 32 * 8) || cudaMalloc(&part, 400 * 32 * 4096 * 8)) {
    printf("alloc failed\n");
    return 1;
  }
  printf("alloc ok\n");
  fflush(stdout);
  double* h = (double*)malloc(N * 8);
  for (i64 i = 0; i < N; ++i) h[i] = (i % 1000) * 1e-3 - 0.5;
  cudaMemcpy(X, h, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(P, h, 160000 * 32 * 8, cudaMemcpyHostToDevice);
  struct Shape { i64 L, I, R; } shapes[] = {{1, 400, 160000}, {30, 400, 400}};
  for (auto s : shapes) {
    run<4, 1, 32, 16, 4, 1>("cur WM4 WK1 BK16 S4", X, P, s.L, s.I, s.R, 30, part, 2, 0);
    run<4, 1, 32, 16, 4, 1, true>("cur NOLOAD", X, P, s.L, s.I, s.R, 30, part, 2, 0);
    run<5, 1, 32, 16, 4, 2, true>("WM5 ACC2 NOLOAD", X, P, s.L, s.I, s.R, 30, part, 2, 0);
    run<5, 1, 32, 16, 4, 2, true, true>("WM5 ACC2 NOLOAD V128", X, P, s.L, s.I, s.R, 30, part, 2, 0);
    run<5, 1, 32, 16, 4, 2, false, true>("WM5 ACC2 V128", X, P, s.L, s.I, s.R, 30, part, 2, 0);
    run<5, 1, 32, 16, 4, 1, false, true>("WM5 V128", X, P, s.L, s.I, s.R, 30, part, 2, 0);
    run<5, 1, 32, 32, 3, 2, false, true>("WM5 ACC2 V128 BK32 S3", X, P, s.L, s.I, s.R, 30, part, 2, 0);
    run<5, 2, 32, 32, 3, 2, false, true>("WM5 WK2 ACC2 V128 BK32 S3", X, P, s.L, s.I, s.R, 30, part, 2, 0);
    run<5, 1, 32, 16, 3, 2, false, true>("WM5 ACC2 V128 S3", X, P, s.L, s.I, s.R, 30, part, 2, 0);
  }
  return 0;
}
