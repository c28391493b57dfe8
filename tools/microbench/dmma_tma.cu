// TMA-fed FP64 DMMA sketch Y[i,c] = sum_{a,b} X[a,i,b] P[a,c,b]: one producer
// warp streams 128B-swizzled K-tiles (16 doubles) of X and P through an
// S-stage mbarrier ring; WM consumer warps (16 rows each) run mma.m16n8k4.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_tma dmma_tma.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstdint>
typedef long long i64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b0));
}
// element (r, k) of a 128B-swizzled box with 16-double rows
__device__ __forceinline__ int swz(int r, int k) { return r * 16 + ((((k >> 1) ^ (r & 7))) << 1) + (k & 1); }

template <int WM, int BN, int S, int ACC, int WK>
__global__ void __launch_bounds__((WM * WK + 1) * 32) sk_tma(const __grid_constant__ CUtensorMap mx,
                                                        const __grid_constant__ CUtensorMap mp, i64 I, i64 cols,
                                                        i64 nbt, i64 tps, i64 total, double* __restrict__ part) {
  constexpr int BM = WM * 16, NT = BN / 8, ABYTES = BM * 128, BBYTES = BN * 128, STAGE = ABYTES + BBYTES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const i64 t0 = blockIdx.y * tps;
  const i64 t1 = t0 + tps < total ? t0 + tps : total;
  const int nk = int(t1 - t0);
  const int m0 = blockIdx.x * BM, n0 = blockIdx.z * BN;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WM * WK);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  if (w == WM * WK) {  // producer
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % S;
        if (kt >= S) mbar_wait(&empty[s], uint32_t(((kt / S) - 1) & 1));
        const i64 tt = t0 + kt, a = tt / nbt, b0 = (tt - a * nbt) * 16;
        mbar_arrive_tx(&full[s], STAGE);
        unsigned char* st = smem + s * STAGE;
        tma3(st, &mx, int(b0), m0, int(a), &full[s]);
        tma3(st + ABYTES, &mp, int(b0), n0, int(a), &full[s]);
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  double acc[ACC][NT][4];
#pragma unroll
  for (int q = 0; q < ACC; ++q)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[q][j][0] = acc[q][j][1] = acc[q][j][2] = acc[q][j][3] = 0.0;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % S;
    mbar_wait(&full[s], uint32_t((kt / S) & 1));
    const double* A = reinterpret_cast<const double*>(smem + s * STAGE);
    const double* B = reinterpret_cast<const double*>(smem + s * STAGE + ABYTES);
    const int r0 = (w % WM) * 16 + g;
#pragma unroll
    for (int kk = (w / WM) * 4; kk < 16; kk += 4 * WK) {
      const double a0 = A[swz(r0, kk + t)];
      const double a1 = A[swz(r0 + 8, kk + t)];
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[(kk >> 2) % ACC][j], a0, a1, B[swz(j * 8 + g, kk + t)]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int q = 1; q < ACC; ++q)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[0][j][e] += acc[q][j][e];
  if (WK > 1) {
    // k-groups > 0 park their accumulators in the (drained) stage ring, group 0 adds them in order
    asm volatile("bar.sync 1, %0;\n" ::"r"(WM * WK * 32));
    double* red = reinterpret_cast<double*>(smem);
    if (w >= WM)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) red[((w - WM) * 32 + lane) * NT * 4 + j * 4 + e] = acc[0][j][e];
    asm volatile("bar.sync 1, %0;\n" ::"r"(WM * WK * 32));
    if (w >= WM) return;
    for (int q = 1; q < WK; ++q)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[0][j][e] += red[(((q - 1) * WM + w) * 32 + lane) * NT * 4 + j * 4 + e];
  }
  const i64 r0 = m0 + (w % WM) * 16 + g;
  double* out = part + i64(blockIdx.y) * cols * I;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const i64 c0 = n0 + j * 8 + 2 * t;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const i64 i = r0 + (e >> 1) * 8, c = c0 + (e & 1);
      if (i < I && c < cols) out[c * I + i] = acc[0][j][e];
    }
  }
}

static CUtensorMap tmap3(const double* base, i64 d0, i64 d1, i64 d2, int b0, int b1) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(d2)};
  const cuuint64_t strides[2] = {cuuint64_t(d0) * 8, cuuint64_t(d0 * d1) * 8};
  const cuuint32_t box[3] = {cuuint32_t(b0), cuuint32_t(b1), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
                                      box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", int(r));
  return m;
}

double ref_check(const double* hX, const double* hP, const double* hY, i64 L, i64 I, i64 R, i64 cols) {
  double md = 0;
  for (int i = 0; i < I; i += 37)
    for (int c = 0; c < cols; c += 7) {
      double s = 0;
      for (i64 a = 0; a < L; ++a)
        for (i64 b = 0; b < R; ++b) s += hX[(a * I + i) * R + b] * hP[(a * cols + c) * R + b];
      md = std::max(md, std::fabs(s - hY[c * I + i]) / (1e-30 + std::fabs(s)));
    }
  return md;
}

template <int WM, int BN, int S, int ACC, int WK = 1>
void run(const char* name, const double* X, const double* P, i64 L, i64 I, i64 R, i64 cols, double* part, double* Y,
         int waves, const double* hX, const double* hP) {
  constexpr int BM = WM * 16;
  const size_t smem = size_t(S) * (BM + BN) * 128 + 1024;
  auto k = sk_tma<WM, BN, S, ACC, WK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, (WM * WK + 1) * 32, smem);
  const i64 mt = (I + BM - 1) / BM, nt = (cols + BN - 1) / BN, nbt = (R + 15) / 16, total = L * nbt;
  i64 want = std::max<i64>(1, (waves * i64(per_sm) * 148) / (mt * nt));
  const i64 tps = std::max<i64>(1, (total + want - 1) / want), splits = (total + tps - 1) / tps;
  const CUtensorMap mx = tmap3(X, R, I, L, 16, BM), mp = tmap3(P, R, cols, L, 16, BN);
  dim3 grid{unsigned(mt), unsigned(splits), unsigned(nt)};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<grid, (WM * WK + 1) * 32, smem>>>(mx, mp, I, cols, nbt, tps, total, part);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) k<<<grid, (WM * WK + 1) * 32, smem>>>(mx, mp, I, cols, nbt, tps, total, part);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1e3 * ms / reps;
  // reduce splits on host for a spot check
  double* hpart = (double*)malloc(splits * cols * I * 8);
  cudaMemcpy(hpart, part, splits * cols * I * 8, cudaMemcpyDeviceToHost);
  double* hY = (double*)calloc(cols * I, 8);
  for (i64 q = 0; q < splits; ++q)
    for (i64 e = 0; e < cols * I; ++e) hY[e] += hpart[q * cols * I + e];
  const double err = ref_check(hX, hP, hY, L, I, R, cols);
  free(hpart);
  free(hY);
  printf("%-26s L=%lld I=%lld R=%lld: %7.1f us  %5.1f TF  %6.0f GB/s  occ=%d/SM splits=%lld relerr=%.1e %s\n", name, L, I,
         R, us, 2.0 * L * I * R * cols / us * 1e-6, L * I * R * 8.0 / us * 1e-3, per_sm, splits, err,
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  const i64 N = 400 * 160000;
  double *X, *P, *part;
  if (cudaMalloc(&X, N * 8) || cudaMalloc(&P, 160000 * 32 * 8) || cudaMalloc(&part, 400 * 32 * 4096 * 8)) return 1;
  double* hX = (double*)malloc(N * 8);
  double* hP = (double*)malloc(160000 * 32 * 8);
  for (i64 i = 0; i < N; ++i) hX[i] = ((i * 2654435761ll) % 1000) * 1e-3 - 0.5;
  for (i64 i = 0; i < 160000 * 32; ++i) hP[i] = ((i * 40503ll) % 997) * 1e-3 - 0.5;
  cudaMemcpy(X, hX, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(P, hP, 160000 * 32 * 8, cudaMemcpyHostToDevice);
  struct Shape { i64 L, I, R; } shapes[] = {{1, 400, 160000}, {30, 400, 400}};
  for (auto s : shapes) {
    run<4, 32, 4, 1>("WM4 S4", X, P, s.L, s.I, s.R, 30, part, nullptr, 2, hX, hP);
    run<4, 32, 4, 2>("WM4 S4 ACC2", X, P, s.L, s.I, s.R, 30, part, nullptr, 2, hX, hP);
    run<4, 32, 2, 1>("WM4 S2", X, P, s.L, s.I, s.R, 30, part, nullptr, 2, hX, hP);
    run<5, 32, 3, 1>("WM5 S3", X, P, s.L, s.I, s.R, 30, part, nullptr, 2, hX, hP);
    run<5, 32, 2, 1>("WM5 S2", X, P, s.L, s.I, s.R, 30, part, nullptr, 2, hX, hP);
    run<5, 32, 3, 2>("WM5 S3 ACC2", X, P, s.L, s.I, s.R, 30, part, nullptr, 2, hX, hP);
    run<3, 32, 4, 1>("WM3 S4", X, P, s.L, s.I, s.R, 30, part, nullptr, 2, hX, hP);
    run<5, 32, 3, 1>("WM5 S3 w4", X, P, s.L, s.I, s.R, 30, part, nullptr, 4, hX, hP);
    run<5, 32, 3, 1>("WM5 S3 w1", X, P, s.L, s.I, s.R, 30, part, nullptr, 1, hX, hP);
  }
  return 0;
}
