// (1) one issuing warp alternating between nd accumulators; (2) accumulator at
// column 80 (not 32-aligned): correctness of a K=32 product there.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cstdlib>
#include "tc.cuh"
using namespace rcpg::tc;
constexpr int N = 80;
__global__ void k(int nd, int steps, long long* cyc, const float* A, const float* B, float* D, int dcol) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32;
  for (int e = tid; e < N * 32; e += blockDim.x) {
    const int r = e / 32, kk = e % 32;
    *reinterpret_cast<float*>(sm + sw128_offset(r, kk)) = B[e];
  }
  if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  if (w == 0) tmem_alloc(&tbase, 512);
  fence_proxy_async(); fence_before_sync(); __syncthreads(); fence_after_sync();
  const uint32_t tmem = tbase, b = smem_u32(sm);
  {
    float v[32];
    for (int kk = 0; kk < 32; ++kk) v[kk] = A[(w * 32 + lane) * 32 + kk];
    tmem_st32(tmem + tmem_lane(w) + 448, v);
    tmem_st_wait();
  }
  fence_before_sync(); __syncthreads();
  const uint32_t id = idesc_tf32(128, N, 0, 0);
  if (tid == 0) {
    fence_after_sync();
    for (int j = 0; j < 4; ++j) mma_tf32_ta(tmem + dcol, tmem + 448 + 8 * j, sdesc_sw128(b + 32 * j), id, j > 0);
    mma_commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  fence_after_sync();
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tmem_ld8(tmem + tmem_lane(w) + dcol + c, v);
    for (int q = 0; q < 8; ++q) D[(w * 32 + lane) * N + c + q] = v[q];
  }
  fence_before_sync(); __syncthreads();
  if (tid == 0) {
    fence_after_sync();
    const long long t0 = clock64();
    for (int q = 0; q < steps; ++q)
#pragma unroll
      for (int j = 0; j < 12; ++j) mma_tf32_ta(tmem + 96 * (j % nd), tmem + 448 + 8 * (j & 3), sdesc_sw128(b), id, 1);
    mma_commit(&bar[1]);
    mbar_wait(&bar[1], 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (w == 0) tmem_dealloc(tmem, 512);
}
int main() {
  long long* dc; cudaMalloc(&dc, 148 * 8);
  std::vector<float> A(128 * 32), B(N * 32), D(128 * N);
  srand(3);
  for (auto& x : A) x = float(rand() % 17 - 8);
  for (auto& x : B) x = float(rand() % 13 - 6);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = N * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int dcol : {0, 80, 160, 240, 16}) for (int nd : {1, 2, 4}) {
    k<<<148, 128, smem>>>(nd, 2000, dc, dA, dB, dD, dcol);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
      double s = 0; for (int kk = 0; kk < 32; ++kk) s += double(A[m * 32 + kk]) * B[n * 32 + kk];
      err = fmax(err, fabs(s - D[m * N + n]));
    }
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("dcol=%3d err=%.1e | 1 warp alternating %d accumulators: %.1f cycles/MMA\n", dcol, err, nd, double(c) / 24000);
  }
  return 0;
}
