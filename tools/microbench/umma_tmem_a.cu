// tcgen05.mma kind::tf32 with the A operand in TMEM (written by tcgen05.st,
// lane = row m, one tf32 per 32-bit column) and B in smem (K-major
// SWIZZLE_128B): correctness for N in {16, 80, 128} and back-to-back rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_1703_09074_b200/csrc umma_tmem_a.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "tc.cuh"

using namespace rcpg::tc;

constexpr int M = 128, K = 32;
constexpr uint32_t ACOL = 256;  // A at TMEM columns [256, 288)

__global__ void ta_kernel(const float* A, const float* B, int N, int iters, float* D, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32;
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K, c = k / 4;
    *reinterpret_cast<float*>(sm + (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) * 16) + (k % 4) * 4) = B[e];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (w == 0) tmem_alloc(&tbase, 512);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tbase;
  {
    float v[32];
    const int m = w * 32 + lane;
    for (int k = 0; k < 32; ++k) v[k] = A[m * K + k];
    tmem_st32(tmem + (uint32_t(w * 32) << 16) + ACOL, v);
    tmem_st_wait();
  }
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  const uint32_t id = idesc_tf32(M, N, 0, 0);
  const uint32_t b = smem_u32(sm);
  if (tid == 0) {
    fence_after_sync();
    for (int j = 0; j < K / 8; ++j)
      mma_tf32_ta(tmem, tmem + ACOL + 8 * j, sdesc(b + j * 32, 16, 1024) | (uint64_t(2) << 61), id, j > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after_sync();
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tmem_ld8(tmem + (uint32_t(w * 32) << 16) + c, v);
    for (int q = 0; q < 8; ++q) D[(w * 32 + lane) * N + c + q] = v[q];
  }
  fence_before_sync();
  __syncthreads();
  if (tid == 0) {
    fence_after_sync();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int j = 0; j < K / 8; ++j)
        mma_tf32_ta(tmem + 128, tmem + ACOL + 8 * j, sdesc(b + j * 32, 16, 1024) | (uint64_t(2) << 61), id, 1);
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    cyc[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (w == 0) tmem_dealloc(tmem, 512);
}

int main() {
  const int iters = 2000;
  int bad = 0;
  for (int N : {16, 48, 80, 128}) {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    srand(5);
    for (auto& x : A) x = float(rand() % 17 - 8);
    for (auto& x : B) x = float(rand() % 13 - 6);
    float *dA, *dB, *dD;
    long long* dc;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMalloc(&dc, 148 * 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const int smem = N * K * 4;
    cudaFuncSetAttribute(ta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    ta_kernel<<<148, 128, smem>>>(dA, dB, N, iters, dD, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("N=%d: %s\n", N, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += double(A[m * K + k]) * B[n * K + k];
        err = fmax(err, fabs(s - D[m * N + n]));
      }
    long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    const double per = double(c) / (iters * 4.0);
    printf("A in TMEM: N=%3d err=%.1e  %.1f cycles/MMA(128x%dx8)  %.0f MAC/clk/SM\n", N, err, per, N,
           double(M) * N * 8 / per);
    bad |= err != 0;
  }
  return bad;
}
