// tcgen05.mma kind::tf32 throughput from shared memory: back-to-back MMAs
// (M = 128, N, K = 8) on resident tiles, K-major, SWIZZLE_NONE vs SWIZZLE_128B.
// Also checks SWIZZLE_128B K-major correctness (one K = 32 product).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_1703_09074_b200/csrc umma_rate.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#include "tc.cuh"

using namespace rcpg::tc;

constexpr int M = 128, K = 32;

// byte offset of element (r, k) of a K-major rows x 32 tf32 tile
__host__ __device__ int off_kmajor(int r, int k, bool sw) {
  if (!sw) return (r / 8) * ((K / 4) * 128) + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4;
  // SWIZZLE_128B atom: 8 rows x 128 B (32 tf32), chunk c of row r at ((c ^ r%8) * 16)
  const int c = k / 4;
  return (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) * 16) + (k % 4) * 4;
}

__device__ uint64_t desc_for(uint32_t base, int k8, bool sw) {
  if (!sw) return sdesc(base + k8 * 256, 128, (K / 4) * 128);
  return sdesc(base + k8 * 32, 16, 1024) | (uint64_t(2) << 61);
}

__global__ void rate_kernel(const float* A, const float* B, int N, bool sw, int iters, float* D, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  float* sA = reinterpret_cast<float*>(sm);
  float* sB = reinterpret_cast<float*>(sm + M * K * 4);
  const int tid = threadIdx.x;
  for (int e = tid; e < M * K; e += blockDim.x)
    *reinterpret_cast<float*>(sm + off_kmajor(e / K, e % K, sw)) = A[e];
  for (int e = tid; e < N * K; e += blockDim.x)
    *reinterpret_cast<float*>(sm + M * K * 4 + off_kmajor(e / K, e % K, sw)) = B[e];
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tbase, 256);
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tbase;
  const uint32_t id = idesc_tf32(M, N, 0, 0);
  const uint32_t a = smem_u32(sA), b = smem_u32(sB);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    // correctness: one K = 32 product into columns [0, N)
    for (int j = 0; j < K / 8; ++j) mma_tf32(tmem, desc_for(a, j, sw), desc_for(b, j, sw), id, j > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after_sync();
  const int w = tid / 32, lane = tid % 32;
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tmem_ld8(tmem + (uint32_t(w * 32) << 16) + c, v);
    for (int q = 0; q < 8; ++q) D[(w * 32 + lane) * N + c + q] = v[q];
  }
  fence_before_sync();
  __syncthreads();
  if (tid == 0) {
    fence_after_sync();
    t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int j = 0; j < K / 8; ++j) mma_tf32(tmem + 128, desc_for(a, j, sw), desc_for(b, j, sw), id, 1);
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (tid < 32) tmem_dealloc(tmem, 256);
}

int main() {
  const int iters = 2000;
  for (int sw = 0; sw < 2; ++sw)
    for (int N : {16, 64, 80, 128}) {
      std::vector<float> A(M * K), B(N * K), D(M * N);
      srand(7);
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
      const int smem = 1024 + (M + N) * K * 4;
      cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int grid : {1, 148}) {
        rate_kernel<<<grid, 128, smem>>>(dA, dB, N, sw, iters, dD, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("sw=%d N=%d: %s\n", sw, N, cudaGetErrorString(e));
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
        const double macs = double(M) * N * 8 / per;
        printf("sw128=%d N=%3d grid=%3d: err=%.1e  %.1f cycles/MMA(128x%dx8)  %.0f MAC/clk/SM  (%.2f PF tf32 @1.9GHz x148)\n",
               sw, N, grid, err, per, N, macs, macs * 2 * 1.9e9 * 148 / 1e15);
      }
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dD);
      cudaFree(dc);
    }
  return 0;
}
