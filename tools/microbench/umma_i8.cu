// tcgen05.mma kind::i8 (s8 x s8 -> s32): A in TMEM (lane = row m, four int8
// K-elements per 32-bit column, K = 32 per MMA -> 8 columns) or in smem, B in
// smem (K-major SWIZZLE_128B, 128 int8 per row atom, +32 B per K32 step):
// correctness for several N and the back-to-back rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_1703_09074_b200/csrc umma_i8.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc.cuh"

using namespace rcpg::tc;

constexpr int M = 128, K = 128;  // four K32 steps
constexpr uint32_t ACOL = 256;   // A at TMEM columns [256, 288)

__host__ __device__ constexpr uint32_t idesc_i8(int M_, int N_) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N_ >> 3) << 17) | (uint32_t(M_ >> 4) << 24);
}

__device__ __forceinline__ void mma_i8_ta(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

// byte offset of int8 element (r, k) in a K-major SW128 tile (128 B rows)
__host__ __device__ constexpr int sw128_b(int r, int k) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 4) ^ (r & 7))) << 4) + (k & 15);
}

__global__ void i8_kernel(const int8_t* A, const int8_t* B, int N, int iters, int a_tmem, int* D, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32;
  unsigned char* sA = sm;               // M x 128 B
  unsigned char* sB = sm + M * 128;     // N x 128 B
  for (int e = tid; e < M * K; e += blockDim.x) sA[sw128_b(e / K, e % K)] = (unsigned char)A[e];
  for (int e = tid; e < N * K; e += blockDim.x) sB[sw128_b(e / K, e % K)] = (unsigned char)B[e];
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
    // row m = 32 w + lane: 128 int8 = 32 words, word c holds k = 4c..4c+3
    float v[32];
    const int m = w * 32 + lane;
    for (int c = 0; c < 32; ++c) {
      uint32_t u = 0;
      for (int q = 0; q < 4; ++q) u |= uint32_t((unsigned char)A[m * K + 4 * c + q]) << (8 * q);
      v[c] = __uint_as_float(u);
    }
    tmem_st32(tmem + (uint32_t(w * 32) << 16) + ACOL, v);
    tmem_st_wait();
  }
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  const uint32_t id = idesc_i8(M, N);
  const uint32_t a = smem_u32(sA), b = smem_u32(sB);
  if (tid == 0) {
    fence_after_sync();
    for (int j = 0; j < K / 32; ++j) {
      if (a_tmem)
        mma_i8_ta(tmem, tmem + ACOL + 8 * j, sdesc_sw128(b + j * 32), id, j > 0);
      else
        mma_i8_ss(tmem, sdesc_sw128(a + j * 32), sdesc_sw128(b + j * 32), id, j > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after_sync();
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tmem_ld8(tmem + (uint32_t(w * 32) << 16) + c, v);
    for (int q = 0; q < 8; ++q) D[(w * 32 + lane) * N + c + q] = __float_as_int(v[q]);
  }
  fence_before_sync();
  __syncthreads();
  if (tid == 0) {
    fence_after_sync();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int j = 0; j < K / 32; ++j) {
        if (a_tmem)
          mma_i8_ta(tmem + 128, tmem + ACOL + 8 * j, sdesc_sw128(b + j * 32), id, 1);
        else
          mma_i8_ss(tmem + 128, sdesc_sw128(a + j * 32), sdesc_sw128(b + j * 32), id, 1);
      }
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
  for (int a_tmem : {0, 1})
    for (int N : {16, 32, 64, 128}) {
      std::vector<int8_t> A(M * K), B(N * K);
      std::vector<int> D(M * N);
      srand(7 + N);
      for (auto& x : A) x = int8_t(rand() % 255 - 127);
      for (auto& x : B) x = int8_t(rand() % 255 - 127);
      int8_t *dA, *dB;
      int* dD;
      long long* dc;
      cudaMalloc(&dA, A.size());
      cudaMalloc(&dB, B.size());
      cudaMalloc(&dD, D.size() * 4);
      cudaMalloc(&dc, 148 * 8);
      cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
      cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
      const int smem = (M + N) * 128;
      cudaFuncSetAttribute(i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      i8_kernel<<<148, 128, smem>>>(dA, dB, N, iters, a_tmem, dD, dc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("N=%d: %s\n", N, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      long long maxerr = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          long long s = 0;
          for (int k = 0; k < K; ++k) s += int(A[m * K + k]) * int(B[n * K + k]);
          maxerr = std::max(maxerr, std::llabs(s - D[m * N + n]));
        }
      long long c = 0;
      cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      const double per = double(c) / (iters * 4.0);
      printf("i8 A in %s: N=%3d maxerr=%lld  %.1f cycles/MMA(128x%dx32)  %.0f MAC/clk/SM\n", a_tmem ? "TMEM" : "smem",
             N, maxerr, per, N, double(M) * N * 32 / per);
      bad |= maxerr != 0;
    }
  return bad;
}
