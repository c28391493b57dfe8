// Pins the tcgen05 kind::tf32 encodings used by csrc/passes_tc.cu:
//  (1) K-major A / K-major B, SWIZZLE_NONE core matrices, M=128, N in {16, 80, 128}, K=32 (4 MMAs)
//  (2) MN-major A / K-major B
//  (3) whether the tensor core truncates or rounds fp32 -> tf32 on input
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_1703_09074_b200/csrc umma_tf32.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "tc.cuh"

using namespace rcpg::tc;

constexpr int M = 128, K = 32;

// A: M x K (element (m, k) at A[m*K + k]); B: N x K (element (n, k) at B[n*K + k]).
// D[m][n] = sum_k A(m,k) B(n,k)
template <bool A_MN>
__global__ void one_gemm(const float* A, const float* B, int N, float* D, int KS, int MS, int LBO, int SBO) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  float* sA = reinterpret_cast<float*>(sm);
  float* sB = sA + M * K;
  const int tid = threadIdx.x;
  // fill A
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    int off;
    if (!A_MN)
      off = (m / 8) * ((K / 4) * 128) + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4;
    else if (MS >= 0)
      off = (k / 8) * KS + (m / 4) * MS + (k % 8) * 16 + (m % 4) * 4;
    else {  // MN-major SWIZZLE_128B: atom = 8 k-rows x 128 B (32 m); m-groups LBO apart, k-groups SBO apart
      const int r = k % 8, c = (m % 32) / 4;
      off = (m / 32) * 1024 + (k / 8) * 4096 + r * 128 + ((c ^ r) * 16) + (m % 4) * 4;
    }
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(sA) + off) = A[e];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    const int off = (n / 8) * ((K / 4) * 128) + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4;
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(sB) + off) = B[e];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tbase, 128);
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, N, A_MN ? 1 : 0, 0);
    for (int j = 0; j < K / 8; ++j) {
      uint64_t ad, bd;
      if (!A_MN)
        ad = sdesc(smem_u32(sA) + j * 256, 128, (K / 4) * 128);
      else
        ad = sdesc(smem_u32(sA) + j * KS, LBO, SBO) | (MS < 0 ? (uint64_t(2) << 61) : 0);
      bd = sdesc(smem_u32(sB) + j * 256, 128, (K / 4) * 128);
      mma_tf32(tmem, ad, bd, id, j > 0);
    }
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
  if (tid < 32) tmem_dealloc(tmem, 128);
}

static float tf32_trunc(float x) {
  unsigned u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}
static float tf32_rne(float x) {
  unsigned u;
  memcpy(&u, &x, 4);
  u += 0xFFFu + ((u >> 13) & 1u);
  u &= 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

int run(bool amn, int N, int mode, int KS = 4096, int MS = 128, int LBO = 4096, int SBO = 128) {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1234 + N);
  for (auto& x : A) x = (mode == 0) ? float(rand() % 17 - 8) : 1.0f + float(rand() % 8192) * (1.0f / 8388608.0f);
  for (auto& x : B) x = (mode == 0) ? float(rand() % 13 - 6) : 1.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xFF, D.size() * 4);
  const int smem = (M + N) * K * 4;
  if (amn) {
    cudaFuncSetAttribute(one_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    one_gemm<true><<<1, 128, smem>>>(dA, dB, N, dD, KS, MS, LBO, SBO);
  } else {
    cudaFuncSetAttribute(one_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    one_gemm<false><<<1, 128, smem>>>(dA, dB, N, dD, 0, 0, 0, 0);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("A_MN=%d N=%d: CUDA error %s\n", amn, N, cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double err_exact = 0, err_trunc = 0, err_rne = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0, st = 0, sr = 0;
      for (int k = 0; k < K; ++k) {
        s += double(A[m * K + k]) * B[n * K + k];
        st += double(tf32_trunc(A[m * K + k])) * tf32_trunc(B[n * K + k]);
        sr += double(tf32_rne(A[m * K + k])) * tf32_rne(B[n * K + k]);
      }
      const double d = D[m * N + n];
      err_exact = fmax(err_exact, fabs(d - s));
      err_trunc = fmax(err_trunc, fabs(d - st));
      err_rne = fmax(err_rne, fabs(d - sr));
    }
  printf("KS=%d MS=%d LBO=%d SBO=%d A_MN=%d N=%3d mode=%d: max|D-exact|=%.3e  max|D-trunc|=%.3e  max|D-rne|=%.3e  D[0]=%.9g\n", KS, MS, LBO, SBO, amn, N, mode,
         err_exact, err_trunc, err_rne, D[0]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return 0;
}

int main() {
  int bad = 0;
  for (int N : {16, 80}) bad |= run(false, N, 0);
  bad |= run(true, 80, 0, 4096, 128, 4096, 128);
  bad |= run(true, 80, 0, 4096, 128, 128, 4096);
  bad |= run(true, 80, 0, 128, 512, 128, 512);
  bad |= run(true, 80, 0, 128, 512, 512, 128);
  bad |= run(true, 80, 0, 4096, -1, 1024, 4096);
  bad |= run(true, 80, 0, 4096, -1, 4096, 1024);
  bad |= run(true, 128, 0, 4096, -1, 1024, 4096);
  bad |= run(false, 16, 1);  // rounding probe: low mantissa bits set in A
  return bad;
}
