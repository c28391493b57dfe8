// Per-step MMA-issue pattern of passes_tc.cu in isolation: 12 MMAs (tf32,
// A TMEM, B smem SW128, 128x80x8) per step, rotating A slots / B stages, with
// 0, 1 or 3 tcgen05.commit per step and optional fence::after_thread_sync.
#include <cstdio>
#include "tc.cuh"
using namespace rcpg::tc;
constexpr int N = 80;
__global__ void k(int commits, int rot, int steps, long long* cyc) {
  const int fence = 0;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int e = tid; e < 6 * 2 * N * 128 / 4; e += blockDim.x) reinterpret_cast<float*>(sm)[e] = 1.0f;
  if (tid == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (tid < 32) tmem_alloc(&tbase, 512);
  fence_proxy_async(); fence_before_sync(); __syncthreads(); fence_after_sync();
  const uint32_t tmem = tbase, b = smem_u32(sm);
  if (tid == 0) {
    const uint32_t id = idesc_tf32(128, N, 0, 0);
    const long long t0 = clock64();
    for (int q = 0; q < steps; ++q) {
      if (fence) fence_after_sync();
      const uint32_t ahi = tmem + 192 + ((rot & 1) ? (q % 5) * 64 : 0), alo = ahi + 32;
      const uint32_t bh0 = b + ((rot & 2) ? (q % 6) * 2 * N * 128 : 0), bl0 = bh0 + N * 128;
      const uint32_t d = tmem + ((rot & 4) ? 96 * (q & 1) : 0);
      for (int k8 = 0; k8 < 4; ++k8) {
        mma_tf32_ta(d, alo + 8 * k8, sdesc_sw128(bh0 + 32 * k8), id, 1);
        mma_tf32_ta(d, ahi + 8 * k8, sdesc_sw128(bl0 + 32 * k8), id, 1);
        mma_tf32_ta(d, ahi + 8 * k8, sdesc_sw128(bh0 + 32 * k8), id, 1);
      }
      for (int c = 0; c < commits; ++c) mma_commit(&bar[c]);
    }
    mma_commit(&bar[3]);
    mbar_wait(&bar[3], 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (tid < 32) tmem_dealloc(tmem, 512);
}
int main() {
  long long* dc; cudaMalloc(&dc, 148 * 8);
  const int smem = 6 * 2 * N * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int commits : {0, 1})
    for (int fence : {0, 1, 2, 3, 4, 7}) {
      k<<<148, 128, smem>>>(commits, fence, 4000, dc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
      long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      printf("commits/step=%d rot(A=1,B=2,D=4)=%d: %.1f cycles/step (%.1f per MMA)\n", commits, fence, double(c) / 4000, double(c) / 48000);
    }
  return 0;
}
