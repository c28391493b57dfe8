// Is the ~45-cycle tf32 MMA floor (M=128, small N) a per-issuing-warp limit or
// a tensor-pipe limit? 1 vs 2 vs 4 issuing warps, each into its own accumulator.
#include <cstdio>
#include "tc.cuh"
using namespace rcpg::tc;
template <int N>
__global__ void k(int nwarps, int steps, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32;
  for (int e = tid; e < 2 * N * 128 / 4; e += blockDim.x) reinterpret_cast<float*>(sm)[e] = 1.0f;
  if (tid == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (w == 0) tmem_alloc(&tbase, 512);
  fence_proxy_async(); fence_before_sync(); __syncthreads(); fence_after_sync();
  const uint32_t tmem = tbase, b = smem_u32(sm);
  if (w < nwarps && lane == 0) {
    const uint32_t id = idesc_tf32(128, N, 0, 0);
    const uint32_t d = tmem + w * 96;
    const uint32_t a = tmem + 384 + 8 * w;
    const uint64_t bd = sdesc_sw128(b);
    const long long t0 = clock64();
    for (int q = 0; q < steps; ++q) {
#pragma unroll
      for (int j = 0; j < 12; ++j) mma_tf32_ta(d, a, bd, id, 1);
    }
    mma_commit(&bar[w]);
    mbar_wait(&bar[w], 0);
    cyc[blockIdx.x * 4 + w] = clock64() - t0;
  }
  __syncthreads();
  if (w == 0) tmem_dealloc(tmem, 512);
}
template <int N>
void run(long long* dc) {
  const int smem = 2 * N * 128 + 1024;
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int nw : {1, 2, 4}) {
    k<N><<<148, 128, smem>>>(nw, 2000, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return; }
    long long c[4]; cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < nw; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("N=%3d issuing warps=%d: %.1f cycles per MMA (all warps' MMAs / wall)\n", N, nw, double(mx) / (2000.0 * 12 * nw));
  }
}
int main() {
  long long* dc; cudaMalloc(&dc, 148 * 4 * 8);
  run<16>(dc); run<80>(dc); run<96>(dc);
  return 0;
}
