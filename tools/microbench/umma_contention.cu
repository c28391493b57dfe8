// MMA issue rate (tf32, A in TMEM, B in smem SW128, M=128, N=80, K=8) while
// other warps (a) idle, (b) tcgen05.st 64 columns per round into other TMEM
// columns, (c) stream LDS/STS over a 64 KB smem buffer, (d) both.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_1703_09074_b200/csrc umma_contention.cu
#include <cstdio>
#include "tc.cuh"
using namespace rcpg::tc;

constexpr int N = 80;
__global__ void k(int mode, int iters, long long* cyc, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32;
  for (int e = tid; e < (N * 128 + 65536) / 4; e += blockDim.x) reinterpret_cast<float*>(sm)[e] = 1.0f;
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (w == 1) tmem_alloc(&tbase, 512);
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tbase;
  const uint32_t b = smem_u32(sm);
  float acc = 0;
  if (w == 1) {
    if (lane == 0) {
      const uint32_t id = idesc_tf32(128, N, 0, 0);
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it)
        for (int j = 0; j < 12; ++j)
          mma_tf32_ta(tmem + 128 * (it & 1), tmem + 256 + 8 * (j & 7), sdesc_sw128(b + (j & 3) * 32), id, 1);
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      cyc[blockIdx.x] = clock64() - t0;
      stop = 1;
    }
  } else if (w >= 2) {
    const int qd = w & 3;
    float v[32];
    for (int i = 0; i < 32; ++i) v[i] = float(i + lane);
    int r = 0;
    while (!stop) {
      if (mode & 1) {
        tmem_st32(tmem + tmem_lane(qd) + 384 + (r & 1) * 64, v);
        tmem_st32(tmem + tmem_lane(qd) + 416 + (r & 1) * 64, v);
        tmem_st_wait();
      }
      if (mode & 2) {
        const unsigned char* src = sm + N * 128;
#pragma unroll 4
        for (int e = tid - 64; e < 65536 / 16; e += 128) {
          float4 x = *reinterpret_cast<const float4*>(src + 16 * ((e + r * 7) & 4095));
          acc += x.x;
          *reinterpret_cast<float4*>(const_cast<unsigned char*>(src) + 16 * ((e + r * 13) & 4095)) = x;
        }
      }
      if (mode == 0) __nanosleep(100);
      ++r;
    }
  }
  fence_before_sync();
  __syncthreads();
  if (acc == 12345.f) sink[0] = acc;
  if (w == 1) tmem_dealloc(tmem, 512);
}

int main() {
  long long* dc; float* s;
  cudaMalloc(&dc, 148 * 8); cudaMalloc(&s, 4);
  const int smem = N * 128 + 65536;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"idle", "tcgen05.st", "smem LDS/STS", "both"};
  for (int mode = 0; mode < 4; ++mode) {
    k<<<148, 192, smem>>>(mode, 2000, dc, s);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("%-14s %.1f cycles / MMA (128x%dx8, A TMEM)\n", names[mode], double(c) / (2000 * 12), N);
  }
  return 0;
}
