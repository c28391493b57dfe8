// TMA streaming-rate probe for the fp32 sketch's X feed: a 1024 x 1M fp32 view
// (4 GiB, rows 4 MiB apart, the C3 mode-0 sketch) streamed by one producer
// thread per CTA through an S-stage mbarrier ring; one consumer warp only
// waits and frees the stage. Variants: rows per box, consecutive K boxes per
// stage (contiguous bytes per row), stages, CTAs per SM, and a contiguous view.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu -lcuda
#include <cuda.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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
__device__ __forceinline__ void tma2(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}

// item = (m-tile fastest, K split); stage = NB boxes of {32, BR} at consecutive K
template <int BR, int NB, int S, int ORD>
__global__ void __launch_bounds__(64) stream(const __grid_constant__ CUtensorMap mx, i64 mtiles, i64 kt_total, i64 tps,
                                             i64 items, int* sink) {
  constexpr int BOX = BR * 128, STAGE = NB * BOX;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S], empty[S];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  int q = 0;
  int acc = 0;
  for (i64 id = blockIdx.x; id < items; id += gridDim.x) {
    const i64 nsp = items / mtiles;
    const i64 mt = ORD == 2 ? id / nsp : id % mtiles, sp = ORD == 2 ? id % nsp : id / mtiles;
    const i64 k0 = sp * tps, k1 = k0 + tps < kt_total ? k0 + tps : kt_total;
    const i64 len = k1 - k0;
    const i64 rot = ORD == 1 ? (mt * (len / NB) / mtiles) * NB : 0;
    for (i64 j = 0; j < len; j += NB, ++q) {
      i64 kt = k0 + j + rot;
      if (kt >= k1) kt -= len;
      if (ORD == 3) {  // G interleaved streams, len / G apart
        constexpr int G = 8;
        const i64 jj = j / NB, per = (len / NB + G - 1) / G;
        const i64 t = (jj % G) * per + jj / G;
        kt = k0 + (t < len / NB ? t : jj) * NB;
      } else if (ORD == 4) {  // stride permutation (P coprime to the tile count)
        const i64 n = len / NB;
        i64 P = 37;
        while (n % P == 0) P += 2;
        kt = k0 + ((j / NB) * P % n) * NB;
      }
      const int s = q % S;
      if (w == 0) {
        if (lane == 0) {
          if (q >= S) mbar_wait(&empty[s], uint32_t(((q / S) - 1) & 1));
          mbar_arrive_tx(&full[s], STAGE);
#pragma unroll
          for (int b = 0; b < NB; ++b) tma2(smem + s * STAGE + b * BOX, &mx, int((kt + b) * 32), int(mt * BR), &full[s]);
        }
      } else {
        mbar_wait(&full[s], uint32_t((q / S) & 1));
        acc += smem[s * STAGE + lane * 4];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
  }
  if (acc == 123456789) *sink = acc;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn enc() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  return reinterpret_cast<EncodeFn>(f);
}

template <int BR, int NB, int S, int ORD = 0>
void run(const char* name, float* X, i64 rows, i64 cols, int cps, CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  CUtensorMap m;
  const cuuint64_t d[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t st[1] = {cuuint64_t(cols) * 4};
  const cuuint32_t box[2] = {32, BR};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("%s: encode failed %d\n", name, int(r));
    return;
  }
  const int smem = NB * BR * 128 * S + 1024;
  cudaFuncSetAttribute(stream<BR, NB, S, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const i64 mtiles = rows / BR, kt_total = cols / 32;
  const int grid = 148 * cps;
  i64 splits = (8 * 148 + mtiles - 1) / mtiles;
  i64 tps = (kt_total + splits - 1) / splits;
  tps = (tps + NB - 1) / NB * NB;
  splits = (kt_total + tps - 1) / tps;
  const i64 items = mtiles * splits;
  int* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int it = 0; it < 2; ++it) stream<BR, NB, S, ORD><<<grid, 64, smem>>>(m, mtiles, kt_total, tps, items, sink);
  cudaEventRecord(a);
  const int reps = 5;
  for (int it = 0; it < reps; ++it) stream<BR, NB, S, ORD><<<grid, 64, smem>>>(m, mtiles, kt_total, tps, items, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, stream<BR, NB, S, ORD>, 64, smem);
  printf("%-36s ord %d box {32,%3d} x%d S=%2d stage %3d KB cps=%d (occ %d): %7.1f us  %6.2f TB/s %s\n", name, ORD, BR, NB, S,
         NB * BR * 128 / 1024, cps, nb, 1e3 * ms / reps, double(rows * cols * 4) * reps / (ms * 1e-3) / 1e12,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(sink);
}

int main() {
  const i64 rows = 1024, cols = i64(1) << 20;
  float* X;
  if (cudaMalloc(&X, size_t(rows * cols * 4)) != cudaSuccess) return 1;
  cudaMemset(X, 0, size_t(rows * cols * 4));
  run<128, 1, 6, 0>("sketch now", X, rows, cols, 1);
  run<128, 1, 6, 3>("sketch, 8 streams", X, rows, cols, 1);
  run<128, 1, 6, 4>("sketch, stride perm", X, rows, cols, 1);
  run<128, 1, 4, 4>("sketch, stride perm, 3 CTAs", X, rows, cols, 3);
  run<128, 1, 12, 4>("sketch, stride perm, S12", X, rows, cols, 1);
  run<128, 1, 6, 0>("C4 mode0 now", X, 128, 8388608, 1);
  run<128, 1, 6, 3>("C4 mode0 8 streams", X, 128, 8388608, 1);
  run<128, 1, 6, 4>("C4 mode0 stride perm", X, 128, 8388608, 1);
  run<128, 1, 6, 0>("C5 mode0 now", X, 2000, 500000, 1);
  run<128, 1, 6, 4>("C5 mode0 stride perm", X, 2000, 500000, 1);
  run<128, 1, 6, 0>("4KB rows", X, cols, rows, 1);
  run<128, 1, 6, 4>("4KB rows stride perm", X, cols, rows, 1);
  run<128, 1, 6, 0>("contiguous 16KB boxes", X, rows * cols / 32, 32, 1);
  return 0;
}
