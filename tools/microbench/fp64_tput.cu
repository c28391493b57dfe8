// Issue throughput of independent fp64 DMUL+DADD (the LU update's pair) and of
// the fp64 compare/select on one SM, by warps per CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_tput fp64_tput.cu
#include <cstdio>

template <int CH>
__global__ void tput(double* out, long long* cyc, double m) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __dsub_rn(x[c], __dmul_rn(m, x[(c + 1) % CH]));
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
__global__ void tput32(float* out, long long* cyc, float m) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fsub_rn(x[c], __fmul_rn(m, x[(c + 1) % CH]));
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 4096 * sizeof(double));
  cudaMallocManaged(&c, 16 * sizeof(long long));
  for (int nt : {32, 128, 256, 416, 512, 1024}) {
    tput<16><<<1, nt>>>(d, c, 1e-9);
    cudaDeviceSynchronize();
    tput<16><<<1, nt>>>(d, c, 1e-9);
    cudaDeviceSynchronize();
    const double pairs = 256.0 * 16 * nt / 32;  // warp-level DMUL+DSUB pairs
    printf("f64 threads %4d: %.2f warp-pairs/clk/SM (%.1f cycles per warp pair)\n", nt, pairs / c[0], c[0] / (256.0 * 16));
    tput32<16><<<1, nt>>>((float*)d, c, 1e-9f);
    cudaDeviceSynchronize();
    printf("f32 threads %4d: %.2f warp-pairs/clk/SM\n", nt, pairs / c[0]);
  }
  return 0;
}
