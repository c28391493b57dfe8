// Latency of dependent fp64 operations on one warp (clock64 around chains).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat fp64_lat.cu
#include <cstdio>

__global__ void lat(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-9;
  long long t0, t1;
  constexpr int N = 256;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  cyc[0] = (t1 - t0) / N;
  // DMUL chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = x * 1.0000001;
  t1 = clock64();
  cyc[1] = (t1 - t0) / N;
  // sqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = sqrt(x) + 1.0;
  t1 = clock64();
  cyc[2] = (t1 - t0) / N;
  // division chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = 3.0 / x + 0.5;
  t1 = clock64();
  cyc[3] = (t1 - t0) / N;
  // rsqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = rsqrt(x) + 1.0;
  t1 = clock64();
  cyc[4] = (t1 - t0) / N;
  // smem round trip (store then dependent load)
  __shared__ double sm[64];
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    sm[threadIdx.x & 31] = x;
    __syncwarp();
    x = sm[(threadIdx.x + 1) & 31] + 1.0;
  }
  t1 = clock64();
  cyc[5] = (t1 - t0) / N;
  // __syncthreads cost (256 threads)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64();
  cyc[6] = (t1 - t0) / N;
  out[threadIdx.x] = x;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1024 * sizeof(double));
  cudaMallocManaged(&c, 16 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) {
    lat<<<1, 256>>>(d, c, 2.0);
    cudaDeviceSynchronize();
  }
  const char* nm[] = {"dfma", "dmul", "sqrt+dadd", "div+dadd", "rsqrt+dadd", "sts+syncwarp+lds+dadd", "syncthreads(256)"};
  for (int i = 0; i < 7; ++i) printf("%-24s %lld cycles\n", nm[i], c[i]);
  return 0;
}
