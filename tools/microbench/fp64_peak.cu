// Measures FP64 issue peaks on the device: SIMT DFMA vs DMMA (mma.sync f64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m16n8k4_kernel(double* out, int iters) {
  double acc[4][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = 0.5;
  double b0 = 0.25;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
                   : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double acc[4][2] = {};
  double a0 = threadIdx.x * 1e-3, b0 = 0.25;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a0), "d"(b0));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += acc[j][0] + acc[j][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int threads : {256, 512, 1024}) {
      dim3 grid(sms * 2);
      float ms;
      cudaEventRecord(a);
      dfma_kernel<<<grid, threads>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      double fl = 2.0 * 8 * iters * double(grid.x) * threads;
      printf("DFMA threads=%d: %.1f TFLOPS\n", threads, fl / ms / 1e9);
      cudaEventRecord(a);
      dmma_m16n8k4_kernel<<<grid, threads>>>(out, iters / 8);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      fl = 2.0 * 16 * 8 * 4 * 4 * (iters / 8) * double(grid.x) * (threads / 32);
      printf("DMMA m16n8k4 threads=%d: %.1f TFLOPS\n", threads, fl / ms / 1e9);
      cudaEventRecord(a);
      dmma_m8n8k4_kernel<<<grid, threads>>>(out, iters / 8);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      fl = 2.0 * 8 * 8 * 4 * 4 * (iters / 8) * double(grid.x) * (threads / 32);
      printf("DMMA m8n8k4 threads=%d: %.1f TFLOPS\n", threads, fl / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
