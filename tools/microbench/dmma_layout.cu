// Checks the m16n8k4 f64 mma.sync fragment layout used by passes_dmma.cu.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = A[g * 4 + t], a1 = A[(g + 8) * 4 + t];  // A row-major 16x4
  double b0 = B[t * 8 + g];                          // B 4x8 (k, n)
  double c[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b0));
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}
int main() {
  double hA[64], hB[32], hC[128], ref[128];
  for (int i = 0; i < 64; ++i) hA[i] = (i * 7 % 13) - 6;
  for (int i = 0; i < 32; ++i) hB[i] = (i * 5 % 11) - 5;
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int kk = 0; kk < 4; ++kk) s += hA[m * 4 + kk] * hB[kk * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *A, *B, *C;
  cudaMalloc(&A, 512); cudaMalloc(&B, 256); cudaMalloc(&C, 1024);
  cudaMemcpy(A, hA, 512, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, 1024, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128; ++i) bad += hC[i] != ref[i];
  printf("m16n8k4 f64 layout mismatches: %d (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
  return bad;
}
