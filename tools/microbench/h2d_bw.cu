// Pinned host -> device bandwidth of a 512 MB tensor: one copy, or split over 2 / 4 streams
// (can concurrent copy engines beat a single cudaMemcpyAsync on this link?).
// nvcc -O3 -o h2d_bw h2d_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 512000000;
  char *h, *d;
  cudaMallocHost(&h, n);
  cudaMalloc(&d, n);
  for (size_t i = 0; i < n; i += 4096) h[i] = char(i);
  cudaStream_t st[8];
  for (auto& s : st) cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int parts : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, st[0]);
      for (int p = 1; p < parts; ++p) cudaStreamWaitEvent(st[p], a, 0);
      const size_t chunk = (n / parts + 255) & ~size_t(255);
      cudaEvent_t done[8];
      for (int p = 0; p < parts; ++p) {
        const size_t off = p * chunk, len = off + chunk <= n ? chunk : n - off;
        cudaMemcpyAsync(d + off, h + off, len, cudaMemcpyHostToDevice, st[p]);
        if (p) {
          cudaEventCreate(&done[p]);
          cudaEventRecord(done[p], st[p]);
          cudaStreamWaitEvent(st[0], done[p], 0);
        }
      }
      cudaEventRecord(b, st[0]);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("streams %d: %.3f ms  %.1f GB/s\n", parts, ms, n / ms / 1e6);
    }
  }
  return 0;
}
