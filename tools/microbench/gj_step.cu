// Why does a Gauss-Jordan elimination step on a small smem matrix (R = 50)
// cost ~1.6 us in the ALS / QR kernels? Variants of the same step loop.
#include <cstdio>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int VAR>
__global__ void gj(int R, double* out, long long* ns) {
  extern __shared__ double sm[];
  double* A = sm; double* X = sm + R * R;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < R * R; e += nt) A[e] = (e % R == e / R) ? R + 1.0 : 1.0 / (1 + (e % 7));
  __syncthreads();
  unsigned long long t0 = gt();
  double* src = A; double* dst = X;
  for (int rep = 0; rep < 10; ++rep)
  for (int k = 0; k < R; ++k) {
    const double p = src[k + k * R];
    double ip;
    if (VAR == 1) ip = __drcp_rn(p); else ip = 1.0 / p;
    if (VAR == 3) {  // restrict-qualified, loads hoisted ahead of stores
      const double* __restrict__ sp = src;
      double* __restrict__ dp = dst;
      const double aik0 = lane < R ? sp[lane + k * R] : 0.0;
      const double aik1 = lane + 32 < R ? sp[lane + 32 + k * R] : 0.0;
      for (int j = wid; j < R; j += nw) {
        const double akj = sp[k + j * R] * ip;
        const double s0 = lane < R ? sp[lane + j * R] : 0.0;
        const double s1 = lane + 32 < R ? sp[lane + 32 + j * R] : 0.0;
        double v0, v1;
        if (j != k) {
          v0 = (lane != k) ? s0 - aik0 * akj : akj;
          v1 = (lane + 32 != k) ? s1 - aik1 * akj : akj;
        } else {
          v0 = (lane != k) ? -aik0 * ip : ip;
          v1 = (lane + 32 != k) ? -aik1 * ip : ip;
        }
        if (lane < R) dp[lane + j * R] = v0;
        if (lane + 32 < R) dp[lane + 32 + j * R] = v1;
      }
    } else if (VAR == 2) {  // branch-free full update, precomputed column k
      for (int j = wid; j < R; j += nw) {
        const double akj = src[k + j * R] * ip;
        for (int i = lane; i < R; i += 32) dst[i + j * R] = src[i + j * R] - src[i + k * R] * akj;
      }
    } else {
      for (int j = wid; j < R; j += nw) {
        const double akj = src[k + j * R] * ip;
        for (int i = lane; i < R; i += 32) {
          const double aik = src[i + k * R];
          double v;
          if (j != k) v = (i != k) ? src[i + j * R] - aik * akj : akj;
          else v = (i != k) ? -aik * ip : ip;
          dst[i + j * R] = v;
        }
      }
    }
    __syncthreads();
    double* t = src; src = dst; dst = t;
  }
  unsigned long long t1 = gt();
  if (tid == 0) { ns[0] = (long long)(t1 - t0); out[0] = src[0]; }
}

int main() {
  double* o; long long* ns; cudaMalloc(&o, 8); cudaMalloc(&ns, 8);
  for (int R : {32, 50, 64})
    for (int nt : {128, 256, 512}) {
      long long h[3];
      gj<0><<<1, nt, 2 * R * R * 8>>>(R, o, ns); cudaMemcpy(&h[0], ns, 8, cudaMemcpyDeviceToHost);
      gj<1><<<1, nt, 2 * R * R * 8>>>(R, o, ns); cudaMemcpy(&h[1], ns, 8, cudaMemcpyDeviceToHost);
      gj<2><<<1, nt, 2 * R * R * 8>>>(R, o, ns); cudaMemcpy(&h[2], ns, 8, cudaMemcpyDeviceToHost);
      long long h3; gj<3><<<1, nt, 2 * R * R * 8>>>(R, o, ns); cudaMemcpy(&h3, ns, 8, cudaMemcpyDeviceToHost);
      printf("R=%d threads=%d: per step ns: baseline %.0f  drcp %.0f  branchfree %.0f  restrict+hoist %.0f\n", R, nt, h[0] / (10.0 * R),
             h[1] / (10.0 * R), h[2] / (10.0 * R), h3 / (10.0 * R));
    }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
