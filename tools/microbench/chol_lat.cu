// Standalone timing of chol_inv_regs (copied from factor.cu by tools/microbench/gen_chol_lat.py)
#include <cstdio>
template <int KR, int KC>
__device__ void chol_inv_regs(double* A, double* X, int n, int ld, double* dg, int* fail) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  __shared__ double rowbuf[2][32 * KC];
  __shared__ double s_d[32 * KC];
  double v[KR][KC];
#pragma unroll
  for (int k = 0; k < KR; ++k)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int r = wid + k * nw, c = lane + 32 * m;
      v[k][m] = (r < n && c < n && c >= r) ? A[r + c * ld] : 0.0;  // I part: identity minus its diagonal
    }
  if (wid == 0)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[0][lane + 32 * m] = v[0][m];
  __syncthreads();
  int bad = 0;
  int nxw = 1 % nw, nxk = 1 / nw;  // owner (warp, slot) of row j + 1, advanced per step (no integer division)
  for (int j = 0; j < n; ++j) {
    const double* rj = rowbuf[j & 1];
    // every shared read of the step is issued before the reciprocal
    const double d = rj[j];
    double tk[KR], aj[KC];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = wid + k * nw;
      tk[k] = (r > j && r < n) ? rj[r] : 0.0;
    }
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int c = lane + 32 * m;
      aj[m] = c == j ? 1.0 : (c < n ? rj[c] : 0.0);
    }
    bad |= !(d > 0.0);
    const double rd = d > 0.0 ? 1.0 / d : 1.0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = wid + k * nw;
      if (r > j && r < n) {
        const double t = tk[k] * rd;  // U(j, r)
#pragma unroll
        for (int m = 0; m < KC; ++m) {
          const int c = lane + 32 * m;
          if (c < n && (c >= r || c <= j)) v[k][m] -= t * aj[m];
        }
      }
    }
    if (j + 1 < n && wid == nxw) {
#pragma unroll
      for (int k = 0; k < KR; ++k)
        if (k == nxk)
#pragma unroll
          for (int m = 0; m < KC; ++m) rowbuf[(j + 1) & 1][lane + 32 * m] = v[k][m];
    }
    if (++nxw == nw) {
      nxw = 0;
      ++nxk;
    }
    if (tid == 0) s_d[j] = d;
    __syncthreads();
  }
  if (tid == 0 && bad) *fail = 1;
  for (int j = tid; j < n; j += blockDim.x) dg[j] = s_d[j] > 0.0 ? sqrt(s_d[j]) : 1.0;
  // R(r, c) = sqrt(d_r) U(r, c) (upper), X = R^{-1}: X(c, r) = (U^{-T})(r, c) / sqrt(d_r)
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int r = wid + k * nw;
    if (r < n) {
      const double dr = s_d[r];
      const double sq = dr > 0.0 ? sqrt(dr) : 1.0, rs = 1.0 / sq, rd = dr > 0.0 ? 1.0 / dr : 1.0;
#pragma unroll
      for (int m = 0; m < KC; ++m) {
        const int c = lane + 32 * m;
        if (c >= n) continue;
        if (c < r) {
          X[c + r * ld] = v[k][m] * rs;
        } else if (c == r) {
          X[r + r * ld] = rs;
          A[r + r * ld] = sq;
        } else {
          X[c + r * ld] = 0.0;
          A[r + c * ld] = (v[k][m] * rd) * sq;
        }
      }
    }
  }
  __syncthreads();
}

template <int KR, int KC>
__device__ void sign_reconstruct_regs(double* G, int n, int ld, int rows, double* sgn) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  __shared__ double rowbuf[2][32 * KC];
  double v[KR][KC];
#pragma unroll
  for (int k = 0; k < KR; ++k)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int r = wid + k * nw, c = lane + 32 * m;
      v[k][m] = (r < n && c < n) ? G[r + c * ld] : 0.0;
    }
  if (wid == 0)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[0][lane + 32 * m] = v[0][m];
  __syncthreads();
  int nxw = 1 % nw, nxk = 1 / nw;  // owner of row k0 + 1
  for (int k0 = 0; k0 < n; ++k0) {
    const double* rk = rowbuf[k0 & 1];
    const double gkk = rk[k0];
    double ak[KC];
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int c = lane + 32 * m;
      ak[m] = c < n ? rk[c] : 0.0;
    }
    const int mk = k0 >> 5, lk = k0 & 31;
    double gik[KR];  // G(r, k0): lane lk of this warp holds it
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      double x = 0.0;
#pragma unroll
      for (int m = 0; m < KC; ++m)
        if (m == mk) x = v[k][m];
      gik[k] = __shfl_sync(0xffffffffu, x, lk);
    }
    const double sk = (gkk > 0.0) != (k0 == rows - 1) ? -1.0 : 1.0;
    const double rd = 1.0 / (sk * gkk - 1.0);
    if (tid == 0) sgn[k0] = sk;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = wid + k * nw;
      if (r > k0 && r < n) {
        const double l = (sk * gik[k]) * rd;
#pragma unroll
        for (int m = 0; m < KC; ++m) {
          const int c = lane + 32 * m;
          if (c > k0 && c < n) v[k][m] -= l * ak[m];
        }
      }
    }
    if (k0 + 1 < n && wid == nxw) {
#pragma unroll
      for (int k = 0; k < KR; ++k)
        if (k == nxk)
#pragma unroll
          for (int m = 0; m < KC; ++m) rowbuf[(k0 + 1) & 1][lane + 32 * m] = v[k][m];
    }
    if (++nxw == nw) {
      nxw = 0;
      ++nxk;
    }
    __syncthreads();
  }
}

template <int KR, int KC>
__global__ void run(const double* G0, double* out, long long* cyc, int n, int ld) {
  extern __shared__ double sm[];
  double *A = sm, *X = sm + 96 * 97;
  __shared__ double dg[96];
  __shared__ int fail;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) A[(e % n) + (e / n) * ld] = G0[e];
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  long long t0 = clock64();
  chol_inv_regs<KR, KC>(A, X, n, ld, dg, &fail);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) out[e] = X[(e % n) + (e / n) * ld];
}

int main() {
  for (int n : {30, 70}) {
    double* h = new double[n * n];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) h[i + j * n] = (i == j ? n : 0.0) + 1.0 / (1 + i + j);
    double *G, *o;
    long long* c;
    cudaMalloc(&G, n * n * 8);
    cudaMalloc(&o, n * n * 8);
    cudaMallocManaged(&c, 64);
    cudaMemcpy(G, h, n * n * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(run<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 96 * 97 * 8);
    cudaFuncSetAttribute(run<12, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 96 * 97 * 8);
    for (int rep = 0; rep < 3; ++rep) {
      if (n <= 32) run<4, 1><<<1, 256, 2 * 96 * 97 * 8>>>(G, o, c, n, n + 1);
      else run<12, 3><<<1, 256, 2 * 96 * 97 * 8>>>(G, o, c, n, n + 1);
      cudaDeviceSynchronize();
    }
    printf("n=%d chol_inv_regs: %lld cycles (%.1f per step) err=%s\n", n, c[0], double(c[0]) / n,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
