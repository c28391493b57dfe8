// Per-step latency of a one-CTA elimination chain (the CholeskyQR2 /
// sign-reconstruction / small-LU pattern): each step reads a published
// shared value, forms a reciprocal, updates register-resident entries and
// publishes the next row behind one __syncthreads. clock64 per variant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_lat step_lat.cu
#include <cstdio>

template <int V>
__global__ void chain(double* out, long long* cyc, int n) {
  __shared__ double row[2][64];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  double v[4];
  for (int k = 0; k < 4; ++k) v[k] = 1.0 + 1e-3 * (tid + k);
  if (tid < 64) row[0][tid] = 2.0 + tid;
  __syncthreads();
  long long t0 = clock64();
  for (int j = 0; j < n; ++j) {
    const double* rj = row[j & 1];
    const double d = rj[j & 31];
    double rd;
    if (V == 0) rd = 1.0 / d;           // IEEE division
    else if (V == 1) rd = __drcp_rn(d); // IEEE reciprocal
    else if (V == 2) rd = d;            // no reciprocal (floor)
    else {                               // MUFU seed + 2 Newton steps (not IEEE)
      float f = __frcp_rn(float(d));
      rd = double(f);
      rd = rd * (2.0 - d * rd);
      rd = rd * (2.0 - d * rd);
    }
    const double aj = rj[lane];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = wid + k * nw;
      if (r > j) v[k] -= (rj[r & 63] * rd) * aj;
    }
    if (wid == (j + 1) % nw) row[(j + 1) & 1][lane] = v[0];
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[V] = (t1 - t0) / n;
  out[tid] = v[0] + v[1] + v[2] + v[3];
}

__global__ void bar_only(long long* cyc, int n) {
  long long t0 = clock64();
  for (int j = 0; j < n; ++j) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1024 * sizeof(double));
  cudaMallocManaged(&c, 16 * sizeof(long long));
  for (int threads : {128, 256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      chain<0><<<1, threads>>>(d, c, 30);
      chain<1><<<1, threads>>>(d, c, 30);
      chain<2><<<1, threads>>>(d, c, 30);
      chain<3><<<1, threads>>>(d, c, 30);
      bar_only<<<1, threads>>>(c, 30);
      cudaDeviceSynchronize();
    }
    printf("threads %4d: div %lld  drcp %lld  none %lld  newton %lld  bar-only %lld cycles/step\n", threads, c[0], c[1],
           c[2], c[3], c[4]);
  }
  return 0;
}
