// Per-step latency of the register-resident Gauss-Jordan of the ALS pinv
// (als.cu gj_inverse_regs) and variants: reciprocal flavour, two pivots per
// barrier. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 gj_regs.cu
#include <cstdio>
#include <cmath>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int RV>
__device__ __forceinline__ double recip(double p) {
  if (RV == 0) return 1.0 / p;
  if (RV == 1) return __drcp_rn(p);
  if (RV == 2) {  // approximate reciprocal + two Newton steps
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
    double e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    e = fma(-p, r, 1.0);
    return fma(r, e, r);
  }
  return p;  // RV == 3: no reciprocal (latency floor)
}

template <int KR, int KC, int RV, bool TWO>
__global__ void gj(const double* Ain, double* Aout, int R, long long* ns) {
  extern __shared__ double rowbuf_raw[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  double (*rowbuf)[32 * KC] = reinterpret_cast<double (*)[32 * KC]>(rowbuf_raw);  // [4][32*KC]
  double v[KR][KC];
#pragma unroll
  for (int q = 0; q < KR; ++q)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int i = wid + q * nw, j = lane + 32 * m;
      v[q][m] = (i < R && j < R) ? Ain[i + j * R] : 0.0;
    }
  // rows 0 (and 1) published
  if (wid == 0)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[0][lane + 32 * m] = v[0][m];
  if (TWO && wid == 1 % nw)
#pragma unroll
    for (int q = 0; q < KR; ++q)
      if (q == 1 / nw)
#pragma unroll
        for (int m = 0; m < KC; ++m) rowbuf[1][lane + 32 * m] = v[q][m];
  __syncthreads();
  const unsigned long long t0 = gt();
  if (!TWO) {
    for (int k = 0; k < R; ++k) {
      const double* rk = rowbuf[k & 1];
      const double p = rk[k];
      double rkj[KC];
#pragma unroll
      for (int m = 0; m < KC; ++m) rkj[m] = rk[lane + 32 * m];
      const int mk = k >> 5, lk = k & 31;
      double aik[KR];
#pragma unroll
      for (int q = 0; q < KR; ++q) {
        double x = 0.0;
#pragma unroll
        for (int m = 0; m < KC; ++m)
          if (m == mk) x = v[q][m];
        aik[q] = __shfl_sync(0xffffffffu, x, lk);
      }
      const double ip = recip<RV>(p);
#pragma unroll
      for (int m = 0; m < KC; ++m) {
        const int j = lane + 32 * m;
        const double akj = rkj[m] * ip;
#pragma unroll
        for (int q = 0; q < KR; ++q) {
          const int i = wid + q * nw;
          if (j != k)
            v[q][m] = (i != k) ? v[q][m] - aik[q] * akj : akj;
          else
            v[q][m] = (i != k) ? -aik[q] * ip : ip;
        }
      }
      const int k1 = k + 1;
      if (k1 < R && wid == k1 % nw) {
#pragma unroll
        for (int q = 0; q < KR; ++q)
          if (q == k1 / nw)
#pragma unroll
            for (int m = 0; m < KC; ++m) rowbuf[k1 & 1][lane + 32 * m] = v[q][m];
      }
      __syncthreads();
    }
  } else {
    // two pivots per barrier: rows k and k+1 (as of step k-1) are published;
    // every thread applies step k, then step k+1 with row k+1 updated locally
    // by the same expressions its owner would use
    for (int k = 0; k < R; k += 2) {
      const double* rk = rowbuf[(k >> 1) & 1 ? 2 : 0];
      const double* rk1 = rowbuf[(k >> 1) & 1 ? 3 : 1];
      const double p = rk[k];
      const double ip = recip<RV>(p);
      double rkj[KC], r1j[KC];
#pragma unroll
      for (int m = 0; m < KC; ++m) {
        rkj[m] = rk[lane + 32 * m];
        r1j[m] = rk1[lane + 32 * m];
      }
      const bool has2 = k + 1 < R;
      // row k+1 after step k (i = k+1 != k)
      const double a1k = rk1[k];
      double r1n[KC];
#pragma unroll
      for (int m = 0; m < KC; ++m) {
        const int j = lane + 32 * m;
        r1n[m] = (j != k) ? r1j[m] - a1k * (rkj[m] * ip) : -a1k * ip;
      }
      const int k1 = k + 1;
      double x1 = 0.0;
#pragma unroll
      for (int m = 0; m < KC; ++m)
        if (m == (k1 >> 5)) x1 = r1n[m];
      x1 = __shfl_sync(0xffffffffu, x1, k1 & 31);
      const double p1 = has2 ? x1 : 1.0;
      const double ip1 = recip<RV>(p1);
      const int mk = k >> 5, lk = k & 31;
      double aik[KR];
#pragma unroll
      for (int q = 0; q < KR; ++q) {
        double x = 0.0;
#pragma unroll
        for (int m = 0; m < KC; ++m)
          if (m == mk) x = v[q][m];
        aik[q] = __shfl_sync(0xffffffffu, x, lk);
      }
#pragma unroll
      for (int m = 0; m < KC; ++m) {
        const int j = lane + 32 * m;
        const double akj = rkj[m] * ip;
#pragma unroll
        for (int q = 0; q < KR; ++q) {
          const int i = wid + q * nw;
          if (j != k)
            v[q][m] = (i != k) ? v[q][m] - aik[q] * akj : akj;
          else
            v[q][m] = (i != k) ? -aik[q] * ip : ip;
        }
      }
      if (has2) {
        const int mk1 = k1 >> 5, lk1 = k1 & 31;
#pragma unroll
        for (int q = 0; q < KR; ++q) {
          double x = 0.0;
#pragma unroll
          for (int m = 0; m < KC; ++m)
            if (m == mk1) x = v[q][m];
          aik[q] = __shfl_sync(0xffffffffu, x, lk1);
        }
#pragma unroll
        for (int m = 0; m < KC; ++m) {
          const int j = lane + 32 * m;
          const double akj = r1n[m] * ip1;
#pragma unroll
          for (int q = 0; q < KR; ++q) {
            const int i = wid + q * nw;
            if (j != k1)
              v[q][m] = (i != k1) ? v[q][m] - aik[q] * akj : akj;
            else
              v[q][m] = (i != k1) ? -aik[q] * ip1 : ip1;
          }
        }
      }
      // publish rows k+2, k+3 (as of step k+1)
      const int nb = ((k >> 1) + 1) & 1 ? 2 : 0;
#pragma unroll
      for (int d = 2; d < 4; ++d) {
        const int kk = k + d;
        if (kk < R && wid == kk % nw)
#pragma unroll
          for (int q = 0; q < KR; ++q)
            if (q == kk / nw)
#pragma unroll
              for (int m = 0; m < KC; ++m) rowbuf[nb + d - 2][lane + 32 * m] = v[q][m];
      }
      __syncthreads();
    }
  }
  const unsigned long long t1 = gt();
#pragma unroll
  for (int q = 0; q < KR; ++q)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int i = wid + q * nw, j = lane + 32 * m;
      if (i < R && j < R) Aout[i + j * R] = v[q][m];
    }
  if (tid == 0) ns[0] = (long long)(t1 - t0);
}


// the static-slot version now in als.cu (copied)
template <int KR, int KC>
__device__ void gj_inverse_regs(double* A, int R, int* ok, double* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  double (*rowbuf)[32 * KC] = reinterpret_cast<double (*)[32 * KC]>(scratch);
  double v[KR][KC];
#pragma unroll
  for (int q = 0; q < KR; ++q)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int i = wid + q * nw, j = lane + 32 * m;
      v[q][m] = (i < R && j < R) ? A[i + j * R] : 0.0;
    }
  if (wid == 0)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[0][lane + 32 * m] = v[0][m];
  __syncthreads();
  int bad = 0;
  // pivot k = q * nw + w: the slot q of the pivot row (and of the next one,
  // q or q + 1) is a compile-time index, so v stays in registers (a runtime
  // slot index made the compiler keep v on the stack: ~1.2 us per step)
#pragma unroll
  for (int q0 = 0; q0 < KR; ++q0) {
    for (int w = 0; w < nw; ++w) {
      const int k = q0 * nw + w;
      if (k >= R) break;
      const double* rk = rowbuf[k & 1];
      const double p = rk[k];
      double rkj[KC];
#pragma unroll
      for (int m = 0; m < KC; ++m) rkj[m] = rk[lane + 32 * m];
      const int mk = k >> 5, lk = k & 31;
      double aik[KR];
#pragma unroll
      for (int q = 0; q < KR; ++q) {
        double x = v[q][0];
#pragma unroll
        for (int m = 1; m < KC; ++m) x = (m == mk) ? v[q][m] : x;
        aik[q] = __shfl_sync(0xffffffffu, x, lk);
      }
      bad |= !(p > 0.0);
      const double ip = 1.0 / p;
      // the general update on every entry (one FMA: v - aik akj), then the
      // column-k entries (-aik / p, lane lk) and row k (akj, its pivot 1 / p)
      // overwritten: the values of the branchy per-entry form, a quarter of
      // the instructions
      double akj[KC];
#pragma unroll
      for (int m = 0; m < KC; ++m) akj[m] = rkj[m] * ip;
#pragma unroll
      for (int m = 0; m < KC; ++m)
#pragma unroll
        for (int q = 0; q < KR; ++q) v[q][m] = fma(-aik[q], akj[m], v[q][m]);
      if (lane == lk)
#pragma unroll
        for (int m = 0; m < KC; ++m)
          if (m == mk)
#pragma unroll
            for (int q = 0; q < KR; ++q) v[q][m] = -aik[q] * ip;
      if (wid == w)
#pragma unroll
        for (int m = 0; m < KC; ++m) v[q0][m] = (lane + 32 * m == k) ? ip : akj[m];
      // publish row k + 1: warp w + 1, slot q0 -- or warp 0, slot q0 + 1
      if (k + 1 < R) {
        double* dst = rowbuf[(k + 1) & 1];
        if (w + 1 < nw) {
          if (wid == w + 1)
#pragma unroll
            for (int m = 0; m < KC; ++m) dst[lane + 32 * m] = v[q0][m];
        } else if (q0 + 1 < KR) {
          if (wid == 0)
#pragma unroll
            for (int m = 0; m < KC; ++m) dst[lane + 32 * m] = v[q0 + 1 < KR ? q0 + 1 : q0][m];
        }
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int q = 0; q < KR; ++q)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int i = wid + q * nw, j = lane + 32 * m;
      if (i < R && j < R) A[i + j * R] = v[q][m];
    }
  if (tid == 0 && bad) *ok = 0;
  __syncthreads();
}

template <int KR, int KC>
__global__ void gj_new(const double* Ain, double* Aout, int R, long long* ns) {
  extern __shared__ double sc[];
  __shared__ int ok;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Aout[e] = Ain[e];
  __syncthreads();
  const unsigned long long t0 = gt();
  gj_inverse_regs<KR, KC>(Aout, R, &ok, sc);
  const unsigned long long t1 = gt();
  if (threadIdx.x == 0) ns[0] = (long long)(t1 - t0);
}

// two pivots per barrier with compile-time slots (nw even): pivots k = q0 nw + w
// and k + 1 (warp w + 1, same slot); rows k + 2, k + 3 published for the next pair
template <int KR, int KC>
__device__ void gj2_inverse_regs(double* A, int R, int* ok, double* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  double (*rowbuf)[32 * KC] = reinterpret_cast<double (*)[32 * KC]>(scratch);  // [4]
  double v[KR][KC];
#pragma unroll
  for (int q = 0; q < KR; ++q)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int i = wid + q * nw, j = lane + 32 * m;
      v[q][m] = (i < R && j < R) ? A[i + j * R] : 0.0;
    }
  if (wid == 0)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[0][lane + 32 * m] = v[0][m];
  if (wid == 1)
#pragma unroll
    for (int m = 0; m < KC; ++m) rowbuf[1][lane + 32 * m] = v[0][m];
  __syncthreads();
  int bad = 0, pb = 0;
#pragma unroll
  for (int q0 = 0; q0 < KR; ++q0) {
    for (int w = 0; w < nw; w += 2) {
      const int k = q0 * nw + w;
      if (k >= R) break;
      const bool has2 = k + 1 < R;
      const double* rk = rowbuf[pb];
      const double* rk1 = rowbuf[pb + 1];
      const double p = rk[k];
      const double ip = 1.0 / p;
      double akj[KC], r1[KC];
#pragma unroll
      for (int m = 0; m < KC; ++m) {
        akj[m] = rk[lane + 32 * m] * ip;
        r1[m] = rk1[lane + 32 * m];
      }
      // row k + 1 after step k (i = k + 1 != k)
      const double a1k = rk1[k];
#pragma unroll
      for (int m = 0; m < KC; ++m) r1[m] = (lane + 32 * m == k) ? -a1k * ip : fma(-a1k, akj[m], r1[m]);
      const int k1 = k + 1, mk = k >> 5, lk = k & 31, mk1 = k1 >> 5, lk1 = k1 & 31;
      double x1 = r1[0];
#pragma unroll
      for (int m = 1; m < KC; ++m) x1 = (m == mk1) ? r1[m] : x1;
      const double p1 = has2 ? __shfl_sync(0xffffffffu, x1, lk1) : 1.0;
      const double ip1 = 1.0 / p1;
      bad |= !(p > 0.0) || !(p1 > 0.0);
      // step k
      double aik[KR];
#pragma unroll
      for (int q = 0; q < KR; ++q) {
        double x = v[q][0];
#pragma unroll
        for (int m = 1; m < KC; ++m) x = (m == mk) ? v[q][m] : x;
        aik[q] = __shfl_sync(0xffffffffu, x, lk);
      }
#pragma unroll
      for (int m = 0; m < KC; ++m)
#pragma unroll
        for (int q = 0; q < KR; ++q) v[q][m] = fma(-aik[q], akj[m], v[q][m]);
      if (lane == lk)
#pragma unroll
        for (int m = 0; m < KC; ++m)
          if (m == mk)
#pragma unroll
            for (int q = 0; q < KR; ++q) v[q][m] = -aik[q] * ip;
      if (wid == w)
#pragma unroll
        for (int m = 0; m < KC; ++m) v[q0][m] = (lane + 32 * m == k) ? ip : akj[m];
      if (has2) {
        double ak1j[KC];
#pragma unroll
        for (int m = 0; m < KC; ++m) ak1j[m] = r1[m] * ip1;
#pragma unroll
        for (int q = 0; q < KR; ++q) {
          double x = v[q][0];
#pragma unroll
          for (int m = 1; m < KC; ++m) x = (m == mk1) ? v[q][m] : x;
          aik[q] = __shfl_sync(0xffffffffu, x, lk1);
        }
#pragma unroll
        for (int m = 0; m < KC; ++m)
#pragma unroll
          for (int q = 0; q < KR; ++q) v[q][m] = fma(-aik[q], ak1j[m], v[q][m]);
        if (lane == lk1)
#pragma unroll
          for (int m = 0; m < KC; ++m)
            if (m == mk1)
#pragma unroll
              for (int q = 0; q < KR; ++q) v[q][m] = -aik[q] * ip1;
        if (wid == w + 1)
#pragma unroll
          for (int m = 0; m < KC; ++m) v[q0][m] = (lane + 32 * m == k1) ? ip1 : ak1j[m];
      }
      // publish rows k + 2, k + 3 (warps w + 2, w + 3 of slot q0, or 0, 1 of q0 + 1)
      const int nb = pb ^ 2;
      if (w + 2 < nw) {
        if (wid == w + 2 || wid == w + 3)
#pragma unroll
          for (int m = 0; m < KC; ++m) rowbuf[nb + (wid - w - 2)][lane + 32 * m] = v[q0][m];
      } else if (q0 + 1 < KR) {
        if (wid < 2)
#pragma unroll
          for (int m = 0; m < KC; ++m) rowbuf[nb + wid][lane + 32 * m] = v[q0 + 1 < KR ? q0 + 1 : q0][m];
      }
      pb = nb;
      __syncthreads();
    }
  }
#pragma unroll
  for (int q = 0; q < KR; ++q)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int i = wid + q * nw, j = lane + 32 * m;
      if (i < R && j < R) A[i + j * R] = v[q][m];
    }
  if (tid == 0 && bad) *ok = 0;
  __syncthreads();
}

template <int KR, int KC>
__global__ void gj2_new(const double* Ain, double* Aout, int R, long long* ns) {
  extern __shared__ double sc[];
  __shared__ int ok;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Aout[e] = Ain[e];
  __syncthreads();
  const unsigned long long t0 = gt();
  gj2_inverse_regs<KR, KC>(Aout, R, &ok, sc);
  const unsigned long long t1 = gt();
  if (threadIdx.x == 0) ns[0] = (long long)(t1 - t0);
}

template <int KR, int KC, int RV, bool TWO>
double run(int R, int nt, const double* dA, double* dO, long long* dns, const double* hA, double* hO) {
  if (RV == 8)
    gj2_new<KR, KC><<<1, nt, 4 * 32 * KC * 8>>>(dA, dO, R, dns);
  else if (RV == 9)
    gj_new<KR, KC><<<1, nt, 4 * 32 * KC * 8>>>(dA, dO, R, dns);
  else
    gj<KR, KC, RV, TWO><<<1, nt, 4 * 32 * KC * 8>>>(dA, dO, R, dns);
  long long ns;
  cudaMemcpy(&ns, dns, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hO, dO, R * R * 8, cudaMemcpyDeviceToHost);
  // residual |A X - I|
  double err = 0;
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      double s = 0;
      for (int k = 0; k < R; ++k) s += hA[i + k * R] * hO[k + j * R];
      err = fmax(err, fabs(s - (i == j)));
    }
  printf("  RV=%d two=%d: %.0f ns/step  |AX-I| %.1e\n", RV, int(TWO), double(ns) / R, err);
  return err;
}

int main() {
  for (int R : {32, 50, 64}) {
    const int nt = 256;
    double hA[64 * 64], hO[64 * 64];
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j) hA[i + j * R] = (i == j ? R : 0.0) + 1.0 / (1 + ((i + j) % 7));
    double *dA, *dO;
    long long* dns;
    cudaMalloc(&dA, R * R * 8);
    cudaMalloc(&dO, R * R * 8);
    cudaMalloc(&dns, 8);
    cudaMemcpy(dA, hA, R * R * 8, cudaMemcpyHostToDevice);
    printf("R=%d threads=%d\n", R, nt);
    for (int rep = 0; rep < 2; ++rep) {
      run<8, 2, 9, false>(R, nt, dA, dO, dns, hA, hO);
      run<8, 2, 8, false>(R, nt, dA, dO, dns, hA, hO);
      run<8, 2, 0, false>(R, nt, dA, dO, dns, hA, hO);
      run<8, 2, 1, false>(R, nt, dA, dO, dns, hA, hO);
      run<8, 2, 2, false>(R, nt, dA, dO, dns, hA, hO);
      run<8, 2, 3, false>(R, nt, dA, dO, dns, hA, hO);
      run<8, 2, 0, true>(R, nt, dA, dO, dns, hA, hO);
      run<8, 2, 2, true>(R, nt, dA, dO, dns, hA, hO);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
