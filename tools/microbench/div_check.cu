// Exhaustive-random check of the LU's reciprocal-based division (factor.cu
// lu_div) against IEEE x / piv, fp64 and fp32, |x| <= |piv| and beyond.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o div_check div_check.cu
#include <cstdio>
#include <cstdint>
template <typename T>
__device__ __forceinline__ T lu_div(T x, T piv, T rp) {
  T q = x * rp;
  q = fma(fma(-q, piv, x), rp, q);
  q = fma(fma(-q, piv, x), rp, q);
  const T ax = fabs(x);
  constexpr T lo = sizeof(T) == 8 ? T(0x1p-900) : T(0x1p-90);
  constexpr T hi = sizeof(T) == 8 ? T(0x1p+900) : T(0x1p+90);
  return (ax >= lo && ax <= hi) ? q : x / piv;
}
__device__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull; z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
template <typename T>
__global__ void check(unsigned long long* bad, uint64_t seed, int wide) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  for (int it = 0; it < 64; ++it) {
    const uint64_t a = mix(seed ^ (i * 64 + it)), b = mix(a);
    T x, p;
    if constexpr (sizeof(T) == 8) {
      // random mantissas, exponents within +-60 (wide: +-600)
      const int ex = int(a % (wide ? 1200 : 120)) - (wide ? 600 : 60), ep = int(b % (wide ? 1200 : 120)) - (wide ? 600 : 60);
      x = ldexp(1.0 + double(a >> 12) * 0x1p-52, ex) * ((a & 1) ? -1 : 1);
      p = ldexp(1.0 + double(b >> 12) * 0x1p-52, ep) * ((b & 2) ? -1 : 1);
    } else {
      const int ex = int(a % (wide ? 160 : 40)) - (wide ? 80 : 20), ep = int(b % (wide ? 160 : 40)) - (wide ? 80 : 20);
      x = ldexpf(1.0f + float(a >> 41) * 0x1p-23f, ex) * ((a & 1) ? -1 : 1);
      p = ldexpf(1.0f + float(b >> 41) * 0x1p-23f, ep) * ((b & 2) ? -1 : 1);
    }
    const T rp = T(1) / p;
    const T q = lu_div(x, p, rp), w = x / p;
    if (!(q == w)) atomicAdd(bad, 1ull);
  }
}
int main() {
  unsigned long long* bad;
  cudaMallocManaged(&bad, 8);
  for (int wide = 0; wide < 2; ++wide) {
    *bad = 0;
    for (int s = 0; s < 8; ++s) check<double><<<4096, 256>>>(bad, 1234 + s, wide);
    cudaDeviceSynchronize();
    printf("f64 wide=%d: %llu mismatches of %llu\n", wide, *bad, 8ull * 4096 * 256 * 64);
    *bad = 0;
    for (int s = 0; s < 8; ++s) check<float><<<4096, 256>>>(bad, 99 + s, wide);
    cudaDeviceSynchronize();
    printf("f32 wide=%d: %llu mismatches of %llu\n", wide, *bad, 8ull * 4096 * 256 * 64);
  }
  return 0;
}
