// SPDX-License-Identifier: MIT
// Host launchers for the streamed tensor passes (see passes.cuh) and the
// Omega generator (compress.hpp:118-124, random.hpp:75-94).
#include <type_traits>

#include "passes.cuh"
#include "rng.cuh"
#include "runtime.cuh"

namespace rcpg {

namespace {

template <typename T>
struct TileCfg;
template <>
struct TileCfg<float> {
  static constexpr int BM = 128, BK = 32;
};
template <>
struct TileCfg<double> {
  static constexpr int BM = 64, BK = 32;
};

template <typename T, int BM, int BN, int BK, bool TXM, class LD, class EP>
void launch_tile_gemm(dim3 grid, const LD& ld, const EP& ep, cudaStream_t st) {
  auto kern = tile_gemm_kernel<T, BM, BN, BK, TXM, LD, EP>;
  const size_t smem = sizeof(TileSmem<T, BM, BN, BK>);
  static const size_t lim = enable_max_dyn_smem(kern);  // per instantiation
  if (smem > lim) throw std::runtime_error("tile_gemm: shared memory tile too large");
  kern<<<grid, kThreads, smem, st>>>(ld, ep);
  count_launch();
  RCPG_LAUNCHED();
}

int pick_bn(i64 cols) {
  if (cols <= 16) return 16;
  if (cols <= 32) return 32;
  if (cols <= 48) return 48;
  if (cols <= 64) return 64;
  return 80;
}

constexpr int kRedChunks = 8;

template <typename T, typename TO = T>
__global__ void __launch_bounds__(32 * kRedChunks) reduce_partials_kernel(const T* __restrict__ part, i64 splits, i64 n, TO* __restrict__ out,
                                       const int* skip) {
  // block = 32 consecutive outputs (lanes, coalesced) x kRedChunks warps; warp w
  // sums its contiguous chunk of splits in order, warp 0 adds the chunk sums in
  // chunk order: a fixed summation order, independent of the launch geometry
  if (skip != nullptr && *skip) return;
  __shared__ double chunk_sum[kRedChunks][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const i64 e = blockIdx.x * i64(32) + lane;
  const i64 per = (splits + kRedChunks - 1) / kRedChunks;
  const i64 q0 = w * per, q1 = q0 + per < splits ? q0 + per : splits;
  double s = 0.0;
  if (e < n) {
    const T* p = part + e;
#pragma unroll 8
    for (i64 q = q0; q < q1; ++q) s += double(__ldcs(p + q * n));
  }
  chunk_sum[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < n) {
    double t = chunk_sum[0][lane];
#pragma unroll
    for (int c = 1; c < kRedChunks; ++c) t += chunk_sum[c][lane];
    out[e] = TO(t);
  }
}

template <typename T, int BN>
void sketch_bn(const T* X, ModeView v, const T* P, i64 cols, T* part, i64 splits, i64 tiles_per_split,
               i64 total, cudaStream_t st, const int* skip) {
  constexpr int BM = TileCfg<T>::BM, BK = TileCfg<T>::BK;
  const i64 mt = ceil_div(v.I, BM), nt = ceil_div(cols, BN);
  dim3 grid{unsigned(mt), unsigned(splits), unsigned(nt)};
  SketchEpilogue<T, BM, BN> ep{part, v.I, cols};
  if (v.R > 1) {
    SketchLoader<T, BM, BN, BK> ld{X, P, v.L, v.I, v.R, cols, ceil_div(v.R, BK), tiles_per_split, total, skip};
    launch_tile_gemm<T, BM, BN, BK, false>(grid, ld, ep, st);
  } else {
    SketchLastLoader<T, BM, BN, BK> ld{X, P, v.L, v.I, cols, tiles_per_split, total, skip};
    launch_tile_gemm<T, BM, BN, BK, false>(grid, ld, ep, st);
  }
}

template <typename T>
void sketch_plan(ModeView v, i64 cols, int num_sms, i64& splits, i64& tiles_per_split, i64& total) {
  constexpr int BM = TileCfg<T>::BM, BK = TileCfg<T>::BK;
  const int BN = pick_bn(cols);
  const i64 mt = ceil_div(v.I, BM), nt = ceil_div(cols, BN);
  total = v.R > 1 ? v.L * ceil_div(v.R, BK) : ceil_div(v.L, BK);
  i64 want = ceil_div(i64(4) * num_sms, mt * nt);
  want = std::max<i64>(1, std::min<i64>(want, 65535));
  tiles_per_split = std::max<i64>(1, ceil_div(total, want));
  splits = ceil_div(total, tiles_per_split);
}

// SIMT fallbacks of the mixed (fp32 X, fp64 panel and arithmetic) passes
template <int BN>
void sketch_bn_mixed(const float* X, ModeView v, const double* P, i64 cols, double* part, i64 splits,
                     i64 tiles_per_split, i64 total, cudaStream_t st, const int* skip) {
  constexpr int BM = TileCfg<double>::BM, BK = TileCfg<double>::BK;
  const i64 mt = ceil_div(v.I, BM), nt = ceil_div(cols, BN);
  dim3 grid{unsigned(mt), unsigned(splits), unsigned(nt)};
  SketchEpilogue<double, BM, BN> ep{part, v.I, cols};
  if (v.R > 1) {
    SketchLoader<double, BM, BN, BK, float, double> ld{X,    P,          v.L,   v.I, v.R, cols, ceil_div(v.R, BK),
                                                       tiles_per_split, total, skip};
    launch_tile_gemm<double, BM, BN, BK, false>(grid, ld, ep, st);
  } else {
    SketchLastLoader<double, BM, BN, BK, float, double> ld{X, P, v.L, v.I, cols, tiles_per_split, total, skip};
    launch_tile_gemm<double, BM, BN, BK, false>(grid, ld, ep, st);
  }
}

template <int BN, typename TO>
void project_bn_mixed(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, TO* O, cudaStream_t st) {
  constexpr int BM = TileCfg<double>::BM, BK = TileCfg<double>::BK;
  const i64 nt = ceil_div(cols, BN), kt = ceil_div(v.I, BK);
  if (v.R > 1) {
    for (i64 a0 = 0; a0 < v.L; a0 += 65535) {
      const i64 na = std::min<i64>(65535, v.L - a0);
      dim3 grid{unsigned(ceil_div(v.R, BM)), unsigned(na), unsigned(nt)};
      const i64 off = a0 * v.I * v.R, ooff = a0 * cols * v.R;
      ProjectLoader<double, BM, BN, BK, float, double> ld{X + off, Q, v.I, v.R, cols, ldq, kt};
      ProjectEpilogue<double, BM, BN, TO> ep{O + ooff, v.R, cols};
      launch_tile_gemm<double, BM, BN, BK, true>(grid, ld, ep, st);
    }
  } else {
    dim3 grid{unsigned(ceil_div(v.L, BM)), 1u, unsigned(nt)};
    ProjectLastLoader<double, BM, BN, BK, float, double> ld{X, Q, v.L, v.I, cols, ldq, kt};
    ProjectLastEpilogue<double, BM, BN, TO> ep{O, v.L, cols};
    launch_tile_gemm<double, BM, BN, BK, false>(grid, ld, ep, st);
  }
}

__global__ void widen_kernel(const float* __restrict__ src, double* __restrict__ dst, i64 n) {
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
    dst[i] = double(src[i]);
}

__global__ void narrow_kernel(const double* __restrict__ src, float* __restrict__ dst, i64 n) {
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
    dst[i] = float(src[i]);
}

template <typename TO>
void sketch_mixed_impl(const float* X, ModeView v, const double* P, i64 cols, TO* Y, double* scratch,
                       i64 scratch_doubles, int num_sms, cudaStream_t st, const int* skip);
template <typename TO>
void project_mixed_impl(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, TO* O, cudaStream_t st);

}  // namespace

i64 sketch_mixed_scratch_doubles(ModeView v, i64 cols, int num_sms) {
  i64 splits = 1, tps, total;
  sketch_plan<double>(v, cols, num_sms, splits, tps, total);
  if (v.R > 1) splits = std::max(splits, sketch_dmma_f32_splits(v, cols, num_sms, tps, total));
  return ceil_div(splits * cols * v.I, 4) * 4;
}

namespace {
template <typename TO>
void sketch_mixed_impl(const float* X, ModeView v, const double* P, i64 cols, TO* Y, double* scratch,
                       i64 scratch_doubles, int num_sms, cudaStream_t st, const int* skip) {
  i64 splits = 0, tps, total;
  bool done = false;
  if (v.R > 1) {
    splits = sketch_dmma_f32_splits(v, cols, num_sms, tps, total);
    if (splits * cols * v.I > scratch_doubles) throw std::runtime_error("sketch_mixed: scratch too small");
    done = sketch_dmma_f32(X, v, P, cols, scratch, num_sms, skip, st);
  }
  if (!done) {
    sketch_plan<double>(v, cols, num_sms, splits, tps, total);
    if (splits * cols * v.I > scratch_doubles) throw std::runtime_error("sketch_mixed: scratch too small");
    switch (pick_bn(cols)) {
      case 16: sketch_bn_mixed<16>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
      case 32: sketch_bn_mixed<32>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
      case 48: sketch_bn_mixed<48>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
      case 64: sketch_bn_mixed<64>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
      default: sketch_bn_mixed<80>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
    }
  }
  // fp64 partials summed in a fixed order, then one rounding to fp32 (TO = float),
  // or kept in fp64 (TO = double: a rank's partial of a sharded sum)
  const i64 n = cols * v.I;
  reduce_partials_kernel<double, TO><<<unsigned(ceil_div(n, 32)), 32 * kRedChunks, 0, st>>>(scratch, splits, n, Y,
                                                                                             skip);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename TO>
void project_mixed_impl(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, TO* O, cudaStream_t st) {
  if (v.R > 1 && project_dmma_f32(X, v, Q, ldq, cols, O, st)) return;
  switch (pick_bn(cols)) {
    case 16: project_bn_mixed<16, TO>(X, v, Q, ldq, cols, O, st); break;
    case 32: project_bn_mixed<32, TO>(X, v, Q, ldq, cols, O, st); break;
    case 48: project_bn_mixed<48, TO>(X, v, Q, ldq, cols, O, st); break;
    case 64: project_bn_mixed<64, TO>(X, v, Q, ldq, cols, O, st); break;
    default: project_bn_mixed<80, TO>(X, v, Q, ldq, cols, O, st); break;
  }
}
}  // namespace

void sketch_mixed(const float* X, ModeView v, const double* P, i64 cols, float* Y, double* scratch,
                  i64 scratch_doubles, int num_sms, cudaStream_t st, const int* skip) {
  sketch_mixed_impl<float>(X, v, P, cols, Y, scratch, scratch_doubles, num_sms, st, skip);
}

void sketch_mixed(const float* X, ModeView v, const double* P, i64 cols, double* Y, double* scratch,
                  i64 scratch_doubles, int num_sms, cudaStream_t st, const int* skip) {
  sketch_mixed_impl<double>(X, v, P, cols, Y, scratch, scratch_doubles, num_sms, st, skip);
}

void project_mixed(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, float* O, cudaStream_t st) {
  project_mixed_impl<float>(X, v, Q, ldq, cols, O, st);
}

void project_mixed(const float* X, ModeView v, const double* Q, i64 ldq, i64 cols, double* O, cudaStream_t st) {
  project_mixed_impl<double>(X, v, Q, ldq, cols, O, st);
}

void narrow_f64(const double* src, float* dst, i64 n, cudaStream_t st) {
  if (n <= 0) return;
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(n, 256), 148 * 16)));
  narrow_kernel<<<blocks, 256, 0, st>>>(src, dst, n);
  count_launch();
  RCPG_LAUNCHED();
}

void widen_f32(const float* src, double* dst, i64 n, cudaStream_t st) {
  if (n <= 0) return;
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(n, 256), 148 * 16)));
  widen_kernel<<<blocks, 256, 0, st>>>(src, dst, n);
  count_launch();
  RCPG_LAUNCHED();
}

template <typename T>
constexpr bool use_dmma(const ModeView& v) {
  return std::is_same<T, double>::value && v.R > 1;
}

template <typename T>
i64 sketch_scratch_elems(ModeView v, i64 cols, int num_sms) {
  i64 splits, tps, total;
  if (use_dmma<T>(v))
    splits = sketch_dmma_splits(v, cols, num_sms, tps, total);
  else
    sketch_plan<T>(v, cols, num_sms, splits, tps, total);
  i64 extra = 0;
  if (std::is_same<T, float>::value && v.R > 1) {
    splits = std::max(splits, sketch_tc_splits(v, cols, num_sms, tps, total));
    extra = sketch_tc_panel_floats(v, cols);
  }
  return ceil_div(splits * cols * v.I, 4) * 4 + extra;
}

template <typename T>
void sketch(const T* X, ModeView v, const T* P, i64 cols, T* Y, T* scratch, i64 scratch_elems, int num_sms,
            cudaStream_t st, const int* skip) {
  i64 splits, tps, total;
  bool tc = false;
  if constexpr (std::is_same<T, float>::value) tc = tc_sketch_ok(X, P, v);
  if (tc) {
    splits = sketch_tc_splits(v, cols, num_sms, tps, total);
    if (splits * cols * v.I > scratch_elems) throw std::runtime_error("sketch: scratch too small");
    if constexpr (std::is_same<T, float>::value) {
      const i64 pf = sketch_tc_panel_floats(v, cols);
      // the blocked panel copy lives behind the partials (16-byte aligned) when the caller's scratch has room
      const i64 off = ceil_div(splits * cols * v.I, 4) * 4;
      float* pblk = (pf > 0 && off + pf <= scratch_elems) ? scratch + off : nullptr;
      sketch_tc(X, v, P, cols, scratch, pblk, num_sms, skip, st);
    }
  } else if (use_dmma<T>(v)) {
    splits = sketch_dmma_splits(v, cols, num_sms, tps, total);
    if (splits * cols * v.I > scratch_elems) throw std::runtime_error("sketch: scratch too small");
    if constexpr (std::is_same<T, double>::value) sketch_dmma(X, v, P, cols, scratch, num_sms, skip, st);
  } else {
  sketch_plan<T>(v, cols, num_sms, splits, tps, total);
  if (splits * cols * v.I > scratch_elems) throw std::runtime_error("sketch: scratch too small");
  switch (pick_bn(cols)) {
    case 16: sketch_bn<T, 16>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
    case 32: sketch_bn<T, 32>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
    case 48: sketch_bn<T, 48>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
    case 64: sketch_bn<T, 64>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
    default: sketch_bn<T, 80>(X, v, P, cols, scratch, splits, tps, total, st, skip); break;
  }
  }
  const i64 n = cols * v.I;
  reduce_partials_kernel<T, T><<<unsigned(ceil_div(n, 32)), 32 * kRedChunks, 0, st>>>(scratch, splits, n, Y, skip);
  count_launch();
  RCPG_LAUNCHED();
}

namespace {
// split-K factor of a last-mode projection: ~4 CTAs per SM, at least 2 K tiles each
template <typename T>
i64 project_last_splits(ModeView v, i64 cols, int num_sms, i64& tps) {
  constexpr int BM = TileCfg<T>::BM, BK = TileCfg<T>::BK;
  const i64 mt = ceil_div(v.L, BM), nt = ceil_div(cols, pick_bn(cols)), kt = ceil_div(v.I, BK);
  const i64 want = std::min<i64>(ceil_div(i64(4) * num_sms, mt * nt), kt / 2);
  if (v.R != 1 || want < 2) {
    tps = 0;
    return 1;
  }
  tps = ceil_div(kt, want);
  return ceil_div(kt, tps);
}

template <typename T, int BN>
void project_bn(const T* X, ModeView v, const T* Q, i64 ldq, i64 cols, T* O, cudaStream_t st, T* scratch,
                i64 scratch_elems) {
  constexpr int BM = TileCfg<T>::BM, BK = TileCfg<T>::BK;
  const i64 nt = ceil_div(cols, BN), kt = ceil_div(v.I, BK);
  if (v.R == 1 && scratch != nullptr) {
    // a small output (C2's last mode: 900 x 30 from 15 CTAs) splits K and sums
    // the partials in a fixed order (reduce_partials): 26 -> ~8 us
    i64 tps = 0;
    const i64 splits = project_last_splits<T>(v, cols, device_caps().num_sms, tps);
    if (splits > 1 && splits * v.L * cols <= scratch_elems) {
      dim3 grid{unsigned(ceil_div(v.L, BM)), unsigned(splits), unsigned(nt)};
      ProjectLastLoader<T, BM, BN, BK> ld{X, Q, v.L, v.I, cols, ldq, kt, nullptr, tps};
      ProjectLastPartEpilogue<T, BM, BN> ep{scratch, v.L, cols};
      launch_tile_gemm<T, BM, BN, BK, false>(grid, ld, ep, st);
      const i64 n = v.L * cols;
      reduce_partials_kernel<T, T><<<unsigned(ceil_div(n, 32)), 32 * kRedChunks, 0, st>>>(scratch, splits, n, O,
                                                                                         nullptr);
      count_launch();
      RCPG_LAUNCHED();
      return;
    }
  }
  if (v.R > 1) {
    // batch over a in chunks of 65535 (gridDim.y limit)
    for (i64 a0 = 0; a0 < v.L; a0 += 65535) {
      const i64 na = std::min<i64>(65535, v.L - a0);
      dim3 grid{unsigned(ceil_div(v.R, BM)), unsigned(na), unsigned(nt)};
      const i64 off = a0 * v.I * v.R, ooff = a0 * cols * v.R;
      ProjectLoader<T, BM, BN, BK> ld{X + off, Q, v.I, v.R, cols, ldq, kt};
      ProjectEpilogue<T, BM, BN> ep{O + ooff, v.R, cols};
      launch_tile_gemm<T, BM, BN, BK, true>(grid, ld, ep, st);
    }
  } else {
    dim3 grid{unsigned(ceil_div(v.L, BM)), 1u, unsigned(nt)};
    ProjectLastLoader<T, BM, BN, BK> ld{X, Q, v.L, v.I, cols, ldq, kt};
    ProjectLastEpilogue<T, BM, BN> ep{O, v.L, cols};
    launch_tile_gemm<T, BM, BN, BK, false>(grid, ld, ep, st);
  }
}
}  // namespace

template <typename T>
i64 project_scratch_elems(ModeView v, i64 cols, int num_sms) {
  i64 tps = 0;
  const i64 splits = project_last_splits<T>(v, cols, num_sms, tps);
  return splits > 1 ? splits * v.L * cols : 0;
}

template <typename T>
void project(const T* X, ModeView v, const T* Q, i64 ldq, i64 cols, T* O, cudaStream_t st, T* scratch,
             i64 scratch_elems) {
  if constexpr (std::is_same<T, double>::value) {
    if (v.R > 1) {
      project_dmma(X, v, Q, ldq, cols, O, st);
      return;
    }
  } else {
    if (tc_project_ok(X, Q, v, ldq)) {
      project_tc(X, v, Q, ldq, cols, O, device_caps().num_sms, st);
      return;
    }
  }
  switch (pick_bn(cols)) {
    case 16: project_bn<T, 16>(X, v, Q, ldq, cols, O, st, scratch, scratch_elems); break;
    case 32: project_bn<T, 32>(X, v, Q, ldq, cols, O, st, scratch, scratch_elems); break;
    case 48: project_bn<T, 48>(X, v, Q, ldq, cols, O, st, scratch, scratch_elems); break;
    case 64: project_bn<T, 64>(X, v, Q, ldq, cols, O, st, scratch, scratch_elems); break;
    default: project_bn<T, 80>(X, v, Q, ldq, cols, O, st, scratch, scratch_elems); break;
  }
}

// ---------------------------------------------------------------- Omega
namespace {
template <typename T, typename TV = T>
__global__ void omega_panel_kernel(u64 s0, KoldaMap km, i64 J, i64 R, i64 cols, int distribution, T* P, i64 Jg) {
  for (i64 s = blockIdx.x * i64(blockDim.x) + threadIdx.x; s < J; s += i64(gridDim.x) * blockDim.x) {
    const i64 a = s / R, b = s - a * R;
    const i64 j = kolda_index(km, a, b);
    T* dst = P + a * cols * R + b;
    for (i64 c = 0; c < cols; ++c) {
      const u64 e = u64(c) * u64(Jg) + u64(j);  // Jg: rows of the (global) unfolding
      const double v = distribution == 0 ? normal_at(s0, e) : uniform_sym_at(s0, e);
      dst[c * R] = T(TV(v));
    }
  }
}
// Gaussian Omega, one Box-Muller pair per thread and column: entries e = c Jg + j
// and e + 1 form pair e / 2 (cos, sin). With Jg even and j even they share the
// column c, and j + 1 increments the fastest Kolda digit, whose storage stride
// (in panel rows) is `sig` -- so the thread owning row s (that digit even)
// writes rows s and s + sig, both coalesced across the warp, and every pair is
// computed once instead of twice.
template <typename T, typename TV = T>
__global__ void omega_pairs_kernel(u64 s0, KoldaMap km, i64 J, i64 R, i64 cols, T* P, i64 Jg, i64 sig, i64 Ef) {
  const i64 half = J / 2;
  for (i64 q = blockIdx.x * i64(blockDim.x) + threadIdx.x; q < half; q += i64(gridDim.x) * blockDim.x) {
    const i64 lo = q % sig, rest = q / sig;
    const i64 t = rest % (Ef / 2), hi = rest / (Ef / 2);
    const i64 s = hi * Ef * sig + 2 * t * sig + lo;  // storage row with an even fastest Kolda digit
    const i64 a = s / R, b = s - a * R;
    const i64 s2 = s + sig, a2 = s2 / R, b2 = s2 - a2 * R;
    const i64 j = kolda_index(km, a, b);
    T* d1 = P + a * cols * R + b;
    T* d2 = P + a2 * cols * R + b2;
    for (i64 c = blockIdx.y; c < cols; c += gridDim.y) {  // column groups: small panels spread over the SMs
      double cs, sn;
      normal_pair(s0, (u64(c) * u64(Jg) + u64(j)) >> 1, cs, sn);
      d1[c * R] = T(TV(cs));
      d2[c * R] = T(TV(sn));
    }
  }
}
}  // namespace

namespace {
// TV: the Scalar type the reference stores Omega in (Matrix<S>, compress.hpp:120);
// T: the panel's storage type (fp64 for the fp32 configs' faithful passes)
template <typename T, typename TV>
void omega_panel_impl(u64 seed, i64 mode, const KoldaMap& km, ModeView v, i64 cols, int distribution, T* P,
                      cudaStream_t st, i64 J_global) {
  const u64 s0 = derive_seed(seed, stream_id(kDomainCompress, u64(mode)));
  const i64 J = v.L * v.R;
  const i64 Jg = J_global > 0 ? J_global : J;
  // fastest Kolda digit: low mode 0 if there are low modes, else high mode 0;
  // its stride in panel rows s = a R + b
  i64 Ef, sig;
  if (km.n_low > 0) {
    Ef = km.low_ext[0];
    sig = v.R;
    for (int m = 1; m < km.n_low; ++m) sig *= km.low_ext[m];
  } else {
    Ef = km.n_high > 0 ? km.high_ext[0] : 1;
    sig = 1;
    for (int m = 1; m < km.n_high; ++m) sig *= km.high_ext[m];
  }
  // (a slab's last digit carries an offset but is never the fastest Kolda digit
  // when there are other high modes; with one high mode Ef is its local extent)
  const bool pairs = distribution == 0 && Jg % 2 == 0 && J % 2 == 0 && Ef % 2 == 0 && Ef >= 2 &&
                     !(km.n_low == 0 && km.n_high == 1 && km.high_last_off % 2 != 0);
  if (pairs) {
    const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(J / 2, 256), 148 * 16)));
    // a thread evaluates its row pair's columns one after the other (a chain of
    // fp64 log / sincos): panels with few rows get column groups in grid.y until
    // ~8 CTAs per SM are in flight (C2 mode 0: 313 x 4 CTAs instead of 313)
    const int ygroups = int(std::max<i64>(1, std::min<i64>(cols, ceil_div(i64(148) * 8, i64(blocks)))));
    omega_pairs_kernel<T, TV><<<dim3(unsigned(blocks), unsigned(ygroups)), 256, 0, st>>>(s0, km, J, v.R, cols, P, Jg,
                                                                                       sig, Ef);
    count_launch();
    RCPG_LAUNCHED();
    return;
  }
  const int blocks = int(std::max<i64>(1, std::min<i64>(ceil_div(J, 256), 148 * 16)));
  omega_panel_kernel<T, TV><<<blocks, 256, 0, st>>>(s0, km, J, v.R, cols, distribution, P, Jg);
  count_launch();
  RCPG_LAUNCHED();
}
}  // namespace

template <typename T>
void omega_panel(u64 seed, i64 mode, const KoldaMap& km, ModeView v, i64 cols, int distribution, T* P,
                 cudaStream_t st, i64 J_global) {
  omega_panel_impl<T, T>(seed, mode, km, v, cols, distribution, P, st, J_global);
}

void omega_panel_f32_as_f64(u64 seed, i64 mode, const KoldaMap& km, ModeView v, i64 cols, int distribution,
                            double* P, cudaStream_t st, i64 J_global) {
  omega_panel_impl<double, float>(seed, mode, km, v, cols, distribution, P, st, J_global);
}

#define RCPG_INST(T)                                                                                     \
  template i64 sketch_scratch_elems<T>(ModeView, i64, int);                                              \
  template void sketch<T>(const T*, ModeView, const T*, i64, T*, T*, i64, int, cudaStream_t, const int*);             \
  template void project<T>(const T*, ModeView, const T*, i64, i64, T*, cudaStream_t, T*, i64);           \
  template i64 project_scratch_elems<T>(ModeView, i64, int);                                                \
  template void omega_panel<T>(u64, i64, const KoldaMap&, ModeView, i64, int, T*, cudaStream_t, i64);
RCPG_INST(float)
RCPG_INST(double)
#undef RCPG_INST

}  // namespace rcpg
