// SPDX-License-Identifier: MIT
// FP32 streamed passes on the 5th-generation tensor cores: TMA -> smem,
// operand A in TMEM, tcgen05.mma kind::tf32 into TMEM accumulators, fp32
// accuracy through the 3xTF32 split
//   x = hi + lo, hi = TF32(x), lo = x - hi (exact in fp32),
//   a.b ~= hi_a.hi_b + hi_a.lo_b + lo_a.hi_b   (dropped lo.lo ~ 2^-22 |a||b|).
//
//   sketch  Y[i, c]    = sum_{a,b} X[a, i, b] P[a, c, b]   M = i, N = c, K = (a, b)
//   project O[a, c, b] = sum_i X[a, i, b] Q[i, c]          M = b, N = c, K = i
// (mode views with R > 1; the X_(n) Omega, X_(n)^T Q, X_(n) Z and Q^T X_(n)
// products of compress.hpp:118-145.)
//
// Facts pinned on hardware (tools/microbench/umma_*.cu): kind::tf32
// truncates fp32 inputs (so the raw value is the hi operand); it accepts
// K-major operands only (MN-major returned zeros); an MMA reading both
// operands from smem is bound by the ~128 B/clk smem read port (A = 4 KB per
// M=128,K=8 step), while an A operand in TMEM leaves the port to B.
//
// Hence the dataflow per K-tile (32 values of the reduction index):
//   warp 0 (1 thread)  TMA: X tile and panel tile -> smem stage (128B swizzle,
//                      out-of-range rows / columns zero-filled by the TMA unit)
//   warps 2-5          row m = TMEM lane: read row m of the X tile (sketch: a
//                      K-contiguous row; projection: one column of the
//                      b-contiguous tile, i.e. the transpose, conflict-free),
//                      tcgen05.st hi and lo into a TMEM A slot; lo plane of the
//                      panel tile -> smem
//   warps 1, 6         two MMA issuers (1 thread each, different SM
//                      sub-partitions): 6 x tcgen05.mma (M=128, N=BN, K=8; A
//                      from TMEM, B from smem) each, for half of the K-tile's
//                      K=8 steps, into their own accumulator; commit -> frees
//                      the stage and the A slot
// One issuing warp sustains one tf32 MMA per ~45 cycles whatever N is (the
// tensor pipe needs N/2 cycles: 40 at N = 80), so a single issuer caps a
// K-tile at 12 x 45 cycles; two issuers reach the pipe rate. The epilogue
// adds the two accumulators (fixed order: deterministic).
// Stages (smem), A slots (TMEM) and the accumulators (TMEM) are handed
// between the roles with mbarriers, so TMA, conversion and MMA of different
// K-tiles overlap. CTAs are persistent (one per SM) over work items; when
// TMEM allows (BN <= 80) the accumulator pair alternates between two column
// blocks, so the epilogue of item j (tcgen05.ld -> coalesced stores) overlaps
// item j+1's MMAs.
#include <cuda.h>  // CUtensorMap and its enums (entry point fetched at run time)

#include <cstdlib>
#include <string>

#include "passes.cuh"
#include "runtime.cuh"
#include "tc.cuh"

namespace rcpg {

namespace {

using namespace tc;

constexpr int kThreads = 224;  // warp 0 TMA, warps 1 + 6 MMA, warps 2-5 convert + epilogue
constexpr int kIssuers = 2;
constexpr int kBM = 128, kBK = 32;
constexpr uint32_t kTmemCols = 512;
constexpr int kSmemBudget = 216 * 1024;

template <int BN, bool PROJ>
struct Plan {
  static constexpr int A_BYTES = kBM * kBK * 4;  // 16 KB
  static constexpr int B_BYTES = BN * kBK * 4;
  static constexpr int B_CH = B_BYTES / 16;
  static constexpr int STAGE = A_BYTES + 2 * B_BYTES;  // raw X | raw panel | panel lo
  static constexpr int S = (kSmemBudget / STAGE) < 8 ? (kSmemBudget / STAGE) : 8;
  static constexpr int SMEM = S * STAGE + 1024;  // + alignment slack (SWIZZLE_128B wants 1024 B)
  static constexpr uint32_t TX = A_BYTES + B_BYTES;
  // TMEM: DBUF x kIssuers accumulators of BN columns, then A slots of 64
  // columns (hi | lo) from a 32-aligned column.
  // sketch: few, long work items -> one accumulator pair, more A slots;
  // projection: many short items -> double-buffered accumulators if they fit
  static constexpr int DBUF = (PROJ && 2 * kIssuers * BN + 3 * 64 <= int(kTmemCols)) ? 2 : 1;
  static constexpr uint32_t ACOL0 = uint32_t((DBUF * kIssuers * BN + 31) / 32 * 32);
  static constexpr int SA_FIT = int((kTmemCols - ACOL0) / 64);
  static constexpr int SA = SA_FIT < 6 ? SA_FIT : 6;
  __host__ __device__ static constexpr uint32_t dcol(int buf, int issuer) {
    return uint32_t((buf * kIssuers + issuer) * BN);
  }
  static constexpr uint32_t IDESC = idesc_tf32(kBM, BN, 0, 0);
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 128, "UMMA N for M = 128");
  static_assert(S >= 3 && SA >= 3, "pipeline depth");
};

struct TcArgs {
  i64 L, I, R, cols;
  i64 items;     // work items (all CTAs)
  i64 n_mtiles;  // sketch: i-tiles; projection: b-tiles
  i64 n_ntiles;
  i64 nbt, tps, total;  // sketch: K-tiles per slab row, K-tiles per split, total K-tiles
  float* out;           // sketch: partials [split][c][i]; projection: O (a, c, b)
  const int* skip;
};

// Work item id -> (n-tile fastest, then m-tile, then split / slab): CTAs
// running concurrently share a K range (sketch) or slab (projection), so the
// panel tile they all read stays in L2.
struct Item {
  i64 hi;  // sketch: K split; projection: slab a
  i64 m0;
  i64 nt;
  i64 t0;  // sketch: first K-tile
  int nk;  // K-tiles
};

template <bool PROJ>
__device__ __forceinline__ Item item_of(const TcArgs& p, i64 id) {
  Item it;
  it.nt = id % p.n_ntiles;
  const i64 rest = id / p.n_ntiles;
  it.m0 = (rest % p.n_mtiles) * kBM;
  it.hi = rest / p.n_mtiles;
  if (PROJ) {
    it.t0 = 0;
    it.nk = int((p.I + kBK - 1) / kBK);
  } else {
    it.t0 = it.hi * p.tps;
    it.nk = int(min(p.tps, p.total - it.t0));
  }
  return it;
}

__device__ __forceinline__ float lo_part(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int BN, bool PROJ>
__global__ void __launch_bounds__(kThreads, 1)
    tc_pass_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmP, TcArgs p) {
  using G = Plan<BN, PROJ>;
  constexpr int S = G::S;
  if (p.skip != nullptr && *p.skip) return;
  extern __shared__ unsigned char smem_dyn[];
  unsigned char* smem = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t full[S], sdone[S], empty[S], aslot[G::SA], accf[2], acce[2];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sdone[s], 128);
      mbar_init(&empty[s], kIssuers);
    }
    for (int s = 0; s < G::SA; ++s) mbar_init(&aslot[s], kIssuers);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], kIssuers);
      mbar_init(&acce[b], 128);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmP);
  }
  if (warp == 1) tmem_alloc(&tmem_sh, kTmemCols);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_sh;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      int q = 0;
      for (i64 id = blockIdx.x; id < p.items; id += gridDim.x) {
        const Item it = item_of<PROJ>(p, id);
        const int n0 = int(it.nt) * BN;
        i64 a = 0, bt = 0;
        if (!PROJ) {
          a = it.t0 / p.nbt;
          bt = it.t0 - a * p.nbt;
        }
        for (int kt = 0; kt < it.nk; ++kt, ++q) {
          const int s = q % S;
          if (q >= S) mbar_wait(&empty[s], uint32_t(((q / S) - 1) & 1));
          unsigned char* st = smem + s * G::STAGE;
          mbar_arrive_tx(&full[s], G::TX);
          if (!PROJ) {
            tma_load_3d(st, &tmX, int(bt * kBK), int(it.m0), int(a), &full[s]);
            tma_load_3d(st + G::A_BYTES, &tmP, int(bt * kBK), n0, int(a), &full[s]);
            if (++bt == p.nbt) {
              bt = 0;
              ++a;
            }
          } else {
#pragma unroll
            for (int g = 0; g < 4; ++g)
              tma_load_3d(st + g * 4096, &tmX, int(it.m0) + 32 * g, kt * kBK, int(it.hi), &full[s]);
            tma_load_2d(st + G::A_BYTES, &tmP, kt * kBK, n0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1 || warp == 6) {
    // ------------------------------------------------------ MMA issuers
    if (lane == 0) {
      const int who = warp == 1 ? 0 : 1;  // K=8 steps {2 who, 2 who + 1} of every K-tile
      int q = 0, j = 0;
      for (i64 id = blockIdx.x; id < p.items; id += gridDim.x, ++j) {
        const Item it = item_of<PROJ>(p, id);
        const int buf = j % G::DBUF;
        const uint32_t d = tmem + G::dcol(buf, who);
        for (int kt = 0; kt < it.nk; ++kt, ++q) {
          const int s = q % S, slot = q % G::SA;
          mbar_wait(&sdone[s], uint32_t((q / S) & 1));
          if (kt == 0 && j >= G::DBUF) mbar_wait(&acce[buf], uint32_t(((j / G::DBUF) - 1) & 1));
          fence_after_sync();
          const uint32_t ahi = tmem + G::ACOL0 + uint32_t(slot) * 64, alo = ahi + 32;
          const uint32_t bhi = smem_u32(smem + s * G::STAGE + G::A_BYTES), blo = bhi + G::B_BYTES;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int k8 = 2 * who + u;
            const uint64_t bh = sdesc_sw128(bhi + 32 * k8), bl = sdesc_sw128(blo + 32 * k8);
            mma_tf32_ta(d, alo + 8 * k8, bh, G::IDESC, (kt > 0 || u > 0) ? 1u : 0u);
            mma_tf32_ta(d, ahi + 8 * k8, bl, G::IDESC, 1u);
            mma_tf32_ta(d, ahi + 8 * k8, bh, G::IDESC, 1u);
          }
          mma_commit(&empty[s]);
          mma_commit(&aslot[slot]);
          if (kt == it.nk - 1) mma_commit(&accf[buf]);
        }
      }
    }
  } else {
    // ---------------------------------------- convert + epilogue (128 thr)
    const int qd = warp & 3;  // TMEM lane quadrant this warp may access
    const int m = qd * 32 + lane;
    const int ctid = threadIdx.x - 64;
    const uint32_t my_lanes = tmem + tmem_lane(qd);

    auto epilogue = [&](i64 id, int j) {
      const int buf = j % G::DBUF;
      mbar_wait(&accf[buf], uint32_t((j / G::DBUF) & 1));
      fence_after_sync();
      const Item it = item_of<PROJ>(p, id);
      const i64 n0 = it.nt * BN;
      const i64 row = it.m0 + m;
      const i64 nrows = PROJ ? p.R : p.I;
      float* out = p.out + it.hi * p.cols * nrows;  // sketch: split slab; projection: slab a
      const uint32_t t0 = my_lanes + G::dcol(buf, 0), t1 = my_lanes + G::dcol(buf, 1);
#pragma unroll
      for (int c8 = 0; c8 < BN; c8 += 8) {
        float v[8], w[8];
        tmem_ld8(t0 + c8, v);
        tmem_ld8(t1 + c8, w);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] += w[u];
        if (row < nrows) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (n0 + c8 + u < p.cols) out[(n0 + c8 + u) * nrows + row] = v[u];
        }
      }
      fence_before_sync();
      mbar_arrive(&acce[buf]);
    };

    int q = 0, j = 0;
    i64 prev = -1;
    for (i64 id = blockIdx.x; id < p.items; id += gridDim.x, ++j) {
      const Item it = item_of<PROJ>(p, id);
      for (int kt = 0; kt < it.nk; ++kt, ++q) {
        const int s = q % S, slot = q % G::SA;
        unsigned char* st = smem + s * G::STAGE;
        mbar_wait(&full[s], uint32_t((q / S) & 1));
        float hi[32], lo[32];
        if (!PROJ) {
          // row m of the K-major tile: chunk c stored at c ^ (m % 8)
          const unsigned char* row = st + (m >> 3) * 1024 + (m & 7) * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = *reinterpret_cast<const float4*>(row + ((c ^ (m & 7)) << 4));
            hi[4 * c] = x.x;
            hi[4 * c + 1] = x.y;
            hi[4 * c + 2] = x.z;
            hi[4 * c + 3] = x.w;
          }
        } else {
          // column m of the b-contiguous tile: box qd holds b in [m0 + 32 qd, +32),
          // row k (= i) at k * 128, chunk (lane / 4) ^ (k % 8)
          const unsigned char* box = st + qd * 4096 + (lane & 3) * 4;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            hi[k] = *reinterpret_cast<const float*>(box + k * 128 + ((((lane >> 2) ^ (k & 7))) << 4));
        }
        // lo plane of the panel tile (same swizzled positions)
        {
          const unsigned char* braw = st + G::A_BYTES;
          unsigned char* blo = st + G::A_BYTES + G::B_BYTES;
          constexpr int NB = (G::B_CH + 127) / 128;
          float4 x[NB];
#pragma unroll
          for (int u = 0; u < NB; ++u)
            if (ctid + 128 * u < G::B_CH) x[u] = *reinterpret_cast<const float4*>(braw + 16 * (ctid + 128 * u));
#pragma unroll
          for (int u = 0; u < NB; ++u)
            if (ctid + 128 * u < G::B_CH)
              *reinterpret_cast<float4*>(blo + 16 * (ctid + 128 * u)) =
                  make_float4(lo_part(x[u].x), lo_part(x[u].y), lo_part(x[u].z), lo_part(x[u].w));
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) lo[k] = lo_part(hi[k]);
        // only the TMEM store waits for the A slot to drain
        if (q >= G::SA) mbar_wait(&aslot[slot], uint32_t(((q / G::SA) - 1) & 1));
        fence_after_sync();
        const uint32_t acol = G::ACOL0 + uint32_t(slot) * 64;
        tmem_st32(my_lanes + acol, hi);
        tmem_st32(my_lanes + acol + 32, lo);
        tmem_st_wait();
        fence_proxy_async();
        fence_before_sync();
        mbar_arrive(&sdone[s]);
        if (kt == 0 && prev >= 0) epilogue(prev, j - 1);
      }
      prev = id;
    }
    if (prev >= 0) epilogue(prev, j - 1);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// ------------------------------------------------------------------ host
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    RCPG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (f == nullptr || q != cudaDriverEntryPointSuccess)
      throw CudaFailure("cuTensorMapEncodeTiled is not available from the driver", cudaErrorNotSupported);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// fp32 tiled map, SWIZZLE_128B, zero fill out of range. dims/strides innermost first.
CUtensorMap tensor_map(const float* base, cuuint32_t rank, const cuuint64_t* dims, const cuuint64_t* strides,
                       const cuuint32_t* box) {
  CUtensorMap m;
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(base), dims,
                                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaFailure("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")", cudaErrorInvalidValue);
  return m;
}

int pick_bn_tc(i64 cols) {
  if (cols >= 128) return 128;
  return int((cols + 15) / 16 * 16);
}

template <int BN, bool PROJ>
void launch(const CUtensorMap& mx, const CUtensorMap& mp, const TcArgs& a, int grid, cudaStream_t st) {
  static const size_t lim = enable_max_dyn_smem(tc_pass_kernel<BN, PROJ>);
  if (size_t(Plan<BN, PROJ>::SMEM) > lim) throw std::runtime_error("tc pass: smem plan too large");
  tc_pass_kernel<BN, PROJ><<<grid, kThreads, Plan<BN, PROJ>::SMEM, st>>>(mx, mp, a);
  count_launch();
  RCPG_LAUNCHED();
}

template <bool PROJ>
void dispatch(int bn, const CUtensorMap& mx, const CUtensorMap& mp, const TcArgs& a, int grid, cudaStream_t st) {
  switch (bn) {
    case 16: launch<16, PROJ>(mx, mp, a, grid, st); break;
    case 32: launch<32, PROJ>(mx, mp, a, grid, st); break;
    case 48: launch<48, PROJ>(mx, mp, a, grid, st); break;
    case 64: launch<64, PROJ>(mx, mp, a, grid, st); break;
    case 80: launch<80, PROJ>(mx, mp, a, grid, st); break;
    case 96: launch<96, PROJ>(mx, mp, a, grid, st); break;
    case 112: launch<112, PROJ>(mx, mp, a, grid, st); break;
    default: launch<128, PROJ>(mx, mp, a, grid, st); break;
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr i64 kMaxCoord = (i64(1) << 31) - 1;

}  // namespace

bool tc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RCPG_NO_TC");
    return !(e != nullptr && e[0] == '1');
  }();
  return on;
}

bool tc_sketch_ok(const float* X, const float* P, ModeView v) {
  return tc_enabled() && v.R > 1 && v.R % 4 == 0 && v.R <= kMaxCoord && v.I <= kMaxCoord && v.L <= kMaxCoord &&
         aligned16(X) && aligned16(P);
}

bool tc_project_ok(const float* X, const float* Q, ModeView v, i64 ldq) {
  return tc_enabled() && v.R > 1 && v.R % 4 == 0 && ldq % 4 == 0 && v.R <= kMaxCoord && v.I <= kMaxCoord &&
         v.L <= kMaxCoord && aligned16(X) && aligned16(Q);
}

i64 sketch_tc_splits(ModeView v, i64 cols, int num_sms, i64& tps, i64& total) {
  const i64 tiles = ceil_div(v.I, kBM) * ceil_div(cols, pick_bn_tc(cols));
  total = v.L * ceil_div(v.R, kBK);
  // ~8 work items per SM keeps the persistent grid's tail short
  i64 want = std::max<i64>(1, ceil_div(i64(8) * num_sms, tiles));
  want = std::min<i64>(want, total);
  tps = std::max<i64>(1, ceil_div(total, want));
  return ceil_div(total, tps);
}

void sketch_tc(const float* X, ModeView v, const float* P, i64 cols, float* part, int num_sms, const int* skip,
               cudaStream_t st) {
  const int bn = pick_bn_tc(cols);
  TcArgs a{};
  a.L = v.L;
  a.I = v.I;
  a.R = v.R;
  a.cols = cols;
  a.out = part;
  a.skip = skip;
  const i64 splits = sketch_tc_splits(v, cols, num_sms, a.tps, a.total);
  a.nbt = ceil_div(v.R, kBK);
  a.n_mtiles = ceil_div(v.I, kBM);
  a.n_ntiles = ceil_div(cols, bn);
  a.items = splits * a.n_mtiles * a.n_ntiles;
  const cuuint64_t xd[3] = {cuuint64_t(v.R), cuuint64_t(v.I), cuuint64_t(v.L)};
  const cuuint64_t xs[2] = {cuuint64_t(v.R) * 4, cuuint64_t(v.I * v.R) * 4};
  const cuuint32_t xb[3] = {kBK, kBM, 1};
  const cuuint64_t pd[3] = {cuuint64_t(v.R), cuuint64_t(cols), cuuint64_t(v.L)};
  const cuuint64_t ps[2] = {cuuint64_t(v.R) * 4, cuuint64_t(cols * v.R) * 4};
  const cuuint32_t pb[3] = {kBK, cuuint32_t(bn), 1};
  const CUtensorMap mx = tensor_map(X, 3, xd, xs, xb);
  const CUtensorMap mp = tensor_map(P, 3, pd, ps, pb);
  const int grid = int(std::min<i64>(a.items, num_sms));
  dispatch<false>(bn, mx, mp, a, grid, st);
}

void project_tc(const float* X, ModeView v, const float* Q, i64 ldq, i64 cols, float* O, int num_sms,
                cudaStream_t st) {
  const int bn = pick_bn_tc(cols);
  TcArgs a{};
  a.L = v.L;
  a.I = v.I;
  a.R = v.R;
  a.cols = cols;
  a.out = O;
  a.n_mtiles = ceil_div(v.R, kBM);
  a.n_ntiles = ceil_div(cols, bn);
  a.items = v.L * a.n_mtiles * a.n_ntiles;
  const cuuint64_t xd[3] = {cuuint64_t(v.R), cuuint64_t(v.I), cuuint64_t(v.L)};
  const cuuint64_t xs[2] = {cuuint64_t(v.R) * 4, cuuint64_t(v.I * v.R) * 4};
  const cuuint32_t xb[3] = {32, kBK, 1};
  const cuuint64_t qd[2] = {cuuint64_t(v.I), cuuint64_t(cols)};
  const cuuint64_t qs[1] = {cuuint64_t(ldq) * 4};
  const cuuint32_t qb[2] = {kBK, cuuint32_t(bn)};
  const CUtensorMap mx = tensor_map(X, 3, xd, xs, xb);
  const CUtensorMap mq = tensor_map(Q, 2, qd, qs, qb);
  const int grid = int(std::min<i64>(a.items, num_sms));
  dispatch<true>(bn, mx, mq, a, grid, st);
}

}  // namespace rcpg
