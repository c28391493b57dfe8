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
  int pblk;             // sketch panel: 0 (a, c, b) map; 1 blocked raw; 2 blocked hi | lo planes
  i64 cpad;             // blocked panel: columns per K-tile block (n-tiles x BN)
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
          mbar_arrive_tx(&full[s], G::TX + (!PROJ && p.pblk == 2 ? uint32_t(G::B_BYTES) : 0u));
          if (!PROJ) {
            tma_load_3d(st, &tmX, int(bt * kBK), int(it.m0), int(a), &full[s]);
            if (p.pblk == 0) {
              tma_load_3d(st + G::A_BYTES, &tmP, int(bt * kBK), n0, int(a), &full[s]);
            } else {  // K-tile block (a, bt): rows [plane][cpad] of 32 contiguous values
              const i64 blk = (a * p.nbt + bt) * (p.pblk == 2 ? 2 : 1);
              tma_load_2d(st + G::A_BYTES, &tmP, 0, int(blk * p.cpad + n0), &full[s]);
              if (p.pblk == 2) tma_load_2d(st + G::A_BYTES + G::B_BYTES, &tmP, 0, int((blk + 1) * p.cpad + n0), &full[s]);
            }
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
        // lo plane of the panel tile (same swizzled positions), unless it came by TMA
        if (PROJ || p.pblk != 2) {
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

// ------------------------------------------------- residual (relerr)
// ||X - Xhat||^2 and ||X||^2 with Xhat on tcgen05 (kruskal.hpp:187-194):
// rows p of X (all modes but the last, row-major) x the last mode k,
//   Xhat[p, k] = sum_r coef[p, r] C[k, r],  coef[p, r] = lambda_r prod_m A_m[d_m(p), r],
// an M = 128 (p) x N = 128 (k) x K = R (padded) GEMM per work item, 3xTF32.
// The coef rows are formed by the epilogue warps (lane = row = TMEM lane)
// and stored hi / lo into TMEM (A operand); C^T hi / lo (K-major, prepared
// once) and the X tile arrive by TMA; the epilogue reads Xhat from TMEM and
// X from smem and accumulates both sums in fp64. Out-of-range rows / columns
// are zero on both sides (zero coef, TMA zero fill), so they add nothing.
constexpr int kResMaxOrder = 8;
constexpr int kRBM = 128, kRBN = 64;
// warp 0 TMA, warp 1 MMA, warps 2-9 coef + epilogue: two warps per TMEM lane
// quadrant, each taking one 32-column box of an item (with four epilogue warps,
// one per scheduler, the epilogue had no latency hiding: C5 3.2 TB/s)
constexpr int kResThreads = 320;
constexpr int kResEpi = kResThreads - 64;  // epilogue threads (mbarrier arrival counts)

struct ResArgs {
  i64 P, E;
  int R, N;                      // rank, tensor order
  i64 ext[kResMaxOrder];         // extents of modes 0 .. N-2
  const float* f[kResMaxOrder];
  const float* w;
  i64 mtiles, ntiles, items, chunk;
  double* part;  // [gridDim][2]
};

// Items are (m-tile, n-tile) with the n-tile fastest: the coef rows of an
// m-tile are formed once and stay in TMEM for all of its n-tiles. X tiles
// stream through an SX-deep ring freed by the epilogue (the kernel's bytes);
// the C^T tiles (hi | lo, from L2) through an SB-deep ring freed by the MMA
// commit (a C^T tile is reloaded per item; with only two in flight the MMA
// waited on its L2 latency and the epilogue on the MMA: ncu, C5).
template <int KP>
struct ResPlan {
  static constexpr int KB = KP / 32;                  // 32-wide swizzle boxes along K
  static constexpr int B_PLANE = KP * kRBN * 4;       // one plane of the C^T tile
  static constexpr int X_BYTES = kRBM * kRBN * 4;     // 32 KB: 2 boxes of 32 columns
  static constexpr int B_STAGE = 2 * B_PLANE;
  static constexpr int SB = KP >= 64 ? 3 : 4;
  static constexpr int SX_FIT = (200 * 1024 - SB * B_STAGE) / X_BYTES;
  static constexpr int SX = SX_FIT < 6 ? SX_FIT : 6;
  static constexpr int SMEM = SX * X_BYTES + SB * B_STAGE + 1024;
  static constexpr uint32_t ACOL = 0;                 // A slots: 2 x (hi KP | lo KP)
  static constexpr uint32_t DCOL = 4 * KP;            // accumulators: NACC x kRBN
  static constexpr int NACC = 4;                      // MMA runs up to 3 items ahead of the epilogue
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t IDESC = idesc_tf32(kRBM, kRBN, 0, 0);
  static_assert(DCOL + NACC * kRBN <= TMEM_COLS, "TMEM plan");
  static_assert(SX >= 2, "X ring depth");
};

template <int KP>
__global__ void __launch_bounds__(kResThreads, 1)
    residual_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmBh,
                       const __grid_constant__ CUtensorMap tmBl, ResArgs p) {
  using G = ResPlan<KP>;
  constexpr int SX = G::SX, SB = G::SB;
  extern __shared__ unsigned char smem_dyn[];
  unsigned char* smem = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
  unsigned char* bsm = smem + SX * G::X_BYTES;  // C^T ring
  constexpr int NA = G::NACC;
  __shared__ __align__(8) uint64_t fullx[SX], emptyx[SX], fullb[SB], emptyb[SB], afull[2], aempty[2], accf[NA], acce[NA];
  __shared__ uint32_t tmem_sh;
  __shared__ double red[2][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 c0 = i64(blockIdx.x) * p.chunk;
  const i64 c1 = c0 + p.chunk < p.items ? c0 + p.chunk : p.items;
  const int n_items = c1 > c0 ? int(c1 - c0) : 0;
  const i64 mt0 = c0 / p.ntiles;  // first m-tile of this CTA; A slot of m-tile mt = (mt - mt0) & 1

  if (threadIdx.x == 0) {
    for (int b = 0; b < SX; ++b) {
      mbar_init(&fullx[b], 1);
      mbar_init(&emptyx[b], kResEpi);
    }
    for (int b = 0; b < SB; ++b) {
      mbar_init(&fullb[b], 1);
      mbar_init(&emptyb[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], kResEpi);
      mbar_init(&aempty[b], 1);
    }
    for (int b = 0; b < NA; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], kResEpi);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmBh);
    tma_prefetch_desc(&tmBl);
  }
  if (warp == 1) tmem_alloc(&tmem_sh, G::TMEM_COLS);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_sh;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int j = 0; j < n_items; ++j) {
        const i64 id = c0 + j, mt = id / p.ntiles, nt = id - mt * p.ntiles;
        const int sx = j % SX, sb = j % SB;
        if (j >= SX) mbar_wait(&emptyx[sx], uint32_t(((j / SX) - 1) & 1));
        unsigned char* xs = smem + sx * G::X_BYTES;
        mbar_arrive_tx(&fullx[sx], G::X_BYTES);
#pragma unroll
        for (int g = 0; g < kRBN / 32; ++g)
          tma_load_2d(xs + g * (kRBM * 128), &tmX, int(nt * kRBN) + 32 * g, int(mt * kRBM), &fullx[sx]);
        if (j >= SB) mbar_wait(&emptyb[sb], uint32_t(((j / SB) - 1) & 1));
        unsigned char* bs = bsm + sb * G::B_STAGE;
        mbar_arrive_tx(&fullb[sb], G::B_STAGE);
#pragma unroll
        for (int kb = 0; kb < G::KB; ++kb) {
          tma_load_2d(bs + kb * (kRBN * 128), &tmBh, 32 * kb, int(nt * kRBN), &fullb[sb]);
          tma_load_2d(bs + G::B_PLANE + kb * (kRBN * 128), &tmBl, 32 * kb, int(nt * kRBN), &fullb[sb]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      for (int j = 0; j < n_items; ++j) {
        const i64 id = c0 + j, mt = id / p.ntiles, nt = id - mt * p.ntiles;
        const int sb = j % SB, buf = j % NA, u = int((mt - mt0) & 1);
        const int tloc = int(mt - mt0);
        const bool first = (nt == 0 || j == 0), last = (nt == p.ntiles - 1 || j == n_items - 1);
        mbar_wait(&fullb[sb], uint32_t((j / SB) & 1));
        if (first) mbar_wait(&afull[u], uint32_t((tloc >> 1) & 1));
        if (j >= NA) mbar_wait(&acce[buf], uint32_t(((j / NA) - 1) & 1));
        fence_after_sync();
        const uint32_t d = tmem + G::DCOL + uint32_t(buf) * kRBN;
        const uint32_t ah = tmem + G::ACOL + uint32_t(u) * 2 * KP, al = ah + KP;
        const uint32_t bh0 = smem_u32(bsm + sb * G::B_STAGE), bl0 = bh0 + G::B_PLANE;
#pragma unroll
        for (int k8 = 0; k8 < KP / 8; ++k8) {
          const uint32_t off = uint32_t((k8 >> 2) * (kRBN * 128) + (k8 & 3) * 32);
          const uint64_t bh = sdesc_sw128(bh0 + off), bl = sdesc_sw128(bl0 + off);
          mma_tf32_ta(d, al + 8 * k8, bh, G::IDESC, k8 > 0 ? 1u : 0u);
          mma_tf32_ta(d, ah + 8 * k8, bl, G::IDESC, 1u);
          mma_tf32_ta(d, ah + 8 * k8, bh, G::IDESC, 1u);
        }
        mma_commit(&accf[buf]);
        mma_commit(&emptyb[sb]);
        if (last) mma_commit(&aempty[u]);
      }
    }
  } else {
    // ------------------------------------- coef rows + residual epilogue
    const int qd = warp & 3, gq = (warp - 2) >> 2;  // lane quadrant, column half
    const int m = qd * 32 + lane;
    const uint32_t my_lanes = tmem + tmem_lane(qd);
    double acc_r = 0.0, acc_x = 0.0;
    // coef rows of m-tile mt -> A slot (mt - mt0) & 1, formed one m-tile ahead
    // of the MMA (at the first item of m-tile t: coef(t + 1)), so the MMA never
    // waits on these gathers
    auto form_coef = [&](i64 mt) {
      const int tloc = int(mt - mt0), u = tloc & 1;
      const i64 prow = mt * kRBM + m;
      const bool valid = prow < p.P;
      i64 dig[kResMaxOrder];
      {
        i64 rem = valid ? prow : 0;
        for (int q = p.N - 2; q >= 0; --q) {
          dig[q] = rem % p.ext[q];
          rem /= p.ext[q];
        }
      }
      if (tloc >= 2) mbar_wait(&aempty[u], uint32_t(((tloc >> 1) - 1) & 1));
      fence_after_sync();
#pragma unroll
      for (int h = 0; h < KP / 32; ++h) {
        if ((h & 1) != gq) continue;  // the two warps of a quadrant split the coef columns
        float hi[32], lo[32];
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          const int r = 32 * h + rr;
          hi[rr] = (valid && r < p.R) ? p.w[r] : 0.f;
        }
        for (int q = p.N - 2; q >= 0; --q) {  // all 32 loads of a mode in flight together
          const float* fq = p.f[q] + dig[q];
          const i64 eq = p.ext[q];
          float fv[32];
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) fv[rr] = (32 * h + rr < p.R) ? __ldg(fq + i64(32 * h + rr) * eq) : 0.f;
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) hi[rr] *= fv[rr];
        }
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) lo[rr] = hi[rr] - __uint_as_float(__float_as_uint(hi[rr]) & 0xFFFFE000u);
        tmem_st32(my_lanes + G::ACOL + uint32_t(u) * 2 * KP + 32 * h, hi);
        tmem_st32(my_lanes + G::ACOL + uint32_t(u) * 2 * KP + KP + 32 * h, lo);
      }
      tmem_st_wait();
      fence_before_sync();
      mbar_arrive(&afull[u]);
    };
    const i64 mt_last = n_items > 0 ? (c1 - 1) / p.ntiles : mt0 - 1;
    if (n_items > 0) {
      form_coef(mt0);
      if (mt0 + 1 <= mt_last) form_coef(mt0 + 1);
    }
    for (int j = 1; j <= n_items; ++j) {
      if (j > 0) {
        const int jj = j - 1, pb = jj % NA;
        const int xsl = jj % SX;
        mbar_wait(&accf[pb], uint32_t((jj / NA) & 1));
        mbar_wait(&fullx[xsl], uint32_t((jj / SX) & 1));
        fence_after_sync();
        const unsigned char* xs = smem + xsl * G::X_BYTES;
        const uint32_t taddr = my_lanes + G::DCOL + uint32_t(pb) * kRBN;
        // 32 accumulator columns per TMEM load, one wait per load (not per 8 columns);
        // the X reads of the 32-column box are issued before the wait
        static_assert(kRBN == 64, "one 32-column box per epilogue warp group");
        {
          const int c32 = 32 * gq;
          uint32_t xr[32];
          tmem_ld32_nw(taddr + c32, xr);
          const unsigned char* box = xs + (c32 >> 5) * (kRBM * 128) + m * 128;
          float4 xq[8];
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) xq[ch] = *reinterpret_cast<const float4*>(box + ((ch ^ (m & 7)) << 4));
          tmem_ld_wait();
#pragma unroll
          for (int c8 = 0; c8 < 32; c8 += 8) {
            const float4 x0 = xq[c8 >> 2], x1 = xq[(c8 >> 2) + 1];
            const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
            float sr = 0.f, sx = 0.f;  // 8-term partial sums, then fp64 (same order as before)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float dd = xv[u] - __uint_as_float(xr[c8 + u]);
              sr = fmaf(dd, dd, sr);
              sx = fmaf(xv[u], xv[u], sx);
            }
            acc_r += double(sr);
            acc_x += double(sx);
          }
        }
        fence_before_sync();
        mbar_arrive(&acce[pb]);
        mbar_arrive(&emptyx[xsl]);
      }
      if (j < n_items) {
        const i64 id = c0 + j, mt = id / p.ntiles, nt = id - mt * p.ntiles;
        if (nt == 0 && mt > mt0 && mt + 1 <= mt_last) form_coef(mt + 1);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc_r += __shfl_xor_sync(0xffffffffu, acc_r, o);
      acc_x += __shfl_xor_sync(0xffffffffu, acc_x, o);
    }
    if (lane == 0) {
      red[0][warp - 2] = acc_r;
      red[1][warp - 2] = acc_x;
    }
  }
  fence_before_sync();
  __syncthreads();
  if (threadIdx.x == 0) {
    double r0 = 0.0, r1 = 0.0;
    for (int q = 0; q < 8; ++q) {
      r0 += red[0][q];
      r1 += red[1][q];
    }
    p.part[2 * blockIdx.x] = r0;
    p.part[2 * blockIdx.x + 1] = r1;
  }
  if (warp == 1) {
    fence_after_sync();
    tmem_dealloc(tmem, G::TMEM_COLS);
  }
}

// C^T hi / lo planes (E x KP, K-major, zero beyond R) from the column-major last factor
__global__ void residual_ct_kernel(const float* C, i64 E, int R, int KP, float* hi, float* lo) {
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < E * KP; e += i64(gridDim.x) * blockDim.x) {
    const i64 k = e / KP;
    const int r = int(e - k * KP);
    const float v = r < R ? C[k + i64(r) * E] : 0.f;
    hi[e] = v;
    lo[e] = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  }
}

// Blocked sketch panel: K-tile block (a, bt) holds [plane][cpad][32] with the
// 32 b values of column c contiguous (zero beyond R and cols), so one panel
// tile is a single contiguous TMA box instead of BN rows R*4 bytes apart.
// planes == 2 stores hi (raw) and lo = x - TF32(x).
__global__ void __launch_bounds__(256) panel_block_kernel(const float* __restrict__ P, i64 L, i64 R, i64 cols, i64 nbt,
                                                          i64 cpad, int planes, float* __restrict__ PB) {
  // one K-tile block per CTA iteration: one 64-bit division per block, then
  // (c, kk) = (e / 32, e % 32): 128-byte reads per column, contiguous writes
  const int per = int(cpad) * 32;
  for (i64 blk = blockIdx.x; blk < L * nbt; blk += gridDim.x) {
    const i64 a = blk / nbt, b0 = (blk - a * nbt) * kBK;
    const float* src = P + a * cols * R + b0;
    float* dst = PB + blk * planes * i64(per);
    for (int e = threadIdx.x; e < per; e += blockDim.x) {
      const int c = e >> 5, kk = e & 31;
      const float v = (c < cols && b0 + kk < R) ? __ldg(src + i64(c) * R + kk) : 0.f;
      dst[e] = v;
      if (planes == 2) dst[per + e] = lo_part(v);
    }
  }
}

int panel_block_mode() {
  static const int m = [] {
    const char* e = std::getenv("RCPG_TC_PBLK");
    return e != nullptr ? std::atoi(e) : 1;
  }();
  return m;
}

}  // namespace

// fp64 3-D tiled map over a (d0 fastest, d1, d2) view with row pitch `pitch` (0: d0), box {16, b1, 1}
// (128 B rows), SWIZZLE_128B, zero fill out of range: the DMMA sketch operands.
void tensor_map_f64_3d(void* out, const double* base, i64 d0, i64 d1, i64 d2, int b1, i64 pitch) {
  if (pitch <= 0) pitch = d0;
  static_assert(sizeof(CUtensorMap) == 128, "tensor map size");
  const cuuint64_t dims[3] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(d2)};
  const cuuint64_t strides[2] = {cuuint64_t(pitch) * 8, cuuint64_t(pitch * d1) * 8};
  const cuuint32_t box[3] = {16, cuuint32_t(b1), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_tiled()(static_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                                    const_cast<double*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaFailure("cuTensorMapEncodeTiled (f64) failed (" + std::to_string(int(r)) + ")", cudaErrorInvalidValue);
}

void tensor_map_f32_3d_sw64(void* out, const float* base, i64 d0, i64 d1, i64 d2, int b1, i64 pitch) {
  if (pitch <= 0) pitch = d0;
  const cuuint64_t dims[3] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(d2)};
  const cuuint64_t strides[2] = {cuuint64_t(pitch) * 4, cuuint64_t(pitch * d1) * 4};
  const cuuint32_t box[3] = {16, cuuint32_t(b1), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_tiled()(static_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                    const_cast<float*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaFailure("cuTensorMapEncodeTiled (f32, 64B swizzle) failed (" + std::to_string(int(r)) + ")",
                      cudaErrorInvalidValue);
}

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

// Only for streamed passes over big tensors whose panel is small next to X
// (I >= 8 cols: the copy costs <= ~25% of the pass's bytes and is re-read by
// >= 8 m-tiles). Measured (bench.py, one B200): C5 mode-0 sketch 6.24 -> 5.59 ms,
// X Z 6.20 -> 5.59 ms; C3 1.76 -> 1.72 / 3.55 -> 3.45 ms; C4 mode 0 (I = 128,
// a 1.6 GB panel) 2.3 -> 4.7 ms, hence the rule.
constexpr i64 kPanelBlockMinElems = i64(1) << 26;

bool panel_block_pays(ModeView v, i64 cols) { return v.L * v.I * v.R >= kPanelBlockMinElems && v.I >= 8 * cols; }

i64 sketch_tc_panel_floats(ModeView v, i64 cols) {
  if (panel_block_mode() == 0 || !panel_block_pays(v, cols)) return 0;
  const int bn = pick_bn_tc(cols);
  return v.L * ceil_div(v.R, kBK) * ceil_div(cols, bn) * bn * 32 * (panel_block_mode() == 2 ? 2 : 1);
}

void sketch_tc(const float* X, ModeView v, const float* P, i64 cols, float* part, float* pblk, int num_sms,
               const int* skip, cudaStream_t st) {
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
  a.cpad = a.n_ntiles * bn;
  const i64 blk_rows = v.L * a.nbt * a.cpad * 2;
  a.pblk = (pblk != nullptr && blk_rows <= kMaxCoord && panel_block_pays(v, cols)) ? panel_block_mode() : 0;
  const CUtensorMap mx = tensor_map(X, 3, xd, xs, xb);
  CUtensorMap mp;
  if (a.pblk != 0) {
    const int planes = a.pblk == 2 ? 2 : 1;
    panel_block_kernel<<<int(std::min<i64>(v.L * a.nbt, i64(num_sms) * 8)), 256, 0, st>>>(P, v.L, v.R, cols, a.nbt,
                                                                                       a.cpad, planes, pblk);
    count_launch();
    RCPG_LAUNCHED();
    const cuuint64_t pd[2] = {32, cuuint64_t(v.L * a.nbt * a.cpad * planes)};
    const cuuint64_t ps[1] = {128};
    const cuuint32_t pb[2] = {kBK, cuuint32_t(bn)};
    mp = tensor_map(pblk, 2, pd, ps, pb);
  } else {
    const cuuint64_t pd[3] = {cuuint64_t(v.R), cuuint64_t(cols), cuuint64_t(v.L)};
    const cuuint64_t ps[2] = {cuuint64_t(v.R) * 4, cuuint64_t(cols * v.R) * 4};
    const cuuint32_t pb[3] = {kBK, cuuint32_t(bn), 1};
    mp = tensor_map(P, 3, pd, ps, pb);
  }
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

bool tc_residual_ok(const i64* shape, int order, int rank) {
  // the TMA coordinates are 32-bit: the last extent E and the row index p < P
  // (the product of the leading modes) must both fit, else the SIMT residual runs
  i64 P = 1;
  for (int m = 0; m + 1 < order; ++m) P *= shape[m];
  return tc_enabled() && order >= 2 && rank <= 64 && shape[order - 1] % 4 == 0 && shape[order - 1] <= kMaxCoord &&
         P <= kMaxCoord;
}

size_t residual_tc_scratch_floats(i64 E, int rank) { return size_t(2 * E * (rank <= 32 ? 32 : 64)); }

void residual_tc(const float* X, const i64* shape, int order, const float* const* factors, const float* weights,
                 int rank, float* ct_scratch, double* part, int num_sms, int& blocks, cudaStream_t st) {
  const int KP = rank <= 32 ? 32 : 64;
  ResArgs a{};
  a.N = order;
  a.R = rank;
  a.E = shape[order - 1];
  a.P = 1;
  for (int m = 0; m < order - 1; ++m) {
    a.ext[m] = shape[m];
    a.f[m] = factors[m];
    a.P *= shape[m];
  }
  a.w = weights;
  a.mtiles = ceil_div(a.P, kRBM);
  a.ntiles = ceil_div(a.E, kRBN);
  a.items = a.mtiles * a.ntiles;
  blocks = int(std::max<i64>(1, std::min<i64>(a.items, num_sms)));
  a.chunk = ceil_div(a.items, blocks);
  blocks = int(ceil_div(a.items, a.chunk));
  a.part = part;
  float* hi = ct_scratch;
  float* lo = ct_scratch + a.E * KP;
  residual_ct_kernel<<<int(std::min<i64>(ceil_div(a.E * KP, 256), 1024)), 256, 0, st>>>(factors[order - 1], a.E,
                                                                                           rank, KP, hi, lo);
  const cuuint64_t xd[2] = {cuuint64_t(a.E), cuuint64_t(a.P)};
  const cuuint64_t xs[1] = {cuuint64_t(a.E) * 4};
  const cuuint32_t xb[2] = {32, kRBM};
  const cuuint64_t bd[2] = {cuuint64_t(KP), cuuint64_t(a.E)};
  const cuuint64_t bs[1] = {cuuint64_t(KP) * 4};
  const cuuint32_t bb[2] = {32, kRBN};
  const CUtensorMap mx = tensor_map(X, 2, xd, xs, xb);
  const CUtensorMap mh = tensor_map(hi, 2, bd, bs, bb);
  const CUtensorMap ml = tensor_map(lo, 2, bd, bs, bb);
  if (KP == 32) {
    static const size_t lim = enable_max_dyn_smem(residual_tc_kernel<32>);
    if (size_t(ResPlan<32>::SMEM) > lim) throw std::runtime_error("residual_tc: smem plan too large");
    residual_tc_kernel<32><<<blocks, kResThreads, ResPlan<32>::SMEM, st>>>(mx, mh, ml, a);
  } else {
    static const size_t lim = enable_max_dyn_smem(residual_tc_kernel<64>);
    if (size_t(ResPlan<64>::SMEM) > lim) throw std::runtime_error("residual_tc: smem plan too large");
    residual_tc_kernel<64><<<blocks, kResThreads, ResPlan<64>::SMEM, st>>>(mx, mh, ml, a);
  }
  count_launch(2);
  RCPG_LAUNCHED();
}

}  // namespace rcpg
