// SPDX-License-Identifier: MIT
// Tall-skinny factorizations (plu_basis / thin_qr), see factor.cu.
#pragma once

#include "comm.cuh"
#include "common.cuh"

namespace rcpg {

constexpr int kMaxPanelCols = 256;  // widest sketch panel l = k + p supported

// Device workspace for the cooperative factorization kernels.
struct FactorWork {
  i64* keys = nullptr;        // [J_max] per-row physical / Kolda positions
  void* cands = nullptr;      // [2][max_blocks] pivot candidates
  GridBarrier* bar = nullptr;
  int* info = nullptr;        // [4]
  double* part = nullptr;     // [2][max_blocks][kMaxPanelCols + 1]
  void* tau = nullptr;        // [kMaxPanelCols] (double-sized)
  void* diag = nullptr;       // [kMaxPanelCols]
  double* cqr_work = nullptr; // [cqr_rows * kMaxPanelCols] CholeskyQR2 scratch
  i64 cqr_rows = 0;           // largest I for the single-CTA CholeskyQR2 path
  int max_blocks = 0;
  unsigned long long* prof = nullptr;  // optional phase timers (RCPG_PROFILE_LU)
  double* rowk = nullptr;     // [kMaxPanelCols] Householder: row k before its update
  bool faithful_qr = false;   // thin_qr: always the faithful Householder (no CholeskyQR2)
  unsigned* ctr = nullptr;    // [kMaxPanelCols + 1] grid LU per-step chunk counters
};

size_t factor_cand_bytes();

// ------------------------------------------------ sharded
constexpr int kDluMaxRanks = 64;

// Locates a global panel row (its Kolda index) among the slabs of the last
// mode: kmg is the unsharded Kolda map, Rg the unsharded R of the mode view.
struct SlabMap {
  KoldaMap kmg;
  i64 Rg = 1, Es = 1;
  int nranks = 1;
  i64 lo[kDluMaxRanks] = {}, hi[kDluMaxRanks] = {};
};

struct DluWork {
  i64* phys = nullptr;        // [J local]
  void* cand_loc = nullptr;   // [G] candidates
  void* cand_all = nullptr;   // [nranks][G]
  void* U = nullptr;          // [n] pivot row
  void* state = nullptr;      // dlu_state_bytes()
  int G = 0;                  // CTAs per rank (equal on all ranks)
};
size_t dlu_state_bytes();

// Row-sharded FullPivLU (P^{-1} L of the rows this rank holds); km maps the
// local rows to their global Kolda index (high_last_off set). Returns r.
template <typename T>
int plu_basis_dist(T* A, T* Z, i64 J, i64 R, int n, i64 J_global, const KoldaMap& km, const SlabMap& sm, Comm& comm,
                   const DluWork& w, cudaStream_t st);

void init_row_keys(const KoldaMap& km, i64 J, i64 R, i64* keys, cudaStream_t st);

// Z (J x r panel, r = min(J, n)) = P^{-1} L of the complete-pivoting LU of the
// J x n panel A (A is destroyed). Returns r.
template <typename T>
int plu_basis(T* A, T* Z, i64 J, i64 R, int n, const KoldaMap& km, FactorWork& w, cudaStream_t st);

// Q (J x r panel) of the Householder QR of A (destroyed); rank warning flag
// written to *rank_warning_dev when non-null. Returns r.
template <typename T>
int thin_qr(T* A, T* Q, i64 J, i64 R, int n, const KoldaMap& km, FactorWork& w, int* rank_warning_dev,
            cudaStream_t st);

}  // namespace rcpg
