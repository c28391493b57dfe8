// SPDX-License-Identifier: MIT
// Tall-skinny factorizations (plu_basis / thin_qr), see factor.cu.
#pragma once

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
};

size_t factor_cand_bytes();

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
