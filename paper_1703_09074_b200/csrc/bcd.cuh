// SPDX-License-Identifier: MIT
// Block coordinate descent (bcd_solve, solve.hpp:264-376) on a device tensor.
#pragma once

#include "als.cuh"

namespace rcpg {

// Whether the one-launch BCD kernel handles these extents (every extent <= 12288
// and the per-component columns fit in shared memory).
bool bcd_supported(const i64* shape, int order, int rank);

// The whole bcd_solve in one cooperative launch, after init_factors (factors in
// fs, mode 0 zero) and als_start (state). res / loo: S elements each. part:
// >= 2 * num_sms * (max extent + 1) doubles. The trace (one entry per inner
// iteration, solve.hpp:320-321), iterations (state->it - 1), converged and the
// error iteration land in the state / trace arrays like the ALS loop's.
template <typename T>
void bcd_solve(const T* X, T* res, T* loo, const i64* shape, int order, const FactorSet<T>& fs, T* weights,
               double tol, int max_iter, double* trace_fit, double* trace_sec, AlsState* state, double* part,
               i64 part_elems, GridBarrier* bar, cudaStream_t st);

}  // namespace rcpg
