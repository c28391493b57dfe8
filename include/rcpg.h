/* SPDX-License-Identifier: MIT
 *
 * rcpg — C ABI of the B200-native randomized CP (rCP) hot path.
 *
 * Drop-in boundary for the reference's C++ entry points:
 *   rcp::decompose      /root/reference/proj/include/rcp/solve.hpp:381-398
 *   rcp::compress       /root/reference/proj/include/rcp/compress.hpp:86-146
 *   rcp::als_solve      /root/reference/proj/include/rcp/solve.hpp:183-262
 *   rcp::recover        /root/reference/proj/include/rcp/kruskal.hpp:198-220
 *   rcp::relative_error /root/reference/proj/include/rcp/kruskal.hpp:187-194
 * Plain pointers and sizes only; no exceptions cross this boundary (errors
 * are status codes, SURVEY.md §8(b) "Status codes"). Everything computes on
 * the GPU; there is no CPU fallback — without a CUDA device every compute
 * entry point returns RCPG_CUDA_ERROR.
 *
 * Conventions
 *   - Tensors are dense, row-major (last index fastest), exactly the
 *     reference's Tensor storage (tensor.hpp:14-18).
 *   - Matrices (bases Q_n, factors) are column-major, like the reference's
 *     Eigen matrices (types.hpp:16-23).
 *   - dtype: RCPG_F32 / RCPG_F64 (the reference's Scalar = float / double).
 *   - One context per host thread; calls are synchronous from the caller's
 *     point of view.
 */
#ifndef RCPG_H
#define RCPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RCPG_OK = 0,
  RCPG_INVALID_ARGUMENT = 1, /* -> std::invalid_argument (types.hpp:30-32)            */
  RCPG_SOLVER_ERROR = 2,     /* -> rcp::SolverError (solve.hpp:48-57); see           */
                             /*    rcpg_last_error_iteration()                        */
  RCPG_CUDA_ERROR = 3,       /* -> std::runtime_error                                 */
  RCPG_OOM = 4,              /* -> std::bad_alloc / runtime_error                     */
  RCPG_NCCL_ERROR = 5        /* -> std::runtime_error                                 */
} rcpg_status;

typedef enum { RCPG_F32 = 0, RCPG_F64 = 1 } rcpg_dtype;

/* rcp::RandomDistribution (compress.hpp:16) */
typedef enum { RCPG_GAUSSIAN = 0, RCPG_UNIFORM = 1 } rcpg_distribution;
/* rcp::PowerStabilizer (compress.hpp:21) */
typedef enum { RCPG_STAB_LU = 0, RCPG_STAB_QR = 1 } rcpg_stabilizer;
/* rcp::SolveMethod / rcp::InitMethod (solve.hpp:19-20) */
typedef enum { RCPG_ALS = 0, RCPG_BCD = 1 } rcpg_method;
typedef enum { RCPG_INIT_EIGENVECTORS = 0, RCPG_INIT_RANDOM = 1 } rcpg_init;

/* Mirror of rcp::CompressConfig (compress.hpp:23-33). `modes` keeps the
 * reference's three states: modes_present = 0 -> disengaged (all modes);
 * modes_present = 1 -> use modes[0..n_modes) (n_modes may be 0 = none). */
typedef struct {
  int64_t target_rank;      /* k; 0 inherits the CP rank inside decompose   */
  int64_t oversampling;     /* p (default 10)                               */
  int32_t power_iterations; /* q (default 2)                                */
  int32_t distribution;     /* rcpg_distribution                            */
  int32_t stabilizer;       /* rcpg_stabilizer                              */
  int32_t modes_present;
  int64_t n_modes;
  const int64_t* modes;     /* 0-based mode indices                         */
  uint64_t seed;            /* Omega stream seed (compress.hpp:32)          */
} rcpg_compress_config;

/* Mirror of rcp::DecomposeConfig (solve.hpp:22-31). */
typedef struct {
  int64_t rank;
  int32_t method;     /* rcpg_method; only RCPG_ALS is on this path      */
  int32_t randomized; /* bool                                            */
  rcpg_compress_config compress;
  double tol;         /* default 1e-5                                    */
  int32_t max_iter;   /* default 500                                     */
  int32_t init;       /* rcpg_init                                       */
  uint64_t seed;      /* initialization stream                           */
} rcpg_decompose_config;

/* Caller-owned result buffers for rcpg_decompose (rcp::Kruskal + FitTrace,
 * kruskal.hpp:16-30, solve.hpp:35-45). Output pointers may be NULL. */
typedef struct {
  void* weights;             /* [rank], dtype of the tensor                      */
  void* factors;             /* sum_n I_n x rank, column-major, concatenated     */
  int32_t* trace_iteration;  /* [trace_capacity]                                 */
  double* trace_fit;         /* [trace_capacity]                                 */
  double* trace_seconds;     /* [trace_capacity] seconds since solver start      */
  int32_t trace_capacity;    /* entries written = min(iterations, capacity)     */
  int32_t iterations;        /* out: FitTrace::iterations                       */
  int32_t converged;         /* out: FitTrace::converged                        */
  double final_relative_error; /* out: FitTrace::final_relative_error          */
} rcpg_result;

typedef struct rcpg_context rcpg_context;
typedef struct rcpg_tensor rcpg_tensor;
typedef struct rcpg_compressed rcpg_compressed;

/* ---- context ----------------------------------------------------------- */
rcpg_status rcpg_create(int device, rcpg_context** out);
void rcpg_destroy(rcpg_context* ctx);
const char* rcpg_last_error(const rcpg_context* ctx);
int32_t rcpg_last_error_iteration(const rcpg_context* ctx); /* SolverError::iteration() */
const char* rcpg_version(void);

/* ---- device tensors (rcp::Tensor, tensor.hpp:19-108) ------------------- */
/* Copies a row-major host tensor to HBM (rcp::Tensor constructor). */
rcpg_status rcpg_tensor_upload(rcpg_context* ctx, rcpg_dtype dtype, int32_t order,
                               const int64_t* shape, const void* host, rcpg_tensor** out);
/* Borrows an existing device allocation (no copy; caller keeps ownership). */
rcpg_status rcpg_tensor_wrap_device(rcpg_context* ctx, rcpg_dtype dtype, int32_t order,
                                    const int64_t* shape, void* device_ptr, rcpg_tensor** out);
rcpg_status rcpg_tensor_download(rcpg_context* ctx, const rcpg_tensor* t, void* host);
void* rcpg_tensor_device_ptr(const rcpg_tensor* t);
void rcpg_tensor_free(rcpg_tensor* t);

/* ---- compress (compress.hpp:86-146) ------------------------------------ */
rcpg_status rcpg_compress(rcpg_context* ctx, const rcpg_tensor* t, const rcpg_compress_config* cfg,
                          rcpg_compressed** out);
int32_t rcpg_compressed_order(const rcpg_compressed* c);
void rcpg_compressed_shape(const rcpg_compressed* c, int64_t* shape);
/* Compressed tensor, row-major, to host. */
rcpg_status rcpg_compressed_download(rcpg_context* ctx, const rcpg_compressed* c, void* host);
/* ModeBasis (types.hpp:60-76): identity flag, dim, number of columns
 * (0 for identity), rank_warning; Q copied column-major (dim x cols). */
void rcpg_compressed_basis_info(const rcpg_compressed* c, int32_t mode, int32_t* identity, int64_t* dim,
                                int64_t* cols, int32_t* rank_warning);
rcpg_status rcpg_compressed_basis_download(rcpg_context* ctx, const rcpg_compressed* c, int32_t mode,
                                           void* host);
void rcpg_compressed_free(rcpg_compressed* c);

/* ---- decompose (solve.hpp:381-398) ------------------------------------- */
rcpg_status rcpg_decompose(rcpg_context* ctx, const rcpg_tensor* t, const rcpg_decompose_config* cfg,
                           rcpg_result* result);
/* Convenience: host tensor in, host result out (upload inside the call). */
rcpg_status rcpg_decompose_host(rcpg_context* ctx, rcpg_dtype dtype, int32_t order, const int64_t* shape,
                                const void* host, const rcpg_decompose_config* cfg, rcpg_result* result);

/* ---- sharding across GPUs (no counterpart in the serial
 * reference) ------------------------------------------------------------------
 * One context per GPU / rank. A tensor split in slabs along its LAST mode (or,
 * with the *_mode variants, its FIRST mode) is decomposed with the same
 * rcpg_decompose / rcpg_compress calls on every rank (collectively); results
 * (model, trace, compressed tensor) are replicated. */
/* 128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it). */
rcpg_status rcpg_comm_unique_id(void* out128);
/* Join an NCCL communicator of nranks ranks (one per GPU, one process each). */
rcpg_status rcpg_comm_init_nccl(rcpg_context* ctx, int32_t nranks, int32_t rank, const void* id128);
/* Virtual ranks inside one process (ctxs[r] is rank r; one host thread each,
 * any devices, including one shared GPU): tests the sharded path on one GPU. */
rcpg_status rcpg_comm_init_loopback(rcpg_context** ctxs, int32_t n);
rcpg_status rcpg_comm_rank(rcpg_context* ctx, int32_t* rank, int32_t* size);
/* The balanced contiguous split [lo, hi) of [0, extent) used for slabs (host only). */
void rcpg_slab_range(int64_t extent, int32_t nranks, int32_t rank, int64_t* lo, int64_t* hi);
/* Slab [lo, hi) of mode `mode` (0 or order-1) of a device tensor (copied; `full` unchanged). */
rcpg_status rcpg_tensor_slab_mode(rcpg_context* ctx, const rcpg_tensor* full, int32_t mode, int64_t lo, int64_t hi,
                                  rcpg_tensor** out);
/* Slab [lo, hi) of the last mode of a device tensor (copied; `full` unchanged). */
rcpg_status rcpg_tensor_slab(rcpg_context* ctx, const rcpg_tensor* full, int64_t lo, int64_t hi, rcpg_tensor** out);
/* Slab from host: global_shape of the whole tensor, host_slab row-major with
 * last extent hi - lo. */
rcpg_status rcpg_tensor_upload_slab(rcpg_context* ctx, rcpg_dtype dtype, int32_t order, const int64_t* global_shape,
                                    int64_t lo, int64_t hi, const void* host_slab, rcpg_tensor** out);
/* Slab of mode `mode` from host: host_slab row-major with extent hi - lo in that mode. */
rcpg_status rcpg_tensor_upload_slab_mode(rcpg_context* ctx, rcpg_dtype dtype, int32_t order,
                                         const int64_t* global_shape, int32_t mode, int64_t lo, int64_t hi,
                                         const void* host_slab, rcpg_tensor** out);

/* ---- model utilities on device ------------------------------------------ */
/* relative_error (kruskal.hpp:187-194) of a Kruskal model (weights [R],
 * factors column-major concatenated, host pointers) against a device tensor;
 * accumulated in double. */
rcpg_status rcpg_relative_error(rcpg_context* ctx, const rcpg_tensor* t, int64_t rank, const void* weights,
                                const void* factors, double* out);

/* recover (kruskal.hpp:198-220): the full-space model of a model fitted on the
 * compressed tensor. Inputs: order, rank R, the compressed extents, the small
 * model (weights [R], factors column-major concatenated, extent_m x R each) and
 * the bases as rcpg_projection_residual_bases takes them plus their row counts
 * `dims` (identity: the factor is copied, dims[m] must equal its extent; else
 * Q_m is dims[m] x cols[m] with cols[m] = the compressed extent). A_m = Q_m A~_m,
 * then normalize (kruskal.hpp:117-176). Outputs: weights [R] and the factors
 * (dims[m] x R, concatenated). Errors as the reference: INVALID_ARGUMENT with
 * "recover: ..." messages. */
rcpg_status rcpg_recover(rcpg_context* ctx, rcpg_dtype dtype, int32_t order, int64_t rank,
                         const int64_t* small_extents, const void* weights, const void* factors,
                         const int32_t* identity, const int64_t* dims, const int64_t* cols, const void* q_concat,
                         void* out_weights, void* out_factors);

/* als_solve (solve.hpp:183-262): CP-ALS on the tensor itself (no compression;
 * cfg->method and cfg->randomized are ignored), with the fit trace and the
 * final relative error of the returned model. */
rcpg_status rcpg_als_solve(rcpg_context* ctx, const rcpg_tensor* t, const rcpg_decompose_config* cfg,
                           rcpg_result* res);

/* ---- bound validation (compress.hpp:148-164, diagnostics.hpp:36-86) ---- */
/* projection_residual: ||t - t x_n Q_n Q_n^T ...||_F over the compressed modes of
 * `c` (the result of rcpg_compress on t); fp64 accumulation. */
rcpg_status rcpg_projection_residual(rcpg_context* ctx, const rcpg_tensor* t, const rcpg_compressed* c, double* out);
/* The same with host bases (rcp::CompressionResult): per mode identity flag and column
 * count, the non-identity Q_n (dim x cols, column-major) concatenated in mode order. */
rcpg_status rcpg_projection_residual_bases(rcpg_context* ctx, const rcpg_tensor* t, const int32_t* identity,
                                          const int64_t* cols, const void* q_concat, double* out);
/* theorem_bound: per-mode tail energies sum_{j >= k} sigma_j^2 of every unfolding
 * (tail_energies[order]) and bound = sqrt(1 + k/(p-1)) sqrt(sum of tails);
 * k >= 2, p >= 2, k < every extent <= 2048. (validate_bound = this plus `trials`
 * rcpg_compress(q = 0) / rcpg_projection_residual calls with the trial seeds;
 * see include/rcp_b200/rcp.hpp.) */
rcpg_status rcpg_theorem_bound(rcpg_context* ctx, const rcpg_tensor* t, int64_t k, int64_t p, double* tail_energies,
                               double* bound);

/* ---- diagnostics (not on the reference API; used by tests/bench) -------- */
/* Materializes Omega_n (rows x cols, column-major) exactly as compress.hpp:118-124
 * draws it, on the device, and copies it to host. */
rcpg_status rcpg_sketch_matrix(rcpg_context* ctx, rcpg_dtype dtype, uint64_t seed, int64_t mode,
                               int64_t rows, int64_t cols, int32_t distribution, void* host);
/* One streamed mode-n pass on host inputs (mode view L x I x R of a row-major
 * tensor, x[(a*I + i)*R + b]):
 *   kind 0, sketch:     out[c*I + i]     = sum_{a,b} x[a,i,b] p[(a*cols + c)*R + b]
 *   kind 1, projection: out[(a*cols + c)*R + b] = sum_i x[a,i,b] p[i + c*I]
 * (the X_(n) Omega / X_(n)^T Q / Q^T X_(n) products of compress.hpp:118-145). */
rcpg_status rcpg_stream_pass(rcpg_context* ctx, rcpg_dtype dtype, int32_t kind, int64_t L, int64_t I, int64_t R,
                             int64_t cols, const void* x, const void* p, void* out);
/* plu_basis / thin_qr (compress.hpp:47-73) of a host column-major matrix, on device. */
rcpg_status rcpg_plu_basis(rcpg_context* ctx, rcpg_dtype dtype, int64_t rows, int64_t cols, const void* in,
                           void* out);
rcpg_status rcpg_thin_qr(rcpg_context* ctx, rcpg_dtype dtype, int64_t rows, int64_t cols, const void* in,
                         void* out, int32_t* rank_warning);
/* Per-pass device timings (CUDA events) of the last compress/decompose call.
 * names: NUL-separated list in `names` (capacity names_cap); returns count. */
int32_t rcpg_pass_timings(const rcpg_context* ctx, char* names, int32_t names_cap, double* ms,
                          double* bytes, int32_t cap);
/* Start of each pass of the last call, ms after the first pass started (same
 * order as rcpg_pass_timings); gaps between passes are device idle time. */
int32_t rcpg_pass_offsets(const rcpg_context* ctx, double* start_ms, int32_t cap);
/* Number of kernels the library launched since context creation. */
int64_t rcpg_kernel_launches(const rcpg_context* ctx);
/* Synthetic test-data generator on device (not the hot path): dense
 * reconstruction of a Kruskal model given on the host (weights [R] and
 * column-major factors, double) plus add_noise (synthetic.hpp:42-58) with
 * amplitude SNR `snr` (<= 0: no noise) drawn from stream (noise_seed, noise)
 * by the counter form of the reference's sequential Box-Muller stream. */
rcpg_status rcpg_synth(rcpg_context* ctx, rcpg_dtype dtype, int32_t order, const int64_t* shape, int64_t rank,
                       const double* weights, const double* factors, double snr, uint64_t noise_seed,
                       rcpg_tensor** out);
rcpg_status rcpg_synchronize(rcpg_context* ctx);
/* Context options (no counterpart in the reference; defaults keep its semantics):
 *   "fp32_arith"  0 (default): fp32 tensors run every GEMM with fp32 operands and
 *                 fp64 products/sums rounded once to float (the oracle's
 *                 double-accumulated GEMMs), factorizations in the reference's
 *                 float operation order; 1: 3xTF32 tcgen05 passes (fast, ~1e-7
 *                 relative per pass, not bit-faithful). Env RCPG_FP32=fast sets 1.
 *   "omega_host"  0 (default): Omega on the device (CUDA libm, a few ulp from
 *                 glibc on ~0.1% of draws); 1: Omega evaluated on the host with
 *                 the reference's std::log/sin/cos and uploaded (bit-identical).
 *   "pass_timing" 0 (default): no instrumentation; 1: a CUDA event pair around
 *                 every pass of a decomposition, read with rcpg_pass_timings
 *                 (~60 event records per call: C2 3.8 -> 4.1 ms). */
rcpg_status rcpg_set_option(rcpg_context* ctx, const char* name, int64_t value);
rcpg_status rcpg_get_option(const rcpg_context* ctx, const char* name, int64_t* value);
/* Device time (CUDA events) of plu_basis (kind 0) / thin_qr (kind 1) on a
 * rows x cols device-resident panel, averaged over reps calls. */
rcpg_status rcpg_bench_factor(rcpg_context* ctx, rcpg_dtype dtype, int32_t kind, int64_t rows, int64_t cols,
                              int32_t reps, double* ms_per_call);
/* CUDA events on the library's stream (device timing of whole calls):
 * record into slot [0, 64); elapsed milliseconds between two recorded slots. */
rcpg_status rcpg_event_record(rcpg_context* ctx, int32_t slot);
rcpg_status rcpg_event_elapsed(rcpg_context* ctx, int32_t slot_a, int32_t slot_b, double* ms);
/* Page-lock / unlock a host buffer for asynchronous H2D/D2H (e2e timing). */
rcpg_status rcpg_host_register(rcpg_context* ctx, void* ptr, size_t bytes);
rcpg_status rcpg_host_unregister(rcpg_context* ctx, void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* RCPG_H */
