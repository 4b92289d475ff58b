/*
 * rsm_b200.h -- C-ABI of the B200-native RSM (arXiv 1411.0814) hot path.
 *
 * Plain C types only (pointers, sizes, POD structs); no exceptions cross it.
 * Every entry point returns an rsm_status (0 = ok) whose values are the
 * reference's process exit codes (rsm::exit_code, include/rsm/error.hpp:38-46
 * of the reference); rsm_last_error() gives the message.
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/proj):
 *   rsm_decompose         <- rsm::decompose            include/rsm/solver.hpp:77, src/solver.cpp:119-146
 *   rsm_make_trial_params <- rsm::trial_params         include/rsm/solver.hpp:36, src/harvest.cpp:11-35
 *   rsm_select            <- attempt-order selection in harvest_gram (stage-1 parity hook)
 *                                                      src/harvest.cpp:79-120, src/sampler.cpp:27-87
 *   rsm_harvest_gram      <- rsm::harvest_gram         include/rsm/solver.hpp:53-54, src/harvest.cpp:79-120
 *   rsm_solve_v           <- rsm::solve_v              include/rsm/solver.hpp:65, src/solver.cpp:15-62
 *   rsm_solve_u           <- rsm::solve_u              include/rsm/solver.hpp:74-75, src/solver.cpp:64-89
 *   rsm_masked_residual_norm <- rsm::masked_residual_norm include/rsm/core.hpp:94, src/core.cpp:35-39
 *   rsm_generate          <- rsm::generate (observed matrix only) include/rsm/synth.hpp:29, src/synth.cpp:12-57
 *   rsm_ctx_generate      <- rsm::generate on the device (same streams; mask bit-exact, values to a few ulps)
 *   rsm_ctx_als / rsm_als <- rsm::baseline_als         include/rsm/solver.hpp:79-81, src/als.cpp:11-44
 *   rsm_load_matrix_csv   <- rsm::load_matrix          include/rsm/io.hpp:14, src/io.cpp:56-99
 *   rsm_save_matrix_csv   <- rsm::save_matrix          include/rsm/io.hpp:18, src/io.cpp:101-116
 *   rsm_dataset_checksum  <- rsm::dataset_checksum     include/rsm/io.hpp:22, src/io.cpp:140-154
 *   rsm_sample            <- rsm::sample_m1 / sample_m2 (one attempt) include/rsm/sampler.hpp:41-47,
 *                                                      src/sampler.cpp:12-87
 *   rsm_small_singular_vectors <- rsm::small_singular_vectors include/rsm/spectra.hpp:61,
 *                                                      src/spectra.cpp:48-86
 *   rsm_gram_update       <- GramAccumulator::accumulate / accumulate_dense / merge
 *                                                      include/rsm/spectra.hpp:36-43, src/spectra.cpp:7-46
 *   rsm_masked_objective  <- rsm::masked_objective     include/rsm/core.hpp:95, src/core.cpp:41-44
 *
 * Host buffers are caller-owned; device memory is owned by the context.
 * Calls are synchronous on return, one host thread per context. Matrices
 * are row-major FP64 with NaN (ignored) at hidden cells plus a uint8 mask,
 * exactly rsm::MaskedMatrix (include/rsm/core.hpp:22-57).
 */
#ifndef RSM_B200_H
#define RSM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t rsm_status;
#define RSM_OK 0
#define RSM_ERR_INTERNAL 1              /* errc::internal (also CUDA/NCCL failures) */
#define RSM_ERR_INVALID_CONFIG 2        /* errc::invalid_config */
#define RSM_ERR_PARSE_IO 3              /* errc::parse_io */
#define RSM_ERR_INSUFFICIENT_COVERAGE 4 /* errc::insufficient_coverage */

#define RSM_MODE_M1 0 /* column branch (rsm::Mode::M1) */
#define RSM_MODE_M2 1 /* row branch    (rsm::Mode::M2) */

/* rsm::RsmConfig (include/rsm/solver.hpp:13-23) with TrialPlan flattened
 * (include/rsm/planner.hpp:12-18): trials + epsilon are what decompose uses. */
typedef struct {
  int64_t rank;
  int32_t mode;
  int64_t block;
  int64_t vectors_per_trial;
  uint64_t trials;
  double epsilon;
  uint64_t seed;
  double gram_rank_tol;
  int64_t min_dim;
  int32_t workers; /* accepted and ignored: results never depend on it */
} rsm_config;

/* rsm::TrialParams (include/rsm/solver.hpp:27-34) */
typedef struct {
  int32_t mode;
  int64_t block;
  int64_t ell;
  int64_t rank;
  int64_t min_count;
  uint64_t seed;
} rsm_trial_params;

/* rsm::DecompositionReport (include/rsm/core.hpp:81-90) */
typedef struct {
  double e;
  uint64_t trials_attempted;
  uint64_t trials_accepted;
  uint64_t z;
  int64_t underdetermined_rows;
  int64_t gram_rank;
  int32_t borderline_rank_gate;
  double wall_time;
} rsm_report;

typedef struct rsm_ctx rsm_ctx;

/* Fills cfg with the reference defaults (RsmConfig{} + TrialPlan{}). */
void rsm_config_default(rsm_config* cfg);

/* Message of the last failing call on ctx (or of the last context-free call
 * when ctx is NULL). Valid until the next call on the same context. */
const char* rsm_last_error(const rsm_ctx* ctx);

/* ---------------------------------------------------------------- context */
/* world/rank/nccl_id: world==1 for a single GPU (nccl_id ignored). For
 * world>1, nccl_id points to the 128-byte ncclUniqueId produced by
 * rsm_nccl_unique_id on rank 0 and broadcast by the caller. */
rsm_status rsm_ctx_create(rsm_ctx** out, int device, int world, int rank, const void* nccl_id);
rsm_status rsm_ctx_destroy(rsm_ctx* ctx);
rsm_status rsm_nccl_unique_id(void* out128);

/* In-process rank group whose collectives go through host memory instead of
 * NCCL (test / diagnostic hook): `world` contexts, possibly on one GPU, each
 * driven by its own host thread, take the multi-rank code path -- trial
 * shards, the accumulator and column-count all-reduce, row shards and the U
 * all-gather -- with sums formed in rank order on every rank. */
typedef struct rsm_host_group rsm_host_group;
rsm_status rsm_host_group_create(int world, rsm_host_group** out);
rsm_status rsm_host_group_destroy(rsm_host_group* g);
rsm_status rsm_ctx_create_host_group(rsm_ctx** out, int device, rsm_host_group* g, int rank);
/* Work split across ranks (host-only, no device): rank owns [lo, hi) of
 * total units -- accepted trials in stage 2-3, rows in stage 5. */
void rsm_shard_range(int64_t total, int world, int rank, int64_t* lo, int64_t* hi);
/* cudaStream_t the context launches on (for event timing by callers). */
void* rsm_ctx_stream(rsm_ctx* ctx);

/* Upload a masked matrix (host buffers) into the context: H2D copy, device
 * bit-packing of the mask, device transpose when m < n. */
rsm_status rsm_ctx_load(rsm_ctx* ctx, const double* values, const uint8_t* mask, int64_t m,
                        int64_t n);
/* Same from device buffers already resident in HBM (no H2D). */
rsm_status rsm_ctx_load_device(rsm_ctx* ctx, const double* d_values, const uint8_t* d_mask,
                               int64_t m, int64_t n);

/* Generate the reference's synthetic instance (rsm::generate, src/synth.cpp:12-57;
 * same streams as rsm_generate below) directly on the device and load it into
 * the context (no host buffers, no H2D). The mask is bit-exact with
 * rsm_generate; values agree to a few ulps (device log/cos in Box-Muller). */
rsm_status rsm_ctx_generate(rsm_ctx* ctx, int64_t m, int64_t n, int64_t r, double rho, double sigma,
                            uint64_t seed);
/* Copy the loaded matrix back: values (m x n FP64, NaN where hidden) and the
 * bit-packed row mask (m x nwp u32, bit j%32 of word j/32; nwp written to
 * *nwp); either buffer may be NULL. */
rsm_status rsm_ctx_fetch_matrix(rsm_ctx* ctx, double* values, uint32_t* words, int64_t* nwp);

/* decompose on the loaded matrix. U (m x r) and V (n x r) row-major host
 * buffers may be NULL to leave the factors on the device
 * (rsm_ctx_fetch_factors copies them later). */
rsm_status rsm_ctx_decompose(rsm_ctx* ctx, const rsm_config* cfg, double* U, double* V,
                             rsm_report* rep);
rsm_status rsm_ctx_fetch_factors(rsm_ctx* ctx, double* U, double* V);

/* Alternating masked least squares baseline on the loaded matrix; replaces
 * rsm::baseline_als (include/rsm/solver.hpp:79-81, src/als.cpp:11-44):
 * V from Rng(seed, ALS_INIT=6, column).next_normal(), `iterations` rounds of
 * U = rows(M; V), V = rows(M^T; U), then U = rows(M; V). The report carries
 * e, underdetermined_rows (last U step) and wall_time. */
rsm_status rsm_ctx_als(rsm_ctx* ctx, int64_t r, int64_t iterations, uint64_t seed, double* U, double* V,
                       rsm_report* rep);

/* Stage entry points on the loaded matrix, for the oriented problem
 * (m >= n as loaded; call these only for the matrix as given). */
rsm_status rsm_ctx_select(rsm_ctx* ctx, const rsm_trial_params* p, uint64_t trials,
                          uint64_t* accepted_attempts /* trials or NULL */,
                          int64_t* survivors /* trials or NULL */, uint64_t* attempted,
                          uint64_t* accepted);
rsm_status rsm_ctx_harvest_gram(rsm_ctx* ctx, const rsm_trial_params* p, uint64_t trials,
                                double* G /* n*n or NULL */, uint64_t* attempted,
                                uint64_t* accepted, uint64_t* z);
/* G == NULL uses the accumulator left on the device by the last harvest. */
rsm_status rsm_ctx_solve_v(rsm_ctx* ctx, const double* G, int64_t n, int64_t r, double tol,
                           double* V /* n*r */, int64_t* gram_rank, int32_t* borderline,
                           double* w_small /* r+1 smallest eigenvalues or NULL */);
/* V == NULL uses the basis left on the device by the last solve_v. */
rsm_status rsm_ctx_solve_u(rsm_ctx* ctx, const double* V, int64_t r, double* U /* m*r or NULL */,
                           int64_t* underdetermined_rows, double* sum_sq_resid);

/* Per-stage device time (ms) of the last decompose, CUDA events on the
 * context stream: [0] select, [1] svd, [2] gram, [3] gram-reduce,
 * [4] solve_v, [5] solve_u, [6] total. Returns the number written. */
int rsm_ctx_stage_ms(rsm_ctx* ctx, double* ms, int cap);
/* Kernel launches issued by the last decompose. */
int64_t rsm_ctx_launch_count(rsm_ctx* ctx);
/* Decompositions on this context that were re-run because the speculative
 * selection (one chunk enqueued ahead of stages 2-5) did not
 * reach the trial count or saw a support longer than stage 2 was sized for
 * (diagnostic; the results are those of the re-run). */
int64_t rsm_ctx_rerun_count(rsm_ctx* ctx);
/* Bytes the last rsm_ctx_load copied host -> device: the values plus the
 * mask bit-packed on the host (rsm_ctx_load_device: 0). */
int64_t rsm_ctx_last_load_h2d_bytes(rsm_ctx* ctx);
/* Stage-4 eigensolver diagnostics of the last solve_v: [0] outer iterations,
 * [1] matvecs, [2] lambda_max, [3] spectrum upper bound, [4] max residual of
 * the wanted Ritz pairs, [5] block size, [6] cooperative grid, [7..] phase
 * clocks (cycles, CTA 0). */
int rsm_ctx_solver_stats(rsm_ctx* ctx, double* out, int cap);

/* --------------------------------------------------------- one-shot API */
/* Reference-shaped calls on host buffers (use a per-device default context). */
rsm_status rsm_make_trial_params(const rsm_config* cfg, int64_t m, int64_t n, rsm_trial_params* out);
rsm_status rsm_decompose(const double* values, const uint8_t* mask, int64_t m, int64_t n,
                         const rsm_config* cfg, double* U, double* V, rsm_report* rep);
rsm_status rsm_als(const double* values, const uint8_t* mask, int64_t m, int64_t n, int64_t r,
                   int64_t iterations, uint64_t seed, double* U, double* V, rsm_report* rep);
rsm_status rsm_harvest_gram(const double* values, const uint8_t* mask, int64_t m, int64_t n,
                            const rsm_trial_params* p, uint64_t trials, double* G,
                            uint64_t* attempted, uint64_t* accepted, uint64_t* z);
/* Minor eigenvectors (solver.cpp:15-62) by Chebyshev-filtered subspace
 * iteration, not the full dsyev spectrum: the rank-gate threshold uses a
 * power-iteration estimate of lambda_max (a lower bound after >= 8 matvecs),
 * so gram_rank and borderline can differ from the reference only for an
 * eigenvalue within that estimate's error of tol * lambda_max. */
rsm_status rsm_solve_v(const double* G, int64_t n, int64_t r, double tol, double* V,
                       int64_t* gram_rank, int32_t* borderline);
/* Row solves (solver.cpp:64-89). Deviation from the reference's COD: a row's
 * rank is decided on its r x r normal matrix (Cholesky pivot <= 1e-10 of the
 * largest diagonal -> eigen-decomposition pseudo-inverse, rank = eigenvalues
 * above 64 eps of the largest) instead of Eigen's column-pivoted QR of the
 * gathered basis rows. Exactly deficient rows (fewer than r observations, a
 * rank-deficient V_O) are flagged and solved at minimum norm as the
 * reference does; rows with cond(V_O) between ~1e5 and ~1e15 can be
 * classified differently. */
rsm_status rsm_solve_u(const double* values, const uint8_t* mask, int64_t m, int64_t n,
                       const double* V, int64_t r, double* U, int64_t* underdetermined_rows);
rsm_status rsm_masked_residual_norm(const double* values, const uint8_t* mask, int64_t m,
                                    int64_t n, const double* U, const double* V, int64_t r,
                                    double* e);

/* -------------------------------------------- per-call building blocks */
/* The reference's single-trial and accumulator functions, one call at a time
 * on the device (the decomposition above never calls them; they serve the
 * drop-in header's attempt_trial / sample_m* / GramAccumulator surface).
 *
 * rsm_sample: attempt `trial_index` of the TRIAL stream draws `count` indices
 * (mode 1 = M2: rows of the m x n matrix; mode 0 = M1: columns), sorted
 * (drawn[count], bit-exact with the reference), and keeps every column (M2) /
 * row (M1) observed on all of them, ascending, in kept[] (capacity n for M2,
 * m for M1), *nkept of them. count <= 16 on the device. */
rsm_status rsm_sample(const double* values, const uint8_t* mask, int64_t m, int64_t n, int32_t mode,
                      int64_t count, uint64_t seed, uint64_t trial_index, int64_t* drawn, int64_t* kept,
                      int64_t* nkept);
/* rsm::small_singular_vectors: the ell right singular vectors of the p x q
 * row-major S with the smallest singular values, ascending, each sign-fixed
 * (largest-magnitude entry positive); zeta is ell x q, sv the singular values
 * (0 for vectors past the rank). The reference's validation and messages;
 * on the device min(p, q) <= 32. Vectors of a repeated (e.g. zero) singular
 * value are a basis of its space, as any SVD's are. */
rsm_status rsm_small_singular_vectors(const double* S, int64_t p, int64_t q, int64_t r, int64_t ell,
                                      double* zeta, double* sv);
/* G (n x n, host, in/out) += sum_v x_v x_v^T over the nvec dense rows of X
 * (nvec x n; may be NULL when nvec = 0), then += G2 when G2 is not NULL:
 * per element in vector order with separate multiply and add, bit-identical
 * to GramAccumulator::accumulate/accumulate_dense followed by merge. */
rsm_status rsm_gram_update(double* G, int64_t n, const double* X, int64_t nvec, const double* G2);
/* rsm::masked_objective: norm 0 = Frobenius (sqrt of the observed squared
 * residual); any other norm fails with the reference's invalid_config. */
rsm_status rsm_masked_objective(const double* values, const uint8_t* mask, int64_t m, int64_t n,
                                const double* U, const double* V, int64_t r, int32_t norm, double* out);

/* FP64 DFMA throughput of the device (TFLOP/s), the roofline denominator of
 * the FP64-bound stages (not in MEASURED_PEAKS.json). */
rsm_status rsm_fp64_peak_tflops(int device, double* tflops);
/* FP64 tensor-core (DMMA m8n8k4) throughput of the device (TFLOP/s). */
rsm_status rsm_dmma_peak_tflops(int device, double* tflops);

/* Host input generator (reference synth streams, observed matrix only),
 * rows [row0, row0+rows) of an m x n instance; multithreaded. */
rsm_status rsm_generate(int64_t m, int64_t n, int64_t r, double rho, double sigma, uint64_t seed,
                        int64_t row0, int64_t rows, double* values, uint8_t* mask);

/* Structured-missingness generator (BASELINE config 5; no reference
 * counterpart): affine-camera tracks, points x (2 frames)
 * columns, rank 4, each point visible over one contiguous frame window of
 * length uniform in [wmin, wmax]; rows [row0, row0+rows). The streams are
 * documented in src synth.cpp and DESIGN.md. */
rsm_status rsm_generate_tracks(int64_t points, int64_t frames, int64_t wmin, int64_t wmax, double sigma,
                               uint64_t seed, int64_t row0, int64_t rows, double* values, uint8_t* mask);

/* ------------------------------------------------------------- loader */
/* NaN-CSV masked matrix (rsm::load_matrix, io.cpp:56-99): one row per line,
 * empty or "nan" (any case) cells hidden. *values (m x n, NaN at hidden
 * cells) and *mask (m x n) are malloc'd by the library; release them with
 * rsm_free. Parse failures return RSM_ERR_PARSE_IO with the reference's
 * messages. */
rsm_status rsm_load_matrix_csv(const char* path, double** values, uint8_t** mask, int64_t* m, int64_t* n);
/* rsm::save_matrix (io.cpp:101-116): hidden cells as NaN, %.17g values. */
rsm_status rsm_save_matrix_csv(const char* path, const double* values, const uint8_t* mask, int64_t m,
                               int64_t n);
/* rsm::dataset_checksum (io.cpp:140-154): FNV-1a over dims, mask, values. */
rsm_status rsm_dataset_checksum(const double* values, const uint8_t* mask, int64_t m, int64_t n,
                                uint64_t* out);
void rsm_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
