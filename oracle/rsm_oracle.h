/*
 * rsm_oracle.h -- CPU restatement of the reference RSM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the B200 product
 * (paper_1411_0814_b200/). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. Nothing in the product
 * path links or calls this code.
 *
 * Every function restates the reference algorithm (paths relative to
 * /root/reference/proj) in plain C, literally: the Gram accumulator sums the
 * harvested singular vectors one by one in attempt order exactly like
 * src/harvest.cpp:110-117 + src/spectra.cpp:7-23, it does NOT use the
 * rank-r identity the GPU uses, so agreement is a real cross-check.
 *
 * Pinning: stage-1 selection is pinned bit-exactly against the reference's own
 * compiled sampler/harvest code (oracle/_ref, see oracle/Makefile); stages 2-5
 * are pinned against the reference's tests/properties and against oracle/_ref
 * (reference solver.cpp/spectra.cpp compiled with builder-written Eigen and
 * LAPACKE shims), see tests/test_oracle_pin.py.
 */
#ifndef RSM_ORACLE_H
#define RSM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror include/rsm_b200.h and rsm::exit_code (include/rsm/error.hpp:38-46) */
#define ORC_OK 0
#define ORC_INTERNAL 1
#define ORC_INVALID 2
#define ORC_COVERAGE 4

typedef struct {
  int32_t mode;      /* 0 = M1 (column branch), 1 = M2 (row branch) */
  int64_t block;     /* l (M1) or k (M2) */
  int64_t ell;       /* 0 = adaptive (M2) */
  int64_t rank;
  int64_t min_count;
  uint64_t seed;
} orc_params;

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
} orc_config;

typedef struct {
  double e;
  uint64_t trials_attempted;
  uint64_t trials_accepted;
  uint64_t z;
  int64_t underdetermined_rows;
  int64_t gram_rank;
  int32_t borderline;
} orc_report;

/* rng.hpp:12-57 */
uint64_t orc_rng_state(uint64_t seed, uint64_t tag, uint64_t index);
uint64_t orc_next_u64(uint64_t* st);
double orc_next_unit(uint64_t* st);
uint64_t orc_next_below(uint64_t* st, uint64_t bound);
double orc_next_normal(uint64_t* st);

/* sampler.cpp:12-23 : count sorted distinct indices drawn from [0,pool) */
void orc_draw(int64_t pool, int64_t count, uint64_t* st, int64_t* out);

/* sampler.cpp:58-87 (M2) and :27-56 (M1). Returns the survivor count q
 * (cols for M2, rows for M1); idx_out receives the drawn rows/cols (block
 * entries), surv_out (may be NULL) the survivors. Acceptance is q >= min_count. */
int64_t orc_sample(const uint8_t* mask, int64_t m, int64_t n, int32_t mode, int64_t block,
                   uint64_t seed, uint64_t attempt, int64_t* idx_out, int64_t* surv_out);

/* harvest.cpp:11-35 */
int orc_trial_params(const orc_config* cfg, int64_t m, int64_t n, orc_params* out);

/* harvest.cpp:79-120 selection only: the attempt-order prefix of accepted
 * attempts. accepted_list (may be NULL) gets up to `trials` attempt ids;
 * q_list (may be NULL) their survivor counts. */
int orc_select(const uint8_t* mask, int64_t m, int64_t n, const orc_params* p, uint64_t trials,
               uint64_t* accepted_list, int64_t* q_list, uint64_t* attempted, uint64_t* accepted);

/* spectra.cpp:48-86: the ell smallest right singular vectors of S (p x q,
 * row-major), each sign-fixed, as columns of zeta (q x ell, column t at
 * zeta + t*q); sv (ell) the singular values. */
int orc_small_singular_vectors(const double* S, int64_t p, int64_t q, int64_t r, int64_t ell,
                               double* zeta, double* sv);

/* harvest.cpp:79-120 with spectra.cpp:7-23: literal Gram accumulation. G is
 * n x n row-major and zero-initialised by the callee. */
int orc_harvest(const double* Y, const uint8_t* mask, int64_t m, int64_t n, const orc_params* p,
                uint64_t trials, double* G, uint64_t* attempted, uint64_t* accepted, uint64_t* z);

/* solver.cpp:15-62 (LAPACKE dsyev from scipy's bundled OpenBLAS). G is
 * overwritten. V is n x r row-major. w_out (may be NULL) receives all n
 * ascending eigenvalues. */
int orc_solve_v(double* G, int64_t n, int64_t r, double tol, double* V, int64_t* gram_rank,
                int32_t* borderline, double* w_out);

/* solver.cpp:64-89 + detail/row_solve.hpp:12-36: per-row complete orthogonal
 * decomposition least squares. */
int orc_solve_u(const double* Y, const uint8_t* mask, int64_t m, int64_t n, const double* V,
                int64_t r, double* U, int64_t* flagged);

/* one row of detail/row_solve.hpp; returns 1 when the row is full rank */
int orc_solve_row(const double* A, const double* y, int64_t nj, int64_t r, double* u);

/* core.cpp:15-39 */
/* baseline_als (src/als.cpp:11-44): V from Rng(seed, ALS_INIT=6, i).next_normal,
 * `iterations` rounds of U = solve_u(M, V), V = solve_u(M^T, U), a final U step;
 * e = masked_residual_norm(M, F), flagged = the last U step's count. */
int orc_als(const double* Y, const uint8_t* mask, int64_t m, int64_t n, int64_t r, int64_t iterations,
            uint64_t seed, double* U, double* V, int64_t* flagged, double* e);

double orc_masked_residual_norm(const double* Y, const uint8_t* mask, int64_t m, int64_t n,
                                const double* U, const double* V, int64_t r);

/* solver.cpp:93-146 (without wall time). U: m x r, V: n x r. */
int orc_decompose(const double* Y, const uint8_t* mask, int64_t m, int64_t n,
                  const orc_config* cfg, double* U, double* V, orc_report* rep);

/* synth.cpp:12-71 restricted to the observed matrix (Y and mask), for a row
 * block [row0, row0+rows). Y hidden cells are NaN. A is m x r, B r x n are
 * generated by the callee from the per-row streams. */
/* config-5 track generator restated from its specification (this library's
 * rsm_generate_tracks; the reference has no counterpart). */
void orc_generate_tracks(int64_t points, int64_t frames, int64_t wmin, int64_t wmax, double sigma,
                         uint64_t seed, double* Y, uint8_t* W);

void orc_generate_rows(int64_t m, int64_t n, int64_t r, double rho, double sigma, uint64_t seed,
                       int64_t row0, int64_t rows, double* Y, uint8_t* mask);

#ifdef __cplusplus
}
#endif
#endif
