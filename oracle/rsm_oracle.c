/*
 * rsm_oracle.c -- CPU restatement of the reference RSM hot path (test
 * infrastructure; see rsm_oracle.h for the contract and pinning notes).
 *
 * Reference paths below are relative to /root/reference/proj.
 */
#include "rsm_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng --- */
/* include/rsm/rng.hpp:12-57: counter-based splitmix64 streams */

static uint64_t orc_mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

uint64_t orc_rng_state(uint64_t seed, uint64_t tag, uint64_t index) {
  uint64_t s = orc_mix(seed + 0x9e3779b97f4a7c15ull * tag); /* rng.hpp:15 */
  return orc_mix(s + 0xbf58476d1ce4e5b9ull * index);        /* rng.hpp:16 */
}

uint64_t orc_next_u64(uint64_t* st) { /* rng.hpp:19-22 */
  *st += 0x9e3779b97f4a7c15ull;
  return orc_mix(*st);
}

double orc_next_unit(uint64_t* st) { /* rng.hpp:25-27 */
  return ((double)(orc_next_u64(st) >> 11) + 0.5) * 0x1.0p-53;
}

uint64_t orc_next_below(uint64_t* st, uint64_t bound) { /* rng.hpp:30-36 */
  const uint64_t limit = bound * (UINT64_MAX / bound);
  for (;;) {
    uint64_t v = orc_next_u64(st);
    if (v < limit) return v % bound;
  }
}

double orc_next_normal(uint64_t* st) { /* rng.hpp:40-44 */
  double u1 = orc_next_unit(st);
  double u2 = orc_next_unit(st);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* --------------------------------------------------------------- sampler --- */

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* sampler.cpp:12-23: partial Fisher-Yates over a fresh identity permutation
 * of [0,pool), first `count` slots, sorted. The identity permutation is kept
 * virtual (a position->value map of the touched slots); the output is the
 * same as the reference's iota+swap. */
void orc_draw(int64_t pool, int64_t count, uint64_t* st, int64_t* out) {
  int64_t* key = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * count + 2));
  int64_t* val = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * count + 2));
  int64_t nmap = 0;
#define ORC_GET(p, res)                              \
  do {                                               \
    res = (p);                                       \
    for (int64_t _i = 0; _i < nmap; ++_i)            \
      if (key[_i] == (p)) { res = val[_i]; break; }  \
  } while (0)
#define ORC_SET(p, v)                                          \
  do {                                                         \
    int64_t _f = -1;                                           \
    for (int64_t _i = 0; _i < nmap; ++_i)                      \
      if (key[_i] == (p)) { _f = _i; break; }                  \
    if (_f < 0) { key[nmap] = (p); val[nmap] = (v); ++nmap; }  \
    else val[_f] = (v);                                        \
  } while (0)
  for (int64_t t = 0; t < count; ++t) {
    const int64_t j = t + (int64_t)orc_next_below(st, (uint64_t)(pool - t));
    int64_t vt, vj;
    ORC_GET(t, vt);
    ORC_GET(j, vj);
    ORC_SET(t, vj);
    ORC_SET(j, vt);
  }
  for (int64_t t = 0; t < count; ++t) ORC_GET(t, out[t]);
#undef ORC_GET
#undef ORC_SET
  free(key);
  free(val);
  qsort(out, (size_t)count, sizeof(int64_t), cmp_i64);
}

int64_t orc_sample(const uint8_t* mask, int64_t m, int64_t n, int32_t mode, int64_t block,
                   uint64_t seed, uint64_t attempt, int64_t* idx_out, int64_t* surv_out) {
  uint64_t st = orc_rng_state(seed, 5 /* stream::TRIAL */, attempt); /* sampler.hpp:36 */
  int64_t q = 0;
  if (mode == 1) { /* sample_m2, sampler.cpp:58-87 */
    orc_draw(m, block, &st, idx_out);
    for (int64_t j = 0; j < n; ++j) {
      int full = 1;
      for (int64_t t = 0; t < block; ++t)
        if (!mask[idx_out[t] * n + j]) { full = 0; break; }
      if (full) {
        if (surv_out) surv_out[q] = j;
        ++q;
      }
    }
  } else { /* sample_m1, sampler.cpp:27-56 */
    orc_draw(n, block, &st, idx_out);
    for (int64_t i = 0; i < m; ++i) {
      int full = 1;
      for (int64_t c = 0; c < block; ++c)
        if (!mask[i * n + idx_out[c]]) { full = 0; break; }
      if (full) {
        if (surv_out) surv_out[q] = i;
        ++q;
      }
    }
  }
  return q;
}

/* --------------------------------------------------------------- harvest --- */

int orc_trial_params(const orc_config* cfg, int64_t m, int64_t n, orc_params* p) {
  /* harvest.cpp:11-35 */
  const int64_t mn = m < n ? m : n;
  if (cfg->rank < 1) return ORC_INVALID;
  if (cfg->rank >= mn) return ORC_INVALID;
  p->mode = cfg->mode;
  p->rank = cfg->rank;
  p->seed = cfg->seed;
  p->block = cfg->block > 0 ? cfg->block : cfg->rank + 1;
  if (p->block <= cfg->rank) return ORC_INVALID;
  const int64_t pool = cfg->mode == 0 ? n : m;
  if (p->block > pool) return ORC_INVALID;
  p->min_count = cfg->min_dim > 0 ? cfg->min_dim : cfg->rank + 1;
  if (p->min_count < cfg->rank + 1) return ORC_INVALID;
  if (cfg->mode == 0) {
    p->ell = cfg->vectors_per_trial > 0 ? cfg->vectors_per_trial : p->block - cfg->rank;
    if (p->ell > p->block - cfg->rank) return ORC_INVALID;
  } else {
    p->ell = cfg->vectors_per_trial;
  }
  return ORC_OK;
}

int orc_select(const uint8_t* mask, int64_t m, int64_t n, const orc_params* p, uint64_t trials,
               uint64_t* accepted_list, int64_t* q_list, uint64_t* attempted, uint64_t* accepted) {
  if (trials < 1) return ORC_INVALID;
  const uint64_t budget = 20 * trials; /* harvest.cpp:85 */
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)p->block);
  uint64_t att = 0, acc = 0;
  while (acc < trials && att < budget) { /* consumption order, harvest.cpp:110-117 */
    const int64_t q = orc_sample(mask, m, n, p->mode, p->block, p->seed, att, idx, NULL);
    if (q >= p->min_count) {
      if (accepted_list) accepted_list[acc] = att;
      if (q_list) q_list[acc] = q;
      ++acc;
    }
    ++att;
  }
  free(idx);
  *attempted = att;
  *accepted = acc;
  return ORC_OK;
}

/* --------------------------------------------------------------- spectra --- */

/* One-sided (Hestenes) Jacobi on the columns of B (rows x cols, row-major):
 * on return the columns are mutually orthogonal and V (cols x cols,
 * row-major) holds the accumulated rotations, B_in * V = B_out. */
static void orc_jacobi_cols(double* B, int64_t rows, int64_t cols, double* V) {
  for (int64_t i = 0; i < cols; ++i)
    for (int64_t j = 0; j < cols; ++j) V[i * cols + j] = (i == j) ? 1.0 : 0.0;
  const double tol = (double)(rows > 1 ? rows : 1) * DBL_EPSILON;
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (int64_t i = 0; i < cols - 1; ++i)
      for (int64_t j = i + 1; j < cols; ++j) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int64_t k = 0; k < rows; ++k) {
          const double x = B[k * cols + i], y = B[k * cols + j];
          a += x * x;
          b += y * y;
          g += x * y;
        }
        if (a == 0.0 || b == 0.0 || fabs(g) <= tol * sqrt(a * b)) continue;
        rotated = 1;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int64_t k = 0; k < rows; ++k) {
          const double x = B[k * cols + i], y = B[k * cols + j];
          B[k * cols + i] = c * x - s * y;
          B[k * cols + j] = s * x + c * y;
        }
        for (int64_t k = 0; k < cols; ++k) {
          const double x = V[k * cols + i], y = V[k * cols + j];
          V[k * cols + i] = c * x - s * y;
          V[k * cols + j] = s * x + c * y;
        }
      }
    if (!rotated) break;
  }
}

/* Orthonormal completion: Q (q x q, column-major: column c at Q+c*q) whose
 * first K columns are the given orthonormal columns (column-major in W,
 * possibly sign-flipped) and whose remaining columns span the complement.
 * Householder QR of W applied to the identity. */
static void orc_complete_basis(const double* W, int64_t q, int64_t K, double* Q) {
  double* H = (double*)malloc(sizeof(double) * (size_t)(q * K));
  double* beta = (double*)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
  memcpy(H, W, sizeof(double) * (size_t)(q * K));
  for (int64_t k = 0; k < K; ++k) {
    double* h = H + k * q;
    double nrm = 0.0;
    for (int64_t i = k; i < q; ++i) nrm += h[i] * h[i];
    nrm = sqrt(nrm);
    const double alpha = h[k] >= 0 ? -nrm : nrm;
    double vnorm2 = 0.0;
    h[k] -= alpha; /* v = x - alpha e_k */
    for (int64_t i = k; i < q; ++i) vnorm2 += h[i] * h[i];
    beta[k] = vnorm2 > 0 ? 2.0 / vnorm2 : 0.0;
    for (int64_t j = k + 1; j < K; ++j) {
      double* x = H + j * q;
      double d = 0.0;
      for (int64_t i = k; i < q; ++i) d += h[i] * x[i];
      d *= beta[k];
      for (int64_t i = k; i < q; ++i) x[i] -= d * h[i];
    }
  }
  for (int64_t c = 0; c < q; ++c) {
    double* x = Q + c * q;
    for (int64_t i = 0; i < q; ++i) x[i] = (i == c) ? 1.0 : 0.0;
    for (int64_t k = K - 1; k >= 0; --k) {
      const double* h = H + k * q;
      double d = 0.0;
      for (int64_t i = k; i < q; ++i) d += h[i] * x[i];
      d *= beta[k];
      for (int64_t i = k; i < q; ++i) x[i] -= d * h[i];
    }
  }
  free(H);
  free(beta);
}

/* spectra.cpp:48-86 */
int orc_small_singular_vectors(const double* S, int64_t p, int64_t q, int64_t r, int64_t ell,
                               double* zeta, double* sv_out) {
  if (q - r < 1) return ORC_INVALID;              /* :51 */
  if (p < r + 1) return ORC_INVALID;              /* :52 */
  if (ell < 1 || ell > q - r) return ORC_INVALID; /* :53 */

  const int64_t K = p < q ? p : q; /* min(p,q) singular values exist */
  double* Vfull = (double*)malloc(sizeof(double) * (size_t)(q * q)); /* column-major */
  double* sig = (double*)malloc(sizeof(double) * (size_t)K);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)K);

  if (p >= q) {
    /* tall/square: Jacobi on the q columns of S gives the full V directly */
    double* B = (double*)malloc(sizeof(double) * (size_t)(p * q));
    double* V = (double*)malloc(sizeof(double) * (size_t)(q * q));
    memcpy(B, S, sizeof(double) * (size_t)(p * q));
    orc_jacobi_cols(B, p, q, V);
    for (int64_t j = 0; j < q; ++j) {
      double s = 0.0;
      for (int64_t k = 0; k < p; ++k) s += B[k * q + j] * B[k * q + j];
      sig[j] = sqrt(s);
      order[j] = j;
    }
    /* descending singular values (stable insertion sort) */
    for (int64_t a = 1; a < K; ++a) {
      int64_t x = order[a], b = a - 1;
      while (b >= 0 && sig[order[b]] < sig[x]) { order[b + 1] = order[b]; --b; }
      order[b + 1] = x;
    }
    for (int64_t c = 0; c < q; ++c)
      for (int64_t i = 0; i < q; ++i) Vfull[c * q + i] = V[i * q + order[c]];
    double* sorted = (double*)malloc(sizeof(double) * (size_t)K);
    for (int64_t c = 0; c < K; ++c) sorted[c] = sig[order[c]];
    memcpy(sig, sorted, sizeof(double) * (size_t)K);
    free(sorted);
    free(B);
    free(V);
  } else {
    /* wide: Jacobi on the p rows of S (columns of S^T); rotated rows are
     * sigma_i v_i^T. Columns past the nonzero ones are completed to an
     * orthonormal basis of R^q (the kernel, singular value 0). */
    double* B = (double*)malloc(sizeof(double) * (size_t)(q * p)); /* S^T, q x p row-major */
    double* U = (double*)malloc(sizeof(double) * (size_t)(p * p));
    for (int64_t i = 0; i < p; ++i)
      for (int64_t j = 0; j < q; ++j) B[j * p + i] = S[i * q + j];
    orc_jacobi_cols(B, q, p, U);
    for (int64_t i = 0; i < p; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < q; ++j) s += B[j * p + i] * B[j * p + i];
      sig[i] = sqrt(s);
      order[i] = i;
    }
    for (int64_t a = 1; a < K; ++a) {
      int64_t x = order[a], b = a - 1;
      while (b >= 0 && sig[order[b]] < sig[x]) { order[b + 1] = order[b]; --b; }
      order[b + 1] = x;
    }
    int64_t nz = 0;
    double* W = (double*)malloc(sizeof(double) * (size_t)(q * p));
    double* sorted = (double*)malloc(sizeof(double) * (size_t)K);
    for (int64_t c = 0; c < K; ++c) {
      const int64_t i = order[c];
      sorted[c] = sig[i];
      if (sig[i] > 0.0) {
        for (int64_t j = 0; j < q; ++j) W[nz * q + j] = B[j * p + i] / sig[i];
        ++nz;
      }
    }
    memcpy(sig, sorted, sizeof(double) * (size_t)K);
    orc_complete_basis(W, q, nz, Vfull);
    /* keep the exact Jacobi vectors for the nonzero part (the completion may
     * have flipped their signs; the sign fix below makes that irrelevant) */
    for (int64_t c = 0; c < nz; ++c)
      for (int64_t j = 0; j < q; ++j) Vfull[c * q + j] = W[c * q + j];
    free(sorted);
    free(W);
    free(B);
    free(U);
  }

  for (int64_t t = 0; t < ell; ++t) { /* :64-82 */
    const int64_t c = q - 1 - t;
    const double* col = Vfull + c * q;
    if (sv_out) sv_out[t] = c < K ? sig[c] : 0.0;
    int64_t arg = 0;
    double best = -1.0;
    for (int64_t i = 0; i < q; ++i) {
      const double a = fabs(col[i]);
      if (a > best) { best = a; arg = i; }
    }
    const double flip = col[arg] < 0.0 ? -1.0 : 1.0;
    for (int64_t i = 0; i < q; ++i) zeta[t * q + i] = flip * col[i];
  }
  free(Vfull);
  free(sig);
  free(order);
  return ORC_OK;
}

/* harvest.cpp:37-51 (attempt_trial) + :79-120 (consumption) with the literal
 * spectra.cpp:7-23 accumulation. */
int orc_harvest(const double* Y, const uint8_t* mask, int64_t m, int64_t n, const orc_params* p,
                uint64_t trials, double* G, uint64_t* attempted, uint64_t* accepted, uint64_t* z) {
  if (trials < 1) return ORC_INVALID;
  memset(G, 0, sizeof(double) * (size_t)(n * n));
  const uint64_t budget = 20 * trials;
  const int64_t maxsurv = m > n ? m : n;
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)p->block);
  int64_t* surv = (int64_t*)malloc(sizeof(int64_t) * (size_t)maxsurv);
  uint64_t att = 0, acc = 0, zz = 0;
  int status = ORC_OK;
  while (acc < trials && att < budget) {
    const int64_t q = orc_sample(mask, m, n, p->mode, p->block, p->seed, att, idx, surv);
    ++att;
    if (q < p->min_count) continue;
    /* Submatrix S: rows x cols, and the column support of the vectors */
    int64_t rows, cols;
    const int64_t *ridx, *cidx;
    if (p->mode == 1) { rows = p->block; cols = q; ridx = idx; cidx = surv; }
    else { rows = q; cols = p->block; ridx = surv; cidx = idx; }
    double* S = (double*)malloc(sizeof(double) * (size_t)(rows * cols));
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t j = 0; j < cols; ++j) S[i * cols + j] = Y[ridx[i] * n + cidx[j]];
    int64_t ell;
    if (p->mode == 1) {
      const int64_t avail = cols - p->rank;
      ell = p->ell > 0 ? (p->ell < avail ? p->ell : avail) : avail;
    } else {
      ell = p->ell;
    }
    double* zeta = (double*)malloc(sizeof(double) * (size_t)(cols * (ell > 0 ? ell : 1)));
    status = orc_small_singular_vectors(S, rows, cols, p->rank, ell, zeta, NULL);
    if (status != ORC_OK) { free(S); free(zeta); break; }
    for (int64_t t = 0; t < ell; ++t) { /* GramAccumulator::accumulate, spectra.cpp:7-23 */
      const double* v = zeta + t * cols;
      for (int64_t a = 0; a < cols; ++a) {
        double* row = G + cidx[a] * n;
        const double va = v[a];
        for (int64_t b = 0; b < cols; ++b) row[cidx[b]] += va * v[b];
      }
      ++zz;
    }
    free(S);
    free(zeta);
    ++acc;
  }
  free(idx);
  free(surv);
  *attempted = att;
  *accepted = acc;
  *z = zz;
  return status;
}

/* ---------------------------------------------------------------- solver --- */

extern int scipy_LAPACKE_dsyev(int layout, char jobz, char uplo, int n, double* a, int lda,
                               double* w);
extern void scipy_openblas_set_num_threads(int);

int orc_solve_v(double* G, int64_t n, int64_t r, double tol, double* V, int64_t* gram_rank,
                int32_t* borderline, double* w_out) {
  /* solver.cpp:15-62 */
  if (n < 1) return ORC_INVALID;
  if (r < 1 || r >= n) return ORC_INVALID;
  if (!(tol > 0.0)) return ORC_INVALID;
  scipy_openblas_set_num_threads(1); /* OPENBLAS_NUM_THREADS=1, tools/rsm.cpp:222 */
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  const int info = scipy_LAPACKE_dsyev(102 /* COL_MAJOR */, 'V', 'L', (int)n, G, (int)n, w);
  if (info != 0) { free(w); return ORC_INTERNAL; }
  if (w_out) memcpy(w_out, w, sizeof(double) * (size_t)n);
  const double lambda_max = w[n - 1] > 0.0 ? w[n - 1] : 0.0;
  const double threshold = tol * lambda_max;
  int64_t significant = 0;
  for (int64_t i = 0; i < n; ++i)
    if (w[i] > threshold) ++significant;
  if (significant < n - r) { free(w); return ORC_COVERAGE; }
  *gram_rank = significant;
  *borderline = !(w[r] > 10.0 * threshold);
  for (int64_t c = 0; c < r; ++c) {
    const double* col = G + c * n;
    int64_t arg = 0;
    double best = -1.0;
    for (int64_t i = 0; i < n; ++i) {
      const double mag = fabs(col[i]);
      if (mag > best) { best = mag; arg = i; }
    }
    const double flip = col[arg] < 0.0 ? -1.0 : 1.0;
    for (int64_t i = 0; i < n; ++i) V[i * r + c] = flip * col[i];
  }
  free(w);
  return ORC_OK;
}

/* Eigen::makeHouseholder semantics: x = [c0; tail] -> beta, tau, essential
 * stored in x[1..]. Returns beta. */
static double orc_householder(double* x, int64_t len, double* tau) {
  double tail = 0.0;
  for (int64_t i = 1; i < len; ++i) tail += x[i] * x[i];
  const double c0 = x[0];
  if (tail <= DBL_MIN) {
    *tau = 0.0;
    for (int64_t i = 1; i < len; ++i) x[i] = 0.0;
    return c0;
  }
  double beta = sqrt(c0 * c0 + tail);
  if (c0 >= 0.0) beta = -beta;
  for (int64_t i = 1; i < len; ++i) x[i] /= (c0 - beta);
  *tau = (beta - c0) / beta;
  return beta;
}

/* apply H = I - tau v v^T (v = [1; ess]) to the vector y (length len) */
static void orc_apply_h(const double* ess, double tau, double* y, int64_t len) {
  if (tau == 0.0) return;
  double d = y[0];
  for (int64_t i = 1; i < len; ++i) d += ess[i] * y[i];
  d *= tau;
  y[0] -= d;
  for (int64_t i = 1; i < len; ++i) y[i] -= d * ess[i];
}

/* detail/row_solve.hpp:12-36: complete orthogonal decomposition least squares
 * with Eigen's ColPivHouseholderQR rank rule (threshold eps*min(nj,r) times
 * the largest pivot) and the minimum-norm solution on deficiency.
 * A is nj x r column-major (column k at A + k*nj). */
int orc_solve_row(const double* A_in, const double* y_in, int64_t nj, int64_t r, double* u) {
  if (nj == 0) {
    for (int64_t k = 0; k < r; ++k) u[k] = 0.0;
    return 0;
  }
  double* A = (double*)malloc(sizeof(double) * (size_t)(nj * r));
  double* y = (double*)malloc(sizeof(double) * (size_t)nj);
  double* tau = (double*)malloc(sizeof(double) * (size_t)r);
  double* nupd = (double*)malloc(sizeof(double) * (size_t)r);
  double* ndir = (double*)malloc(sizeof(double) * (size_t)r);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)r);
  memcpy(A, A_in, sizeof(double) * (size_t)(nj * r));
  memcpy(y, y_in, sizeof(double) * (size_t)nj);
  const int64_t size = nj < r ? nj : r;
  double maxnorm = 0.0;
  for (int64_t k = 0; k < r; ++k) {
    double s = 0.0;
    for (int64_t i = 0; i < nj; ++i) s += A[k * nj + i] * A[k * nj + i];
    nupd[k] = ndir[k] = sqrt(s);
    perm[k] = k;
    if (nupd[k] > maxnorm) maxnorm = nupd[k];
  }
  const double thr_helper = (maxnorm * DBL_EPSILON) * (maxnorm * DBL_EPSILON) / (double)nj;
  const double norm_downdate_threshold = sqrt(DBL_EPSILON);
  int64_t nonzero = size;
  double maxpivot = 0.0;
  for (int64_t k = 0; k < size; ++k) {
    int64_t big = k;
    for (int64_t j = k + 1; j < r; ++j)
      if (nupd[j] > nupd[big]) big = j;
    const double big_sq = nupd[big] * nupd[big];
    if (nonzero == size && big_sq < thr_helper * (double)(nj - k)) nonzero = k;
    if (big != k) {
      for (int64_t i = 0; i < nj; ++i) {
        double t = A[k * nj + i]; A[k * nj + i] = A[big * nj + i]; A[big * nj + i] = t;
      }
      double t = nupd[k]; nupd[k] = nupd[big]; nupd[big] = t;
      t = ndir[k]; ndir[k] = ndir[big]; ndir[big] = t;
      int64_t pt = perm[k]; perm[k] = perm[big]; perm[big] = pt;
    }
    double* col = A + k * nj + k;
    const double beta = orc_householder(col, nj - k, &tau[k]);
    col[0] = beta;
    if (fabs(beta) > maxpivot) maxpivot = fabs(beta);
    for (int64_t j = k + 1; j < r; ++j) orc_apply_h(col, tau[k], A + j * nj + k, nj - k);
    for (int64_t j = k + 1; j < r; ++j) {
      if (nupd[j] != 0.0) {
        double t = fabs(A[j * nj + k]) / nupd[j];
        t = (1.0 + t) * (1.0 - t);
        if (t < 0.0) t = 0.0;
        const double t2 = t * (nupd[j] / ndir[j]) * (nupd[j] / ndir[j]);
        if (t2 <= norm_downdate_threshold) {
          double s = 0.0;
          for (int64_t i = k + 1; i < nj; ++i) s += A[j * nj + i] * A[j * nj + i];
          ndir[j] = sqrt(s);
          nupd[j] = ndir[j];
        } else {
          nupd[j] *= sqrt(t);
        }
      }
    }
  }
  const double premult = maxpivot * (DBL_EPSILON * (double)size);
  int64_t rank = 0;
  for (int64_t i = 0; i < nonzero; ++i)
    if (fabs(A[i * nj + i]) > premult) ++rank;

  double* z = (double*)calloc((size_t)r, sizeof(double));
  if (rank > 0) {
    /* c = Q^T y restricted to the first `rank` reflectors */
    for (int64_t k = 0; k < rank; ++k) orc_apply_h(A + k * nj + k, tau[k], y + k, nj - k);
    if (rank == r) {
      for (int64_t i = r - 1; i >= 0; --i) {
        double s = y[i];
        for (int64_t j = i + 1; j < r; ++j) s -= A[j * nj + i] * z[j];
        z[i] = s / A[i * nj + i];
      }
    } else {
      /* minimum-norm solution of [R11 R12] w = c1 via QR of W^T (r x rank) */
      double* Wt = (double*)malloc(sizeof(double) * (size_t)(r * rank)); /* column-major r x rank */
      double* tw = (double*)malloc(sizeof(double) * (size_t)rank);
      for (int64_t i = 0; i < rank; ++i)
        for (int64_t j = 0; j < r; ++j) Wt[i * r + j] = (j >= i) ? A[j * nj + i] : 0.0;
      for (int64_t k = 0; k < rank; ++k) {
        double* col = Wt + k * r + k;
        const double beta = orc_householder(col, r - k, &tw[k]);
        col[0] = beta;
        for (int64_t j = k + 1; j < rank; ++j) orc_apply_h(col, tw[k], Wt + j * r + k, r - k);
      }
      /* W^T = Q2 R2 -> W = R2^T Q2^T; solve R2^T s = c1, then w = Q2 [s; 0] */
      double* s = (double*)calloc((size_t)r, sizeof(double));
      for (int64_t i = 0; i < rank; ++i) {
        double acc = y[i];
        for (int64_t j = 0; j < i; ++j) acc -= Wt[i * r + j] * s[j];
        s[i] = acc / Wt[i * r + i];
      }
      for (int64_t k = rank - 1; k >= 0; --k) orc_apply_h(Wt + k * r + k, tw[k], s + k, r - k);
      for (int64_t j = 0; j < r; ++j) z[j] = s[j];
      free(s);
      free(Wt);
      free(tw);
    }
  }
  for (int64_t k = 0; k < r; ++k) u[perm[k]] = z[k];
  free(z);
  free(A);
  free(y);
  free(tau);
  free(nupd);
  free(ndir);
  free(perm);
  return (nj >= r && rank == r) ? 1 : 0;
}

int orc_solve_u(const double* Y, const uint8_t* mask, int64_t m, int64_t n, const double* V,
                int64_t r, double* U, int64_t* flagged) {
  /* solver.cpp:64-89 (serial twin: reference.cpp:27-38) */
  if (r < 1) return ORC_INVALID;
  double* A = (double*)malloc(sizeof(double) * (size_t)(n * r));
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t fl = 0;
  for (int64_t i = 0; i < m; ++i) {
    int64_t nj = 0;
    for (int64_t j = 0; j < n; ++j)
      if (mask[i * n + j]) ++nj;
    int64_t t = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (!mask[i * n + j]) continue;
      for (int64_t k = 0; k < r; ++k) A[k * nj + t] = V[j * r + k];
      y[t] = Y[i * n + j];
      ++t;
    }
    if (!orc_solve_row(A, y, nj, r, U + i * r)) ++fl;
  }
  free(A);
  free(y);
  *flagged = fl;
  return ORC_OK;
}

double orc_masked_residual_norm(const double* Y, const uint8_t* mask, int64_t m, int64_t n,
                                const double* U, const double* V, int64_t r) {
  /* core.cpp:15-39 */
  int64_t w = 0;
  for (int64_t p = 0; p < m * n; ++p) w += mask[p];
  if (w == 0) return NAN;
  double ss = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    const double* ui = U + i * r;
    for (int64_t j = 0; j < n; ++j) {
      if (!mask[i * n + j]) continue;
      const double* vj = V + j * r;
      double p = 0.0;
      for (int64_t k = 0; k < r; ++k) p += ui[k] * vj[k];
      const double d = Y[i * n + j] - p;
      ss += d * d;
    }
  }
  return sqrt(ss) / sqrt((double)w);
}

static int orc_decompose_oriented(const double* Y, const uint8_t* mask, int64_t m, int64_t n,
                                  const orc_config* cfg, double* U, double* V, orc_report* rep) {
  /* solver.cpp:93-115 */
  orc_params p;
  int st = orc_trial_params(cfg, m, n, &p);
  if (st) return st;
  double* G = (double*)malloc(sizeof(double) * (size_t)(n * n));
  st = orc_harvest(Y, mask, m, n, &p, cfg->trials, G, &rep->trials_attempted,
                   &rep->trials_accepted, &rep->z);
  if (!st) st = orc_solve_v(G, n, cfg->rank, cfg->gram_rank_tol, V, &rep->gram_rank,
                            &rep->borderline, NULL);
  free(G);
  if (st) return st;
  return orc_solve_u(Y, mask, m, n, V, cfg->rank, U, &rep->underdetermined_rows);
}

int orc_decompose(const double* Y, const uint8_t* mask, int64_t m, int64_t n,
                  const orc_config* cfg, double* U, double* V, orc_report* rep) {
  /* solver.cpp:119-146 */
  memset(rep, 0, sizeof(*rep));
  const int64_t mn = m < n ? m : n;
  if (cfg->rank < 1 || cfg->rank >= mn) return ORC_INVALID;
  if (!(cfg->epsilon > 0.0 && cfg->epsilon < 1.0)) return ORC_INVALID;
  if (cfg->trials < 1) return ORC_INVALID;
  int64_t w = 0;
  for (int64_t q = 0; q < m * n; ++q) w += mask[q];
  if (w == 0) return ORC_COVERAGE;
  int st;
  if (m >= n) {
    st = orc_decompose_oriented(Y, mask, m, n, cfg, U, V, rep);
  } else {
    /* core.hpp:50-56 transposed(): hidden cells NaN, mask transposed */
    double* Yt = (double*)malloc(sizeof(double) * (size_t)(m * n));
    uint8_t* Mt = (uint8_t*)malloc((size_t)(m * n));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) {
        Mt[j * m + i] = mask[i * n + j];
        Yt[j * m + i] = mask[i * n + j] ? Y[i * n + j] : NAN;
      }
    st = orc_decompose_oriented(Yt, Mt, n, m, cfg, V, U, rep);
    free(Yt);
    free(Mt);
  }
  if (st) return st;
  rep->e = orc_masked_residual_norm(Y, mask, m, n, U, V, cfg->rank);
  return ORC_OK;
}

/* ----------------------------------------------------------------- synth --- */

int orc_als(const double* Y, const uint8_t* mask, int64_t m, int64_t n, int64_t r, int64_t iterations,
            uint64_t seed, double* U, double* V, int64_t* flagged, double* e) {
  /* als.cpp:17-20 */
  if (r < 1 || r >= (m < n ? m : n)) return 2;
  if (iterations < 1) return 2;
  int64_t known = 0;
  for (int64_t q = 0; q < m * n; ++q) known += mask[q] ? 1 : 0;
  if (known == 0) return 4;
  for (int64_t i = 0; i < n; ++i) { /* als.cpp:22-26 */
    uint64_t st = orc_rng_state(seed, 6 /* ALS_INIT */, (uint64_t)i);
    for (int64_t k = 0; k < r; ++k) V[i * r + k] = orc_next_normal(&st);
  }
  /* M^T (core.hpp MaskedMatrix::transposed) */
  double* YT = (double*)malloc(sizeof(double) * (size_t)(m * n));
  uint8_t* WT = (uint8_t*)malloc((size_t)(m * n));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      YT[j * m + i] = Y[i * n + j];
      WT[j * m + i] = mask[i * n + j];
    }
  int64_t fl = 0, flt = 0;
  int st = 0;
  for (int64_t it = 0; it < iterations && st == 0; ++it) { /* als.cpp:29-32 */
    st = orc_solve_u(Y, mask, m, n, V, r, U, &fl);
    if (st == 0) st = orc_solve_u(YT, WT, n, m, U, r, V, &flt);
  }
  if (st == 0) st = orc_solve_u(Y, mask, m, n, V, r, U, &fl); /* als.cpp:33 */
  free(YT);
  free(WT);
  if (st) return st;
  *flagged = fl;
  *e = orc_masked_residual_norm(Y, mask, m, n, U, V, r); /* als.cpp:40 */
  return 0;
}

void orc_generate_rows(int64_t m, int64_t n, int64_t r, double rho, double sigma, uint64_t seed,
                       int64_t row0, int64_t rows, double* Y, uint8_t* mask) {
  /* synth.cpp:12-57 (observed matrix only; streams are per row, so any row
   * block is generated independently). Ybar = A*B summed in k order. */
  (void)m;
  double* B = (double*)malloc(sizeof(double) * (size_t)(r * n));
  for (int64_t k = 0; k < r; ++k) {
    uint64_t st = orc_rng_state(seed, 2 /* FACTOR_B */, (uint64_t)k);
    for (int64_t j = 0; j < n; ++j) B[k * n + j] = orc_next_normal(&st);
  }
  double* a = (double*)malloc(sizeof(double) * (size_t)r);
  for (int64_t ii = 0; ii < rows; ++ii) {
    const int64_t i = row0 + ii;
    uint64_t sa = orc_rng_state(seed, 1 /* FACTOR_A */, (uint64_t)i);
    for (int64_t k = 0; k < r; ++k) a[k] = orc_next_normal(&sa);
    uint64_t sn = orc_rng_state(seed, 3 /* NOISE */, (uint64_t)i);
    uint64_t sm = orc_rng_state(seed, 4 /* MASK */, (uint64_t)i);
    double* yrow = Y + ii * n;
    uint8_t* mrow = mask + ii * n;
    for (int64_t j = 0; j < n; ++j) {
      double ybar = 0.0;
      for (int64_t k = 0; k < r; ++k) ybar += a[k] * B[k * n + j];
      yrow[j] = ybar;
    }
    if (sigma > 0.0)
      for (int64_t j = 0; j < n; ++j) yrow[j] += sigma * orc_next_normal(&sn);
    for (int64_t j = 0; j < n; ++j) {
      const int known = orc_next_unit(&sm) <= rho;
      mrow[j] = (uint8_t)known;
      if (!known) yrow[j] = NAN;
    }
  }
  free(a);
  free(B);
}


void orc_generate_tracks(int64_t points, int64_t frames, int64_t wmin, int64_t wmax, double sigma,
                         uint64_t seed, double* Y, uint8_t* W) {
  const int64_t n = 2 * frames;
  for (int64_t i = 0; i < points; ++i) {
    uint64_t sp = orc_rng_state(seed, 16 /* TRACK_POINT */, (uint64_t)i);
    const double X[4] = {2.0 * orc_next_unit(&sp) - 1.0, 2.0 * orc_next_unit(&sp) - 1.0,
                         2.0 * orc_next_unit(&sp) - 1.0, 1.0};
    uint64_t sw = orc_rng_state(seed, 18 /* TRACK_WINDOW */, (uint64_t)i);
    const int64_t L = wmin + (int64_t)orc_next_below(&sw, (uint64_t)(wmax - wmin + 1));
    const int64_t f0 = (int64_t)orc_next_below(&sw, (uint64_t)(frames - L + 1));
    uint64_t sn = orc_rng_state(seed, 19 /* TRACK_NOISE */, (uint64_t)i);
    for (int64_t j = 0; j < n; ++j) {
      const int64_t f = j / 2;
      if (f < f0 || f >= f0 + L) {
        Y[i * n + j] = NAN;
        W[i * n + j] = 0;
        continue;
      }
      /* camera row (j % 2) of frame f: entries 4*(j%2) .. +3 of the frame's stream */
      uint64_t sc = orc_rng_state(seed, 17 /* TRACK_CAMERA */, (uint64_t)f);
      double P[8];
      for (int q = 0; q < 8; ++q) P[q] = orc_next_normal(&sc);
      double s = 0.0;
      for (int q = 0; q < 4; ++q) s += P[(j % 2) * 4 + q] * X[q];
      if (sigma > 0.0) s += sigma * orc_next_normal(&sn);
      Y[i * n + j] = s;
      W[i * n + j] = 1;
    }
  }
}
