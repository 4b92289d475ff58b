// rsm_internal.h -- kernel argument blocks and launchers shared between the
// stage kernels (k_*.cu) and the host orchestration (rsm_ctx.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>

namespace rsmk {

// Host-side launch configuration, memoised per (kernel, block, dynamic smem):
// cudaFuncSetAttribute / cudaOccupancy* cost microseconds of host time, and
// after the selection's host sync every microsecond of it is GPU idle time.
// ensure_smem raises a kernel's dynamic-shared-memory limit once (only ever
// upwards); occupancy returns blocks per SM for (kernel, threads, smem).
void ensure_smem(const void* fn, size_t smem);
int occupancy(const void* fn, int threads, size_t smem);

// device-resident selection state (stage 1 compaction)
struct SelState {
  unsigned long long acc;             // accepted so far, capped at T
  unsigned long long acc_before;      // accepted before the current chunk
  unsigned long long attempted_done;  // attempt id + 1 of the T-th acceptance, 0 = not yet
  int qmax;                           // largest survivor count among accepted trials
  int pad;
  unsigned long long qsum;            // sum of the accepted trials' survivor counts (z)
};

struct SvdArgs {
  const double* Y;       // oriented values, m x n row-major
  int64_t m, n;
  const uint32_t* bitsR; // m x nwp row-major mask words
  int64_t nwp;
  const uint32_t* bitsC; // n x mwp column-major mask words (column branch)
  int64_t mwp;
  const int32_t* t_idx;  // T x block drawn indices (global trial numbering)
  int64_t t_lo, t_hi;    // this rank's trial range
  int block;             // K
  int rex;               // top vectors kept (q - ell)
  uint32_t* t_cm;        // local trials x cmw support words
  int64_t cmw;
  int64_t npad;          // expanded column count (multiple of 128)
  double* Vout;          // local trials x (rp/2) planes x npad x 2 (see k_svd.cu), or null
  int8_t* Wq;            // or: int8 digit slices [S][Kpad][npad], rows t*rex + p (k_gram_i8.cu)
  int64_t Kpad;
  int S;                 // digit slices (gram_i8_slices)
  int* colcnt;           // n per-column trial counts
  double* scratch;       // per-CTA vector scratch when shared memory is too small
  uint32_t* scratch_u32; // per-CTA 2*mwp words (column branch)
  int64_t Lpad;
  int use_smem;
  int max_outer;         // one-sided Jacobi rotations per trial (at most)
  int fast_basis;        // r = block - 1 (either branch): top-r basis from the Gram (no Jacobi)
  // speculative launch (decompose enqueues stages 2-5 before the selection's
  // outcome is on the host): trials at or past *sel_acc and trials whose
  // support exceeds Lcap are skipped; the host checks the selection state
  // after its one synchronisation and re-runs when either happened
  const unsigned long long* sel_acc;
  int64_t Lcap;
};

struct GramArgs {
  const uint32_t* t_cm;
  const double* V;  // expanded top vectors, SvdArgs::Vout layout
  int64_t T;       // local trial count
  int64_t cmw;
  int64_t npad;
  int R;
  int nslices;
  int lag;         // stage-3 ring: refill the stage released lag groups ago
  int accumulate;  // add to P instead of overwriting (trial chunks after the first)
  const int2* tiles;
  double* P;       // nslices x npad x npad partials
};

// stage 3 on tcgen05 (k_gram_i8.cu): int8 slices Wq[S][Kpad][npad] (MN-major)
struct GramI8Args {
  const int8_t* W;
  int64_t npad, Kpad;
  int64_t Kc;        // K rows per work unit (multiple of 32, <= gram_i8_kmax())
  int nk;            // K-chunks (P slices)
  int ntiles;        // 128 x 64 tiles touching the upper triangle
  const int2* tiles;
  double* P;         // nk x npad x npad partials (-W^T W per K-chunk)
  int accumulate;    // add to P (trial chunks after the first)
  int diag;          // RSM_I8_DIAG: 0 normal, 1 loads only, 2 MMAs only (timing experiments)
  int S;             // digit slices (gram_i8_slices)
};

struct EigArgs {
  const double* G;  // n x n
  int64_t n;
  int r, b;         // wanted, block
  double tol;       // gram_rank_tol
  int rows_per_cta;
  int rpw;          // rows per warp
  int gres;         // set by launch_eig: G rows resident in shared memory
  int kc;           // set by launch_eig: iterate rows staged per bulk copy
  const int* zero_rows;  // exactly-zero rows of G (k_zero_rows), or null
  double* X;        // n x ld  (3 buffers)
  double* Y;
  double* Z;
  double* part;     // grid x PARTW partials
  double* V;        // n x r output
  double* w;        // b Ritz values output
  int* istat;       // [0] status, [1] gram_rank (low), [2] borderline, [3] outer its, [4] matvecs
  double* dstat;    // [0] lambda_max, [1] ub, [2] max residual
  int max_outer;
  const int* cnt;   // per-column trial counts when G = diag(cnt) - PSD (else null)
  double amp;       // Chebyshev filter amplification cap (degree choice)
  int dmax;         // and degree cap
  int rr0_probe;     // first outer iteration: top Ritz value by power iteration only
  double* hout;      // pinned host block for w / dstat / istat (see k_eig.cu publish), or null
  int init_cq;       // CholQR of the random start block (0: the first filter takes it as is)
  double shift0;     // relative diagonal shift of the first CholQR pass after a filter
  int probe_its;     // power iterations of the probe round
};

struct SolveUArgs {
  const double* Y;
  const uint32_t* bitsR;
  int64_t m, n, nwp;
  int64_t row_lo, row_hi;
  const double* V;  // n x r
  double* U;        // m x r (rows row_lo..row_hi written)
  double* rowres;   // m residual^2 per row
  int* flagged;     // count (integer atomics)
  int r;
  const double* Ugiven;  // non-null: rows' solutions given (m x r), only the residual pass
                         // counts (masked_residual_norm through the stage-5 arithmetic)
  const double* Apre;    // non-null: rows' packed normal matrices (m x r(r+1)/2, k_normal_i8.cu)
  int pf;                // k_solve_u_preg: rows ahead pulled toward L2 by a bulk prefetch (0: none)
};

// rsm_ctx.cu: message for rsm_last_error(NULL) from host-only entry points
void set_host_error(const std::string& msg);

// k_prep.cu
void launch_pack_rows(const uint8_t* mask, int64_t m, int64_t n, uint32_t* bits, int64_t nwp,
                      cudaStream_t s);
void launch_unpack_rows(const uint32_t* bits, int64_t m, int64_t n, int64_t nwp, uint8_t* mask,
                        cudaStream_t s);
void launch_pack_cols(const uint8_t* mask, int64_t m, int64_t n, uint32_t* bits, int64_t mwp,
                      cudaStream_t s);
void launch_transpose(const double* Y, const uint8_t* M, int64_t m, int64_t n, double* Yt,
                      uint8_t* Mt, cudaStream_t s);
void launch_count_bits(const uint32_t* bits, int64_t nwords, unsigned long long* out,
                       cudaStream_t s);
// k_synth.cu: device generator (B is r x n scratch)
void launch_generate(int64_t m, int64_t n, int64_t r, double rho, double sigma, uint64_t seed, double* B,
                     int64_t nwp, double* Y, uint32_t* bits, int sms, cudaStream_t s);
// k_select.cu
void launch_select(const uint32_t* bits, int64_t stride, int64_t nwords, int64_t pool, int block,
                   uint64_t seed, uint64_t a0, int64_t count, int32_t* idx_out, int32_t* q_out,
                   cudaStream_t s);
void launch_accept(const int32_t* q, const int32_t* idx, int64_t count, int32_t min_count,
                   int block, uint64_t a0, int32_t* blockcnt, SelState* st, uint64_t T,
                   uint64_t* t_attempt, int32_t* t_q, int32_t* t_idx, cudaStream_t s);
// k_svd.cu
size_t svd_smem_fixed(int64_t cmw, bool m2);
void launch_svd(const SvdArgs& a, bool m2, int grid, size_t smem, cudaStream_t s);
int svd_occupancy(bool m2, size_t smem);
bool launch_svd_warp(const SvdArgs& a, int sms, cudaStream_t s);  // row branch, k <= 9
int64_t svd_warp_lcap(int K, int64_t Lest, int64_t cmw);
// k_gram.cu
int gram_cols_per_lane(int R);
int gram_ctas_per_sm(int R);
void launch_gram(const GramArgs& a, int ntiles, cudaStream_t s);
void launch_gram_reduce(const double* P, int nslices, int64_t npad, int64_t n, const int* cnt,
                        double* G, cudaStream_t s);
// k_gram_i8.cu
int gram_i8_slices();
int64_t gram_i8_kmax();
void gram_i8_tiles(int64_t npad, std::vector<int2>& t);
cudaError_t launch_gram_i8(const GramI8Args& a, int sms, cudaStream_t s);
// k_eig.cu
int eig_part_width(int b);
cudaError_t launch_eig(const EigArgs& a, int grid, cudaStream_t s);
int eig_max_grid();
void launch_sign_fix(double* V, int64_t n, int r, cudaStream_t s);
void launch_zero_rows(const double* G, int64_t n, const int* cnt, int* out, cudaStream_t s);
// k_dropin.cu (drop-in header utilities, one call at a time)
void launch_sample_one(const uint32_t* bits, int64_t stride, int64_t nwords, int64_t pool, int count, uint64_t seed,
                       uint64_t index, int32_t* drawn, uint32_t* words, int32_t* kept, int64_t* nkept,
                       cudaStream_t s);
size_t small_svd_scratch_doubles(int p, int q);
void launch_small_svd(const double* S, int p, int q, int ell, double* scratch, double* zeta, double* sv,
                      cudaStream_t s);
void launch_gram_update(double* G, int64_t n, const double* X, int64_t nvec, const double* G2, cudaStream_t s);
// k_normal_i8.cu: stage 5's normal matrices on the tensor cores
struct NormalI8Args {
  const uint32_t* bits;  // m x nwp row-major mask words
  int64_t m, n, nwp;
  const double* V;       // n x r basis
  int r;
  int8_t* Bq;            // normal_i8_bq_bytes(r, n) scratch: the basis products' int8 digits
  double* Apre;          // m x r(r+1)/2 packed upper normal matrices (output)
  int b_resident;        // set by the launcher: B loaded once per CTA
};
size_t normal_i8_bq_bytes(int r, int64_t n);
cudaError_t launch_normal_i8(const NormalI8Args& a, int sms, cudaStream_t s);
// k_solve_u.cu
void launch_solve_u(const SolveUArgs& a, cudaStream_t s);
// returns the launches made
int launch_sum_rows(const double* v, int64_t n, double* out, cudaStream_t s, unsigned* counter = nullptr);
void launch_residual(const double* Y, const uint32_t* bitsR, int64_t m, int64_t n, int64_t nwp,
                     const double* U, const double* V, int r, double* rowres, cudaStream_t s);

}  // namespace rsmk
