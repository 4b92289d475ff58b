// k_eig.cu -- stage 4: the r minor eigenvectors of the n x n accumulator.
//
// Reference: solve_v (solver.cpp:15-62, paths relative to
// /root/reference/proj) calls LAPACKE_dsyev for the full spectrum, applies
// the rank gate on w > tol * lambda_max and returns the r eigenvectors of
// the smallest eigenvalues, sign-fixed. Here a single cooperative persistent
// kernel runs Chebyshev-filtered block subspace iteration (Zhou & Saad's
// scaled filter) aimed at the low end of the PSD spectrum:
//   * ub = ||G||_inf bounds the spectrum from above;
//   * a block of b >= r+2 vectors is filtered with a degree-d Chebyshev
//     polynomial damping [a, ub] (a = largest Ritz value of the block,
//     d chosen so the amplification stays below EigArgs::amp = 1e10: CholQR2
//     with its shifted retry keeps such blocks orthonormal, and the larger
//     degree saves an outer round at configs 1, 3 and 4),
//     re-orthonormalised by CholQR2 and Rayleigh-Ritz projected;
//   * it stops when the residuals of the r+1 lowest Ritz pairs fall below
//     1e-12 ub, which makes the r+1 lowest Ritz values the eigenvalues the
//     rank gate needs and the first r Ritz vectors the basis;
//   * one extra column runs a plain power iteration for lambda_max (used only
//     in the rank-gate threshold tol * lambda_max).
// G is read from L2 by every matvec (each CTA owns a contiguous row block;
// the iterate is staged through shared memory in 64-row chunks). All grid
// reductions write per-CTA partials and every CTA sums them in the same
// fixed order, so the result is bitwise reproducible. When n <= 16 the block
// is the whole space and a single Rayleigh-Ritz step is the exact
// eigendecomposition.
#include <algorithm>
#include <cooperative_groups.h>

#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace cg = cooperative_groups;

namespace rsmk {

using namespace rsmd;

namespace {

constexpr int ET = 256;        // threads per CTA
constexpr int BMAX = 16;       // max block size
constexpr int LDM = BMAX + 1;  // + power column
constexpr int DYN_BYTES = 212 * 1024;  // dynamic shared memory: staged iterate (+ the CTA's rows of G)

struct EigShared {
  double pad0;
  double H[BMAX * BMAX];
  double S[BMAX * BMAX];
  double red[LDM * (LDM + 1) / 2 + 2 * LDM + 8];
  double theta[BMAX];
  double dinv[BMAX];  // reciprocal diagonal of the Cholesky factor in S
  double cs[64];
  int pairs[64];
  int flag[4];
  double red2[(ET / 32) * 34];  // matvec cross-warp partials
  unsigned long long xbar;      // mbarrier of the iterate's bulk copies
};

__device__ __forceinline__ int pw_of(int b) { return (b + 1) * (b + 2) / 2 + 2 * (b + 1) + 8; }

// Y(rows) = G * X, ncol <= NC columns, leading dimension ld. The CTA's rows
// are taken in pairs; each pair gets 8/npairs warps that split the k range,
// and a lane accumulates both rows x all columns over its k's in registers
// (every x element is loaded once per pair, every G element once). Partials
// are reduced by recursive halving within the warp and in a fixed order
// across the k-split warps, so Y is bitwise reproducible. gs holds the CTA's
// G rows in shared memory (nullptr: read them from global / L2); X is read
// with coherent loads (it was written by other CTAs before the grid sync).
template <int NC>
__device__ void matvec(const EigArgs& a, const double* __restrict__ Xin, double* __restrict__ Yout,
                       double* __restrict__ Yown, int ncol, int ld, int row_lo, int row_hi, const double* gs,
                       double* xs, EigShared& sh, unsigned& xphase) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = a.n;
  const int npair = (row_hi - row_lo + 1) / 2;
  constexpr int W = ET / 32;
  const int kc = a.kc;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&sh.xbar);
  for (int pb = 0; pb < npair; pb += W) {
    const int np = (npair - pb) < W ? (npair - pb) : W;
    const int wk = W / np;  // warps per pair
    const int pi = warp / wk, ks = warp % wk;
    double v[32];  // [row][col] for cols 0..15
    double ext[2] = {0.0, 0.0};  // col 16
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = 0.0;
    const int i0 = row_lo + 2 * (pb + pi);
    const bool act = pi < np;
    const bool has1 = act && i0 + 1 < row_hi;
    // the second row of an odd tail re-reads the first; its sums are dropped
    const double* g0 = gs ? gs + (int64_t)(i0 - row_lo) * n : a.G + (int64_t)i0 * n;
    const double* g1 = has1 ? g0 + n : g0;
    for (int64_t k0 = 0; k0 < n; k0 += kc) {
      const int kn = (int)((n - k0) < kc ? (n - k0) : kc);
      __syncthreads();  // the previous chunk (or matvec) is done with xs
      if (tid == 0) {
        // X was written by other CTAs before the grid sync (generic proxy);
        // order those writes before the bulk copy's (async proxy) reads
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        const unsigned bytes = (unsigned)(((int64_t)kn * ld + 1) / 2 * 16);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                (unsigned)__cvta_generic_to_shared(xs)),
            "l"(Xin + k0 * ld), "r"(bytes), "r"(bar)
            : "memory");
      }
      {
        unsigned done = 0;
        do {
          asm volatile(
              "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
              : "=r"(done)
              : "r"(bar), "r"(xphase)
              : "memory");
        } while (!done);
        xphase ^= 1u;
      }
      if (act) {
        // NC columns are read per row regardless of ncol (xs is padded;
        // products in columns >= ncol are never written out)
        const int kb = kn * ks / wk, ke = kn * (ks + 1) / wk;
        auto body = [&](auto ldg) {
#pragma unroll 2
          for (int k = kb + lane; k < ke; k += 32) {
            const double* x = xs + (int64_t)k * ld;
            double xv[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) xv[j] = x[j];
            const double ga = ldg(g0 + k0 + k);
            const double gb = ldg(g1 + k0 + k);
#pragma unroll
            for (int j = 0; j < NC && j < 16; ++j) {
              v[j] = fma(ga, xv[j], v[j]);
              v[16 + j] = fma(gb, xv[j], v[16 + j]);
            }
            if (NC > 16) {
              ext[0] = fma(ga, xv[NC > 16 ? 16 : 0], ext[0]);
              ext[1] = fma(gb, xv[NC > 16 ? 16 : 0], ext[1]);
            }
          }
        };
        if (gs) body([](const double* p) { return *p; });
        else body([](const double* p) { return __ldg(p); });
      }
    }
    warp_reduce_halving<32>(v, lane);  // lane l: value l = (row l/16, col l%16)
    if (NC > 16) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ext[0] += __shfl_xor_sync(0xffffffffu, ext[0], o);
        ext[1] += __shfl_xor_sync(0xffffffffu, ext[1], o);
      }
    }
    double* red2 = sh.red2;
    red2[warp * 34 + lane] = v[0];
    if (lane < 2) red2[warp * 34 + 32 + lane] = ext[lane & 1];
    __syncthreads();
    if (act && ks == 0) {
      double s = 0.0;
      for (int q = 0; q < wk; ++q) s += red2[(pi * wk + q) * 34 + lane];
      const int row = i0 + (lane >> 4), col = lane & 15;
      if (col < ncol && (lane < 16 || has1)) {
        Yout[(int64_t)row * ld + col] = s;
        Yown[(row - row_lo) * ld + col] = s;
      }
      if (NC > 16 && ncol > 16 && lane < 2 && (lane == 0 || has1)) {
        double e = 0.0;
        for (int q = 0; q < wk; ++q) e += red2[(pi * wk + q) * 34 + 32 + lane];
        Yout[(int64_t)(i0 + lane) * ld + 16] = e;
        Yown[(i0 + lane - row_lo) * ld + 16] = e;
      }
    }
    __syncthreads();
  }
}

// partial of value e of this CTA for reduction buffer buf; layout [buf][e][cta]
// so one warp reads the grid's partials of a value with coalesced loads
__device__ __forceinline__ double* pslot(const EigArgs& a, int buf, int pw, int e) {
  return a.part + ((size_t)buf * pw + e) * gridDim.x + blockIdx.x;
}

// grid reduction of cnt values from part[buf] into sh.red; op 0 = sum, 1 = max.
// One warp per value: lanes sum a strided subset of the CTAs' partials, then a
// butterfly; the order is fixed, so every CTA gets bitwise identical results.
__device__ void grid_reduce(const EigArgs& a, cg::grid_group& grid, int buf, int cnt, int op,
                            int pw, EigShared& sh) {
  grid.sync();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nc = (int)gridDim.x;  // <= 32 * 5
  constexpr int VU = 4;            // values per warp per round (all loads in flight)
  for (int e0 = warp; e0 < cnt; e0 += (ET / 32) * VU) {
    double s[VU];
#pragma unroll
    for (int u = 0; u < VU; ++u) {
      const int e = e0 + u * (ET / 32);
      s[u] = op ? -1.0 : 0.0;
      if (e < cnt) {
        const double* base = a.part + ((size_t)buf * pw + e) * nc;
#pragma unroll
        for (int cc = 0; cc < 5; ++cc) {
          const int c = lane + 32 * cc;
          if (c < nc) {
            const double v = base[c];
            s[u] = op ? fmax(s[u], v) : s[u] + v;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < VU; ++u) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, s[u], o);
        s[u] = op ? fmax(s[u], t) : s[u] + t;
      }
      const int e = e0 + u * (ET / 32);
      if (lane == 0 && e < cnt) sh.red[e] = s[u];
    }
  }
  __syncthreads();
}

// local Gram partial of columns [0, nc) of X over own rows -> part[buf]; plus
// optional squared norm of column pc (pc < 0: none) at index nc*(nc+1)/2
__device__ void gram_partial(const EigArgs& a, const double* Xo, int nc, int ld, int pc, int nr, int buf,
                             int pw) {
  const int P = nc * (nc + 1) / 2;
  for (int p = threadIdx.x; p < P + 1; p += ET) {
    int i = 0, j = 0;
    if (p < P) {
      int rem = p;
      while (rem >= nc - i) { rem -= nc - i; ++i; }
      j = i + rem;
    } else {
      if (pc < 0) continue;
      i = j = pc;
    }
    double s = 0.0;
    for (int lr = 0; lr < nr; ++lr) s += Xo[lr * ld + i] * Xo[lr * ld + j];
    *pslot(a, buf, pw, p) = s;
  }
}

// Whole CTA (ET = 16 x 16 threads): Cholesky of the nc x nc matrix (nc <= 16)
// given packed (upper) in sh.red; lower factor to sh.S and its reciprocal
// diagonal to sh.dinv. Thread (i, j) keeps L(i, j) in a register; per step the
// pivot's reciprocal square root and the scaled column go through sh.cs (two
// CTA barriers), then every thread updates its own entry -- the arithmetic
// and its order per entry are those of the right-looking loop (pivot d *
// rsqrt(d), column * rsqrt(d), fma(-L(i,k), L(j,k), L(i,j)) for k ascending).
// Retries with a diagonal shift when the matrix is not numerically positive.
// (One warp working in shared memory took ~9 k cycles per 10 x 10 factor:
// index divisions and three warp barriers per step.)
__device__ void chol_cta(int nc, EigShared& sh, double shift0) {
  const int tid = threadIdx.x, i = tid >> 4, j = tid & 15;
  const bool live = i < nc && j <= i;
  double tr = 0.0;
  for (int k = 0; k < nc; ++k) tr += fabs(sh.red[k * nc - k * (k - 1) / 2]);
  double shift = shift0 * tr;
  const double a0 = live ? sh.red[j * nc - j * (j - 1) / 2 + (i - j)] : 0.0;
  double l = 0.0;
#pragma unroll 1
  for (int attempt = 0; attempt < 4; ++attempt) {
    l = a0 + ((live && i == j) ? shift : 0.0);
    bool ok = true;
#pragma unroll 1
    for (int k = 0; k < nc; ++k) {
      if (i == k && j == k) {
        const double d = l;
        ok = d > 0.0;
        const double inv = ok ? rsqrt_fast(d) : 0.0;
        l = ok ? d * inv : 0.0;
        sh.cs[0] = inv;
      }
      __syncthreads();
      if (live && j == k && i > k) {
        l *= sh.cs[0];
        sh.cs[1 + i] = l;
      }
      __syncthreads();
      if (live && j > k) l = fma(-sh.cs[1 + i], sh.cs[1 + j], l);
    }
    if (blockIdx.x == 0 && tid == 0) sh.flag[3] += 1;  // attempts (statistics)
    if (__syncthreads_and(ok ? 1 : 0)) break;
    shift = (shift == 0.0) ? 1e-14 * tr : shift * 100.0;
  }
  if (live) sh.S[i * BMAX + j] = l;
  if (live && i == j) sh.dinv[i] = 1.0 / l;
  __syncthreads();
}

// Whole CTA: cyclic Jacobi on the symmetric K x K matrix A (sh.H, leading
// dimension BMAX, K <= 16) with the absolute threshold 16 eps ||A||_F
// (warp_jacobi_abs's; LAPACK-level absolute eigenvalue accuracy). Thread
// (i, j) keeps A(i, j) and V(i, j) in registers with shared-memory copies the
// others read. Round-robin ordering: each step the Kp/2 pair threads form
// their rotations (Rutishauser's formulas, two rsqrt and no division), then
// every thread applies J^T A J and V J to its own entry from four (two)
// neighbours: three CTA barriers per step instead of one warp's ~1.9 k cycles
// of shuffles. The four products are summed (t1 + t4) + (t2 + t3), symmetric
// in (i, j), so A stays exactly symmetric. On return A's diagonal holds the
// eigenvalues and V (sh.S) the vectors in matching column order. Returns the
// sweep count.
__device__ int jacobi_cta(double* A, double* V, int K, EigShared& sh, int max_sweeps) {
  const int tid = threadIdx.x, i = tid >> 4, j = tid & 15;
  const int Kp = (K + 1) & ~1;
  const bool live = i < K && j < K;
  double a = live ? A[i * BMAX + j] : 0.0;
  double v = (i == j) ? 1.0 : 0.0;
  double* cs = sh.cs;      // [2 * BMAX]: c_i, sigma_i of index i's rotation
  int* part = sh.pairs;    // [BMAX]: partner of index i (itself: no rotation)
  {
    double f = warp_sum(a * a);
    if ((tid & 31) == 0) sh.red2[tid >> 5] = f;
    V[i * BMAX + j] = v;
    __syncthreads();
    f = 0.0;
    for (int w = 0; w < ET / 32; ++w) f += sh.red2[w];
    cs[2 * BMAX] = fmax(16.0 * 2.220446049250313e-16 * sqrt(f), 1e-300);
    __syncthreads();
  }
  const double thr = cs[2 * BMAX];
  if (K < 2) return 0;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (!__syncthreads_or((live && i < j && fabs(a) > thr) ? 1 : 0)) break;
#pragma unroll 1
    for (int step = 0; step < Kp - 1; ++step) {
      if (tid < Kp / 2) {
        const int x = (tid == 0) ? 0 : ((tid - 1 + step) % (Kp - 1)) + 1;
        const int y = ((Kp - 2 - tid + step) % (Kp - 1)) + 1;
        const int p = x < y ? x : y, q = x < y ? y : x;
        double c = 1.0, sn = 0.0;
        if (q < K) {
          const double off = A[p * BMAX + q];
          if (fabs(off) > thr) {
            const double dd = A[q * BMAX + q] - A[p * BMAX + p], ee = 2.0 * off;
            const double r2 = fma(dd, dd, ee * ee);
            const double rr = r2 * rsqrt_fast(r2);
            const double w = rr + fabs(dd);
            const double g = rsqrt_fast(2.0 * rr * w);
            c = w * g;
            sn = (dd >= 0.0 ? ee : -ee) * g;
          }
          part[p] = sn != 0.0 ? q : p;
          part[q] = sn != 0.0 ? p : q;
          cs[2 * p] = c;
          cs[2 * p + 1] = -sn;  // x_p' = c x_p - s x_q
          cs[2 * q] = c;
          cs[2 * q + 1] = sn;   // x_q' = s x_p + c x_q
        } else {
          part[p] = p;
          cs[2 * p] = 1.0;
          cs[2 * p + 1] = 0.0;
        }
      }
      __syncthreads();
      double an = a, vn = v;
      if (live) {
        const int pi = part[i], pj = part[j];
        const double ci = cs[2 * i], si = cs[2 * i + 1], cj = cs[2 * j], sj = cs[2 * j + 1];
        if (pi != i || pj != j) {
          const double t1 = __dmul_rn(__dmul_rn(ci, cj), a);
          const double t2 = __dmul_rn(__dmul_rn(ci, sj), A[i * BMAX + pj]);
          const double t3 = __dmul_rn(__dmul_rn(si, cj), A[pi * BMAX + j]);
          const double t4 = __dmul_rn(__dmul_rn(si, sj), A[pi * BMAX + pj]);
          an = __dadd_rn(__dadd_rn(t1, t4), __dadd_rn(t2, t3));
          if (j == pi && i != j) an = 0.0;  // the rotated pair's off-diagonal entry
        }
        if (pj != j) vn = fma(cj, v, sj * V[i * BMAX + pj]);
      }
      __syncthreads();
      if (live) {
        A[i * BMAX + j] = an;
        V[i * BMAX + j] = vn;
      }
      a = an;
      v = vn;
      __syncthreads();
    }
  }
  return sweep;
}

// X(own rows) <- X R^{-1}, R = L^T with L in sh.S (smem copy and global)
__device__ void apply_rinv(double* X, double* Xo, int nc, int ld, int row_lo, int nr, EigShared& sh) {
  for (int lr = threadIdx.x; lr < nr; lr += ET) {
    double y[BMAX];
    double* x = Xo + lr * ld;
    double* xg = X + (int64_t)(row_lo + lr) * ld;
#pragma unroll
    for (int j = 0; j < BMAX; ++j) {
      if (j < nc) {
        double s = x[j];
#pragma unroll
        for (int i = 0; i < BMAX; ++i)
          if (i < j) s -= y[i] * sh.S[j * BMAX + i];
        y[j] = s * sh.dinv[j];
      }
    }
#pragma unroll
    for (int j = 0; j < BMAX; ++j)
      if (j < nc) {
        x[j] = y[j];
        xg[j] = y[j];
      }
  }
}

__device__ void cholqr(const EigArgs& a, cg::grid_group& grid, double* X, double* Xo, int nc, int ld, int pc,
                       int row_lo, int nr, int& buf, int pw, EigShared& sh) {
  const bool tme = blockIdx.x == 0 && threadIdx.x == 0;
  long long t0 = clock64();
  gram_partial(a, Xo, nc, ld, pc, nr, buf, pw);
  long long t1 = clock64();
  const int P = nc * (nc + 1) / 2;
  grid_reduce(a, grid, buf, P + 1, 0, pw, sh);
  long long t2 = clock64();
  buf ^= 1;
  // the first pass after a filter (pc >= 0) meets a Gram conditioned up to
  // the filter's amplification: it may start from the shift its retry would reach
  chol_cta(nc, sh, pc >= 0 ? a.shift0 : 0.0);
  long long t3 = clock64();
  apply_rinv(X, Xo, nc, ld, row_lo, nr, sh);
  if (tme) {
    a.dstat[16] += (double)(t1 - t0);
    a.dstat[17] += (double)(t2 - t1);
    a.dstat[18] += (double)(t3 - t2);
    a.dstat[19] += (double)(clock64() - t3);
  }
  if (pc >= 0) {
    const double nrm = sqrt(sh.red[P]);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int lr = threadIdx.x; lr < nr; lr += ET) {
      const double v = Xo[lr * ld + pc] * inv;
      Xo[lr * ld + pc] = v;
      X[(int64_t)(row_lo + lr) * ld + pc] = v;
    }
  }
  __syncthreads();
}

// CTA 0, thread 0, last: Ritz values, statistics and status straight into the
// caller's pinned host block (no device->host copies on the stream):
// [0, 32) w, [32, 64) dstat, [64, 68) istat
__device__ void publish(const EigArgs& a) {
  if (!a.hout) return;
  for (int j = 0; j < a.b; ++j) a.hout[j] = a.w[j];
  for (int i = 0; i < 32; ++i) a.hout[32 + i] = a.dstat[i];
  int* hi = reinterpret_cast<int*>(a.hout + 64);
  for (int i = 0; i < 8; ++i) hi[i] = a.istat[i];
}

}  // namespace

template <int NC>
__global__ void __launch_bounds__(ET, 1) k_eig(EigArgs a) {
  cg::grid_group grid = cg::this_grid();
  const long long t_start = clock64();
  __shared__ EigShared sh;
  if (blockIdx.x == 0 && threadIdx.x < 16) a.dstat[16 + threadIdx.x] = 0.0;
  if (threadIdx.x == 0) sh.flag[3] = 0;
  extern __shared__ __align__(16) double dyn[];
  const int tid = threadIdx.x;
  const int64_t n = a.n;
  const int b = a.b, r = a.r, ld = b + 1, pcol = b;
  const int pw = pw_of(b);
  const int row_lo = (int)((int64_t)blockIdx.x * a.rows_per_cta < n ? blockIdx.x * a.rows_per_cta : n);
  const int row_hi = (int)((int64_t)(blockIdx.x + 1) * a.rows_per_cta < n ? (blockIdx.x + 1) * a.rows_per_cta : n);
  int buf = 0;
  int matvecs = 0;
  const bool full = (b >= n);  // block = whole space
  if (a.zero_rows && *a.zero_rows > r) {
    // more than r exact zero eigenvalues: the rank gate fails (solver.cpp:34-39)
    if (blockIdx.x == 0 && tid == 0) {
      a.istat[0] = 3;
      a.istat[3] = 0;
      a.istat[4] = 0;
      for (int i = 0; i < 16; ++i) a.dstat[i] = 0.0;
      publish(a);
    }
    return;
  }
  // dynamic shared memory: [own rows of X, Y, Z][G rows when resident][iterate chunk]
  const int nr = row_hi - row_lo;
  const int own = ((a.rows_per_cta * ld) + 1) & ~1;
  double* Xo = dyn;
  double* Yo = dyn + own;
  double* Zo = dyn + 2 * own;
  double* Wo = dyn + 3 * own;  // scratch
  double* gdyn = dyn + 4 * own;
  const double* gs = nullptr;
  double* xs = gdyn + (a.gres ? (((int64_t)a.rows_per_cta * n + 1) & ~int64_t(1)) : 0);
  unsigned xphase = 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&sh.xbar)),
                 "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (a.gres) {
    // the CTA's rows of G (written by the previous kernel): one bulk copy on
    // the iterate's mbarrier when n is even (16-byte rows), else a plain loop
    const int64_t tot = (int64_t)(row_hi - row_lo) * n;
    const double* src = a.G + (int64_t)row_lo * n;
    if ((n & 1) == 0 && tot > 0) {
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&sh.xbar);
      if (tid == 0) {
        const unsigned bytes = (unsigned)(tot * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                (unsigned)__cvta_generic_to_shared(gdyn)),
            "l"(src), "r"(bytes), "r"(bar)
            : "memory");
      }
      unsigned done = 0;
      do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(xphase)
            : "memory");
      } while (!done);
      xphase ^= 1u;
    } else {
      for (int64_t e = tid; e < tot; e += ET) gdyn[e] = __ldg(src + e);
      __syncthreads();
    }
    gs = gdyn;
  }

  // ---- ub: an upper bound of the spectrum ----
  // With the accumulator's structure G = diag(count) - sum E V V^T E^T (a PSD
  // matrix subtracted from a diagonal), lambda_max(G) <= max count: a tight,
  // rigorous bound (a.cnt, up to rounding of the PSD part). Otherwise (a G
  // supplied by the caller) ||G||_inf.
  {
    double mx = 0.0;
    const int warp = tid >> 5, lane = tid & 31;
    if (a.cnt) {
      for (int row = row_lo + tid; row < row_hi; row += ET) mx = fmax(mx, (double)a.cnt[row]);
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    } else {
      for (int row = row_lo + warp; row < row_hi; row += ET / 32) {
        double s = 0.0;
        for (int64_t k = lane; k < n; k += 32) s += fabs(__ldg(a.G + (int64_t)row * n + k));
        s = warp_sum(s);
        mx = fmax(mx, s);
      }
    }
    if (lane == 0) sh.red[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double m2 = 0.0;
      for (int w = 0; w < ET / 32; ++w) m2 = fmax(m2, sh.red[w]);
      *pslot(a, buf, pw, 0) = m2;
    }
    grid_reduce(a, grid, buf, 1, 1, pw, sh);
    buf ^= 1;
  }
  double ub = sh.red[0] > 0.0 ? sh.red[0] * (1.0 + 1e-10) : 1.0;  // rigorous

  // ---- initial block: identity (full) or hashed pseudo-random columns ----
  double* X = a.X;
  double* Y = a.Y;
  double* Z = a.Z;
  for (int e = tid; e < nr * ld; e += ET) {
    const int lr = e / ld, j = e % ld, row = row_lo + lr;
    double v;
    if (full) v = (j == row) ? 1.0 : 0.0;
    else v = (double)(mix(0x51ed270b27c3e1a5ull ^ ((uint64_t)row * 131 + j)) >> 11) * 0x1.0p-53 - 0.5;
    if (j == pcol) v = 1.0 + 0.01 * ((double)(mix(0xabcdefull + row) >> 11) * 0x1.0p-53);
    X[(int64_t)row * ld + j] = v;
    Xo[e] = v;
  }
  __syncthreads();
  // the random start block is well conditioned: one CholQR orthonormalises it
  if (!full && a.init_cq) cholqr(a, grid, X, Xo, b, ld, pcol, row_lo, nr, buf, pw, sh);

  double acut = 0.5 * ub;
  double maxres = 0.0, lmax = 0.0;
  int outer = 0, status = 1;
  // phase clocks (CTA 0, thread 0): [0] filter, [1] CholQR2, [2] RR matvec+reduce,
  // [3] small eigensolve, [4] rotate+residual, [5] setup before the loop
  long long tacc[6] = {0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
  const long long t_setup = tlast - t_start;  // G rows to smem, ub, initial CholQR
  const bool tme = blockIdx.x == 0 && tid == 0;
  long long jac_sweeps = 0, jac_cyc = 0, mv_cyc = 0, sync_cyc = 0;
#define EIG_T(i)                          \
  do {                                    \
    if (tme) {                            \
      const long long t_ = clock64();     \
      tacc[i] += t_ - tlast;              \
      tlast = t_;                         \
    }                                     \
  } while (0)
  EIG_T(5);
  for (; outer < a.max_outer; ++outer) {
    {
      // ---- Chebyshev filter of degree d on [acut, ub], normalised at 0, then
      // CholQR2 and the Rayleigh-Ritz product, as ONE loop over matvec steps
      // (a single inlined copy of the matvec: the kernel is large enough for
      // instruction fetch to show): step 1 forms Y = (G X - c X) sigma / e
      // from X, steps 2..d the three-term recurrence from Y and X (the block
      // rotates (X, Y, Z) <- (Y, Z, X) after each), step d + 1 is Z = G X of
      // the re-orthonormalised block. full: no filter, d = 0 ----
      double e = 1.0, c = 0.0, sigma = 0.0, tau = 0.0;
      int d = 0;
      if (!full) {
        e = 0.5 * (ub - acut);
        c = 0.5 * (ub + acut);
        const double x0 = fabs(c / e);
        const double growth = x0 + sqrt(x0 * x0 - 1.0);
        d = (int)floor(log(a.amp) / log(growth));
        d = d < 2 ? 2 : (d > a.dmax ? a.dmax : d);
        sigma = e / (0.0 - c);
        tau = 2.0 / sigma;
      }
#pragma unroll 1
      for (int it = 1; it <= d + 1; ++it) {
        const bool first = it == 1, rr = it == d + 1;
        if (rr && !full) {
          // filtered block is in Y
          { double* t = X; X = Y; Y = t; t = Xo; Xo = Yo; Yo = t; }
          __syncthreads();
          EIG_T(0);
#pragma unroll 1
          for (int pass = 0; pass < 2; ++pass)  // CholQR2 (one inlined copy)
            cholqr(a, grid, X, Xo, b, ld, pass == 0 ? pcol : -1, row_lo, nr, buf, pw, sh);
          EIG_T(1);
        }
        const long long t0 = clock64();
        grid.sync();  // the iterate (X at steps 1 and d + 1, Y between) is complete
        const long long t1 = clock64();
        matvec<NC>(a, (first || rr) ? X : Y, Z, Zo, ld, ld, row_lo, row_hi, gs, xs, sh, xphase);
        if (tme && !first && !rr) {
          sync_cyc += t1 - t0;
          mv_cyc += clock64() - t1;
        }
        ++matvecs;
        if (rr) break;
        if (first) {
          for (int q = tid; q < nr * ld; q += ET) {
            const int j = q % ld;
            const double y = (j == pcol) ? Zo[q] / ub : (Zo[q] - c * Xo[q]) * (sigma / e);
            Yo[q] = y;
            Y[(int64_t)row_lo * ld + q] = y;
          }
          continue;
        }
        const double sigma2 = 1.0 / (tau - sigma);
        for (int q = tid; q < nr * ld; q += ET) {
          const int j = q % ld;
          const double z = (j == pcol) ? Zo[q] / ub
                                       : (Zo[q] - c * Yo[q]) * (2.0 * sigma2 / e) - sigma * sigma2 * Xo[q];
          Zo[q] = z;
          Z[(int64_t)row_lo * ld + q] = z;
        }
        double* t = X; X = Y; Y = Z; Z = t;
        t = Xo; Xo = Yo; Yo = Zo; Zo = t;
        sigma = sigma2;
      }
    }
    // ---- Rayleigh-Ritz ----
    {
      const int P = b * (b + 1) / 2;
      for (int p = tid; p < P + 2; p += ET) {
        double s = 0.0;
        if (p < P) {
          int i = 0, rem = p;
          while (rem >= b - i) { rem -= b - i; ++i; }
          const int j = i + rem;
          for (int lr = 0; lr < nr; ++lr) s += Xo[lr * ld + i] * Zo[lr * ld + j];
        } else if (p == P) {
          for (int lr = 0; lr < nr; ++lr) s += Xo[lr * ld + pcol] * Zo[lr * ld + pcol];
        } else {
          for (int lr = 0; lr < nr; ++lr) s += Xo[lr * ld + pcol] * Xo[lr * ld + pcol];
        }
        *pslot(a, buf, pw, p) = s;
      }
      grid_reduce(a, grid, buf, P + 2, 0, pw, sh);
      buf ^= 1;
      if (sh.red[P + 1] > 0.0) lmax = sh.red[P] / sh.red[P + 1];
      // symmetric H from the packed upper triangle
      for (int e2 = tid; e2 < b * b; e2 += ET) {
        int i = e2 / b, j = e2 % b;
        if (i > j) { const int t = i; i = j; j = t; }
        const int p = i * b - i * (i - 1) / 2 + (j - i);
        sh.H[(e2 / b) * BMAX + (e2 % b)] = sh.red[p];
      }
      __syncthreads();
      EIG_T(2);
      // Probe round (first outer iteration): the filtered block cannot have
      // converged yet, and the next filter needs only the top Ritz value for
      // its damping interval -- a Rayleigh quotient of H by power iteration
      // (a lower bound: the interval only widens) instead of the full b x b
      // eigensolve, rotation and residuals. Subspace iteration depends on the
      // span alone, so the CholQR basis carries on unrotated.
      if (a.rr0_probe && !full && outer == 0 && outer + 1 < a.max_outer) {
        if (tid < 32) {
          const int l = tid;
          double x = l < b ? 1.0 : 0.0;
          double yv = 0.0;
          for (int itp = 0; itp < a.probe_its; ++itp) {
            yv = 0.0;
            for (int j = 0; j < b; ++j) {
              const double xj = __shfl_sync(0xffffffffu, x, j);
              if (l < b) yv = fma(sh.H[l * BMAX + j], xj, yv);
            }
            const double nn = warp_sum(yv * yv);
            x = nn > 0.0 ? yv * rsqrt(nn) : x;
          }
          yv = 0.0;
          for (int j = 0; j < b; ++j) {
            const double xj = __shfl_sync(0xffffffffu, x, j);
            if (l < b) yv = fma(sh.H[l * BMAX + j], xj, yv);
          }
          const double te = warp_sum(x * yv);
          if (l == 0) sh.theta[b - 1] = te;
        }
        __syncthreads();
        const double te = sh.theta[b - 1];
        if (lmax > 0.0 && !a.cnt) ub = fmin(ub, fmax(1.1 * lmax, 1.1 * te));
        acut = te;
        if (!(acut < 0.999 * ub)) acut = 0.999 * ub;
        if (acut <= 0.0) acut = 1e-6 * ub;
        continue;
      }
      {
        const long long tj = clock64();
        const int sw = jacobi_cta(sh.H, sh.S, b, sh, 60);
        if (tme) {
          jac_sweeps += sw;
          jac_cyc += clock64() - tj;
        }
        // ascending order (ties: the lower index first, as a stable selection
        // sort): eigenpair j moves to its rank
        const int i = tid >> 4, j = tid & 15;
        if (tid < b) {
          const double th = sh.H[tid * BMAX + tid];
          int rank = 0;
          for (int k = 0; k < b; ++k) {
            const double tk = sh.H[k * BMAX + k];
            rank += (tk < th || (tk == th && k < tid)) ? 1 : 0;
          }
          sh.theta[rank] = th;
          sh.pairs[tid] = rank;
        }
        const double x = (i < b && j < b) ? sh.S[i * BMAX + j] : 0.0;
        __syncthreads();
        if (i < b && j < b) sh.S[i * BMAX + sh.pairs[j]] = x;
      }
      __syncthreads();
    }
    EIG_T(3);
    // X <- X S, Z <- Z S (own rows); residual partials
    {
      // X <- X S (own rows); the rotated Z only enters the residuals
      // ||Z S_j - theta_j X S_j||^2, so it is not stored. New X values and the
      // squared residual terms go to scratch first (X is still being read).
      for (int q = tid; q < nr * b; q += ET) {
        const int lr = q / b, j = q % b;
        double sx = 0.0, sz = 0.0;
        for (int i = 0; i < b; ++i) {
          const double sij = sh.S[i * BMAX + j];
          sx = fma(Xo[lr * ld + i], sij, sx);
          sz = fma(Zo[lr * ld + i], sij, sz);
        }
        const double d = sz - sh.theta[j] * sx;
        Yo[lr * ld + j] = sx;
        Wo[lr * ld + j] = d * d;
      }
      __syncthreads();
      for (int q = tid; q < nr * b; q += ET) {
        const int lr = q / b, j = q % b;
        const double v = Yo[lr * ld + j];
        Xo[lr * ld + j] = v;
        X[(int64_t)(row_lo + lr) * ld + j] = v;
      }
      for (int j = tid; j < b; j += ET) {
        double s2 = 0.0;
        for (int lr = 0; lr < nr; ++lr) s2 += Wo[lr * ld + j];
        *pslot(a, buf, pw, j) = s2;
      }
      grid_reduce(a, grid, buf, b, 0, pw, sh);
      buf ^= 1;
    }
    EIG_T(4);
    // the r wanted pairs must converge; the (r+1)-th Ritz value only has to be
    // resolved against the rank-gate thresholds: either converged too, or
    // clearly above 10 tol lambda_max (eigenvalues that small are amplified by
    // the filter exactly like the wanted ones, so they would be in the block)
    // Coverage certificate: Ritz values bound the eigenvalues from above
    // (lambda_k <= theta_k, Rayleigh-Ritz interlacing), and the power-column
    // estimate bounds lambda_max from below, so theta_{r+1} <= tol * lmax
    // proves at least r+1 eigenvalues at or below the reference's threshold:
    // the rank gate of solver.cpp:34-39 fails, whatever the rest of the
    // spectrum (e.g. columns no trial covered give exact zero eigenvalues).
    if (!full && r < b && lmax > 0.0 && sh.theta[r] <= a.tol * lmax) {
      status = 3;
      ++outer;
      break;
    }
    maxres = 0.0;
    for (int j = 0; j < r && j < b; ++j) maxres = fmax(maxres, sqrt(sh.red[j]));
    bool sep = true;
    if (r < b) {
      const double rr = sqrt(sh.red[r]);
      const double gate = 10.0 * a.tol * fmax(lmax, 0.0);
      sep = rr <= 1e-12 * ub || (sh.theta[r] - rr > 1e3 * gate && sh.theta[r] - rr > 1e-8 * ub);
    }
    // 1e-13 ub: one filter pass gains ~6 digits, so this rarely costs an extra
    // pass, and it keeps the basis (and a noiseless e) at dsyev's accuracy
    if (full || (maxres <= 1e-13 * ub && sep)) { status = 0; ++outer; break; }
    // tighten the damping interval's top: ||G||_inf can exceed lambda_max
    // several-fold; the power column's Rayleigh quotient (a lower bound after
    // >= 8 matvecs) with a 10% margin is used instead. A mild underestimate
    // only amplifies the top eigenvalues by T_d(1+eps), negligible next to the
    // wanted end's T_d(|x0|).
    if (outer == 0 && lmax > 0.0 && !a.cnt) ub = fmin(ub, fmax(1.1 * lmax, 1.1 * sh.theta[b - 1]));
    acut = sh.theta[b - 1];
    if (!(acut < 0.999 * ub)) acut = 0.999 * ub;
    if (acut <= 0.0) acut = 1e-6 * ub;
  }
  if (status == 1 && maxres <= 1e-9 * ub) status = 0;  // converged to a looser bound
  const long long t_loop_end = clock64();
  // ---- outputs, sign-fixed (solver.cpp:47-60): each column's largest-
  // magnitude entry made positive, the first index winning ties. Per-CTA
  // candidates (signed value, row) -> partials, one grid sync, every CTA
  // scans the candidates in CTA order (rows ascend with the CTA index) ----
  {
    __shared__ double flip[BMAX];
    if (tid < r) {
      double best = -1.0, val = 0.0;
      int arg = row_lo;
      for (int lr = 0; lr < nr; ++lr) {
        const double x = Xo[lr * ld + tid];
        if (fabs(x) > best) { best = fabs(x); val = x; arg = row_lo + lr; }
      }
      *pslot(a, buf, pw, tid) = nr > 0 ? val : 0.0;
      *pslot(a, buf, pw, r + tid) = nr > 0 ? (double)arg : -1.0;
    }
    grid.sync();
    {
      // warp j scans column j's candidates: lane l takes a contiguous run of
      // CTAs (first maximum within it), then an arg-max butterfly in which the
      // lower CTA index wins ties -- the first index over the whole column
      const int warp = tid >> 5, lane = tid & 31;
      const int nc = (int)gridDim.x, per = (nc + 31) / 32;
      for (int j = warp; j < r; j += ET / 32) {
        double best = -1.0, val = 0.0;
        int at = nc;
        for (int cta = lane * per; cta < nc && cta < (lane + 1) * per; ++cta) {
          const double x = a.part[((size_t)buf * pw + j) * nc + cta];
          const double id = a.part[((size_t)buf * pw + r + j) * nc + cta];
          if (id >= 0.0 && fabs(x) > best) { best = fabs(x); val = x; at = cta; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
          const double v2 = __shfl_xor_sync(0xffffffffu, val, o);
          const int a2 = __shfl_xor_sync(0xffffffffu, at, o);
          if (b2 > best || (b2 == best && a2 < at)) { best = b2; val = v2; at = a2; }
        }
        if (lane == 0) flip[j] = val < 0.0 ? -1.0 : 1.0;
      }
    }
    __syncthreads();
    for (int q = tid; q < nr * r; q += ET) {
      const int lr = q / r, j = q % r;
      a.V[(int64_t)(row_lo + lr) * r + j] = flip[j] * Xo[lr * ld + j];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    for (int j = 0; j < b; ++j) a.w[j] = sh.theta[j];
    a.istat[0] = status;
    a.istat[3] = outer;
    a.istat[4] = matvecs;
    a.dstat[0] = full ? sh.theta[b - 1] : lmax;
    a.dstat[1] = ub;
    a.dstat[2] = maxres;
    for (int i = 0; i < 6; ++i) a.dstat[3 + i] = (double)tacc[i];
    a.dstat[9] = (double)jac_sweeps;
    a.dstat[10] = (double)jac_cyc;
    a.dstat[11] = (double)mv_cyc;
    a.dstat[12] = (double)sync_cyc;
    a.dstat[20] = (double)sync_cyc;  // grid syncs before the filter's matvecs
    a.dstat[21] = (double)t_setup;
    a.dstat[22] = (double)(clock64() - t_loop_end);  // sign fix + outputs
    a.dstat[23] = (double)(clock64() - t_start);
    a.dstat[24] = (double)sh.flag[3];
    publish(a);
  }
#undef EIG_T
}

// Exactly-zero rows of G (columns no trial covered: count 0 when G is our
// harvest, else rows whose n entries are all 0.0) are exact zero eigenvalues;
// more than r of them fail the reference's rank gate outright.
__global__ void k_zero_rows(const double* __restrict__ G, int64_t n, const int* __restrict__ cnt,
                            int* __restrict__ out) {
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int nw = (int)((gridDim.x * (int64_t)blockDim.x) >> 5);
  int z = 0;
  for (int64_t i = warp; i < n; i += nw) {
    bool zero;
    if (cnt) zero = cnt[i] == 0;
    else {
      bool nz = false;
      for (int64_t k = lane; k < n; k += 32) nz |= G[i * n + k] != 0.0;
      zero = !__any_sync(0xffffffffu, nz);
    }
    z += zero ? 1 : 0;
  }
  if (lane == 0 && z) atomicAdd(out, z);
}

// sign fix (solver.cpp:47-60): the largest-magnitude entry of each column is
// made positive, the first index winning ties. One warp per column.
__global__ void k_sign_fix(double* V, int64_t n, int r) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < r; c += blockDim.x >> 5) {
    double best = -1.0;
    int64_t arg = 0;
    for (int64_t i = lane; i < n; i += 32) {
      const double m = fabs(V[i * r + c]);
      if (m > best) { best = m; arg = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
    }
    const double flip = V[arg * r + c] < 0.0 ? -1.0 : 1.0;
    for (int64_t i = lane; i < n; i += 32) V[i * r + c] *= flip;
  }
}

int eig_part_width(int b) { return (b + 1) * (b + 2) / 2 + 2 * (b + 1) + 8; }

int eig_max_grid() {
  int dev = 0, sms = 0, nb = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  nb = occupancy((const void*)k_eig<17>, ET, DYN_BYTES);
  return sms * (nb > 0 ? nb : 1);
}

cudaError_t launch_eig(const EigArgs& a0, int grid, cudaStream_t s) {
  EigArgs a = a0;
  const int ld = a.b + 1;
  // the whole iterate in shared memory when it fits, else even-sized chunks;
  // the CTA's G rows stay resident when there is room next to it
  const size_t xrow = sizeof(double) * (size_t)ld;
  const size_t own = sizeof(double) * 4 * ((((size_t)a.rows_per_cta * ld) + 1) & ~(size_t)1);
  const size_t pad = sizeof(double) * 32 + own;  // own-row buffers ride along with the padding
  const size_t xfull = xrow * (size_t)a.n + pad;
  const size_t gbytes = sizeof(double) * (((size_t)a.rows_per_cta * (size_t)a.n + 1) & ~(size_t)1);
  size_t dyn;
  if (xfull <= (size_t)DYN_BYTES) {
    a.kc = (int)a.n;
    a.gres = xfull + gbytes <= (size_t)DYN_BYTES ? 1 : 0;
    dyn = xfull + (a.gres ? gbytes : 0);
  } else {
    a.gres = 0;
    a.kc = (int)(((DYN_BYTES - pad) / xrow) & ~(size_t)1);
    dyn = xrow * (size_t)a.kc + pad;
  }
  void* args[] = {(void*)&a};
  if (a.b + 1 <= 12) {
    ensure_smem((const void*)k_eig<12>, DYN_BYTES);
    return cudaLaunchCooperativeKernel((void*)k_eig<12>, dim3(grid), dim3(ET), args, dyn, s);
  }
  ensure_smem((const void*)k_eig<17>, DYN_BYTES);
  return cudaLaunchCooperativeKernel((void*)k_eig<17>, dim3(grid), dim3(ET), args, dyn, s);
}

void launch_zero_rows(const double* G, int64_t n, const int* cnt, int* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(int), s);
  int blocks = (int)std::min<int64_t>(148 * 4, (n + 7) / 8);
  k_zero_rows<<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(G, n, cnt, out);
}

void launch_sign_fix(double* V, int64_t n, int r, cudaStream_t s) {
  k_sign_fix<<<1, 512, 0, s>>>(V, n, r);
}

}  // namespace rsmk
