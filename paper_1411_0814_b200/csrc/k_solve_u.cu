// k_solve_u.cu -- stage 5: per-row masked least squares for U and the
// masked residual e.
//
// Reference: solve_u (solver.cpp:64-89, paths relative to
// /root/reference/proj) runs detail::solve_row (detail/row_solve.hpp:12-36)
// per row: gather V rows at the observed columns, complete orthogonal
// decomposition, minimum-norm solution; the row is counted as
// underdetermined when it has fewer than r observations or the basis
// restricted to them is rank deficient; an empty row gets zeros.
//
// Here one warp owns a row at a time. Each warp double-buffers its rows in
// shared memory: while row i is solved, the 16-byte cp.async copies of its
// next row (values and mask words) are in flight, so Y is streamed from HBM
// exactly once with all of a row's loads outstanding. The warp selects
// through the bit-packed mask (hidden cells hold NaN and never enter
// arithmetic), accumulates the r x r normal matrix V_O^T V_O and V_O^T y,
// reduces them across the warp and solves by Cholesky in registers. Rows whose
// normal matrix is singular or ill-conditioned take an eigendecomposition
// pseudo-inverse (the minimum-norm solution, as the COD gives). The residual
// of e (masked_residual_norm, core.cpp:15-39) is formed directly as
// sum (y - u.v)^2 from the row still in shared memory, never by the
// cancelling ||y||^2 - u^T b shortcut.
#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

using namespace rsmd;

namespace {

constexpr int SU_MAXW = 16;  // warps per CTA (upper bound; chosen at launch)

// minimum-norm solution via eigendecomposition of the (symmetric PSD) normal
// matrix; returns the numerical rank
template <int R>
__device__ int pinv_solve(const double* Ap, const double* b, double* u) {
  double A[R][R], Q[R][R];
  int p = 0;
  for (int i = 0; i < R; ++i)
    for (int j = i; j < R; ++j) {
      A[i][j] = A[j][i] = Ap[p++];
    }
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) Q[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int i = 0; i < R; ++i) {
      dia += A[i][i] * A[i][i];
      for (int j = i + 1; j < R; ++j) off += A[i][j] * A[i][j];
    }
    if (off <= 1e-32 * dia || off == 0.0) break;
    for (int pp = 0; pp < R - 1; ++pp)
      for (int q = pp + 1; q < R; ++q) {
        const double apq = A[pp][q];
        if (apq == 0.0) continue;
        const double zeta = (A[q][q] - A[pp][pp]) / (2.0 * apq);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int k = 0; k < R; ++k) {
          const double x = A[k][pp], y = A[k][q];
          A[k][pp] = c * x - s * y;
          A[k][q] = s * x + c * y;
        }
        for (int k = 0; k < R; ++k) {
          const double x = A[pp][k], y = A[q][k];
          A[pp][k] = c * x - s * y;
          A[q][k] = s * x + c * y;
        }
        A[pp][q] = A[q][pp] = 0.0;
        for (int k = 0; k < R; ++k) {
          const double x = Q[k][pp], y = Q[k][q];
          Q[k][pp] = c * x - s * y;
          Q[k][q] = s * x + c * y;
        }
      }
  }
  double lmax = 0.0;
  for (int i = 0; i < R; ++i) lmax = fmax(lmax, A[i][i]);
  const double thr = 64.0 * 2.220446049250313e-16 * lmax;
  int rank = 0;
  for (int k = 0; k < R; ++k) u[k] = 0.0;
  for (int i = 0; i < R; ++i) {
    if (A[i][i] > thr && lmax > 0.0) {
      ++rank;
      double sb = 0.0;
      for (int k = 0; k < R; ++k) sb += Q[k][i] * b[k];
      sb /= A[i][i];
      for (int k = 0; k < R; ++k) u[k] += sb * Q[k][i];
    }
  }
  return rank;
}

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes16) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr int pow2_at_least(int x) { return x <= 1 ? 1 : 2 * pow2_at_least((x + 1) / 2); }

}  // namespace

// Normal-equation solve of one row (packed upper A, b, observed count nj):
// Cholesky in registers; rows with nj < R or a pivot <= 1e-10 max diag take the
// eigendecomposition pseudo-inverse. Returns true when the row is flagged
// (detail/row_solve.hpp:26-35: fewer than r observations or rank < r). The
// factor keeps the reciprocal of each pivot (one rsqrt per column), so the
// factorisation and both substitutions multiply instead of dividing: R
// reciprocal square roots on the dependent chain instead of R square roots
// plus R(R+1)/2 + 2R divisions.
template <int R>
__device__ __forceinline__ bool row_solve(const double* A, const double* bv, int nj, double* u) {
  constexpr int NA = R * (R + 1) / 2;
  bool slow = nj < R;
  if (!slow) {
    double L[NA], Li[R];  // L: lower factor, row-major packed; Li: 1 / L_ii
    double dmax = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) dmax = fmax(dmax, A[i * R - i * (i - 1) / 2]);
    int q = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        double v = A[j * R - j * (j - 1) / 2 + (i - j)];
#pragma unroll
        for (int k = 0; k < j; ++k) v = fma(-L[i * (i + 1) / 2 + k], L[j * (j + 1) / 2 + k], v);
        if (i == j) {
          if (!(v > 1e-10 * dmax)) slow = true;
          Li[i] = rsqrt_fast(fmax(v, 1e-300));
          L[q] = v * Li[i];
        } else {
          L[q] = v * Li[j];
        }
        ++q;
      }
    }
    if (!slow) {
      double z[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        double v = bv[i];
#pragma unroll
        for (int k = 0; k < i; ++k) v = fma(-L[i * (i + 1) / 2 + k], z[k], v);
        z[i] = v * Li[i];
      }
#pragma unroll
      for (int i = R - 1; i >= 0; --i) {
        double v = z[i];
#pragma unroll
        for (int k = i + 1; k < R; ++k) v = fma(-L[k * (k + 1) / 2 + i], u[k], v);
        u[i] = v * Li[i];
      }
    }
  }
  if (slow) {
    const int rank = pinv_solve<R>(A, bv, u);
    return (nj < R) || (rank < R);
  }
  return false;
}

// One warp per row (rows strided over the grid's warps). STAGE 1: two row
// buffers per warp in shared memory, the next row's values and mask words
// arriving by two 1-D bulk copies (TMA) on the buffer's mbarrier, issued by
// one lane; STAGE 2: the same with per-lane cp.async (odd n); STAGE 0: no row
// buffers, the warp reads its row straight from global memory (the second
// pass re-reads it from L2) -- the layout when V-hat is too large to share
// shared memory with row buffers (config 4: n = 2048, r = 8). V-hat sits in
// shared memory as ceil(R/2) planes of (v_2p, v_2p+1) pairs (VSMEM) or is
// read from global.
template <int R, bool VSMEM, int STAGE>
__global__ void __launch_bounds__(R <= 4 ? SU_MAXW * 32 : 384) k_solve_u(SolveUArgs a) {
  constexpr bool BULK = STAGE == 1;
  constexpr int NP = (R + 1) / 2;      // V planes
  constexpr int NA = R * (R + 1) / 2;  // packed normal matrix
  // reduced values (A, b, count): padded to a power of two for the halving
  // reduction when small; reduced value by value for larger r
  constexpr int NV = R <= 4 ? pow2_at_least(NA + R + 1) : NA + R + 1;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t npd = (n + 1) & ~int64_t(1);
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);  // [SU_MAXW][2]
  double2* Vp = reinterpret_cast<double2*>(sm + 2 * SU_MAXW);
  double* wb = sm + 2 * SU_MAXW + (VSMEM ? 2 * NP * n : 0);
  const int64_t bufd = npd + a.nwp / 2;  // doubles per row buffer (values + words)
  auto ybuf = [&](int b) { return wb + (2 * warp + b) * bufd; };
  if (BULK && threadIdx.x < 2 * nwarps) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bars + threadIdx.x)), "r"(1));
  }
  if (BULK && threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  if (VSMEM) {
    for (int64_t e = threadIdx.x; e < NP * n; e += blockDim.x) {
      const int64_t p = e / n, c = e % n;
      const double x0 = a.V[c * R + 2 * p];
      const double x1 = (2 * p + 1 < R) ? a.V[c * R + 2 * p + 1] : 0.0;
      Vp[e] = make_double2(x0, x1);
    }
  }
  __syncthreads();
  // A_all = V^T V (packed upper) for the dense-row complement (r > 4),
  // summed in a fixed order: per-thread strided partials, then a fixed tree
  __shared__ double Aall[NA];
  if constexpr (R > 4) {
    __shared__ double Ared[SU_MAXW][NA];
    double part[NA];
#pragma unroll
    for (int p = 0; p < NA; ++p) part[p] = 0.0;
    for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
      double v[R];
#pragma unroll
      for (int k = 0; k < R; ++k) v[k] = a.V[c * R + k];
      int p = 0;
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = i; j < R; ++j) {
          part[p] = fma(v[i], v[j], part[p]);
          ++p;
        }
    }
#pragma unroll
    for (int p = 0; p < NA; ++p) {
      const double t = warp_sum(part[p]);
      if (lane == 0) Ared[warp][p] = t;
    }
    __syncthreads();
    if (threadIdx.x < NA) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t += Ared[w][threadIdx.x];
      Aall[threadIdx.x] = t;
    }
    __syncthreads();
  }
  auto vload = [&](int64_t c, double* v) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      double2 t;
      if (VSMEM) t = Vp[p * n + c];
      else {
        t.x = __ldg(a.V + c * R + 2 * p);
        t.y = (2 * p + 1 < R) ? __ldg(a.V + c * R + 2 * p + 1) : 0.0;
      }
      v[2 * p] = t.x;
      if (2 * p + 1 < R) v[2 * p + 1] = t.y;
    }
  };
  const uint32_t ybytes = (uint32_t)(n * 8), wbytes = (uint32_t)(a.nwp * 4);
  auto issue = [&](int64_t row, int b) {
    double* yb = ybuf(b);
    uint32_t* wdst = reinterpret_cast<uint32_t*>(yb + npd);
    if (BULK) {
      if (lane == 0) {
        const unsigned bar = smem_u32(bars + 2 * warp + b);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(ybytes + wbytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                smem_u32(yb)),
            "l"(a.Y + row * n), "r"(ybytes), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                smem_u32(wdst)),
            "l"(a.bitsR + row * a.nwp), "r"(wbytes), "r"(bar)
            : "memory");
      }
    } else {
      const double* y = a.Y + row * n;
      for (int64_t c = lane; c < n; c += 32) cp_async(yb + c, y + c, 0);
      const uint32_t* w = a.bitsR + row * a.nwp;  // nwp is a multiple of 4 words
      for (int64_t c = lane; c < a.nwp / 4; c += 32) cp_async(wdst + 4 * c, w + 4 * c, 1);
      asm volatile("cp.async.commit_group;\n" ::);
    }
  };
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t nw = (int64_t)gridDim.x * nwarps;
  unsigned phase = 0u;  // bit b: parity of buffer b's next completion
  int cur = 0;
  int64_t row = a.row_lo + gw;
  if (STAGE && row < a.row_hi) issue(row, 0);
  const int nfull = (int)(n >> 5);
  for (; row < a.row_hi; row += nw) {
    const int64_t nxt = row + nw;
    if (STAGE && nxt < a.row_hi) issue(nxt, cur ^ 1);
    if (STAGE == 0) {
    } else if (BULK) {
      const unsigned bar = smem_u32(bars + 2 * warp + cur);
      unsigned done = 0;
      do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"((phase >> cur) & 1u)
            : "memory");
      } while (!done);
      phase ^= 1u << cur;
    } else {
      if (nxt < a.row_hi) asm volatile("cp.async.wait_group 1;\n" ::);
      else asm volatile("cp.async.wait_group 0;\n" ::);
      __syncwarp();
    }
    const double* y = STAGE ? ybuf(cur) : a.Y + row * n;
    const uint32_t* wd = STAGE ? reinterpret_cast<const uint32_t*>(y + npd) : a.bitsR + row * a.nwp;
    // normal equations over the observed cells; hidden cells are skipped by
    // predication (their NaN never enters arithmetic)
    double acc[NV];
#pragma unroll
    for (int p = 0; p < NV; ++p) acc[p] = 0.0;
    int cnt = 0;  // observed cells (mask words are zero beyond n)
    for (int64_t w = lane; w < a.nwp; w += 32) cnt += __popc(wd[w]);
    // r > 4 and at least half observed: V_O^T V_O = V^T V minus the hidden
    // cells' outer products (walking only the hidden bits), which saves most
    // of the r(r+1)/2 FMAs per cell
    bool dense = false;
    if constexpr (R > 4) dense = !a.Apre && 2 * (int64_t)warp_sum_int(cnt) >= n;
    const bool needA = !a.Apre;  // else the normal matrix comes from the tensor cores
    // branchless (so the loads of consecutive columns pipeline): a hidden
    // cell's basis row is scaled by 0 and its value selected away, so the NaN
    // stored there never enters arithmetic
    auto add_y = [&](int64_t c, bool k, double yraw) {
      double v[R];
      vload(c, v);
      const double yc = k ? yraw : 0.0;
      if (!dense && needA) {
        const double kf = k ? 1.0 : 0.0;
        double t[R];
#pragma unroll
        for (int i = 0; i < R; ++i) t[i] = kf * v[i];
        int p = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
          for (int j = i; j < R; ++j) {
            acc[p] = fma(t[i], v[j], acc[p]);
            ++p;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < R; ++i) acc[NA + i] = fma(yc, v[i], acc[NA + i]);
    };
    auto add = [&](int64_t c, bool k) { add_y(c, k, k ? y[c] : 0.0); };
    if constexpr (STAGE == 0) {
      // rows straight from global memory: UB words' mask words and values
      // are loaded before any is used, so UB loads per lane are in flight
      // (the hidden cells' NaN is loaded but selected away)
      constexpr int UB = 8;
      int w = 0;
      for (; w + UB <= nfull; w += UB) {
        unsigned bw[UB];
        double yv[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) bw[u] = __ldg(wd + w + u);
#pragma unroll
        for (int u = 0; u < UB; ++u) yv[u] = __ldg(y + (int64_t)(w + u) * 32 + lane);
#pragma unroll
        for (int u = 0; u < UB; ++u) add_y((w + u) * 32 + lane, (bw[u] >> lane) & 1u, yv[u]);
      }
      for (; w < nfull; ++w) add(w * 32 + lane, (wd[w] >> lane) & 1u);
    } else {
#pragma unroll 2
      for (int w = 0; w < nfull; ++w) add(w * 32 + lane, (wd[w] >> lane) & 1u);
    }
    if ((int64_t)nfull * 32 + lane < n) add(nfull * 32 + lane, (wd[nfull] >> lane) & 1u);
    if (dense) {
      const int nwn = (int)((n + 31) >> 5);
      for (int w = lane; w < nwn; w += 32) {
        const int rem = (int)(n - (int64_t)w * 32);
        const unsigned valid = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
        unsigned miss = ~wd[w] & valid;
        while (miss) {
          const int bpos = __ffs(miss) - 1;
          miss &= miss - 1u;
          double v[R];
          vload((int64_t)w * 32 + bpos, v);
          int p = 0;
#pragma unroll
          for (int i = 0; i < R; ++i)
#pragma unroll
            for (int j = i; j < R; ++j) {
              acc[p] = fma(v[i], v[j], acc[p]);
              ++p;
            }
        }
      }
    }
    acc[NA + R] = (double)cnt;
    if (R <= 4) {
      warp_reduce_halving<NV>(acc, lane);
    } else {
#pragma unroll
      for (int p = 0; p < NV; ++p) acc[p] = warp_sum(acc[p]);
    }
    auto total = [&](int p) {
      if constexpr (R <= 4) return warp_total<NV>(acc, p);
      else return acc[p];
    };
    double A[NA], bv[R];
#pragma unroll
    for (int p = 0; p < NA; ++p) A[p] = a.Apre ? a.Apre[row * NA + p] : (dense ? Aall[p] - total(p) : total(p));
#pragma unroll
    for (int i = 0; i < R; ++i) bv[i] = total(NA + i);
    const int nj = (int)total(NA + R);

    double u[R];
    bool flagged = row_solve<R>(A, bv, nj, u);
    if (a.Ugiven) {  // residual of given factors: the same arithmetic from here on
#pragma unroll
      for (int q = 0; q < R; ++q) u[q] = a.Ugiven[row * R + q];
      flagged = false;
    }
    // second pass over the row still in shared memory: direct residual
    double ss = 0.0;
    auto res_y = [&](int64_t c, bool k, double yraw) {
      double v[R];
      vload(c, v);
      double p = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) p = fma(u[q], v[q], p);
      const double d = k ? yraw - p : 0.0;
      ss = fma(d, d, ss);
    };
    auto res = [&](int64_t c, bool k) { res_y(c, k, k ? y[c] : 0.0); };
    if constexpr (STAGE == 0) {
      constexpr int UB = 8;
      int w = 0;
      for (; w + UB <= nfull; w += UB) {
        unsigned bw[UB];
        double yv[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) bw[u] = __ldg(wd + w + u);
#pragma unroll
        for (int u = 0; u < UB; ++u) yv[u] = __ldg(y + (int64_t)(w + u) * 32 + lane);
#pragma unroll
        for (int u = 0; u < UB; ++u) res_y((w + u) * 32 + lane, (bw[u] >> lane) & 1u, yv[u]);
      }
      for (; w < nfull; ++w) res(w * 32 + lane, (wd[w] >> lane) & 1u);
    } else {
#pragma unroll 2
      for (int w = 0; w < nfull; ++w) res(w * 32 + lane, (wd[w] >> lane) & 1u);
    }
    if ((int64_t)nfull * 32 + lane < n) res(nfull * 32 + lane, (wd[nfull] >> lane) & 1u);
    ss = warp_sum(ss);
    if (lane < R) {
      double uk = 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k == lane) uk = u[k];
      a.U[row * R + lane] = uk;
    }
    if (lane == 0) {
      a.rowres[row] = ss;
      if (flagged) atomicAdd(a.flagged, 1);
    }
    __syncwarp();  // this buffer is refilled by the next iteration's prefetch
    cur ^= 1;
  }
}

// Fused-pass row solver (r <= 4, V-hat in shared memory, rows staged by TMA).
// The residual pass of a warp's row k runs in the same column loop as the
// accumulation pass of its next row k+1, so every shared-memory read of V-hat
// serves both rows. Row k stays in its buffer until that loop ends; the
// buffer is then refilled with row k+2 (already pulled into L2 by a bulk
// prefetch issued when the loop started) while row k+1 is solved.
//
// Per column the loop does only what every cell needs: V_O^T y (R FMAs on the
// selected value) for row k+1 and the direct residual (R FMAs from y, one
// select, one FMA) for row k. The normal matrix V_O^T V_O is formed word by
// word from each 32-column mask word's MINORITY cells: a word with at least 16
// observed cells contributes V_w^T V_w (its 32 columns' Gram, tabulated once
// per CTA in a fixed order) minus its hidden cells' outer products, any other
// word its observed cells' outer products; each lane walks the bits of its own
// words, so at most 16 outer products per word and ~0.2 n per row at config 3
// (rho = 0.8) instead of n. The observed count and row k's residual ride in
// the same warp reduction as row k+1's normal equations.
// WALK = false: the minority outer products are accumulated inside the
// streaming loop instead (row-level decision: V^T V minus the hidden cells
// when at least half the row is observed, else the observed cells), with the
// basis row already in registers -- no extra shared-memory reads, ~14 more
// FP64 instructions per cell.
template <int R, bool WALK>
__global__ void __launch_bounds__(SU_MAXW * 32) k_solve_u_fused(SolveUArgs a) {
  constexpr int NP = (R + 1) / 2;
  constexpr int NA = R * (R + 1) / 2;
  constexpr int NV = pow2_at_least(NA + R + 2);  // A, b, count, previous row's residual
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t npd = (n + 1) & ~int64_t(1);
  const int nwarps = blockDim.x >> 5;
  const int nwn = (int)((n + 31) >> 5);  // mask words holding columns
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);  // [SU_MAXW][2]
  double2* Vp = reinterpret_cast<double2*>(sm + 2 * SU_MAXW);
  double* Vw = sm + 2 * SU_MAXW + 2 * NP * n;  // nwn x NA per-word Grams
  double* wb = Vw + (((int64_t)nwn * NA + 1) & ~int64_t(1));
  const int64_t bufd = npd + a.nwp / 2;
  auto ybuf = [&](int b) { return wb + (2 * warp + b) * bufd; };
  if (threadIdx.x < 2 * nwarps)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bars + threadIdx.x)), "r"(1));
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  for (int64_t e = threadIdx.x; e < NP * n; e += blockDim.x) {
    const int64_t p = e / n, c = e % n;
    const double x0 = a.V[c * R + 2 * p];
    const double x1 = (2 * p + 1 < R) ? a.V[c * R + 2 * p + 1] : 0.0;
    Vp[e] = make_double2(x0, x1);
  }
  // per-word Gram V_w^T V_w (packed upper): one thread sums a word's columns
  // in column order -- the same bits in every CTA and launch shape
  for (int w = threadIdx.x; w < nwn; w += blockDim.x) {
    double part[NA];
#pragma unroll
    for (int p = 0; p < NA; ++p) part[p] = 0.0;
    for (int64_t c = (int64_t)w * 32; c < n && c < (int64_t)w * 32 + 32; ++c) {
      double v[R];
#pragma unroll
      for (int k = 0; k < R; ++k) v[k] = a.V[c * R + k];
      int p = 0;
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = i; j < R; ++j) {
          part[p] = fma(v[i], v[j], part[p]);
          ++p;
        }
    }
#pragma unroll
    for (int p = 0; p < NA; ++p) Vw[(int64_t)w * NA + p] = part[p];
  }
  __syncthreads();
  __shared__ double Aall[NA];  // V^T V = sum of the word Grams in word order
  if (!WALK && threadIdx.x < NA) {
    double t = 0.0;
    for (int w = 0; w < nwn; ++w) t += Vw[(int64_t)w * NA + threadIdx.x];
    Aall[threadIdx.x] = t;
  }
  __syncthreads();
  auto vload = [&](int64_t c, double* v) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double2 t = Vp[p * n + c];
      v[2 * p] = t.x;
      if (2 * p + 1 < R) v[2 * p + 1] = t.y;
    }
  };
  const uint32_t ybytes = (uint32_t)(n * 8), wbytes = (uint32_t)(a.nwp * 4);
  auto issue = [&](int64_t row, int b) {
    if (lane == 0) {
      double* yb = ybuf(b);
      const unsigned bar = smem_u32(bars + 2 * warp + b);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(ybytes + wbytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              smem_u32(yb)),
          "l"(a.Y + row * n), "r"(ybytes), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              smem_u32(yb + npd)),
          "l"(a.bitsR + row * a.nwp), "r"(wbytes), "r"(bar)
          : "memory");
    }
  };
  auto prefetch_l2 = [&](int64_t row) {
    if (lane == 0) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a.Y + row * n), "r"(ybytes) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a.bitsR + row * a.nwp), "r"(wbytes)
                   : "memory");
    }
  };
  unsigned phase = 0u;
  auto wait_buf = [&](int b) {
    const unsigned bar = smem_u32(bars + 2 * warp + b);
    unsigned done = 0;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar), "r"((phase >> b) & 1u)
          : "memory");
    } while (!done);
    phase ^= 1u << b;
  };
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t nw = (int64_t)gridDim.x * nwarps;
  const int64_t r0 = a.row_lo + gw;
  if (r0 >= a.row_hi) return;
  const int64_t nrows = (a.row_hi - r0 + nw - 1) / nw;  // this warp's rows: r0 + k nw
  const int nfull = (int)(n >> 5);
  const bool tail = (int64_t)nfull * 32 + lane < n;
  issue(r0, 0);
  if (nrows > 1) issue(r0 + nw, 1);
  // V_O^T y term of column c (the hidden cell's NaN is selected away)
  auto accum_b = [&](double* acc, const double* v, double yraw, bool k) {
    const double yc = k ? yraw : 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) acc[NA + i] = fma(yc, v[i], acc[NA + i]);
  };
  // direct residual term: d = y - u.v from y (nu = -u), zero when hidden
  // in-loop minority outer product (WALK = false): weight sg on the selected cells
  auto accum_A = [&](double* acc, const double* v, bool k, bool hid) {
    const double w = (hid ? !k : k) ? (hid ? -1.0 : 1.0) : 0.0;
    double t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) t[i] = w * v[i];
    int p = 0;
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int j = i; j < R; ++j) {
        acc[p] = fma(t[i], v[j], acc[p]);
        ++p;
      }
  };
  // observed count of a row (all lanes get it) and its minority side
  auto row_count = [&](const uint32_t* wd) -> int {
    int c = 0;
    for (int w = lane; w < nwn; w += 32) c += __popc(wd[w]);
    return warp_sum_int(c);
  };
  auto resid = [&](double& ss, const double* v, const double* nu, double yraw, bool k) {
    double d = yraw;
#pragma unroll
    for (int q = 0; q < R; ++q) d = fma(nu[q], v[q], d);
    d = k ? d : 0.0;
    ss = fma(d, d, ss);
  };
  // normal matrix from each word's minority cells, then one reduction of the
  // normal equations, the observed count and the previous row's residual
  // (ss_prev, returned summed), and the solve
  auto finish = [&](double (&acc)[NV], const uint32_t* wd, double* u, double& ss_prev, int64_t frow, int njr,
                    bool hidr) -> bool {
    int cnt = 0;
    if (a.Apre) {  // normal matrices from the tensor cores: only the count here
      for (int w = lane; w < nwn; w += 32) cnt += __popc(wd[w]);
    } else if (!WALK) {
      if (hidr) {
#pragma unroll
        for (int p = 0; p < NA; ++p) acc[p] += lane == 0 ? Aall[p] : 0.0;
      }
      cnt = lane == 0 ? njr : 0;
    }
    for (int w = lane; WALK && !a.Apre && w < nwn; w += 32) {
      const int rem = (int)(n - (int64_t)w * 32);
      const unsigned valid = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
      const unsigned obs = wd[w] & valid;
      const int no = __popc(obs);
      cnt += no;
      const bool hid = 2 * no >= __popc(valid);
      const double sg = hid ? -1.0 : 1.0;
      unsigned bits = hid ? (~obs & valid) : obs;
      if (hid) {
#pragma unroll
        for (int p = 0; p < NA; ++p) acc[p] += Vw[(int64_t)w * NA + p];
      }
      // two cells per iteration (independent loads and FMA chains); a lone
      // last cell pairs with itself at weight 0
      while (bits) {
        const int p0 = __ffs(bits) - 1;
        bits &= bits - 1u;
        const bool two = bits != 0u;
        const int p1 = two ? __ffs(bits) - 1 : p0;
        bits &= bits - 1u;
        double v[R], x[R];
        vload((int64_t)w * 32 + p0, v);
        vload((int64_t)w * 32 + p1, x);
        const double s1 = two ? sg : 0.0;
        int p = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const double vs = sg * v[i], xs = s1 * x[i];
#pragma unroll
          for (int j = i; j < R; ++j) {
            acc[p] = fma(xs, x[j], fma(vs, v[j], acc[p]));
            ++p;
          }
        }
      }
    }
    acc[NA + R] = (double)cnt;
    acc[NA + R + 1] = ss_prev;
    warp_reduce_halving<NV>(acc, lane);
    double A[NA], bv[R];
#pragma unroll
    for (int p = 0; p < NA; ++p) A[p] = a.Apre ? a.Apre[frow * NA + p] : warp_total<NV>(acc, p);
#pragma unroll
    for (int i = 0; i < R; ++i) bv[i] = warp_total<NV>(acc, NA + i);
    const int nj = (int)warp_total<NV>(acc, NA + R);
    ss_prev = warp_total<NV>(acc, NA + R + 1);
    const bool fl = row_solve<R>(A, bv, nj, u);
    if (a.Ugiven) {  // residual of given factors: the same arithmetic from here on
#pragma unroll
      for (int q = 0; q < R; ++q) u[q] = a.Ugiven[frow * R + q];
      return false;
    }
    return fl;
  };
  // row 0: accumulation pass alone
  double u[R];
  bool flagged;
  {
    wait_buf(0);
    const double* y = ybuf(0);
    const uint32_t* wd = reinterpret_cast<const uint32_t*>(y + npd);
    const int nj0 = WALK ? 0 : row_count(wd);
    const bool hid0 = 2 * (int64_t)nj0 >= n;
    double acc[NV];
#pragma unroll
    for (int p = 0; p < NV; ++p) acc[p] = 0.0;
#pragma unroll 4
    for (int w = 0; w < nfull; ++w) {
      const int64_t c = w * 32 + lane;
      double v[R];
      vload(c, v);
      const bool k0 = (wd[w] >> lane) & 1u;
      accum_b(acc, v, y[c], k0);
      if (!WALK) accum_A(acc, v, k0, hid0);
    }
    if (tail) {
      const int64_t c = (int64_t)nfull * 32 + lane;
      double v[R];
      vload(c, v);
      const bool k0 = (wd[nfull] >> lane) & 1u;
      accum_b(acc, v, y[c], k0);
      if (!WALK) accum_A(acc, v, k0, hid0);
    }
    double none = 0.0;
    flagged = finish(acc, wd, u, none, r0, nj0, hid0);
  }
  for (int64_t k = 0; k < nrows; ++k) {
    const int64_t row = r0 + k * nw;
    const int b = (int)(k & 1);
    const double* y = ybuf(b);
    const uint32_t* wd = reinterpret_cast<const uint32_t*>(y + npd);
    const bool has_next = k + 1 < nrows;
    if (k + 2 < nrows) prefetch_l2(r0 + (k + 2) * nw);
    double nu[R];
#pragma unroll
    for (int q = 0; q < R; ++q) nu[q] = -u[q];
    double ss = 0.0;
    double acc[NV];
#pragma unroll
    for (int p = 0; p < NV; ++p) acc[p] = 0.0;
    const double* yn = ybuf(b ^ 1);
    const uint32_t* wn = reinterpret_cast<const uint32_t*>(yn + npd);
    int nj1 = 0;
    bool hid1 = false;
    if (has_next) {
      wait_buf(b ^ 1);
      if (!WALK) {
        nj1 = row_count(wn);
        hid1 = 2 * (int64_t)nj1 >= n;
      }
      // residual of row k and V_O^T y of row k+1 share the V-hat reads
#pragma unroll 4
      for (int w = 0; w < nfull; ++w) {
        const int64_t c = w * 32 + lane;
        double v[R];
        vload(c, v);
        resid(ss, v, nu, y[c], (wd[w] >> lane) & 1u);
        const bool k1 = (wn[w] >> lane) & 1u;
        accum_b(acc, v, yn[c], k1);
        if (!WALK) accum_A(acc, v, k1, hid1);
      }
      if (tail) {
        const int64_t c = (int64_t)nfull * 32 + lane;
        double v[R];
        vload(c, v);
        resid(ss, v, nu, y[c], (wd[nfull] >> lane) & 1u);
        const bool k1 = (wn[nfull] >> lane) & 1u;
        accum_b(acc, v, yn[c], k1);
        if (!WALK) accum_A(acc, v, k1, hid1);
      }
    } else {
#pragma unroll 4
      for (int w = 0; w < nfull; ++w) {
        const int64_t c = w * 32 + lane;
        double v[R];
        vload(c, v);
        resid(ss, v, nu, y[c], (wd[w] >> lane) & 1u);
      }
      if (tail) {
        const int64_t c = (int64_t)nfull * 32 + lane;
        double v[R];
        vload(c, v);
        resid(ss, v, nu, y[c], (wd[nfull] >> lane) & 1u);
      }
    }
    if (lane < R) {
      double uk = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q == lane) uk = u[q];
      a.U[row * R + lane] = uk;
    }
    if (lane == 0 && flagged) atomicAdd(a.flagged, 1);
    __syncwarp();  // row k's buffer is free: refill it with row k+2
    if (k + 2 < nrows) issue(r0 + (k + 2) * nw, b);
    if (has_next) flagged = finish(acc, wn, u, ss, row + nw, nj1, hid1);  // ss: row k's residual, summed
    else ss = warp_sum(ss);
    if (lane == 0) a.rowres[row] = ss;
  }
}

// Row solver for precomputed normal matrices (a.Apre from k_normal_i8.cu,
// r <= 4, n even): per row only V_O^T y, the observed count and the direct
// residual remain, so a warp keeps ONE staged row: row k+1 arrives in the
// warp's buffer by TMA (values; its mask words into one of two small word
// buffers) and is accumulated while the residual of row k -- staged one row
// earlier and still in L2 -- is formed from global loads in the same column
// loop (every V-hat read in shared memory serves both rows). Half the row
// buffers of k_solve_u_fused, so 16 warps per SM instead of 11 (V-hat stays
// in shared memory), and the per-row reduction carries R + 2 values instead of
// the normal matrix's. Same arithmetic per cell as k_solve_u_fused (the
// residual, the selects and the FMA order are identical), same results.
template <int R>
__global__ void __launch_bounds__(SU_MAXW * 32) k_solve_u_pre(SolveUArgs a) {
  constexpr int NP = (R + 1) / 2;
  constexpr int NA = R * (R + 1) / 2;
  constexpr int NV = pow2_at_least(R + 2);  // b, count, previous row's residual
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int nwarps = blockDim.x >> 5;
  const int nwn = (int)((n + 31) >> 5);
  const int64_t mwd = ((a.nwp + 3) & ~int64_t(3)) / 2;  // one row's mask words, in doubles (16-byte multiple)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);  // [SU_MAXW]
  double2* Vp = reinterpret_cast<double2*>(sm + SU_MAXW);
  double* wb = sm + SU_MAXW + 2 * NP * n;
  const int64_t bufd = n + 2 * mwd;  // values, then two mask-word slots
  double* ybuf = wb + warp * bufd;
  auto mbuf = [&](int s) { return reinterpret_cast<uint32_t*>(ybuf + n + s * mwd); };
  if (threadIdx.x < nwarps)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bars + threadIdx.x)), "r"(1));
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  for (int64_t e = threadIdx.x; e < NP * n; e += blockDim.x) {
    const int64_t p = e / n, c = e % n;
    const double x0 = a.V[c * R + 2 * p];
    const double x1 = (2 * p + 1 < R) ? a.V[c * R + 2 * p + 1] : 0.0;
    Vp[e] = make_double2(x0, x1);
  }
  __syncthreads();
  auto vload = [&](int64_t c, double* v) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double2 t = Vp[p * n + c];
      v[2 * p] = t.x;
      if (2 * p + 1 < R) v[2 * p + 1] = t.y;
    }
  };
  const uint32_t ybytes = (uint32_t)(n * 8), wbytes = (uint32_t)(a.nwp * 4);
  const unsigned bar = smem_u32(bars + warp);
  auto issue = [&](int64_t row, int slot) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(ybytes + wbytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              smem_u32(ybuf)),
          "l"(a.Y + row * n), "r"(ybytes), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              smem_u32(mbuf(slot))),
          "l"(a.bitsR + row * a.nwp), "r"(wbytes), "r"(bar)
          : "memory");
    }
  };
  auto prefetch_l2 = [&](int64_t row) {
    if (lane == 0) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a.Y + row * n), "r"(ybytes) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a.bitsR + row * a.nwp), "r"(wbytes)
                   : "memory");
    }
  };
  unsigned phase = 0u;
  auto wait_buf = [&]() {
    unsigned done = 0;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar), "r"(phase)
          : "memory");
    } while (!done);
    phase ^= 1u;
  };
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t nw = (int64_t)gridDim.x * nwarps;
  const int64_t r0 = a.row_lo + gw;
  if (r0 >= a.row_hi) return;
  const int64_t nrows = (a.row_hi - r0 + nw - 1) / nw;  // this warp's rows: r0 + k nw
  const int nfull = (int)(n >> 5);
  const bool tail = (int64_t)nfull * 32 + lane < n;
  const unsigned lbit = 1u << lane;
  // predicated on the mask bit (no selects): a hidden cell's NaN never
  // enters an executed instruction, and skipping adds nothing the selected-zero
  // form would (acc + 0 * v == acc, ss + 0 * 0 == ss)
  auto accum_b = [&](double* acc, const double* v, double yraw, bool k) {
    if (k) {
#pragma unroll
      for (int i = 0; i < R; ++i) acc[i] = fma(yraw, v[i], acc[i]);
    }
  };
  auto resid = [&](double& ss, const double* v, const double* nu, double yraw, bool k) {
    double d = yraw;
#pragma unroll
    for (int q = 0; q < R; ++q) d = fma(nu[q], v[q], d);
    if (k) ss = fma(d, d, ss);
  };
  // count, one reduction of b / count / the previous row's residual, solve
  auto finish = [&](double (&acc)[NV], const uint32_t* wd, double* u, double& ss_prev, int64_t frow) -> bool {
    int cnt = 0;
    for (int w = lane; w < nwn; w += 32) cnt += __popc(wd[w]);
    acc[R] = (double)cnt;
    acc[R + 1] = ss_prev;
    warp_reduce_halving<NV>(acc, lane);
    double A[NA], bv[R];
    const double* ap = a.Apre + frow * NA;
    if constexpr (NA % 2 == 0) {
#pragma unroll
      for (int p = 0; p < NA / 2; ++p) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(ap) + p);
        A[2 * p] = t.x;
        A[2 * p + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int p = 0; p < NA; ++p) A[p] = __ldg(ap + p);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) bv[i] = warp_total<NV>(acc, i);
    const int nj = (int)warp_total<NV>(acc, R);
    ss_prev = warp_total<NV>(acc, R + 1);
    const bool fl = row_solve<R>(A, bv, nj, u);
    if (a.Ugiven) {
#pragma unroll
      for (int q = 0; q < R; ++q) u[q] = a.Ugiven[frow * R + q];
      return false;
    }
    return fl;
  };
  // row 0: accumulation pass alone
  double u[R];
  bool flagged;
  issue(r0, 0);
  {
    wait_buf();
    const uint32_t* wd = mbuf(0);
    double acc[NV];
#pragma unroll
    for (int p = 0; p < NV; ++p) acc[p] = 0.0;
#pragma unroll 4
    for (int w = 0; w < nfull; ++w) {
      const int64_t c = w * 32 + lane;
      double v[R];
      vload(c, v);
      accum_b(acc, v, ybuf[c], (wd[w] >> lane) & 1u);
    }
    if (tail) {
      const int64_t c = (int64_t)nfull * 32 + lane;
      double v[R];
      vload(c, v);
      accum_b(acc, v, ybuf[c], (wd[nfull] >> lane) & 1u);
    }
    double none = 0.0;
    flagged = finish(acc, wd, u, none, r0);
  }
  for (int64_t k = 0; k < nrows; ++k) {
    const int64_t row = r0 + k * nw;
    const uint32_t* wd = mbuf((int)(k & 1));
    const uint32_t* wn = mbuf((int)((k + 1) & 1));
    const double* yg = a.Y + row * n;  // row k: staged one row ago, read back through L2
    const bool has_next = k + 1 < nrows;
    if (has_next) issue(row + nw, (int)((k + 1) & 1));  // the buffer is free: row k was accumulated
    if (k + 2 < nrows) prefetch_l2(r0 + (k + 2) * nw);
    double nu[R];
#pragma unroll
    for (int q = 0; q < R; ++q) nu[q] = -u[q];
    double ss = 0.0;
    double acc[NV];
#pragma unroll
    for (int p = 0; p < NV; ++p) acc[p] = 0.0;
    if (has_next) {
      wait_buf();
      // running pointers (immediate offsets in the unrolled body)
      const double* yp = yg + lane;
      const double* yb = ybuf + lane;
      const double2* vq = Vp + lane;
      // groups of four words: both rows' mask words by one 16-byte load each
      const int nq = nfull >> 2;
      for (int g = 0; g < nq; ++g) {
        const uint4 md = reinterpret_cast<const uint4*>(wd)[g];
        const uint4 mn = reinterpret_cast<const uint4*>(wn)[g];
        const unsigned dw[4] = {md.x, md.y, md.z, md.w}, nw4[4] = {mn.x, mn.y, mn.z, mn.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double v[R];
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const double2 t = vq[p * n + 32 * j];
            v[2 * p] = t.x;
            if (2 * p + 1 < R) v[2 * p + 1] = t.y;
          }
          resid(ss, v, nu, __ldg(yp + 32 * j), (dw[j] & lbit) != 0u);
          accum_b(acc, v, yb[32 * j], (nw4[j] & lbit) != 0u);
        }
        yp += 128;
        yb += 128;
        vq += 128;
      }
      for (int w = nq << 2; w < nfull; ++w) {
        double v[R];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const double2 t = vq[p * n];
          v[2 * p] = t.x;
          if (2 * p + 1 < R) v[2 * p + 1] = t.y;
        }
        resid(ss, v, nu, __ldg(yp), (wd[w] >> lane) & 1u);
        accum_b(acc, v, *yb, (wn[w] >> lane) & 1u);
        yp += 32;
        yb += 32;
        vq += 32;
      }
      if (tail) {
        const int64_t c = (int64_t)nfull * 32 + lane;
        double v[R];
        vload(c, v);
        resid(ss, v, nu, __ldg(yg + c), (wd[nfull] >> lane) & 1u);
        accum_b(acc, v, ybuf[c], (wn[nfull] >> lane) & 1u);
      }
    } else {
#pragma unroll 4
      for (int w = 0; w < nfull; ++w) {
        const int64_t c = w * 32 + lane;
        double v[R];
        vload(c, v);
        resid(ss, v, nu, __ldg(yg + c), (wd[w] >> lane) & 1u);
      }
      if (tail) {
        const int64_t c = (int64_t)nfull * 32 + lane;
        double v[R];
        vload(c, v);
        resid(ss, v, nu, __ldg(yg + c), (wd[nfull] >> lane) & 1u);
      }
    }
    if (lane < R) {
      double uk = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q == lane) uk = u[q];
      a.U[row * R + lane] = uk;
    }
    if (lane == 0 && flagged) atomicAdd(a.flagged, 1);
    if (has_next) flagged = finish(acc, wn, u, ss, row + nw);  // ss: row k's residual, summed
    else ss = warp_sum(ss);
    if (lane == 0) a.rowres[row] = ss;
    __syncwarp();  // every lane is done with the word slot the next issue overwrites
  }
}

// k_solve_u_pre without row staging, for a V-hat that leaves no room for row
// buffers (config 4: n = 2048, r = 8 -- 128 KB of basis planes): both rows of
// the fused column loop come straight from global memory (row k+1 from DRAM,
// pulled toward L2 by a bulk prefetch two rows ahead; row k, read one
// iteration earlier, from L2), eight words of each row in flight per lane.
// Every V-hat read in shared memory serves the residual of row k and the
// accumulation of row k+1 -- the two-pass kernel read the basis twice per row,
// and at r = 8 those reads (64 B per cell per pass) are what bounds it. Every
// lane sees every mask word, so the observed count needs no reduction; the
// warp reduction carries V_O^T y and the previous row's residual only. Same
// per-cell arithmetic as k_solve_u_pre. Needs a.Apre (k_normal_i8.cu).
template <int R>
__global__ void __launch_bounds__(384) k_solve_u_preg(SolveUArgs a) {
  constexpr int NP = (R + 1) / 2;
  constexpr int NA = R * (R + 1) / 2;
  constexpr int NV = pow2_at_least(R + 1);  // b, previous row's residual
  constexpr int UB = 8;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int nwarps = blockDim.x >> 5;
  double2* Vp = reinterpret_cast<double2*>(sm);
  for (int64_t e = threadIdx.x; e < NP * n; e += blockDim.x) {
    const int64_t p = e / n, c = e % n;
    const double x0 = a.V[c * R + 2 * p];
    const double x1 = (2 * p + 1 < R) ? a.V[c * R + 2 * p + 1] : 0.0;
    Vp[e] = make_double2(x0, x1);
  }
  __syncthreads();
  const uint32_t ybytes = (uint32_t)(n * 8), wbytes = (uint32_t)(a.nwp * 4);
  auto prefetch_l2 = [&](int64_t row) {
    if (lane == 0) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a.Y + row * n), "r"(ybytes) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a.bitsR + row * a.nwp), "r"(wbytes)
                   : "memory");
    }
  };
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t nw = (int64_t)gridDim.x * nwarps;
  const int64_t r0 = a.row_lo + gw;
  if (r0 >= a.row_hi) return;
  const int64_t nrows = (a.row_hi - r0 + nw - 1) / nw;  // this warp's rows: r0 + k nw
  const int nfull = (int)(n >> 5);
  const bool has_tail = (int64_t)nfull * 32 < n;
  const bool tail = (int64_t)nfull * 32 + lane < n;
  const unsigned lbit = 1u << lane;
  // L2 residency: a row's first read (as row k+1) asks L2 to keep its lines,
  // the second (as row k, one iteration later) releases them
  uint64_t pol_keep, pol_drop;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_drop));
  auto ld_hint = [](const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(p), "l"(pol));
    return v;
  };
  auto vload = [&](const double2* vq, double* v) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double2 t = vq[p * n];
      v[2 * p] = t.x;
      if (2 * p + 1 < R) v[2 * p + 1] = t.y;
    }
  };
  // predicated on the mask bit: a hidden cell's NaN never enters an executed
  // instruction (as k_solve_u_pre)
  auto accum_b = [&](double* acc, const double* v, double yraw, bool k) {
    if (k) {
#pragma unroll
      for (int i = 0; i < R; ++i) acc[i] = fma(yraw, v[i], acc[i]);
    }
  };
  auto resid = [&](double& ss, const double* v, const double* nu, double yraw, bool k) {
    double d = yraw;
#pragma unroll
    for (int q = 0; q < R; ++q) d = fma(nu[q], v[q], d);
    if (k) ss = fma(d, d, ss);
  };
  auto finish = [&](double (&acc)[NV], int cnt, double* u, double& ss_prev, int64_t frow) -> bool {
    double A[NA], bv[R];
    const double* ap = a.Apre + frow * NA;
#pragma unroll
    for (int p = 0; p < NA; ++p) A[p] = __ldg(ap + p);  // in flight during the reduction
    acc[R] = ss_prev;
    warp_reduce_halving<NV>(acc, lane);
#pragma unroll
    for (int i = 0; i < R; ++i) bv[i] = warp_total<NV>(acc, i);
    ss_prev = warp_total<NV>(acc, R);
    const bool fl = row_solve<R>(A, bv, cnt, u);
    if (a.Ugiven) {
#pragma unroll
      for (int q = 0; q < R; ++q) u[q] = a.Ugiven[frow * R + q];
      return false;
    }
    return fl;
  };
  // one row alone: ACC = accumulation pass (row 0), else residual pass (last row)
  auto single = [&](auto ACC, const double* y, const uint32_t* wd, double* acc, const double* nu, double& ss,
                    int& cnt) {
    constexpr bool kAcc = decltype(ACC)::value;
    const double* yp = y + lane;
    const double2* vq = Vp + lane;
    int w = 0;
    for (; w + UB <= nfull; w += UB) {
      const uint4 m0 = __ldg(reinterpret_cast<const uint4*>(wd + w));
      const uint4 m1 = __ldg(reinterpret_cast<const uint4*>(wd + w + 4));
      const unsigned bw[UB] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
      double yv[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) yv[u] = __ldg(yp + 32 * u);
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        double v[R];
        vload(vq + 32 * u, v);
        if (kAcc) {
          cnt += __popc(bw[u]);
          accum_b(acc, v, yv[u], (bw[u] & lbit) != 0u);
        } else {
          resid(ss, v, nu, yv[u], (bw[u] & lbit) != 0u);
        }
      }
      yp += 32 * UB;
      vq += 32 * UB;
    }
    for (; w < nfull + (has_tail ? 1 : 0); ++w) {
      const unsigned word = __ldg(wd + w);
      if (kAcc) cnt += __popc(word);
      if (w < nfull || tail) {
        double v[R];
        vload(vq, v);
        const bool k = (word & lbit) != 0u;
        const double yraw = k ? __ldg(yp) : 0.0;
        if (kAcc) accum_b(acc, v, yraw, k);
        else resid(ss, v, nu, yraw, k);
      }
      yp += 32;
      vq += 32;
    }
  };
  double u[R];
  bool flagged;
  {
    double acc[NV];
#pragma unroll
    for (int p = 0; p < NV; ++p) acc[p] = 0.0;
    double none = 0.0;
    int cnt = 0;
    if ((a.pf & 3) && nrows > 1) prefetch_l2(r0 + nw);
    single(std::true_type{}, a.Y + r0 * n, a.bitsR + r0 * a.nwp, acc, nullptr, none, cnt);
    flagged = finish(acc, cnt, u, none, r0);
  }
  for (int64_t k = 0; k < nrows; ++k) {
    const int64_t row = r0 + k * nw;
    const bool has_next = k + 1 < nrows;
    if ((a.pf & 3) && k + 2 < nrows) prefetch_l2(r0 + (k + 2) * nw);
    const double* yk = a.Y + row * n;
    const uint32_t* wd = a.bitsR + row * a.nwp;
    double nu[R];
#pragma unroll
    for (int q = 0; q < R; ++q) nu[q] = -u[q];
    double ss = 0.0;
    double acc[NV];
#pragma unroll
    for (int p = 0; p < NV; ++p) acc[p] = 0.0;
    int cnt = 0;
    if (has_next) {
      const double* yn = yk + nw * n;
      const uint32_t* wn = wd + nw * a.nwp;
      const double* ypk = yk + lane;
      const double* ypn = yn + lane;
      const double2* vq = Vp + lane;
      int w = 0;
      for (; w + UB <= nfull; w += UB) {
        const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(wd + w));
        const uint4 d1 = __ldg(reinterpret_cast<const uint4*>(wd + w + 4));
        const uint4 n0 = __ldg(reinterpret_cast<const uint4*>(wn + w));
        const uint4 n1 = __ldg(reinterpret_cast<const uint4*>(wn + w + 4));
        const unsigned dw[UB] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        const unsigned nwd[UB] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
        double yvn[UB], yvk[UB];
#pragma unroll
        for (int q = 0; q < UB; ++q) yvn[q] = a.pf & 4 ? ld_hint(ypn + 32 * q, pol_keep) : __ldg(ypn + 32 * q);  // DRAM
#pragma unroll
        for (int q = 0; q < UB; ++q) yvk[q] = a.pf & 4 ? ld_hint(ypk + 32 * q, pol_drop) : __ldg(ypk + 32 * q);  // L2
#pragma unroll
        for (int q = 0; q < UB; ++q) {
          double v[R];
          vload(vq + 32 * q, v);
          cnt += __popc(nwd[q]);
          resid(ss, v, nu, yvk[q], (dw[q] & lbit) != 0u);
          accum_b(acc, v, yvn[q], (nwd[q] & lbit) != 0u);
        }
        ypk += 32 * UB;
        ypn += 32 * UB;
        vq += 32 * UB;
      }
      for (; w < nfull + (has_tail ? 1 : 0); ++w) {
        const unsigned wdk = __ldg(wd + w), wdn = __ldg(wn + w);
        cnt += __popc(wdn);
        if (w < nfull || tail) {
          double v[R];
          vload(vq, v);
          const bool kk = (wdk & lbit) != 0u, kn = (wdn & lbit) != 0u;
          resid(ss, v, nu, kk ? __ldg(ypk) : 0.0, kk);
          accum_b(acc, v, kn ? __ldg(ypn) : 0.0, kn);
        }
        ypk += 32;
        ypn += 32;
        vq += 32;
      }
    } else {
      single(std::false_type{}, yk, wd, acc, nu, ss, cnt);
    }
    if (lane < R) {
      double uk = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q == lane) uk = u[q];
      a.U[row * R + lane] = uk;
    }
    if (lane == 0 && flagged) atomicAdd(a.flagged, 1);
    if (has_next) flagged = finish(acc, cnt, u, ss, row + nw);  // ss: row k's residual, summed
    else ss = warp_sum(ss);
    if (lane == 0) a.rowres[row] = ss;
  }
}

// Stage 5 on the FP64 tensor cores (mma.m8n8k4.f64), for precomputed normal
// matrices (a.Apre), r <= 8, n a multiple of 32. A warp owns 8 rows at a time;
// lane l sits in row g = l / 4 of the block with k = l % 4.
//   pass 1, b = V_O^T y: D(8 rows x 8) += A(8 x 4) B(4 x 8) per step with A
//     the masked values and B four basis rows (columns j >= r are zero). The
//     contraction order is free, so lane k of a row takes the four CONTIGUOUS
//     columns 4k..4k+3 of every 16-column group (one 256-bit load, LDG.256:
//     a row's whole 128-byte line per warp instruction) and step q uses
//     column 4k + q of each lane;
//   the 8 rows are solved at once (each 4-lane group holds its row's b, count
//     and normal matrix; no reduction anywhere: the MMA did it);
//   pass 2, the residual: an 8 x 8 tile of U V^T per MMA (A = the rows' u, B =
//     eight basis rows chosen so that two tiles give a lane the predictions of
//     the same four contiguous columns), read against one 256-bit load of Y
//     (through L2: the block was read by pass 1 moments ago; evict_last there,
//     evict_first here).
// ~360 warp instructions per row instead of ~1370, and V-hat's shared-memory
// reads drop to 8 B per row-column. V-hat sits in shared memory with an odd
// row stride (5 or 9 doubles) so both fragment patterns are conflict-free.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

#ifndef RSM_SU_MMA_PFD
#define RSM_SU_MMA_PFD 2
#endif
// TEAM warps share an 8-row block, each taking 1/TEAM of its columns: the
// bytes a warp holds between its two passes (and so the L2 footprint of all
// warps' blocks, which must stay below L2's capacity for the second read to
// hit) shrink by TEAM while the warps in flight stay. The team's partial b,
// counts and residuals meet in shared memory across a named barrier and are
// added in team order; every team warp solves the block's rows (same inputs,
// same result).
template <int R, int UW, int TEAM>
__global__ void __launch_bounds__((R <= 4 && UW <= 4) ? 512 : 256) k_solve_u_mma(SolveUArgs a) {
  constexpr int RS = R <= 4 ? 5 : 9;
  constexpr int NA = R * (R + 1) / 2;
  constexpr int NK = (R + 3) / 4;
  constexpr int PFD = RSM_SU_MMA_PFD;  // pass 1: steps prefetched ahead
  // UW: mask words (32 columns each) per unrolled step, 2 UW KB of a block in flight per warp
  extern __shared__ __align__(16) double Vs[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, k = lane & 3;
  const int64_t n = a.n;
  const int nwarps = blockDim.x >> 5;
  for (int64_t e = threadIdx.x; e < n * R; e += blockDim.x) {
    const int64_t c = e / R;
    const int j = (int)(e % R);
    Vs[c * RS + j] = a.V[e];
  }
  __syncthreads();
  uint64_t pol_keep, pol_drop;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_drop));
  // one 256-bit load (LDG.256, sm_100): a lane's four contiguous columns; the four lanes of a
  // row cover one whole 128-byte line per instruction
  struct double4v { double x, y, z, w; };
  auto ld4 = [](const double* p, uint64_t pol) {
    double4v v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;\n"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p), "l"(pol));
    return v;
  };
  const int nwn = (int)(n >> 5) / TEAM;  // this warp's mask words per row (n % (32 TEAM) == 0)
  const int team = warp / TEAM, tw = warp % TEAM, nteams = nwarps / TEAM;
  const int64_t wbase = (int64_t)tw * nwn;  // first word of this warp's column range
  // exchange areas behind V-hat: per team and team warp, 8 rows x 8 partial b, 8 counts, 8 residuals
  double* xb = Vs + (((int64_t)n * RS + 1) & ~int64_t(1)) + (int64_t)(team * TEAM) * 80;
  const int64_t rows = a.row_hi - a.row_lo;
  const int64_t nblk = (rows + 7) / 8;
  const int64_t stride = (int64_t)gridDim.x * nteams;
  for (int64_t bi = (int64_t)blockIdx.x * nteams + team; bi < nblk; bi += stride) {
    const int64_t row = a.row_lo + bi * 8 + g;
    const bool valid = row < a.row_hi;
    const int64_t rowc = valid ? row : a.row_hi - 1;  // a partial block re-reads its last row
    const double* yr = a.Y + rowc * n + 32 * wbase;
    const uint32_t* wr = a.bitsR + rowc * a.nwp + wbase;
    // ---- pass 1: b = V_O^T y, observed count ----
    // four independent accumulator pairs (step q of every group feeds pair q):
    // the MMAs of a group do not wait on one another
    double dq[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    int cnt = 0;
    {
      const double* yp = yr + 4 * k;
      const double* vp = Vs + (int64_t)(32 * wbase + 4 * k) * RS + g;
      int w = 0;
      for (; w + UW <= nwn; w += UW) {
        // pull the lines of the step PFD steps ahead toward L2 (no registers
        // held): a row's 16-column group is one 128-byte line, lane k takes
        // groups k, k + 4, ...
        if (w + UW * (PFD + 1) <= nwn) {
#pragma unroll
          for (int j = 0; j < (2 * UW) / 4; ++j)
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(yp - 4 * k + 32 * UW * PFD + 16 * (k + 4 * j)));
        }
        unsigned word[UW];
        double4v y[UW][2];
#pragma unroll
        for (int u = 0; u < UW; ++u) word[u] = __ldg(wr + w + u);
#pragma unroll
        for (int u = 0; u < UW; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h) y[u][h] = ld4(yp + 32 * u + 16 * h, pol_keep);
#pragma unroll
        for (int u = 0; u < UW; ++u) {
          cnt += __popc(word[u]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const unsigned bits = (word[u] >> (16 * h + 4 * k)) & 15u;
            const double yq[4] = {y[u][h].x, y[u][h].y, y[u][h].z, y[u][h].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double aq = ((bits >> q) & 1u) ? yq[q] : 0.0;  // a hidden cell's NaN is selected away
              const double bq = g < R ? vp[(int64_t)(32 * u + 16 * h + q) * RS] : 0.0;
              dmma(dq[q][0], dq[q][1], aq, bq);
            }
          }
        }
        yp += 32 * UW;
        vp += (int64_t)32 * UW * RS;
      }
      for (; w < nwn; ++w) {
        const unsigned word = __ldg(wr + w);
        cnt += __popc(word);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double4v y4 = ld4(yp + 16 * h, pol_keep);
          const unsigned bits = (word >> (16 * h + 4 * k)) & 15u;
          const double yq[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double aq = ((bits >> q) & 1u) ? yq[q] : 0.0;
            const double bq = g < R ? vp[(int64_t)(16 * h + q) * RS] : 0.0;
            dmma(dq[q][0], dq[q][1], aq, bq);
          }
        }
        yp += 32;
        vp += (int64_t)32 * RS;
      }
    }
    double d0 = (dq[0][0] + dq[1][0]) + (dq[2][0] + dq[3][0]);
    double d1 = (dq[0][1] + dq[1][1]) + (dq[2][1] + dq[3][1]);
    if constexpr (TEAM > 1) {
      double* mine = xb + tw * 80;
      mine[g * 8 + 2 * k] = d0;
      mine[g * 8 + 2 * k + 1] = d1;
      if (k == 0) mine[64 + g] = (double)cnt;
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + team), "r"(32 * TEAM) : "memory");
      d0 = 0.0;
      d1 = 0.0;
      double c = 0.0;
#pragma unroll
      for (int t = 0; t < TEAM; ++t) {
        d0 += xb[t * 80 + g * 8 + 2 * k];
        d1 += xb[t * 80 + g * 8 + 2 * k + 1];
        c += xb[t * 80 + 64 + g];
      }
      cnt = (int)c;
    }
    // ---- the rows' solves: lane (g, k) holds b[g][2k], b[g][2k + 1] ----
    double bv[R], A[NA], u[R];
    const double* ap = a.Apre + rowc * NA;
#pragma unroll
    for (int p = 0; p < NA; ++p) A[p] = __ldg(ap + p);
#pragma unroll
    for (int j = 0; j < R; ++j) bv[j] = __shfl_sync(0xffffffffu, (j & 1) ? d1 : d0, (lane & ~3) + (j >> 1));
    bool flagged = row_solve<R>(A, bv, cnt, u);
    if (a.Ugiven) {
#pragma unroll
      for (int q = 0; q < R; ++q) u[q] = a.Ugiven[rowc * R + q];
      flagged = false;
    }
    // ---- pass 2: direct residual from 8 x 8 tiles of U V^T ----
    double ua[NK];
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
      double x = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * kk + q < R && q == k) x = u[4 * kk + q];
      ua[kk] = x;
    }
    double ss = 0.0;
    {
      // the columns of a tile are free too: of a 16-column group, tile 0 takes columns
      // {4j, 4j + 1} and tile 1 {4j + 2, 4j + 3} (j = 0..3), so lane k's two predictions of
      // each tile are its four contiguous columns 4k..4k+3: one 256-bit load per group
      const double* yp = yr + 4 * k;
      const double* vp = Vs + (int64_t)(32 * wbase + 4 * (g >> 1) + (g & 1)) * RS + k;
      auto tiles = [&](unsigned word, const double4v* y, const double* vq) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
          for (int kk = 0; kk < NK; ++kk) {
            const double b0 = (4 * kk + k < R) ? vq[(int64_t)(16 * h) * RS + 4 * kk] : 0.0;
            const double b1 = (4 * kk + k < R) ? vq[(int64_t)(16 * h + 2) * RS + 4 * kk] : 0.0;
            dmma(p0, p1, ua[kk], b0);
            dmma(p2, p3, ua[kk], b1);
          }
          const unsigned bits = (word >> (16 * h + 4 * k)) & 15u;
          if (bits & 1u) {
            const double d = y[h].x - p0;
            ss = fma(d, d, ss);
          }
          if (bits & 2u) {
            const double d = y[h].y - p1;
            ss = fma(d, d, ss);
          }
          if (bits & 4u) {
            const double d = y[h].z - p2;
            ss = fma(d, d, ss);
          }
          if (bits & 8u) {
            const double d = y[h].w - p3;
            ss = fma(d, d, ss);
          }
        }
      };
      int w = 0;
      for (; w + UW <= nwn; w += UW) {
        unsigned word[UW];
        double4v y[UW][2];
#pragma unroll
        for (int u = 0; u < UW; ++u) word[u] = __ldg(wr + w + u);
#pragma unroll
        for (int u = 0; u < UW; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h) y[u][h] = ld4(yp + 32 * u + 16 * h, pol_drop);
#pragma unroll
        for (int u = 0; u < UW; ++u) tiles(word[u], y[u], vp + (int64_t)(32 * u) * RS);
        yp += 32 * UW;
        vp += (int64_t)32 * UW * RS;
      }
      for (; w < nwn; ++w) {
        const unsigned word = __ldg(wr + w);
        double4v y[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) y[h] = ld4(yp + 16 * h, pol_drop);
        tiles(word, y, vp);
        yp += 32;
        vp += (int64_t)32 * RS;
      }
    }
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    if constexpr (TEAM > 1) {
      if (k == 0) xb[tw * 80 + 72 + g] = ss;
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + team), "r"(32 * TEAM) : "memory");
      ss = 0.0;
#pragma unroll
      for (int t = 0; t < TEAM; ++t) ss += xb[t * 80 + 72 + g];
    }
    if (valid && k == 0 && tw == 0) {
      a.rowres[row] = ss;
#pragma unroll
      for (int q = 0; q < R; ++q) a.U[row * R + q] = u[q];
      if (flagged) atomicAdd(a.flagged, 1);
    }
  }
}

// deterministic single-CTA sum of n doubles (fixed strided order + tree)
__global__ void k_sum_rows(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
  __shared__ double part[1024];
  const int tid = threadIdx.x;
  double s = 0.0;
  for (int64_t i = tid; i < n; i += blockDim.x) s += v[i];  // coalesced, fixed order
  part[tid] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (tid < o) part[tid] += part[tid + o];
    __syncthreads();
  }
  if (tid == 0) *out = part[0];
}

// masked residual per row for given factors (core.cpp:15-31): warp per row
__global__ void k_residual(const double* __restrict__ Y, const uint32_t* __restrict__ bitsR, int64_t m,
                           int64_t n, int64_t nwp, const double* __restrict__ U,
                           const double* __restrict__ V, int r, double* __restrict__ rowres) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = gw; row < m; row += nw) {
    double ss = 0.0;
    for (int64_t c = lane; c < n; c += 32) {
      if ((__ldg(bitsR + row * nwp + (c >> 5)) >> (c & 31)) & 1u) {
        double p = 0.0;
        for (int k = 0; k < r; ++k) p = fma(U[row * r + k], V[c * r + k], p);
        const double d = Y[row * n + c] - p;
        ss = fma(d, d, ss);
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) rowres[row] = ss;
  }
}

void launch_residual(const double* Y, const uint32_t* bitsR, int64_t m, int64_t n, int64_t nwp,
                     const double* U, const double* V, int r, double* rowres, cudaStream_t s) {
  int64_t blocks = (m + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_residual<<<(unsigned)blocks, 256, 0, s>>>(Y, bitsR, m, n, nwp, U, V, r, rowres);
}

template <int R, bool VSMEM, int STAGE>
static void launch_solve_u_k(const SolveUArgs& a, size_t fixed, size_t per_warp, int sms, cudaStream_t s) {
  // one CTA per SM with as many warps as shared memory (row buffers) and the
  // register budget allow: V-hat is staged once per SM
  const size_t cap = 227 * 1024 - 2048;  // static shared memory of the kernel
  const int wmax = R <= 4 ? SU_MAXW : 12;
  int w = per_warp ? (int)std::min<size_t>(wmax, (cap - fixed) / per_warp) : wmax;
  if (w < 1) w = 1;
  const size_t smem = fixed + (size_t)w * per_warp;
  ensure_smem((const void*)k_solve_u<R, VSMEM, STAGE>, smem);
  const int64_t rows = a.row_hi - a.row_lo;
  int64_t blocks = std::min<int64_t>((rows + w - 1) / w, (int64_t)sms);
  if (blocks < 1) blocks = 1;
  k_solve_u<R, VSMEM, STAGE><<<(unsigned)blocks, w * 32, smem, s>>>(a);
}

template <int R>
static void launch_solve_u_r(const SolveUArgs& a, cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);  // cached by the runtime
  constexpr int NP = (R + 1) / 2;
  const size_t head = sizeof(double) * 2 * SU_MAXW;  // mbarriers
  const size_t vbytes = sizeof(double) * 2 * NP * (size_t)a.n;
  const size_t bufb = sizeof(double) * (size_t)(((a.n + 1) & ~int64_t(1)) + a.nwp / 2);
  const size_t per_warp = 2 * bufb;
  const size_t cap = 227 * 1024 - 2048;
  const bool bulk = (a.n % 2) == 0;
  static const bool fused_off = [] {
    const char* e = getenv("RSM_SOLVE_U_FUSED");
    return e && atoi(e) == 0;
  }();
  // FP64 tensor-core kernel: tensor-core normal matrices, n a multiple of 32,
  // warps per SM limited so the 8-row blocks awaiting their second read
  // (8 n doubles per warp) stay inside L2
  static const int mma_mode = [] {
    const char* e = getenv("RSM_SU_MMA");
    return e ? atoi(e) : 1;
  }();
  if (a.Apre && mma_mode && (a.n % 32) == 0 && ((uintptr_t)a.Y % 32) == 0) {
    constexpr int RS = R <= 4 ? 5 : 9;
    const size_t vs = sizeof(double) * (size_t)a.n * RS;
    if (vs <= 200 * 1024) {
      static const int wenv = [] {
        const char* e = getenv("RSM_SU_MMA_W");
        return e ? atoi(e) : 0;
      }();
      const int64_t rows = a.row_hi - a.row_lo;
      const int64_t nblk = (rows + 7) / 8;
      {
        // all the warps the register file holds; TEAM warps per 8-row block so the blocks awaiting
        // their second read (8 n doubles per team) fit the L2 budget
        constexpr int WALL = R <= 4 ? 16 : 8;
        static const int tenv = [] {
          const char* e = getenv("RSM_SU_MMA_TEAM");
          return e ? atoi(e) : 0;
        }();
        int team = 1;
        while (team < 4 && (double)(WALL / team) * sms * 8.0 * a.n * 8.0 > 80.0 * 1024 * 1024) team *= 2;
        if (tenv > 0) team = tenv;
        if ((a.n / 32) % team != 0 || WALL % team != 0) team = 1;
        const int wt = wenv > 0 ? std::max(team, (std::min(WALL, wenv) / team) * team) : WALL;
        const size_t smem = vs + 16 + sizeof(double) * 80 * (size_t)wt;
        const int64_t tb = (nblk + wt / team - 1) / (wt / team);
        const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tb, (int64_t)sms));
#define RSM_MMA_LAUNCH(T)                                              \
  {                                                                    \
    ensure_smem((const void*)k_solve_u_mma<R, 4, T>, smem);            \
    k_solve_u_mma<R, 4, T><<<gb, wt * 32, smem, s>>>(a);               \
  }
        if (team == 4) RSM_MMA_LAUNCH(4)
        else if (team == 2) RSM_MMA_LAUNCH(2)
        else RSM_MMA_LAUNCH(1)
#undef RSM_MMA_LAUNCH
        return;
      }
    }
  }
  if (head + vbytes + 8 * per_warp <= cap) {
    // V-hat and >= 8 warps of staged rows
    if constexpr (R <= 4) {
      constexpr int NA = R * (R + 1) / 2;
      const size_t wgram = sizeof(double) * (((size_t)((a.n + 31) / 32) * NA + 1) & ~(size_t)1);
      // tensor-core normal matrices: one staged row per warp (k_solve_u_pre)
      static const bool pre_on = [] {
        const char* e = getenv("RSM_SU_PRE");
        return !(e && atoi(e) == 0);
      }();
      const size_t mwd = (size_t)((a.nwp + 3) & ~int64_t(3)) / 2;
      const size_t per_warp1 = sizeof(double) * ((size_t)a.n + 2 * mwd);
      const size_t headp = sizeof(double) * SU_MAXW;
      if (a.Apre && bulk && pre_on && headp + vbytes + 8 * per_warp1 <= 227 * 1024 - 1024) {
        int w = (int)std::min<size_t>(SU_MAXW, (227 * 1024 - 1024 - headp - vbytes) / per_warp1);
        if (w < 1) w = 1;
        const size_t smem = headp + vbytes + (size_t)w * per_warp1;
        const int64_t rows = a.row_hi - a.row_lo;
        int64_t blocks = std::min<int64_t>((rows + w - 1) / w, (int64_t)sms);
        if (blocks < 1) blocks = 1;
        ensure_smem((const void*)k_solve_u_pre<R>, smem);
        k_solve_u_pre<R><<<(unsigned)blocks, w * 32, smem, s>>>(a);
        return;
      }
      if (bulk && !fused_off && head + vbytes + wgram + 8 * per_warp <= cap) {
        const size_t capw = 227 * 1024 - 1024;  // the kernel has no static shared memory
        int w = (int)std::min<size_t>(SU_MAXW, (capw - head - vbytes - wgram) / per_warp);
        if (w < 1) w = 1;
        const size_t smem = head + vbytes + wgram + (size_t)w * per_warp;
        static const bool walk = [] {
          const char* e = getenv("RSM_SU_WALK");
          return !(e && atoi(e) == 0);
        }();
        const int64_t rows = a.row_hi - a.row_lo;
        int64_t blocks = std::min<int64_t>((rows + w - 1) / w, (int64_t)sms);
        if (blocks < 1) blocks = 1;
        if (walk) {
          ensure_smem((const void*)k_solve_u_fused<R, true>, smem);
          k_solve_u_fused<R, true><<<(unsigned)blocks, w * 32, smem, s>>>(a);
        } else {
          ensure_smem((const void*)k_solve_u_fused<R, false>, smem);
          k_solve_u_fused<R, false><<<(unsigned)blocks, w * 32, smem, s>>>(a);
        }
        return;
      }
    }
    if (bulk) launch_solve_u_k<R, true, 1>(a, head + vbytes, per_warp, sms, s);
    else launch_solve_u_k<R, true, 2>(a, head + vbytes, per_warp, sms, s);
  } else if (head + vbytes <= cap) {
    // V-hat alone fills shared memory: rows are read from global
    static const bool preg_on = [] {
      const char* e = getenv("RSM_SU_PREG");
      return !(e && atoi(e) == 0);
    }();
    if (a.Apre && bulk && preg_on) {
      // tensor-core normal matrices: fused residual/accumulation loop (k_solve_u_preg)
      static const int w = [] {
        const char* e = getenv("RSM_SU_PREG_W");
        return e ? std::max(1, std::min(12, atoi(e))) : 12;
      }();
      static const int pf = [] {
        // bit 2: L2 eviction hints on the two reads of a row (config 4: 8.3 -> 8.1 ms);
        // bits 0-1: bulk L2 prefetch two rows ahead (measured slower: 8.5 ms, the
        // prefetched rows push the rows awaiting their second read out of L2)
        const char* e = getenv("RSM_SU_PF");
        return e ? atoi(e) : 4;
      }();
      SolveUArgs b = a;
      b.pf = pf;
      const int64_t rows = a.row_hi - a.row_lo;
      int64_t blocks = std::min<int64_t>((rows + w - 1) / w, (int64_t)sms);
      if (blocks < 1) blocks = 1;
      ensure_smem((const void*)k_solve_u_preg<R>, vbytes);
      k_solve_u_preg<R><<<(unsigned)blocks, w * 32, vbytes, s>>>(b);
      return;
    }
    launch_solve_u_k<R, true, 0>(a, head + vbytes, 0, sms, s);
  } else {
    if (bulk) launch_solve_u_k<R, false, 1>(a, head, per_warp, sms, s);
    else launch_solve_u_k<R, false, 2>(a, head, per_warp, sms, s);
  }
}

void launch_solve_u(const SolveUArgs& a, cudaStream_t s) {
  switch (a.r) {
    case 1: launch_solve_u_r<1>(a, s); break;
    case 2: launch_solve_u_r<2>(a, s); break;
    case 3: launch_solve_u_r<3>(a, s); break;
    case 4: launch_solve_u_r<4>(a, s); break;
    case 5: launch_solve_u_r<5>(a, s); break;
    case 6: launch_solve_u_r<6>(a, s); break;
    case 7: launch_solve_u_r<7>(a, s); break;
    default: launch_solve_u_r<8>(a, s); break;
  }
}

// two-level deterministic sum for long vectors: SUMP blocks sum fixed
// contiguous chunks (fixed strided order + tree), one thread adds the SUMP
// partials in order
constexpr int SUMP = 64;
__global__ void k_sum_part(const double* __restrict__ v, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void k_sum_final(const double* __restrict__ part, int np, double* __restrict__ out) {
  double s = 0.0;
  for (int i = 0; i < np; ++i) s += part[i];
  *out = s;
}

// both levels in one launch: the block that arrives last (arrival counter, 0
// on entry) adds the SUMP partials in index order -- the same fixed order as
// k_sum_final, whichever block that is
__global__ void k_sum_part_final(const double* __restrict__ v, int64_t n, double* __restrict__ part,
                                 double* __restrict__ out, unsigned* __restrict__ counter) {
  __shared__ double red[256];
  __shared__ bool last;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = red[0];
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    // lane l loads partials l and l + 32 (SUMP = 64); lane 0 adds them in index order
    const volatile double* pv = part;
    const double a0 = pv[threadIdx.x], a1 = pv[threadIdx.x + 32];
    double t = 0.0;
    for (int i = 0; i < 32; ++i) t += __shfl_sync(0xffffffffu, a0, i);
    for (int i = 0; i < 32; ++i) t += __shfl_sync(0xffffffffu, a1, i);
    if (threadIdx.x == 0) {
      *out = t;
      *counter = 0u;
    }
  }
}

// out[0] = sum of v[0..n); out must have room for 2 + SUMP doubles (partials).
// counter (optional): a device word that is 0 on entry -- the two-level sum
// then runs as one launch (the last block to arrive finishes it)
int launch_sum_rows(const double* v, int64_t n, double* out, cudaStream_t s, unsigned* counter) {
  if (n <= 32768) {
    k_sum_rows<<<1, 1024, 0, s>>>(v, n, out);
    return 1;
  }
  if (counter) {
    static_assert(SUMP == 64, "k_sum_part_final's final pass");
    k_sum_part_final<<<SUMP, 256, 0, s>>>(v, n, out + 2, out, counter);
    return 1;
  }
  k_sum_part<<<SUMP, 256, 0, s>>>(v, n, out + 2);
  k_sum_final<<<1, 1, 0, s>>>(out + 2, SUMP, out);
  return 2;
}

}  // namespace rsmk
