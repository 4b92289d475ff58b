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

#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

using namespace rsmd;

namespace {

constexpr int SU_WARPS = 4;

template <int R>
struct RowAcc {
  static constexpr int NP = R * (R + 1) / 2;
  double A[NP];
  double b[R];
  int nj;
};

template <int R>
__device__ __forceinline__ void acc_add(RowAcc<R>& s, const double* v, double y) {
  int p = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
#pragma unroll
    for (int j = i; j < R; ++j) {
      s.A[p] = fma(v[i], v[j], s.A[p]);
      ++p;
    }
    s.b[i] = fma(y, v[i], s.b[i]);
  }
  ++s.nj;
}

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

// issue the copies of one row (values + mask words) into a warp buffer
__device__ __forceinline__ void issue_row(const SolveUArgs& a, int64_t row, double* ybuf, uint32_t* wbuf,
                                          bool vec16) {
  const int lane = threadIdx.x & 31;
  const double* y = a.Y + row * a.n;
  if (vec16) {
    for (int64_t c = lane; c < a.n / 2; c += 32) cp_async(ybuf + 2 * c, y + 2 * c, 1);
  } else {
    for (int64_t c = lane; c < a.n; c += 32) cp_async(ybuf + c, y + c, 0);
  }
  const uint32_t* w = a.bitsR + row * a.nwp;  // nwp is a multiple of 4 words
  for (int64_t c = lane; c < a.nwp / 4; c += 32) cp_async(wbuf + 4 * c, w + 4 * c, 1);
  asm volatile("cp.async.commit_group;\n" ::);
}

}  // namespace

template <int R, bool VSMEM>
__global__ void __launch_bounds__(SU_WARPS * 32) k_solve_u(SolveUArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t npd = (n + 1) & ~int64_t(1);
  double* Vs = sm;
  double* wb = sm + (VSMEM ? ((n * R + 1) & ~int64_t(1)) : 0);
  const int64_t bufd = npd + a.nwp / 2;  // doubles per row buffer (values + words)
  double* yb0 = wb + (2 * warp) * bufd;
  double* yb1 = wb + (2 * warp + 1) * bufd;
  // V in shared memory is stored component-major (Vs[k*n + c]) so the 32
  // lanes of a warp, which own 32 consecutive columns, read consecutive words
  if (VSMEM) {
    for (int64_t e = threadIdx.x; e < n * R; e += blockDim.x) Vs[(e % R) * n + e / R] = a.V[e];
    __syncthreads();
  }
  auto vrow = [&](int64_t c, double* v) {
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = VSMEM ? Vs[k * n + c] : __ldg(a.V + c * R + k);
  };
  const bool vec16 = (n % 2) == 0;
  const int64_t gw = (int64_t)blockIdx.x * SU_WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * SU_WARPS;
  int cur = 0;
  int64_t row = a.row_lo + gw;
  if (row < a.row_hi) issue_row(a, row, yb0, reinterpret_cast<uint32_t*>(yb0 + npd), vec16);
  for (; row < a.row_hi; row += nw) {
    double* ycur = cur ? yb1 : yb0;
    double* ynxt = cur ? yb0 : yb1;
    const int64_t nxt = row + nw;
    if (nxt < a.row_hi) {
      issue_row(a, nxt, ynxt, reinterpret_cast<uint32_t*>(ynxt + npd), vec16);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncwarp();
    const double* y = ycur;
    const uint32_t* wd = reinterpret_cast<const uint32_t*>(ycur + npd);
    RowAcc<R> s;
#pragma unroll
    for (int p = 0; p < RowAcc<R>::NP; ++p) s.A[p] = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) s.b[i] = 0.0;
    s.nj = 0;
    // branchless: unknown cells contribute zero vectors (selected, never
    // multiplied, so the NaN at hidden cells never enters arithmetic)
    const int nfull = (int)(n >> 5);
    for (int w = 0; w < nfull; ++w) {
      const int c = w * 32 + lane;
      const bool k = (wd[w] >> lane) & 1u;
      double v[R];
      vrow(c, v);
#pragma unroll
      for (int q = 0; q < R; ++q) v[q] = k ? v[q] : 0.0;
      acc_add<R>(s, v, k ? y[c] : 0.0);
      s.nj += k ? 0 : -1;  // acc_add counted one
    }
    if ((int64_t)nfull * 32 + lane < n && ((wd[nfull] >> lane) & 1u)) {
      const int c = nfull * 32 + lane;
      double v[R];
      vrow(c, v);
      acc_add<R>(s, v, y[c]);
    }
    // butterfly reduction: every lane ends with the row totals
#pragma unroll
    for (int p = 0; p < RowAcc<R>::NP; ++p) s.A[p] = warp_sum(s.A[p]);
#pragma unroll
    for (int i = 0; i < R; ++i) s.b[i] = warp_sum(s.b[i]);
    const int nj = warp_sum_int(s.nj);

    double u[R];
    bool flagged = false;
    bool slow = nj < R;
    if (!slow) {
      // Cholesky of the packed normal matrix (lower factor, row-major packed)
      double L[RowAcc<R>::NP];
      double dmax = 0.0;
#pragma unroll
      for (int i = 0; i < R; ++i) dmax = fmax(dmax, s.A[i * R - i * (i - 1) / 2]);
      int q = 0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
          double v = s.A[j * R - j * (j - 1) / 2 + (i - j)];
#pragma unroll
          for (int k = 0; k < j; ++k) v -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
          if (i == j) {
            if (!(v > 1e-10 * dmax)) slow = true;
            L[q] = sqrt(fmax(v, 0.0));
          } else {
            L[q] = v / L[j * (j + 1) / 2 + j];
          }
          ++q;
        }
      }
      if (!slow) {
        double z[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          double v = s.b[i];
#pragma unroll
          for (int k = 0; k < i; ++k) v -= L[i * (i + 1) / 2 + k] * z[k];
          z[i] = v / L[i * (i + 1) / 2 + i];
        }
#pragma unroll
        for (int i = R - 1; i >= 0; --i) {
          double v = z[i];
#pragma unroll
          for (int k = i + 1; k < R; ++k) v -= L[k * (k + 1) / 2 + i] * u[k];
          u[i] = v / L[i * (i + 1) / 2 + i];
        }
      }
    }
    if (slow) {
      const int rank = pinv_solve<R>(s.A, s.b, u);
      flagged = (nj < R) || (rank < R);
    }
    // second pass over the row still in shared memory: direct residual
    double ss = 0.0;
    for (int w = 0; w < nfull; ++w) {
      const int c = w * 32 + lane;
      const bool k = (wd[w] >> lane) & 1u;
      double v[R];
      vrow(c, v);
      double p = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) p = fma(u[q], v[q], p);
      const double d = k ? y[c] - p : 0.0;
      ss = fma(d, d, ss);
    }
    if ((int64_t)nfull * 32 + lane < n && ((wd[nfull] >> lane) & 1u)) {
      const int c = nfull * 32 + lane;
      double v[R];
      vrow(c, v);
      double p = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) p = fma(u[q], v[q], p);
      const double d = y[c] - p;
      ss = fma(d, d, ss);
    }
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

template <int R>
static void launch_solve_u_r(const SolveUArgs& a, cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t vbytes = sizeof(double) * (size_t)(((a.n * R) + 1) & ~int64_t(1));
  const size_t bufb = sizeof(double) * (size_t)(((a.n + 1) & ~int64_t(1)) + a.nwp / 2);
  const size_t rows_b = (size_t)SU_WARPS * 2 * bufb;
  const bool vsm = vbytes + rows_b <= 112 * 1024;
  const size_t smem = rows_b + (vsm ? vbytes : 0);
  const int64_t rows = a.row_hi - a.row_lo;
  int occ = 0;
  if (vsm) {
    cudaFuncSetAttribute(k_solve_u<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_solve_u<R, true>, SU_WARPS * 32, smem);
  } else {
    cudaFuncSetAttribute(k_solve_u<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_solve_u<R, false>, SU_WARPS * 32, smem);
  }
  if (occ < 1) occ = 1;
  int64_t blocks = std::min<int64_t>((rows + SU_WARPS - 1) / SU_WARPS, (int64_t)sms * occ);
  if (blocks < 1) blocks = 1;
  if (vsm) k_solve_u<R, true><<<(unsigned)blocks, SU_WARPS * 32, smem, s>>>(a);
  else k_solve_u<R, false><<<(unsigned)blocks, SU_WARPS * 32, smem, s>>>(a);
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

void launch_sum_rows(const double* v, int64_t n, double* out, cudaStream_t s) {
  k_sum_rows<<<1, 1024, 0, s>>>(v, n, out);
}

}  // namespace rsmk
