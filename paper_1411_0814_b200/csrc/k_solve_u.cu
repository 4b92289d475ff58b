// k_solve_u.cu -- stage 5: per-row masked least squares for U and the
// masked residual e.
//
// Reference: solve_u (solver.cpp:64-89, paths relative to
// /root/reference/proj) runs detail::solve_row (detail/row_solve.hpp:12-36)
// per row: gather V rows at the observed columns, complete orthogonal
// decomposition, minimum-norm solution; the row is counted as
// underdetermined when it has fewer than r observations or the basis
// restricted to them is rank deficient; an empty row gets zeros. Here one
// warp owns a row: it streams the row of Y once with 128-bit loads, selects
// through the bit-packed mask (hidden cells hold NaN and are never read into
// arithmetic), accumulates the r x r normal matrix V_O^T V_O and V_O^T y,
// reduces them across the warp and solves by Cholesky in registers. Rows
// whose normal matrix is singular or ill-conditioned fall back to an
// eigendecomposition pseudo-inverse (the minimum-norm solution, as the COD
// gives). The residual of e (masked_residual_norm, core.cpp:15-39) is formed
// directly as sum (y - u.v)^2 in a second pass over the (L1/L2-resident)
// row, never by the cancelling ||y||^2 - u^T b shortcut.
#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

using namespace rsmd;

namespace {

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

}  // namespace

template <int R, bool VSMEM, bool VEC2>
__global__ void __launch_bounds__(256) k_solve_u(SolveUArgs a) {
  extern __shared__ __align__(16) double Vs[];
  const int lane = threadIdx.x & 31;
  const int64_t n = a.n;
  const double* Vp = a.V;
  if (VSMEM) {
    for (int64_t e = threadIdx.x; e < n * R; e += blockDim.x) Vs[e] = a.V[e];
    __syncthreads();
    Vp = Vs;
  }
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = a.row_lo + gw; row < a.row_hi; row += nw) {
    const double* y = a.Y + row * n;
    const uint32_t* mb = a.bitsR + row * a.nwp;
    RowAcc<R> s;
#pragma unroll
    for (int p = 0; p < RowAcc<R>::NP; ++p) s.A[p] = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) s.b[i] = 0.0;
    s.nj = 0;
    if (VEC2) {
      for (int64_t c0 = 2 * lane; c0 < n; c0 += 64) {
        const uint32_t w = __ldg(mb + (c0 >> 5));
        const uint32_t sh = (uint32_t)(c0 & 31);
        const bool k0 = (w >> sh) & 1u, k1 = (w >> (sh + 1)) & 1u;
        if (k0 | k1) {
          const double2 yy = __ldg(reinterpret_cast<const double2*>(y + c0));
          if (k0) acc_add<R>(s, Vp + c0 * R, yy.x);
          if (k1) acc_add<R>(s, Vp + (c0 + 1) * R, yy.y);
        }
      }
    } else {
      for (int64_t c = lane; c < n; c += 32) {
        const uint32_t w = __ldg(mb + (c >> 5));
        if ((w >> (c & 31)) & 1u) acc_add<R>(s, Vp + c * R, __ldg(y + c));
      }
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
          // A(i,j) with i >= j from the upper packing (j, i)
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
    // second pass: direct residual over the known cells
    double ss = 0.0;
    if (VEC2) {
      for (int64_t c0 = 2 * lane; c0 < n; c0 += 64) {
        const uint32_t w = __ldg(mb + (c0 >> 5));
        const uint32_t sh = (uint32_t)(c0 & 31);
        const bool k0 = (w >> sh) & 1u, k1 = (w >> (sh + 1)) & 1u;
        if (k0 | k1) {
          const double2 yy = __ldg(reinterpret_cast<const double2*>(y + c0));
          if (k0) {
            double p = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) p = fma(u[k], Vp[c0 * R + k], p);
            const double d = yy.x - p;
            ss = fma(d, d, ss);
          }
          if (k1) {
            double p = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) p = fma(u[k], Vp[(c0 + 1) * R + k], p);
            const double d = yy.y - p;
            ss = fma(d, d, ss);
          }
        }
      }
    } else {
      for (int64_t c = lane; c < n; c += 32) {
        const uint32_t w = __ldg(mb + (c >> 5));
        if ((w >> (c & 31)) & 1u) {
          double p = 0.0;
#pragma unroll
          for (int k = 0; k < R; ++k) p = fma(u[k], Vp[c * R + k], p);
          const double d = __ldg(y + c) - p;
          ss = fma(d, d, ss);
        }
      }
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
  const size_t vbytes = (size_t)a.n * R * sizeof(double);
  const bool vsm = vbytes <= 96 * 1024;
  const bool vec2 = (a.n % 2) == 0;
  const int64_t rows = a.row_hi - a.row_lo;
  int64_t blocks = (rows + 7) / 8;
  const int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const size_t smem = vsm ? vbytes : 0;
#define RSM_SU(VS, V2)                                                                          \
  do {                                                                                          \
    cudaFuncSetAttribute(k_solve_u<R, VS, V2>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                         (int)smem);                                                            \
    k_solve_u<R, VS, V2><<<(unsigned)blocks, 256, smem, s>>>(a);                                \
  } while (0)
  if (vsm && vec2) RSM_SU(true, true);
  else if (vsm) RSM_SU(true, false);
  else if (vec2) RSM_SU(false, true);
  else RSM_SU(false, false);
#undef RSM_SU
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
