// k_svd.cu -- stage 2: gather of each accepted submatrix and its top right
// singular vectors by one-sided (Hestenes) Jacobi in shared memory, FP64.
//
// Reference: small_singular_vectors (spectra.cpp:48-86, paths relative to
// /root/reference/proj) harvests the ell smallest right singular vectors of S
// from a full-V JacobiSVD; attempt_trial (harvest.cpp:37-51) takes
// ell = cols - rank for the row branch and ell = block - rank for the column
// branch. Their outer products sum to  I - V_top V_top^T  over the trial's
// column support, where V_top holds the q - ell top right singular vectors
// (q = number of columns of S). So this kernel only produces V_top; stage 3
// accumulates the identity form.
//
// The K "vectors" rotated by the Jacobi are the K rows of S for the row
// branch (S is K x q, K = k) and the K columns of S for the column branch
// (S is q_rows x K, K = l). Each outer iteration recomputes their K x K Gram
// from the data in shared memory, diagonalises it with the warp-parallel
// cyclic Jacobi and applies the rotation to the vectors; it stops when the
// recomputed Gram is diagonal to working precision (the one-sided Jacobi
// convergence test), so accuracy is that of one-sided Jacobi, not of the
// squared Gram.
//
// Also emits, per trial, the column-support bit words and their exclusive
// popcount prefix (the compact-index map stage 3 needs), and the per-column
// trial counts (the identity's diagonal) with integer atomics.
#include <algorithm>
#include <type_traits>

#include "rsm_internal.h"
#include "rsm_dev.cuh"

using rsmd::emit_slices4;

namespace rsmk {

using namespace rsmd;

namespace {

// exclusive popcount prefix of nwords words, by warp 0; returns total in *tot
__device__ void warp0_popc_scan(const uint32_t* words, uint32_t* pre, int64_t nwords,
                                int* tot) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int64_t per = (nwords + 31) / 32;
  const int64_t lo = lane * per;
  const int64_t hi = lo + per < nwords ? lo + per : nwords;
  int s = 0;
  for (int64_t w = lo; w < hi; ++w) s += __popc(words[w]);
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  int run = incl - s;
  for (int64_t w = lo; w < hi; ++w) {
    pre[w] = (uint32_t)run;
    run += __popc(words[w]);
  }
  if (lane == 31) *tot = incl;
}

}  // namespace

constexpr int SVD_GRED_PER_WARP = 36;  // K(K+1)/2 Gram partials per warp (K <= 8)
static_assert(4 * 45 <= KMAX * KMAX, "row-branch partials (4 warps, K <= 9) fit in Tmp");

// Gram of the K vectors (K x L, leading dimension Lp) in one pass: each
// thread accumulates all K(K+1)/2 products over its columns, warps reduce by
// recursive halving, lane-holders publish per-warp partials, and threads
// p < K(K+1)/2 sum them in warp order (deterministic). Writes the full
// symmetric K x K into gram (leading dimension KMAX).
template <int K>
__device__ __noinline__ void cta_gram_1pass(const double* vec, int64_t Lp, int64_t L, double* gram, double* gred) {
  constexpr int P = K * (K + 1) / 2;
  constexpr int NV = P <= 4 ? 4 : (P <= 8 ? 8 : (P <= 16 ? 16 : (P <= 32 ? 32 : 64)));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  double g[NV];
#pragma unroll
  for (int p = 0; p < NV; ++p) g[p] = 0.0;
  for (int64_t c = tid; c < L; c += blockDim.x) {
    double x[K];
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = vec[i * Lp + c];
    int p = 0;
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = i; j < K; ++j) {
        g[p] = fma(x[i], x[j], g[p]);
        ++p;
      }
  }
  warp_reduce_halving<NV>(g, lane);
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const double t = warp_total<NV>(g, p);
    if (lane == 0) gred[warp * P + p] = t;
  }
  __syncthreads();
  if (tid < P) {
    double t = 0.0;
    for (int w = 0; w < nwarps; ++w) t += gred[w * P + tid];
    int i = 0, rem = tid;
    while (rem >= K - i) {
      rem -= K - i;
      ++i;
    }
    const int j = i + rem;
    gram[i * KMAX + j] = t;
    gram[j * KMAX + i] = t;
  }
}

// vectors <- W^T vectors (W is K x K, leading dimension KMAX), thread per column
template <int K>
__device__ __noinline__ void cta_rotate(double* vec, int64_t Lp, int64_t L, const double* W) {
  for (int64_t c = threadIdx.x; c < L; c += blockDim.x) {
    double x[K];
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = vec[i * Lp + c];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double y = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) y += W[i * KMAX + j] * x[i];
      vec[j * Lp + c] = y;
    }
  }
}

// Row branch gather in the CTA-per-trial kernel: the K drawn rows' values at
// four support columns per thread are loaded before any is stored (one memory
// round trip per batch), the column counts are bumped as before.
template <int K>
__device__ __noinline__ void cta_gather_rows(const double* __restrict__ Y, int64_t n, const int* idx,
                                             const uint32_t* cm, const uint32_t* pre, double* vec, int64_t Lp,
                                             int* colcnt) {
  constexpr int B = 4;
  int64_t rowoff[K];
#pragma unroll
  for (int i = 0; i < K; ++i) rowoff[i] = (int64_t)idx[i] * n;
  for (int64_t j0 = threadIdx.x; j0 < n; j0 += (int64_t)B * blockDim.x) {
    double x[B][K];
    int64_t cpos[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int64_t j = j0 + (int64_t)q * blockDim.x;
      cpos[q] = -1;
      if (j < n) {
        const uint32_t word = cm[j >> 5], bit = 1u << (j & 31);
        if (word & bit) cpos[q] = pre[j >> 5] + __popc(word & (bit - 1u));
      }
#pragma unroll
      for (int i = 0; i < K; ++i) x[q][i] = cpos[q] >= 0 ? __ldg(Y + rowoff[i] + j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < B; ++q)
      if (cpos[q] >= 0) {
#pragma unroll
        for (int i = 0; i < K; ++i) vec[i * Lp + cpos[q]] = x[q][i];
        atomicAdd(colcnt + j0 + (int64_t)q * blockDim.x, 1);
      }
  }
}

// Column branch gather: vector j of S^T is column idx[j] over the surviving
// rows. Each thread walks its mask words' set bits four rows at a time and
// issues the 4 K loads of a batch before storing any, so a batch costs one
// memory round trip instead of four (the rows are random: every load is its
// own sector).
template <int K>
__device__ __noinline__ void cta_gather_cols(const double* __restrict__ Y, int64_t n, int64_t mwp, const int* idx,
                                             const uint32_t* rw, const uint32_t* rp, double* vec, int64_t Lp) {
  constexpr int B = 4;
  int col[K];
#pragma unroll
  for (int j = 0; j < K; ++j) col[j] = idx[j];
  for (int64_t w = threadIdx.x; w < mwp; w += blockDim.x) {
    uint32_t word = rw[w];
    int64_t c = rp[w];
    while (word) {
      int64_t rows[B];
      int nb = 0;
#pragma unroll
      for (int q = 0; q < B; ++q) {
        rows[q] = -1;
        if (word) {
          rows[q] = w * 32 + (__ffs(word) - 1);
          word &= word - 1;
          nb = q + 1;
        }
      }
      double x[B][K];
#pragma unroll
      for (int q = 0; q < B; ++q)
#pragma unroll
        for (int j = 0; j < K; ++j) x[q][j] = rows[q] >= 0 ? __ldg(Y + rows[q] * n + col[j]) : 0.0;
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (q < nb) {
#pragma unroll
          for (int j = 0; j < K; ++j) vec[j * Lp + c + q] = x[q][j];
        }
      c += nb;
    }
  }
}

// Column branch gather with the l x l Gram accumulated on the way (the r = l - 1
// path needs nothing else from the vectors: see perp_basis_small), nothing
// stored. Same walk as cta_gather_cols; the per-thread partials are reduced as
// in cta_gram_1pass (fixed order). Ends with the Gram published in `gram`
// (the caller synchronises).
template <int K>
__device__ __noinline__ void cta_gather_cols_gram(const double* __restrict__ Y, int64_t n, int64_t mwp,
                                                  const int* idx, const uint32_t* rw, double* gram,
                                                  double* gred) {
  constexpr int B = 4;
  constexpr int P = K * (K + 1) / 2;
  constexpr int NV = P <= 4 ? 4 : (P <= 8 ? 8 : (P <= 16 ? 16 : (P <= 32 ? 32 : 64)));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  int col[K];
#pragma unroll
  for (int j = 0; j < K; ++j) col[j] = idx[j];
  double g[NV];
#pragma unroll
  for (int p = 0; p < NV; ++p) g[p] = 0.0;
  for (int64_t w = tid; w < mwp; w += blockDim.x) {
    uint32_t word = rw[w];
    while (word) {
      int64_t rows[B];
#pragma unroll
      for (int q = 0; q < B; ++q) {
        rows[q] = -1;
        if (word) {
          rows[q] = w * 32 + (__ffs(word) - 1);
          word &= word - 1;
        }
      }
      double x[B][K];
#pragma unroll
      for (int q = 0; q < B; ++q)
#pragma unroll
        for (int j = 0; j < K; ++j) x[q][j] = rows[q] >= 0 ? __ldg(Y + rows[q] * n + col[j]) : 0.0;
#pragma unroll
      for (int q = 0; q < B; ++q) {
        int p = 0;
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int j = i; j < K; ++j) {
            g[p] = fma(x[q][i], x[q][j], g[p]);
            ++p;
          }
      }
    }
  }
  warp_reduce_halving<NV>(g, lane);
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const double t = warp_total<NV>(g, p);
    if (lane == 0) gred[warp * P + p] = t;
  }
  __syncthreads();
  if (tid < P) {
    double t = 0.0;
    for (int w = 0; w < nwarps; ++w) t += gred[w * P + tid];
    int i = 0, rem = tid;
    while (rem >= K - i) {
      rem -= K - i;
      ++i;
    }
    const int j = i + rem;
    gram[i * KMAX + j] = t;
    gram[j * KMAX + i] = t;
  }
}

// threads per CTA: the column branch keeps a trial's vectors out of shared
// memory (Gram accumulated while gathering; the Jacobi fallback's vectors go
// to global scratch unless RSM_SVD_COL_SMEM=1), so four 128-thread trials
// share an SM and one trial's serial parts hide under the others' gathers
// (config 2: 512 threads 1.01 ms, 256 0.84, 128 0.80, 64 0.85 before the
// Gram moved into the gather)
#ifndef RSM_SVD_COL_THREADS
#define RSM_SVD_COL_THREADS 128
#endif
template <bool M2>
constexpr int svd_cta_threads() { return M2 ? 128 : RSM_SVD_COL_THREADS; }

template <int K>
__device__ __noinline__ bool topr_basis_small(const double* Gsm, double* C);
template <int K>
__device__ __noinline__ bool perp_basis_small(const double* Gsm, double* Q, int ldq);

__device__ __forceinline__ bool it_fast(const int* flags) { return flags[3] != 0; }

// runtime-K dispatch of topr_basis_small (row-branch CTA kernel, K <= 9)
__device__ __noinline__ bool topr_basis_rt(int K, const double* Gsm, double* C) {
  switch (K) {
    case 2: return topr_basis_small<2>(Gsm, C);
    case 3: return topr_basis_small<3>(Gsm, C);
    case 4: return topr_basis_small<4>(Gsm, C);
    case 5: return topr_basis_small<5>(Gsm, C);
    case 6: return topr_basis_small<6>(Gsm, C);
    case 7: return topr_basis_small<7>(Gsm, C);
    case 8: return topr_basis_small<8>(Gsm, C);
    case 9: return topr_basis_small<9>(Gsm, C);
    default: return false;
  }
}

// runtime-K dispatch of perp_basis_small (column-branch CTA kernel, K = l <= 8)
__device__ __noinline__ bool perp_basis_rt(int K, const double* Gsm, double* Q, int ldq) {
  switch (K) {
    case 2: return perp_basis_small<2>(Gsm, Q, ldq);
    case 3: return perp_basis_small<3>(Gsm, Q, ldq);
    case 4: return perp_basis_small<4>(Gsm, Q, ldq);
    case 5: return perp_basis_small<5>(Gsm, Q, ldq);
    case 6: return perp_basis_small<6>(Gsm, Q, ldq);
    case 7: return perp_basis_small<7>(Gsm, Q, ldq);
    case 8: return perp_basis_small<8>(Gsm, Q, ldq);
    default: return false;
  }
}

template <bool M2>
__global__ void __launch_bounds__(svd_cta_threads<M2>(), M2 ? 3 : (512 / RSM_SVD_COL_THREADS)) k_svd(SvdArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
  const int K = a.block;
  const int64_t Lp = a.Lpad;

  // shared layout
  double* gram = reinterpret_cast<double*>(smem_raw);  // KMAX*KMAX
  double* W = gram + KMAX * KMAX;                       // KMAX*KMAX
  double* Vacc = W + KMAX * KMAX;                       // KMAX*KMAX (column branch)
  double* Tmp = Vacc + KMAX * KMAX;                     // KMAX*KMAX
  // per-warp Gram partials (warps x 36): the row branch's 4 warps alias Tmp
  // (free during the Gram); the column branch's 16 warps get their own region
  double* gred = M2 ? Tmp : Tmp + KMAX * KMAX;
  double* cs = Tmp + KMAX * KMAX + (M2 ? 0 : (svd_cta_threads<M2>() / 32) * SVD_GRED_PER_WARP);  // 64
  double* sig = cs + 64;                                // KMAX
  int* pairs = reinterpret_cast<int*>(sig + KMAX);      // 64
  int* ord = pairs + 64;                                // KMAX
  int* idx = ord + KMAX;                                // KMAX
  int* flags = idx + KMAX;                              // 4
  uint32_t* cm = reinterpret_cast<uint32_t*>(flags + 4);  // cmw
  uint32_t* pre = cm + a.cmw;                             // cmw
  double* vec;
  {
    size_t off = (size_t)(reinterpret_cast<unsigned char*>(pre + a.cmw) - smem_raw);
    off = (off + 15) & ~(size_t)15;
    vec = a.use_smem ? reinterpret_cast<double*>(smem_raw + off)
                     : a.scratch + (size_t)blockIdx.x * K * Lp;
  }
  uint32_t* rw = a.scratch_u32 + (size_t)blockIdx.x * 2 * a.mwp;  // column branch only
  uint32_t* rp = rw + a.mwp;

  const int64_t t_end = a.sel_acc ? min(a.t_hi, (int64_t)*a.sel_acc) : a.t_hi;
  for (int64_t t = a.t_lo + blockIdx.x; t < t_end; t += gridDim.x) {
    const int64_t tl = t - a.t_lo;  // local index for outputs
    bool colfast = false;            // column branch: basis taken straight from the gathered Gram
    if (tid < K) idx[tid] = a.t_idx[t * K + tid];
    __syncthreads();
    int64_t L;  // vector length
    if (M2) {
      // column support: AND of the K drawn rows' words (sampler.cpp:65-74)
      for (int64_t w = tid; w < a.cmw; w += nth) {
        uint32_t acc = 0;
        if (w < a.nwp) {
          acc = 0xffffffffu;
          for (int i = 0; i < K; ++i) acc &= __ldg(a.bitsR + (int64_t)idx[i] * a.nwp + w);
        }
        cm[w] = acc;
      }
      __syncthreads();
      warp0_popc_scan(cm, pre, a.cmw, &flags[0]);
      __syncthreads();
      L = flags[0];
      if (L > a.Lcap) continue;  // speculative launch only (uniform: L is in shared memory)
      for (int64_t w = tid; w < a.cmw; w += nth) a.t_cm[tl * a.cmw + w] = cm[w];
      // gather S (K x L) row-major into vec (sampler.cpp:80-84)
      if (K >= 2 && K <= 9) {
        switch (K) {
          case 2: cta_gather_rows<2>(a.Y, a.n, idx, cm, pre, vec, Lp, a.colcnt); break;
          case 3: cta_gather_rows<3>(a.Y, a.n, idx, cm, pre, vec, Lp, a.colcnt); break;
          case 4: cta_gather_rows<4>(a.Y, a.n, idx, cm, pre, vec, Lp, a.colcnt); break;
          case 5: cta_gather_rows<5>(a.Y, a.n, idx, cm, pre, vec, Lp, a.colcnt); break;
          case 6: cta_gather_rows<6>(a.Y, a.n, idx, cm, pre, vec, Lp, a.colcnt); break;
          case 7: cta_gather_rows<7>(a.Y, a.n, idx, cm, pre, vec, Lp, a.colcnt); break;
          case 8: cta_gather_rows<8>(a.Y, a.n, idx, cm, pre, vec, Lp, a.colcnt); break;
          default: cta_gather_rows<9>(a.Y, a.n, idx, cm, pre, vec, Lp, a.colcnt); break;
        }
      } else
      for (int64_t j = tid; j < a.n; j += nth) {
        const uint32_t word = cm[j >> 5];
        const uint32_t bit = 1u << (j & 31);
        if (word & bit) {
          const int64_t c = pre[j >> 5] + __popc(word & (bit - 1u));
          for (int i = 0; i < K; ++i) vec[i * Lp + c] = __ldg(a.Y + (int64_t)idx[i] * a.n + j);
          atomicAdd(a.colcnt + j, 1);
        }
      }
    } else {
      // column support = the K drawn columns
      for (int64_t w = tid; w < a.cmw; w += nth) cm[w] = 0;
      __syncthreads();
      if (tid < K) atomicOr(&cm[idx[tid] >> 5], 1u << (idx[tid] & 31));
      __syncthreads();
      warp0_popc_scan(cm, pre, a.cmw, &flags[1]);
      __syncthreads();
      for (int64_t w = tid; w < a.cmw; w += nth) a.t_cm[tl * a.cmw + w] = cm[w];
      if (tid < K) atomicAdd(a.colcnt + idx[tid], 1);
      // surviving rows: AND of the K columns' words (sampler.cpp:34-43)
      for (int64_t w = tid; w < a.mwp; w += nth) {
        uint32_t acc = 0xffffffffu;
        for (int j = 0; j < K; ++j) acc &= __ldg(a.bitsC + (int64_t)idx[j] * a.mwp + w);
        rw[w] = acc;
      }
      __syncthreads();
      warp0_popc_scan(rw, rp, a.mwp, &flags[0]);
      __syncthreads();
      L = flags[0];
      if (L > a.Lcap) continue;  // speculative launch only (uniform: L is in shared memory)
      // r = l - 1: the right singular vectors of the q x l submatrix are the
      // eigenvectors of its l x l Gram, and stage 3 consumes only the
      // projector on the top r of them = I - u u^T, u the smallest
      // eigenvector. Any orthonormal basis of u-perp serves
      // (perp_basis_small: inverse iteration + Householder complement by one
      // lane), so the Gram is accumulated while gathering and the vectors are
      // never stored; without a clear gap the trial is gathered again for
      // the one-sided Jacobi below.
      if (a.fast_basis && a.rex == K - 1 && K >= 2 && K <= 8) {
        switch (K) {
          case 2: cta_gather_cols_gram<2>(a.Y, a.n, a.mwp, idx, rw, gram, gred); break;
          case 3: cta_gather_cols_gram<3>(a.Y, a.n, a.mwp, idx, rw, gram, gred); break;
          case 4: cta_gather_cols_gram<4>(a.Y, a.n, a.mwp, idx, rw, gram, gred); break;
          case 5: cta_gather_cols_gram<5>(a.Y, a.n, a.mwp, idx, rw, gram, gred); break;
          case 6: cta_gather_cols_gram<6>(a.Y, a.n, a.mwp, idx, rw, gram, gred); break;
          case 7: cta_gather_cols_gram<7>(a.Y, a.n, a.mwp, idx, rw, gram, gred); break;
          default: cta_gather_cols_gram<8>(a.Y, a.n, a.mwp, idx, rw, gram, gred); break;
        }
        __syncthreads();
        if (tid == 0) {
          int p = 0;
          for (int i = 0; i < K; ++i)
            for (int j = i; j < K; ++j) Tmp[p++] = gram[i * KMAX + j];
          flags[3] = perp_basis_rt(K, Tmp, Vacc, KMAX) ? 1 : 0;
          if (flags[3])
            for (int i = 0; i < K; ++i) ord[i] = i;
        }
        __syncthreads();
        colfast = flags[3] != 0;
      }
      if (colfast) {
      } else
      // gather S^T (K x L): vector j = column idx[j] over surviving rows
      if (K >= 2 && K <= 8) {
        switch (K) {
          case 2: cta_gather_cols<2>(a.Y, a.n, a.mwp, idx, rw, rp, vec, Lp); break;
          case 3: cta_gather_cols<3>(a.Y, a.n, a.mwp, idx, rw, rp, vec, Lp); break;
          case 4: cta_gather_cols<4>(a.Y, a.n, a.mwp, idx, rw, rp, vec, Lp); break;
          case 5: cta_gather_cols<5>(a.Y, a.n, a.mwp, idx, rw, rp, vec, Lp); break;
          case 6: cta_gather_cols<6>(a.Y, a.n, a.mwp, idx, rw, rp, vec, Lp); break;
          case 7: cta_gather_cols<7>(a.Y, a.n, a.mwp, idx, rw, rp, vec, Lp); break;
          default: cta_gather_cols<8>(a.Y, a.n, a.mwp, idx, rw, rp, vec, Lp); break;
        }
      } else
      for (int64_t w = tid; w < a.mwp; w += nth) {
        uint32_t word = rw[w];
        int64_t c = rp[w];
        while (word) {
          const int b = __ffs(word) - 1;
          word &= word - 1;
          const int64_t i = w * 32 + b;
          for (int j = 0; j < K; ++j) vec[j * Lp + c] = __ldg(a.Y + i * a.n + idx[j]);
          ++c;
        }
      }
      if (!colfast && tid < K * K) Vacc[(tid / K) * KMAX + (tid % K)] = (tid / K == tid % K) ? 1.0 : 0.0;
    }
    __syncthreads();

    // ---- one-sided Jacobi with Gram-accelerated sweeps ----
    const int P = K * (K + 1) / 2;
    // off-diagonals relative to the larger norm: this bounds the rotation of
    // the top-rex subspace (what stage 3 consumes) by ~tol * g_ii / (g_ii - g_jj)
    const double tol_ortho = 1e-14;
    if (!colfast)
    for (int it = 0;; ++it) {
      if (K >= 2 && K <= (M2 ? 9 : 8)) {
        // one pass over the vectors: every thread accumulates all K(K+1)/2
        // products of its columns, warps reduce, partials summed in fixed order
        // (K = 9 only in the 4-warp row branch: its partials fit in Tmp)
        switch (K) {
          case 2: cta_gram_1pass<2>(vec, Lp, L, gram, gred); break;
          case 3: cta_gram_1pass<3>(vec, Lp, L, gram, gred); break;
          case 4: cta_gram_1pass<4>(vec, Lp, L, gram, gred); break;
          case 5: cta_gram_1pass<5>(vec, Lp, L, gram, gred); break;
          case 6: cta_gram_1pass<6>(vec, Lp, L, gram, gred); break;
          case 7: cta_gram_1pass<7>(vec, Lp, L, gram, gred); break;
          case 8: cta_gram_1pass<8>(vec, Lp, L, gram, gred); break;
          default:
            if constexpr (M2) cta_gram_1pass<9>(vec, Lp, L, gram, gred);
            break;
        }
      } else
      for (int p = warp; p < P; p += nwarps) {
        // unrank p -> (i, j), i <= j
        int i = 0, rem = p;
        while (rem >= K - i) { rem -= K - i; ++i; }
        const int j = i + rem;
        const double* vi = vec + i * Lp;
        const double* vj = vec + j * Lp;
        double s = 0.0;
        for (int64_t c = lane; c < L; c += 32) s += vi[c] * vj[c];
        s = warp_sum(s);
        if (lane == 0) {
          gram[i * KMAX + j] = s;
          gram[j * KMAX + i] = s;
        }
      }
      __syncthreads();
      if (M2 && it == 0 && a.fast_basis && a.rex == K - 1 && K <= 9) {
        // r = k - 1: an orthonormal basis of the top-r subspace straight from
        // the Gram (topr_basis_small: one lane, no Jacobi sweeps); its
        // coefficients C (K x r) go to W, the output is V = S^T C
        if (tid == 0) {
          int p = 0;
          for (int i = 0; i < K; ++i)
            for (int j = i; j < K; ++j) Tmp[p++] = gram[i * KMAX + j];
          flags[3] = topr_basis_rt(K, Tmp, W) ? 1 : 0;
        }
        __syncthreads();
        if (flags[3]) break;
      } else if (it == 0 && tid == 0) {
        flags[3] = 0;
      }
      if (warp == 0) {
        int big = 0;
        for (int e = lane; e < K * K; e += 32) {
          const int p = e / K, q = e % K;
          if (p < q) {
            const double g = gram[p * KMAX + q];
            const double d = fmax(gram[p * KMAX + p], gram[q * KMAX + q]);
            if (g != 0.0 && fabs(g) > tol_ortho * d) big = 1;
          }
        }
        big = __any_sync(0xffffffffu, big);
        const bool stop = !big || it >= a.max_outer;
        if (stop) {
          if (lane < K) sig[lane] = sqrt(fmax(gram[lane * KMAX + lane], 0.0));
        } else {
          warp_jacobi_rel(gram, KMAX, W, KMAX, K, cs, pairs, 2.220446049250313e-16, 40);
        }
        if (lane == 0) flags[2] = stop ? 1 : 0;
      }
      __syncthreads();
      if (flags[2]) break;
      // vectors <- W^T vectors (compile-time K up to 8: register arrays)
      if (K >= 2 && K <= 9) {
        switch (K) {
          case 2: cta_rotate<2>(vec, Lp, L, W); break;
          case 3: cta_rotate<3>(vec, Lp, L, W); break;
          case 4: cta_rotate<4>(vec, Lp, L, W); break;
          case 5: cta_rotate<5>(vec, Lp, L, W); break;
          case 6: cta_rotate<6>(vec, Lp, L, W); break;
          case 7: cta_rotate<7>(vec, Lp, L, W); break;
          case 8: cta_rotate<8>(vec, Lp, L, W); break;
          default: cta_rotate<9>(vec, Lp, L, W); break;
        }
      } else
      for (int64_t c = tid; c < L; c += nth) {
        double x[KMAX];
#pragma unroll
        for (int i = 0; i < KMAX; ++i) x[i] = (i < K) ? vec[i * Lp + c] : 0.0;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (j < K) {
            double y = 0.0;
#pragma unroll
            for (int i = 0; i < KMAX; ++i)
              if (i < K) y += W[i * KMAX + j] * x[i];
            vec[j * Lp + c] = y;
          }
        }
      }
      if (!M2) {
        // Vacc <- Vacc W
        for (int e = tid; e < K * K; e += nth) {
          const int r = e / K, cc = e % K;
          double s = 0.0;
          for (int i = 0; i < K; ++i) s += Vacc[r * KMAX + i] * W[i * KMAX + cc];
          Tmp[r * KMAX + cc] = s;
        }
        __syncthreads();
        for (int e = tid; e < K * K; e += nth) Vacc[(e / K) * KMAX + e % K] = Tmp[(e / K) * KMAX + e % K];
      }
      __syncthreads();
    }
    const bool fast = M2 && it_fast(flags);
    // descending singular values, ties by index (stable)
    if (tid == 0 && !it_fast(flags)) {
      for (int i = 0; i < K; ++i) ord[i] = i;
      for (int i = 1; i < K; ++i) {
        const int x = ord[i];
        int b = i - 1;
        while (b >= 0 && sig[ord[b]] < sig[x]) { ord[b + 1] = ord[b]; --b; }
        ord[b + 1] = x;
      }
    }
    __syncthreads();
    // expanded layout (stage 3 streams it with 1-D bulk copies): the trial's
    // top vectors as rp/2 planes of npad (v_{2p}, v_{2p+1}) pairs, zero
    // outside the column support; rp = rex rounded up to even
    const int rex = a.rex, rp = (a.rex + 1) & ~1;
    if (a.Wq) {
      if (M2 && fast) {
        // V = S^T C once per SUPPORT column (L of them, not npad), in place
        // over the first rex = K - 1 rows of the staged submatrix; the
        // expansion below then only looks values up. Four columns per thread
        // per pass, so each coefficient read serves four columns.
        for (int64_t c0 = 4 * (int64_t)tid; c0 < L; c0 += 4 * (int64_t)nth) {
          double xs[4][9];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < 9; ++k) xs[u][k] = (k < K && c0 + u < L) ? vec[k * Lp + c0 + u] : 0.0;
          for (int i = 0; i < rex; ++i) {
            double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int k = 0; k < 9; ++k) {
              const double w = k < K ? W[k * rex + i] : 0.0;
#pragma unroll
              for (int u = 0; u < 4; ++u) v[u] = fma(xs[u][k], w, v[u]);
            }
            // row i < K - 1 of these columns is not read again by this thread
            // (xs holds them) nor by any other (columns are disjoint)
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c0 + u < L) vec[i * Lp + c0 + u] = v[u];
          }
        }
        __syncthreads();
      }
      // int8 digit slices for the tensor-core stage 3 (k_gram_i8.cu): rows
      // tl * rex + i, zero outside the support, four columns per thread
      for (int64_t j0 = 4 * (int64_t)tid; j0 < a.npad; j0 += 4 * (int64_t)nth) {
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = j0 + u;
          int c = -1;
          if (M2) {
            const uint32_t word = cm[j >> 5], bit = 1u << (j & 31);
            if (word & bit) c = (int)pre[j >> 5] + __popc(word & (bit - 1u));
          } else {
            for (int q = 0; q < K; ++q)
              if (idx[q] == j) c = q;
          }
          cc[u] = c;
        }
        if (M2 && fast) {
          int8_t* wp = a.Wq + (tl * rex) * a.npad + j0;
          const int64_t sstride = a.Kpad * a.npad;
          for (int i = 0; i < rex; ++i) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = cc[u] >= 0 ? vec[i * Lp + cc[u]] : 0.0;
            emit_slices4_at(a.S, wp, sstride, v[0], v[1], v[2], v[3]);
            wp += a.npad;
          }
          continue;
        }
        for (int i = 0; i < rex; ++i) {
          double v[4];
          {
            const int o = ord[i];
            const double sg = M2 ? sig[o] : 0.0;
            const double inv = sg > 0.0 ? 1.0 / sg : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              v[u] = 0.0;
              if (cc[u] >= 0) v[u] = M2 ? vec[o * Lp + cc[u]] * inv : Vacc[cc[u] * KMAX + o];
            }
          }
          emit_slices4(a.S, a.Wq, a.Kpad, a.npad, tl * rex + i, j0, v[0], v[1], v[2], v[3]);
        }
      }
      __syncthreads();
      continue;
    }
    double2* vout = reinterpret_cast<double2*>(a.Vout + tl * a.npad * rp);
    for (int64_t j = tid; j < a.npad; j += nth) {
      int c = -1;  // support position of column j
      if (M2) {
        const uint32_t word = cm[j >> 5], bit = 1u << (j & 31);
        if (word & bit) c = (int)pre[j >> 5] + __popc(word & (bit - 1u));
      } else {
        for (int q = 0; q < K; ++q)
          if (idx[q] == j) c = q;
      }
      for (int p = 0; p < rp / 2; ++p) {
        double v[2] = {0.0, 0.0};
        if (c >= 0)
          for (int h = 0; h < 2; ++h) {
            const int i = 2 * p + h;
            if (i < rex) {
              if (M2 && fast) {
                double t = 0.0;
                for (int k = 0; k < K; ++k) t = fma(vec[k * Lp + c], W[k * rex + i], t);
                v[h] = t;
              } else if (M2) {
                // V_top rows over the column support: rotated_row_i[c] / sigma_i
                const int o = ord[i];
                const double sg = sig[o];
                v[h] = sg > 0.0 ? vec[o * Lp + c] / sg : 0.0;
              } else {
                v[h] = Vacc[c * KMAX + ord[i]];
              }
            }
          }
        vout[p * a.npad + j] = make_double2(v[0], v[1]);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Row branch, warp per trial (K = k <= 9): no CTA barriers, 4 independent
// trials per CTA. The warp ANDs the k mask rows' words, scans the popcounts
// (shuffle scan), gathers the k x q submatrix into its shared-memory slice
// (lane = column, coalesced row reads), then runs the same Gram-accelerated
// one-sided Jacobi: every lane accumulates all K(K+1)/2 partial dot products
// of its columns in registers (one pass over the data), a butterfly reduction
// leaves the full Gram in every lane, the convergence test is evaluated
// redundantly (warp-uniform), and only the K x K eigensolve goes through
// shared memory.
// Top-(K-1) right-singular subspace of a K x (q) submatrix S from its K x K
// Gram G = S S^T (packed upper g), for the case r = K - 1 the row branch's
// default k = r + 1 gives. Stage 3 consumes only the projector V_r V_r^T, so
// any orthonormal basis of span(V_r) serves: the smallest eigenvector u of G
// by inverse iteration (Cholesky of G, at most 5 steps, converged when
// successive iterates agree to 1e-14), a Householder reflection H with
// H u = -+e_K whose first K-1 columns Q span u-perp = span(U_r), M = Q^T G Q
// and its Cholesky M = L L^T; then V = S^T C with C = Q L^{-T} is orthonormal
// (V^T V = L^{-1} M L^{-T} = I) and spans the top-r right singular vectors.
// Run by one lane into C (K x (K-1), smem); returns false (the caller falls
// back to the one-sided Jacobi) when G is not clearly separated -- inverse
// iteration not converged or M not safely positive definite.
template <int K>
__device__ __noinline__ bool topr_basis_small(const double* Gsm, double* C) {
  constexpr int R = K - 1;
  constexpr int P = K * (K + 1) / 2;
  auto gat = [&](int i, int j) {  // packed upper G (shared memory)
    const int lo = i < j ? i : j, hi = i < j ? j : i;
    return Gsm[lo * K - lo * (lo - 1) / 2 + (hi - lo)];
  };
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) tr += gat(i, i);
  if (!(tr > 0.0)) return false;
  // Cholesky of G (packed lower) with a floor on the pivots (G may be
  // singular: the floor only regularises the inverse iteration)
  double L[P], Li[K];  // Li: reciprocal pivots (the solves multiply)
  auto li = [](int i, int j) { return i * (i + 1) / 2 + j; };
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double d = gat(j, j);
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[li(j, k)] * L[li(j, k)];
    d = fmax(d, 1e-30 * tr);
    Li[j] = rsqrt_fast(d);
    L[li(j, j)] = d * Li[j];
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double v = gat(i, j);
#pragma unroll
      for (int k = 0; k < j; ++k) v -= L[li(i, k)] * L[li(j, k)];
      L[li(i, j)] = v * Li[j];
    }
  }
  double x[K];
#pragma unroll
  for (int i = 0; i < K; ++i) x[i] = 1.0 + 0.25 * i;
  bool conv = false;
  for (int it = 0; it < 5 && !conv; ++it) {
    double z[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double v = x[i];
#pragma unroll
      for (int k = 0; k < i; ++k) v -= L[li(i, k)] * z[k];
      z[i] = v * Li[i];
    }
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      double v = z[i];
#pragma unroll
      for (int k = i + 1; k < K; ++k) v -= L[li(k, i)] * z[k];
      z[i] = v * Li[i];
    }
    double nz = 0.0, dot = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) nz += z[i] * z[i];
    nz = rsqrt_fast(nz);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      z[i] *= nz;
      dot += z[i] * x[i];
    }
    double diff = 0.0;
    const double sg = dot >= 0.0 ? 1.0 : -1.0;
#pragma unroll
    for (int i = 0; i < K; ++i) diff = fmax(diff, fabs(z[i] - sg * x[i]));
    if (it > 0 && diff <= 1e-14) conv = true;
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = z[i];
  }
  if (!conv) return false;
  // Householder v = x + s e_K, H = I - beta v v^T (H x = -s e_K); the first R
  // columns of H are Q. M = Q^T G Q = (H G H)[0:R, 0:R] with w = G v,
  // gamma = v^T w: (HGH)_ij = G_ij - beta (v_i w_j + w_i v_j) + beta^2 gamma v_i v_j
  const double sgn = x[K - 1] >= 0.0 ? 1.0 : -1.0;
  double v[K];
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = x[i];
  v[K - 1] += sgn;
  double vv = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) vv += v[i] * v[i];
  const double beta = 2.0 / vv;
  double w[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) t += gat(i, k) * v[k];
    w[i] = t;
  }
  double gam = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) gam += v[i] * w[i];
  // Cholesky of M (packed lower, reusing L), pivots well above zero
  double dmax = 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i)
    dmax = fmax(dmax, gat(i, i) - 2.0 * beta * v[i] * w[i] + beta * beta * gam * v[i] * v[i]);
#pragma unroll
  for (int j = 0; j < R; ++j) {
    double d = gat(j, j) - 2.0 * beta * v[j] * w[j] + beta * beta * gam * v[j] * v[j];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[li(j, k)] * L[li(j, k)];
    if (!(d > 1e-8 * dmax)) return false;
    Li[j] = rsqrt_fast(d);
    L[li(j, j)] = d * Li[j];
#pragma unroll
    for (int i = j + 1; i < R; ++i) {
      double t = gat(i, j) - beta * (v[i] * w[j] + w[i] * v[j]) + beta * beta * gam * v[i] * v[j];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= L[li(i, k)] * L[li(j, k)];
      L[li(i, j)] = t * Li[j];
    }
  }
  // C = Q L^{-T}: row i of C solves L c = q_i, q_ij = delta_ij - beta v_i v_j
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double c[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      double t = (i == j ? 1.0 : 0.0) - beta * v[i] * v[j];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= L[li(j, k)] * c[k];
      c[j] = t * Li[j];
    }
#pragma unroll
    for (int j = 0; j < R; ++j) C[i * R + j] = c[j];
  }
  return true;
}

// Column branch, r = l - 1: an orthonormal basis of the top-r right singular
// subspace of the q x K submatrix A from its K x K Gram G = A^T A (packed upper
// g). That subspace is u-perp, u the eigenvector of G's smallest eigenvalue: u
// by the same regularised-Cholesky inverse iteration as topr_basis_small, then
// the Householder reflection H with H u = -+e_K, whose first K - 1 columns are
// the basis. Q (K x K, leading dimension ldq) gets those columns and u as its
// last one. Returns false (the caller runs the one-sided Jacobi) when the
// inverse iteration has not converged to 1e-14 in 16 steps (lambda_K /
// lambda_{K-1} above ~0.1: no clear gap); with a gap the eigenvector's error
// eps * lambda_1 / (lambda_{K-1} - lambda_K) is at rounding level.
template <int K>
__device__ __noinline__ bool perp_basis_small(const double* Gsm, double* Q, int ldq) {
  constexpr int P = K * (K + 1) / 2;
  auto gat = [&](int i, int j) {
    const int lo = i < j ? i : j, hi = i < j ? j : i;
    return Gsm[lo * K - lo * (lo - 1) / 2 + (hi - lo)];
  };
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) tr += gat(i, i);
  if (!(tr > 0.0)) return false;
  double L[P], Li[K];
  auto li = [](int i, int j) { return i * (i + 1) / 2 + j; };
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double d = gat(j, j);
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[li(j, k)] * L[li(j, k)];
    d = fmax(d, 1e-30 * tr);
    Li[j] = rsqrt_fast(d);
    L[li(j, j)] = d * Li[j];
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double v = gat(i, j);
#pragma unroll
      for (int k = 0; k < j; ++k) v -= L[li(i, k)] * L[li(j, k)];
      L[li(i, j)] = v * Li[j];
    }
  }
  double x[K];
#pragma unroll
  for (int i = 0; i < K; ++i) x[i] = 1.0 + 0.25 * i;
  bool conv = false;
  for (int it = 0; it < 16 && !conv; ++it) {
    double z[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double v = x[i];
#pragma unroll
      for (int k = 0; k < i; ++k) v -= L[li(i, k)] * z[k];
      z[i] = v * Li[i];
    }
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      double v = z[i];
#pragma unroll
      for (int k = i + 1; k < K; ++k) v -= L[li(k, i)] * z[k];
      z[i] = v * Li[i];
    }
    double nz = 0.0, dot = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) nz += z[i] * z[i];
    nz = rsqrt_fast(nz);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      z[i] *= nz;
      dot += z[i] * x[i];
    }
    double diff = 0.0;
    const double sg = dot >= 0.0 ? 1.0 : -1.0;
#pragma unroll
    for (int i = 0; i < K; ++i) diff = fmax(diff, fabs(z[i] - sg * x[i]));
    if (it > 0 && diff <= 1e-14) conv = true;
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = z[i];
  }
  if (!conv) return false;
  // one exact renormalisation (rsqrt_fast is a Newton approximation)
  double nx = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) nx += x[i] * x[i];
  nx = 1.0 / sqrt(nx);
#pragma unroll
  for (int i = 0; i < K; ++i) x[i] *= nx;
  const double sgn = x[K - 1] >= 0.0 ? 1.0 : -1.0;
  double v[K];
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = x[i];
  v[K - 1] += sgn;
  double vv = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) vv += v[i] * v[i];
  const double beta = 2.0 / vv;
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int j = 0; j < K - 1; ++j) Q[i * ldq + j] = (i == j ? 1.0 : 0.0) - beta * v[i] * v[j];
    Q[i * ldq + K - 1] = x[i];
  }
  return true;
}

constexpr int SVDW_WARPS = 4;
// largest k whose warp kernel takes the top-r basis path (r = k - 1) before
// falling back to one-sided Jacobi (config 4: k = 9)
#ifndef RSM_FASTK
#define RSM_FASTK 9
#endif
constexpr int FASTK = RSM_FASTK;

template <int K>
__global__ void __launch_bounds__(SVDW_WARPS * 32) k_svd_warp(SvdArgs a) {
  constexpr int P = K * (K + 1) / 2;
  extern __shared__ __align__(16) double smw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t Lp = a.Lpad;
  const int64_t per_warp = K * Lp + 2 * K * K + 64 + 32 + a.cmw;  // doubles
  double* S = smw + warp * per_warp;
  double* Gs = S + K * Lp;
  double* Ws = Gs + K * K;
  double* cs = Ws + K * K;
  int* pairs = reinterpret_cast<int*>(cs + 64);
  uint32_t* cm = reinterpret_cast<uint32_t*>(cs + 96);
  uint32_t* pre = cm + a.cmw;
  const int rex = a.rex, rp = (a.rex + 1) & ~1;
  const int64_t nwarps = (int64_t)gridDim.x * SVDW_WARPS;

  const int64_t t_end = a.sel_acc ? min(a.t_hi, (int64_t)*a.sel_acc) : a.t_hi;
  for (int64_t t = a.t_lo + (int64_t)blockIdx.x * SVDW_WARPS + warp; t < t_end; t += nwarps) {
    const int64_t tl = t - a.t_lo;
    const int myidx = lane < K ? a.t_idx[t * K + lane] : 0;
    int rows[K];
#pragma unroll
    for (int i = 0; i < K; ++i) rows[i] = __shfl_sync(0xffffffffu, myidx, i);
    // support words + exclusive popcount prefix (warp scan over lanes, words
    // w = s*32 + lane)
    int run = 0;
    for (int64_t w0 = 0; w0 < a.cmw; w0 += 32) {
      const int64_t w = w0 + lane;
      uint32_t acc = 0;
      if (w < a.nwp && w < a.cmw) {
        acc = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < K; ++i) acc &= __ldg(a.bitsR + (int64_t)rows[i] * a.nwp + w);
      }
      const int c = __popc(acc);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (w < a.cmw) {
        cm[w] = acc;
        pre[w] = (uint32_t)(run + incl - c);
        a.t_cm[tl * a.cmw + w] = acc;
      }
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    const int L = run;
    if (L > a.Lcap) continue;  // speculative launch only (see SvdArgs)
    __syncwarp();
    // gather S (K x L): lane = column within each 32-column word. Every
    // support cell is copied global -> shared by an asynchronous 8-byte copy
    // (cp.async), so all of a trial's K x L loads are in flight at once and
    // the warp waits for them once (one memory round trip per trial)
    {
      // four words per step: their support words and prefixes by one 16-byte
      // shared-memory load each (cmw is a multiple of 4; words past n are 0),
      // the copies' global addresses as immediate offsets of K running row
      // pointers
      const unsigned sb = (unsigned)__cvta_generic_to_shared(S);
      const unsigned Lp8 = 8u * (unsigned)Lp;
      const double* yrow[K];
#pragma unroll
      for (int i = 0; i < K; ++i) yrow[i] = a.Y + (int64_t)rows[i] * a.n + lane;
      int* cc = a.colcnt + lane;
      const uint32_t below = (1u << lane) - 1u;
      const uint32_t lbit = 1u << lane;
      auto cell = [&](auto J, uint32_t word, uint32_t p) {
        constexpr int OFF = decltype(J)::value;
        if (word & lbit) {  // support bits exist only for j < n
          unsigned dst = sb + 8u * (p + (unsigned)__popc(word & below));
#pragma unroll
          for (int i = 0; i < K; ++i) {
            asm volatile("cp.async.ca.shared.global [%0], [%1+%2], 8;\n" ::"r"(dst), "l"(yrow[i]), "n"(OFF * 256)
                         : "memory");
            dst += Lp8;
          }
          atomicAdd(cc + 32 * OFF, 1);
        }
      };
      for (int w = 0; w < (int)a.cmw; w += 4) {
        const uint4 c4 = *reinterpret_cast<const uint4*>(cm + w);
        const uint4 p4 = *reinterpret_cast<const uint4*>(pre + w);
        cell(std::integral_constant<int, 0>{}, c4.x, p4.x);
        cell(std::integral_constant<int, 1>{}, c4.y, p4.y);
        cell(std::integral_constant<int, 2>{}, c4.z, p4.z);
        cell(std::integral_constant<int, 3>{}, c4.w, p4.w);
#pragma unroll
        for (int i = 0; i < K; ++i) yrow[i] += 128;
        cc += 128;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    // one-sided Jacobi, Gram-accelerated. The Gram of the rotated vectors is
    // accumulated in the rotation pass itself (one read of S per iteration).
    double g[P];
#pragma unroll
    for (int p = 0; p < P; ++p) g[p] = 0.0;
    for (int c = lane; c < L; c += 32) {
      double x[K];
#pragma unroll
      for (int i = 0; i < K; ++i) x[i] = S[i * Lp + c];
      int p = 0;
#pragma unroll
      for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = i; j < K; ++j) {
          g[p] = fma(x[i], x[j], g[p]);
          ++p;
        }
    }
    bool fast = false;
    for (int it = 0;; ++it) {
      bool reduced = false;
      if constexpr (K <= FASTK) {
        if (it == 0 && rex == K - 1 && a.fast_basis) {
          // r = k - 1: an orthonormal basis of the top-r subspace straight
          // from the Gram (see topr_basis_small), no Jacobi rotations. Only one
          // lane needs the Gram: a halving reduction (~NH shuffles instead of
          // 5 P) leaves each total in one lane, which stores it.
          constexpr int NH = P <= 16 ? 16 : (P <= 32 ? 32 : 64);
          constexpr int PL = NH > 32 ? NH / 32 : 1, LPV = NH < 32 ? 32 / NH : 1;
          double h[NH];
#pragma unroll
          for (int p = 0; p < NH; ++p) h[p] = p < P ? g[p] : 0.0;
          warp_reduce_halving<NH>(h, lane);
          if (lane % LPV == 0) {
#pragma unroll
            for (int q = 0; q < PL; ++q) {
              const int j = (lane / LPV) * PL + q;
              if (j < P) Gs[j] = h[q];
            }
          }
          __syncwarp();
          if (lane == 0) Gs[K * K - 1] = topr_basis_small<K>(Gs, Ws) ? 1.0 : 0.0;
          __syncwarp();
          fast = Gs[K * K - 1] != 0.0;
          __syncwarp();
          if (fast) break;
#pragma unroll
          for (int p = 0; p < P; ++p) g[p] = Gs[p];  // the Jacobi path wants the totals in every lane
          reduced = true;
        }
      }
      if (!reduced) {
#pragma unroll
        for (int p = 0; p < P; ++p) g[p] = warp_sum(g[p]);
      }
      bool big = false;
      {
        int p = 0;
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int j = i; j < K; ++j) {
            if (j > i) {
              const double dii = g[i * K - i * (i - 1) / 2];
              const double djj = g[j * K - j * (j - 1) / 2];
              if (g[p] != 0.0 && fabs(g[p]) > 1e-14 * fmax(dii, djj)) big = true;
            }
            ++p;
          }
      }
      if (!big || it >= a.max_outer) break;  // warp-uniform
      {
        int p = 0;
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int j = i; j < K; ++j) {
            if (lane == 0) {
              Gs[i * K + j] = g[p];
              Gs[j * K + i] = g[p];
            }
            ++p;
          }
      }
      __syncwarp();
      warp_jacobi_reg<K, true>(Gs, K, Ws, K, 40);
      __syncwarp();
#pragma unroll
      for (int p = 0; p < P; ++p) g[p] = 0.0;
      for (int c = lane; c < L; c += 32) {
        double x[K], y[K];
#pragma unroll
        for (int i = 0; i < K; ++i) x[i] = S[i * Lp + c];
#pragma unroll
        for (int j = 0; j < K; ++j) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < K; ++i) t = fma(Ws[i * K + j], x[i], t);
          y[j] = t;
          S[j * Lp + c] = t;
        }
        int p = 0;
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int j = i; j < K; ++j) {
            g[p] = fma(y[i], y[j], g[p]);
            ++p;
          }
      }
      __syncwarp();
    }
    if constexpr (K <= FASTK) {
      if (fast) {
        // V = S^T C (K x r coefficients in Ws), expanded layout
        constexpr int R1 = K - 1;
        constexpr int RPX1 = (R1 + 1) & ~1;
        double cf[K][RPX1];
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int j = 0; j < RPX1; ++j) cf[i][j] = j < R1 ? Ws[i * R1 + j] : 0.0;
        const int lmax = L > 0 ? L - 1 : 0;
        if (a.Wq) {
          // int8 digit slices (k_gram_i8.cu): lane = 4 consecutive columns
          // V = S^T C first in compact form, in place over rows 0..r-1 of S
          // (each support column once: L of them, not npad), then expanded
          for (int c = lane; c < L; c += 32) {
            double x[K], t[R1];
#pragma unroll
            for (int i = 0; i < K; ++i) x[i] = S[i * Lp + c];
#pragma unroll
            for (int p = 0; p < R1; ++p) {
              double acc = 0.0;
#pragma unroll
              for (int i = 0; i < K; ++i) acc = fma(x[i], cf[i][p], acc);
              t[p] = acc;
            }
#pragma unroll
            for (int p = 0; p < R1; ++p) S[p * Lp + c] = t[p];
          }
          __syncwarp();
          const int64_t sstride = a.Kpad * a.npad;
          int8_t* wq = a.Wq + tl * rex * a.npad + 4 * lane;
          const int sh0 = (4 * lane) & 31;  // bit of the lane's first column within its word
          for (int64_t j0 = 4 * lane; j0 < a.npad; j0 += 128, wq += 128) {
            const uint32_t word = cm[j0 >> 5];
            int c0 = (int)pre[j0 >> 5] + __popc(word & ((1u << sh0) - 1u));
            const uint32_t nib = (word >> sh0) & 15u;
            int cu[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              cu[u] = c0 < lmax ? c0 : lmax;
              c0 += (nib >> u) & 1u;
            }
            // the vector loop stays rolled: one copy of the digit emission in
            // the instruction stream (the kernel is fetch-sensitive)
            int8_t* wp = wq;
            const double* sp = S;
#pragma unroll 1
            for (int p = 0; p < R1; ++p) {
              double v[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const double t = sp[cu[u]];
                v[u] = ((nib >> u) & 1u) ? t : 0.0;
              }
              emit_slices4_at(a.S, wp, sstride, v[0], v[1], v[2], v[3]);
              wp += a.npad;
              sp += Lp;
            }
          }
          __syncwarp();
          continue;
        }
        double2* vout = reinterpret_cast<double2*>(a.Vout + tl * a.npad * rp);
        for (int64_t j = lane; j < a.npad; j += 32) {
          const uint32_t word = cm[j >> 5], bit = 1u << (j & 31);
          const bool in = (word & bit) != 0;
          int c = (int)pre[j >> 5] + __popc(word & (bit - 1u));
          c = c < lmax ? c : lmax;
          double x[K];
#pragma unroll
          for (int i = 0; i < K; ++i) x[i] = S[i * Lp + c];
#pragma unroll
          for (int p = 0; p < RPX1 / 2; ++p) {
            double v0 = 0.0, v1 = 0.0;
#pragma unroll
            for (int i = 0; i < K; ++i) {
              v0 = fma(x[i], cf[i][2 * p], v0);
              v1 = fma(x[i], cf[i][2 * p + 1], v1);
            }
            vout[p * a.npad + j] = make_double2(in ? v0 : 0.0, in ? v1 : 0.0);
          }
        }
        __syncwarp();
        continue;
      }
    }
    // descending norms (stable), then the top rows, normalised. The sort is a
    // compile-time bubble network on (sigma, row) pairs, so both stay in
    // registers (no dynamically indexed local arrays).
    double sig[K];
    int ord[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      sig[i] = sqrt(fmax(g[i * K - i * (i - 1) / 2], 0.0));
      ord[i] = i;
    }
    // stable bubble sort on K <= 9 entries (ties keep the lower index first)
#pragma unroll
    for (int pass = 0; pass < K - 1; ++pass)
#pragma unroll
      for (int j = 0; j < K - 1 - pass; ++j)
        if (sig[j] < sig[j + 1]) {
          const double ts = sig[j];
          sig[j] = sig[j + 1];
          sig[j + 1] = ts;
          const int ti = ord[j];
          ord[j] = ord[j + 1];
          ord[j + 1] = ti;
        }
    // row i of the output: S row ord[i] scaled by 1/sigma_i (0 when excluded)
    constexpr int RPX = (K + 1) & ~1;
    double scl[RPX];
    const double* srow[RPX];
#pragma unroll
    for (int i = 0; i < RPX; ++i) {
      const bool use = i < K && i < rex && sig[i < K ? i : 0] > 0.0;
      scl[i] = use ? 1.0 / sig[i < K ? i : 0] : 0.0;
      srow[i] = S + (int64_t)(i < K ? ord[i] : 0) * Lp;
    }
    // expanded layout (see k_svd): rp/2 planes of npad pairs, zero outside
    // the support
    const int lmax = L > 0 ? L - 1 : 0;
    if (a.Wq) {
      // int8 digit slices (k_gram_i8.cu): lane = 4 consecutive columns
      for (int64_t j0 = 4 * lane; j0 < a.npad; j0 += 128) {
        int cidx[4];
        bool in[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = j0 + u;
          const uint32_t word = cm[j >> 5], bit = 1u << (j & 31);
          in[u] = (word & bit) != 0;
          const int c = (int)pre[j >> 5] + __popc(word & (bit - 1u));
          cidx[u] = c < lmax ? c : lmax;
        }
#pragma unroll
        for (int p = 0; p < RPX; ++p) {
          if (p >= rex) break;
          double v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = in[u] ? srow[p][cidx[u]] * scl[p] : 0.0;
          emit_slices4(a.S, a.Wq, a.Kpad, a.npad, tl * rex + p, j0, v[0], v[1], v[2], v[3]);
        }
      }
      __syncwarp();
      continue;
    }
    double2* vout = reinterpret_cast<double2*>(a.Vout + tl * a.npad * rp);
    for (int64_t j = lane; j < a.npad; j += 32) {
      const uint32_t word = cm[j >> 5], bit = 1u << (j & 31);
      const bool in = (word & bit) != 0;
      int c = (int)pre[j >> 5] + __popc(word & (bit - 1u));
      c = c < lmax ? c : lmax;
#pragma unroll
      for (int p = 0; p < RPX / 2; ++p) {
        if (p >= rp / 2) break;
        const double v0 = in ? srow[2 * p][c] * scl[2 * p] : 0.0;
        const double v1 = in ? srow[2 * p + 1][c] * scl[2 * p + 1] : 0.0;
        vout[p * a.npad + j] = make_double2(v0, v1);
      }
    }
    __syncwarp();
  }
}

size_t svd_warp_smem(int K, int64_t Lpad, int64_t cmw) {
  return sizeof(double) * (size_t)SVDW_WARPS * (K * Lpad + 2 * K * K + 64 + 32 + cmw);
}

static const void* svd_warp_fn(int K) {
  switch (K) {
    case 2: return (const void*)k_svd_warp<2>;
    case 3: return (const void*)k_svd_warp<3>;
    case 4: return (const void*)k_svd_warp<4>;
    case 5: return (const void*)k_svd_warp<5>;
    case 6: return (const void*)k_svd_warp<6>;
    case 7: return (const void*)k_svd_warp<7>;
    case 8: return (const void*)k_svd_warp<8>;
    case 9: return (const void*)k_svd_warp<9>;
    default: return nullptr;
  }
}

// speculative stage-2 bound: the largest even support length >= Lest for which
// the warp kernel keeps the occupancy it has at Lest (the shared memory the
// bound costs is then free); Lest itself when the warp kernel does not apply
int64_t svd_warp_lcap(int K, int64_t Lest, int64_t cmw) {
  Lest = std::max<int64_t>(2, (Lest + 1) & ~int64_t(1));
  const void* fn = svd_warp_fn(K);
  if (!fn || svd_warp_smem(K, Lest, cmw) > 200 * 1024) return Lest;
  const int occ0 = occupancy(fn, SVDW_WARPS * 32, svd_warp_smem(K, Lest, cmw));
  auto keeps = [&](int64_t L) {
    const size_t sm = svd_warp_smem(K, L, cmw);
    return sm <= 200 * 1024 && occupancy(fn, SVDW_WARPS * 32, sm) >= occ0;
  };
  int64_t lo = Lest, hi = Lest + 2;  // even lengths; lo keeps occ0
  while (keeps(hi)) {
    lo = hi;
    hi *= 2;
  }
  while (hi - lo > 2) {
    const int64_t mid = ((lo + hi) / 2) & ~int64_t(1);
    if (keeps(mid)) lo = mid;
    else hi = mid;
  }
  return lo;
}

bool launch_svd_warp(const SvdArgs& a, int sms, cudaStream_t s) {
  const int K = a.block;
  if (K < 2 || K > 9) return false;
  const size_t smem = svd_warp_smem(K, a.Lpad, a.cmw);
  if (smem > 200 * 1024) return false;
  const int64_t Tl = a.t_hi - a.t_lo;
#define RSM_SVDW(KK)                                                                                \
  case KK: {                                                                                        \
    int occ = occupancy((const void*)k_svd_warp<KK>, SVDW_WARPS * 32, smem);                       \
    if (occ < 1) occ = 1;                                                                           \
    const int64_t grid = std::min<int64_t>((Tl + SVDW_WARPS - 1) / SVDW_WARPS, (int64_t)sms * occ); \
    k_svd_warp<KK><<<(unsigned)std::max<int64_t>(grid, 1), SVDW_WARPS * 32, smem, s>>>(a);          \
    return true;                                                                                    \
  }
  switch (K) {
    RSM_SVDW(2) RSM_SVDW(3) RSM_SVDW(4) RSM_SVDW(5) RSM_SVDW(6) RSM_SVDW(7) RSM_SVDW(8) RSM_SVDW(9)
    default: return false;
  }
#undef RSM_SVDW
}

size_t svd_smem_fixed(int64_t cmw, bool m2) {
  const int gred = m2 ? 0 : svd_cta_threads<false>() / 32 * SVD_GRED_PER_WARP;
  size_t s = sizeof(double) * (4 * KMAX * KMAX + gred + 64 + KMAX) + sizeof(int) * (64 + 3 * KMAX + 4) +
             sizeof(uint32_t) * 2 * (size_t)cmw;
  return (s + 15) & ~(size_t)15;
}

void launch_svd(const SvdArgs& a, bool m2, int grid, size_t smem, cudaStream_t s) {
  if (m2) {
    ensure_smem((const void*)k_svd<true>, smem);
    k_svd<true><<<grid, svd_cta_threads<true>(), smem, s>>>(a);
  } else {
    ensure_smem((const void*)k_svd<false>, smem);
    k_svd<false><<<grid, svd_cta_threads<false>(), smem, s>>>(a);
  }
}

int svd_occupancy(bool m2, size_t smem) {
  return m2 ? occupancy((const void*)k_svd<true>, svd_cta_threads<true>(), smem)
            : occupancy((const void*)k_svd<false>, svd_cta_threads<false>(), smem);
}

}  // namespace rsmk
