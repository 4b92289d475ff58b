// k_dropin.cu -- device kernels behind the drop-in header's per-trial and
// accumulator utilities (include/rsm_gpu/rsm.hpp): one attempt's sample,
// the small SVD's constraint vectors and dense Gram updates.
// These are the reference's building blocks exposed one call at a time
// (sampler.cpp:27-87, spectra.cpp:7-86, core.cpp:15-44, paths relative to
// /root/reference/proj); the batched hot path (k_select / k_svd / k_gram*)
// never calls them.
#include <cmath>

#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

using namespace rsmd;

namespace {

constexpr int DT = 256;  // threads per CTA (one CTA per call)

// deterministic block sum (fixed tree), result broadcast to every thread
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

}  // namespace

// sample_m1 / sample_m2 for one attempt: the draw (bit-exact, as k_select),
// then the kept indices of the other dimension: AND of the drawn rows'
// (M2: row-major words) or columns' (M1: column-major words) mask words,
// emitted in ascending order.
__global__ void __launch_bounds__(DT) k_sample_one(const uint32_t* __restrict__ bits, int64_t stride,
                                                   int64_t nwords, int64_t pool, int count, uint64_t seed,
                                                   uint64_t index, int32_t* __restrict__ drawn,
                                                   uint32_t* __restrict__ words, int32_t* __restrict__ kept,
                                                   int64_t* __restrict__ nkept) {
  __shared__ int32_t sd[KMAX];
  if (threadIdx.x == 0) draw_sorted(seed, index, pool, count, sd);
  __syncthreads();
  if (threadIdx.x < count) drawn[threadIdx.x] = sd[threadIdx.x];
  for (int64_t w = threadIdx.x; w < nwords; w += blockDim.x) {
    uint32_t acc = 0xffffffffu;
    for (int t = 0; t < count; ++t) acc &= bits[(int64_t)sd[t] * stride + w];
    words[w] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // ordered emission (words past the dimension are zero)
    int64_t c = 0;
    for (int64_t w = 0; w < nwords; ++w) {
      uint32_t x = words[w];
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1u;
        kept[c++] = (int32_t)(w * 32 + b);
      }
    }
    *nkept = c;
  }
}

// small_singular_vectors (spectra.cpp:48-86) of a p x q submatrix S (row
// major), one CTA. One-sided (Hestenes) Jacobi on the short side, so every
// singular value keeps the relative accuracy of the data:
//   q <= p (q <= 32): rotate the q columns of W = S (length p) pairwise until
//            orthogonal; V = accumulated rotations (q x q), sigma = norms;
//   p < q (p <= 32): rotate the p rows (length q); the normalised rows are
//            the top right singular vectors (rows whose norm is below
//            1e-15 of the largest are rank deficiency: sigma 0), the remaining
//            q - p' columns of V an orthonormal completion (Householder QR of
//            the p' top vectors) with sigma exactly 0, as the structural zeros
//            of a full SVD.
// V's columns sorted by descending sigma; output vector t = column q-1-t
// (ascending sigma; columns past the rank carry sigma 0), sign-fixed so the
// largest-magnitude entry is positive (first index on ties). W and V live in
// global scratch (Wg: p x q, Vg: q x q).
__global__ void __launch_bounds__(DT) k_small_svd(const double* __restrict__ S, int p, int q, int ell,
                                                  double* __restrict__ Wg, double* __restrict__ Vg,
                                                  double* __restrict__ sig, int* __restrict__ ord,
                                                  double* __restrict__ zeta, double* __restrict__ sv) {
  __shared__ double red[DT / 32];
  __shared__ double rot[2];
  __shared__ int flag;
  const int tid = threadIdx.x;
  const bool cols = q <= p;  // tall or square: rotate the q <= 32 columns; wide: the p <= 32 rows
  const int nv = cols ? q : p;           // vectors rotated
  const int len = cols ? p : q;          // their length
  // element e of vector v in W: column v (stride q) or row v (stride 1)
  auto at = [&](int v, int e) -> double& { return cols ? Wg[(int64_t)e * q + v] : Wg[(int64_t)v * q + e]; };
  for (int64_t e = tid; e < (int64_t)p * q; e += blockDim.x) Wg[e] = S[e];
  if (cols)
    for (int e = tid; e < q * q; e += blockDim.x) Vg[e] = (e / q == e % q) ? 1.0 : 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < 80; ++sweep) {
    if (tid == 0) flag = 0;
    __syncthreads();
    for (int i = 0; i < nv - 1; ++i)
      for (int j = i + 1; j < nv; ++j) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int e = tid; e < len; e += blockDim.x) {
          const double x = at(i, e), y = at(j, e);
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
        }
        a = block_sum(a, red);
        b = block_sum(b, red);
        g = block_sum(g, red);
        if (g != 0.0 && fabs(g) > 1e-15 * sqrt(a * b)) {
          const double zeta_ = (b - a) / (2.0 * g);
          const double t = (zeta_ >= 0.0 ? 1.0 : -1.0) / (fabs(zeta_) + sqrt(1.0 + zeta_ * zeta_));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int e = tid; e < len; e += blockDim.x) {
            const double x = at(i, e), y = at(j, e);
            at(i, e) = c * x - s * y;
            at(j, e) = s * x + c * y;
          }
          if (cols)
            for (int e = tid; e < q; e += blockDim.x) {
              const double x = Vg[(int64_t)e * q + i], y = Vg[(int64_t)e * q + j];
              Vg[(int64_t)e * q + i] = c * x - s * y;
              Vg[(int64_t)e * q + j] = s * x + c * y;
            }
          if (tid == 0) flag = 1;
        }
        __syncthreads();
      }
    __syncthreads();
    if (!flag) break;
    __syncthreads();
  }
  // norms, descending order (stable)
  for (int v = 0; v < nv; ++v) {
    double a = 0.0;
    for (int e = tid; e < len; e += blockDim.x) a = fma(at(v, e), at(v, e), a);
    a = block_sum(a, red);
    if (tid == 0) sig[v] = sqrt(a);
  }
  __syncthreads();
  if (tid == 0) {
    for (int v = 0; v < nv; ++v) ord[v] = v;
    for (int i = 1; i < nv; ++i) {
      const int x = ord[i];
      int b = i - 1;
      while (b >= 0 && sig[ord[b]] < sig[x]) { ord[b + 1] = ord[b]; --b; }
      ord[b + 1] = x;
    }
  }
  __syncthreads();
  double* Vfull = Vg;  // q x q, column c = right singular vector of the c-th largest sigma
  int ptop = nv;       // vectors with sigma > 0 (rows case)
  if (!cols) {
    // rows case: top vectors = normalised rows, in descending order, into
    // columns 0..p'-1 of a q x q V; Householder completion for the rest
    if (tid == 0) {
      int c = 0;
      const double smax = sig[ord[0]];
      while (c < nv && sig[ord[c]] > 1e-300 && sig[ord[c]] > 1e-15 * smax) ++c;
      flag = c;
    }
    __syncthreads();
    ptop = flag;
    // H holds the Householder vectors u_i (rows of length q) after the top columns
    double* U = Vg;                          // q x q region: columns 0..ptop-1 = top vectors
    double* Hh = Wg + (int64_t)p * q;        // ptop x q Householder vectors (scratch after W)
    double* beta = sig + 2 * 32;             // ptop betas
    for (int c = 0; c < ptop; ++c) {
      const int v = ord[c];
      const double inv = 1.0 / sig[v];
      for (int e = tid; e < q; e += blockDim.x) U[(int64_t)e * q + c] = at(v, e) * inv;
    }
    __syncthreads();
    // QR of the q x ptop matrix A = U[:, 0:ptop] (copy into Hh as columns)
    double* A = Hh + (int64_t)32 * q;  // q x ptop working copy, column-major
    for (int c = 0; c < ptop; ++c)
      for (int e = tid; e < q; e += blockDim.x) A[(int64_t)c * q + e] = U[(int64_t)e * q + c];
    __syncthreads();
    for (int i = 0; i < ptop; ++i) {
      double nx = 0.0;
      for (int e = i + tid; e < q; e += blockDim.x) nx = fma(A[(int64_t)i * q + e], A[(int64_t)i * q + e], nx);
      nx = sqrt(block_sum(nx, red));
      const double x0 = A[(int64_t)i * q + i];
      const double alpha = x0 >= 0.0 ? -nx : nx;
      // u = x - alpha e_i (entries i..q-1), beta = 2 / u^T u
      for (int e = tid; e < q; e += blockDim.x) Hh[(int64_t)i * q + e] = e < i ? 0.0 : (A[(int64_t)i * q + e] - (e == i ? alpha : 0.0));
      __syncthreads();
      double uu = 0.0;
      for (int e = i + tid; e < q; e += blockDim.x) uu = fma(Hh[(int64_t)i * q + e], Hh[(int64_t)i * q + e], uu);
      uu = block_sum(uu, red);
      if (tid == 0) beta[i] = uu > 0.0 ? 2.0 / uu : 0.0;
      __syncthreads();
      for (int c = i + 1; c < ptop; ++c) {
        double d = 0.0;
        for (int e = i + tid; e < q; e += blockDim.x) d = fma(Hh[(int64_t)i * q + e], A[(int64_t)c * q + e], d);
        d = block_sum(d, red) * beta[i];
        for (int e = i + tid; e < q; e += blockDim.x) A[(int64_t)c * q + e] -= d * Hh[(int64_t)i * q + e];
        __syncthreads();
      }
    }
    // completion: column k >= ptop of Q = H_0 H_1 ... H_{ptop-1} e_k, one
    // thread per column
    for (int k = ptop + tid; k < q; k += blockDim.x) {
      for (int e = 0; e < q; ++e) U[(int64_t)e * q + k] = (e == k) ? 1.0 : 0.0;
      for (int i = ptop - 1; i >= 0; --i) {
        double d = 0.0;
        for (int e = i; e < q; ++e) d = fma(Hh[(int64_t)i * q + e], U[(int64_t)e * q + k], d);
        d *= beta[i];
        for (int e = i; e < q; ++e) U[(int64_t)e * q + k] -= d * Hh[(int64_t)i * q + e];
      }
    }
    __syncthreads();
  }
  // outputs: vector t = column q-1-t of the descending-sigma V
  for (int t = 0; t < ell; ++t) {
    const int c = q - 1 - t;
    // source column of Vfull: cols case -> ord[c]; rows case -> c (already ordered)
    const int src = cols ? ord[c] : c;
    __shared__ double bv[DT];
    __shared__ int bi[DT];
    double best = -1.0;
    int arg = 0;
    for (int e = tid; e < q; e += blockDim.x) {
      const double a = fabs(Vfull[(int64_t)e * q + src]);
      if (a > best) { best = a; arg = e; }
    }
    bv[tid] = best;
    bi[tid] = arg;
    __syncthreads();
    if (tid == 0) {
      double b0 = -1.0;
      int a0 = 0;
      for (int u = 0; u < (int)blockDim.x; ++u)
        if (bv[u] > b0 || (bv[u] == b0 && bi[u] < a0)) { b0 = bv[u]; a0 = bi[u]; }
      rot[0] = Vfull[(int64_t)a0 * q + src] < 0.0 ? -1.0 : 1.0;
      const double s_ = cols ? sig[ord[c]] : (c < ptop ? sig[ord[c]] : 0.0);
      sv[t] = s_;
    }
    __syncthreads();
    for (int e = tid; e < q; e += blockDim.x) zeta[(int64_t)t * q + e] = rot[0] * Vfull[(int64_t)e * q + src];
    __syncthreads();
  }
}

// G (n x n) += sum_v x_v x_v^T (+ G2): every element sums its products in
// vector order with separate multiply and add, as the reference's loops
// (spectra.cpp:22-37, 40-44) do, so the result is bit-identical to them
__global__ void k_gram_update(double* __restrict__ G, int64_t n, const double* __restrict__ X, int64_t nvec,
                              const double* __restrict__ G2) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    double g = G[e];
    for (int64_t v = 0; v < nvec; ++v) {
      const double xi = X[v * n + i];
      if (xi == 0.0) continue;  // accumulate_dense skips zero rows; the sparse form never touches them
      g = __dadd_rn(g, __dmul_rn(xi, X[v * n + j]));
    }
    if (G2) g = __dadd_rn(g, G2[e]);
    G[e] = g;
  }
}

void launch_sample_one(const uint32_t* bits, int64_t stride, int64_t nwords, int64_t pool, int count, uint64_t seed,
                       uint64_t index, int32_t* drawn, uint32_t* words, int32_t* kept, int64_t* nkept,
                       cudaStream_t s) {
  k_sample_one<<<1, DT, 0, s>>>(bits, stride, nwords, pool, count, seed, index, drawn, words, kept, nkept);
}

size_t small_svd_scratch_doubles(int p, int q) {
  // W (p x q) + Householder vectors (32 x q) + working copy (q x 32) | V (q x q)
  return (size_t)p * q + (size_t)64 * q + (size_t)q * q + 160;
}

void launch_small_svd(const double* S, int p, int q, int ell, double* scratch, double* zeta, double* sv,
                      cudaStream_t s) {
  double* W = scratch;
  double* V = W + (size_t)p * q + (size_t)64 * q;
  double* sig = V + (size_t)q * q;  // 32 sigmas + 32 (pad) + 32 betas
  int* ord = reinterpret_cast<int*>(sig + 128);
  k_small_svd<<<1, DT, 0, s>>>(S, p, q, ell, W, V, sig, ord, zeta, sv);
}

void launch_gram_update(double* G, int64_t n, const double* X, int64_t nvec, const double* G2, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((n * n + 255) / 256, 148 * 8);
  k_gram_update<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(G, n, X, nvec, G2);
}

}  // namespace rsmk
