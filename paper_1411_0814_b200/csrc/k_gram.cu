// k_gram.cu -- stage 3: accumulation of the n x n constraint Gram matrix.
//
// Reference: GramAccumulator::accumulate (spectra.cpp:7-23, paths relative
// to /root/reference/proj) adds zeta zeta^T for every harvested vector, in
// attempt order (harvest.cpp:110-117). Per trial the harvested vectors sum to
// I - V V^T on the trial's column support (see k_svd.cu), so
//     G = diag(count) - sum_t  E_t V_t V_t^T E_t^T
// with count[c] = number of trials whose support holds column c. This kernel
// forms the second term with register-resident output tiles: a CTA owns a
// 64 x (32*CPL) tile of G (8 warps x 8 rows, lane = column) and a slice of
// the trial list; every trial's compact V rows that fall into the tile are
// staged in shared memory (zero rows where the trial does not touch the
// tile), and each warp applies the rank-R update to its 8 x 32*CPL block,
// skipping rows outside the support. No atomics: each tile x slice partial
// is written once and stage 3b sums the slices in a fixed order, so G is
// bitwise reproducible. Only tiles touching the upper triangle are computed;
// stage 3b mirrors them (the reference G is exactly symmetric).
#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

template <int R, int CPL>
struct GramCfg {
  static constexpr int TR = 64;
  static constexpr int TC = 32 * CPL;
  static constexpr int CH = (R <= 4) ? 8 : (R <= 8 ? 4 : 2);  // trials per staged chunk
};

template <int R, int CPL>
__global__ void __launch_bounds__(256) k_gram(GramArgs a) {
  using C = GramCfg<R, CPL>;
  constexpr int TR = C::TR, TC = C::TC, CH = C::CH, SPAN = TR + TC;
  extern __shared__ __align__(16) double sm[];
  double* VI = sm;                       // [CH][TR][R]
  double* VJ = VI + CH * TR * R;         // [CH][TC][R]
  uint32_t* rbits = reinterpret_cast<uint32_t*>(VJ + CH * TC * R);  // [CH][2]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 tile = a.tiles[blockIdx.x];
  const int64_t row0 = (int64_t)tile.x * TR, col0 = (int64_t)tile.y * TC;
  const int slice = blockIdx.y;
  const int64_t per = (a.T + a.nslices - 1) / a.nslices;
  const int64_t t_begin = slice * per;
  const int64_t t_end = (t_begin + per < a.T) ? t_begin + per : a.T;

  double acc[8][CPL];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int s = 0; s < CPL; ++s) acc[i][s] = 0.0;

  for (int64_t t0 = t_begin; t0 < t_end; t0 += CH) {
    // ---- stage the chunk's V rows for the tile's row and column ranges ----
    for (int p = tid; p < CH * SPAN; p += 256) {
      const int u = p / SPAN, pos = p % SPAN;
      const int64_t t = t0 + u;
      double* dst = (pos < TR) ? VI + ((int64_t)u * TR + pos) * R
                               : VJ + ((int64_t)u * TC + (pos - TR)) * R;
      bool have = false;
      if (t < t_end) {
        const int64_t c = (pos < TR) ? row0 + pos : col0 + (pos - TR);
        const uint32_t word = __ldg(a.t_cm + t * a.cmw + (c >> 5));
        const uint32_t bit = 1u << (c & 31);
        if (word & bit) {
          const int64_t ci = __ldg(a.t_pre + t * a.cmw + (c >> 5)) + __popc(word & (bit - 1u));
          const double* src = a.V + __ldg(a.t_off + t) + ci * R;
#pragma unroll
          for (int k = 0; k < R; ++k) dst[k] = __ldg(src + k);
          have = true;
        }
      }
      if (!have) {
#pragma unroll
        for (int k = 0; k < R; ++k) dst[k] = 0.0;
      }
    }
    if (tid < CH * 2) {
      const int u = tid >> 1, h = tid & 1;
      const int64_t t = t0 + u;
      rbits[tid] = (t < t_end) ? __ldg(a.t_cm + t * a.cmw + (row0 >> 5) + h) : 0u;
    }
    __syncthreads();
    // ---- rank-R updates of the register tile ----
#pragma unroll 1
    for (int u = 0; u < CH; ++u) {
      const uint32_t rb = (rbits[u * 2 + (warp >> 2)] >> ((warp & 3) * 8)) & 0xffu;
      if (rb == 0) continue;  // warp-uniform
      double vj[CPL][R];
#pragma unroll
      for (int s = 0; s < CPL; ++s)
#pragma unroll
        for (int k = 0; k < R; ++k) vj[s][k] = VJ[((int64_t)u * TC + lane + 32 * s) * R + k];
      const double* vib = VI + ((int64_t)u * TR + warp * 8) * R;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (rb & (1u << i)) {
          double vi[R];
#pragma unroll
          for (int k = 0; k < R; ++k) vi[k] = vib[i * R + k];
#pragma unroll
          for (int s = 0; s < CPL; ++s) {
            double d = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) d = fma(vi[k], vj[s][k], d);
            acc[i][s] -= d;
          }
        }
      }
    }
    __syncthreads();
  }
  // ---- write the slice partial ----
  double* out = a.P + (int64_t)slice * a.npad * a.npad;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = row0 + warp * 8 + i;
#pragma unroll
    for (int s = 0; s < CPL; ++s) out[row * a.npad + col0 + lane + 32 * s] = acc[i][s];
  }
}

// G[a][b] = G[b][a] = sum_slices P[s][a][b] (+count on the diagonal), a <= b.
// One CTA per 32 x 32 upper tile; transposed writes go through smem.
__global__ void k_gram_reduce(const double* __restrict__ P, int nslices, int64_t npad, int64_t n,
                              const int* __restrict__ cnt, double* __restrict__ G) {
  __shared__ double tilebuf[32][33];
  const int64_t bi = (int64_t)blockIdx.y * 32, bj = (int64_t)blockIdx.x * 32;
  if (bj + 31 < bi) return;  // strictly lower tile: produced by its mirror
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += blockDim.y) {
    const int64_t i = bi + r, j = bj + tx;
    double v = 0.0;
    if (i < n && j < n && i <= j) {
      for (int s = 0; s < nslices; ++s) v += P[(int64_t)s * npad * npad + i * npad + j];
      if (i == j) v += (double)cnt[i];
      G[i * n + j] = v;
    }
    tilebuf[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += blockDim.y) {
    const int64_t j = bj + r, i = bi + tx;  // write G[j][i] for i < j
    if (i < n && j < n && i < j) G[j * n + i] = tilebuf[tx][r];
  }
}

template <int R, int CPL>
static void launch_gram_t(const GramArgs& a, int ntiles, cudaStream_t s) {
  using C = GramCfg<R, CPL>;
  const size_t smem = sizeof(double) * (size_t)C::CH * (C::TR + C::TC) * R +
                      sizeof(uint32_t) * C::CH * 2;
  cudaFuncSetAttribute(k_gram<R, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)ntiles, (unsigned)a.nslices);
  k_gram<R, CPL><<<grid, 256, smem, s>>>(a);
}

int gram_cols_per_lane(int R) { return R <= 4 ? 4 : (R <= 8 ? 2 : 1); }

void launch_gram(const GramArgs& a, int ntiles, cudaStream_t s) {
  switch (a.R) {
    case 1: launch_gram_t<1, 4>(a, ntiles, s); break;
    case 2: launch_gram_t<2, 4>(a, ntiles, s); break;
    case 3: launch_gram_t<3, 4>(a, ntiles, s); break;
    case 4: launch_gram_t<4, 4>(a, ntiles, s); break;
    case 5: launch_gram_t<5, 2>(a, ntiles, s); break;
    case 6: launch_gram_t<6, 2>(a, ntiles, s); break;
    case 7: launch_gram_t<7, 2>(a, ntiles, s); break;
    case 8: launch_gram_t<8, 2>(a, ntiles, s); break;
    case 9: launch_gram_t<9, 1>(a, ntiles, s); break;
    case 10: launch_gram_t<10, 1>(a, ntiles, s); break;
    case 11: launch_gram_t<11, 1>(a, ntiles, s); break;
    case 12: launch_gram_t<12, 1>(a, ntiles, s); break;
    case 13: launch_gram_t<13, 1>(a, ntiles, s); break;
    case 14: launch_gram_t<14, 1>(a, ntiles, s); break;
    case 15: launch_gram_t<15, 1>(a, ntiles, s); break;
    default: launch_gram_t<16, 1>(a, ntiles, s); break;
  }
}

void launch_gram_reduce(const double* P, int nslices, int64_t npad, int64_t n, const int* cnt,
                        double* G, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  k_gram_reduce<<<grid, block, 0, s>>>(P, nslices, npad, n, cnt, G);
}

}  // namespace rsmk
