// k_gram.cu -- stage 3: accumulation of the n x n constraint Gram matrix.
//
// Reference: GramAccumulator::accumulate (spectra.cpp:7-23, paths relative
// to /root/reference/proj) adds zeta zeta^T for every harvested vector, in
// attempt order (harvest.cpp:110-117). Per trial the harvested vectors sum to
// I - V V^T on the trial's column support (see k_svd.cu), so
//     G = diag(count) - sum_t  E_t V_t V_t^T E_t^T
// with count[c] = number of trials whose support holds column c.
//
// This kernel forms the second term with register-resident output tiles: a
// CTA owns a 64 x (32*CPL) tile of G (8 warps x 8 rows, lane = column) and a
// slice of the trial list. For every trial the compact V rows that fall into
// the tile's row block and column block are two contiguous segments of the
// trial's V array (k_svd writes the rows in support order with an even
// stride RP), so they are streamed into shared memory with 16-byte
// cp.async copies through an NS-stage ring of CH-trial groups: the copies of
// group g+NS-1 are in flight while group g is computed. The per-trial
// metadata (segment offsets, support words) is loaded one 64-trial batch
// ahead into registers and published to shared memory. Each warp applies
// the rank-R update to its 8 x 32*CPL register block, skipping rows outside
// the support (warp-uniform) and reading zeros for columns outside it.
//
// No atomics: each tile x slice partial is written once and stage 3b sums
// the slices in a fixed order, so G is bitwise reproducible. Only tiles
// touching the upper triangle are computed; stage 3b mirrors them (the
// reference G is exactly symmetric).
#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int R, int CPL>
struct GramCfg {
  static constexpr int RP = (R + 1) & ~1;  // padded row stride (doubles)
  static constexpr int TR = 64;
  static constexpr int TC = 32 * CPL;
  static constexpr int CH = (R <= 4) ? 4 : 2;  // trials per pipeline group
  static constexpr int NS = 3;                 // pipeline depth (groups)
  static constexpr int MB = 64;                // metadata batch (trials)
  static constexpr int SLOT = (TR + TC) * RP;  // doubles per trial slot
};

struct TrialMeta {
  long long srcI, srcJ;  // segment starts in V (doubles)
  unsigned wI[2];
  unsigned wJ[4];
  int preI[2];  // support bits before each row-block word
  int preJ[4];  // support bits before each column-block word
};

}  // namespace

template <int R, int CPL>
__global__ void __launch_bounds__(256, 2) k_gram(GramArgs a) {
  using C = GramCfg<R, CPL>;
  constexpr int RP = C::RP, TR = C::TR, TC = C::TC, CH = C::CH, NS = C::NS, MB = C::MB, SLOT = C::SLOT;
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;                                              // [NS][CH][SLOT]
  TrialMeta* meta = reinterpret_cast<TrialMeta*>(ring + NS * CH * SLOT);  // [2][MB]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 tile = a.tiles[blockIdx.x];
  const int64_t row0 = (int64_t)tile.x * TR, col0 = (int64_t)tile.y * TC;
  const int64_t wrow = row0 >> 5, wcol = col0 >> 5;
  const int slice = blockIdx.y;
  const int64_t per = (a.T + a.nslices - 1) / a.nslices;
  const int64_t tb = slice * per;
  const int64_t te = (tb + per < a.T) ? tb + per : a.T;
  const int64_t ntr = te > tb ? te - tb : 0;
  const int64_t ngroups = (ntr + CH - 1) / CH;

  // ---- metadata of one batch: thread u < MB loads trial tb + b*MB + u ----
  long long m_off = 0;
  unsigned m_pI = 0, m_pJ = 0, m_w[2 + CPL];
  auto meta_load = [&](int64_t b) {
    const int64_t t = tb + b * MB + tid;
    if (tid < MB && b * MB + tid < ntr) {
      m_off = __ldg(a.t_off + t);
      m_pI = __ldg(a.t_pre + t * a.cmw + wrow);
      m_pJ = __ldg(a.t_pre + t * a.cmw + wcol);
      m_w[0] = __ldg(a.t_cm + t * a.cmw + wrow);
      m_w[1] = __ldg(a.t_cm + t * a.cmw + wrow + 1);
#pragma unroll
      for (int s = 0; s < CPL; ++s) m_w[2 + s] = __ldg(a.t_cm + t * a.cmw + wcol + s);
    }
  };
  auto meta_store = [&](int64_t b) {
    if (tid < MB && b * MB + tid < ntr) {
      TrialMeta& m = meta[(b & 1) * MB + tid];
      m.srcI = m_off + (long long)m_pI * RP;
      m.srcJ = m_off + (long long)m_pJ * RP;
      m.wI[0] = m_w[0];
      m.wI[1] = m_w[1];
      m.preI[0] = 0;
      m.preI[1] = __popc(m_w[0]);
      int run = 0;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const unsigned w = s < CPL ? m_w[2 + s] : 0u;
        m.wJ[s] = w;
        m.preJ[s] = run;
        run += __popc(w);
      }
    }
  };
  // Issue the copies of group g into ring stage g % NS: per trial the two
  // compact segments (support rows of the tile's row block, support columns
  // of its column block), contiguous in V, as 16-byte cp.async chunks.
  auto issue = [&](int64_t g) {
    if (g < ngroups) {
      double* st = ring + (g % NS) * CH * SLOT;
      const int64_t i0 = g * CH;
      const int nt = (int)((ntr - i0) < CH ? (ntr - i0) : CH);
#pragma unroll 1
      for (int u = 0; u < nt; ++u) {
        const int64_t i = i0 + u;
        const TrialMeta& m = meta[((i / MB) & 1) * MB + (i % MB)];
        double* slot = st + u * SLOT;
        const int cI = (m.preI[1] + __popc(m.wI[1])) * (RP / 2);
        const int cJ = (m.preJ[3] + __popc(m.wJ[3])) * (RP / 2);
        for (int c = tid; c < cI + cJ; c += 256) {
          if (c < cI) cp_async16(slot + 2 * c, a.V + m.srcI + 2 * c);
          else cp_async16(slot + TR * RP + 2 * (c - cI), a.V + m.srcJ + 2 * (c - cI));
        }
      }
    }
    cp_async_commit();  // (possibly empty) group keeps the wait count uniform
  };

  double acc[8][CPL];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int s = 0; s < CPL; ++s) acc[i][s] = 0.0;

  if (ngroups > 0) {
    meta_load(0);
    meta_store(0);
    meta_load(1);  // batch 1 in registers, published after the first group
    __syncthreads();
#pragma unroll
    for (int g = 0; g < NS - 1; ++g) issue(g);
  }
  const int shI = (warp & 3) * 8;
  for (int64_t g = 0; g < ngroups; ++g) {
    // publish the next metadata batch early enough for the copies that need it
    // (batch b+1 is published one group after batch b starts, long before
    // issue() reaches it; buffer (b+1)&1 last served batch b-1, which is done)
    if (g >= 1 && ((g - 1) * CH) % MB == 0) {
      const int64_t b = ((g - 1) * CH) / MB;
      meta_store(b + 1);
      meta_load(b + 2);
    }
    __syncthreads();  // meta visible; previous compute done with the stage we refill
    issue(g + NS - 1);
    cp_async_wait<NS - 1>();
    __syncthreads();  // group g landed for every thread
    const double* st = ring + (g % NS) * CH * SLOT;
#pragma unroll 1
    for (int u = 0; u < CH; ++u) {
      const int64_t i = g * CH + u;
      if (i >= ntr) break;
      const TrialMeta& m = meta[((i / MB) & 1) * MB + (i % MB)];
      const unsigned wI0 = m.wI[0], wI1 = m.wI[1];
      const unsigned rb = ((warp < 4 ? wI0 : wI1) >> shI) & 0xffu;
      if (rb == 0) continue;  // warp-uniform
      const double* VI = st + u * SLOT;
      const double* VJ = VI + TR * RP;
      // this lane's columns: compact index = support bits below it (zeros outside)
      double vj[CPL][RP];
#pragma unroll
      for (int s = 0; s < CPL; ++s) {
        const unsigned w = m.wJ[s];
        const bool sel = (w >> lane) & 1u;
        const int cj = m.preJ[s] + __popc(w & ((1u << lane) - 1u));
#pragma unroll
        for (int h = 0; h < RP / 2; ++h) {
          const double2 t = sel ? reinterpret_cast<const double2*>(VJ + cj * RP)[h] : make_double2(0.0, 0.0);
          vj[s][2 * h] = t.x;
          vj[s][2 * h + 1] = t.y;
        }
      }
      int ci = (warp < 4) ? __popc(wI0 & ((1u << shI) - 1u)) : m.preI[1] + __popc(wI1 & ((1u << shI) - 1u));
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) {
        if (rb & (1u << r8)) {  // warp-uniform
          double x[RP];
#pragma unroll
          for (int h = 0; h < RP / 2; ++h) {
            const double2 t = reinterpret_cast<const double2*>(VI + ci * RP)[h];
            x[2 * h] = t.x;
            x[2 * h + 1] = t.y;
          }
          ++ci;
#pragma unroll
          for (int s = 0; s < CPL; ++s)
#pragma unroll
            for (int k = 0; k < R; ++k) acc[r8][s] = fma(-x[k], vj[s][k], acc[r8][s]);
        }
      }
    }
  }
  cp_async_wait<0>();
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
static size_t gram_smem() {
  using C = GramCfg<R, CPL>;
  return sizeof(double) * (size_t)C::NS * C::CH * C::SLOT + sizeof(TrialMeta) * 2 * C::MB;
}

template <int R, int CPL>
static void launch_gram_t(const GramArgs& a, int ntiles, cudaStream_t s) {
  const size_t smem = gram_smem<R, CPL>();
  cudaFuncSetAttribute(k_gram<R, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)ntiles, (unsigned)a.nslices);
  k_gram<R, CPL><<<grid, 256, smem, s>>>(a);
}

int gram_cols_per_lane(int R) { return R <= 4 ? 4 : (R <= 8 ? 2 : 1); }

int gram_ctas_per_sm(int) { return 2; }

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
