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
// CTA owns a 64 x (32*CPL) tile of G (NW warps x RPW rows, lane = column)
// and a slice of the trial list. Stage 2 stores each trial's top vectors
// expanded (rp/2 planes of npad (v_2p, v_2p+1) pairs, zero outside the
// support), so the tile's row block and column block of a plane are two
// contiguous 16-byte-aligned runs: they are streamed into shared memory with
// 1-D bulk copies (TMA) through an NS-stage ring of CH-trial groups guarded
// by mbarriers. Each warp applies the rank-R update to its RPW x 32*CPL
// register block, skipping rows outside the support (warp-uniform, on the
// uniform datapath) and reading its columns' pairs conflict-free.
//
// No atomics: each tile x slice partial is written once and stage 3b sums
// the slices in a fixed order, so G is bitwise reproducible. Only tiles
// touching the upper triangle are computed; stage 3b mirrors them (the
// reference G is exactly symmetric).
#include <cstdlib>

#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// 1-D bulk copy global -> shared through the TMA engine, completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int R, int CPL, int RG>
struct GramCfg {
  static constexpr int NW = 8;             // warps
  static constexpr int WPR = NW / RG;      // warps sharing a row group (split columns)
  static constexpr int LCPL = CPL / WPR;   // columns per lane
  static constexpr int RP = (R + 1) & ~1;  // planes * 2
  static constexpr int NP = RP / 2;        // planes
  static constexpr int TR = 64;
  static constexpr int TC = 32 * CPL;
  static constexpr int RPW = TR / RG;          // rows per warp
  static constexpr int CH = (R <= 4) ? 4 : 2;  // trials per ring stage
  static constexpr int NS = 4;                 // ring depth (stages)
  static constexpr int SLOT = (TR + TC) * RP;  // doubles per trial slot
};

}  // namespace

// NW warps own RPW x TC register blocks of the 64 x TC tile and take turns
// feeding the ring (group h is produced by warp h % NW): lane u < CH of the
// producer publishes trial g*CH+u's row-support words in the stage and
// issues its 2*NP bulk copies (row block and column block of every plane),
// completing on the stage's full barrier. Every warp releases a stage through
// its empty barrier; the stage released `lag` groups ago is refilled with the
// group NS ahead of it, so a producer rarely waits for the slowest warp. A
// warp loads the support words of the next group it produces right after
// producing one. Row activity is made warp-uniform with a redux so the
// compiler branches on the uniform datapath.
template <int R, int CPL, int RG>
__global__ void __launch_bounds__(256, 2) k_gram(GramArgs a) {
  using C = GramCfg<R, CPL, RG>;
  constexpr int RP = C::RP, NP = C::NP, TR = C::TR, TC = C::TC, RPW = C::RPW, CH = C::CH, NS = C::NS,
                SLOT = C::SLOT, NW = C::NW, LCPL = C::LCPL;
  static_assert(LCPL >= 1 && LCPL * C::WPR == CPL, "column split");
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;                                                     // [NS][CH][SLOT]
  uint2* rowsup = reinterpret_cast<uint2*>(ring + NS * CH * SLOT);       // [NS][CH]
  int* stage_nt = reinterpret_cast<int*>(rowsup + NS * CH);              // [NS]
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_nt + 2 * ((NS + 1) / 2));  // [NS]
  uint64_t* empty = full + NS;                                           // [NS]

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
  const int64_t tstride = a.npad * RP;  // doubles per trial

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 32);
      mbar_init(empty + s, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ---- producer state: lane u < CH owns trial g*CH + u of its groups ----
  unsigned n_w0 = 0, n_w1 = 0, n_any = 0;
  auto load = [&](int64_t g) {
    const int64_t i = g * CH + lane;
    n_w0 = n_w1 = n_any = 0;
    if (lane < CH && g < ngroups && i < ntr) {
      const uint32_t* cm = a.t_cm + (tb + i) * a.cmw;
      n_w0 = __ldg(cm + wrow);
      n_w1 = __ldg(cm + wrow + 1);
#pragma unroll
      for (int s = 0; s < CPL; ++s) n_any |= __ldg(cm + wcol + s);
    }
  };
  auto produce = [&](int64_t g) {
    const int st = (int)(g % NS);
    const int64_t i = g * CH + lane;
    // a trial with no support rows or no support columns in the tile adds nothing
    const bool live = lane < CH && i < ntr && (n_w0 | n_w1) != 0 && n_any != 0;
    if (lane < CH) rowsup[st * CH + lane] = live ? make_uint2(n_w0, n_w1) : make_uint2(0u, 0u);
    const unsigned bytes = __popc(__ballot_sync(0xffffffffu, live)) * (unsigned)(SLOT * 8);
    if (lane == 0) {
      const int64_t rem = ntr - g * CH;
      stage_nt[st] = (int)(rem < CH ? rem : CH);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(full + st, bytes);
    else mbar_arrive(full + st);
    if (live) {
      double* slot = ring + (st * CH + lane) * SLOT;
      const double* src = a.V + (tb + i) * tstride;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        bulk_g2s(slot + p * TR * 2, src + p * a.npad * 2 + row0 * 2, TR * 16, full + st);
        bulk_g2s(slot + TR * RP + p * TC * 2, src + p * a.npad * 2 + col0 * 2, TC * 16, full + st);
      }
    }
    load(g + NW);  // this warp's next group
  };
  // group h is produced by warp h % NW; groups 0..NS-1 fill the empty ring
  load(warp);
  for (int h = warp; h < NS && h < ngroups; h += NW) produce(h);

  double acc[RPW][LCPL];
#pragma unroll
  for (int i = 0; i < RPW; ++i)
#pragma unroll
    for (int s = 0; s < LCPL; ++s) acc[i][s] = 0.0;

  const int rfirst = (warp % RG) * RPW;      // this warp's rows within the tile
  const int cfirst = (warp / RG) * 32 * LCPL;  // and its first column
  const int wword = rfirst >> 5;             // row-support word of those rows
  const int shI = rfirst & 31;               // bit offset inside it
  constexpr unsigned RMASK = RPW >= 32 ? 0xffffffffu : ((1u << RPW) - 1u);
  for (int64_t g = 0; g < ngroups; ++g) {
    const int st = (int)(g % NS);
    if (g >= a.lag && g + NS - a.lag < ngroups && (int)((g + NS - a.lag) % NW) == warp) {
      // refill the stage group g-lag used once every warp has released it
      mbar_wait(empty + (int)((g - a.lag) % NS), (unsigned)(((g - a.lag) / NS) & 1));
      produce(g + NS - a.lag);
    }
    mbar_wait(full + st, (unsigned)((g / NS) & 1));
    const int nt = stage_nt[st];
#pragma unroll 1
    for (int u = 0; u < nt; ++u) {
      const uint2 ws = rowsup[st * CH + u];
      const unsigned rb = __reduce_or_sync(0xffffffffu, ((wword ? ws.y : ws.x) >> shI) & RMASK);
      if (rb == 0) continue;
      const double* VI = ring + (st * CH + u) * SLOT;
      const double* VJ = VI + TR * RP;
      // this lane's columns (zero outside the support)
      double vj[LCPL][RP];
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int s = 0; s < LCPL; ++s) {
          const double2 t = reinterpret_cast<const double2*>(VJ + p * TC * 2)[cfirst + lane + 32 * s];
          vj[s][2 * p] = t.x;
          vj[s][2 * p + 1] = t.y;
        }
#pragma unroll
      for (int r8 = 0; r8 < RPW; ++r8) {
        if (rb & (1u << r8)) {  // warp-uniform
          double x[RP];
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const double2 t = reinterpret_cast<const double2*>(VI + p * TR * 2)[rfirst + r8];
            x[2 * p] = t.x;
            x[2 * p + 1] = t.y;
          }
#pragma unroll
          for (int s = 0; s < LCPL; ++s)
#pragma unroll
            for (int k = 0; k < R; ++k) acc[r8][s] = fma(-x[k], vj[s][k], acc[r8][s]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
  // ---- write (or add to) the slice partial ----
  double* out = a.P + (int64_t)slice * a.npad * a.npad;
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int64_t row = row0 + rfirst + i;
#pragma unroll
    for (int s = 0; s < LCPL; ++s) {
      double* o = out + row * a.npad + col0 + cfirst + lane + 32 * s;
      *o = a.accumulate ? *o + acc[i][s] : acc[i][s];
    }
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

template <int R, int CPL, int RG>
static size_t gram_smem() {
  using C = GramCfg<R, CPL, RG>;
  return sizeof(double) * (size_t)C::NS * C::CH * C::SLOT + sizeof(uint2) * C::NS * C::CH +
         sizeof(int) * 2 * ((C::NS + 1) / 2) + sizeof(uint64_t) * 2 * C::NS;
}

template <int R, int CPL, int RG>
static void launch_gram_t(const GramArgs& a0, int ntiles, cudaStream_t s) {
  using C = GramCfg<R, CPL, RG>;
  GramArgs a = a0;
  static const int lag_env = [] {
    const char* e = getenv("RSM_GRAM_LAG");
    return e ? atoi(e) : 0;
  }();
  a.lag = lag_env > 0 && lag_env < C::NS ? lag_env : 2;
  const size_t smem = gram_smem<R, CPL, RG>();
  cudaFuncSetAttribute(k_gram<R, CPL, RG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)ntiles, (unsigned)a.nslices);
  k_gram<R, CPL, RG><<<grid, 256, smem, s>>>(a);
}

int gram_cols_per_lane(int R) { return R <= 4 ? 4 : (R <= 8 ? 2 : 1); }

int gram_ctas_per_sm(int) { return 2; }

// row groups per tile: 8 (8 rows x all tile columns per warp) or 4 (16 rows
// x half the columns: half the column reads per trial, twice the row reads)
static int gram_row_groups() {
  static int rg = [] {
    const char* e = getenv("RSM_GRAM_RG");
    return (e && atoi(e) == 4) ? 4 : 8;
  }();
  return rg;
}

template <int R, int CPL>
static void launch_gram_r(const GramArgs& a, int ntiles, cudaStream_t s) {
  if constexpr (CPL >= 2) {
    if (gram_row_groups() == 4) {
      launch_gram_t<R, CPL, 4>(a, ntiles, s);
      return;
    }
  }
  launch_gram_t<R, CPL, 8>(a, ntiles, s);
}

void launch_gram(const GramArgs& a, int ntiles, cudaStream_t s) {
  switch (a.R) {
    case 1: launch_gram_r<1, 4>(a, ntiles, s); break;
    case 2: launch_gram_r<2, 4>(a, ntiles, s); break;
    case 3: launch_gram_r<3, 4>(a, ntiles, s); break;
    case 4: launch_gram_r<4, 4>(a, ntiles, s); break;
    case 5: launch_gram_r<5, 2>(a, ntiles, s); break;
    case 6: launch_gram_r<6, 2>(a, ntiles, s); break;
    case 7: launch_gram_r<7, 2>(a, ntiles, s); break;
    case 8: launch_gram_r<8, 2>(a, ntiles, s); break;
    case 9: launch_gram_r<9, 1>(a, ntiles, s); break;
    case 10: launch_gram_r<10, 1>(a, ntiles, s); break;
    case 11: launch_gram_r<11, 1>(a, ntiles, s); break;
    case 12: launch_gram_r<12, 1>(a, ntiles, s); break;
    case 13: launch_gram_r<13, 1>(a, ntiles, s); break;
    case 14: launch_gram_r<14, 1>(a, ntiles, s); break;
    case 15: launch_gram_r<15, 1>(a, ntiles, s); break;
    default: launch_gram_r<16, 1>(a, ntiles, s); break;
  }
}

void launch_gram_reduce(const double* P, int nslices, int64_t npad, int64_t n, const int* cnt,
                        double* G, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  k_gram_reduce<<<grid, block, 0, s>>>(P, nslices, npad, n, cnt, G);
}

}  // namespace rsmk
