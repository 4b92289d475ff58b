// k_gram_i8.cu -- stage 3 on the 5th-generation tensor cores: the constraint
// Gram G = diag(count) - W^T W as an exact-integer split ("Ozaki") SYRK on
// tcgen05.mma kind::i8 with TMEM accumulators.
//
// Reference: GramAccumulator::accumulate (spectra.cpp:7-23, paths relative to
// /root/reference/proj) adds zeta zeta^T for every harvested vector; per trial
// those sum to I - V_t V_t^T on the trial's support (k_svd.cu), so
//     G = diag(count) - W^T W,   W = [E_1 V_1 | E_2 V_2 | ...]^T  (K x n),
// K = trials * r, every entry of W an entry of an orthonormal basis (|w| <= 1).
//
// Exact split. Each w is written in balanced signed base-256 digits,
//     w = a_0 2^-6 + sum_{1<=s<S} a_s 2^(-6-8s) + e,  a_0 in [-65, 65],
//     a_s in [-128, 127], |e| <= 2^(-7-8(S-1))       (split_i8 below),
// so  w_i w_j ~= sum_{d<S} 2^(-12-8d) * sum_{s+t=d} a_s(i) a_t(j)
// and each inner sum is an INTEGER dot product over K that tcgen05 computes
// exactly in int32 (|sum| <= S * 2^14 * Kc < 2^31 for K-chunks Kc <= 16384).
// The dropped classes (s+t >= S) and e bound the absolute error of one
// product by ~S 2^(2-8S) (S = 6, the default: 8.5e-14; S = 7: 3e-16), below
// the differences between two FP64 summation orders of the reference's own
// loop at these sizes; the per-class FP64 combination in the epilogue rounds
// once per class.
//
// Layout. The slices are stored MN-major: Wq[s][k][col] int8, row k = trial-
// vector, npad columns, so stage 2 writes each trial's vectors as contiguous
// rows. An output tile is 128 rows (G rows = W columns R) x 64 columns (C);
// only tiles touching the upper triangle run and k_gram_reduce mirrors them.
// Per K-step of 32 one 3-D TMA box brings all S slices of A = W[k0:k0+32, R]
// (SWIZZLE_128B, 128-byte rows) and one brings B = W[k0:k0+32, C]
// (SWIZZLE_64B) into a 5/6-stage smem ring. One elected thread issues the
// S(S+1)/2 MMAs (M=128, N=64, K=32, A and B MN-major) into S int32
// accumulators of 64 TMEM columns each (S*64 <= 512 columns). Four epilogue
// warps drain TMEM once per (tile, K-chunk) work unit, combine the classes in
// FP64 and write -sum into the K-chunk's partial (the same P layout k_gram
// uses), which k_gram_reduce sums in a fixed order: G is bitwise reproducible
// and exactly symmetric, with no atomics.
//
// Warp roles (192 threads, one CTA per SM, persistent over work units):
//   warp 0: TMA producer (one lane), warp 1: TMEM owner + MMA issuer (one
//   lane), warps 2-5: epilogue (warp w reads TMEM lanes 32*(w%4)..+31).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

namespace {

constexpr int BM = 128, BN = 64, KS = 32;
constexpr int NTHREADS = 192;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mb_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(su32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  unsigned p = 0;
  asm volatile(
      "{\n .reg .pred e;\n .reg .b32 r;\n elect.sync r|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}\n"
      : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// 32 consecutive int32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// UMMA shared-memory descriptor (tcgen05 "matrix descriptor"): start address,
// leading / stride byte offsets (>> 4), version 1, swizzle mode in [61,64)
__device__ __forceinline__ uint64_t smem_desc(unsigned addr, unsigned lbo, unsigned sbo, unsigned layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
constexpr unsigned kLayoutSW128 = 2, kLayoutSW64 = 4;
// instruction descriptor: D s32, A/B signed int8, both MN-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

template <int S>
struct I8Cfg {
  static constexpr int A_SLICE = KS * BM;        // bytes of one slice of the A box
  static constexpr int B_SLICE = KS * BN;        // and of the B box
  static constexpr int A_STAGE = S * A_SLICE;
  static constexpr int B_STAGE = S * B_SLICE;
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int NST = (220 * 1024) / STAGE;  // ring depth
  static constexpr int SMEM = 1024 + NST * STAGE + 256;
};

}  // namespace

template <int S>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_gram_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GramI8Args a) {
  using C = I8Cfg<S>;
  constexpr int NST = C::NST;
  extern __shared__ __align__(1024) uint8_t smraw[];
  // 1024-byte alignment for the 128B-swizzle atoms
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = sm;
  uint8_t* smB = sm + NST * C::A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * C::STAGE);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nunits = (int64_t)a.ntiles * a.nk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mb_init(full + s, 1);
      mb_init(empty + s, 1);
    }
    mb_init(tfull, 1);
    mb_init(tempty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int st = 0;
      unsigned ph = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t kc = u / a.ntiles;
        const int2 t = a.tiles[u % a.ntiles];
        const int64_t k0 = kc * a.Kc, k1 = min(k0 + a.Kc, a.Kpad);
        for (int64_t k = k0; k < k1; k += KS) {
          mb_wait(empty + st, ph ^ 1u);
          if (a.diag == 2) {  // diagnostic: no loads (MMA rate on stale smem)
            mb_arrive(full + st);
          } else {
            mb_expect_tx(full + st, (unsigned)C::STAGE);
            tma_3d(smA + st * C::A_STAGE, &tmA, t.x * BM, (int)k, 0, full + st);
            tma_3d(smB + st * C::B_STAGE, &tmB, t.y * BN, (int)k, 0, full + st);
          }
          if (++st == NST) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp runs the loop (every value warp-uniform, so descriptors
    // stay in uniform registers) and one elected lane issues: issuing from a
    // lane-0 branch made the compiler broadcast each descriptor per MMA and
    // capped the issue rate at about one MMA per 70 cycles.
    int st = 0;
    unsigned ph = 0, tph = 0;
    const uint64_t adesc0 = smem_desc(su32(smA), 0, 8 * BM, kLayoutSW128);
    const uint64_t bdesc0 = smem_desc(su32(smB), C::B_SLICE, 8 * BN, kLayoutSW64);
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int64_t kc = u / a.ntiles;
      const int64_t k0 = kc * a.Kc, k1 = min(k0 + a.Kc, a.Kpad);
      mb_wait(tempty, tph ^ 1u);  // the epilogue drained the previous unit
      tc_fence_after();
      for (int64_t k = k0; k < k1; k += KS) {
        mb_wait(full + st, ph);
        tc_fence_after();
        if (elect_one()) {
          // descriptor start addresses are in 16-byte units in the low bits.
          // For slice s of A the pairs (s, t), t = 0..S-1-s, land in classes
          // d = s + t, i.e. TMEM columns 64 (s + t): one MMA with the B slices
          // t0.. concatenated along N (the 3-D TMA box stores slice t at
          // t * B_SLICE, which is the descriptor's leading-byte offset between
          // 64-column SW64 atoms) covers up to four of them at once, so A_s is
          // read from shared memory once per 256 columns instead of once per pair.
          const uint64_t ab = adesc0 + (uint64_t)((st * C::A_STAGE) >> 4);
          const uint64_t bb = bdesc0 + (uint64_t)((st * C::B_STAGE) >> 4);
#pragma unroll
          for (int s = 0; s < S; ++s) {
#pragma unroll
            for (int t0 = 0; t0 < S - s; t0 += 4) {
              const int nt = (S - s - t0) < 4 ? (S - s - t0) : 4;
              if (a.diag != 1)  // diag 1: loads only
                mma_i8(tmem + (uint32_t)((s + t0) * BN), ab + (uint64_t)((s * C::A_SLICE) >> 4),
                       bb + (uint64_t)((t0 * C::B_SLICE) >> 4), idesc_n(nt * BN), (k > k0 || s > 0) ? 1u : 0u);
            }
          }
          tc_commit(empty + st);  // frees the stage once these MMAs have read it
        }
        __syncwarp();
        if (++st == NST) {
          st = 0;
          ph ^= 1u;
        }
      }
      if (elect_one()) tc_commit(tfull);  // accumulators complete
      __syncwarp();
      tph ^= 1u;
    }
  } else {
    // ---------------- epilogue: TMEM -> FP64 -> partial ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int rloc = 32 * q + lane;
    unsigned tph = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int64_t kc = u / a.ntiles;
      const int2 t = a.tiles[u % a.ntiles];
      mb_wait(tfull, tph);
      tc_fence_after();
      // a K-chunk past the end of a short trial chunk ran no MMA: it adds 0
      const bool live = kc * a.Kc < a.Kpad;
      const int64_t row = (int64_t)t.x * BM + rloc;
      double* out = a.P + kc * a.npad * a.npad + row * a.npad + (int64_t)t.y * BN;
#pragma unroll 1
      for (int h = 0; h < BN / 32; ++h) {
        double acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.0;
#pragma unroll
        for (int d = S - 1; d >= 0; --d) {  // small classes first
          int v[32];
          tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(d * BN + 32 * h), v);
          const double sc = live ? ldexp(1.0, -12 - 8 * d) : 0.0;
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] = fma((double)v[j], sc, acc[j]);
        }
        double2* o2 = reinterpret_cast<double2*>(out + 32 * h);
        if (a.accumulate) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const double2 p = o2[j];
            o2[j] = make_double2(p.x - acc[2 * j], p.y - acc[2 * j + 1]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) o2[j] = make_double2(-acc[2 * j], -acc[2 * j + 1]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(tempty);
      tph ^= 1u;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* m, const int8_t* W, int64_t npad, int64_t Kpad, int S, int box0, CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)npad, (cuuint64_t)Kpad, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)npad, (cuuint64_t)(npad * Kpad)};
  cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)KS, (cuuint32_t)S};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(W), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int S>
cudaError_t launch_i8_t(const GramI8Args& a, int sms, cudaStream_t s) {
  using C = I8Cfg<S>;
  CUtensorMap ma, mb;
  if (!make_map(&ma, a.W, a.npad, a.Kpad, S, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mb, a.W, a.npad, a.Kpad, S, BN, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  ensure_smem((const void*)k_gram_i8<S>, C::SMEM);
  const int64_t nunits = (int64_t)a.ntiles * a.nk;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nunits, sms));
  k_gram_i8<S><<<grid, NTHREADS, C::SMEM, s>>>(ma, mb, a);
  return cudaGetLastError();
}

}  // namespace

// RSM_I8_SLICES (5..7) overrides the default digit count
int gram_i8_slices() {
  static const int s = [] {
    const char* e = getenv("RSM_I8_SLICES");
    const int v = e ? atoi(e) : rsmd::kGramSlices;
    return v < 5 ? 5 : (v > 7 ? 7 : v);
  }();
  return s;
}

// int32 exactness: a class sums at most S products of |digits| <= 128, so
// |acc| <= S * 16384 * Kc < 2^31 for Kc <= 16384 and S <= 7
int64_t gram_i8_kmax() { return 16384; }

void gram_i8_tiles(int64_t npad, std::vector<int2>& t) {
  t.clear();
  for (int64_t a = 0; a < npad / BM; ++a)
    for (int64_t b = 0; b < npad / BN; ++b)
      if (BN * b + BN - 1 >= BM * a) t.push_back(make_int2((int)a, (int)b));
}

cudaError_t launch_gram_i8(const GramI8Args& a, int sms, cudaStream_t s) {
  switch (a.S) {
    case 5: return launch_i8_t<5>(a, sms, s);
    case 7: return launch_i8_t<7>(a, sms, s);
    default: return launch_i8_t<6>(a, sms, s);
  }
}

}  // namespace rsmk
