// k_normal_i8.cu -- stage 5's per-row normal matrices on the tcgen05 tensor
// cores: A_i = V_O(i)^T V_O(i) = sum_c m_ic v_c v_c^T for every row i at once,
// as an exact-integer GEMM  M (m x n, 0/1) x Q (n x NA*S int8 digits).
//
// Reference: solve_row (detail/row_solve.hpp:12-36, paths relative to
// /root/reference/proj) forms each row's least-squares problem on the basis
// rows at its observed columns; k_solve_u.cu solves it through the r x r
// normal matrix. Its packed upper entries q_cp = v_ci v_cj (|q| <= 1: V-hat
// has orthonormal columns) are written in S = 7 balanced signed base-256
// digits (rsmd::digits_i8, as stage 3's accumulator split), so
//     A_ip = sum_s 2^(-6-8s) * sum_c m_ic a_s(q_cp)
// and every inner sum is an integer dot product the tensor core accumulates
// exactly in int32 (|sum| <= 128 n). The truncation error of the digits is
// <= 2^(-7-48) per q, i.e. <= n 2^-55 (3e-14 at n = 1024) on an entry of
// size ~ observed fraction: below the rounding of an FP64 sum over the row.
//
// Layout. B = Q digits, precomputed once per V-hat (k_q_digits): hq halves of
// n rows x 128 bytes (column p*S + s of the padded N = 128 hq), TMA'd per
// 32-row K-step into an SW128 ring. A = the mask rows' bits, built by the
// four builder warps straight into the SW128 MN-major layout: lane t holds
// row (32w + t)'s mask word for the K-step, a five-stage shuffle butterfly
// transposes the 32 x 32 bit block, each column's 32 bits expand to 32 bytes
// (0/1) stored as two 16-byte chunks. One elected lane issues one MMA (M = 128, N = 128 hq,
// K = 32) per K-step into TMEM; the same four warps drain their TMEM lane
// quarter per 128-row tile, combine the digit columns in FP64 and write the
// packed normal matrices (m x NA, FP64).
//
// Warp roles (448 threads, persistent over 128-row tiles): warps 0-7 build A
// in two groups of four that take alternate K-steps, warps 8-11 drain TMEM
// (two accumulators, so a tile's epilogue overlaps the next tile's MMAs),
// warp 12 owns TMEM and issues MMAs, warp 13 is the TMA producer for B.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

namespace {

constexpr int NS = 7;     // digits per q value
constexpr int KS = 32;    // K per MMA (kind::i8)
constexpr int KSUB = 4;   // MMAs per ring stage
constexpr int SK = KS * KSUB;  // K (mask columns) per stage
constexpr int NTH = 448;
constexpr int NST = 4;    // ring stages

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
__device__ __forceinline__ uint64_t smem_desc(unsigned addr, unsigned lbo, unsigned sbo) {
  // start >> 4, leading / stride byte offsets >> 4, version 1, SWIZZLE_128B
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// no-swizzle (interleaved core-matrix) descriptor: lbo = stride between core
// matrices along K, sbo = along M
__device__ __forceinline__ uint64_t smem_desc_none(unsigned addr, unsigned lbo, unsigned sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// D s32, A/B signed int8, A K-major, B MN-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
// 4 bits -> 4 bytes of 0/1
__device__ __forceinline__ uint32_t spread4(uint32_t x) { return (x * 0x00204081u) & 0x01010101u; }

}  // namespace

// Q digits of V-hat (n x R): column c of B gets, for p < NA (packed upper
// (i, j), i <= j) and s < NS, the s-th digit of v_ci v_cj at column p*NS+s of
// its half (p*NS+s)/128; unused columns are 0. Bq: hq x n x 128 int8.
template <int R>
__global__ void k_q_digits(const double* __restrict__ V, int64_t n, int64_t nr, int8_t* __restrict__ Bq) {
  // one thread per (column c, packed value p); Bq (hq x nr x 128) is zeroed
  // by the launcher, unused columns stay 0
  constexpr int NA = R * (R + 1) / 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * NA; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / NA;
    const int p = (int)(e % NA);
    int i = 0, rem = p;
    while (rem >= R - i) { rem -= R - i; ++i; }
    const int j = i + rem;
    const unsigned long long d = rsmd::digits_i8<NS>(V[c * R + i] * V[c * R + j]);  // byte b = a[NS-1-b]
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int col = p * NS + s;
      Bq[((int64_t)(col >> 7) * nr + c) * 128 + (col & 127)] = (int8_t)((d >> (8 * (NS - 1 - s))) & 0xFF);
    }
  }
}

template <int R, int HQ>
__global__ void __launch_bounds__(NTH, 1)
    k_normal_i8(const __grid_constant__ CUtensorMap tmB, NormalI8Args a) {
  constexpr int NA = R * (R + 1) / 2;
  constexpr int N = 128 * HQ;
  constexpr int A_STAGE = 128 * SK;       // 128 rows x 128 K-bytes (16 KB)
  constexpr int B_STAGE = SK * 128 * HQ;  // 128 K-rows x N bytes, [HQ][128][128]
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = sm;
  uint8_t* smB = sm + NST * A_STAGE;
  // B resident (every K-stage loaded once) when it fits, else a ring
  const bool res = a.b_resident != 0;
  const int nks = (int)((a.n + SK - 1) / SK);  // K-stages per tile
  uint64_t* full = reinterpret_cast<uint64_t*>(smB + (res ? nks : NST) * B_STAGE);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;  // [2]: two TMEM accumulators, tiles alternate
  uint64_t* tempty = tfull + 2;   // [2]
  uint64_t* bres = tempty + 2;    // the resident B's arrival
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bres + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (a.m + 127) / 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mb_init(full + s, res ? 4 : 5);  // 4 builder warps (+ the B producer's expect_tx when streamed)
      mb_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mb_init(tfull + b, 1);
      mb_init(tempty + b, 4);
    }
    mb_init(bres, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
  }
  if (warp == 12) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)), "r"(2 * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp < 8) {
    // ---------------- A builders: two groups of four warps, alternate stages ----------------
    const int grp = warp >> 2, qtr = warp & 3;
    int64_t gs0 = 0;  // global stage index of the tile's first stage (the ring's order)
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, gs0 += nks) {
      const int64_t row = tile * 128 + 32 * qtr + lane;
      const bool rv = row < a.m;
      // four mask words per stage (one 16-byte load; rows are nwp = 4 nks words)
      const uint4* rw = reinterpret_cast<const uint4*>(a.bits + (rv ? row : 0) * a.nwp);
      int ks = (int)((grp - (gs0 & 1)) & 1);  // this group's first stage of the tile
      uint4 nx = (rv && ks < nks) ? __ldg(rw + ks) : make_uint4(0, 0, 0, 0);
      const int ar = 32 * qtr + lane;
      for (; ks < nks; ks += 2) {
        const uint4 w4 = nx;
        nx = (rv && ks + 2 < nks) ? __ldg(rw + ks + 2) : make_uint4(0, 0, 0, 0);
        const int64_t gs = gs0 + ks;
        const int st = (int)(gs % NST);
        const unsigned ph = (unsigned)((gs / NST) & 1);
        mb_wait(empty + st, ph ^ 1u);
        // K-major, no swizzle: row ar's 128 K-bytes are its 4 words' bits as
        // 0/1 bytes; core matrix (row / 8, 16-byte chunk c) at
        // (row / 8) * 128 + c * 2048, row % 8 inside it
        uint8_t* At = smA + st * A_STAGE + (ar >> 3) * 128 + (ar & 7) * 16;
        const uint32_t wj[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t w = wj[j];
          uint4 c0, c1;
          c0.x = spread4(w & 0xF); c0.y = spread4((w >> 4) & 0xF);
          c0.z = spread4((w >> 8) & 0xF); c0.w = spread4((w >> 12) & 0xF);
          c1.x = spread4((w >> 16) & 0xF); c1.y = spread4((w >> 20) & 0xF);
          c1.z = spread4((w >> 24) & 0xF); c1.w = spread4((w >> 28) & 0xF);
          *reinterpret_cast<uint4*>(At + (2 * j) * 2048) = c0;
          *reinterpret_cast<uint4*>(At + (2 * j + 1) * 2048) = c1;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mb_arrive(full + st);
      }
    }
  } else if (warp < 12) {
    // ---------------- epilogue: TMEM lane quarter warp % 4 -> FP64 ----------------
    const int qtr = warp & 3;
    int64_t it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int64_t row = tile * 128 + 32 * qtr + lane;
      const bool rv = row < a.m;
      const int tb = (int)(it & 1);  // this tile's accumulator
      mb_wait(tfull + tb, (unsigned)((it >> 1) & 1));
      tc_fence_after();
      double A[NA];
#pragma unroll
      for (int p = 0; p < NA; ++p) A[p] = 0.0;
      // column blocks last to first and columns high to low: each value's
      // digits are added smallest first
      constexpr int NCB = (NA * NS + 31) / 32;
#pragma unroll
      for (int cbi = NCB - 1; cbi >= 0; --cbi) {
        const int cb = 32 * cbi;
        int v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(tmem + ((uint32_t)(32 * qtr) << 16) + (uint32_t)(tb * N + cb)));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 31; j >= 0; --j) {
          const int col = cb + j;
          if (col < NA * NS) A[col / NS] = fma((double)v[j], ldexp(1.0, -6 - 8 * (col % NS)), A[col / NS]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(tempty + tb);
      if (rv) {
        double* o = a.Apre + row * NA;
#pragma unroll
        for (int p = 0; p < NA; ++p) o[p] = A[p];
      }
    }
  } else if (warp == 12) {
    // ---------------- MMA issuer: KSUB MMAs (K = 32 each) per stage ----------------
    int st = 0;
    unsigned ph = 0;
    int64_t it = 0;  // this CTA's tile count: accumulator it & 1
    if (res) mb_wait(bres, 0);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int tb = (int)(it & 1);
      // the epilogue drained this accumulator's previous tile (two tiles ago)
      mb_wait(tempty + tb, (unsigned)(((it >> 1) & 1) ^ 1u));
      tc_fence_after();
      for (int ks = 0; ks < nks; ++ks) {
        mb_wait(full + st, ph);
        tc_fence_after();
        if (elect_one()) {
          const unsigned abase = su32(smA + st * A_STAGE);
          const unsigned bbase = su32(smB + (res ? ks : st) * B_STAGE);
#pragma unroll
          for (int i = 0; i < KSUB; ++i) {
            // A: K chunks 2i, 2i+1 (LBO 2048 along K, SBO 128 along M);
            // B: K-rows 32i.. of each 128-column half (LBO 16 KB between
            // halves along N, SBO 1 KB between 8-row atoms)
            const uint64_t ad = smem_desc_none(abase + (unsigned)(2 * i * 2048), 2048, 128);
            const uint64_t bd = smem_desc(bbase + (unsigned)(i * KS * 128), SK * 128, 1024);
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)(tb * N)),
                "l"(ad), "l"(bd), "r"(idesc_n(N)), "r"((ks > 0 || i > 0) ? 1u : 0u)
                : "memory");
          }
          tc_commit(empty + st);
        }
        __syncwarp();
        if (++st == NST) {
          st = 0;
          ph ^= 1u;
        }
      }
      if (elect_one()) tc_commit(tfull + tb);
      __syncwarp();
    }
  } else {
    // ---------------- B producer (TMA): 128 K-rows x HQ halves per load ----------------
    if (lane == 0 && res) {
      mb_expect_tx(bres, (unsigned)(nks * B_STAGE));
      for (int ks = 0; ks < nks; ++ks)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];\n" ::"r"(su32(smB + ks * B_STAGE)),
            "l"(&tmB), "r"(0), "r"(ks * SK), "r"(0), "r"(su32(bres))
            : "memory");
    } else if (lane == 0) {
      int st = 0;
      unsigned ph = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int ks = 0; ks < nks; ++ks) {
          mb_wait(empty + st, ph ^ 1u);
          mb_expect_tx(full + st, (unsigned)B_STAGE);
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
              "%4}], [%5];\n" ::"r"(su32(smB + st * B_STAGE)),
              "l"(&tmB), "r"(0), "r"(ks * SK), "r"(0), "r"(su32(full + st))
              : "memory");
          if (++st == NST) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 12) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * N));
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

template <int R, int HQ>
cudaError_t launch_t(const NormalI8Args& a, int sms, cudaStream_t s) {
  const int nks = (int)((a.n + SK - 1) / SK);
  NormalI8Args b = a;
  const int stream_smem = 1024 + NST * (128 * SK + SK * 128 * HQ) + 256;
  const int res_smem = 1024 + NST * 128 * SK + nks * SK * 128 * HQ + 256;
  b.b_resident = res_smem <= 200 * 1024 ? 1 : 0;
  const int SMEM = b.b_resident ? res_smem : stream_smem;
  auto fn = encode_fn();
  if (!fn) return cudaErrorInvalidValue;
  CUtensorMap mb;
  const int64_t nr = ((a.n + SK - 1) / SK) * SK;  // rows of Bq (padded: zero digits)
  cuuint64_t dims[3] = {128, (cuuint64_t)nr, (cuuint64_t)HQ};
  cuuint64_t strides[2] = {128, (cuuint64_t)(128 * nr)};
  cuuint32_t box[3] = {128, (cuuint32_t)SK, (cuuint32_t)HQ};
  cuuint32_t es[3] = {1, 1, 1};
  if (fn(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(a.Bq), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  ensure_smem((const void*)k_normal_i8<R, HQ>, SMEM);
  const int64_t ntiles = (a.m + 127) / 128;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, sms));
  k_normal_i8<R, HQ><<<grid, NTH, SMEM, s>>>(mb, b);
  return cudaGetLastError();
}

template <int R>
cudaError_t launch_r(const NormalI8Args& a, int sms, cudaStream_t s) {
  constexpr int NA = R * (R + 1) / 2;
  constexpr int HQ = (NA * NS + 127) / 128;
  const int64_t nr = ((a.n + SK - 1) / SK) * SK;
  k_q_digits<R><<<(unsigned)std::min<int64_t>((a.n * NA + 255) / 256, 4096), 256, 0, s>>>(a.V, a.n, nr, a.Bq);
  return launch_t<R, HQ>(a, sms, s);
}

}  // namespace

// bytes of the Q-digit buffer (B operand) for rank r and n basis rows
size_t normal_i8_bq_bytes(int r, int64_t n) {
  const int na = r * (r + 1) / 2;
  const int hq = (na * NS + 127) / 128;
  return (size_t)hq * (size_t)(((n + SK - 1) / SK) * SK) * 128;
}

cudaError_t launch_normal_i8(const NormalI8Args& a, int sms, cudaStream_t s) {
  // Bq's unused columns and the padded rows past n are zero
  const size_t bytes = normal_i8_bq_bytes(a.r, a.n);
  cudaMemsetAsync(a.Bq, 0, bytes, s);
  switch (a.r) {
    case 1: return launch_r<1>(a, sms, s);
    case 2: return launch_r<2>(a, sms, s);
    case 3: return launch_r<3>(a, sms, s);
    case 4: return launch_r<4>(a, sms, s);
    case 5: return launch_r<5>(a, sms, s);
    case 6: return launch_r<6>(a, sms, s);
    case 7: return launch_r<7>(a, sms, s);
    case 8: return launch_r<8>(a, sms, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rsmk
