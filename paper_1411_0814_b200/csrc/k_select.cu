// k_select.cu -- stage 1: trial selection, bit-exact with the reference.
//
// Every attempt a draws `block` distinct sorted indices with the counter
// stream Rng(seed, TRIAL=5, a) (sampler.hpp:32-37, rng.hpp:14-36) by the
// partial Fisher-Yates of sampler.cpp:12-23 (the identity permutation is kept
// virtual: a position->value map of the <= 2*block touched slots), then
// counts survivors: AND of the drawn rows' mask words and popc for the row
// branch (sample_m2, sampler.cpp:58-87), or AND of the drawn columns'
// column-major words for the column branch (sample_m1, sampler.cpp:27-56).
// The attempt-order prefix of the first T accepted attempts (consumption
// order and 20x budget of harvest.cpp:79-120) is then compacted with a
// deterministic block scan.
#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

using namespace rsmd;

// One warp handles 32 consecutive attempts: each lane draws the index set of
// one attempt (draws are per-attempt serial integer work), then the warp
// scans the mask words of each of the 32 attempts cooperatively (coalesced
// 128-byte row segments).
__global__ void __launch_bounds__(256) k_select(const uint32_t* __restrict__ bits, int64_t stride,
                                                int64_t nwords, int64_t pool, int block,
                                                uint64_t seed, uint64_t a0, int64_t count,
                                                int32_t* __restrict__ idx_out,
                                                int32_t* __restrict__ q_out, int apw) {
  extern __shared__ int32_t sidx[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int64_t base = ((int64_t)blockIdx.x * warps + warp) * apw;
  int32_t* my = sidx + (size_t)warp * apw * block;
  const int64_t a = base + lane;
  if (lane < apw && a < count) {
    int32_t* out = my + lane * block;
    draw_sorted(seed, a0 + (uint64_t)a, pool, block, out);
    for (int t = 0; t < block; ++t) idx_out[a * block + t] = out[t];
  }
  __syncwarp();
  if (nwords <= 64 && (stride & 3) == 0 && apw == 32) {
    // short scans (row branch, n <= 2048): each lane ANDs its own attempt's
    // rows with 16-byte loads, all of them in flight at once (the words past
    // n up to the stride are zero padding)
    if (lane < apw && a < count) {
      const int32_t* rows = my + lane * block;
      uint4 acc[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) acc[u] = make_uint4(~0u, ~0u, ~0u, ~0u);
      for (int t = 0; t < block; ++t) {
        const uint4* rb = reinterpret_cast<const uint4*>(bits + (int64_t)rows[t] * stride);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          if (4 * u < nwords) {
            const uint4 x = __ldg(rb + u);
            acc[u].x &= x.x;
            acc[u].y &= x.y;
            acc[u].z &= x.z;
            acc[u].w &= x.w;
          }
        }
      }
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (4 * u < nwords) cnt += __popc(acc[u].x) + __popc(acc[u].y) + __popc(acc[u].z) + __popc(acc[u].w);
      q_out[a] = cnt;
    }
    return;
  }
  for (int i = 0; i < apw; ++i) {
    const int64_t ai = base + i;
    if (ai >= count) break;
    const int32_t* rows = my + i * block;
    int cnt = 0;
    for (int64_t w = lane; w < nwords; w += 32) {
      uint32_t acc = 0xffffffffu;
      for (int t = 0; t < block; ++t) acc &= __ldg(bits + (int64_t)rows[t] * stride + w);
      cnt += __popc(acc);
    }
    cnt = warp_sum_int(cnt);
    if (lane == 0) q_out[ai] = cnt;
  }
}

__global__ void k_acc_count(const int32_t* __restrict__ q, int64_t count, int32_t min_count,
                            int32_t* __restrict__ blockcnt) {
  __shared__ int ws[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = (i < count && q[i] >= min_count) ? 1 : 0;
  const int c = __popc(__ballot_sync(0xffffffffu, f));
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += ws[w];
    blockcnt[blockIdx.x] = s;
  }
}

// single block: exclusive scan of the per-block accepted counts and update
// of the running accepted total (capped at T)
__global__ void k_acc_scan(int32_t* __restrict__ blockcnt, int64_t nb, SelState* st,
                           uint64_t T) {
  __shared__ long long wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t per = (nb + blockDim.x - 1) / blockDim.x;
  const int64_t lo = tid * per, hi = (lo + per < nb) ? lo + per : nb;
  long long own = 0;
  for (int64_t b = lo; b < hi; ++b) own += blockcnt[b];
  // block-wide inclusive scan of the per-thread sums (warp scans + a scan of
  // the warp totals)
  long long inc = own;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    long long w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  inc += warp > 0 ? wsum[warp - 1] : 0;
  long long run = inc - own;  // exclusive prefix of this thread's range
  if (tid == (int)blockDim.x - 1) {
    const unsigned long long before = st->acc;
    st->acc_before = before;
    const unsigned long long tot = before + (unsigned long long)inc;
    st->acc = tot < T ? tot : T;
  }
  for (int64_t b = lo; b < hi; ++b) {
    const long long v = blockcnt[b];
    blockcnt[b] = (int32_t)run;  // exclusive offset within the chunk
    run += v;
  }
}

__global__ void k_acc_emit(const int32_t* __restrict__ q, const int32_t* __restrict__ idx,
                           int64_t count, int32_t min_count, int block, uint64_t a0,
                           const int32_t* __restrict__ blockoff, SelState* st, uint64_t T,
                           uint64_t* __restrict__ t_attempt, int32_t* __restrict__ t_q,
                           int32_t* __restrict__ t_idx) {
  __shared__ int ws[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = (i < count && q[i] >= min_count) ? 1 : 0;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) ws[warp] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      const int v = ws[w];
      ws[w] = s;
      s += v;
    }
  }
  __syncthreads();
  const unsigned long long pos = st->acc_before + (unsigned long long)blockoff[blockIdx.x] +
                                 (unsigned long long)(ws[warp] + __popc(bal & ((1u << lane) - 1u)));
  // survivor-count sum of the accepted trials that enter the first T: one
  // 64-bit atomic per warp (integer sums: the order does not matter)
  const unsigned qc = (f && pos < T) ? (unsigned)q[i] : 0u;
  const unsigned qw = __reduce_add_sync(0xffffffffu, qc);
  const unsigned qm = __reduce_max_sync(0xffffffffu, qc);
  if (lane == 0 && qw) {
    atomicAdd(&st->qsum, (unsigned long long)qw);
    atomicMax(&st->qmax, (int)qm);
  }
  if (!f) return;
  if (pos >= T) return;
  t_attempt[pos] = a0 + (uint64_t)i;
  const int32_t qi = q[i];
  t_q[pos] = qi;
  for (int t = 0; t < block; ++t) t_idx[pos * block + t] = idx[i * block + t];
  if (pos == T - 1) st->attempted_done = a0 + (uint64_t)i + 1;
}

void launch_select(const uint32_t* bits, int64_t stride, int64_t nwords, int64_t pool, int block,
                   uint64_t seed, uint64_t a0, int64_t count, int32_t* idx_out, int32_t* q_out,
                   cudaStream_t s) {
  // attempts per warp: 32 (one draw per lane) when an attempt's scan is a
  // few words; 4 when it is long (the column branch scans m/32 words per drawn
  // column), so that enough warps share the scans
  const int apw = nwords > 64 ? 4 : 32;
  const int threads = 256, warps = threads / 32;
  const int64_t per_block = (int64_t)warps * apw;
  const int64_t blocks = (count + per_block - 1) / per_block;
  const size_t smem = (size_t)warps * apw * block * sizeof(int32_t);
  k_select<<<(unsigned)blocks, threads, smem, s>>>(bits, stride, nwords, pool, block, seed, a0,
                                                   count, idx_out, q_out, apw);
}

void launch_accept(const int32_t* q, const int32_t* idx, int64_t count, int32_t min_count,
                   int block, uint64_t a0, int32_t* blockcnt, SelState* st, uint64_t T,
                   uint64_t* t_attempt, int32_t* t_q, int32_t* t_idx, cudaStream_t s) {
  const int threads = 1024;
  const int64_t nb = (count + threads - 1) / threads;
  k_acc_count<<<(unsigned)nb, threads, 0, s>>>(q, count, min_count, blockcnt);
  k_acc_scan<<<1, 1024, 0, s>>>(blockcnt, nb, st, T);
  k_acc_emit<<<(unsigned)nb, threads, 0, s>>>(q, idx, count, min_count, block, a0, blockcnt, st,
                                              T, t_attempt, t_q, t_idx);
}

}  // namespace rsmk
