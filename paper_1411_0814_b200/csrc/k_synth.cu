// k_synth.cu -- device-side synthetic generator: the
// reference's Eq. 31 instance (src/synth.cpp:12-57, paths relative to
// /root/reference/proj) generated straight into the context's HBM layout
// (FP64 Y with NaN at hidden cells + the bit-packed row mask), for
// large-scale throughput runs without a host generator or a 16 GiB upload.
//
// The counter-based splitmix64 stream Rng(seed, tag, index) (rng.hpp:12-57)
// is random-access: its d-th draw (1-based) is mix(s0 + d*gamma), so every
// cell is generated independently. Stream use matches the host generator
// (synth.cpp here): A row i from Rng(seed, 1, i) (draws 2k+1, 2k+2 for factor
// k), B row k from Rng(seed, 2, k) (draws 2j+1, 2j+2 for column j), noise of
// cell (i, j) from Rng(seed, 3, i) draws 2j+1, 2j+2, mask from Rng(seed, 4, i)
// draw j+1 compared with rho. The product A*B is summed in k order with
// separately rounded multiplies and adds, as the host code. The mask is
// therefore bit-exact; values match the host to the last few ulps only,
// because Box-Muller's log/cos come from the device math library instead of
// glibc (the parity tests state that tolerance).
#include "rsm_internal.h"
#include "rsm_dev.cuh"

namespace rsmk {

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ uint64_t stream0(uint64_t seed, uint64_t tag, uint64_t index) {
  return rsmd::rng_state(seed, tag, index);
}
// d-th draw (1-based) of the stream whose constructor state is s0
__device__ __forceinline__ uint64_t draw(uint64_t s0, uint64_t d) { return rsmd::mix(s0 + d * kGamma); }
__device__ __forceinline__ double unit(uint64_t x) { return ((double)(x >> 11) + 0.5) * 0x1.0p-53; }
// normal from draws d, d+1 (Rng::next_normal)
__device__ __forceinline__ double normal(uint64_t s0, uint64_t d) {
  const double u1 = unit(draw(s0, d));
  const double u2 = unit(draw(s0, d + 1));
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586476925286766559, u2)));
}

}  // namespace

// B (r x n): thread per element
__global__ void k_gen_factor_b(int64_t r, int64_t n, uint64_t seed, double* __restrict__ B) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= r * n) return;
  const int64_t k = e / n, j = e % n;
  B[e] = normal(stream0(seed, 2, (uint64_t)k), 2 * (uint64_t)j + 1);
}

// warp per row: values (NaN where hidden) and the row's mask words (nwp per
// row, zero past n)
__global__ void k_gen_rows(int64_t m, int64_t n, int64_t r, double rho, double sigma, uint64_t seed,
                           const double* __restrict__ B, int64_t nwp, double* __restrict__ Y,
                           uint32_t* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < m; i += nw) {
    // factor row: lane k < r draws a_k
    const uint64_t sa = stream0(seed, 1, (uint64_t)i);
    const double mine = lane < r ? normal(sa, 2 * (uint64_t)lane + 1) : 0.0;
    const uint64_t sn = stream0(seed, 3, (uint64_t)i);
    const uint64_t sm = stream0(seed, 4, (uint64_t)i);
    double* y = Y + i * n;
    uint32_t* w = bits + i * nwp;
    for (int64_t j0 = 0; j0 < nwp * 32; j0 += 32) {
      const int64_t j = j0 + lane;
      bool known = false;
      if (j < n) {
        double s = 0.0;
        for (int64_t k = 0; k < r; ++k)
          s = __dadd_rn(s, __dmul_rn(__shfl_sync(0xffffffffu, mine, (int)k), B[k * n + j]));
        if (sigma > 0.0) s = __dadd_rn(s, __dmul_rn(sigma, normal(sn, 2 * (uint64_t)j + 1)));
        known = unit(draw(sm, (uint64_t)j + 1)) <= rho;
        y[j] = known ? s : __longlong_as_double(0x7ff8000000000000ll);
      } else {
        // keep the shuffles of the factor row converged across the warp
        for (int64_t k = 0; k < r; ++k) (void)__shfl_sync(0xffffffffu, mine, (int)k);
      }
      const unsigned word = __ballot_sync(0xffffffffu, known);
      if (lane == 0) w[j0 >> 5] = word;
    }
  }
}

void launch_generate(int64_t m, int64_t n, int64_t r, double rho, double sigma, uint64_t seed, double* B,
                     int64_t nwp, double* Y, uint32_t* bits, int sms, cudaStream_t s) {
  const int64_t nb = r * n;
  k_gen_factor_b<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(r, n, seed, B);
  int64_t blocks = (m + 7) / 8;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  k_gen_rows<<<(unsigned)blocks, 256, 0, s>>>(m, n, r, rho, sigma, seed, B, nwp, Y, bits);
}

}  // namespace rsmk
