// k_prep.cu -- input layout kernels: bit-pack the uint8 observation mask
// (rsm::MaskedMatrix::mask, include/rsm/core.hpp:26 of the reference) into
// row-major words (m x nwp, bit j%32 of word j/32) and column-major words
// (n x mwp) for the column branch, the device transpose used when m < n
// (rsm::MaskedMatrix::transposed, core.hpp:50-56 / solver.cpp:130-140), and
// the observed-cell count (core.hpp:44-48).
#include <map>
#include <mutex>
#include <tuple>

#include "rsm_internal.h"

namespace rsmk {

// one thread per output word; each thread reads 32 consecutive mask bytes
__global__ void k_pack_rows(const uint8_t* __restrict__ mask, int64_t m, int64_t n,
                            uint32_t* __restrict__ bits, int64_t nwp) {
  const int64_t total = m * nwp;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / nwp, w = t % nwp;
    const int64_t j0 = w * 32;
    uint32_t word = 0;
    if (j0 < n) {
      const uint8_t* src = mask + i * n + j0;
      const int64_t cnt = (n - j0) < 32 ? (n - j0) : 32;
      for (int b = 0; b < cnt; ++b) word |= (src[b] ? 1u : 0u) << b;
    }
    bits[t] = word;
  }
}

// inverse of k_pack_rows (the byte mask is rebuilt on demand when the host
// delivered packed words): one thread per byte
__global__ void k_unpack_rows(const uint32_t* __restrict__ bits, int64_t m, int64_t n, int64_t nwp,
                              uint8_t* __restrict__ mask) {
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t % n;
    mask[t] = (uint8_t)((bits[i * nwp + (j >> 5)] >> (j & 31)) & 1u);
  }
}

// column-major: word (j, w) holds rows 32w..32w+31 of column j. Consecutive
// threads take consecutive columns so each byte load instruction is one
// contiguous 32-byte segment of a mask row.
__global__ void k_pack_cols(const uint8_t* __restrict__ mask, int64_t m, int64_t n,
                            uint32_t* __restrict__ bits, int64_t mwp) {
  const int64_t total = n * mwp;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = t / n, j = t % n;
    const int64_t i0 = w * 32;
    uint32_t word = 0;
    if (i0 < m) {
      const int64_t cnt = (m - i0) < 32 ? (m - i0) : 32;
      for (int b = 0; b < cnt; ++b) word |= (mask[(i0 + b) * n + j] ? 1u : 0u) << b;
    }
    bits[j * mwp + w] = word;
  }
}

// 32x32 tiled transpose of values and mask: out (n x m) = in (m x n)^T,
// hidden cells become NaN (core.hpp:50-56 sets only known cells).
__global__ void k_transpose(const double* __restrict__ Y, const uint8_t* __restrict__ M,
                            int64_t m, int64_t n, double* __restrict__ Yt,
                            uint8_t* __restrict__ Mt) {
  __shared__ double ty[32][33];
  __shared__ uint8_t tm[32][33];
  const int64_t bi = blockIdx.y * 32, bj = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = bi + r, j = bj + threadIdx.x;
    if (i < m && j < n) {
      ty[r][threadIdx.x] = Y[i * n + j];
      tm[r][threadIdx.x] = M[i * n + j];
    }
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = bj + r, i = bi + threadIdx.x;
    if (i < m && j < n) {
      const uint8_t k = tm[threadIdx.x][r];
      Mt[j * m + i] = k;
      Yt[j * m + i] = k ? ty[threadIdx.x][r] : __longlong_as_double(0x7ff8000000000000ll);
    }
  }
}

__global__ void k_count_bits(const uint32_t* __restrict__ bits, int64_t nwords,
                             unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nwords;
       t += (int64_t)gridDim.x * blockDim.x)
    c += __popc(bits[t]);
  c = __reduce_add_sync(0xffffffffu, (unsigned)c);  // per-warp partial fits in 32 bits
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);   // integer: order-independent
}

void launch_unpack_rows(const uint32_t* bits, int64_t m, int64_t n, int64_t nwp, uint8_t* mask,
                        cudaStream_t s) {
  int64_t blocks = (m * n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_unpack_rows<<<(unsigned)blocks, 256, 0, s>>>(bits, m, n, nwp, mask);
}

void launch_pack_rows(const uint8_t* mask, int64_t m, int64_t n, uint32_t* bits, int64_t nwp,
                      cudaStream_t s) {
  const int64_t total = m * nwp;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_pack_rows<<<(unsigned)blocks, threads, 0, s>>>(mask, m, n, bits, nwp);
}

void launch_pack_cols(const uint8_t* mask, int64_t m, int64_t n, uint32_t* bits, int64_t mwp,
                      cudaStream_t s) {
  const int64_t total = n * mwp;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_pack_cols<<<(unsigned)blocks, threads, 0, s>>>(mask, m, n, bits, mwp);
}

void launch_transpose(const double* Y, const uint8_t* M, int64_t m, int64_t n, double* Yt,
                      uint8_t* Mt, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
  k_transpose<<<grid, block, 0, s>>>(Y, M, m, n, Yt, Mt);
}

void launch_count_bits(const uint32_t* bits, int64_t nwords, unsigned long long* out,
                       cudaStream_t s) {
  int64_t blocks = (nwords + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_count_bits<<<(unsigned)blocks, 256, 0, s>>>(bits, nwords, out);
}

// ---- memoised launch configuration (rsm_internal.h) ----
namespace {
std::mutex g_cfg_mu;
std::map<std::pair<int, const void*>, size_t> g_smem_set;
std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;
}  // namespace

void ensure_smem(const void* fn, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  size_t& cur = g_smem_set[{dev, fn}];
  if (smem <= cur && cur != 0) return;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess) cur = smem;
}

int occupancy(const void* fn, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    auto it = g_occ.find({dev, fn, threads, smem});
    if (it != g_occ.end()) return it->second;
  }
  ensure_smem(fn, smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem);
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  g_occ[{dev, fn, threads, smem}] = nb;
  return nb;
}

}  // namespace rsmk
