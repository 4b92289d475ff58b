// Latency microbenchmark of the stage-4 small dense kernels on one warp:
// chol_small-style shuffle Cholesky (11 x 11) and warp_jacobi_reg<10>.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1411_0814_b200/csrc scripts/micro/small_bench.cu
#include <cstdio>
#include <cstdint>
#include "rsm_dev.cuh"
using namespace rsmd;

constexpr int BMAX = 16;

__device__ __noinline__ void chol_v1(const double* red, int nc, double* S, double* dinv) {
  const int lane = threadIdx.x;
  double a[BMAX];
#pragma unroll
  for (int j = 0; j < BMAX; ++j) {
    double v = 0.0;
    if (lane < nc && j < nc) {
      const int i0 = lane < j ? lane : j, j0 = lane < j ? j : lane;
      v = red[i0 * nc - i0 * (i0 - 1) / 2 + (j0 - i0)];
    }
    a[j] = v;
  }
#pragma unroll
  for (int k = 0; k < BMAX; ++k) {
    if (k < nc) {
      const double d = __shfl_sync(0xffffffffu, a[k], k);
      const double inv = d > 0.0 ? rsqrt_fast(d) : 0.0;
      const double l = d > 0.0 ? d * inv : 0.0;
      if (lane == k) a[k] = l;
      if (lane > k) a[k] *= inv;
#pragma unroll
      for (int j = k + 1; j < BMAX; ++j) {
        const double ljk = __shfl_sync(0xffffffffu, a[k], j);
        if (j < nc && j <= lane) a[j] = fma(-a[k], ljk, a[j]);
      }
    }
  }
  if (lane < nc) {
    double dg = 1.0;
#pragma unroll
    for (int j = 0; j < BMAX; ++j) {
      if (j <= lane) S[lane * BMAX + j] = a[j];
      if (j == lane) dg = a[j];
    }
    dinv[lane] = 1.0 / dg;
  }
  __syncwarp();
}

// rolled, in shared memory (k_eig.cu chol_small since round 2)
__device__ __noinline__ void chol_v2(const double* red, int nc, double* L, double* dinv) {
  const int lane = threadIdx.x;
#pragma unroll 1
  for (int e = lane; e < nc * nc; e += 32) {
    const int i = e / nc, j = e - i * nc;
    if (j <= i) L[i * BMAX + j] = red[j * nc - j * (j - 1) / 2 + (i - j)];
  }
  __syncwarp();
#pragma unroll 1
  for (int k = 0; k < nc; ++k) {
    const double d = L[k * BMAX + k];
    const double inv = d > 0.0 ? rsqrt_fast(d) : 0.0;
    __syncwarp();
    if (lane == 0) L[k * BMAX + k] = d > 0.0 ? d * inv : 0.0;
    if (k + 1 + lane < nc) L[(k + 1 + lane) * BMAX + k] *= inv;
    __syncwarp();
    const int m = nc - k - 1;
#pragma unroll 1
    for (int e = lane; e < m * m; e += 32) {
      const int ii = e / m, jj = e - ii * m;
      if (jj <= ii) {
        const int i = k + 1 + ii, j = k + 1 + jj;
        L[i * BMAX + j] = fma(-L[i * BMAX + k], L[j * BMAX + k], L[i * BMAX + j]);
      }
    }
    __syncwarp();
  }
  if (lane < nc) dinv[lane] = 1.0 / L[lane * BMAX + lane];
  __syncwarp();
}

__global__ void bench2(double* out, long long* cyc) {
  __shared__ double red[200], S[BMAX * BMAX], dinv[BMAX];
  const int lane = threadIdx.x;
  const int nc = 10;
  for (int p = lane; p < nc * (nc + 1) / 2; p += 32) red[p] = 0.01 * ((p * 37) % 11);
  if (lane < nc) red[lane * nc - lane * (lane - 1) / 2] = nc + lane;
  __syncwarp();
  long long t0 = clock64();
  chol_v1(red, nc, S, dinv);
  long long t1 = clock64();
  chol_v1(red, nc, S, dinv);
  long long t2 = clock64();
  chol_v2(red, nc, S, dinv);
  long long t3 = clock64();
  chol_v2(red, nc, S, dinv);
  long long t4 = clock64();
  if (lane == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
    out[0] = S[5 * BMAX + 3] + dinv[2];
  }
}

__global__ void bench(double* out, long long* cyc) {
  __shared__ double red[200], S[BMAX * BMAX], dinv[BMAX], H[BMAX * BMAX], V[BMAX * BMAX];
  const int lane = threadIdx.x;
  const int nc = 11;
  // SPD: A = I*nc + small symmetric
  for (int p = lane; p < nc * (nc + 1) / 2; p += 32) red[p] = 0.01 * ((p * 37) % 11) ;
  if (lane < nc) red[lane * nc - lane * (lane - 1) / 2] = nc + lane;
  for (int e = lane; e < 10 * 10; e += 32) {
    const int i = e / 10, j = e % 10;
    H[i * BMAX + j] = (i == j) ? 1.0 + i : 0.001 * ((i * 7 + j * 7) % 13);
  }
  __syncwarp();
  long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) chol_v1(red, nc, S, dinv);
  long long t1 = clock64();
  int sw = warp_jacobi_reg<10>(H, BMAX, V, BMAX, 40);
  long long t2 = clock64();
  if (lane == 0) {
    cyc[0] = (t1 - t0) / 10;
    cyc[1] = t2 - t1;
    cyc[2] = sw;
    out[0] = S[5 * BMAX + 3] + H[0];
  }
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  bench<<<1, 32>>>(o, c);
  bench<<<1, 32>>>(o, c);
  long long h[3];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("chol_small(11): %lld cycles; jacobi_reg<10>: %lld cycles, %lld sweeps (%s)\n", h[0], h[1], h[2],
         cudaGetErrorString(cudaGetLastError()));
  long long h2[4];
  bench2<<<1, 32>>>(o, c);
  cudaMemcpy(h2, c, sizeof(h2), cudaMemcpyDeviceToHost);
  printf("chol(10) unrolled/shuffle: first %lld, second %lld; rolled/smem: first %lld, second %lld cycles\n", h2[0],
         h2[1], h2[2], h2[3]);
  return 0;
}
