// Correctness + latency of warp_jacobi_reg<K> on random symmetric matrices:
// residual ||A V - V diag(w)|| and orthogonality ||V^T V - I||.
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include "rsm_dev.cuh"
using namespace rsmd;
template <int K>
__global__ void run(const double* Ain, double* out, long long* cyc, int* sweeps) {
  __shared__ double A[16 * 16], V[16 * 16];
  for (int e = threadIdx.x; e < K * K; e += 32) A[(e / K) * 16 + e % K] = Ain[e];
  __syncwarp();
  long long t0 = clock64();
  int sw = warp_jacobi_reg<K>(A, 16, V, 16, 60);
  long long t1 = clock64();
  for (int e = threadIdx.x; e < K * K; e += 32) { out[e] = V[(e / K) * 16 + e % K]; }
  if (threadIdx.x < K) out[K * K + threadIdx.x] = A[threadIdx.x * 16 + threadIdx.x];
  if (threadIdx.x == 0) { *cyc = t1 - t0; *sweeps = sw; }
}
template <int K>
void test(unsigned seed) {
  double h[K * K];
  srand(seed);
  for (int i = 0; i < K; ++i)
    for (int j = 0; j <= i; ++j) h[i * K + j] = h[j * K + i] = (rand() / (double)RAND_MAX - 0.5) * (i == j ? 10.0 * (i + 1) : 1.0);
  double *dA, *dO; long long* dc; int* ds;
  cudaMalloc(&dA, sizeof(h)); cudaMalloc(&dO, sizeof(double) * (K * K + K)); cudaMalloc(&dc, 8); cudaMalloc(&ds, 4);
  cudaMemcpy(dA, h, sizeof(h), cudaMemcpyHostToDevice);
  run<K><<<1, 32>>>(dA, dO, dc, ds);
  run<K><<<1, 32>>>(dA, dO, dc, ds);
  double o[K * K + K]; long long cyc; int sw;
  cudaMemcpy(o, dO, sizeof(o), cudaMemcpyDeviceToHost); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&sw, ds, 4, cudaMemcpyDeviceToHost);
  double res = 0, orth = 0, nrm = 0;
  for (int i = 0; i < K; ++i) for (int j = 0; j < K; ++j) nrm += h[i * K + j] * h[i * K + j];
  for (int c = 0; c < K; ++c) {
    for (int i = 0; i < K; ++i) {
      double s = 0; for (int k = 0; k < K; ++k) s += h[i * K + k] * o[k * K + c];
      res = fmax(res, fabs(s - o[K * K + c] * o[i * K + c]));
    }
    for (int d = 0; d < K; ++d) { double s = 0; for (int i = 0; i < K; ++i) s += o[i * K + c] * o[i * K + d]; orth = fmax(orth, fabs(s - (c == d))); }
  }
  printf("K=%2d cycles %7lld sweeps %d  residual %.2e (|A| %.1f)  orth %.2e  %s\n", K, cyc, sw, res, sqrt(nrm), orth, cudaGetErrorString(cudaGetLastError()));
}
int main() { test<3>(1); test<5>(2); test<9>(3); test<10>(4); test<11>(5); test<16>(6); return 0; }
