// Probe: GPU-initiated (zero-copy) gather of random 8 KB rows from pinned host
// memory vs cudaMemcpyAsync of the whole matrix. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void gather_rows(const double* __restrict__ host, const int* __restrict__ rows, int nr, int n,
                            double* __restrict__ dev) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = gw; k < nr; k += nw) {
    const int64_t r = rows[k];
    const double2* src = reinterpret_cast<const double2*>(host + r * n);
    double2* dst = reinterpret_cast<double2*>(dev + r * n);
    for (int c = lane; c < n / 2; c += 32) dst[c] = src[c];
  }
}

int main() {
  const int m = 131072, n = 1024;
  const size_t bytes = (size_t)m * n * 8;
  double* h;
  cudaHostAlloc((void**)&h, bytes, cudaHostAllocDefault);
  for (size_t i = 0; i < (size_t)m * n; i += 512) h[i] = 1.0;
  double* d;
  cudaMalloc(&d, bytes);
  std::vector<int> rows(m);
  for (int i = 0; i < m; ++i) rows[i] = i;
  std::mt19937 g(1);
  std::shuffle(rows.begin(), rows.end(), g);
  const int nr = m * 46 / 100;
  std::sort(rows.begin(), rows.begin() + nr);
  int* drows;
  cudaMalloc(&drows, sizeof(int) * nr);
  cudaMemcpy(drows, rows.data(), sizeof(int) * nr, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("memcpy H2D %.1f MB: %.2f ms = %.1f GB/s\n", bytes / 1e6, ms, bytes / ms / 1e6);
  }
  for (int blocks : {148, 296, 592, 1184}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      gather_rows<<<blocks, 256>>>(h, drows, nr, n, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    const double gb = (double)nr * n * 8;
    printf("zero-copy gather %d rows (%.0f MB), %d blocks: %.2f ms = %.1f GB/s (%s)\n", nr, gb / 1e6, blocks, ms,
           gb / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
