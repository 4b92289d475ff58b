// Grid-barrier latency on B200: cooperative-groups grid.sync() against a
// flag barrier (one arrival counter per phase, lead thread spins on an
// acquire load), for the stage-4 kernel's grid of 128 CTAs x 256 threads.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o barrier_bench barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// monotone counter: barrier k completes when the counter reaches k * gridDim.x
__global__ void k_flag(int iters, unsigned* ctr, long long* out) {
  const long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
      const unsigned target = (unsigned)i * gridDim.x;
      while (ld_acquire(ctr) < target) {
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
  long long* d;
  unsigned* ctr;
  cudaMalloc(&d, 8);
  cudaMalloc(&ctr, 4);
  const int iters = 1000;
  for (int grid : {64, 128, 148}) {
    void* args[] = {(void*)&iters, (void*)&d};
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaLaunchCooperativeKernel((void*)k_cg, dim3(grid), dim3(256), args, 0, 0);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    }
    printf("grid %d cg::grid.sync   %.0f cycles\n", grid, (double)h / iters);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 4);
      void* a2[] = {(void*)&iters, (void*)&ctr, (void*)&d};
      cudaLaunchCooperativeKernel((void*)k_flag, dim3(grid), dim3(256), a2, 0, 0);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    }
    printf("grid %d flag barrier     %.0f cycles (%s)\n", grid, (double)h / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
