// Does a predicated-off DFMA cost DFMA-pipe time or only an issue slot?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, unsigned pat, int iters) {
  double acc[16];
  const double a = out[0], b = out[1];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = out[2 + j];
  unsigned m = pat;
  for (int i = 0; i < iters; ++i) {
    m = (m << 1) | (m >> 31);  // rotate: a warp-uniform 1-in-3-ish pattern
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (MODE == 0) {
        acc[j] = fma(a, acc[j], b);
      } else {
        // predicated: the asm forces a predicated DFMA (no branch)
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p fma.rn.f64 %0, %0, %1, %3;\n}\n"
            : "+d"(acc[j])
            : "d"(a), "r"(m & (1u << j)), "d"(b));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  if (s == 1234.5) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 4096);
  double h[32];
  for (int i = 0; i < 32; ++i) h[i] = 0.999;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  unsigned pats[3] = {0xffffffffu, 0x49249249u, 0x0u};
  const char* names[3] = {"all on", "1 in 3 on", "all off"};
  for (int mode = 0; mode < 2; ++mode)
    for (int p = 0; p < (mode ? 3 : 1); ++p) {
      auto run = [&]() {
        if (mode == 0) k<0><<<148 * 4, 256>>>(d, pats[p], iters);
        else k<1><<<148 * 4, 256>>>(d, pats[p], iters);
      };
      run();
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s %-10s %.3f ms\n", mode ? "predicated" : "plain     ", mode ? names[p] : "", ms);
    }
  return 0;
}
