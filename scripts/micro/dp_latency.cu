// Dependent-chain latencies on B200 (one warp): DFMA, DADD, DMUL, the
// float-seeded Newton rsqrt used by the small dense solvers, F2F conversions,
// shared-memory load-to-use, __syncthreads at 256 threads.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dp_latency dp_latency.cu
#include <cstdio>

__device__ __forceinline__ double rsqrt_fast(double v) {
#ifdef SEED_F32
  double r = (double)rsqrtf((float)v);
#else
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(v));
#endif
  const double hv = 0.5 * v;
  r = r * fma(-hv * r, r, 1.5);
  r = r * fma(-hv * r, r, 1.5);
  return r;
}

__global__ void k(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[64];
  double x = x0, y = 1.0 + 1e-9 * threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt_fast(fabs(x) + 1.0);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = (double)((float)x * 1.0001f);
  long long t5 = clock64();
  sm[threadIdx.x & 63] = x;
  __syncwarp();
  int idx = threadIdx.x & 63;
  for (int i = 0; i < n; ++i) idx = (int)sm[idx] & 63;
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t7 = clock64();
  float f = (float)x;
  for (int i = 0; i < n; ++i) f = fmaf(f, 1.0001f, 1e-30f);
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    cyc[6] = t7 - t6; cyc[7] = t8 - t7;
  }
  out[threadIdx.x] = x + idx + f;
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 8 * 256); cudaMalloc(&c, 64);
  const int n = 4096;
  const char* names[] = {"DFMA", "DADD", "DMUL", "rsqrt_fast", "F2F round trip + FMUL", "LDS.64 + F2I chain", "__syncthreads", "FFMA"};
  for (int threads : {32, 256}) {
    k<<<1, threads>>>(d, c, 1.0, n);
    cudaDeviceSynchronize();
    k<<<1, threads>>>(d, c, 1.0, n);
    long long h[8];
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i) printf("threads %3d  %-24s %.1f cycles per dependent op\n", threads, names[i], (double)h[i] / n);
  }
  return 0;
}
