// FP64 microbenchmarks on sm_100a: dependent DFMA latency, DFMA and DMMA
// (mma.sync m8n8k4 f64) throughput. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, int iters) {
  double a = out[0], b = out[1], c = out[2];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c = fma(a, c, b);
  }
  long long t1 = clock64();
  out[3 + threadIdx.x] = c;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int CH>
__global__ void dfma_tp(double* out, int iters) {
  double acc[CH];
  const double a = out[0], b = out[1];
#pragma unroll
  for (int k = 0; k < CH; ++k) acc[k] = out[2 + k];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k) acc[k] = fma(a, acc[k], b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += acc[k];
  if (s == 12345.0) out[0] = s;
}

template <int CH>
__global__ void dmma_tp(double* out, int iters) {
  double a = out[threadIdx.x & 31], b = out[(threadIdx.x + 1) & 31];
  double c[CH][2];
#pragma unroll
  for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}


// half the warps issue DFMA chains, half issue DMMA chains: does the SM run
// the two FP64 paths concurrently?
template <int CH>
__global__ void mixed_tp(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  if (warp & 1) {
    double a = out[threadIdx.x & 31], b = out[(threadIdx.x + 1) & 31];
    double c[CH][2];
#pragma unroll
    for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < CH; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1])
                     : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.0) out[0] = s;
  } else {
    double acc[16];
    const double a = out[0], b = out[1];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = out[2 + k];
    for (int i = 0; i < iters * 2; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fma(a, acc[k], b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += acc[k];
    if (s == 12345.0) out[0] = s;
  }
}

int main() {
  double* d;
  long long* cyc;
  cudaMalloc(&d, 4096 * 8);
  cudaMalloc(&cyc, 8);
  double h[64];
  for (int i = 0; i < 64; ++i) h[i] = 0.999 + 1e-6 * i;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  lat<<<1, 32>>>(d, cyc, 1000);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(d, cyc, 1000);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DFMA latency: %.2f cycles\n", c / 16000.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int threads, double fl_per_thread_iter, int iters) {
    kern<<<sms * 4, threads>>>(d, iters);
    cudaEventRecord(e0);
    kern<<<sms * 4, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = fl_per_thread_iter * threads * (double)sms * 4 * iters;
    printf("%-28s %8.2f TFLOP/s  (%s)\n", name, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run("DFMA 8 chains x 256 thr", dfma_tp<8>, 256, 16, 20000);
  run("DFMA 16 chains x 256 thr", dfma_tp<16>, 256, 32, 10000);
  run("DFMA 4 chains x 128 thr", dfma_tp<4>, 128, 8, 40000);
  run("DMMA 4 chains x 256 thr", dmma_tp<4>, 256, 4 * 512.0 / 32, 5000);
  run("DMMA 8 chains x 256 thr", dmma_tp<8>, 256, 8 * 512.0 / 32, 2500);
  run("DMMA 2 chains x 128 thr", dmma_tp<2>, 128, 2 * 512.0 / 32, 10000);
  // mixed: per DMMA warp-iteration 4*512/32 flops per thread; per DFMA warp-iteration 16*16*2 flops per thread
  {
    const int iters = 20000, threads = 256;
    mixed_tp<4><<<sms * 4, threads>>>(d, iters);
    cudaEventRecord(e0);
    mixed_tp<4><<<sms * 4, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl_dmma = 4 * 512.0 / 32 * (threads / 2) * (double)sms * 4 * iters;
    const double fl_dfma = 2 * 16 * 2.0 * (threads / 2) * (double)sms * 4 * iters;
    printf("mixed DMMA+DFMA warps: %.2f TFLOP/s total (%.2f ms; DMMA share of flops %.2f)\n",
           (fl_dmma + fl_dfma) / ms / 1e9, ms, fl_dmma / (fl_dmma + fl_dfma));
  }
  return 0;
}
