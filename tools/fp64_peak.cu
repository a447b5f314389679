// FP64 pipe microbenchmark for B200 (sm_100a): DFMA throughput with 8
// independent chains per thread, DFMA dependent-chain latency, and the
// throughput of IEEE division / square root (the operations the Riemann
// solvers are built from).  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_lat(double* out, double a, double b, int iters, long long* cyc) {
  double x = threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

__global__ void k_div(double* out, double b, int iters) {
  double x[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = 1.0 + threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = b / x[k] + 1.0;
  }
  double s = x[0] + x[1] + x[2] + x[3];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_sqrt(double* out, int iters) {
  double x[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = 2.0 + threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = sqrt(x[k]) + 1.5;
  }
  double s = x[0] + x[1] + x[2] + x[3];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float ms;
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
  };
  float t_fma = timeit([&] { k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7, iters); });
  double flops = 2.0 * 8 * iters * (double)blocks * threads;
  float t_div = timeit([&] { k_div<<<blocks, threads>>>(out, 0.5, iters / 8); });
  double divs = 4.0 * (iters / 8) * (double)blocks * threads;
  float t_sqrt = timeit([&] { k_sqrt<<<blocks, threads>>>(out, iters / 8); });
  double sqrts = 4.0 * (iters / 8) * (double)blocks * threads;
  k_lat<<<1, 32>>>(out, 0.999999, 1e-7, iters, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"sms\": %d, \"clock_mhz_attr\": %d, \"dfma_tflops\": %.3f, \"dfma_lane_ops_per_clk_per_sm_at_attr_clock\": %.1f, "
         "\"dfma_latency_cycles\": %.2f, \"ddiv_per_s\": %.4e, \"dsqrt_per_s\": %.4e}\n",
         sms, clk / 1000, flops / (t_fma * 1e-3) / 1e12,
         flops / 2 / (t_fma * 1e-3) / (sms * (clk * 1e3)),
         (double)c / iters, divs / (t_div * 1e-3), sqrts / (t_sqrt * 1e-3));
  return 0;
}
