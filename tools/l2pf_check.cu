// cp.async.bulk.prefetch.L2 with growing sizes: the band prefetch of the line
// kernel issues up to nx * 8 bytes per instruction (72 KB worst case); this
// checks that large sizes neither fault nor stall (sizes 16 B .. 16 MiB).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/l2pf_check tools/l2pf_check.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void pf(const char* p, unsigned n) {
  if (threadIdx.x == 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(n) : "memory");
}

int main() {
  char* d = nullptr;
  const size_t cap = 64u << 20;
  if (cudaMalloc(&d, cap) != cudaSuccess) { printf("cudaMalloc failed\n"); return 2; }
  cudaMemset(d, 1, cap);
  int bad = 0;
  for (unsigned n = 16; n <= (16u << 20); n *= 2) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    pf<<<148, 32>>>(d, n);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("size %9u B: %s, %.3f ms\n", n, cudaGetErrorString(e), ms);
    if (e != cudaSuccess) { bad = 1; break; }
  }
  // odd multiples of 16 near the sizes the kernel uses
  const unsigned odd[] = {65536 + 16, 72 * 1024 + 48, 131072 - 16, 300000 - 300000 % 16};
  for (unsigned n : odd) {
    pf<<<148, 32>>>(d + 16, n);
    cudaError_t e = cudaDeviceSynchronize();
    printf("size %9u B (offset 16): %s\n", n, cudaGetErrorString(e));
    if (e != cudaSuccess) { bad = 1; break; }
  }
  printf(bad ? "FAILED\n" : "ok\n");
  return bad;
}
