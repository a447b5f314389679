// Bitwise check of ws::FastMath against the IEEE operations on a B200:
// for random operands over wide exponent ranges, special values and signed
// zero numerators, every
// result whose range flag is set must equal `x / y`, `1.0 / y`, `sqrt(x)`
// bit for bit.  Prints one JSON line; exit code 1 on any mismatch.
// Built and run by tests/test_gpu_fastmath.py (same flags as the library).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../paper_1308_1464_b200/csrc/ws_math.cuh"

using ws::FastMath;

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ double operand(unsigned long long r, int mode) {
  if (mode == 0) {  // physical range: exponent in [-60, 60]
    unsigned long long m = r & 0x000fffffffffffffull;
    long long ex = 1023 + (long long)((r >> 52) % 121) - 60;
    unsigned long long s = (r >> 63) << 63;
    return __longlong_as_double((long long)(s | ((unsigned long long)ex << 52) | m));
  }
  if (mode == 1) {  // any finite or special bit pattern
    return __longlong_as_double((long long)r);
  }
  // extreme exponents near the range tests
  unsigned long long m = r & 0x000fffffffffffffull;
  long long ex = (long long)((r >> 52) % 2047);
  long long pick = (long long)((r >> 40) & 7);
  if (pick < 3) ex = (pick == 0) ? (long long)((r >> 52) % 80) : 2046 - (long long)((r >> 52) % 80);
  return __longlong_as_double((long long)(((r >> 63) << 63) | ((unsigned long long)ex << 52) | m));
}

__global__ void k_check(unsigned long long seed, long long n, unsigned long long* bad,
                        unsigned long long* fast) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const unsigned long long r1 = mix(seed ^ (2 * t)), r2 = mix(seed ^ (2 * t + 1));
    const int mode = (int)(t % 4);
    // mode 3: a signed-zero numerator over any bit pattern (zero-jump path)
    const double x = mode == 3 ? ((r1 & 1) ? -0.0 : 0.0) : operand(r1, mode);
    const double y = operand(r2, mode == 3 ? (int)((r2 >> 7) % 3) : mode);
    bool ok = true;
    double q = FastMath::div(x, y, ok);
    if (ok) {
      atomicAdd(&fast[0], 1ull);
      if (__double_as_longlong(q) != __double_as_longlong(x / y)) atomicAdd(&bad[0], 1ull);
    }
    ok = true;
    q = FastMath::rcp(y, ok);
    if (ok) {
      atomicAdd(&fast[1], 1ull);
      if (__double_as_longlong(q) != __double_as_longlong(1.0 / y)) atomicAdd(&bad[1], 1ull);
    }
    ok = true;
    const double ax = fabs(x);
    q = FastMath::sqrt_(ax, ok);
    if (ok) {
      atomicAdd(&fast[2], 1ull);
      if (__double_as_longlong(q) != __double_as_longlong(sqrt(ax))) atomicAdd(&bad[2], 1ull);
    }
  }
}

int main(int argc, char** argv) {
  long long n = argc > 1 ? atoll(argv[1]) : (1ll << 26);
  unsigned long long *bad, *fast, hb[3], hf[3];
  cudaMalloc(&bad, 24);
  cudaMalloc(&fast, 24);
  cudaMemset(bad, 0, 24);
  cudaMemset(fast, 0, 24);
  k_check<<<148 * 16, 256>>>(0x5eedull, n, bad, fast);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hb, bad, 24, cudaMemcpyDeviceToHost);
  cudaMemcpy(hf, fast, 24, cudaMemcpyDeviceToHost);
  printf("{\"n\": %lld, \"cuda\": \"%s\", \"div_fast\": %llu, \"div_bad\": %llu, \"rcp_fast\": %llu, "
         "\"rcp_bad\": %llu, \"sqrt_fast\": %llu, \"sqrt_bad\": %llu}\n",
         n, cudaGetErrorString(e), hf[0], hb[0], hf[1], hb[1], hf[2], hb[2]);
  return (e != cudaSuccess || hb[0] || hb[1] || hb[2]) ? 1 : 0;
}
