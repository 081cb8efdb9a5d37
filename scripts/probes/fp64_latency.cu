// FP64 / smem latency probe (single warp, dependent chains, clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double y = threadIdx.x * 1e-3;
  for (int i = 0; i < n; ++i) y = y * a;
  long long t2 = clock64();
  __shared__ double sm[64];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  int j = threadIdx.x & 31;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) j = static_cast<int>(sm[j]) & 31;  // dependent smem loads
  long long t4 = clock64();
  double z = 1.0 + threadIdx.x;
  for (int i = 0; i < n; ++i) z = rsqrt(z) + 1.0;
  long long t5 = clock64();
  out[threadIdx.x] = x + y + j + z;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t4 - t3;
    cyc[3] = t5 - t4;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * 8);
  cudaMallocManaged(&cyc, 4 * 8);
  const int n = 4096;
  chain<<<1, 32>>>(out, cyc, 0.999, 1e-3, n);
  chain<<<1, 32>>>(out, cyc, 0.999, 1e-3, n);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: DFMA %.1f  DMUL %.1f  LDS(+cvt) %.1f  rsqrt+add %.1f\n", double(cyc[0]) / n,
         double(cyc[1]) / n, double(cyc[2]) / n, double(cyc[3]) / n);
  return 0;
}
