// FP64 FMA throughput of this GPU (the FP64 roofline denominator):
// every SM fully occupied, 8 independent DFMA chains per thread, CUDA-event timed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dfma_loop(double* out, double a, double b, int iters) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-6 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 256 * sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 1 << 15;
  dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7, 1024);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * kChains * static_cast<double>(iters) * blocks * threads;
    const double tf = flops / (ms * 1e-3) / 1e12;
    best = tf > best ? tf : best;
  }
  const double per_sm_clk = best * 1e12 / 2.0 / sms / (clk * 1e3);
  std::printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"sm_clock_mhz_attr\": %.0f, \"dfma_per_sm_per_clk\": %.1f}\n", best,
              sms, clk / 1e3, per_sm_clk);
  return 0;
}
