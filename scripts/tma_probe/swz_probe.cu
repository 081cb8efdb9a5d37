// Dump the raw smem layout of a SWIZZLE_128B fp64 TMA box (debug aid).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include "../../paper_2210_06528_b200/csrc/tma.cuh"
using namespace mfb;

__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int lines, int with_static) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned long long s_static[32];
  if (with_static && threadIdx.x < 32) s_static[threadIdx.x] = threadIdx.x;
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(sm + lines * 128 + 1024);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, lines * 128);
    tma_load_2d(sm, &map, 0, 0, bar);
  }
  mbar_wait(bar, 0);
  const double* d = reinterpret_cast<const double*>(sm);
  for (int i = threadIdx.x; i < lines * 16; i += blockDim.x) out[i] = d[i];
  if (threadIdx.x == 0) out[lines * 16] = (double)smem_u32(sm) + (with_static ? s_static[3] * 0 : 0);
}

int main(int argc, char** argv) {
  const int lines = argc > 1 ? atoi(argv[1]) : 24, ws = argc > 2 ? atoi(argv[2]) : 0;
  const int R = 200, C = 32;
  double *f, *o;
  cudaMalloc(&f, R * C * 8);
  cudaMalloc(&o, (lines * 16 + 1) * 8);
  static double h[R * C];
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = r * 100 + c;
  cudaMemcpy(f, h, sizeof h, cudaMemcpyHostToDevice);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t str[1] = {(cuuint64_t)C * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)lines};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, f, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = lines * 128 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 128, smem>>>(map, o, lines, ws);
  cudaError_t e = cudaDeviceSynchronize();
  static double ho[4096];
  cudaMemcpy(ho, o, (lines * 16 + 1) * 8, cudaMemcpyDeviceToHost);
  printf("encode=%d run=%s smem_base=%g\n", (int)r, cudaGetErrorString(e), ho[lines * 16]);
  for (int l = 0; l < lines; ++l) {
    printf("line %2d:", l);
    for (int k = 0; k < 8; ++k) printf(" %5g", ho[l * 16 + 2 * k]);  // first double of each 16-B chunk
    printf("\n");
  }
  return 0;
}
