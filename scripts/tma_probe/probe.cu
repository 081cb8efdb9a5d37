// Standalone probe of the TMA/mbarrier helpers (debug aid, not product code).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2210_06528_b200/csrc/tma.cuh"
using namespace mfb;

__global__ void k(const __grid_constant__ CUtensorMap map, const double* src1d, double* out, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) std::uint64_t bar;
  double* tile = reinterpret_cast<double*>(sm);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned bytes = 0;
    if (mode & 1) bytes += 16 * 64 * 8;
    if (mode & 2) bytes += 256;
    mbar_arrive_expect_tx(&bar, bytes);
    if (mode & 1) tma_load_2d(tile, &map, 3, 5, &bar);
    if (mode & 2) bulk_load_1d(sm + 16 * 64 * 8, src1d, 256, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 16 * 64 + 32; i += blockDim.x) out[i] = tile[i];
}

int main() {
  const int M0 = 100, M1 = 150;
  double *f, *o;
  cudaMalloc(&f, M0 * M1 * 8);
  cudaMalloc(&o, 4096 * 8);
  double h[M0 * M1];
  for (int i = 0; i < M0 * M1; ++i) h[i] = i;
  cudaMemcpy(f, h, sizeof h, cudaMemcpyHostToDevice);
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap map;
  cuuint64_t dims[2] = {M1, M0}; cuuint64_t str[1] = {M1 * 8}; cuuint32_t box[2] = {64, 16}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, f, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d\n", (int)r);
  for (int mode = 1; mode <= 3; ++mode) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 64 * 8 + 512);
    k<<<1, 128, 16 * 64 * 8 + 512>>>(map, f + 64, o, mode);
    cudaError_t e = cudaDeviceSynchronize();
    double ho[4];
    cudaMemcpy(ho, o, 32, cudaMemcpyDeviceToHost);
    printf("mode %d: %s  out[0]=%g (expect %d) out[1]=%g\n", mode, cudaGetErrorString(e), ho[0], 5 * M1 + 3, ho[1]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
