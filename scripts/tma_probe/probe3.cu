// Isolate mbarrier / bulk copy / tensor TMA (debug aid, not product code).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda/barrier>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
using barrier = cuda::barrier<cuda::thread_scope_block>;
namespace cde = cuda::device::experimental;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void kA(double* out) {  // mbarrier init + plain arrive + wait
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(blockDim.x) : "memory");
  __syncthreads();
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(su(&bar)), "r"(0) : "memory");
  if (threadIdx.x == 0) out[0] = 42.0;
}

__global__ void kB(const double* src, double* out) {  // 1-D bulk copy
  __shared__ __align__(128) double buf[64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(512) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(buf)),
                 "l"((uint64_t)src), "r"(512), "r"(su(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(su(&bar)), "r"(0) : "memory");
  if (threadIdx.x < 64) out[threadIdx.x] = buf[threadIdx.x];
}

__global__ void kC(const __grid_constant__ CUtensorMap map, double* out, int nbytes) {  // libcu++ TMA reference
  __shared__ alignas(128) double tile[16 * 64];
#pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ barrier bar;
  if (threadIdx.x == 0) {
    init(&bar, blockDim.x);
    cde::fence_proxy_async_shared_cta();
  }
  __syncthreads();
  barrier::arrival_token token;
  if (threadIdx.x == 0) {
    cde::cp_async_bulk_tensor_2d_global_to_shared(tile, &map, 3, 5, bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, nbytes);
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) out[i] = tile[i];
}

int main(int argc, char** argv) {
  const int M0 = 100, M1 = 150;
  double *f, *o;
  cudaMalloc(&f, M0 * M1 * 8);
  cudaMalloc(&o, 4096 * 8);
  static double h[M0 * M1];
  for (int i = 0; i < M0 * M1; ++i) h[i] = i;
  cudaMemcpy(f, h, sizeof h, cudaMemcpyHostToDevice);
  int v = atoi(argv[1]);
  if (v == 1) kA<<<1, 128>>>(o);
  if (v == 2) kB<<<1, 128>>>(f + 64, o);
  if (v == 3) {
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    CUtensorMap map;
    int mode = argc > 2 ? atoi(argv[2]) : 0;
    CUtensorMapDataType dt = mode == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : mode == 1 ? CU_TENSOR_MAP_DATA_TYPE_INT64 :
                             mode == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    int mul = mode == 3 ? 2 : 1;
    cuuint64_t dims[2] = {(cuuint64_t)M1 * mul, M0};
    cuuint64_t str[1] = {M1 * 8};
    cuuint32_t box[2] = {(cuuint32_t)(64 * mul), 16};
    if (mode == 4) { dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT64; box[0] = 16; }
    cuuint32_t es[2] = {1, 1};
    CUresult r;
    if (argc > 3) {
      r = cuTensorMapEncodeTiled(&map, dt, 2, f, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("direct libcuda encode\n");
    } else
    r = enc(&map, dt, 2, f, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode=%d q=%d fn=%p\n", (int)r, (int)q, fnp);
    const unsigned long long* w = reinterpret_cast<const unsigned long long*>(&map);
    for (int i = 0; i < 16; ++i) printf("%016llx%c", w[i], i % 4 == 3 ? '\n' : ' ');
    int drv = 0, rt = 0; cudaDriverGetVersion(&drv); cudaRuntimeGetVersion(&rt); printf("driver %d runtime %d\n", drv, rt);
    kC<<<1, 128>>>(map, o, mode == 4 ? 16 * 16 * 8 : 16 * 64 * 8);
  }
  cudaError_t e = cudaDeviceSynchronize();
  double ho[2] = {0, 0};
  cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
  printf("probe %d: %s out0=%g out1=%g\n", v, cudaGetErrorString(e), ho[0], ho[1]);
  return 0;
}
