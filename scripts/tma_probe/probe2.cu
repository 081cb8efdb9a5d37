// TMA variants probe (debug aid, not product code).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int V>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, double* out, int nbytes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t sbar;
  uint64_t& bar = (V == 1) ? *reinterpret_cast<uint64_t*>(sm + 16 * 64 * 8 + 1024) : sbar;
  unsigned char* base = sm;
  if (V == 6) base = sm + ((1024 - (su(sm) & 1023)) & 1023);  // manual 1024-B alignment
  double* tile = reinterpret_cast<double*>(base);
  // (no printf)
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
    if (V != 2) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (V == 7 || V == 8) {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(nbytes) : "memory");
      __syncwarp();
      if (V == 7)
        asm volatile(
            "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
            "@P cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n}"
            ::"r"(su(tile)), "l"((uint64_t)&map), "r"(3), "r"(5), "r"(su(&bar)) : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(su(tile)), "l"((uint64_t)&map), "r"(3), "r"(5), "r"(su(&bar)) : "memory");
    }
  } else if (threadIdx.x == 0) {
    const CUtensorMap* mp = (V == 4) ? gmap : &map;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(nbytes) : "memory");
    if (V == 5)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su(tile)),
          "l"((uint64_t)mp), "r"(3), "r"(5), "r"(su(&bar))
          : "memory");

    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];" ::"r"(su(tile)),
          "l"((uint64_t)mp), "r"(3), "r"(5), "r"(su(&bar))
          : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(
          su(&bar)),
      "r"(0)
      : "memory");
  __syncthreads();
  if (V == 1 && threadIdx.x == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(su(&bar)) : "memory");
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) out[i] = tile[i];
}

template <int V>
void run(const CUtensorMap& map, const CUtensorMap* gmap, double* o, int M1, int nbytes) {
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 64 * 8 + 2048);
  cudaError_t e;
  if (V == 3) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 16 * 64 * 8 + 2048;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k<V>, map, gmap, o, nbytes);
  } else {
    k<V><<<1, 128, 16 * 64 * 8 + 2048>>>(map, gmap, o, nbytes);
    e = cudaGetLastError();
  }
  cudaError_t e2 = cudaDeviceSynchronize();
  double ho[2] = {0, 0};
  cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
  printf("V%d: launch=%s sync=%s out0=%g (expect %d)\n", V, cudaGetErrorString(e), cudaGetErrorString(e2), ho[0],
         5 * M1 + 3);
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int M0 = 100; const int M1 = argc > 2 ? atoi(argv[2]) : 150;
  double *f, *o;
  CUtensorMap* gm;
  cudaMalloc(&f, M0 * M1 * 8);
  cudaMalloc(&o, 4096 * 8);
  cudaMalloc(&gm, sizeof(CUtensorMap));
  static double h[100 * 1024];
  for (int i = 0; i < M0 * M1; ++i) h[i] = i;
  cudaMemcpy(f, h, sizeof h, cudaMemcpyHostToDevice);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap map;
  cuuint64_t dims[2] = {M1, M0};
  cuuint64_t str[1] = {M1 * 8};
  cuuint32_t box[2] = {(cuuint32_t)(argc > 3 ? atoi(argv[3]) : 64), (cuuint32_t)(argc > 4 ? atoi(argv[4]) : 16)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, f, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaMemcpy(gm, &map, sizeof map, cudaMemcpyHostToDevice);
  printf("encode=%d sizeof=%zu align=%zu\n", (int)r, sizeof(CUtensorMap), alignof(CUtensorMap));
  int v = atoi(argv[1]);
  switch (v) {
    case 1: run<1>(map, gm, o, M1, box[0]*box[1]*8); break;
    case 2: run<2>(map, gm, o, M1, box[0]*box[1]*8); break;
    case 3: run<3>(map, gm, o, M1, box[0]*box[1]*8); break;
    case 4: run<4>(map, gm, o, M1, box[0]*box[1]*8); break;
    case 5: run<5>(map, gm, o, M1, box[0]*box[1]*8); break;
    case 6: run<6>(map, gm, o, M1, box[0]*box[1]*8); break;
    case 7: run<7>(map, gm, o, M1, box[0]*box[1]*8); break;
    case 8: run<8>(map, gm, o, M1, box[0]*box[1]*8); break;
  }
  return 0;
}
