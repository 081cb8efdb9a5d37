// Launch probe2's V1 kernel from its cubin through the driver API (debug aid).
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#define CHK(x)                                                        \
  do {                                                                \
    CUresult r_ = (x);                                                \
    if (r_ != CUDA_SUCCESS) {                                         \
      const char* s_;                                                 \
      cuGetErrorString(r_, &s_);                                      \
      printf("%s -> %d %s\n", #x, (int)r_, s_);                       \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main(int argc, char** argv) {
  CHK(cuInit(0));
  CUdevice dev;
  CHK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CHK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CHK(cuCtxSetCurrent(ctx));
  CUmodule mod;
  CHK(cuModuleLoad(&mod, argv[1]));
  CUfunction fn;
  CHK(cuModuleGetFunction(&fn, mod, "_Z1kILi1EEv14CUtensorMap_stPKS0_Pdi"));
  const int M0 = 100, M1 = 152;
  CUdeviceptr f, o;
  CHK(cuMemAlloc(&f, M0 * M1 * 8));
  CHK(cuMemAlloc(&o, 4096 * 8));
  static double h[M0 * M1];
  for (int i = 0; i < M0 * M1; ++i) h[i] = i;
  CHK(cuMemcpyHtoD(f, h, sizeof h));
  alignas(64) CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)M1, (cuuint64_t)M0};
  cuuint64_t str[1] = {(cuuint64_t)M1 * 8};
  cuuint32_t box[2] = {64, 16};
  cuuint32_t es[2] = {1, 1};
  CHK(cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)f, dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  CUdeviceptr gm = 0;
  int nb = 64 * 16 * 8; void* args[4] = {&map, &gm, &o, &nb};
  CHK(cuFuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 16 * 64 * 8 + 2048));
  CHK(cuLaunchKernel(fn, 1, 1, 1, 128, 1, 1, 16 * 64 * 8 + 2048, 0, args, nullptr));
  CUresult r = cuCtxSynchronize();
  const char* es2;
  cuGetErrorString(r, &es2);
  double ho[2] = {0, 0};
  if (r == CUDA_SUCCESS) cuMemcpyDtoH(ho, o, 16);
  printf("driver-launch: %s out0=%g (expect %d)\n", es2, ho[0], 5 * M1 + 3);
  return 0;
}
