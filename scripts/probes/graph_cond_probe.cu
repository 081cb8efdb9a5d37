#include <cuda_runtime.h>
#include <cstdio>
__global__ void body(cudaGraphConditionalHandle h, int* it, int maxit) {
  if (threadIdx.x == 0) {
    int v = ++(*it);
    cudaGraphSetConditional(h, v < maxit ? 1u : 0u);
  }
}
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  printf("add %s\n", cudaGetErrorString(e));
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  int* it; cudaMalloc(&it, 4); cudaMemset(it, 0, 4);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  body<<<1, 32, 0, s>>>(h, it, 5);
  cudaStreamEndCapture(s, &bodyg);
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %s\n", cudaGetErrorString(e));
  e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int h_it = 0; cudaMemcpy(&h_it, it, 4, cudaMemcpyDeviceToHost);
  printf("launch %s it=%d\n", cudaGetErrorString(e), h_it);
}
