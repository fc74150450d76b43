#include <cuda_runtime.h>
#include <cstdio>
__global__ void decide(int* ctr, cudaGraphConditionalHandle h) {
  int c = ++(*ctr);
  cudaGraphSetConditional(h, c < 5 ? 1 : 0);
}
__global__ void body(int* x) { atomicAdd(x, 1); }
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
  cudaGraphAddNode(&node, g, nullptr, 0, &p);
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  int *x, *c; cudaMalloc(&x, 4); cudaMalloc(&c, 4); cudaMemset(x, 0, 4); cudaMemset(c, 0, 4);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  body<<<1,1,0,s>>>(x);
  decide<<<1,1,0,s>>>(c, h);
  cudaGraph_t out; cudaStreamEndCapture(s, &out);
  cudaGraphExec_t ex; cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  printf("inst %s\n", cudaGetErrorString(e));
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int hx; cudaMemcpy(&hx, x, 4, cudaMemcpyDeviceToHost);
  printf("body ran %d times err %s\n", hx, cudaGetErrorString(cudaGetLastError()));
}
