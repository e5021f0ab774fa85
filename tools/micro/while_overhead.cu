// Microbenchmark: per-iteration cost of a CUDA-graph conditional WHILE loop
// whose body is one kernel (grid G x 256) that decrements a counter.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(unsigned* cnt, cudaGraphConditionalHandle h) {
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned c = --(*cnt);
    if (h) cudaGraphSetConditional(h, c > 0);
  }
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); fflush(stdout); return 1; } } while (0)
int main() {
  unsigned* cnt;
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&cnt, 4));
  for (int G : {1, 148, 1184}) {
    cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h; CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t node; CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    void* args[] = {&cnt, &h};
    cudaKernelNodeParams kp = {}; kp.func = (void*)body; kp.gridDim = dim3(G); kp.blockDim = dim3(256); kp.kernelParams = args;
    cudaGraphNode_t kn; CK(cudaGraphAddKernelNode(&kn, cp.conditional.phGraph_out[0], nullptr, 0, &kp));
    cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
    for (int rep = 0; rep < 2; ++rep) {
      unsigned N = 10000; cudaMemcpy(cnt, &N, 4, cudaMemcpyHostToDevice);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a); cudaGraphLaunch(ex, 0); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("grid %d: %.2f us per iteration (%s)\n", G, ms * 1000 / N, cudaGetErrorString(cudaGetLastError())); fflush(stdout);
    }
    // same kernel launched from the host in a loop, no sync
    unsigned N = 10000; cudaMemcpy(cnt, &N, 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int it = 0; it < 10000; ++it) body<<<G, 256>>>(cnt, (cudaGraphConditionalHandle)0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %d: %.2f us per host launch (async)\n", G, ms * 1000 / 10000);
  }
  return 0;
}
