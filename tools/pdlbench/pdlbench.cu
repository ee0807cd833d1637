// Per-edge cost of dependent kernel launches in a CUDA graph, with and without
// programmatic dependent launch (PDL).  Development probe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdlbench pdlbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(float* buf, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float v = i < n ? buf[i] : 0.f;
#pragma unroll 1
  for (int k = 0; k < 64; ++k) v = v * 1.0001f + 0.5f;  // ~a few us of work
  if (i < n) buf[i] = v;
}

int main() {
  const int n = 148 * 256, chain = 20;
  float* buf;
  cudaMalloc(&buf, n * sizeof(float));
  cudaMemset(buf, 0, n * sizeof(float));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int blocks : {148, 2 * 148}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
      for (int c = 0; c < chain; ++c) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(n / blocks);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl;
        cudaLaunchKernelEx(&cfg, k_step, buf, n, pdl);
      }
      cudaStreamEndCapture(s, &g);
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("inst failed\n"); return 1; }
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 50; ++w) cudaGraphLaunch(ge, s);
      cudaEventRecord(a, s);
      const int reps = 500;
      for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("blocks %d pdl %d: %.2f us per graph of %d kernels = %.2f us per kernel\n", blocks, pdl,
             ms * 1e3 / reps, chain, ms * 1e3 / reps / chain);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
