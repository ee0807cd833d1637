// fp64bench -- measured FP64 pipe throughput of one B200 (DADD, DMUL, DFMA),
// the ceiling k_convert's binary64 work runs against (profiles/r2_convert.md).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64bench fp64bench.cu
#include <cstdio>

template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) x[j] = __dadd_rn(x[j], a);
      if (OP == 1) x[j] = __dmul_rn(x[j], b);
      if (OP == 2) x[j] = __fma_rn(x[j], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"DADD", "DMUL", "DFMA"};
  for (int op = 0; op < 3; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) k<0><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
      if (op == 1) k<1><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
      if (op == 2) k<2><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 8;
    printf("%s: %.1f Gop/s = %.1f ops/clk/SM at %.0f MHz nominal (%d SMs)\n", names[op],
           ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3, sms);
  }
  return 0;
}
