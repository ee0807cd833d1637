// cellbench -- standalone timing of the fused cell kernels (development tool).
//
// Runs the engine's stage sequence on B synthetic C1 frames (random RGB, the
// reference generator's distribution) to reach realistic centres, then times
// k_cell<ACC> and k_cell<final> launches alone with CUDA events.  Built
// against one variant of the kernel sources (see tools/cellbench/run.sh).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_1509_04232_b200/csrc/spx_internal.cuh"

namespace spx {
int launch_convert(const uint8_t*, float*, int64_t, int64_t, int, cudaStream_t, int64_t, int64_t,
                   float);
int launch_records(const double*, const double*, CRec*, int64_t, int64_t, int64_t, int,
                   cudaStream_t, int64_t, int64_t, int64_t);
}  // namespace spx

using namespace spx;

__global__ void k_rand_rgb(uint8_t* p, long long n, unsigned seed) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    p[i] = (uint8_t)(x >> 24);
  }
}

#define CK(x) do { int rc_ = (x); if (rc_) { fprintf(stderr, "%s failed: %d %s\n", #x, rc_, spx_last_error()); return 1; } } while (0)
#define CC(x) do { cudaError_t e_ = (x); if (e_) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 256;
  const int H = argc > 2 ? atoi(argv[2]) : 480, W = argc > 3 ? atoi(argv[3]) : 640;
  const int S = argc > 4 ? atoi(argv[4]) : 16;
  const int reps = 20;
  const int ns_r = (H + S - 1) / S, ns_c = (W + S - 1) / S;
  const long long K = (long long)ns_r * ns_c, hw = (long long)H * W;
  const double xyw = 10.0 / S;
  uint8_t* rgb; float* lab; int32_t* labels; double *cxy[2], *clab[2]; CRec* rec; ClusterAcc* acc;
  int64_t* counts; int32_t* wl;
  CC(cudaMalloc(&rgb, B * hw * 3));
  CC(cudaMalloc(&lab, B * hw * 12));
  CC(cudaMalloc(&labels, B * hw * 4));
  for (int i = 0; i < 2; ++i) {
    CC(cudaMalloc(&cxy[i], B * K * 16));
    CC(cudaMalloc(&clab[i], B * K * 24));
  }
  CC(cudaMalloc(&rec, B * K * sizeof(CRec)));
  CC(cudaMalloc(&acc, B * K * sizeof(ClusterAcc)));
  CC(cudaMalloc(&counts, B * K * 8));
  CC(cudaMalloc(&wl, (B * K + 1) * 4));
  cudaStream_t s = 0;
  k_rand_rgb<<<1184, 256>>>(rgb, B * hw * 3, 12345u);
  CK(launch_convert(rgb, lab, 0, B * hw, 2, s, hw, S, -1.f));
  CK(launch_init(lab, H, W, S, ns_c, cxy[0], clab[0], 0, K, K, B, 0, 1, s, 1, -1, 0));
  CK(launch_records(cxy[0], clab[0], rec, ns_r, ns_c, S, B, s, 0, -1, 0));
  CC(cudaMemsetAsync(acc, 0, B * K * sizeof(ClusterAcc), s));
  int cur = 0;
  for (int it = 0; it < 5; ++it) {
    CK(launch_cell(lab, cxy[cur], clab[cur], rec, labels, acc, nullptr, H, W, S, ns_r, ns_c, xyw,
                   B, true, s, 0, -1, 0));
    CK(launch_reduce_cells(acc, lab, labels, cxy[cur], clab[cur], cxy[cur ^ 1], clab[cur ^ 1],
                           counts, rec, nullptr, wl, wl + B * K, H, W, S, ns_r, ns_c, 16, B, s, 0,
                           -1, 0));
    cur ^= 1;
    int nflag = 0;
    CC(cudaMemcpy(&nflag, wl + B * K, 4, cudaMemcpyDeviceToHost));
    printf("pass %d: %d of %lld clusters flagged for the exact fallback\n", it, nflag, B * K);

  }
  CC(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  {
    for (int w = 0; w < 10; ++w) CK(launch_convert(rgb, lab, 0, B * hw, 2, s, hw, S, -1.f));
    std::vector<float> t(reps);
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0, s);
      CK(launch_convert(rgb, lab, 0, B * hw, 2, s, hw, S, -1.f));
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&t[r], e0, e1);
    }
    float sum = 0.f;
    for (float v : t) sum += v;
    printf("k_convert %dx%dx%d: mean %.4f ms (%.1f Gpx/s)\n", B, H, W, sum / reps,
           B * hw / (sum / reps) / 1e6);
  }
  for (int accf = 1; accf >= 0; --accf) {
    for (int w = 0; w < 3; ++w)
      CK(launch_cell(lab, cxy[cur], clab[cur], rec, labels, acc, nullptr, H, W, S, ns_r, ns_c, xyw,
                     B, accf, s, 0, -1, 0));
    std::vector<float> t(reps);
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0, s);
      CK(launch_cell(lab, cxy[cur], clab[cur], rec, labels, acc, nullptr, H, W, S, ns_r, ns_c, xyw,
                     B, accf, s, 0, -1, 0));
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&t[r], e0, e1);
    }
    float best = 1e9f, sum = 0.f;
    for (float v : t) { best = v < best ? v : best; sum += v; }
    printf("k_cell<%d> %dx%dx%d S=%d: mean %.4f ms  min %.4f ms  (%.1f Gpx/s)\n", accf, B, H, W, S,
           sum / reps, best, B * hw / (sum / reps) / 1e6);
  }
  CC(cudaGetLastError());
  return 0;
}
