// accum.cu -- centre-update partial sums (_core.pyx:200-285).
//
// k_accum_range reproduces accumulate_range exactly: one thread per
// (frame, cluster, strip) folds the strip's matching pixels in row-major
// order in binary64 (colour) and int64 (x, y, count), so the slab is
// bit-identical to the reference's for ANY label map.
//
// accumulate_spill (pixels outside their cluster's 3Sx3S window; never
// produced by association, only by arbitrary label maps) keeps the
// reference's sequential row-major order per cluster: the spilled pixels are
// compacted in scan order (stable), stably sorted by label, and each
// cluster's run is folded into strip 0 in that order.
#include <cub/cub.cuh>

#include "spx_internal.cuh"

namespace spx {

__global__ void k_accum_range(const float* __restrict__ img, const int32_t* __restrict__ labels,
                              int64_t h, int64_t w, double* __restrict__ slab, int64_t n_bl,
                              int64_t s, int64_t ns_c, int64_t tile_len, int64_t k0, int64_t k1,
                              int64_t k_stride, int frames, const int32_t* __restrict__ done) {
  int64_t per_frame = (k1 - k0) * n_bl;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= per_frame * frames) return;
  int64_t f = i / per_frame;
  if (done && done[f]) return;
  int64_t rem = i % per_frame;
  int64_t k = k0 + rem / n_bl;
  int64_t j = rem % n_bl;
  const float* im = img + f * h * w * 3;
  const int32_t* lab = labels + f * h * w;
  int64_t r = k / ns_c, c = k % ns_c;
  int64_t wx0 = (c - 1) * s;
  if (wx0 < 0) wx0 = 0;
  int64_t wx1 = (c + 2) * s;
  if (wx1 > w) wx1 = w;
  int64_t ry0 = (r - 1) * s;
  int64_t ry1 = (r + 2) * s;
  if (ry1 > h) ry1 = h;
  int64_t sy0 = ry0 + j * tile_len;
  if (sy0 < 0) sy0 = 0;
  int64_t sy1 = ry0 + (j + 1) * tile_len;
  if (sy1 > ry1) sy1 = ry1;
  double sl = 0.0, sa = 0.0, sb = 0.0;
  int64_t sx = 0, sy = 0, cnt = 0;
  const int32_t kk = (int32_t)k;
  for (int64_t y = sy0; y < sy1; ++y) {
    const int32_t* row = lab + y * w;
    for (int64_t x = wx0; x < wx1; ++x) {
      if (__ldg(row + x) == kk) {
        const float* p = im + (y * w + x) * 3;
        sl = dadd(sl, (double)__ldg(p));
        sa = dadd(sa, (double)__ldg(p + 1));
        sb = dadd(sb, (double)__ldg(p + 2));
        sx += x;
        sy += y;
        cnt += 1;
      }
    }
  }
  double* o = slab + ((f * k_stride + k) * n_bl + j) * 6;
  o[0] = sl;
  o[1] = sa;
  o[2] = sb;
  o[3] = (double)sx;
  o[4] = (double)sy;
  o[5] = (double)cnt;
}

int launch_accum_range(const float* img, const int32_t* labels, int64_t h, int64_t w,
                       double* slab, int64_t n_bl, int64_t s, int64_t ns_c, int64_t tile_len,
                       int64_t k0, int64_t k1, int64_t k_stride, int frames, const int32_t* done,
                       cudaStream_t st) {
  int64_t n = (k1 - k0) * n_bl * frames;
  if (n <= 0) return SPX_OK;
  k_accum_range<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(img, labels, h, w, slab, n_bl, s,
                                                            ns_c, tile_len, k0, k1, k_stride,
                                                            frames, done);
  SPX_LAUNCH_CHECK("k_accum_range");
  return SPX_OK;
}

// ---- spill -------------------------------------------------------------------

__global__ void k_spill_flags(const int32_t* __restrict__ labels, int64_t h, int64_t w, int64_t s,
                              int64_t ns_c, int64_t n_clusters, uint8_t* __restrict__ flags,
                              int32_t* __restrict__ keys, unsigned long long* __restrict__ count,
                              int* __restrict__ bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= h * w) return;
  int64_t y = i / w, x = i % w;
  int64_t k = labels[i];
  if (k < 0 || k >= n_clusters) {
    atomicExch(bad, 1);
    flags[i] = 0;
    keys[i] = 0;
    return;
  }
  int64_t kr = k / ns_c, kc = k % ns_c;
  bool inside = x >= (kc - 1) * s && x < (kc + 2) * s && y >= (kr - 1) * s && y < (kr + 2) * s;
  flags[i] = inside ? 0 : 1;
  keys[i] = (int32_t)k;
  if (!inside) atomicAdd(count, 1ull);
}

__global__ void k_iota(int32_t* v, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

__global__ void k_gather_keys(const int32_t* __restrict__ idx, const int32_t* __restrict__ labels,
                              int32_t* __restrict__ keys, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = labels[idx[i]];
}

// One thread per run of equal labels in the sorted list: fold in scan order.
__global__ void k_spill_fold(const int32_t* __restrict__ keys, const int32_t* __restrict__ idx,
                             int64_t n, const float* __restrict__ img, int64_t w,
                             double* __restrict__ slab, int64_t n_bl) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i > 0 && keys[i - 1] == keys[i]) return;
  int64_t k = keys[i];
  double* o = slab + k * n_bl * 6;
  double a0 = o[0], a1 = o[1], a2 = o[2], a3 = o[3], a4 = o[4], a5 = o[5];
  for (int64_t q = i; q < n && keys[q] == keys[i]; ++q) {
    int64_t p = idx[q];
    const float* v = img + p * 3;
    a0 = dadd(a0, (double)v[0]);
    a1 = dadd(a1, (double)v[1]);
    a2 = dadd(a2, (double)v[2]);
    a3 = dadd(a3, (double)(p % w));
    a4 = dadd(a4, (double)(p / w));
    a5 = dadd(a5, 1.0);
  }
  o[0] = a0;
  o[1] = a1;
  o[2] = a2;
  o[3] = a3;
  o[4] = a4;
  o[5] = a5;
}

int spill(const float* img, const int32_t* labels, int64_t h, int64_t w, double* slab,
          int64_t n_clusters, int64_t n_bl, int64_t s, int64_t ns_c, int64_t* spills,
          cudaStream_t st) {
  int64_t n = h * w;
  *spills = 0;
  if (n == 0) return SPX_OK;
  if (n > INT32_MAX) {
    set_error("accumulate_spill: image too large for the spill path");
    return SPX_ERR_VALUE;
  }
  uint8_t* flags = nullptr;
  int32_t *keys = nullptr, *idx = nullptr, *sel = nullptr, *skeys = nullptr, *sidx = nullptr;
  unsigned long long* cnt = nullptr;
  int* bad = nullptr;
  int* nsel = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, need = 0;
  int rc = SPX_OK;
  unsigned long long hcnt = 0;
  int hbad = 0;
  unsigned blocks = (unsigned)ceil_div(n, 256);
#define SPILL_CUDA(call)                           \
  do {                                             \
    cudaError_t e__ = (call);                      \
    if (e__ != cudaSuccess) {                      \
      rc = cuda_status(e__, #call);                \
      goto out;                                    \
    }                                              \
  } while (0)
  SPILL_CUDA(cudaMallocAsync(&flags, n, st));
  SPILL_CUDA(cudaMallocAsync(&keys, n * 4, st));
  SPILL_CUDA(cudaMallocAsync(&cnt, 8, st));
  SPILL_CUDA(cudaMallocAsync(&bad, 4, st));
  SPILL_CUDA(cudaMemsetAsync(cnt, 0, 8, st));
  SPILL_CUDA(cudaMemsetAsync(bad, 0, 4, st));
  k_spill_flags<<<blocks, 256, 0, st>>>(labels, h, w, s, ns_c, n_clusters, flags, keys, cnt, bad);
  SPILL_CUDA(cudaGetLastError());
  SPILL_CUDA(cudaMemcpyAsync(&hcnt, cnt, 8, cudaMemcpyDeviceToHost, st));
  SPILL_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
  SPILL_CUDA(cudaStreamSynchronize(st));
  if (hbad) {
    set_error("accumulate_spill: label outside [0, %lld)", (long long)n_clusters);
    rc = SPX_ERR_DIMENSION;
    goto out;
  }
  *spills = (int64_t)hcnt;
  if (hcnt > 0) {
    int64_t m = (int64_t)hcnt;
    SPILL_CUDA(cudaMallocAsync(&idx, n * 4, st));
    SPILL_CUDA(cudaMallocAsync(&sel, m * 4, st));
    SPILL_CUDA(cudaMallocAsync(&skeys, m * 4, st));
    SPILL_CUDA(cudaMallocAsync(&sidx, m * 4, st));
    SPILL_CUDA(cudaMallocAsync(&nsel, 4, st));
    k_iota<<<blocks, 256, 0, st>>>(idx, n);
    SPILL_CUDA(cudaGetLastError());
    // stable compaction of spilled pixel indices (scan order)
    SPILL_CUDA(cub::DeviceSelect::Flagged(nullptr, need, idx, flags, sel, nsel, (int)n, st));
    tmp_bytes = need;
    SPILL_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, keys, skeys, sel, sidx, (int)m, 0,
                                               32, st));
    if (need > tmp_bytes) tmp_bytes = need;
    SPILL_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    need = tmp_bytes;
    SPILL_CUDA(cub::DeviceSelect::Flagged(tmp, need, idx, flags, sel, nsel, (int)n, st));
    k_gather_keys<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(sel, labels, keys, m);
    SPILL_CUDA(cudaGetLastError());
    need = tmp_bytes;
    // radix sort is stable: equal labels keep scan order
    SPILL_CUDA(cub::DeviceRadixSort::SortPairs(tmp, need, keys, skeys, sel, sidx, (int)m, 0, 32,
                                               st));
    k_spill_fold<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(skeys, sidx, m, img, w, slab, n_bl);
    SPILL_CUDA(cudaGetLastError());
  }
out:
  cudaFreeAsync(flags, st);
  cudaFreeAsync(keys, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(bad, st);
  if (idx) cudaFreeAsync(idx, st);
  if (sel) cudaFreeAsync(sel, st);
  if (skeys) cudaFreeAsync(skeys, st);
  if (sidx) cudaFreeAsync(sidx, st);
  if (nsel) cudaFreeAsync(nsel, st);
  if (tmp) cudaFreeAsync(tmp, st);
  if (rc == SPX_OK) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_status(e, "accumulate_spill");
  }
#undef SPILL_CUDA
  return rc;
}

}  // namespace spx

extern "C" int32_t spx_accumulate_range(const float* img, const int32_t* labels, int64_t h,
                                        int64_t w, double* slab, int64_t n_bl, int64_t s,
                                        int64_t ns_c, int64_t tile_len, int64_t k0, int64_t k1,
                                        void* stream) {
  using namespace spx;
  if (s < 1 || ns_c < 1 || tile_len < 1 || n_bl < 1 || k0 < 0) {
    set_error("accumulate_range: bad geometry");
    return SPX_ERR_VALUE;
  }
  return launch_accum_range(img, labels, h, w, slab, n_bl, s, ns_c, tile_len, k0, k1, 0, 1,
                            nullptr, as_stream(stream));
}

extern "C" int32_t spx_accumulate_spill(const float* img, const int32_t* labels, int64_t h,
                                        int64_t w, double* slab, int64_t n_clusters, int64_t n_bl,
                                        int64_t s, int64_t ns_c, int64_t* spills_host,
                                        void* stream) {
  using namespace spx;
  if (s < 1 || ns_c < 1 || n_bl < 1) {
    set_error("accumulate_spill: bad geometry");
    return SPX_ERR_VALUE;
  }
  return spill(img, labels, h, w, slab, n_clusters, n_bl, s, ns_c, spills_host,
               as_stream(stream));
}
