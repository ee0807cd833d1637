// connect.cu -- connectivity cleanup.
//
// Weak (_core.pyx:328-356): a pixel none of whose in-bounds 4-neighbours
// shares its label adopts the left neighbour (top in column 0; (0,0) never
// changes), reading a frozen snapshot; the engine applies it twice
// (engine.py:204-206).  k_weak2 fuses both passes: each CTA computes pass 1
// on its tile plus a 1-pixel halo in shared memory (from a 2-pixel halo of
// the source) and pass 2 on the tile, so labels cross HBM once each way
// (8 B/px instead of 16).
//
// Strict (_core.pyx:359-461) is a sequential scan-order flood fill.  Its
// result is reproduced in parallel:
//   * components are 4-connected equal-label regions; the reference's
//     component order is the scan order of their first pixel, i.e. their
//     minimum linear index, so union-find with min-index roots orders them;
//   * the seed's "first finalized neighbour" is always the left neighbour
//     (up in column 0; none for pixel 0): left/up precede the seed in scan
//     order and cannot be in its component, right/down cannot be finalized;
//   * a component keeps its label iff it is the first component (pixel 0),
//     or it is the first component of that label with size >= min_size and
//     pixel 0's component does not carry the same label (the `used` flag can
//     only be set by such a keeper);
//   * absorbed components take the final value of their seed-left
//     component, resolved by pointer jumping.
#include <climits>

#include "spx_internal.cuh"

namespace spx {

namespace {

constexpr int WTW = 32, WTH = 8;

__device__ __forceinline__ int32_t weak_rule(const int32_t* src, int64_t w, int64_t h, int64_t x,
                                             int64_t y, int pitch, int lx, int ly) {
  // src is a shared-memory tile with pitch; (lx,ly) local coords of (x,y).
  int32_t v = src[ly * pitch + lx];
  int32_t left = x > 0 ? src[ly * pitch + lx - 1] : 0;
  if (x > 0 && left == v) return v;
  if (x < w - 1 && src[ly * pitch + lx + 1] == v) return v;
  int32_t up = y > 0 ? src[(ly - 1) * pitch + lx] : 0;
  if (y > 0 && up == v) return v;
  if (y < h - 1 && src[(ly + 1) * pitch + lx] == v) return v;
  if (x > 0) return left;
  if (y > 0) return up;
  return v;
}

// One pass over rows [y0,y1) (the kernel-protocol weak_band).
__global__ void __launch_bounds__(WTW* WTH) k_weak1(const int32_t* __restrict__ src,
                                                     int32_t* __restrict__ dst, int64_t h,
                                                     int64_t w, int64_t y0, int64_t y1) {
  constexpr int P = WTW + 2;
  __shared__ int32_t t[(WTH + 2) * P];
  int64_t tx0 = (int64_t)blockIdx.x * WTW, ty0 = y0 + (int64_t)blockIdx.y * WTH;
  for (int i = threadIdx.y * WTW + threadIdx.x; i < (WTH + 2) * P; i += WTW * WTH) {
    int ly = i / P, lx = i % P;
    int64_t y = ty0 + ly - 1, x = tx0 + lx - 1;
    t[i] = (y >= 0 && y < h && x >= 0 && x < w) ? src[y * w + x] : 0;
  }
  __syncthreads();
  int64_t x = tx0 + threadIdx.x, y = ty0 + threadIdx.y;
  if (x >= w || y >= y1) return;
  dst[y * w + x] = weak_rule(t, w, h, x, y, P, threadIdx.x + 1, threadIdx.y + 1);
}

// Both passes fused; frames of a batch along blockIdx.z.  32-bit indexing
// (frames < 2^31 px).
// Output rows [y0, y1) of a buffer of h rows (row strips pass their halo
// rows in the buffer and only their own rows as the output range; image
// edges coincide with buffer edges, interior strip edges have >= 2 halo rows).
//
// Work unit: a group of 4 horizontally adjacent pixels.  The source tile
// (WG x HG outputs, 8-column / 2-row halo) is staged as int4 groups; pass 1
// is evaluated group-wise on the tile plus a 4-column / 1-row halo into a
// second int4 tile, pass 2 group-wise on the output tile.  A group reads its
// own, the upper and the lower int4 and one word on each side: 5 shared
// loads per 4 pixels per pass.
constexpr int WG = 128, HG = 32;
constexpr int NG0 = WG / 4 + 4, R0G = HG + 4;  // source groups: cols [x0-8, x0+WG+8)
constexpr int NG1 = WG / 4 + 2, R1G = HG + 2;  // pass-1 groups: cols [x0-4, x0+WG+4)

// Pixels outside the image hold kOut in the tiles, a value no pipeline label
// takes (labels are cluster ids >= 0), so "neighbour in bounds and equal"
// is a plain comparison and "in bounds" is `!= kOut`.
constexpr int kOut = INT_MIN;

__device__ __forceinline__ int4 weak_rule4(int4 v, int4 up, int4 dn, int lft, int rgt) {
  const int vv[4] = {v.x, v.y, v.z, v.w};
  const int uu[4] = {up.x, up.y, up.z, up.w};
  const int dd[4] = {dn.x, dn.y, dn.z, dn.w};
  int o[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int L = k == 0 ? lft : vv[k - 1];
    const int R = k == 3 ? rgt : vv[k + 1];
    const int c = vv[k];
    const bool keep = (L == c) | (R == c) | (uu[k] == c) | (dd[k] == c);
    o[k] = keep ? c : (L != kOut ? L : (uu[k] != kOut ? uu[k] : c));
  }
  return make_int4(o[0], o[1], o[2], o[3]);
}

__global__ void __launch_bounds__(256) k_weak2(const int32_t* __restrict__ src,
                                               int32_t* __restrict__ dst, int h, int w, int y0,
                                               int y1) {
  __shared__ int4 t0[R0G][NG0];
  __shared__ int4 t1[R1G][NG1];
  const long long fo = (long long)blockIdx.z * h * w;
  const int32_t* s = src + fo;
  int32_t* d = dst + fo;
  const int tx0 = blockIdx.x * WG, ty0 = y0 + blockIdx.y * HG;
  const int tid = threadIdx.x;
  const bool vec = (w & 3) == 0;
  for (int i = tid; i < R0G * NG0; i += 256) {
    const int r = i / NG0, g = i - r * NG0;
    const int y = ty0 - 2 + r, x = tx0 - 8 + 4 * g;
    int4 v = make_int4(kOut, kOut, kOut, kOut);
    if (y >= 0 && y < h) {
      const int32_t* row = s + (long long)y * w;
      if (vec && x >= 0 && x + 4 <= w) {
        v = __ldg(reinterpret_cast<const int4*>(row + x));
      } else {
        v.x = (x >= 0 && x < w) ? __ldg(row + x) : kOut;
        v.y = (x + 1 >= 0 && x + 1 < w) ? __ldg(row + x + 1) : kOut;
        v.z = (x + 2 >= 0 && x + 2 < w) ? __ldg(row + x + 2) : kOut;
        v.w = (x + 3 >= 0 && x + 3 < w) ? __ldg(row + x + 3) : kOut;
      }
    }
    t0[r][g] = v;
  }
  __syncthreads();
  // pass 1 on rows [ty0-1, ty0+HG+1), cols [tx0-4, tx0+WG+4)
  for (int i = tid; i < R1G * NG1; i += 256) {
    const int r = i / NG1, g = i - r * NG1;
    int4 o = weak_rule4(t0[r + 1][g + 1], t0[r][g + 1], t0[r + 2][g + 1], t0[r + 1][g].w,
                        t0[r + 1][g + 2].x);
    // out-of-image positions stay kOut for pass 2 (the rule keeps c = kOut:
    // its in-image neighbours never equal kOut, its left / up may be kOut)
    const int4 c = t0[r + 1][g + 1];
    o.x = c.x == kOut ? kOut : o.x;
    o.y = c.y == kOut ? kOut : o.y;
    o.z = c.z == kOut ? kOut : o.z;
    o.w = c.w == kOut ? kOut : o.w;
    t1[r][g] = o;
  }
  __syncthreads();
  // pass 2 on the output tile
  for (int i = tid; i < HG * (WG / 4); i += 256) {
    const int r = i / (WG / 4), g = i - r * (WG / 4);
    const int y = ty0 + r, x = tx0 + 4 * g;
    if (y >= y1 || x >= w) continue;
    const int4 o = weak_rule4(t1[r + 1][g + 1], t1[r][g + 1], t1[r + 2][g + 1], t1[r + 1][g].w,
                              t1[r + 1][g + 2].x);
    int32_t* out = d + (long long)y * w + x;
    if (vec) {
      *reinterpret_cast<int4*>(out) = o;
    } else {
      const int oo[4] = {o.x, o.y, o.z, o.w};
      for (int k = 0; k < 4; ++k)
        if (x + k < w) out[k] = oo[k];
    }
  }
}

// ---- strict -------------------------------------------------------------------

__device__ __forceinline__ int32_t uf_find(const int32_t* parent, int32_t x) {
  int32_t p = parent[x];
  while (p != x) {
    x = p;
    p = parent[x];
  }
  return x;
}

__device__ __forceinline__ void uf_unite(int32_t* parent, int32_t a, int32_t b) {
  while (true) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a > b) {
      int32_t t = a;
      a = b;
      b = t;
    }
    int32_t old = atomicMin(parent + b, a);
    if (old == b) return;
    b = old;
  }
}

__global__ void k_cc_init(int32_t* parent, int32_t* size, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    parent[i] = (int32_t)i;
    size[i] = 0;
  }
}

__global__ void k_cc_union(const int32_t* __restrict__ lab, int32_t* parent, int64_t h, int64_t w,
                           int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t local = i % (h * w);
  int64_t x = local % w, y = local / w;
  int32_t v = lab[i];
  if (x < w - 1 && lab[i + 1] == v) uf_unite(parent, (int32_t)i, (int32_t)(i + 1));
  if (y < h - 1 && lab[i + w] == v) uf_unite(parent, (int32_t)i, (int32_t)(i + w));
}

__global__ void k_cc_flatten(int32_t* parent, int32_t* size, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t r = uf_find(parent, (int32_t)i);
  parent[i] = r;
  atomicAdd(size + r, 1);
}

__global__ void k_cc_first(const int32_t* __restrict__ lab, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ size, int32_t* first, int64_t hw,
                           int64_t n, int64_t nlab, int64_t min_size) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || parent[i] != (int32_t)i || size[i] < min_size) return;
  int64_t f = i / hw;
  atomicMin(first + f * nlab + lab[i], (int32_t)i);
}

__global__ void k_cc_next(const int32_t* __restrict__ lab, const int32_t* __restrict__ parent,
                          const int32_t* __restrict__ size, const int32_t* __restrict__ first,
                          int32_t* nxt, int64_t w, int64_t hw, int64_t n, int64_t nlab,
                          int64_t min_size) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || parent[i] != (int32_t)i) return;
  int64_t f = i / hw, base = f * hw, local = i - base;
  int32_t v = lab[i];
  bool keep = local == 0 ||
              (size[i] >= min_size && first[f * nlab + v] == (int32_t)i && lab[base] != v);
  if (keep) {
    nxt[i] = (int32_t)i;
  } else {
    int64_t adj = (local % w > 0) ? i - 1 : i - w;
    nxt[i] = parent[adj];
  }
}

__global__ void k_cc_jump(const int32_t* __restrict__ parent, int32_t* nxt, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || parent[i] != (int32_t)i) return;
  nxt[i] = nxt[nxt[i]];
}

__global__ void k_cc_write(const int32_t* __restrict__ lab, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ nxt, int32_t* __restrict__ dst, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dst[i] = lab[nxt[parent[i]]];
}

__global__ void k_max_label(const int32_t* __restrict__ lab, int64_t n, int* out, int* neg) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int v = i < n ? lab[i] : 0;
  if (i < n && v < 0) atomicExch(neg, 1);
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, v);
}

}  // namespace

int launch_weak1(const int32_t* src, int32_t* dst, int64_t h, int64_t w, int64_t y0, int64_t y1,
                 cudaStream_t st) {
  if (y1 <= y0 || w <= 0) return SPX_OK;
  dim3 grid((unsigned)ceil_div(w, WTW), (unsigned)ceil_div(y1 - y0, WTH));
  k_weak1<<<grid, dim3(WTW, WTH), 0, st>>>(src, dst, h, w, y0, y1);
  SPX_LAUNCH_CHECK("k_weak1");
  return SPX_OK;
}

int launch_weak2(const int32_t* src, int32_t* dst, int64_t h, int64_t w, int frames,
                 cudaStream_t st, int64_t y0, int64_t y1) {
  if (y1 < 0) y1 = h;
  if (y1 <= y0 || w <= 0 || frames <= 0) return SPX_OK;
  if (h * w >= (int64_t)1 << 31 || frames > 65535) {
    set_error("weak: frame too large for the fused kernel");
    return SPX_ERR_VALUE;
  }
  dim3 grid((unsigned)ceil_div(w, WG), (unsigned)ceil_div(y1 - y0, HG), (unsigned)frames);
  k_weak2<<<grid, 256, 0, st>>>(src, dst, (int)h, (int)w, (int)y0, (int)y1);
  SPX_LAUNCH_CHECK("k_weak2");
  return SPX_OK;
}

// scratch: parent, size, nxt (n each) and first (frames * nlab), all int32.
int launch_strict(const int32_t* src, int32_t* dst, int64_t h, int64_t w, int frames,
                  int64_t nlab, int64_t min_size, int32_t* parent, int32_t* size, int32_t* nxt,
                  int32_t* first, cudaStream_t st) {
  int64_t hw = h * w, n = hw * frames;
  if (n == 0) return SPX_OK;
  if (n >= INT32_MAX) {
    set_error("strict_fill: %lld pixels exceed the int32 component index", (long long)n);
    return SPX_ERR_VALUE;
  }
  unsigned b = (unsigned)ceil_div(n, 256);
  k_cc_init<<<b, 256, 0, st>>>(parent, size, n);
  SPX_CUDA(cudaMemsetAsync(first, 0x7f, (size_t)(frames * nlab) * 4, st));
  k_cc_union<<<b, 256, 0, st>>>(src, parent, h, w, n);
  k_cc_flatten<<<b, 256, 0, st>>>(parent, size, n);
  k_cc_first<<<b, 256, 0, st>>>(src, parent, size, first, hw, n, nlab, min_size);
  k_cc_next<<<b, 256, 0, st>>>(src, parent, size, first, nxt, w, hw, n, nlab, min_size);
  int rounds = 1;
  while ((1ll << rounds) < n) ++rounds;
  for (int r = 0; r <= rounds; ++r) k_cc_jump<<<b, 256, 0, st>>>(parent, nxt, n);
  k_cc_write<<<b, 256, 0, st>>>(src, parent, nxt, dst, n);
  SPX_LAUNCH_CHECK("strict_fill kernels");
  return SPX_OK;
}

int strict_fill_alloc(const int32_t* src, int32_t* dst, int64_t h, int64_t w, int64_t min_size,
                      cudaStream_t st) {
  int64_t n = h * w;
  if (n == 0) return SPX_OK;
  int* mx = nullptr;
  int32_t *parent = nullptr, *size = nullptr, *nxt = nullptr, *first = nullptr;
  int hm[2] = {0, 0};
  int rc = SPX_OK;
  SPX_CUDA(cudaMallocAsync(&mx, 8, st));
  SPX_CUDA(cudaMemsetAsync(mx, 0, 8, st));
  k_max_label<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(src, n, mx, mx + 1);
  SPX_CUDA(cudaMemcpyAsync(hm, mx, 8, cudaMemcpyDeviceToHost, st));
  SPX_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(mx, st);
  if (hm[1]) {
    set_error("strict_fill: negative label");
    return SPX_ERR_VALUE;
  }
  int64_t nlab = (int64_t)hm[0] + 1;
  SPX_CUDA(cudaMallocAsync(&parent, n * 4, st));
  SPX_CUDA(cudaMallocAsync(&size, n * 4, st));
  SPX_CUDA(cudaMallocAsync(&nxt, n * 4, st));
  SPX_CUDA(cudaMallocAsync(&first, nlab * 4, st));
  rc = launch_strict(src, dst, h, w, 1, nlab, min_size, parent, size, nxt, first, st);
  cudaFreeAsync(parent, st);
  cudaFreeAsync(size, st);
  cudaFreeAsync(nxt, st);
  cudaFreeAsync(first, st);
  if (rc == SPX_OK) SPX_CUDA(cudaStreamSynchronize(st));
  return rc;
}

}  // namespace spx

extern "C" int32_t spx_weak_band(const int32_t* src, int32_t* dst, int64_t h, int64_t w,
                                 int64_t y0, int64_t y1, void* stream) {
  using namespace spx;
  if (y0 < 0 || y1 > h || w < 0) {
    set_error("weak_band: rows [%lld,%lld) outside image", (long long)y0, (long long)y1);
    return SPX_ERR_DIMENSION;
  }
  return launch_weak1(src, dst, h, w, y0, y1, as_stream(stream));
}

extern "C" int32_t spx_strict_fill(const int32_t* src, int32_t* dst, int64_t h, int64_t w,
                                   int64_t min_size, void* stream) {
  using namespace spx;
  if (h < 0 || w < 0) {
    set_error("strict_fill: bad shape");
    return SPX_ERR_DIMENSION;
  }
  return strict_fill_alloc(src, dst, h, w, min_size, as_stream(stream));
}
