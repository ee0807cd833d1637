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
// Components are labelled tile by tile in shared memory first (k_cc_local),
// joined across tile borders (k_cc_border) and resolved per pixel
// (k_cc_resolve, which also lists the components for the later passes).
#include <algorithm>
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
#ifndef SPX_WEAK_WG
#define SPX_WEAK_WG 128
#endif
#ifndef SPX_WEAK_HG
#define SPX_WEAK_HG 16
#endif
constexpr int WG = SPX_WEAK_WG, HG = SPX_WEAK_HG;  // 128x16 tiles: 21 KB smem, 0.19 ms per 256 C1 frames (32 rows: 0.22)
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

// The rule for pixels whose left and upper neighbours are in the image
// (interior tiles): an isolated pixel always adopts its left neighbour.
__device__ __forceinline__ int4 weak_rule4_inner(int4 v, int4 up, int4 dn, int lft, int rgt) {
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
    o[k] = keep ? c : L;
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
  // interior tiles (source window and output fully inside the image, the
  // common case) skip every bounds test and out-of-image mask
  const bool inner = vec && tx0 >= 8 && tx0 + WG + 8 <= w && ty0 >= 2 && ty0 + HG + 2 <= h &&
                     ty0 + HG <= y1;
  if (inner) {
    for (int i = tid; i < R0G * NG0; i += 256) {
      const int r = i / NG0, g = i - r * NG0;
      t0[r][g] = __ldg(reinterpret_cast<const int4*>(s + (long long)(ty0 - 2 + r) * w + tx0 - 8) + g);
    }
    __syncthreads();
    // (every pass-1 and pass-2 pixel of an inner tile has its left and upper
    // neighbours in the image: columns >= tx0 - 4 >= 4, rows >= ty0 - 1 >= 1)
    for (int i = tid; i < R1G * NG1; i += 256) {
      const int r = i / NG1, g = i - r * NG1;
      t1[r][g] = weak_rule4_inner(t0[r + 1][g + 1], t0[r][g + 1], t0[r + 2][g + 1],
                                  t0[r + 1][g].w, t0[r + 1][g + 2].x);
    }
    __syncthreads();
    for (int i = tid; i < HG * (WG / 4); i += 256) {
      const int r = i / (WG / 4), g = i - r * (WG / 4);
      *reinterpret_cast<int4*>(d + (long long)(ty0 + r) * w + tx0 + 4 * g) =
          weak_rule4_inner(t1[r + 1][g + 1], t1[r][g + 1], t1[r + 2][g + 1], t1[r + 1][g].w,
                           t1[r + 1][g + 2].x);
    }
    return;
  }
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

// Union-find over pixel indices with min-index roots (ECL-CC style): links
// only ever point to smaller indices, so concurrent path halving (each step
// re-points x at its grandparent) keeps every pointer valid.
__device__ __forceinline__ int32_t uf_find(int32_t* parent, int32_t x) {
  int32_t p = parent[x];
  while (p != x) {
    const int32_t g = parent[p];
    if (g != p) parent[x] = g;  // halve the path
    x = p;
    p = g;
  }
  return x;
}
// Read-only find, for the flatten pass: there every pixel also stores its
// root, and a concurrent halving store could replace a stored root with a
// mere ancestor.
__device__ __forceinline__ int32_t uf_root(const int32_t* parent, int32_t x) {
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

// Per-pixel kernels run on a (column blocks, rows, frames) grid: pixel
// (x, y) of frame f has global index f*h*w + y*w + x (< 2^31).
struct PixIdx {
  int x, y, f, i;  // i: global index
  bool in;
};
__device__ __forceinline__ PixIdx pix_idx(int h, int w) {
  PixIdx q;
  q.x = blockIdx.x * blockDim.x + threadIdx.x;
  q.y = blockIdx.y;
  q.f = blockIdx.z;
  q.in = q.x < w;
  q.i = (q.f * h + q.y) * w + q.x;
  return q;
}

// ---- component labelling ------------------------------------------------------
// (A) k_cc_local: one block per 64 x 16 tile labels the tile's components in
//     shared memory (union-find with min-index roots, then a flatten and the
//     component sizes) and writes every pixel's tile-local root as a global
//     index, the local root's count into `size`.  Row-major order inside a
//     tile is the frame's scan order restricted to it, so a local root is the
//     minimum global index of its piece.
// (B) k_cc_border: the tiles' bottom rows and right columns unite with the
//     neighbouring tiles (global min-index union-find over the local roots).
// (C) k_cc_resolve: every pixel's root, and each tile-local root adds its
//     count to its component's root (B's path halving may already have
//     re-pointed a local root, so (A) marks them by a non-zero count).
constexpr int CTW = 64, CTH = 16, CTN = CTW * CTH;

__device__ __forceinline__ int s_find(int* par, int x) {
  int p = par[x];
  while (p != x) {
    const int g = par[p];
    if (g != p) par[x] = g;
    x = p;
    p = g;
  }
  return x;
}
__device__ __forceinline__ void s_unite(int* par, int a, int b) {
  while (true) {
    a = s_find(par, a);
    b = s_find(par, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(par + b, a);
    if (old == b) return;
    b = old;
  }
}

__global__ void __launch_bounds__(256) k_cc_local(const int32_t* __restrict__ lab,
                                                  int32_t* __restrict__ parent,
                                                  int32_t* __restrict__ size, int h, int w) {
  __shared__ int t_lab[CTN];
  __shared__ int t_par[CTN];
  __shared__ int t_cnt[CTN];
  const int tx0 = blockIdx.x * CTW, ty0 = blockIdx.y * CTH;
  const int base = blockIdx.z * h * w;
  const int tw = min(CTW, w - tx0), th = min(CTH, h - ty0);
  for (int i = threadIdx.x; i < CTN; i += 256) {
    const int r = i / CTW, c = i - r * CTW;
    t_lab[i] = (r < th && c < tw) ? __ldg(lab + base + (ty0 + r) * w + tx0 + c) : 0;
    t_par[i] = i;
    t_cnt[i] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < CTN; i += 256) {
    const int r = i / CTW, c = i - r * CTW;
    if (r >= th || c >= tw) continue;
    const int v = t_lab[i];
    if (c + 1 < tw && t_lab[i + 1] == v) s_unite(t_par, i, i + 1);
    if (r + 1 < th && t_lab[i + CTW] == v) s_unite(t_par, i, i + CTW);
  }
  __syncthreads();
  int root[CTN / 256];
#pragma unroll
  for (int k = 0; k < CTN / 256; ++k) {
    const int i = threadIdx.x + 256 * k;
    int x = i, p = t_par[x];
    while (p != x) {  // read-only chase (no writers in this phase)
      x = p;
      p = t_par[x];
    }
    root[k] = x;
    const int r = i / CTW, c = i - r * CTW;
    if (r < th && c < tw) atomicAdd(t_cnt + x, 1);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < CTN / 256; ++k) {
    const int i = threadIdx.x + 256 * k;
    const int r = i / CTW, c = i - r * CTW;
    if (r >= th || c >= tw) continue;
    const int x = root[k];
    const int gi = base + (ty0 + r) * w + tx0 + c;
    parent[gi] = base + (ty0 + x / CTW) * w + tx0 + x % CTW;
    size[gi] = x == i ? t_cnt[i] : 0;  // > 0 marks the tile-local roots for (C)
  }
}

__global__ void __launch_bounds__(128) k_cc_border(const int32_t* __restrict__ lab,
                                                   int32_t* parent, int h, int w) {
  const int tx0 = blockIdx.x * CTW, ty0 = blockIdx.y * CTH;
  const int base = blockIdx.z * h * w;
  const int t = threadIdx.x;
  if (t < CTW) {  // bottom row: unite downwards
    const int x = tx0 + t, y = ty0 + CTH - 1;
    if (x < w && y + 1 < h) {
      const int gi = base + y * w + x;
      if (__ldg(lab + gi) == __ldg(lab + gi + w)) uf_unite(parent, gi, gi + w);
    }
  } else if (t < CTW + CTH) {  // right column: unite rightwards
    const int x = tx0 + CTW - 1, y = ty0 + (t - CTW);
    if (y < h && x + 1 < w) {
      const int gi = base + y * w + x;
      if (__ldg(lab + gi) == __ldg(lab + gi + 1)) uf_unite(parent, gi, gi + 1);
    }
  }
}

__global__ void k_cc_resolve(int32_t* parent, int32_t* size, int32_t* roots, int32_t* nroots,
                             int h, int w) {
  const PixIdx q = pix_idx(h, w);
  const int32_t r = q.in ? uf_root(parent, q.i) : -1;
  const bool root = q.in && r == q.i;
  if (q.in) {
    parent[q.i] = r;
    // a tile-local root (count > 0) that is not its component's root adds
    // its count there; only component roots receive adds, a root never adds
    const int32_t c = size[q.i];
    if (c > 0 && r != q.i) atomicAdd(size + r, c);
  }
  // compact list of the components (any order): one global atomic per block
  __shared__ int bcount, bbase;
  if (threadIdx.x == 0) bcount = 0;
  __syncthreads();
  const int slot = root ? atomicAdd(&bcount, 1) : 0;
  __syncthreads();
  if (threadIdx.x == 0) bbase = bcount ? atomicAdd(nroots, bcount) : 0;
  __syncthreads();
  if (root) roots[bbase + slot] = q.i;
}

// (over the component list; sizes are final once (C) has run)
__global__ void k_cc_first(const int32_t* __restrict__ lab, const int32_t* __restrict__ size,
                           const int32_t* __restrict__ roots, const int32_t* __restrict__ nroots,
                           int32_t* first, int hw, int64_t nlab, int64_t min_size) {
  const int n = *nroots;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int32_t i = roots[j];
    if (size[i] < min_size) continue;
    atomicMin(first + (i / hw) * nlab + lab[i], i);
  }
}

__global__ void k_cc_next(const int32_t* __restrict__ lab, const int32_t* __restrict__ parent,
                          const int32_t* __restrict__ size, const int32_t* __restrict__ first,
                          const int32_t* __restrict__ roots, const int32_t* __restrict__ nroots,
                          int32_t* nxt, int w, int hw, int64_t nlab, int64_t min_size) {
  const int n = *nroots;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int32_t i = roots[j];
    const int f = i / hw, base = f * hw;
    const int32_t v = lab[i];
    const bool keep = i == base ||
                      (size[i] >= min_size && first[f * nlab + v] == i && lab[base] != v);
    // absorbed: the root of the seed's left neighbour (up in column 0)
    const int x = (i - base) % w;
    nxt[i] = keep ? i : parent[x > 0 ? i - 1 : i - w];
  }
}

// Final value of each component: pointer jumping on nxt over the compact
// list of components (nxt[r] <- nxt[nxt[r]]), ceil(log2(h*w)) + 1 rounds --
// absorption chains never leave a frame and strictly decrease in seed index,
// so they are shorter than h*w -- after which nxt[r] is r's keeper.  Racing
// updates only ever shortcut to a later node of the same chain.  (On random
// noise frames nearly every component is a 1-2 pixel fragment and chains run
// to hundreds of links, which rules out per-component chain walking.)
// Round `round` records whether it changed anything in changed[round]; a
// round after one that changed nothing returns at once (converged).
#ifndef SPX_JU
#define SPX_JU 4
#endif
__global__ void k_cc_jump(const int32_t* __restrict__ roots, const int32_t* __restrict__ nroots,
                          int32_t* nxt, int32_t* changed, int round) {
  if (round > 0 && changed[round - 1] == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) changed[round] = 0;
    return;
  }
  const int n = *nroots;
  bool any = false;
  // four independent components per thread and step: their dependent
  // gathers (roots -> nxt -> nxt) are in flight together
  const int stride = gridDim.x * blockDim.x;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += SPX_JU * stride) {
    int32_t r[SPX_JU], a[SPX_JU], b[SPX_JU];
#pragma unroll
    for (int u = 0; u < SPX_JU; ++u) r[u] = j + u * stride < n ? roots[j + u * stride] : -1;
#pragma unroll
    for (int u = 0; u < SPX_JU; ++u) a[u] = r[u] >= 0 ? nxt[r[u]] : 0;
#pragma unroll
    for (int u = 0; u < SPX_JU; ++u) b[u] = r[u] >= 0 ? nxt[a[u]] : 0;
#pragma unroll
    for (int u = 0; u < SPX_JU; ++u)
      if (r[u] >= 0 && a[u] != b[u]) {
        nxt[r[u]] = b[u];
        any = true;
      }
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) changed[round] = 1;
}

__global__ void k_cc_write(const int32_t* __restrict__ lab, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ nxt, int32_t* __restrict__ dst, int h,
                           int w) {
  const PixIdx q = pix_idx(h, w);
  if (!q.in) return;
  dst[q.i] = lab[nxt[parent[q.i]]];
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

// scratch: parent, size, nxt (n each) and first (frames * nlab + kStrictExtra),
// all int32;
// src and dst must not overlap (dst holds the component list meanwhile).
static int launch_strict_chunk(const int32_t* src, int32_t* dst, int64_t h, int64_t w,
                               int frames, int64_t nlab, int64_t min_size, int32_t* parent,
                               int32_t* size, int32_t* nxt, int32_t* first, cudaStream_t st);

// Frames are independent: a batch whose pixel indices would overflow int32
// runs in chunks of whole frames (same buffers, offset by the chunk).
int launch_strict(const int32_t* src, int32_t* dst, int64_t h, int64_t w, int frames,
                  int64_t nlab, int64_t min_size, int32_t* parent, int32_t* size, int32_t* nxt,
                  int32_t* first, cudaStream_t st) {
  const int64_t hw = h * w;
  if (hw == 0 || frames <= 0) return SPX_OK;
  if (hw >= INT32_MAX) {
    set_error("strict_fill: %lld pixels per frame exceed the int32 component index",
              (long long)hw);
    return SPX_ERR_VALUE;
  }
  const int fc = (int)std::min<int64_t>(frames, (INT32_MAX - 1) / hw);
  for (int f0 = 0; f0 < frames; f0 += fc) {
    const int nf = std::min(fc, frames - f0);
    const int64_t o = (int64_t)f0 * hw;
    const int rc = launch_strict_chunk(src + o, dst + o, h, w, nf, nlab, min_size, parent + o,
                                       size + o, nxt + o, first, st);
    if (rc) return rc;
  }
  return SPX_OK;
}

static int launch_strict_chunk(const int32_t* src, int32_t* dst, int64_t h, int64_t w,
                               int frames, int64_t nlab, int64_t min_size, int32_t* parent,
                               int32_t* size, int32_t* nxt, int32_t* first, cudaStream_t st) {
  int64_t hw = h * w, n = hw * frames;
  if (n == 0) return SPX_OK;
  if (h > 65535 || frames > 65535) {
    set_error("strict_fill: at most 65535 rows and 65535 frames per launch");
    return SPX_ERR_VALUE;
  }
  const dim3 grid((unsigned)ceil_div(w, 256), (unsigned)h, (unsigned)frames);
  const int H = (int)h, W = (int)w;
  SPX_CUDA(cudaMemsetAsync(first, 0x7f, (size_t)(frames * nlab) * 4, st));
  // The component list lives in dst until the final write; its length and
  // the per-round change flags in the kStrictExtra ints after `first`.
  int32_t* nroots = first + frames * nlab;
  int32_t* changed = nroots + 1;
  SPX_CUDA(cudaMemsetAsync(nroots, 0, kStrictExtra * sizeof(int32_t), st));
  const dim3 tiles((unsigned)ceil_div(w, CTW), (unsigned)ceil_div(h, CTH), (unsigned)frames);
  k_cc_local<<<tiles, 256, 0, st>>>(src, parent, size, H, W);
  k_cc_border<<<tiles, 128, 0, st>>>(src, parent, H, W);
  k_cc_resolve<<<grid, 256, 0, st>>>(parent, size, dst, nroots, H, W);
  const unsigned lb = (unsigned)std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 16);
  k_cc_first<<<lb, 256, 0, st>>>(src, size, dst, nroots, first, (int)hw, nlab, min_size);
  k_cc_next<<<lb, 256, 0, st>>>(src, parent, size, first, dst, nroots, nxt, W, (int)hw, nlab,
                                min_size);
  int rounds = 1;
  while ((1ll << rounds) < hw) ++rounds;
  const unsigned jb = (unsigned)std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 8);
  for (int r = 0; r <= rounds; ++r) k_cc_jump<<<jb, 256, 0, st>>>(dst, nroots, nxt, changed, r);
  k_cc_write<<<grid, 256, 0, st>>>(src, parent, nxt, dst, H, W);
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
  SPX_CUDA(cudaMallocAsync(&first, (nlab + kStrictExtra) * 4, st));
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
