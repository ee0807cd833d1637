// centers.cu -- cluster-centre seeding, gradient perturbation, centre update
// reduction and the early-stop shift.  One thread per cluster: these are
// O(K) stages (K = 1,200 clusters per 640x480 frame) whose cost is a few
// reads per cluster; batching frames gives the parallelism.
#include <algorithm>

#include <functional>
#include <vector>

#include "spx_internal.cuh"

namespace spx {

// _core.pyx:110-120 _gradient, exact binary64.
__device__ __forceinline__ double gradient_at(const LabView& im, int64_t x, int64_t y) {
  double dl = dsub((double)im.get(y, x + 1, 0), (double)im.get(y, x - 1, 0));
  double da = dsub((double)im.get(y, x + 1, 1), (double)im.get(y, x - 1, 1));
  double db = dsub((double)im.get(y, x + 1, 2), (double)im.get(y, x - 1, 2));
  double gx = dadd(dadd(dmul(dl, dl), dmul(da, da)), dmul(db, db));
  dl = dsub((double)im.get(y + 1, x, 0), (double)im.get(y - 1, x, 0));
  da = dsub((double)im.get(y + 1, x, 1), (double)im.get(y - 1, x, 1));
  db = dsub((double)im.get(y + 1, x, 2), (double)im.get(y - 1, x, 2));
  double gy = dadd(dadd(dmul(dl, dl), dmul(da, da)), dmul(db, db));
  return dadd(gx, gy);
}

// _core.pyx:123-156 perturb for one centre (in place).
__device__ __forceinline__ void perturb_one(const LabView& im, int64_t h, int64_t w, double* cxy,
                                            double* clab) {
  int64_t ix = (int64_t)cxy[0], iy = (int64_t)cxy[1];
  if (ix < 1 || ix > w - 2 || iy < 1 || iy > h - 2) return;
  double best = gradient_at(im, ix, iy);
  int64_t bx = ix, by = iy;
  for (int dy = -1; dy < 2; ++dy)
    for (int dx = -1; dx < 2; ++dx) {
      if (dx == 0 && dy == 0) continue;
      int64_t nx = ix + dx, ny = iy + dy;
      if (nx < 1 || nx > w - 2 || ny < 1 || ny > h - 2) continue;
      double g = gradient_at(im, nx, ny);
      if (g < best) {
        best = g;
        bx = nx;
        by = ny;
      }
    }
  cxy[0] = (double)bx;
  cxy[1] = (double)by;
  clab[0] = im.get(by, bx, 0);
  clab[1] = im.get(by, bx, 1);
  clab[2] = im.get(by, bx, 2);
}

// _core.pyx:86-107 (+ optional perturb).  Clusters [k0,k1) of each of
// `frames` frames; `planar` selects the engine's [3][H][W] Lab layout.
// Row strips: the buffer holds local rows (hl of them, starting at global
// cell row row_off); h is the GLOBAL image height and all coordinates are
// global.  Whole frames: hl == h, row_off == 0.
__global__ void k_init(const float* __restrict__ img, int64_t h, int64_t w, int64_t s,
                       int64_t ns_c, double* __restrict__ cxy, double* __restrict__ clab,
                       int64_t k0, int64_t k1, int64_t k_stride, int frames, int perturb,
                       int do_init, int planar, int64_t hl, int64_t row_off, CRec* rec,
                       ClusterAcc* acc, int32_t* zero_ints, int n_zero) {
  int64_t nk = k1 - k0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_zero) zero_ints[i] = 0;
  if (i >= nk * frames) return;
  int64_t f = i / nk;
  int64_t k = k0 + i % nk;
  const int64_t pst = planar ? plane_of(hl * w) : hl * w;
  LabView im{img + f * pst * 3, w, pst, planar != 0};
  im.yoff = row_off * s;
  double* xy = cxy + (f * k_stride + k) * 2;
  double* lab = clab + (f * k_stride + k) * 3;
  if (do_init) {
    int64_t r = k / ns_c + row_off, c = k % ns_c;
    int64_t ix = c * s + s / 2;
    if (ix > w - 1) ix = w - 1;
    int64_t iy = r * s + s / 2;
    if (iy > h - 1) iy = h - 1;
    xy[0] = (double)ix;
    xy[1] = (double)iy;
    lab[0] = im.get(iy, ix, 0);
    lab[1] = im.get(iy, ix, 1);
    lab[2] = im.get(iy, ix, 2);
  }
  if (perturb) perturb_one(im, h, w, xy, lab);
  if (rec)
    rec[f * k_stride + k] = make_record(xy[0], xy[1], lab[0], lab[1], lab[2],
                                        (int)(k / ns_c + row_off), (int)(k % ns_c), (int)s);
  if (acc) acc[f * k_stride + k] = ClusterAcc{};
}

int launch_init(const float* img, int64_t h, int64_t w, int64_t s, int64_t ns_c, double* cxy,
                double* clab, int64_t k0, int64_t k1, int64_t k_stride, int frames, int perturb,
                int do_init, cudaStream_t st, int planar, int64_t hl, int64_t row_off,
                CRec* rec, ClusterAcc* acc, int32_t* zero_ints, int n_zero) {
  int64_t n = std::max<int64_t>((k1 - k0) * frames, n_zero);
  if (n <= 0) return SPX_OK;
  if (hl < 0) hl = h;
  k_init<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(img, h, w, s, ns_c, cxy, clab, k0, k1,
                                                     k_stride, frames, perturb, do_init, planar,
                                                     hl, row_off, rec, acc, zero_ints, n_zero);
  SPX_LAUNCH_CHECK("k_init");
  return SPX_OK;
}

// _core.pyx:288-325 reduce_range: pairwise tree over strips, then divide.
// Clusters [k0,k1) of each frame; frames whose done flag is set are skipped.
__global__ void k_reduce(double* __restrict__ slab, int64_t n_bl, const double* __restrict__ prev_xy,
                         const double* __restrict__ prev_lab, double* __restrict__ out_xy,
                         double* __restrict__ out_lab, int64_t* __restrict__ out_counts,
                         int64_t k0, int64_t k1, int64_t k_stride, int frames,
                         const int32_t* __restrict__ done) {
  int64_t nk = k1 - k0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nk * frames) return;
  int64_t f = i / nk;
  if (done && done[f]) return;
  int64_t k = f * k_stride + k0 + i % nk;
  double* sk = slab + k * n_bl * 6;
  int64_t m = n_bl;
  while (m > 1) {
    int64_t half = m >> 1;
    for (int64_t j = 0; j < half; ++j)
      for (int comp = 0; comp < 6; ++comp)
        sk[j * 6 + comp] = dadd(sk[2 * j * 6 + comp], sk[(2 * j + 1) * 6 + comp]);
    if (m & 1)
      for (int comp = 0; comp < 6; ++comp) sk[half * 6 + comp] = sk[(m - 1) * 6 + comp];
    m = half + (m & 1);
  }
  double cnt = sk[5];
  if (cnt > 0.0) {
    out_lab[k * 3] = ddiv(sk[0], cnt);
    out_lab[k * 3 + 1] = ddiv(sk[1], cnt);
    out_lab[k * 3 + 2] = ddiv(sk[2], cnt);
    out_xy[k * 2] = ddiv(sk[3], cnt);
    out_xy[k * 2 + 1] = ddiv(sk[4], cnt);
  } else {
    out_lab[k * 3] = prev_lab[k * 3];
    out_lab[k * 3 + 1] = prev_lab[k * 3 + 1];
    out_lab[k * 3 + 2] = prev_lab[k * 3 + 2];
    out_xy[k * 2] = prev_xy[k * 2];
    out_xy[k * 2 + 1] = prev_xy[k * 2 + 1];
  }
  out_counts[k] = (int64_t)cnt;
}

int launch_reduce(double* slab, int64_t n_bl, const double* prev_xy, const double* prev_lab,
                  double* out_xy, double* out_lab, int64_t* out_counts, int64_t k0, int64_t k1,
                  int64_t k_stride, int frames, const int32_t* done, cudaStream_t st) {
  int64_t n = (k1 - k0) * frames;
  if (n <= 0) return SPX_OK;
  k_reduce<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(slab, n_bl, prev_xy, prev_lab, out_xy,
                                                       out_lab, out_counts, k0, k1, k_stride,
                                                       frames, done);
  SPX_LAUNCH_CHECK("k_reduce");
  return SPX_OK;
}

// numpy pairwise summation of |new - old| (engine.py:196; numpy
// loops_utils.h.src pairwise_sum: <8 sequential, <=128 eight accumulators,
// else split at n/2 rounded down to a multiple of 8).
__device__ double pairwise_absdiff(const double* a, const double* b, int64_t n) {
  // Iterative post-order traversal of the recursion tree (depth <= 64).
  struct Frame { int64_t off, n; int state; double left; };
  Frame stack[64];
  int top = 0;
  stack[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (top >= 0) {
    Frame& fr = stack[top];
    if (fr.n <= 128) {
      double res;
      const double* x = a + fr.off;
      const double* y = b + fr.off;
      if (fr.n < 8) {
        res = 0.0;
        for (int64_t i = 0; i < fr.n; ++i) res = dadd(res, fabs(dsub(x[i], y[i])));
      } else {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = fabs(dsub(x[j], y[j]));
        int64_t i;
        for (i = 8; i < fr.n - (fr.n % 8); i += 8)
          for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], fabs(dsub(x[i + j], y[i + j])));
        res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
        for (; i < fr.n; ++i) res = dadd(res, fabs(dsub(x[i], y[i])));
      }
      ret = res;
      --top;
      continue;
    }
    int64_t n2 = fr.n / 2;
    n2 -= n2 % 8;
    if (fr.state == 0) {
      fr.state = 1;
      stack[top + 1] = {fr.off, n2, 0, 0.0};
      ++top;
    } else if (fr.state == 1) {
      fr.left = ret;
      fr.state = 2;
      stack[top + 1] = {fr.off + n2, fr.n - n2, 0, 0.0};
      ++top;
    } else {
      ret = dadd(fr.left, ret);
      --top;
    }
  }
  return ret;
}

// Per-frame shift; sets done[f] when shift < threshold (engine.py:196-200).
__global__ void k_shift(const double* __restrict__ new_xy, const double* __restrict__ old_xy,
                        int64_t k, int frames, double* __restrict__ shift_out,
                        int32_t* __restrict__ done, int32_t* __restrict__ passes,
                        double threshold) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= frames) return;
  if (done && done[f]) return;
  double sh = pairwise_absdiff(new_xy + (int64_t)f * k * 2, old_xy + (int64_t)f * k * 2, 2 * k);
  if (shift_out) shift_out[f] = sh;
  if (passes) passes[f] += 1;
  // The flag takes effect after the association that follows (engine.py:197-200).
  if (done && threshold >= 0.0 && sh < threshold) done[f] = 2;
}

// ---- the same sum with the recursion tree evaluated in parallel -------------
// numpy's pairwise_sum is a fixed binary tree over n values (leaves: the
// <= 128-element blocks summed with eight accumulators; inner nodes:
// left + right).  ShiftTree builds that tree once per n on the host; the
// kernel sums every leaf in parallel, then evaluates the inner nodes level by
// level (height 1 first: nodes of equal height are independent), one block
// per frame -- the same additions in the same association as the recursion,
// so bit-identical to numpy (tests: engine early stop vs the oracle).

// Sum of the n values x[i] (or |x[i] - y[i]| when y != null) of one leaf.
__device__ double leaf_sum(const double* x, const double* y, int n) {
  auto v = [&](int i) { return y ? fabs(dsub(x[i], y[i])) : x[i]; };
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = dadd(res, v(i));
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = v(j);
  int i;
  for (i = 8; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], v(i + j));
  double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; i < n; ++i) res = dadd(res, v(i));
  return res;
}

struct TreeDev {
  const long long* leaf_off;
  const int* leaf_n;
  const int3* inner;      // (dst, left, right) value indices, by height
  const int* lev_start;   // nlev + 1 offsets into inner
  int nleaf, ninner, nlev, nvals, root;
};

__global__ void __launch_bounds__(256) k_shift_tree(const double* __restrict__ x,
                                                    const double* __restrict__ y,
                                                    int64_t frame_stride, TreeDev t,
                                                    double* __restrict__ scratch,
                                                    double* __restrict__ shift_out,
                                                    int32_t* __restrict__ done,
                                                    int32_t* __restrict__ passes,
                                                    double threshold) {
  const int f = blockIdx.x;
  if (done && done[f]) return;  // block-uniform
  const double* xf = x + (int64_t)f * frame_stride;
  const double* yf = y ? y + (int64_t)f * frame_stride : nullptr;
  double* vals = scratch + (int64_t)f * t.nvals;
  for (int i = threadIdx.x; i < t.nleaf; i += blockDim.x)
    vals[i] = leaf_sum(xf + t.leaf_off[i], yf ? yf + t.leaf_off[i] : nullptr, t.leaf_n[i]);
  __syncthreads();
  for (int l = 0; l < t.nlev; ++l) {
    for (int j = t.lev_start[l] + threadIdx.x; j < t.lev_start[l + 1]; j += blockDim.x) {
      const int3 q = t.inner[j];
      vals[q.x] = dadd(vals[q.y], vals[q.z]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double sh = vals[t.root];
    if (shift_out) shift_out[f] = sh;
    if (passes) passes[f] += 1;
    if (done && threshold >= 0.0 && sh < threshold) done[f] = 2;
  }
}

void ShiftTree::release() {
  for (void* q : {(void*)leaf_off, (void*)leaf_n, (void*)inner, (void*)lev_start, (void*)scratch})
    if (q) cudaFree(q);
  leaf_off = nullptr, leaf_n = nullptr, inner = nullptr, lev_start = nullptr, scratch = nullptr;
  n = -1;
}

ShiftTree::~ShiftTree() { release(); }

int ShiftTree::build(int64_t n_values, int max_frames) {
  if (n == n_values && frames >= max_frames) return SPX_OK;
  release();
  std::vector<long long> loff;
  std::vector<int> ln;
  struct Node { int dst, l, r, h; };
  std::vector<Node> nodes;
  // returns (value index, height); inner value indices are assigned after
  // the leaves are counted, so record them as negative placeholders first
  std::function<std::pair<int, int>(int64_t, int64_t)> rec = [&](int64_t off, int64_t m) {
    if (m <= 128) {
      loff.push_back(off);
      ln.push_back((int)m);
      return std::make_pair((int)loff.size() - 1, 0);
    }
    int64_t m2 = m / 2;
    m2 -= m2 % 8;
    auto L = rec(off, m2);
    auto R = rec(off + m2, m - m2);
    nodes.push_back({-(int)nodes.size() - 1, L.first, R.first, 1 + std::max(L.second, R.second)});
    return std::make_pair(nodes.back().dst, nodes.back().h);
  };
  const auto top = rec(0, std::max<int64_t>(n_values, 0));
  const int nl = (int)loff.size();
  auto fix = [&](int v) { return v < 0 ? nl + (-v - 1) : v; };
  int hmax = 0;
  for (auto& q : nodes) hmax = std::max(hmax, q.h);
  std::vector<int3> in;
  std::vector<int> ls(1, 0);
  for (int h = 1; h <= hmax; ++h) {
    for (auto& q : nodes)
      if (q.h == h) in.push_back(make_int3(fix(q.dst), fix(q.l), fix(q.r)));
    ls.push_back((int)in.size());
  }
  n = n_values;
  frames = std::max(1, max_frames);
  nleaf = nl;
  ninner = (int)in.size();
  nlev = hmax;
  nvals = nl + ninner;
  root = fix(top.first);
  SPX_CUDA(cudaMalloc(&leaf_off, nl * sizeof(long long)));
  SPX_CUDA(cudaMalloc(&leaf_n, nl * sizeof(int)));
  SPX_CUDA(cudaMalloc(&inner, std::max<size_t>(1, in.size()) * sizeof(int3)));
  SPX_CUDA(cudaMalloc(&lev_start, ls.size() * sizeof(int)));
  SPX_CUDA(cudaMalloc(&scratch, (size_t)frames * nvals * sizeof(double)));
  SPX_CUDA(cudaMemcpy(leaf_off, loff.data(), nl * sizeof(long long), cudaMemcpyHostToDevice));
  SPX_CUDA(cudaMemcpy(leaf_n, ln.data(), nl * sizeof(int), cudaMemcpyHostToDevice));
  if (!in.empty())
    SPX_CUDA(cudaMemcpy(inner, in.data(), in.size() * sizeof(int3), cudaMemcpyHostToDevice));
  SPX_CUDA(cudaMemcpy(lev_start, ls.data(), ls.size() * sizeof(int), cudaMemcpyHostToDevice));
  return SPX_OK;
}

int ShiftTree::launch(const double* x, const double* y, int64_t frame_stride, int nframes,
                      double* shift_out, int32_t* done, int32_t* passes, double threshold,
                      cudaStream_t st) {
  if (nframes > frames) {
    set_error("shift tree built for %d frames, %d requested", frames, nframes);
    return SPX_ERR_VALUE;
  }
  if (nframes <= 0) return SPX_OK;
  TreeDev t{leaf_off, leaf_n, inner, lev_start, nleaf, ninner, nlev, nvals, root};
  k_shift_tree<<<(unsigned)nframes, 256, 0, st>>>(x, y, frame_stride, t, scratch, shift_out, done,
                                                  passes, threshold);
  SPX_LAUNCH_CHECK("k_shift_tree");
  return SPX_OK;
}

// done: 0 running, 2 = stops after the next association, 1 = stopped.
__global__ void k_commit_done(int32_t* done, int frames) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < frames && done[f] == 2) done[f] = 1;
}

int launch_shift(const double* new_xy, const double* old_xy, int64_t k, int frames,
                 double* shift_out, int32_t* done, int32_t* passes, double threshold,
                 cudaStream_t st) {
  k_shift<<<(unsigned)ceil_div(frames, 64), 64, 0, st>>>(new_xy, old_xy, k, frames, shift_out,
                                                         done, passes, threshold);
  SPX_LAUNCH_CHECK("k_shift");
  return SPX_OK;
}

int launch_commit_done(int32_t* done, int frames, cudaStream_t st) {
  k_commit_done<<<(unsigned)ceil_div(frames, 64), 64, 0, st>>>(done, frames);
  SPX_LAUNCH_CHECK("k_commit_done");
  return SPX_OK;
}

}  // namespace spx

using namespace spx;

extern "C" int32_t spx_init_centers_range(const float* img, int64_t h, int64_t w, int64_t s,
                                          int64_t ns_c, double* cxy, double* clab, int64_t k0,
                                          int64_t k1, void* stream) {
  if (s < 1 || ns_c < 1 || k0 < 0) {
    set_error("init_centers_range: bad grid (s=%lld ns_c=%lld)", (long long)s, (long long)ns_c);
    return SPX_ERR_VALUE;
  }
  return launch_init(img, h, w, s, ns_c, cxy, clab, k0, k1, 0, 1, 0, 1, as_stream(stream), 0, -1, 0);
}

extern "C" int32_t spx_perturb_range(const float* img, int64_t h, int64_t w, double* cxy,
                                     double* clab, int64_t k0, int64_t k1, void* stream) {
  if (k0 < 0) {
    set_error("perturb_range: negative cluster index");
    return SPX_ERR_VALUE;
  }
  return launch_init(img, h, w, 1, 1, cxy, clab, k0, k1, 0, 1, 1, 0, as_stream(stream), 0, -1, 0);
}

extern "C" int32_t spx_reduce_range(double* slab, int64_t n_bl, const double* prev_xy,
                                    const double* prev_lab, double* out_xy, double* out_lab,
                                    int64_t* out_counts, int64_t k0, int64_t k1, void* stream) {
  if (n_bl < 1 || k0 < 0) {
    set_error("reduce_range: n_bl must be >= 1");
    return SPX_ERR_VALUE;
  }
  return launch_reduce(slab, n_bl, prev_xy, prev_lab, out_xy, out_lab, out_counts, k0, k1, 0, 1,
                       nullptr, as_stream(stream));
}

extern "C" int32_t spx_center_shift(const double* new_xy, const double* old_xy, int64_t k,
                                    double* out_dev, void* stream) {
  if (k < 0) {
    set_error("center_shift: negative cluster count");
    return SPX_ERR_VALUE;
  }
  // per-call tree (the API form; the engine keeps its tree)
  ShiftTree t;
  int rc = t.build(2 * k, 1);
  if (rc) return rc;
  rc = t.launch(new_xy, old_xy, 0, 1, out_dev, nullptr, nullptr, -1.0, as_stream(stream));
  if (rc) return rc;
  SPX_CUDA(cudaStreamSynchronize(as_stream(stream)));  // the tree is freed on return
  return SPX_OK;
}

extern "C" int32_t spx_pairwise_sum(const double* x, int64_t n, double* out_dev, void* stream) {
  if (n < 0) {
    set_error("pairwise_sum: negative length");
    return SPX_ERR_VALUE;
  }
  ShiftTree t;
  int rc = t.build(n, 1);
  if (rc) return rc;
  rc = t.launch(x, nullptr, 0, 1, out_dev, nullptr, nullptr, -1.0, as_stream(stream));
  if (rc) return rc;
  SPX_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return SPX_OK;
}
