// strips.cu -- row-strip decomposition of one large image (SURVEY.md §8(e),
// config C5: 16384^2 split across GPUs).
//
// Rank r owns whole cell rows [lo, hi) of the global grid, hence the clusters
// of those rows and the pixel rows [lo*S, min(hi*S, H)).  Its buffers cover a
// LOCAL window of one extra cell row above and below (clipped at the image):
//   * association of own pixels needs the centres of the neighbouring cell
//     row -> halo CENTRES are received after every update;
//   * own pixels add to the accumulators of the neighbours' boundary
//     clusters -> those boundary-cluster PARTIAL SUMS are sent to the owner,
//     which adds them to its own (order-free and exact under the certified-sum
//     condition, see cell.cu; x / y / count are integers);
//   * the exact fallback for a flagged boundary cluster and the final weak
//     connectivity read S rows of the neighbour's labels -> halo LABEL rows;
//   * the halo RGB rows are part of the rank's input, so Lab needs no
//     exchange.
// Each exchange is a pack (device kernel / copies into a contiguous send
// buffer) + transport (the host: NCCL send/recv between ranks, or plain
// device copies when several strips share one process) + unpack.  The
// transported bytes per iteration and neighbour are ns_c * 40 B of centres,
// ns_c * 48 B of partial sums and S * W * 4 B of labels.  Results are
// bit-identical to the single-GPU engine for any strip count.
#include <algorithm>
#include <cstring>

#include "spx_internal.cuh"

namespace spx {
int launch_convert(const uint8_t*, float*, int64_t, int64_t, int, cudaStream_t, int64_t, int64_t,
                   float);
int launch_records(const double*, const double*, CRec*, int64_t, int64_t, int64_t, int,
                   cudaStream_t, int64_t, int64_t, int64_t);
int launch_weak2(const int32_t*, int32_t*, int64_t, int64_t, int, cudaStream_t, int64_t, int64_t);
bool cell_path_ok(int64_t, int64_t, int64_t, int64_t);

namespace {

// dst[i] += src[i] for n accumulators (integer fields added as integers).
__global__ void k_absdiff(const double* __restrict__ a, const double* __restrict__ b,
                          double* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fabs(dsub(a[i], b[i]));
}

__global__ void k_add_acc(ClusterAcc* __restrict__ dst, const ClusterAcc* __restrict__ src, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const ClusterAcc a = src[i];
  ClusterAcc& d = dst[i];
  d.s[0] = dadd(d.s[0], a.s[0]);
  d.s[1] = dadd(d.s[1], a.s[1]);
  d.s[2] = dadd(d.s[2], a.s[2]);
  d.sx += a.sx;
  d.sy += a.sy;
  d.cf += a.cf;
}

}  // namespace

struct Strip {
  spx_settings g;            // global settings
  int64_t lo = 0, hi = 0;    // own cell rows (global)
  int64_t rl0 = 0, nrl = 0;  // local grid: global row of local row 0, local row count
  int64_t own0 = 0, own1 = 0;    // own rows in the local grid
  int64_t y0 = 0, hl = 0;        // local pixel rows: global row of row 0, count
  int64_t oy0 = 0, oy1 = 0;      // own pixel rows (local)
  int64_t K = 0, n_bl = 0;
  int device = 0;
  double xy_weight = 0.0;
  int cur = 0;
  float* lab = nullptr;
  int32_t* labels = nullptr;
  int32_t* out = nullptr;
  double* cxy[2] = {nullptr, nullptr};
  double* clab[2] = {nullptr, nullptr};
  CRec* rec = nullptr;
  ClusterAcc* acc = nullptr;
  int32_t* worklist = nullptr;
  int64_t* counts = nullptr;

  ~Strip() {
    cudaSetDevice(device);
    for (void* q : {(void*)lab, (void*)labels, (void*)out, (void*)cxy[0], (void*)cxy[1],
                    (void*)clab[0], (void*)clab[1], (void*)rec, (void*)acc, (void*)worklist,
                    (void*)counts})
      if (q) cudaFree(q);
  }

  bool has_up() const { return lo > 0; }
  bool has_down() const { return hi < g.ns_r; }

  int init(const spx_settings& st, int64_t l, int64_t h_, int dev) {
    g = st;
    lo = l;
    hi = h_;
    device = dev;
    SPX_CUDA(cudaSetDevice(dev));
    rl0 = std::max<int64_t>(lo - 1, 0);
    nrl = std::min<int64_t>(hi + 1, g.ns_r) - rl0;
    own0 = lo - rl0;
    own1 = hi - rl0;
    y0 = rl0 * g.s;
    hl = std::min<int64_t>((rl0 + nrl) * g.s, g.height) - y0;
    oy0 = lo * g.s - y0;
    oy1 = std::min<int64_t>(hi * g.s, g.height) - y0;
    K = nrl * g.ns_c;
    n_bl = ceil_div(3 * g.s, g.tile_len);
    xy_weight = g.compactness / (double)g.s;
    const int64_t hw = hl * g.width;
    SPX_CUDA(cudaMalloc(&lab, plane_of(hw) * 3 * sizeof(float)));
    SPX_CUDA(cudaMalloc(&labels, hw * sizeof(int32_t)));
    SPX_CUDA(cudaMalloc(&out, hw * sizeof(int32_t)));
    SPX_CUDA(cudaMemset(labels, 0xff, hw * sizeof(int32_t)));
    for (int i = 0; i < 2; ++i) {
      SPX_CUDA(cudaMalloc(&cxy[i], K * 2 * sizeof(double)));
      SPX_CUDA(cudaMalloc(&clab[i], K * 3 * sizeof(double)));
      SPX_CUDA(cudaMemset(cxy[i], 0, K * 2 * sizeof(double)));
      SPX_CUDA(cudaMemset(clab[i], 0, K * 3 * sizeof(double)));
    }
    SPX_CUDA(cudaMalloc(&rec, K * sizeof(CRec)));
    SPX_CUDA(cudaMalloc(&acc, K * sizeof(ClusterAcc)));
    SPX_CUDA(cudaMemset(acc, 0, K * sizeof(ClusterAcc)));
    SPX_CUDA(cudaMalloc(&worklist, (K + 1) * sizeof(int32_t)));
    SPX_CUDA(cudaMalloc(&counts, K * sizeof(int64_t)));
    SPX_CUDA(cudaMemset(counts, 0, K * sizeof(int64_t)));
    return SPX_OK;
  }

  // convert the local window (own + halo pixel rows), seed own clusters
  int begin(const uint8_t* rgb_local, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t hw = hl * g.width;
    int rc = launch_convert(rgb_local, lab, 0, hw, g.color_space, s, hw, g.s, -1.f);
    if (rc) return rc;
    cur = 0;
    const int64_t k0 = own0 * g.ns_c, k1 = own1 * g.ns_c;
    if ((rc = launch_init(lab, g.height, g.width, g.s, g.ns_c, cxy[0], clab[0], k0, k1, K, 1, 0, 1,
                          s, 1, hl, rl0)))
      return rc;
    if (g.perturb &&
        (rc = launch_init(lab, g.height, g.width, g.s, g.ns_c, cxy[0], clab[0], k0, k1, K, 1, 1, 0,
                          s, 1, hl, rl0)))
      return rc;
    SPX_CUDA(cudaMemsetAsync(acc, 0, K * sizeof(ClusterAcc), s));
    return launch_records(cxy[0], clab[0], rec, nrl, g.ns_c, g.s, 1, s, k0, k1, rl0);
  }

  // Own cell rows split for overlapping the exchanges: the boundary rows
  // (own0 with an upper neighbour, own1 - 1 with a lower one) are the only
  // ones whose association reads halo centres and whose pixels contribute to
  // halo clusters / label halos; the interior rows need nothing from the
  // neighbours.  part: 0 all own rows, 1 interior, 2 boundary.
  void rows_of(int part, int64_t r[4]) const {  // up to two ranges [r0,r1), [r2,r3)
    const int64_t up = has_up() ? 1 : 0, dn = has_down() ? 1 : 0;
    const int64_t i0 = std::min(own0 + up, own1), i1 = std::max(i0, own1 - dn);
    r[0] = r[1] = r[2] = r[3] = 0;
    if (part == 0) {
      r[0] = own0, r[1] = own1;
    } else if (part == 1) {
      r[0] = i0, r[1] = i1;
    } else {
      r[0] = own0, r[1] = i0;  // top boundary row (if any)
      r[2] = std::max(i1, i0), r[3] = own1;
      if (r[1] >= r[2]) r[1] = r[3], r[2] = r[3] = 0;  // adjacent: one range
    }
  }

  int associate(bool with_update, int part, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    int64_t r[4];
    rows_of(part, r);
    for (int i = 0; i < 4; i += 2) {
      if (r[i + 1] <= r[i]) continue;
      const int rc = launch_cell(lab, cxy[cur], clab[cur], rec, labels, acc, nullptr, hl, g.width,
                                 g.s, nrl, g.ns_c, xy_weight, 1, with_update, s, r[i], r[i + 1],
                                 rl0);
      if (rc) return rc;
    }
    return SPX_OK;
  }

  // part 0: the whole update; 1: interior clusters (before the neighbours'
  // partial sums arrive); 2: boundary clusters, then the exact fallback over
  // every flagged cluster of this iteration (needs the label halos).
  int update(int part, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int nxt = cur ^ 1;
    int64_t r[4];
    rows_of(part, r);
    int rc;
    auto reduce = [&](int64_t a, int64_t b, int mode) {
      return launch_reduce_cells(acc, lab, labels, cxy[cur], clab[cur], cxy[nxt], clab[nxt],
                                 counts, rec, nullptr, worklist, worklist + K, hl, g.width, g.s,
                                 nrl, g.ns_c, g.tile_len, 1, s, a, b, rl0, mode);
    };
    if (part == 0) {
      rc = reduce(own0, own1, kReduceAndExact);
    } else if (part == 1) {
      rc = reduce(r[0], r[1], kReduceAppendFirst);  // zeroes the count even if empty
    } else if (r[1] > r[0] && r[3] > r[2]) {
      rc = reduce(r[0], r[1], kReduceAppend);
      if (!rc) rc = reduce(r[2], r[3], kReduceAppendLast);
    } else if (r[1] > r[0] || r[3] > r[2]) {
      rc = r[1] > r[0] ? reduce(r[0], r[1], kReduceAppendLast) : reduce(r[2], r[3], kReduceAppendLast);
    } else {  // no neighbours: the interior part reduced every own cluster
      rc = reduce(own0, own1, kExactOnly);
    }
    if (rc) return rc;
    if (part != 1) cur = nxt;  // halo centres of the new buffer arrive by exchange
    return SPX_OK;
  }

  // |new - old| of the own clusters' centres (x, y per cluster) after an
  // update, for the early-stop shift over all clusters (engine.py:196).
  int shift_local(double* out, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t c = g.ns_c, no = (own1 - own0) * c;
    k_absdiff<<<(unsigned)ceil_div(std::max<int64_t>(2 * no, 1), 256), 256, 0, s>>>(
        cxy[cur] + own0 * c * 2, cxy[cur ^ 1] + own0 * c * 2, out, 2 * no);
    SPX_LAUNCH_CHECK("k_absdiff");
    return SPX_OK;
  }

  // ---- exchange buffers ----------------------------------------------------
  // centres: ns_c * (2 + 3) doubles = cxy row then clab row
  int pack_centres(double* up, double* down, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t c = g.ns_c;
    if (up && has_up()) {
      SPX_CUDA(cudaMemcpyAsync(up, cxy[cur] + own0 * c * 2, c * 16, cudaMemcpyDeviceToDevice, s));
      SPX_CUDA(cudaMemcpyAsync(up + 2 * c, clab[cur] + own0 * c * 3, c * 24,
                               cudaMemcpyDeviceToDevice, s));
    }
    if (down && has_down()) {
      SPX_CUDA(cudaMemcpyAsync(down, cxy[cur] + (own1 - 1) * c * 2, c * 16,
                               cudaMemcpyDeviceToDevice, s));
      SPX_CUDA(cudaMemcpyAsync(down + 2 * c, clab[cur] + (own1 - 1) * c * 3, c * 24,
                               cudaMemcpyDeviceToDevice, s));
    }
    return SPX_OK;
  }
  // from_up: the upper neighbour's bottom own row -> my local row own0 - 1
  int unpack_centres(const double* from_up, const double* from_down, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t c = g.ns_c;
    int rc;
    if (from_up && has_up()) {
      const int64_t r = own0 - 1;
      SPX_CUDA(cudaMemcpyAsync(cxy[cur] + r * c * 2, from_up, c * 16, cudaMemcpyDeviceToDevice, s));
      SPX_CUDA(cudaMemcpyAsync(clab[cur] + r * c * 3, from_up + 2 * c, c * 24,
                               cudaMemcpyDeviceToDevice, s));
      if ((rc = launch_records(cxy[cur], clab[cur], rec, nrl, c, g.s, 1, s, r * c, (r + 1) * c, rl0)))
        return rc;
    }
    if (from_down && has_down()) {
      const int64_t r = own1;
      SPX_CUDA(cudaMemcpyAsync(cxy[cur] + r * c * 2, from_down, c * 16, cudaMemcpyDeviceToDevice,
                               s));
      SPX_CUDA(cudaMemcpyAsync(clab[cur] + r * c * 3, from_down + 2 * c, c * 24,
                               cudaMemcpyDeviceToDevice, s));
      if ((rc = launch_records(cxy[cur], clab[cur], rec, nrl, c, g.s, 1, s, r * c, (r + 1) * c, rl0)))
        return rc;
    }
    return SPX_OK;
  }
  // partial sums my pixels added to the neighbours' boundary clusters
  int pack_sums(ClusterAcc* up, ClusterAcc* down, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t c = g.ns_c;
    if (up && has_up()) {
      ClusterAcc* src = acc + (own0 - 1) * c;
      SPX_CUDA(cudaMemcpyAsync(up, src, c * sizeof(ClusterAcc), cudaMemcpyDeviceToDevice, s));
      SPX_CUDA(cudaMemsetAsync(src, 0, c * sizeof(ClusterAcc), s));
    }
    if (down && has_down()) {
      ClusterAcc* src = acc + own1 * c;
      SPX_CUDA(cudaMemcpyAsync(down, src, c * sizeof(ClusterAcc), cudaMemcpyDeviceToDevice, s));
      SPX_CUDA(cudaMemsetAsync(src, 0, c * sizeof(ClusterAcc), s));
    }
    return SPX_OK;
  }
  int unpack_sums(const ClusterAcc* from_up, const ClusterAcc* from_down, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t c = g.ns_c;
    const unsigned b = (unsigned)ceil_div(c, 128);
    if (from_up && has_up()) k_add_acc<<<b, 128, 0, s>>>(acc + own0 * c, from_up, (int)c);
    if (from_down && has_down()) k_add_acc<<<b, 128, 0, s>>>(acc + (own1 - 1) * c, from_down, (int)c);
    SPX_LAUNCH_CHECK("k_add_acc");
    return SPX_OK;
  }
  // S label rows at each edge of my own pixel rows
  int64_t label_rows() const { return g.s; }
  int pack_labels(int32_t* up, int32_t* down, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t w = g.width, n = std::min<int64_t>(g.s, oy1 - oy0);
    if (up && has_up())
      SPX_CUDA(cudaMemcpyAsync(up, labels + oy0 * w, n * w * 4, cudaMemcpyDeviceToDevice, s));
    if (down && has_down())
      SPX_CUDA(cudaMemcpyAsync(down, labels + (oy1 - n) * w, n * w * 4, cudaMemcpyDeviceToDevice,
                               s));
    return SPX_OK;
  }
  int unpack_labels(const int32_t* from_up, const int32_t* from_down, cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t w = g.width;
    if (from_up && has_up())  // rows [oy0 - S, oy0): the upper neighbour's last S own rows
      SPX_CUDA(cudaMemcpyAsync(labels + (oy0 - g.s) * w, from_up, g.s * w * 4,
                               cudaMemcpyDeviceToDevice, s));
    if (from_down && has_down()) {  // rows [oy1, hl)
      const int64_t n = hl - oy1;
      SPX_CUDA(cudaMemcpyAsync(labels + oy1 * w, from_down, n * w * 4, cudaMemcpyDeviceToDevice,
                               s));
    }
    return SPX_OK;
  }

  // weak connectivity on own rows (strict: none here); labels carry global
  // cluster ids
  int finish(int32_t* out_labels, double* out_xy, double* out_lab, int64_t* out_counts,
             cudaStream_t s) {
    SPX_CUDA(cudaSetDevice(device));
    const int64_t w = g.width;
    int rc;
    const int32_t* src = labels;
    if (g.connectivity == 1) {
      if ((rc = launch_weak2(labels, out, hl, w, 1, s, oy0, oy1))) return rc;
      src = out;
    }
    // connectivity 2 (strict): the raw labels; strict connectivity is a
    // whole-image scan-order pass, which the caller runs over the gathered
    // strips (strips.py)
    const int64_t n = (oy1 - oy0) * w;  // labels already carry global ids
    SPX_CUDA(cudaMemcpyAsync(out_labels, src + oy0 * w, n * 4, cudaMemcpyDeviceToDevice, s));
    const int64_t c = g.ns_c, no = (own1 - own0) * c;
    if (out_xy)
      SPX_CUDA(cudaMemcpyAsync(out_xy, cxy[cur] + own0 * c * 2, no * 16, cudaMemcpyDeviceToDevice, s));
    if (out_lab)
      SPX_CUDA(cudaMemcpyAsync(out_lab, clab[cur] + own0 * c * 3, no * 24, cudaMemcpyDeviceToDevice,
                               s));
    if (out_counts)
      SPX_CUDA(cudaMemcpyAsync(out_counts, counts + own0 * c, no * 8, cudaMemcpyDeviceToDevice, s));
    return SPX_OK;
  }
};

}  // namespace spx

struct spx_strip {
  spx::Strip s;
};

using spx::as_stream;

extern "C" {

int32_t spx_strip_create(const spx_settings* st, int64_t row_lo, int64_t row_hi, int32_t device,
                         spx_strip** out) {
  using namespace spx;
  *out = nullptr;
  if (!st || row_lo < 0 || row_hi > st->ns_r || row_hi <= row_lo) {
    set_error("strip rows [%lld, %lld) outside the grid", (long long)row_lo, (long long)row_hi);
    return SPX_ERR_INVALID_SETTINGS;
  }
  if (!cell_path_ok(st->height, st->width, st->s, st->tile_len)) {
    set_error("row strips need the fused cell path (4 <= S <= 255, ceil(3S / tile_len) <= 64)");
    return SPX_ERR_INVALID_SETTINGS;
  }
  spx_strip* s = new spx_strip();
  int rc = s->s.init(*st, row_lo, row_hi, device);
  if (rc) {
    delete s;
    return rc;
  }
  *out = s;
  return SPX_OK;
}

int32_t spx_strip_destroy(spx_strip* s) {
  delete s;
  return SPX_OK;
}

int32_t spx_strip_geometry(spx_strip* s, int64_t* out6) {
  // local pixel rows [y0, y0 + hl) of the input window, own pixel rows
  // [y0 + oy0, y0 + oy1), own cell rows [lo, hi)
  out6[0] = s->s.y0;
  out6[1] = s->s.hl;
  out6[2] = s->s.y0 + s->s.oy0;
  out6[3] = s->s.y0 + s->s.oy1;
  out6[4] = s->s.lo;
  out6[5] = s->s.hi;
  return SPX_OK;
}

int32_t spx_strip_begin(spx_strip* s, const uint8_t* rgb_window, void* stream) {
  return s->s.begin(rgb_window, as_stream(stream));
}
int32_t spx_strip_associate(spx_strip* s, int32_t with_update, void* stream) {
  return s->s.associate(with_update != 0, 0, as_stream(stream));
}

int32_t spx_strip_update(spx_strip* s, void* stream) { return s->s.update(0, as_stream(stream)); }

int32_t spx_strip_associate_part(spx_strip* s, int32_t with_update, int32_t part, void* stream) {
  if (part < 0 || part > 2) {
    spx::set_error("strip part must be 0 (all), 1 (interior) or 2 (boundary)");
    return SPX_ERR_VALUE;
  }
  return s->s.associate(with_update != 0, part, as_stream(stream));
}

int32_t spx_strip_update_part(spx_strip* s, int32_t part, void* stream) {
  if (part < 0 || part > 2) {
    spx::set_error("strip part must be 0 (all), 1 (interior) or 2 (boundary)");
    return SPX_ERR_VALUE;
  }
  return s->s.update(part, as_stream(stream));
}

int32_t spx_strip_shift_local(spx_strip* s, double* out, void* stream) {
  return s->s.shift_local(out, as_stream(stream));
}
int32_t spx_strip_pack_centres(spx_strip* s, double* up, double* down, void* stream) {
  return s->s.pack_centres(up, down, as_stream(stream));
}

int32_t spx_strip_unpack_centres(spx_strip* s, const double* from_up, const double* from_down,
                                 void* stream) {
  return s->s.unpack_centres(from_up, from_down, as_stream(stream));
}
int32_t spx_strip_pack_sums(spx_strip* s, void* up, void* down, void* stream) {
  return s->s.pack_sums((spx::ClusterAcc*)up, (spx::ClusterAcc*)down, as_stream(stream));
}
int32_t spx_strip_unpack_sums(spx_strip* s, const void* from_up, const void* from_down,
                              void* stream) {
  return s->s.unpack_sums((const spx::ClusterAcc*)from_up, (const spx::ClusterAcc*)from_down,
                          as_stream(stream));
}
int32_t spx_strip_pack_labels(spx_strip* s, int32_t* up, int32_t* down, void* stream) {
  return s->s.pack_labels(up, down, as_stream(stream));
}
int32_t spx_strip_unpack_labels(spx_strip* s, const int32_t* from_up, const int32_t* from_down,
                                void* stream) {
  return s->s.unpack_labels(from_up, from_down, as_stream(stream));
}
int32_t spx_strip_finish(spx_strip* s, int32_t* labels, double* cxy, double* clab, int64_t* counts,
                         void* stream) {
  return s->s.finish(labels, cxy, clab, counts, as_stream(stream));
}

}  // extern "C"
