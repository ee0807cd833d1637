// cell.cu -- the engine's fused association + centre-update path.
//
// Work unit: one grid cell (S x S pixels).  All pixels of a cell share the
// same 9 candidate centres, so a warp (or half-warp for S = 8) loads them once
// into registers and streams the cell's pixels in runs of 4 (three 128-bit
// loads of HWC Lab per run).  Distances are evaluated two pixels at a time
// with Blackwell's packed FFMA2/FADD2/FMUL2, square roots on MUFU.RSQ, and
// the same rigorous fp32 -> binary64 argmin certificate as assoc.cu (uncertain
// pixels are re-evaluated with the reference's exact binary64 order).
//
// With ACC the kernel also produces the centre-update partial sums for every
// (cell, candidate slot): the run's slot nibbles and Lab values are staged in
// shared memory and 9 (or 27) "owner" lanes fold them per slot in binary64
// (colour) and int32 (x, y, count).  The reduce kernel adds the 9 partials of
// each cluster in a fixed order.
//
// Exactness of the sums: the reference folds the
// colour sums left-to-right in binary64 (_core.pyx:233-243).  If every member
// value v of a cluster is 0 or has 2^-tau_exp <= |v| < 128, every partial sum
// of any subset of the cluster is an exact binary64 number (members are
// multiples of ulp(2^tau) and |sum| < count * 128 <= 2^53 ulp), so the
// reference's fold, its strip tree, and our fixed-order sum all equal the
// exact sum.  Pixels outside that range set a flag bit; the reduce kernel
// recomputes flagged clusters with the reference's exact strip fold.
#include <cmath>

#include "spx_internal.cuh"

namespace spx {

namespace {

__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float rsq(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// sqrt of a packed pair as q * rsqrt(q) (q >= 1e-30 by construction).
__device__ __forceinline__ unsigned long long sqrt2(unsigned long long q) {
  float q0, q1;
  f2_unpack(q, q0, q1);
  return mul2(q, f2_pack(rsq(q0), rsq(q1)));
}

__device__ __forceinline__ bool fin_small(double v) { return fabs(v) < 1e15; }

// Out-of-range flag for the certified sums: nonzero |v| < tau or |v| >= 128
// (NaN/inf included).
__device__ __forceinline__ unsigned sum_flag(float v, float tau) {
  float a = fabsf(v);
  return (a != 0.f && a < tau) || !(a < 128.f) ? 1u : 0u;
}

}  // namespace

struct CellParams {
  const float* img;        // [F][H][W][3]
  const double* cxy;       // [F][K][2]  (current centres, binary64)
  const double* clab;      // [F][K][3]
  const CRec* rec;         // [F][K]     fp32 records of the current centres
  int32_t* labels;         // [F][H][W]
  Part* part;              // [F][K][9]  (ACC only)
  const int32_t* done;     // per frame, skip == 1 (may be null)
  int h, w, s, ns_r, ns_c, frames;
  int lanes_per_cell;      // 32 or 16
  int runs_per_row;        // S / 4
  int runs;                // S * S / 4
  double xy_weight;
  float w32, k_mp, k_mc, k_xy, k_const, k_rel;
  float tau;               // certified-sum lower magnitude
};

// Exact binary64 argmin over the candidates in reference order (_core.pyx:181-197).
__device__ __noinline__ int exact_argmin(const double* __restrict__ cxy, const double* __restrict__ clab,
                                         float pl, float pa, float pb, int x, int y, int pr, int pc,
                                         int ns_r, int ns_c, double xy_weight) {
  int best_k = pr * ns_c + pc;
  double best_d = pix_dist_exact(pl, pa, pb, cxy[2 * best_k], cxy[2 * best_k + 1], clab[3 * best_k],
                                 clab[3 * best_k + 1], clab[3 * best_k + 2], x, y, xy_weight);
  for (int t = 1; t < 9; ++t) {
    int kr = pr + off_r(t), kc = pc + off_c(t);
    if (kr < 0 || kr >= ns_r || kc < 0 || kc >= ns_c) continue;
    int k = kr * ns_c + kc;
    double d = pix_dist_exact(pl, pa, pb, cxy[2 * k], cxy[2 * k + 1], clab[3 * k], clab[3 * k + 1],
                              clab[3 * k + 2], x, y, xy_weight);
    if (d < best_d) {
      best_d = d;
      best_k = k;
    }
  }
  return best_k;
}

template <bool ACC>
__global__ void __launch_bounds__(128) k_cell(CellParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lpc = p.lanes_per_cell;
  const int cpw = 32 / lpc;                       // cells per warp
  const int ci = lane / lpc, ll = lane % lpc;     // cell within warp, lane within cell
  const int S = p.s;
  const int cells_per_frame = p.ns_r * p.ns_c;
  const long long gcell = ((long long)blockIdx.x * (blockDim.x >> 5) + warp) * cpw + ci;
  const long long total_cells = (long long)cells_per_frame * p.frames;
  // per-cell smem: slot bytes [runs] words + Lab [4][runs] float4
  const int cell_bytes = p.runs * 4 + p.runs * 4 * 16;
  unsigned char* cbuf = smem + (size_t)((threadIdx.x >> 5) * cpw + ci) * cell_bytes;
  uint32_t* slot_words = reinterpret_cast<uint32_t*>(cbuf);
  float4* labv = reinterpret_cast<float4*>(cbuf + p.runs * 4);

  bool active = gcell < total_cells;
  int f = 0, cr = 0, cc = 0;
  if (active) {
    f = (int)(gcell / cells_per_frame);
    int cell = (int)(gcell % cells_per_frame);
    cr = cell / p.ns_c;
    cc = cell % p.ns_c;
    if (p.done && p.done[f] == 1) active = false;
  }

  // ---- candidates: 9 records, relative to this cell's origin ----------------
  float cl[9], ca[9], cb[9], cx[9], cy[9];
  unsigned valid = 0;
  float mc = 0.f, mxy = 0.f;
  bool all_ok = true;
  if (active) {
    const CRec* rf = p.rec + (long long)f * cells_per_frame;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      int kr = cr + off_r(t), kc = cc + off_c(t);
      bool in = kr >= 0 && kr < p.ns_r && kc >= 0 && kc < p.ns_c;
      CRec r = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 1.f};
      if (in) {
        const float4* q = reinterpret_cast<const float4*>(rf + kr * p.ns_c + kc);
        float4 v0 = __ldg(q), v1 = __ldg(q + 1);
        r = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        valid |= 1u << t;
      }
      cl[t] = r.l;
      ca[t] = r.a;
      cb[t] = r.b;
      cx[t] = __fadd_rn(r.xr, (float)(off_c(t) * S));
      cy[t] = __fadd_rn(r.yr, (float)(off_r(t) * S));
      if (in) {
        mc = fmaxf(mc, r.mag_lab);
        mxy = fmaxf(mxy, fmaxf(fabsf(cx[t]), fabsf(cy[t])));
        all_ok = all_ok && (r.ok != 0.f);
      }
    }
  }
  // Cell constant part of 2A: k_mc*Mc + k_xy*(3*Mxy + 2S) + k_const
  float two_a_cell = __fmaf_rn(mc, p.k_mc, __fmaf_rn(__fmaf_rn(3.f, mxy, 2.f * S), p.k_xy, p.k_const));
  if (!all_ok) two_a_cell = INFINITY;
  const unsigned long long W2 = f2_pack(p.w32, p.w32);
  const unsigned long long TINY2 = f2_pack(1e-30f, 1e-30f);
  const int x_cell = cc * S, y_cell = cr * S;
  const long long img_base = (long long)f * p.h * p.w;

  if (active) {
    for (int j = ll; j < p.runs; j += lpc) {
      const int row = j / p.runs_per_row;
      const int c4 = (j - row * p.runs_per_row) * 4;
      const int y = y_cell + row, x = x_cell + c4;
      uint32_t word = 0xFFFFFFFFu;  // slot bytes; 0xFF = no pixel
      if (y < p.h && x < p.w) {
        const long long pix = img_base + (long long)y * p.w + x;
        const float4* src = reinterpret_cast<const float4*>(p.img + pix * 3);
        float4 v0 = __ldg(src), v1 = __ldg(src + 1), v2 = __ldg(src + 2);
        float L[4] = {v0.x, v0.w, v1.z, v2.y};
        float A[4] = {v0.y, v1.x, v1.w, v2.z};
        float B[4] = {v0.z, v1.y, v2.x, v2.w};
        const unsigned long long NL01 = f2_pack(-L[0], -L[1]), NL23 = f2_pack(-L[2], -L[3]);
        const unsigned long long NA01 = f2_pack(-A[0], -A[1]), NA23 = f2_pack(-A[2], -A[3]);
        const unsigned long long NB01 = f2_pack(-B[0], -B[1]), NB23 = f2_pack(-B[2], -B[3]);
        const float xr0 = (float)c4;
        const unsigned long long NX01 = f2_pack(-xr0, -(xr0 + 1.f));
        const unsigned long long NX23 = f2_pack(-(xr0 + 2.f), -(xr0 + 3.f));
        const float yr = (float)row;
        unsigned k1[4] = {0x7F7FFFFFu, 0x7F7FFFFFu, 0x7F7FFFFFu, 0x7F7FFFFFu};
        unsigned k2[4] = {0x7F7FFFFFu, 0x7F7FFFFFu, 0x7F7FFFFFu, 0x7F7FFFFFu};
#pragma unroll
        for (int t = 0; t < 9; ++t) {
          const unsigned long long CL = f2_pack(cl[t], cl[t]);
          const unsigned long long CA = f2_pack(ca[t], ca[t]);
          const unsigned long long CB = f2_pack(cb[t], cb[t]);
          const unsigned long long CX = f2_pack(cx[t], cx[t]);
          const float dy = __fsub_rn(cy[t], yr);
          const float dyy = __fmaf_rn(dy, dy, 1e-30f);
          const unsigned long long DYY = f2_pack(dyy, dyy);
          unsigned long long d01, d23;
          {
            unsigned long long dl = add2(CL, NL01), da = add2(CA, NA01), db = add2(CB, NB01);
            unsigned long long q = fma2(db, db, fma2(da, da, fma2(dl, dl, TINY2)));
            unsigned long long dx = add2(CX, NX01);
            unsigned long long r = fma2(dx, dx, DYY);
            d01 = fma2(W2, sqrt2(r), sqrt2(q));
          }
          {
            unsigned long long dl = add2(CL, NL23), da = add2(CA, NA23), db = add2(CB, NB23);
            unsigned long long q = fma2(db, db, fma2(da, da, fma2(dl, dl, TINY2)));
            unsigned long long dx = add2(CX, NX23);
            unsigned long long r = fma2(dx, dx, DYY);
            d23 = fma2(W2, sqrt2(r), sqrt2(q));
          }
          float D[4];
          f2_unpack(d01, D[0], D[1]);
          f2_unpack(d23, D[2], D[3]);
          const bool vt = (valid >> t) & 1u;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            unsigned key = vt ? ((__float_as_uint(D[i]) & ~15u) | (unsigned)t) : 0x7F7FFFFFu;
            k2[i] = min(k2[i], max(k1[i], key));
            k1[i] = min(k1[i], key);
          }
        }
        int lab4[4];
        word = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float mp = fabsf(L[i]) + fabsf(A[i]) + fabsf(B[i]);
          const float f2v = __uint_as_float(k2[i]);
          const float thr = __fmaf_rn(f2v, p.k_rel, __fmaf_rn(mp, p.k_mp, two_a_cell));
          const float gap = __fsub_rn(f2v, __uint_as_float(k1[i]));
          int t = (int)(k1[i] & 15u);
          int k = (cr + off_r(t)) * p.ns_c + (cc + off_c(t));
          if (!(gap > thr) || !(mp < 1e15f)) {
            k = exact_argmin(p.cxy + (long long)f * cells_per_frame * 2,
                             p.clab + (long long)f * cells_per_frame * 3, L[i], A[i], B[i],
                             x + i, y, cr, cc, p.ns_r, p.ns_c, p.xy_weight);
            const int idx = (k / p.ns_c - cr + 1) * 3 + (k % p.ns_c - cc + 1);
            t = idx < 4 ? idx + 1 : (idx == 4 ? 0 : idx);  // (dr,dc) -> scan slot
          }
          lab4[i] = k;
          if (ACC) {
            unsigned fl = sum_flag(L[i], p.tau) | sum_flag(A[i], p.tau) | sum_flag(B[i], p.tau);
            word |= ((unsigned)t | (fl << 4)) << (8 * i);
          }
        }
        int4* dst = reinterpret_cast<int4*>(p.labels + pix);
        *dst = make_int4(lab4[0], lab4[1], lab4[2], lab4[3]);
        if (ACC) {
          labv[0 * p.runs + j] = make_float4(L[0], A[0], B[0], 0.f);
          labv[1 * p.runs + j] = make_float4(L[1], A[1], B[1], 0.f);
          labv[2 * p.runs + j] = make_float4(L[2], A[2], B[2], 0.f);
          labv[3 * p.runs + j] = make_float4(L[3], A[3], B[3], 0.f);
        }
      }
      if (ACC) slot_words[j] = word;
    }
  }
  if (!ACC) return;
  __syncwarp();

  // ---- owner lanes: fold each slot's members -------------------------------
  const int segs = lpc / 9;  // 3 (32 lanes) or 1 (16 lanes)
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  int sx = 0, sy = 0, cnt = 0;
  unsigned flag = 0;
  const int slot = ll % 9, seg = ll / 9;
  if (active && seg < segs) {
    const int w0 = (p.runs * seg) / segs, w1 = (p.runs * (seg + 1)) / segs;
    const uint32_t rep = 0x01010101u * (uint32_t)slot;
    for (int wi = w0; wi < w1; ++wi) {
      uint32_t wv = slot_words[wi];
      uint32_t z = (wv & 0x0F0F0F0Fu) ^ rep;  // zero byte <=> slot match
      // exact zero-byte detection (no false positives across bytes)
      uint32_t m = ~(((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z | 0x7F7F7F7Fu);
      m &= ~((wv & 0x80808080u));  // 0xFF marks "no pixel"
      while (m) {
        const int bit = __ffs(m) - 1;
        const int i = bit >> 3;
        m &= m - 1;
        const float4 v = labv[i * p.runs + wi];
        s0 = dadd(s0, (double)v.x);
        s1 = dadd(s1, (double)v.y);
        s2 = dadd(s2, (double)v.z);
        const int row = wi / p.runs_per_row;
        sx += (wi - row * p.runs_per_row) * 4 + i;
        sy += row;
        cnt += 1;
        flag |= (wv >> (i * 8 + 4)) & 1u;
      }
    }
  }
  // combine the segments (fixed order: seg 0 + seg 1 + seg 2)
  const unsigned full = 0xFFFFFFFFu;
  if (segs > 1) {
#pragma unroll
    for (int g = 1; g < 3; ++g) {
      const int srcl = (lane & ~(lpc - 1)) + slot + 9 * g;
      double t0 = __shfl_sync(full, s0, srcl), t1 = __shfl_sync(full, s1, srcl),
             t2 = __shfl_sync(full, s2, srcl);
      int ux = __shfl_sync(full, sx, srcl), uy = __shfl_sync(full, sy, srcl),
          uc = __shfl_sync(full, cnt, srcl);
      unsigned uf = __shfl_sync(full, flag, srcl);
      if (seg == 0) {
        s0 = dadd(s0, t0);
        s1 = dadd(s1, t1);
        s2 = dadd(s2, t2);
        sx += ux;
        sy += uy;
        cnt += uc;
        flag |= uf;
      }
    }
  }
  if (active && seg == 0) {
    Part* o = p.part + (gcell * 9 + slot);
    Part r;
    r.s[0] = s0;
    r.s[1] = s1;
    r.s[2] = s2;
    r.sx = sx;
    r.sy = sy;
    r.cnt = cnt;
    r.flag = (int)flag;
    *o = r;
  }
}

namespace {

// fp32 filter records of the current centres (after init / perturb).
__global__ void k_records(const double* __restrict__ cxy, const double* __restrict__ clab,
                          CRec* __restrict__ rec, int ns_c, int s, int k_per_frame, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int k = (int)(i % k_per_frame);
  int kr = k / ns_c, kc = k % ns_c;
  double x = cxy[2 * i], y = cxy[2 * i + 1];
  double l = clab[3 * i], a = clab[3 * i + 1], b = clab[3 * i + 2];
  CRec r;
  r.l = __double2float_rn(l);
  r.a = __double2float_rn(a);
  r.b = __double2float_rn(b);
  r.xr = __double2float_rn(dsub(x, (double)kc * s));
  r.yr = __double2float_rn(dsub(y, (double)kr * s));
  bool ok = fin_small(x) && fin_small(y) && fin_small(l) && fin_small(a) && fin_small(b);
  r.mag_lab = fmaxf(fabsf(r.l), fmaxf(fabsf(r.a), fabsf(r.b)));
  r.mag_xy = fmaxf(fabsf(r.xr), fabsf(r.yr));
  r.ok = ok ? 1.f : 0.f;
  rec[i] = r;
}

// Reference strip fold for one (cluster, strip): _core.pyx:221-255 verbatim
// order (row-major, binary64 colour, integer x/y/count).
__device__ void strip_fold(const float* __restrict__ img, const int32_t* __restrict__ lab, int h,
                           int w, int k, int j, int s, int ns_c, int tile_len, double out[6]) {
  int r = k / ns_c, c = k % ns_c;
  int wx0 = max((c - 1) * s, 0), wx1 = min((c + 2) * s, w);
  int ry0 = (r - 1) * s, ry1 = min((r + 2) * s, h);
  int sy0 = max(ry0 + j * tile_len, 0), sy1 = min(ry0 + (j + 1) * tile_len, ry1);
  double sl = 0.0, sa = 0.0, sb = 0.0;
  long long sx = 0, sy = 0, cnt = 0;
  for (int y = sy0; y < sy1; ++y)
    for (int x = wx0; x < wx1; ++x)
      if (__ldg(lab + (long long)y * w + x) == k) {
        const float* px = img + ((long long)y * w + x) * 3;
        sl = dadd(sl, (double)__ldg(px));
        sa = dadd(sa, (double)__ldg(px + 1));
        sb = dadd(sb, (double)__ldg(px + 2));
        sx += x;
        sy += y;
        cnt += 1;
      }
  out[0] = sl;
  out[1] = sa;
  out[2] = sb;
  out[3] = (double)sx;
  out[4] = (double)sy;
  out[5] = (double)cnt;
}

struct ReduceParams {
  const Part* part;
  const float* img;
  const int32_t* labels;
  const double* prev_xy;
  const double* prev_lab;
  double* out_xy;
  double* out_lab;
  int64_t* counts;
  CRec* rec;
  const int32_t* done;
  int h, w, s, ns_r, ns_c, frames, n_bl, tile_len;
};

__device__ __forceinline__ void write_centre(const ReduceParams& p, long long gk, int kr, int kc,
                                             double cnt, double sl, double sa, double sb,
                                             double sx, double sy) {
  double l, a, b, x, y;
  if (cnt > 0.0) {  // _core.pyx:313-320
    l = ddiv(sl, cnt);
    a = ddiv(sa, cnt);
    b = ddiv(sb, cnt);
    x = ddiv(sx, cnt);
    y = ddiv(sy, cnt);
  } else {
    l = p.prev_lab[3 * gk];
    a = p.prev_lab[3 * gk + 1];
    b = p.prev_lab[3 * gk + 2];
    x = p.prev_xy[2 * gk];
    y = p.prev_xy[2 * gk + 1];
  }
  p.out_lab[3 * gk] = l;
  p.out_lab[3 * gk + 1] = a;
  p.out_lab[3 * gk + 2] = b;
  p.out_xy[2 * gk] = x;
  p.out_xy[2 * gk + 1] = y;
  p.counts[gk] = (int64_t)cnt;
  CRec r;
  r.l = __double2float_rn(l);
  r.a = __double2float_rn(a);
  r.b = __double2float_rn(b);
  r.xr = __double2float_rn(dsub(x, (double)kc * p.s));
  r.yr = __double2float_rn(dsub(y, (double)kr * p.s));
  r.mag_lab = fmaxf(fabsf(r.l), fmaxf(fabsf(r.a), fabsf(r.b)));
  r.mag_xy = fmaxf(fabsf(r.xr), fabsf(r.yr));
  r.ok = (fin_small(x) && fin_small(y) && fin_small(l) && fin_small(a) && fin_small(b)) ? 1.f : 0.f;
  p.rec[gk] = r;
}

// One lane per cluster: fixed-order sum of the 9 (cell, slot) partials that
// belong to it.  Clusters with a flagged member are recomputed by the whole
// warp with the reference strip folds + pairwise strip tree (_core.pyx:300-311).
__global__ void __launch_bounds__(128) k_reduce_cells(ReduceParams p) {
  __shared__ double strips[4][32][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = p.ns_r * p.ns_c;
  const long long gk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = gk < (long long)K * p.frames;
  int f = 0, k = 0, kr = 0, kc = 0;
  bool todo = false, flagged = false;
  if (in) {
    f = (int)(gk / K);
    k = (int)(gk % K);
    kr = k / p.ns_c;
    kc = k % p.ns_c;
    todo = !(p.done && p.done[f]);
  }
  if (todo) {
    const Part* pf = p.part + (long long)f * K * 9;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    long long sx = 0, sy = 0, cnt = 0;
    int fl = 0;
    // cell (kr - dr, kc - dc) sees this cluster at offset (dr, dc)
    for (int dr = -1; dr <= 1; ++dr)
      for (int dc = -1; dc <= 1; ++dc) {
        const int r2 = kr - dr, c2 = kc - dc;
        if (r2 < 0 || r2 >= p.ns_r || c2 < 0 || c2 >= p.ns_c) continue;
        const int idx = (dr + 1) * 3 + (dc + 1);
        const int t = idx < 4 ? idx + 1 : (idx == 4 ? 0 : idx);
        const Part q = pf[(long long)(r2 * p.ns_c + c2) * 9 + t];
        s0 = dadd(s0, q.s[0]);
        s1 = dadd(s1, q.s[1]);
        s2 = dadd(s2, q.s[2]);
        sx += (long long)q.sx + (long long)q.cnt * c2 * p.s;
        sy += (long long)q.sy + (long long)q.cnt * r2 * p.s;
        cnt += q.cnt;
        fl |= q.flag;
      }
    flagged = fl != 0;
    if (!flagged)
      write_centre(p, gk, kr, kc, (double)cnt, s0, s1, s2, (double)sx, (double)sy);
  }
  // exact fallback for flagged clusters, one at a time per warp
  unsigned need = __ballot_sync(0xFFFFFFFFu, flagged);
  while (need) {
    const int src = __ffs(need) - 1;
    need &= need - 1;
    const int fk = __shfl_sync(0xFFFFFFFFu, k, src);
    const int ff = __shfl_sync(0xFFFFFFFFu, f, src);
    const float* im = p.img + (long long)ff * p.h * p.w * 3;
    const int32_t* lb = p.labels + (long long)ff * p.h * p.w;
    if (lane < p.n_bl) strip_fold(im, lb, p.h, p.w, fk, lane, p.s, p.ns_c, p.tile_len, strips[warp][lane]);
    __syncwarp();
    if (lane == 0) {
      double (*sk)[6] = strips[warp];
      int m = p.n_bl;
      while (m > 1) {  // pairwise tree, _core.pyx:301-311
        int half = m >> 1;
        for (int i = 0; i < half; ++i)
          for (int comp = 0; comp < 6; ++comp) sk[i][comp] = dadd(sk[2 * i][comp], sk[2 * i + 1][comp]);
        if (m & 1)
          for (int comp = 0; comp < 6; ++comp) sk[half][comp] = sk[m - 1][comp];
        m = half + (m & 1);
      }
      write_centre(p, (long long)ff * K + fk, fk / p.ns_c, fk % p.ns_c, sk[0][5], sk[0][0], sk[0][1],
                   sk[0][2], sk[0][3], sk[0][4]);
    }
    __syncwarp();
  }
}

__global__ void k_fill_i32(int32_t* v, int n, int value) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = value;
}

}  // namespace

// ---- launchers ----------------------------------------------------------------

bool cell_path_ok(int64_t h, int64_t w, int64_t s, int64_t tile_len) {
  int64_t n_bl = ceil_div(3 * s, tile_len);
  return s % 4 == 0 && s >= 8 && s <= 32 && w % 4 == 0 && n_bl <= 32 &&
         h * w * 3 < (int64_t)1 << 40 && h < (1 << 30) && w < (1 << 30);
}

size_t cell_smem_bytes(int64_t s, bool acc) {
  if (!acc) return 0;
  int runs = (int)(s * s / 4);
  int lpc = runs >= 32 ? 32 : 16;
  int cpw = 32 / lpc;
  return (size_t)4 * cpw * (runs * 4 + runs * 4 * 16);
}

void assoc_bound_coefficients(double xy_weight, float& w32, float& k_mp, float& k_mc, float& k_xy,
                              float& k_const, float& k_rel);

int launch_cell(const float* img, const double* cxy, const double* clab, const CRec* rec,
                int32_t* labels, Part* part, const int32_t* done, int64_t h, int64_t w, int64_t s,
                int64_t ns_r, int64_t ns_c, double xy_weight, int frames, bool acc,
                cudaStream_t st) {
  CellParams p;
  p.img = img;
  p.cxy = cxy;
  p.clab = clab;
  p.rec = rec;
  p.labels = labels;
  p.part = part;
  p.done = done;
  p.h = (int)h;
  p.w = (int)w;
  p.s = (int)s;
  p.ns_r = (int)ns_r;
  p.ns_c = (int)ns_c;
  p.frames = frames;
  p.runs = (int)(s * s / 4);
  p.runs_per_row = (int)(s / 4);
  p.lanes_per_cell = p.runs >= 32 ? 32 : 16;
  p.xy_weight = xy_weight;
  assoc_bound_coefficients(xy_weight, p.w32, p.k_mp, p.k_mc, p.k_xy, p.k_const, p.k_rel);
  // tau = 2^k with 9 S^2 <= 2^(23 + k)  (certified sums, see header)
  int kexp = -23;
  while ((double)std::ldexp(1.0, 23 + kexp) < 9.0 * (double)(s * s)) ++kexp;
  p.tau = (float)std::ldexp(1.0, kexp);
  const int cpw = 32 / p.lanes_per_cell;
  const long long cells = ns_r * ns_c * (long long)frames;
  const long long warps = ceil_div(cells, cpw);
  const unsigned blocks = (unsigned)ceil_div(warps, 4);
  const size_t smem = cell_smem_bytes(s, acc);
  if (acc) {
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
      SPX_CUDA(cudaFuncSetAttribute(k_cell<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      configured = smem;
    }
    k_cell<true><<<blocks, 128, smem, st>>>(p);
  } else {
    k_cell<false><<<blocks, 128, 0, st>>>(p);
  }
  SPX_LAUNCH_CHECK("k_cell");
  return SPX_OK;
}

int launch_records(const double* cxy, const double* clab, CRec* rec, int64_t ns_r, int64_t ns_c,
                   int64_t s, int frames, cudaStream_t st) {
  long long n = ns_r * ns_c * (long long)frames;
  k_records<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(cxy, clab, rec, (int)ns_c, (int)s,
                                                        (int)(ns_r * ns_c), n);
  SPX_LAUNCH_CHECK("k_records");
  return SPX_OK;
}

int launch_reduce_cells(const Part* part, const float* img, const int32_t* labels,
                        const double* prev_xy, const double* prev_lab, double* out_xy,
                        double* out_lab, int64_t* counts, CRec* rec, const int32_t* done,
                        int64_t h, int64_t w, int64_t s, int64_t ns_r, int64_t ns_c,
                        int64_t tile_len, int frames, cudaStream_t st) {
  ReduceParams p;
  p.part = part;
  p.img = img;
  p.labels = labels;
  p.prev_xy = prev_xy;
  p.prev_lab = prev_lab;
  p.out_xy = out_xy;
  p.out_lab = out_lab;
  p.counts = counts;
  p.rec = rec;
  p.done = done;
  p.h = (int)h;
  p.w = (int)w;
  p.s = (int)s;
  p.ns_r = (int)ns_r;
  p.ns_c = (int)ns_c;
  p.frames = frames;
  p.n_bl = (int)ceil_div(3 * s, tile_len);
  p.tile_len = (int)tile_len;
  long long n = ns_r * ns_c * (long long)frames;
  k_reduce_cells<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(p);
  SPX_LAUNCH_CHECK("k_reduce_cells");
  return SPX_OK;
}

int launch_fill_i32(int32_t* v, int n, int value, cudaStream_t st) {
  k_fill_i32<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(v, n, value);
  SPX_LAUNCH_CHECK("k_fill_i32");
  return SPX_OK;
}

}  // namespace spx
