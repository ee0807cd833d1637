// cell.cu -- the engine's fused association + centre-update path.
//
// Work unit: one grid cell (S x S pixels).  All pixels of a cell share the
// same 9 candidate centres, so the cell's LPC lanes (2 to 32 by S and launch
// size, cell_lpc) stage the 9 fp32 candidate records in shared memory and
// stream the cell's
// pixels in runs of 4 (one 128-bit load per planar Lab channel; the final
// pass stages its runs with cp.async).  Distances are evaluated two pixels
// at a time with Blackwell's packed FFMA2/FADD2/FMUL2 (the candidate as a
// broadcast scalar operand), square roots with MUFU (sqrt.approx.ftz), and a
// rigorous fp32 -> binary64 argmin certificate: pixels whose best and
// second-best keys are closer than the error bound are re-evaluated with the
// reference's exact binary64 order.
//
// With ACC the kernel also produces the centre update: each lane adds its
// pixels' colour (binary64) and packed x / y / count / flag counters
// (integer) into lane-private per-slot accumulators in shared memory; at the
// end of a cell the LPC lane entries of each slot are summed and added to
// the cluster's ClusterAcc with global atomics (f64 atomicAdd for colour).
//
// Determinism / exactness of the sums: the
// reference folds each strip's colour values left to right in binary64 and
// combines strips with a pairwise tree (_core.pyx:233-311).  If every member
// value v of a cluster is 0 or has 2^k <= |v| < 128 with 9 S^2 <= 2^(23+k),
// every partial sum of any subset of the cluster is an exact binary64 number,
// so the reference's fold, its tree and ANY order of our lane sums and
// atomics give the same (exact) result -- the atomics' order cannot matter.
// Pixels outside that range carry a flag (sign bit of Lab channel 0, set by
// the engine's convert); a cluster with a flagged member is queued and
// recomputed by k_exact_clusters (S <= 32) / k_exact_wide (S > 32) with the
// reference's strip folds and tree.  k_reduce_cells divides the exact sums
// (k_update runs the reduce and k_exact_clusters as one launch).  For
// S > 42 the engine uses wide mode instead (per-(cluster, strip) sums, see
// "wide cells" below).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>

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
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
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
__device__ __forceinline__ float sqa(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

}  // namespace

struct CellParams {
  const float* img;        // [F][H][W][3]
  const double* cxy;       // [F][K][2]  (current centres, binary64)
  const double* clab;      // [F][K][3]
  const CRec* rec;         // [F][K]     fp32 records of the current centres
  int32_t* labels;         // [F][H][W]
  ClusterAcc* acc;         // [F][K]     (ACC only) atomically accumulated sums
  const int32_t* done;     // per frame, skip == 1 (may be null)
  int32_t* wl;             // (ACC, may be null) flagged clusters are appended here
  int32_t* wl_n;           //   by their first flagged contribution
  int h, w, s, ns_r, ns_c, frames;
  long long plane;         // planar Lab channel stride (plane_of(h * w))
  int cr0, cr1;            // cell rows processed (local grid)
  int row_off;             // global cell row of local row 0 (strips; 0 otherwise)
  int runs_per_row;        // ceil(S / 4)
  int runs;                // S * runs_per_row
  int groups_per_warp;     // cell groups walked by one warp
  int parts, part_runs;    // warps per cell group and runs per warp (small launches, LPC 32)
  unsigned row_magic;      // ceil(2^32 / runs_per_row)
  double xy_weight;
  float w32, k_mp, k_mc, k_xy, k_const, k_rel;
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

// Shared-memory layout per warp (CPW = 32 / LPC cells per warp).
//   cand[CPW][9]:   fp32 candidate l, a, b, x (cell relative); the packed
//                   FADD2/FFMA2 ops take them as broadcast scalar operands
//   cy[CPW][9]:     candidate y (cell relative)
//   cand_k[CPW][9]: cluster id of each candidate slot
//   acc (ACC):      lane-private per-slot accumulators, lane-interleaved so
//                   any per-lane slot choice is bank-conflict free:
//                   accd[9][3][32] double, acci[9][32] uint64 (packed
//                   count | flags<<11 | sum_x<<22 | sum_y<<43).
// With LPC >= 8 the per-warp block is <= 10 KB, so 16 warps fit the 164 KB
// shared-memory carve-out and leave 92 KB of L1 for the Lab stream.
// Warps per k_cell block (same 16 warps per SM either way: the register
// budget is per SM).  Two: 256 C1 frames with 4 lanes 4.316 -> 4.291 ms,
// fused pass 0.585 -> 0.578 ms (C4 within 0.4%); eight: 5% slower.
#ifndef SPX_CELL_WARPS
#define SPX_CELL_WARPS 2
#endif
constexpr int kWarps = SPX_CELL_WARPS;
constexpr int kCellMaxS = 255;
// Cell groups walked by one warp (at most).  Measured with 4 lanes, 256 C1
// frames (bench_configs, late round 2): 1 group per warp -- more, shorter
// warps, smaller tails -- fused pass 0.598 -> 0.584 ms, step 4.327 -> 4.310
// ms; C4 6.96 -> 6.89 ms; C3 equal (2 and 3 in between, 8 worse).
#ifndef SPX_GPW
#define SPX_GPW 1
#endif
constexpr int kGroupsPerWarp = SPX_GPW;
#ifndef SPX_CELL_WARPS_SMALL
#define SPX_CELL_WARPS_SMALL 32
#endif
constexpr int kCellWarpsSmall = SPX_CELL_WARPS_SMALL;  // warps per SM a small LPC-32 launch aims for
#ifndef SPX_MINB
#define SPX_MINB 4  // resident blocks per SM the register budget is sized for
#endif
#ifndef SPX_MINB_FIN
// the final (no-accumulation) pass: 16 warps per SM like the accumulating
// one (with 4 lanes per cell at S = 16: 0.434 vs 0.438 ms at 20 warps; with
// 8 lanes 20 warps had been 1% faster)
#define SPX_MINB_FIN SPX_MINB
#endif
#ifndef SPX_PAIRMIN
#define SPX_PAIRMIN 1  // top-2 keys merged two candidates at a time (cellbench: -0.8% / -1.6%)
#endif
// (rounded up to 16 bytes: the accumulators behind it take 16-byte accesses)
__host__ __device__ constexpr size_t cand_bytes(int lpc) {
  return ((size_t)(32 / lpc) * 9 * 24 + 15) & ~(size_t)15;
}
// Accumulator columns start on bank 0 (stride 32 entries), so the per-pixel
// updates (lane l touches entry l of its slot's column) are conflict-free
// whatever slots the lanes pick; in the epilogue, where a lane sums a whole
// column of its cell, each lane starts at a rotated 16-byte offset so the
// lanes' reads spread over the banks.
constexpr size_t kAccBytes = 9 * 3 * 32 * sizeof(double) + 9 * 32 * sizeof(uint64_t);
// Aligned runs of the final pass are staged by cp.async into a per-lane
// double buffer in shared memory instead of a register prefetch (cellbench,
// 256 C1 frames: 0.469 -> 0.455 ms); the accumulating pass keeps the
// register prefetch (its shared memory already holds the accumulators, and
// staging measured no better there).
#ifndef SPX_CPA
#define SPX_CPA 1
#endif
#ifndef SPX_CPA_ACC
#define SPX_CPA_ACC 0
#endif
__host__ __device__ constexpr bool cpa_on(bool acc) { return acc ? SPX_CPA_ACC : SPX_CPA; }
// cp.async run staging: [2 buffers][3 channels][32 lanes] float4
constexpr size_t kStageBytes = 2 * 3 * 32 * 16;
__host__ __device__ constexpr size_t warp_smem(int lpc, bool acc) {
  return cand_bytes(lpc) + (acc ? kAccBytes : 0) + (cpa_on(acc) ? kStageBytes : 0);
}

// Work unit: a group of CPW = 32 / LPC cells of one frame; a warp walks
// up to kGroupsPerWarp consecutive groups (fewer when the launch would not
// fill the GPU).  Each cell's LPC lanes stage its 9
// candidates in shared memory, then stream the cell's pixels in runs of 4
// (one 128-bit load per planar channel); LPC = 16 for S >= 16, LPC = 4 for
// small cells (S = 8, 12) so each lane still gets several runs per cell.
// AL: every run is 4 whole pixels at a 16-byte aligned address (S % 4 == 0
// and W % 4 == 0): 128-bit loads and stores.  Otherwise a cell row ends in a
// partial run (S % 4 pixels) and runs may start anywhere: the run's pixels
// are loaded and stored one by one and the pixels past the cell (or image)
// edge are masked out of the labels, the certificate and the sums.
template <bool ACC, int LPC, bool AL>
__global__ void __launch_bounds__(kWarps * 32, (ACC ? SPX_MINB : SPX_MINB_FIN) * 4 / kWarps)
    k_cell(CellParams p) {
  constexpr int CPW = 32 / LPC;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = lane / LPC, ll = lane % LPC;  // cell within warp, lane within cell
  const int S = p.s;
  const int K = p.ns_r * p.ns_c;
  const int f = blockIdx.y;
  if (p.done && p.done[f] == 1) return;  // whole block: one frame
  const int n_cells = (p.cr1 - p.cr0) * p.ns_c;
  const int g_begin = (blockIdx.x * kWarps + warp) * p.groups_per_warp;
  const int g_end = min(g_begin + p.groups_per_warp, (n_cells + CPW - 1) / CPW * p.parts);
  if (g_begin >= g_end) return;  // whole warp

  unsigned char* wbase = smem + (size_t)warp * warp_smem(LPC, ACC);
  float4* cand = reinterpret_cast<float4*>(wbase) + ci * 9;
  float* cyv = reinterpret_cast<float*>(wbase + CPW * 9 * 16) + ci * 9;
  int* cand_k = reinterpret_cast<int*>(wbase + CPW * 9 * 20) + ci * 9;
  double* accd = reinterpret_cast<double*>(wbase + cand_bytes(LPC));
  unsigned long long* acci =
      reinterpret_cast<unsigned long long*>(wbase + cand_bytes(LPC) + 9 * 3 * 32 * sizeof(double));
  constexpr bool CPA = AL && cpa_on(ACC);
  float4* stage = reinterpret_cast<float4*>(wbase + cand_bytes(LPC) + (ACC ? kAccBytes : 0));

  const long long hw = (long long)p.h * p.w, pl = p.plane;
  const float* fimg = p.img + (long long)f * 3 * pl;
  const CRec* frec = p.rec + (long long)f * K;
  const long long img_base = (long long)f * hw;
  const unsigned rmag = p.row_magic;
  // row = j / runs_per_row via a 32-bit reciprocal (exact for j, rpr < 2^16)
  auto run_pos = [&](int jj, int& row, int& c4) {
    row = rmag ? (int)__umulhi((unsigned)jj, rmag) : jj;  // rmag = 0: one run per row
    c4 = (jj - row * p.runs_per_row) * 4;
  };
  // valid pixels of the run starting at cell column c4, image column x
  auto run_len = [&](int c4, int x) { return AL ? 4 : min(4, min(S - c4, p.w - x)); };
  // CPA: the run's three float4 are copied into this lane's stage buffer
  auto stage_run = [&](bool ok, int y, int x, int buf) {
    if (!ok) return;
    const float* q = fimg + (long long)y * p.w + x;
    float4* d = stage + buf * 96 + lane;
    const unsigned sd = (unsigned)__cvta_generic_to_shared(d);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sd), "l"(q));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sd + 512), "l"(q + pl));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sd + 1024), "l"(q + 2 * pl));
  };
  auto load_run = [&](bool ok, int y, int x, int nv, float4& Lx, float4& Ax, float4& Bx) {
    if (!ok) return;
    SPX_DCHECK(y >= 0 && y < p.h && x >= 0 && nv >= 1 && x + nv <= p.w);
    const float* q = fimg + (long long)y * p.w + x;
    if (AL) {
      Lx = __ldg(reinterpret_cast<const float4*>(q));
      Ax = __ldg(reinterpret_cast<const float4*>(q + pl));
      Bx = __ldg(reinterpret_cast<const float4*>(q + 2 * pl));
    } else {
      float l[4] = {0.f, 0.f, 0.f, 0.f}, a[4] = {0.f, 0.f, 0.f, 0.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < nv) {
          l[i] = __ldg(q + i);
          a[i] = __ldg(q + pl + i);
          b[i] = __ldg(q + 2 * pl + i);
        }
      Lx = make_float4(l[0], l[1], l[2], l[3]);
      Ax = make_float4(a[0], a[1], a[2], a[3]);
      Bx = make_float4(b[0], b[1], b[2], b[3]);
    }
  };
  // first run of the lane in its cell (LPC 32: per part, below)
  int row0 = 0, c40 = 0;
  if (LPC < 32) run_pos(ll, row0, c40);
  for (int grp = g_begin; grp < g_end; ++grp) {
    // ---- geometry (local grid) -----------------------------------------------
    // LPC 32 (one cell per warp): group = (cell, part), the part's runs
    // [j0, j1) of the cell; narrower cells take whole cells (parts == 1)
    const int cg = LPC == 32 ? grp / p.parts : grp;
    const int j0 = LPC == 32 ? (grp - cg * p.parts) * p.part_runs : 0;
    const int j1 = LPC == 32 ? min(p.runs, j0 + p.part_runs) : p.runs;
    if (LPC == 32) run_pos(j0 + ll, row0, c40);
    const int cell = p.cr0 * p.ns_c + cg * CPW + ci;
    const bool active = cg * CPW + ci < n_cells;
    const int cr = active ? cell / p.ns_c : 0;
    const int cc = active ? cell - cr * p.ns_c : 0;
    const int x_cell = cc * S, y_cell = cr * S;  // local pixel origin
    const int y_glob0 = (cr + p.row_off) * S;    // global y of the cell's row 0
    // first run of this lane (its latency overlaps the staging below)
    bool ok_n = active && j0 + ll < j1 && y_cell + row0 < p.h && x_cell + c40 < p.w;
    int row_n = row0, c4_n = c40;
    float4 Ln = make_float4(0.f, 0.f, 0.f, 0.f), An = Ln, Bn = Ln;
    int buf = 0;
    if (CPA) {
      stage_run(ok_n, y_cell + row0, x_cell + c40, 0);
      asm volatile("cp.async.commit_group;" ::: "memory");
    } else {
      load_run(ok_n, y_cell + row0, x_cell + c40, run_len(c40, x_cell + c40), Ln, An, Bn);
    }

    // ---- stage the 9 candidates (the cell's lanes, 9 / LPC each) --------------
    float mc = 0.f, mxy = 0.f, okf = 1.f;
#pragma unroll
    for (int t0 = 0; t0 < 9; t0 += LPC) {
      const int t = t0 + ll;
      if (active && t < 9) {
        const int kr = cr + off_r(t), kc = cc + off_c(t);
        float4 cp;
        float cyt = 0.f;
        if (kr >= 0 && kr < p.ns_r && kc >= 0 && kc < p.ns_c) {
          const float4* q = reinterpret_cast<const float4*>(frec + kr * p.ns_c + kc);
          const float4 v0 = __ldg(q), v1 = __ldg(q + 1);
          const float cxt = __fadd_rn(v0.w, (float)(off_c(t) * S));
          cyt = __fadd_rn(v1.x, (float)(off_r(t) * S));
          cp = make_float4(v0.x, v0.y, v0.z, cxt);
          mc = fmaxf(mc, v1.y);
          mxy = fmaxf(mxy, fmaxf(fabsf(cxt), fabsf(cyt)));
          okf = fminf(okf, v1.w);
        } else {
          // Out of the grid: colour 1e18 away makes D ~1e18, never the argmin.
          cp = make_float4(1e18f, 0.f, 0.f, 0.f);
        }
        cand[t] = cp;
        cyv[t] = cyt;
        cand_k[t] = kr * p.ns_c + kc;  // only read for in-grid winners
      }
    }
    // cell-wide maxima over the cell's lanes (xor butterfly inside the group)
#pragma unroll
    for (int o = LPC / 2; o; o >>= 1) {
      mc = fmaxf(mc, __shfl_xor_sync(0xFFFFFFFFu, mc, o));
      mxy = fmaxf(mxy, __shfl_xor_sync(0xFFFFFFFFu, mxy, o));
      okf = fminf(okf, __shfl_xor_sync(0xFFFFFFFFu, okf, o));
    }
    if (ACC) {
      float4* z = reinterpret_cast<float4*>(accd);
#pragma unroll
      for (int i = lane; i < (int)(kAccBytes / 16); i += 32) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();

    // Cell constant of 2A: k_mc*Mc + k_xy*(3*Mxy + 2S) + k_const
    float two_a_cell =
        __fmaf_rn(mc, p.k_mc, __fmaf_rn(__fmaf_rn(3.f, mxy, 2.f * S), p.k_xy, p.k_const));
    if (okf == 0.f) two_a_cell = INFINITY;

    for (int j = j0 + ll; j < j1; j += LPC) {
      const int row = row_n, c4 = c4_n;
      const bool ok = ok_n;
      float4 Lv = Ln, Av = An, Bv = Bn;
      // prefetch the lane's next run of this cell (software pipelining)
      if (j + LPC < j1) {
        run_pos(j + LPC, row_n, c4_n);
        ok_n = active && y_cell + row_n < p.h && x_cell + c4_n < p.w;
        if (CPA)
          stage_run(ok_n, y_cell + row_n, x_cell + c4_n, buf ^ 1);
        else
          load_run(ok_n, y_cell + row_n, x_cell + c4_n, run_len(c4_n, x_cell + c4_n), Ln, An, Bn);
      }
      if (CPA) {
        // this run's copies (the group before the one just issued) are done;
        // the buffer the next run is copied into was read by the previous
        // iteration, whose values are consumed by now
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        const float4* sb = stage + buf * 96 + lane;
        if (ok) {
          Lv = sb[0];
          Av = sb[32];
          Bv = sb[64];
        }
        buf ^= 1;
      }
      if (!ok) continue;
      const int y = y_cell + row, x = x_cell + c4;
      const int nv = run_len(c4, x);  // valid pixels of this run (4 when AL)
      const long long pix = img_base + (long long)y * p.w + x;  // label index
      // Channel 0 carries the certified-sum flag in its sign bit (set by the
      // engine's planar convert; channel 0 is never negative): strip it.
      const unsigned fl4 = (__float_as_uint(Lv.x) >> 31) | ((__float_as_uint(Lv.y) >> 31) << 1) |
                           ((__float_as_uint(Lv.z) >> 31) << 2) |
                           ((__float_as_uint(Lv.w) >> 31) << 3);
      const float L[4] = {fabsf(Lv.x), fabsf(Lv.y), fabsf(Lv.z), fabsf(Lv.w)};
      const float A[4] = {Av.x, Av.y, Av.z, Av.w};
      const float B[4] = {Bv.x, Bv.y, Bv.z, Bv.w};
      const unsigned long long L01 = f2_pack(L[0], L[1]), L23 = f2_pack(L[2], L[3]);
      const unsigned long long A01 = f2_pack(Av.x, Av.y), A23 = f2_pack(Av.z, Av.w);
      const unsigned long long B01 = f2_pack(Bv.x, Bv.y), B23 = f2_pack(Bv.z, Bv.w);
      const float xr0 = (float)c4;
      const unsigned long long X01 = f2_pack(xr0, xr0 + 1.f);
      const unsigned long long X23 = f2_pack(xr0 + 2.f, xr0 + 3.f);
      const float yr = (float)row;
      unsigned k1[4] = {0x7F7FFFFFu, 0x7F7FFFFFu, 0x7F7FFFFFu, 0x7F7FFFFFu};
      unsigned k2[4] = {0x7F7FFFFFu, 0x7F7FFFFFu, 0x7F7FFFFFu, 0x7F7FFFFFu};
      unsigned kp[4];  // SPX_PAIRMIN: the first key of a candidate pair
      (void)kp;
      const float w32 = p.w32;
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const float4 cv = cand[t];
        const float dyf = __fsub_rn(cyv[t], yr);
        const float dyyf = __fmul_rn(dyf, dyf);
        const unsigned long long dyy = f2_pack(dyyf, dyyf);
        const unsigned long long cl = f2_pack(cv.x, cv.x), ca = f2_pack(cv.y, cv.y),
                                 cb = f2_pack(cv.z, cv.z), cx = f2_pack(cv.w, cv.w);
        float Q[4], R[4];
        {
          unsigned long long dl = sub2(cl, L01), da = sub2(ca, A01), db = sub2(cb, B01);
          unsigned long long q = fma2(db, db, fma2(da, da, mul2(dl, dl)));
          unsigned long long dx = sub2(cx, X01);
          unsigned long long r = fma2(dx, dx, dyy);
          f2_unpack(q, Q[0], Q[1]);
          f2_unpack(r, R[0], R[1]);
        }
        {
          unsigned long long dl = sub2(cl, L23), da = sub2(ca, A23), db = sub2(cb, B23);
          unsigned long long q = fma2(db, db, fma2(da, da, mul2(dl, dl)));
          unsigned long long dx = sub2(cx, X23);
          unsigned long long r = fma2(dx, dx, dyy);
          f2_unpack(q, Q[2], Q[3]);
          f2_unpack(r, R[2], R[3]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          // D = sqrt(q) + w * sqrt(r) (MUFU.SQRT; error bound in DESIGN.md)
          const float d = __fmaf_rn(w32, sqa(R[i]), sqa(Q[i]));
          const unsigned key = (__float_as_uint(d) & ~15u) | (unsigned)t;
#if SPX_PAIRMIN
          // candidate 0 seeds the best key; later candidates merge in pairs:
          // the two smallest of {k1 <= k2} u {lo <= hi} are min(k1, lo) and
          // min(max(k1, lo), k2, hi) -- 5 min/max per 2 candidates, not 6
          if (t == 0) {
            k1[i] = key;
          } else if (t & 1) {
            kp[i] = key;
          } else {
            const unsigned lo = min(kp[i], key), hi = max(kp[i], key);
            k2[i] = min(min(k2[i], hi), max(k1[i], lo));
            k1[i] = min(k1[i], lo);
          }
#else
          k2[i] = min(k2[i], max(k1[i], key));
          k1[i] = min(k1[i], key);
#endif
        }
      }
      // certificate for the 4 pixels; uncertain ones (rare) take the exact path
      int t[4];
      bool unsure = false;
      unsigned need = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float mp = fabsf(L[i]) + fabsf(A[i]) + fabsf(B[i]);
        const float f2v = __uint_as_float(k2[i]);
        const float thr = __fmaf_rn(f2v, p.k_rel, __fmaf_rn(mp, p.k_mp, two_a_cell));
        const float gap = __fsub_rn(f2v, __uint_as_float(k1[i]));
        t[i] = (int)(k1[i] & 15u);
        // Lab comes from the engine's convert (|v| < 300): no magnitude guard
        // needed; NaN or overflow make `gap > thr` false, i.e. unsure.
        const bool u = !(gap > thr) && i < nv;
        need |= (unsigned)u << i;
        unsure |= u;
      }
      if (unsure) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (need >> i & 1u) {
            const int k = exact_argmin(p.cxy + (long long)f * K * 2, p.clab + (long long)f * K * 3,
                                       L[i], A[i], B[i], x + i, y_glob0 + row, cr, cc, p.ns_r,
                                       p.ns_c, p.xy_weight);
            const int idx = (k / p.ns_c - cr + 1) * 3 + (k % p.ns_c - cc + 1);
            t[i] = idx < 4 ? idx + 1 : (idx == 4 ? 0 : idx);  // (dr,dc) -> scan slot
          }
        }
      }
      int lab4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        SPX_DCHECK(t[i] >= 0 && t[i] < 9);
        SPX_DCHECK(i >= nv || (cand_k[t[i]] >= 0 && cand_k[t[i]] < K));
        lab4[i] = cand_k[t[i]] + p.row_off * p.ns_c;  // GLOBAL ids
      }
      SPX_DCHECK(y < p.h && x + nv <= p.w && pix + nv <= (long long)p.frames * hw);
      if (ACC) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (!AL && i >= nv) break;
          double* d = accd + t[i] * 96 + lane;
          d[0] = dadd(d[0], (double)L[i]);
          d[32] = dadd(d[32], (double)A[i]);
          d[64] = dadd(d[64], (double)B[i]);
          acci[t[i] * 32 + lane] += 1ull | ((unsigned long long)((fl4 >> i) & 1u) << 11) |
                                    ((unsigned long long)(c4 + i) << 22) |
                                    ((unsigned long long)row << 43);
        }
      }
      if (AL) {
        *reinterpret_cast<int4*>(p.labels + pix) = make_int4(lab4[0], lab4[1], lab4[2], lab4[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < nv) p.labels[pix + i] = lab4[i];
      }
    }
    if (ACC) {
      __syncwarp();
      // ---- per-cell column reduction: 9 slots x (3 colour + 1 packed int) ---
      // column c < 27: colour (slot c/3, channel c%3); 27 <= c < 36: ints of
      // slot c-27.  The LPC lane entries of a column are summed in a
      // lane-rotated order (any order is exact under the certified-sum
      // condition; flagged clusters are recomputed by k_exact_clusters) and
      // go straight into the owning cluster's accumulator with global atomics.
      constexpr int NQ = LPC / 2;  // 16-byte pairs per column
      const int lane0 = ci * LPC;
      if (active) {
        ClusterAcc* fa = p.acc + (long long)f * K;
        for (int col = ll; col < 36; col += LPC) {
          if (col < 27) {
            const double2* src = reinterpret_cast<const double2*>(accd + col * 32 + lane0);
            double sacc = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const double2 v = src[(q + ll) & (NQ - 1)];
              sacc = dadd(dadd(sacc, v.x), v.y);
            }
            // an empty (or out-of-grid) slot sums to +0.0: nothing to add
            SPX_DCHECK(sacc == 0.0 || (cand_k[col / 3] >= 0 && cand_k[col / 3] < K));
            if (sacc != 0.0) atomicAdd(&fa[cand_k[col / 3]].s[col % 3], sacc);
          } else {
            const ulonglong2* src =
                reinterpret_cast<const ulonglong2*>(acci + (col - 27) * 32 + lane0);
            // Each lane entry packs count | flags << 11 | sum_x << 22 |
            // sum_y << 43 of at most 2047 pixels (cell_path_ok).  Up to
            // S = 45 a cell has <= 2047 pixels, so the packed entries of its
            // lanes add without carries between fields; larger cells unpack.
            unsigned long long cnt = 0, flg = 0, sxr = 0, syr = 0;
            if (S <= 45) {
              unsigned long long tot = 0;
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                const ulonglong2 v = src[(q + ll) & (NQ - 1)];
                tot += v.x + v.y;
              }
              cnt = tot & 2047ull;
              flg = (tot >> 11) & 2047ull;
              sxr = (tot >> 22) & 0x1FFFFFull;
              syr = tot >> 43;
            } else {
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                const ulonglong2 v = src[(q + ll) & (NQ - 1)];
                cnt += (v.x & 2047ull) + (v.y & 2047ull);
                flg += ((v.x >> 11) & 2047ull) + ((v.y >> 11) & 2047ull);
                sxr += ((v.x >> 22) & 0x1FFFFFull) + ((v.y >> 22) & 0x1FFFFFull);
                syr += (v.x >> 43) + (v.y >> 43);
              }
            }
            if (cnt) {
              SPX_DCHECK(cand_k[col - 27] >= 0 && cand_k[col - 27] < K && flg <= cnt);
              ClusterAcc* o = fa + cand_k[col - 27];
              atomicAdd(&o->sx, sxr + cnt * (unsigned long long)x_cell);
              atomicAdd(&o->sy, syr + cnt * (unsigned long long)y_glob0);
              const unsigned long long add = cnt | (flg << 32);
              if (p.wl && flg) {
                // the contribution that turns the cluster's flag count
                // nonzero enqueues it for k_exact_clusters (exactly once)
                if ((atomicAdd(&o->cf, add) >> 32) == 0)
                  p.wl[atomicAdd(p.wl_n, 1)] = (int32_t)((long long)f * K + cand_k[col - 27]);
              } else {
                atomicAdd(&o->cf, add);
              }
            }
          }
        }
      }
    }
    __syncwarp();  // smem (candidates, accumulators) is rewritten by the next group
  }
}

namespace {

// fp32 filter records of the current centres (after init / perturb).
__global__ void k_records(const double* __restrict__ cxy, const double* __restrict__ clab,
                          CRec* __restrict__ rec, int ns_c, int s, int k_per_frame, long long n,
                          int k0, int k1, int row_off) {
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int nk = k1 - k0;
  const long long f = j / nk;
  int k = k0 + (int)(j % nk);
  const long long i = f * k_per_frame + k;
  const int kr = k / ns_c + row_off, kc = k % ns_c;
  const CRec r = make_record(cxy[2 * i], cxy[2 * i + 1], clab[3 * i], clab[3 * i + 1],
                             clab[3 * i + 2], kr, kc, s);
  rec[i] = r;
}

struct ReduceParams {
  ClusterAcc* acc;
  const float* img;
  const int32_t* labels;
  const double* prev_xy;
  const double* prev_lab;
  double* out_xy;
  double* out_lab;
  int64_t* counts;
  CRec* rec;
  const int32_t* done;
  int32_t* worklist;       // flagged clusters (global index f*K + k)
  int32_t* worklist_n;
  int32_t* wl_reset;       // (may be null) zeroed by k_reduce_cells: the next pass's count
  bool append;             // k_reduce_cells enqueues flagged clusters (else k_cell did)
  int h, w, s, ns_r, ns_c, frames, n_bl, tile_len;
  long long plane;         // planar Lab channel stride (plane_of(h * w))
  bool win_staged;         // k_exact_clusters stages the label window in smem
  float tau_strip;         // k_exact_wide: certified range of one strip's members
  int kr0, kr1;            // cluster rows reduced (local grid)
  int row_off;             // global cell row of local row 0
};

// Store cluster gk's new centre q = {l, a, b, x, y} (already divided, or
// the previous centre for an empty cluster, _core.pyx:313-320), its count and
// its fp32 record.
__device__ __forceinline__ void write_centre(const ReduceParams& p, long long gk, int kr, int kc,
                                             double cnt, const double* q) {
  const double l = q[0], a = q[1], b = q[2], x = q[3], y = q[4];
  p.out_lab[3 * gk] = l;
  p.out_lab[3 * gk + 1] = a;
  p.out_lab[3 * gk + 2] = b;
  p.out_xy[2 * gk] = x;
  p.out_xy[2 * gk + 1] = y;
  p.counts[gk] = (int64_t)cnt;
  const CRec r = make_record(x, y, l, a, b, kr + p.row_off, kc, p.s);
  p.rec[gk] = r;
}

// One lane per cluster: fixed-order sum of the 9 (cell, slot) partials that
// belong to it.  Clusters with a flagged member are recomputed by the whole
// warp with the reference strip folds + pairwise strip tree (_core.pyx:300-311).
__device__ __forceinline__ void centre_values(const ReduceParams& p, long long gk, int kr, int kc,
                                              double cnt, double sl, double sa, double sb,
                                              double sx, double sy, double* xy, double* lab,
                                              CRec& r) {
  if (cnt > 0.0) {  // _core.pyx:313-320
    // five independent IEEE divisions: branch-free fast paths first (they
    // interleave), the rare guarded-out operands redone with ddiv
    const double num[5] = {sl, sa, sb, sx, sy};
    double q[5];
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 5; ++i) ok &= ddiv_fastpath(num[i], cnt, q[i]);
    if (!ok)
#pragma unroll
      for (int i = 0; i < 5; ++i) q[i] = ddiv(num[i], cnt);
    lab[0] = q[0];
    lab[1] = q[1];
    lab[2] = q[2];
    xy[0] = q[3];
    xy[1] = q[4];
  } else {
    lab[0] = p.prev_lab[3 * gk];
    lab[1] = p.prev_lab[3 * gk + 1];
    lab[2] = p.prev_lab[3 * gk + 2];
    xy[0] = p.prev_xy[2 * gk];
    xy[1] = p.prev_xy[2 * gk + 1];
  }
  r.l = __double2float_rn(lab[0]);
  r.a = __double2float_rn(lab[1]);
  r.b = __double2float_rn(lab[2]);
  r.xr = __double2float_rn(dsub(xy[0], (double)kc * p.s));
  r.yr = __double2float_rn(dsub(xy[1], (double)(kr + p.row_off) * p.s));
  r.mag_lab = fmaxf(fabsf(r.l), fmaxf(fabsf(r.a), fabsf(r.b)));
  r.mag_xy = fmaxf(fabsf(r.xr), fabsf(r.yr));
  r.ok = (fin_small(xy[0]) && fin_small(xy[1]) && fin_small(lab[0]) && fin_small(lab[1]) &&
          fin_small(lab[2]))
             ? 1.f
             : 0.f;
}

// One thread per cluster: the sums of the cell partials, divided as in
// _core.pyx:313-320; the block's 128 consecutive clusters are staged in
// shared memory and written out with coalesced 16-byte stores (the per-
// cluster AoS records would otherwise leave as 8 scattered stores per
// thread).  Flagged clusters are left to k_exact_clusters (which may run
// concurrently on another stream).
constexpr int kRedT = 128;
#ifndef SPX_REDPER
#define SPX_REDPER 1
#endif
constexpr int kRedPer = SPX_REDPER;  // clusters per thread: their loads are in flight together
constexpr int kRedN = kRedT * kRedPer;

__device__ __forceinline__ void reduce_cells_body(const ReduceParams& p, int bx, int f) {
  __shared__ __align__(16) double s_xy[kRedN * 2];
  __shared__ __align__(16) double s_lab[kRedN * 3];
  __shared__ __align__(16) long long s_cnt[kRedN];
  __shared__ __align__(16) CRec s_rec[kRedN];
  __shared__ bool s_fl[kRedN];  // flagged: k_exact_clusters owns its outputs
  if (p.wl_reset && bx == 0 && f == 0 && threadIdx.x == 0) *p.wl_reset = 0;
  const int K = p.ns_r * p.ns_c;
  const int nk = (p.kr1 - p.kr0) * p.ns_c;
  if (p.done && p.done[f]) return;  // whole block: one frame
  const int j0 = bx * kRedN;
  const int n = min(kRedN, nk - j0);
  const long long gk0 = (long long)f * K + p.kr0 * p.ns_c + j0;
  const int t = threadIdx.x;
  double4 s012[kRedPer];
  ulonglong2 syc[kRedPer];
#pragma unroll
  for (int c = 0; c < kRedPer; ++c) {
    const int i = c * kRedT + t;
    if (i < n) {
      const ClusterAcc* a = p.acc + gk0 + i;
      s012[c] = *reinterpret_cast<const double4*>(a);  // s[0..2], sx
      syc[c] = *reinterpret_cast<const ulonglong2*>(&a->sy);
    }
  }
#pragma unroll
  for (int c = 0; c < kRedPer; ++c) {
    const int i = c * kRedT + t;
    if (i >= n) break;
    const long long gk = gk0 + i;
    const int k = p.kr0 * p.ns_c + j0 + i;
    const int kr = k / p.ns_c, kc = k - kr * p.ns_c;
    ClusterAcc* a = p.acc + gk;
    // consume and clear for the next pass
    *reinterpret_cast<double4*>(a) = make_double4(0.0, 0.0, 0.0, 0.0);
    *reinterpret_cast<ulonglong2*>(&a->sy) = make_ulonglong2(0ull, 0ull);
    const unsigned long long sx = (unsigned long long)__double_as_longlong(s012[c].w);
    const unsigned long long cnt = syc[c].y & 0xFFFFFFFFull, fl = syc[c].y >> 32;
    if (fl != 0 && p.append) p.worklist[atomicAdd(p.worklist_n, 1)] = (int32_t)gk;
    s_fl[i] = fl != 0;
    centre_values(p, gk, kr, kc, (double)cnt, s012[c].x, s012[c].y, s012[c].z, (double)sx,
                  (double)syc[c].x, s_xy + 2 * i, s_lab + 3 * i, s_rec[i]);
    s_cnt[i] = (long long)cnt;
  }
  __syncthreads();
  // coalesced copies of the block's contiguous output ranges, flagged
  // clusters skipped (k_exact_clusters may run concurrently and owns them)
  {
    const double2* sx2 = reinterpret_cast<const double2*>(s_xy);
    double2* gx2 = reinterpret_cast<double2*>(p.out_xy + 2 * gk0);
    for (int i = t; i < n; i += kRedT)
      if (!s_fl[i]) gx2[i] = sx2[i];
    double* gl = p.out_lab + 3 * gk0;
    for (int i = t; i < 3 * n; i += kRedT)
      if (!s_fl[i / 3]) gl[i] = s_lab[i];
    for (int i = t; i < n; i += kRedT)
      if (!s_fl[i]) p.counts[gk0 + i] = s_cnt[i];
    const float4* sr = reinterpret_cast<const float4*>(s_rec);
    float4* gr = reinterpret_cast<float4*>(p.rec + gk0);
    for (int i = t; i < 2 * n; i += kRedT)
      if (!s_fl[i >> 1]) gr[i] = sr[i];
  }
}

__global__ void __launch_bounds__(kRedT) k_reduce_cells(ReduceParams p) {
  reduce_cells_body(p, blockIdx.x, blockIdx.y);
}

// Exact recomputation of flagged clusters (certificate failed).  One block
// per cluster, built for latency -- at small batches this kernel's chain of
// dependent steps IS the pass's update time:
//  (1) the worklist count and the block's first item load together;
//  (2) the 3S x 3S window of labels is staged into shared memory with one
//      round of cp.async (16-byte copies when aligned);
//  (3) each warp takes row strips (strip j = rows [ry0 + j*tile_len, ...),
//      an independent reference fold from 0.0, _core.pyx:233-243) and walks
//      the strip in row-major order, 4 x 32 window positions per step: a
//      ballot finds the members and their row-major ranks, the members'
//      L / a / b are copied with cp.async into a compact array, and lanes
//      0..2 fold the three channels in order once the array is half full and
//      at the end of the strip (one fold per strip in practice);
//  (4) lanes 0..5 of warp 0 run the pairwise strip tree (_core.pyx:300-311)
//      for one component each and lanes 0..4 divide one component each.
// Pipeline labels never spill, so the window holds every member.
#ifndef SPX_EXW
#define SPX_EXW 3
#endif
#ifndef SPX_EXG
#define SPX_EXG 16
#endif
constexpr int kExWarps = SPX_EXW;  // 3 = n_bl for the default tile_len 16 (3S / 16 strips when S = 16)
constexpr int kExCap = 256;        // compacted members per warp and fold round

constexpr int kExMaxStrips = 64;   // n_bl <= 64 (cell_path_ok)
// The 3S x 3S window of labels is staged in shared memory up to this size;
// larger windows (S > 48) are read from global memory (L2) in place.
constexpr size_t kExWinSmemMax = 88 * 1024;
size_t exact_win_bytes(int64_t s) { return (size_t)9 * s * s * sizeof(int32_t); }
bool exact_win_staged(int64_t s) { return exact_win_bytes(s) <= kExWinSmemMax; }
size_t exact_smem_bytes(int64_t s) {  // compact values + the window's labels (staged)
  return (size_t)kExWarps * 3 * kExCap * sizeof(float) +
         (exact_win_staged(s) ? exact_win_bytes(s) : 0);
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Warp 0 of an exact-fallback block, after the strips' sums are in
// strips[0..n_bl): lane t < 6 runs the pairwise strip tree of component t
// (_core.pyx:300-311), lanes 0..4 divide one component each
// (_core.pyx:313-320), lane 0 stores.
__device__ __forceinline__ void finish_cluster(const ReduceParams& p, double (*strips)[6],
                                               double* qv, int gk, int r, int c, int lane) {
  if (lane < 6) {
    int m = p.n_bl;
#pragma unroll 1
    while (m > 1) {
      const int half = m >> 1;
#pragma unroll 1
      for (int i = 0; i < half; ++i)
        strips[i][lane] = dadd(strips[2 * i][lane], strips[2 * i + 1][lane]);
      if (m & 1) strips[half][lane] = strips[m - 1][lane];
      m = half + (m & 1);
    }
  }
  __syncwarp();
  const double cnt = strips[0][5];
  if (lane < 5) {
    double q;
    if (cnt > 0.0) {
      q = ddiv_ilp(strips[0][lane], cnt);
    } else {  // empty: keep the previous centre
      q = lane < 3 ? p.prev_lab[3LL * gk + lane] : p.prev_xy[2LL * gk + (lane - 3)];
    }
    qv[lane] = q;
  }
  __syncwarp();
  if (lane == 0) write_centre(p, gk, r, c, cnt, qv);
}

// Items first, first + stride, ... of the worklist; blocks of >= kExWarps
// warps (warps beyond kExWarps only help stage the window).
__device__ __forceinline__ void exact_clusters_body(const ReduceParams& p, int first, int stride) {
  extern __shared__ __align__(16) unsigned char ex_smem[];
  __shared__ double strips[kExMaxStrips][6];
  __shared__ double qv[6];
  float* const cv_all = reinterpret_cast<float*>(ex_smem);  // [kExWarps][3][kExCap]
  int32_t* const win_s = reinterpret_cast<int32_t*>(cv_all + kExWarps * 3 * kExCap);
  const bool staged = p.win_staged;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* const cw = cv_all + warp * 3 * kExCap;
  const int K = p.ns_r * p.ns_c;
  const long long hw = (long long)p.h * p.w;
  const long long cap = (long long)p.frames * K;  // worklist capacity
  // (1) independent loads: the count and this block's first item (in bounds)
  const int n = *p.worklist_n;
  int gk_next = (long long)first < cap ? p.worklist[first] : 0;
  for (int item = first; item < n; item += stride) {
    const int gk = gk_next;
    if (item + (long long)stride < n) gk_next = p.worklist[item + stride];
    const int ff = gk / K, fk = gk - ff * K;
    // a frame that stopped early has no update this pass (k_cell enqueued its
    // clusters during its final association)
    if (p.done && p.done[ff]) continue;  // block-uniform
    const float* im = p.img + (long long)ff * 3 * p.plane;  // planar [3][plane]
    const int32_t* lb = p.labels + (long long)ff * hw;
    const int r = fk / p.ns_c, c = fk - r * p.ns_c;
    const int gid = fk + p.row_off * p.ns_c;  // labels carry global ids
    const int wx0 = max((c - 1) * p.s, 0), wx1 = min((c + 2) * p.s, p.w);
    const int ry0 = (r - 1) * p.s, ry1 = min((r + 2) * p.s, p.h);
    const int ya0 = max(ry0, 0);
    const int ww = wx1 - wx0, wrows = ry1 - ya0;
    SPX_DCHECK(gk >= 0 && (long long)gk < cap && ww > 0 && ww <= 3 * p.s && wrows > 0 &&
               wrows <= 3 * p.s && p.n_bl <= kExMaxStrips);
    // the window's labels: staged (row stride ww) or in place (row stride w)
    const int32_t* const win = staged ? win_s : lb + (long long)ya0 * p.w + wx0;
    const int wst = staged ? ww : p.w;
    // (2) the window's labels, one round trip
    if (!staged) {
    } else if (((wx0 | ww | p.w) & 3) == 0) {
      const int q4 = ww >> 2;
#pragma unroll 1
      for (int i = threadIdx.x; i < wrows * q4; i += blockDim.x) {
        const int rr = i / q4, cq = i - rr * q4;
        SPX_DCHECK(rr * ww + 4 * cq + 4 <= 9 * p.s * p.s);
        cp_async16(win_s + rr * ww + 4 * cq, lb + (long long)(ya0 + rr) * p.w + wx0 + 4 * cq);
      }
    } else {
#pragma unroll 1
      for (int i = threadIdx.x; i < wrows * ww; i += blockDim.x) {
        const int rr = i / ww, cc = i - rr * ww;
        SPX_DCHECK(i < 9 * p.s * p.s);
        cp_async4(win_s + i, lb + (long long)(ya0 + rr) * p.w + wx0 + cc);
      }
    }
#pragma unroll 1
    for (int i = threadIdx.x; i < p.n_bl * 6; i += blockDim.x) (&strips[0][0])[i] = 0.0;
    cp_async_wait_all();
    __syncthreads();
    // (3) strips: row-major walk of the strip's window rectangle, 4 x 32
    // positions per step (position i = row i / ww, column i % ww); a ballot
    // per 32 positions gives the members their row-major ranks
    const int dq = 32 / ww, dr = 32 - dq * ww;
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll 1
    for (int j = warp; warp < kExWarps && j < p.n_bl; j += kExWarps) {
      const int ya = max(ry0 + j * p.tile_len, 0);
      const int yz = min(ry0 + (j + 1) * p.tile_len, ry1);
      if (ya >= yz) continue;  // warp-uniform
      const int n_rect = (yz - ya) * ww;
      double acc = 0.0;                           // lanes 0..2: channel fold
      unsigned long long lx = 0, ly = 0, lc = 0;  // lane sums of x, global y, count
      int rr = lane / ww, cc = lane - (lane / ww) * ww;  // this lane's position
      int o = 0;                                  // members copied, not yet folded
      // lanes 0..2 fold the copied members of one channel each, in order;
      // channel 0 carries the certified-sum flag in its sign bit: |L|
      auto fold = [&]() {
        cp_async_wait_all();
        __syncwarp();
        if (lane < 3) {
          const float* src = cw + lane * kExCap;
          const bool l0 = lane == 0;
          int i = 0;
#pragma unroll 4
          for (; i + 4 <= o; i += 4) {
            float v0 = src[i], v1 = src[i + 1], v2 = src[i + 2], v3 = src[i + 3];
            if (l0) {
              v0 = fabsf(v0);
              v1 = fabsf(v1);
              v2 = fabsf(v2);
              v3 = fabsf(v3);
            }
            acc = dadd(acc, (double)v0);
            acc = dadd(acc, (double)v1);
            acc = dadd(acc, (double)v2);
            acc = dadd(acc, (double)v3);
          }
#pragma unroll 1
          for (; i < o; ++i) acc = dadd(acc, (double)(l0 ? fabsf(src[i]) : src[i]));
        }
        __syncwarp();
        o = 0;
      };
#pragma unroll 1
      for (int base = 0; base < n_rect; base += 128) {
        if (o > kExCap - 128) fold();  // room for this step's members
        int ry[4], cx[4];
        bool hit[4];
        unsigned msk[4];
        ry[0] = rr;
        cx[0] = cc;
#pragma unroll
        for (int u = 1; u < 4; ++u) {
          ry[u] = ry[u - 1] + dq;
          cx[u] = cx[u - 1] + dr;
          if (cx[u] >= ww) {
            cx[u] -= ww;
            ++ry[u];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool in = base + 32 * u + lane < n_rect;
          SPX_DCHECK(!in || (ya + ry[u] < ya0 + wrows && cx[u] >= 0 && cx[u] < ww));
          hit[u] = in && win[(long long)(ya - ya0 + ry[u]) * wst + cx[u]] == gid;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) msk[u] = __ballot_sync(0xFFFFFFFFu, hit[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (hit[u]) {
            const int q = o + __popc(msk[u] & lt_mask);
            SPX_DCHECK(q < kExCap);
            const int y = ya + ry[u];
            const float* g0 = im + (long long)y * p.w + wx0 + cx[u];
            cp_async4(cw + q, g0);
            cp_async4(cw + kExCap + q, g0 + p.plane);
            cp_async4(cw + 2 * kExCap + q, g0 + 2 * p.plane);
            lx += (unsigned long long)(wx0 + cx[u]);
            ly += (unsigned long long)(y + p.row_off * p.s);
            lc += 1;
          }
          o += __popc(msk[u]);
        }
        rr = ry[3] + dq;
        cc = cx[3] + dr;
        if (cc >= ww) {
          cc -= ww;
          ++rr;
        }
      }
      if (o) fold();
#pragma unroll
      for (int sh = 16; sh; sh >>= 1) {
        lx += __shfl_xor_sync(0xFFFFFFFFu, lx, sh);
        ly += __shfl_xor_sync(0xFFFFFFFFu, ly, sh);
        lc += __shfl_xor_sync(0xFFFFFFFFu, lc, sh);
      }
      if (lane < 3) strips[j][lane] = acc;
      if (lane == 0) {
        strips[j][3] = (double)lx;
        strips[j][4] = (double)ly;
        strips[j][5] = (double)lc;
      }
    }
    __syncthreads();
    // (4) warp 0: strip tree, divisions, store
    if (warp == 0) finish_cluster(p, strips, qv, gk, r, c, lane);
    __syncthreads();  // the window and strips are reused by the next item
  }
}

__global__ void __launch_bounds__(kExWarps * 32) k_exact_clusters(ReduceParams p) {
  exact_clusters_body(p, blockIdx.x, gridDim.x);
}

// The update of one pass as ONE launch (single-stream engine path): blocks
// [0, red_blocks * frames) reduce (k_reduce_cells), the rest run the exact
// fallback over the worklist k_cell filled (k_exact_clusters) -- the two
// parts are independent, and one launch replaces a fork / join across two
// streams (the chain a single frame waits on).
__global__ void __launch_bounds__(kRedT) k_update(ReduceParams p, int red_blocks) {
  const int nred = red_blocks * p.frames;
  if ((int)blockIdx.x < nred)
    reduce_cells_body(p, blockIdx.x % red_blocks, blockIdx.x / red_blocks);
  else
    exact_clusters_body(p, blockIdx.x - nred, gridDim.x - nred);
}

// Exact recomputation for large cells (S > 32), where most clusters are
// flagged (the certified range 2^k <= |v| < 128 narrows as 9 S^2 grows).
// One block of kWideWarps warps per cluster, warp w taking strips w,
// w + kWideWarps, ... (an independent reference fold each,
// _core.pyx:233-243).  A strip has at most tile_len * 3S members, so a much
// wider range is certified per strip: if every member value of a channel is
// 0 or tau_strip <= |v| < 128 (tau_strip = 2^k with tile_len * 3S <=
// 2^(23+k)), every partial sum of that channel is exact and the strip's
// fold equals any-order sum -- lanes accumulate their members in binary64
// and the warp adds the lane sums.  Only channels with an uncertified member
// (rare) are refolded sequentially: row-major units of 256 columns, labels
// and values loaded coalesced, members found by ballot, lanes 0..2 folding
// in order with the values arriving by shuffle.
constexpr int kWideWarps = 8;
// kWideCh: 32-column chunks per unit (8, 12 or 16 by window width, so a
// window row of up to 512 columns is one unit)
template <int kWideCh>
__global__ void __launch_bounds__(kWideWarps * 32) k_exact_wide(ReduceParams p) {
  __shared__ double strips[kExMaxStrips][6];
  __shared__ double qv[6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = p.ns_r * p.ns_c;
  const long long hw = (long long)p.h * p.w;
  const int n = *p.worklist_n;
  const unsigned tau_bits = __float_as_uint(p.tau_strip);
  for (int item = blockIdx.x; item < n; item += gridDim.x) {
    const int gk = p.worklist[item];
    const int ff = gk / K, fk = gk - ff * K;
    if (p.done && p.done[ff]) continue;  // block-uniform
    const float* im = p.img + (long long)ff * 3 * p.plane;
    const int32_t* lb = p.labels + (long long)ff * hw;
    const int r = fk / p.ns_c, c = fk - r * p.ns_c;
    const int gid = fk + p.row_off * p.ns_c;
    const int wx0 = max((c - 1) * p.s, 0), wx1 = min((c + 2) * p.s, p.w);
    const int ry0 = (r - 1) * p.s, ry1 = min((r + 2) * p.s, p.h);
    const int nseg = (wx1 - wx0 + 32 * kWideCh - 1) / (32 * kWideCh);
    SPX_DCHECK(gk >= 0 && gk < p.frames * K && p.n_bl <= kExMaxStrips && wx1 > wx0);
#pragma unroll 1
    for (int i = threadIdx.x; i < p.n_bl * 6; i += blockDim.x) (&strips[0][0])[i] = 0.0;
    __syncthreads();
#pragma unroll 1
    for (int j = warp; j < p.n_bl; j += kWideWarps) {
      const int ya = max(ry0 + j * p.tile_len, 0);
      const int yz = min(ry0 + (j + 1) * p.tile_len, ry1);
      if (ya >= yz) continue;  // warp-uniform
      const int units = (yz - ya) * nseg;
      auto unit_xy = [&](int u, int& y, int& x0) {
        y = ya + u / nseg;
        x0 = wx0 + (u % nseg) * 32 * kWideCh + lane;
      };
      // ---- pass 1: lane sums of the members (exact if certified) ---------
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      unsigned bad = 0;  // channels with an uncertified member (bits 0..2)
      unsigned long long lx = 0, ly = 0, lc = 0;
      int lb_n[kWideCh];
      auto load_labels = [&](int u) {
        int y, x0;
        unit_xy(u, y, x0);
        const long long row = (long long)y * p.w;
#pragma unroll
        for (int ch = 0; ch < kWideCh; ++ch) {
          const int x = x0 + 32 * ch;
          lb_n[ch] = x < wx1 ? __ldg(lb + row + x) : -1;
        }
      };
      auto cert = [&](float v) {  // 0, or tau_strip <= |v| < 128
        const unsigned a = __float_as_uint(v) & 0x7FFFFFFFu;
        return a == 0u || (a >= tau_bits && a < 0x43000000u);
      };
      load_labels(0);
#pragma unroll 1
      for (int u = 0; u < units; ++u) {
        int lbv[kWideCh];
#pragma unroll
        for (int ch = 0; ch < kWideCh; ++ch) lbv[ch] = lb_n[ch];
        if (u + 1 < units) load_labels(u + 1);  // the next unit's labels in flight
        int y, x0;
        unit_xy(u, y, x0);
        const long long row = (long long)y * p.w;
        const unsigned long long yg = (unsigned long long)(y + p.row_off * p.s);
        float lv[kWideCh], av[kWideCh], bv[kWideCh];
#pragma unroll
        for (int ch = 0; ch < kWideCh; ++ch) {  // member values only (one read per pixel)
          const bool hit = lbv[ch] == gid;
          const long long o = row + x0 + 32 * ch;
          lv[ch] = hit ? fabsf(__ldg(im + o)) : 0.f;  // channel 0: |L| (flag bit)
          av[ch] = hit ? __ldg(im + p.plane + o) : 0.f;
          bv[ch] = hit ? __ldg(im + 2 * p.plane + o) : 0.f;
        }
#pragma unroll
        for (int ch = 0; ch < kWideCh; ++ch) {
          if (lbv[ch] == gid) {
            s0 = dadd(s0, (double)lv[ch]);
            s1 = dadd(s1, (double)av[ch]);
            s2 = dadd(s2, (double)bv[ch]);
            bad |= (cert(lv[ch]) ? 0u : 1u) | (cert(av[ch]) ? 0u : 2u) | (cert(bv[ch]) ? 0u : 4u);
            lx += (unsigned long long)(x0 + 32 * ch);
            ly += yg;
            ++lc;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        lx += __shfl_xor_sync(0xFFFFFFFFu, lx, o);
        ly += __shfl_xor_sync(0xFFFFFFFFu, ly, o);
        lc += __shfl_xor_sync(0xFFFFFFFFu, lc, o);
        s0 = dadd(s0, __shfl_xor_sync(0xFFFFFFFFu, s0, o));
        s1 = dadd(s1, __shfl_xor_sync(0xFFFFFFFFu, s1, o));
        s2 = dadd(s2, __shfl_xor_sync(0xFFFFFFFFu, s2, o));
        bad |= __shfl_xor_sync(0xFFFFFFFFu, bad, o);
      }
      // ---- pass 2 (uncertified channels): the reference's ordered fold ----
      double acc = lane == 0 ? s0 : (lane == 1 ? s1 : s2);
      if (bad) {  // warp-uniform
        const bool mine = lane < 3 && (bad >> lane & 1u);
        if (mine) acc = 0.0;
#pragma unroll 1
        for (int u = 0; u < units; ++u) {
          int y, x0;
          unit_xy(u, y, x0);
          const long long row = (long long)y * p.w;
#pragma unroll 1
          for (int ch = 0; ch < kWideCh; ++ch) {
            const int x = x0 + 32 * ch;
            const bool hit = x < wx1 && __ldg(lb + row + x) == gid;
            unsigned m = __ballot_sync(0xFFFFFFFFu, hit);
            float v0 = 0.f, v1 = 0.f, v2 = 0.f;
            if (hit) {
              v0 = fabsf(__ldg(im + row + x));
              v1 = __ldg(im + p.plane + row + x);
              v2 = __ldg(im + 2 * p.plane + row + x);
            }
            while (m) {  // warp-uniform: members in column order
              const int b = __ffs(m) - 1;
              m &= m - 1;
              const float w0 = __shfl_sync(0xFFFFFFFFu, v0, b);
              const float w1 = __shfl_sync(0xFFFFFFFFu, v1, b);
              const float w2 = __shfl_sync(0xFFFFFFFFu, v2, b);
              const float v = lane == 0 ? w0 : (lane == 1 ? w1 : w2);
              if (mine) acc = dadd(acc, (double)v);
            }
          }
        }
      }
      if (lane < 3) strips[j][lane] = acc;
      if (lane == 0) {
        strips[j][3] = (double)lx;
        strips[j][4] = (double)ly;
        strips[j][5] = (double)lc;
      }
    }
    __syncthreads();
    if (warp == 0) finish_cluster(p, strips, qv, gk, r, c, lane);
    __syncthreads();  // strips are reused by the next item
  }
}

// ---- wide cells (S > 42): per-(cluster, strip) sums ------------------------
//
// With large cells nearly every cluster has a member outside the certified
// range 2^k <= |v| < 128 (9 S^2 <= 2^(23+k): S = 118 needs |v| >= 2^-6), so
// the cluster-level certificate of k_cell fails everywhere and the exact
// fallback re-reads each cluster's 3S x 3S window -- every pixel nine times.
// The reference's strips are the natural unit instead: a strip holds at most
// tile_len * 3S members, so its own certified range is far wider (S = 118:
// |v| >= 2^-10; 0.7% of strip channels fail on random frames).  Wide mode:
//  (A) k_strip_acc reads every pixel once (its label and Lab) and adds it to
//      its cluster's strip: one warp per cell walks the cell row by row
//      into lane-private per-slot accumulators (as k_cell) and, whenever the
//      rows of a slot row's clusters cross a strip boundary, sums the slot
//      columns and adds them to the (cluster, strip) entry with atomics --
//      exact in any order for a certified channel.  A channel with an
//      uncertified member marks the entry; the first mark enqueues it.
//  (B) k_strip_refold folds each marked channel again in the reference's
//      row-major order (_core.pyx:233-243) over the strip's window rows.
//  (C) k_reduce_strips runs the pairwise strip tree and the divisions
//      (_core.pyx:300-320) per cluster and clears the entries.
struct WideParams {
  const float* img;        // planar Lab [F][3][plane]
  const int32_t* labels;   // [F][H][W]
  StripAcc* sacc;          // [F][K][n_bl]
  const int32_t* done;
  long long* wl;           // (gk << 8) | strip, entries with an uncertified channel
  int32_t* wl_n;
  int h, w, s, ns_r, ns_c, frames, n_bl, tile_len;
  long long plane;
  unsigned long long ns_c_magic;   // ceil(2^64 / ns_c): k / ns_c = umul64hi(k, magic)
  int bands, band_rows;            // k_strip_acc: warps per cell, rows per warp
};

constexpr int kWideAccBytes = 9 * 3 * 32 * 8 + 9 * 32 * 8 + 9 * 32;  // colour, ints, bad bits
constexpr int kWideWarpSmem = (kWideAccBytes + 15) & ~15;

// kPx: pixels per lane and cell row, ceil(S / 32); SG: fewer than 3 cluster
// columns (slots from a division instead of the id offset)
// Warps per k_strip_acc block (4: 16 3631x3859 frames, S = 118 / 84: 16.8 /
// 17.6 ms per call; 2: 17.3 / 17.4 -- mixed, 4 kept; more than 4 need the
// dynamic shared-memory opt-in)
#ifndef SPX_SACC_WARPS
#define SPX_SACC_WARPS 4
#endif
constexpr int kSaccWarps = SPX_SACC_WARPS;
template <int kPx, bool SG>
__global__ void __launch_bounds__(kSaccWarps * 32) k_strip_acc(WideParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.y;
  if (p.done && p.done[f] == 1) return;  // whole block: one frame
  const int K = p.ns_r * p.ns_c;
  const int wid = blockIdx.x * kSaccWarps + warp;
  const int cell = wid / p.bands, band = wid - cell * p.bands;
  if (cell >= K) return;  // whole warp
  unsigned char* wb = smem + warp * kWideWarpSmem;
  double* accd = reinterpret_cast<double*>(wb);                                  // [9][3][32]
  unsigned long long* acci = reinterpret_cast<unsigned long long*>(wb + 6912);   // [9][32]
  unsigned char* badb = wb + 6912 + 2304;                                        // [9][32]
  for (int i = lane; i < kWideAccBytes / 16; i += 32)
    reinterpret_cast<float4*>(wb)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int S = p.s;
  const int cr = cell / p.ns_c, cc = cell - cr * p.ns_c;
  const int x_cell = cc * S, y_cell = cr * S;
  const int cols = min(S, p.w - x_cell);
  // this warp's band of the cell's rows (small launches split cells)
  const int yl0 = band * p.band_rows, rows = min(min(S, p.h - y_cell), yl0 + p.band_rows);
  if (yl0 >= rows) return;  // whole warp
  SPX_DCHECK(cols > 0 && cols <= 32 * kPx);
  const long long hw = (long long)p.h * p.w;
  const float* fimg = p.img + (long long)f * 3 * p.plane;
  const int32_t* flab = p.labels + (long long)f * hw;
  StripAcc* fsa = p.sacc + (long long)f * K * p.n_bl;
  const bool small_grid = SG;
  const long long pl = p.plane;
  const int ns_c = p.ns_c;
  const int kbase = (cr - 1) * p.ns_c + (cc - 1);  // id of slot (0, 0)
  // a lane's pixels of a cell row: columns lane, lane + 32, ... (coalesced
  // 4-byte loads)
  int lb[kPx];
  float L[kPx], A[kPx], B[kPx];
  // per-lane row pointers, advanced one image row per load (the band's
  // first row first)
  const long long o0 = (long long)(y_cell + yl0) * p.w + x_cell + lane;
  const int32_t* lr = flab + o0;
  const float* ir0 = fimg + o0;
  const float* ir1 = ir0 + pl;
  const float* ir2 = ir0 + 2 * pl;
  const int w = p.w;
  auto load_row = [&]() {
#pragma unroll
    for (int u = 0; u < kPx; ++u) {
      const bool in = lane + 32 * u < cols;
      lb[u] = in ? lr[32 * u] : 0;
      L[u] = in ? __ldg(ir0 + 32 * u) : 0.f;
      A[u] = in ? __ldg(ir1 + 32 * u) : 0.f;
      B[u] = in ? __ldg(ir2 + 32 * u) : 0.f;
    }
    lr += w;
    ir0 += w;
    ir1 += w;
    ir2 += w;
  };
  // next strip boundary (last row of a strip) of each slot row dr: rows yl
  // with yl + 1 + (2 - dr) S a multiple of tile_len
  int nb[3];
#pragma unroll
  for (int dr = 0; dr < 3; ++dr) {
    const int m = ((2 - dr) * S + 1) % p.tile_len;
    const int b0 = m ? p.tile_len - m : 0;  // first boundary row of the cell
    nb[dr] = yl0 <= b0 ? b0 : b0 + (yl0 - b0 + p.tile_len - 1) / p.tile_len * p.tile_len;
  }
  load_row();
  __syncwarp();
#pragma unroll 1
  for (int yl = yl0; yl < rows; ++yl) {
    int clb[kPx];
    float cL[kPx], cA[kPx], cB[kPx];
#pragma unroll
    for (int u = 0; u < kPx; ++u) {
      clb[u] = lb[u];
      cL[u] = L[u];
      cA[u] = A[u];
      cB[u] = B[u];
    }
    if (yl + 1 < rows) load_row();  // the next row's loads in flight
    const unsigned long long pk_row = 1ull | ((unsigned long long)yl << 43);
    // a lane's pixels of one slot are summed in registers first
    int tc = -1;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
    unsigned long long ci = 0;
    unsigned cb = 0;
    auto put = [&]() {
      double* d = accd + tc * 96 + lane;
      d[0] = dadd(d[0], c0);
      d[32] = dadd(d[32], c1);
      d[64] = dadd(d[64], c2);
      acci[tc * 32 + lane] += ci;
      badb[tc * 32 + lane] |= (unsigned char)cb;
    };
#pragma unroll
    for (int u = 0; u < kPx; ++u) {
      const int xr = lane + 32 * u;  // cell-relative column
      if (xr >= cols) break;
      int t;  // slot (dr, dc), row-major
      if (small_grid) {
        const unsigned k = (unsigned)clb[u];
        const int kr = p.ns_c_magic ? (int)__umul64hi((unsigned long long)k, p.ns_c_magic)
                                    : (int)k;
        const int kc = (int)k - kr * p.ns_c;
        t = (kr - cr + 1) * 3 + (kc - cc + 1);
      } else {  // ns_c >= 3: the offset from slot 0's id names the slot
        const int dk = clb[u] - kbase;
        const int dr = (dk >= ns_c) + (dk >= 2 * ns_c);
        t = dr * 3 + (dk - dr * ns_c);
      }
      SPX_DCHECK(t >= 0 && t < 9);
      // channel 0's sign bit: the engine's convert flags pixels with a
      // channel outside the strip's certified range (wide mode); such a
      // strip has all three channels refolded
      const unsigned bits = __float_as_uint(cL[u]);
      const float l = __uint_as_float(bits & 0x7FFFFFFFu);
      const unsigned bb = (bits >> 31) * 7u;
      const unsigned long long pk = pk_row + ((unsigned long long)xr << 22);
      // branch-free run merge: a new slot spills the old run (rare) and
      // restarts the sums from zero (0.0 + v == v exactly)
      const bool same = t == tc;
      if (!same && tc >= 0) put();
      c0 = dadd(same ? c0 : 0.0, (double)l);
      c1 = dadd(same ? c1 : 0.0, (double)cA[u]);
      c2 = dadd(same ? c2 : 0.0, (double)cB[u]);
      ci = (same ? ci : 0ull) + pk;
      cb = (same ? cb : 0u) | bb;
      tc = t;
    }
    if (tc >= 0) put();
    // Slot row dr holds clusters of cluster row cr - 1 + dr, whose windows
    // start at row (cr + dr - 2) S: their strips end where
    // yl + 1 + (2 - dr) S is a multiple of tile_len (or at the cell's end).
#pragma unroll
    for (int dr = 0; dr < 3; ++dr) {
      const int rel = yl + (2 - dr) * S;  // row yl from the window top
      if (yl == nb[dr]) nb[dr] += p.tile_len;
      else if (yl + 1 < rows) continue;  // warp-uniform
      const int kr = cr - 1 + dr;
      if (kr < 0 || kr >= p.ns_r) continue;
      const int j = rel / p.tile_len;
      SPX_DCHECK(j >= 0 && j < p.n_bl);
      __syncwarp();
      // the slot row's three slots: each lane takes its own entries, the
      // warp reduces them (any order: exact for certified channels; marked
      // ones are refolded by k_strip_refold), lane 0 adds them to the entry
#pragma unroll 1
      for (int dc = 0; dc < 3; ++dc) {
        const int kc = cc - 1 + dc, t = dr * 3 + dc;
        if (kc < 0 || kc >= p.ns_c) continue;  // warp-uniform (no members)
        const unsigned long long v = acci[t * 32 + lane];
        const unsigned cnt = __reduce_add_sync(0xFFFFFFFFu, (unsigned)(v & 2047ull));
        if (cnt == 0u) continue;  // nothing added since the last flush (entries zero)
        const unsigned sxr = __reduce_add_sync(0xFFFFFFFFu, (unsigned)((v >> 22) & 0x1FFFFFull));
        const unsigned syr = __reduce_add_sync(0xFFFFFFFFu, (unsigned)(v >> 43));
        const unsigned bad = __reduce_or_sync(0xFFFFFFFFu, (unsigned)badb[t * 32 + lane]);
        double* d = accd + t * 96 + lane;
        double s0 = d[0], s1 = d[32], s2 = d[64];
        d[0] = 0.0;
        d[32] = 0.0;
        d[64] = 0.0;
        acci[t * 32 + lane] = 0ull;
        badb[t * 32 + lane] = 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          s0 = dadd(s0, __shfl_xor_sync(0xFFFFFFFFu, s0, o));
          s1 = dadd(s1, __shfl_xor_sync(0xFFFFFFFFu, s1, o));
          s2 = dadd(s2, __shfl_xor_sync(0xFFFFFFFFu, s2, o));
        }
        if (lane == 0) {
          StripAcc* e = fsa + ((long long)kr * p.ns_c + kc) * p.n_bl + j;
          if (s0 != 0.0) atomicAdd(&e->s[0], s0);
          if (s1 != 0.0) atomicAdd(&e->s[1], s1);
          if (s2 != 0.0) atomicAdd(&e->s[2], s2);
          atomicAdd(&e->sx, (unsigned long long)sxr + (unsigned long long)cnt * x_cell);
          atomicAdd(&e->sy, (unsigned long long)syr + (unsigned long long)cnt * y_cell);
          atomicAdd(&e->cnt, cnt);
          if (bad && atomicOr(&e->bad, bad) == 0u)
            p.wl[atomicAdd(p.wl_n, 1)] =
                (((long long)f * K + (long long)kr * p.ns_c + kc) << 8) | j;
        }
      }
      __syncwarp();
    }
  }
}

// (B) one warp per marked (cluster, strip): the marked channels folded in
// the reference's order over the strip's window rows (_core.pyx:233-243):
// 32 columns at a time, members ranked by ballot and compacted into shared
// memory, lanes 0..2 folding them in order.
constexpr int kRefoldCap = 512;  // compacted members per warp and fold round
#ifndef SPX_REFOLD_G
#define SPX_REFOLD_G 8
#endif
constexpr int kRefoldG = SPX_REFOLD_G;  // units of 32 columns loaded per group
__global__ void __launch_bounds__(128) k_strip_refold(WideParams p) {
  __shared__ float cvals[4][3][kRefoldCap];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* const cw = &cvals[warp][0][0];
  const unsigned lt_mask = (1u << lane) - 1u;
  const int n = *p.wl_n;
  const int K = p.ns_r * p.ns_c;
  const long long hw = (long long)p.h * p.w;
  for (int item = blockIdx.x * 4 + warp; item < n; item += gridDim.x * 4) {
    const long long it = p.wl[item];
    const long long gk = it >> 8;
    const int j = (int)(it & 255);
    const int ff = (int)(gk / K), fk = (int)(gk - (long long)ff * K);
    StripAcc* e = p.sacc + gk * p.n_bl + j;
    const unsigned bad = e->bad;
    SPX_DCHECK(bad != 0u && bad < 8u && j < p.n_bl);
    const float* im = p.img + (long long)ff * 3 * p.plane;
    const int32_t* lb = p.labels + (long long)ff * hw;
    const int r = fk / p.ns_c, c = fk - r * p.ns_c;
    const int wx0 = max((c - 1) * p.s, 0), wx1 = min((c + 2) * p.s, p.w);
    const int ry0 = (r - 1) * p.s, ry1 = min((r + 2) * p.s, p.h);
    const int ya = max(ry0 + j * p.tile_len, 0), yz = min(ry0 + (j + 1) * p.tile_len, ry1);
    const bool mine = lane < 3 && (bad >> lane & 1u);
    double acc = 0.0;
    int o = 0;  // members compacted, not yet folded
    // lanes 0..2 fold their (marked) channel over the compacted members
    auto fold = [&]() {
      __syncwarp();
      if (mine) {
        const float* src = cw + lane * kRefoldCap;
        int i = 0;
#pragma unroll 1
        for (; i + 4 <= o; i += 4) {
          const float v0 = src[i], v1 = src[i + 1], v2 = src[i + 2], v3 = src[i + 3];
          acc = dadd(acc, (double)v0);
          acc = dadd(acc, (double)v1);
          acc = dadd(acc, (double)v2);
          acc = dadd(acc, (double)v3);
        }
#pragma unroll 1
        for (; i < o; ++i) acc = dadd(acc, (double)src[i]);
      }
      __syncwarp();
      o = 0;
    };
    // units of 32 columns in row-major order; groups of kRefoldG units are loaded
    // one group ahead (labels and values together); members get their
    // row-major ranks from ballots and are compacted into shared memory
    const int chunks = (wx1 - wx0 + 31) >> 5;
    const int units = (yz - ya) * chunks;
    int g_lb[kRefoldG];
    float g_v0[kRefoldG], g_v1[kRefoldG], g_v2[kRefoldG];
    auto load4 = [&](int u0) {
#pragma unroll
      for (int q = 0; q < kRefoldG; ++q) {
        const int u = u0 + q;
        const int ry = u / chunks, ch = u - ry * chunks;
        const int x = wx0 + 32 * ch + lane;
        const bool in = u < units && x < wx1;
        const long long off = (long long)(ya + ry) * p.w + x;
        g_lb[q] = in ? __ldg(lb + off) : -1;
        g_v0[q] = in ? __ldg(im + off) : 0.f;
        g_v1[q] = in ? __ldg(im + p.plane + off) : 0.f;
        g_v2[q] = in ? __ldg(im + 2 * p.plane + off) : 0.f;
      }
    };
    load4(0);
#pragma unroll 1
    for (int u0 = 0; u0 < units; u0 += kRefoldG) {
      int c_lb[kRefoldG];
      float c_v0[kRefoldG], c_v1[kRefoldG], c_v2[kRefoldG];
#pragma unroll
      for (int q = 0; q < kRefoldG; ++q) {
        c_lb[q] = g_lb[q];
        c_v0[q] = g_v0[q];
        c_v1[q] = g_v1[q];
        c_v2[q] = g_v2[q];
      }
      if (u0 + kRefoldG < units) load4(u0 + kRefoldG);
      if (o > kRefoldCap - 32 * kRefoldG) fold();  // room for this group's members
#pragma unroll
      for (int q = 0; q < kRefoldG; ++q) {
        const bool hit = c_lb[q] == fk;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, hit);
        if (hit) {
          const int pos = o + __popc(m & lt_mask);
          cw[pos] = fabsf(c_v0[q]);  // channel 0: |L| (cluster-level flag bit)
          cw[kRefoldCap + pos] = c_v1[q];
          cw[2 * kRefoldCap + pos] = c_v2[q];
        }
        o += __popc(m);
      }
    }
    if (o) fold();
    if (mine) e->s[lane] = acc;
  }
}

// (C) one warp per cluster: the strip entries into shared memory (cleared
// in global memory for the next pass), then the strip tree, the divisions
// and the stores of finish_cluster.
__global__ void __launch_bounds__(128) k_reduce_strips(ReduceParams p, StripAcc* sacc,
                                                       int32_t* wl_n) {
  __shared__ double strips[4][kExMaxStrips][6];
  __shared__ double qv[4][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = p.ns_r * p.ns_c;
  const int f = blockIdx.y;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *wl_n = 0;  // B has read it
  if (p.done && p.done[f]) return;
  const int k = blockIdx.x * 4 + warp;
  if (k >= K) return;  // whole warp
  const long long gk = (long long)f * K + k;
  StripAcc* e = sacc + gk * p.n_bl;
  for (int j = lane; j < p.n_bl; j += 32) {
    const StripAcc v = e[j];
    strips[warp][j][0] = v.s[0];
    strips[warp][j][1] = v.s[1];
    strips[warp][j][2] = v.s[2];
    strips[warp][j][3] = (double)v.sx;
    strips[warp][j][4] = (double)v.sy;
    strips[warp][j][5] = (double)v.cnt;
    e[j] = StripAcc{{0.0, 0.0, 0.0}, 0ull, 0ull, 0u, 0u};
  }
  __syncwarp();
  const int r = k / p.ns_c, c = k - r * p.ns_c;
  finish_cluster(p, strips[warp], qv[warp], (int)gk, r, c, lane);
}

}  // namespace

// ---- launchers ----------------------------------------------------------------

// Any S in [4, 255] (runs of 4 pixels, the last one of a cell row partial
// when S % 4 != 0; a lane walks at most ceil(S/4) * S / 32 runs, i.e. <= 2047
// pixels, the width of the packed per-lane count) and any frame size (planar
// planes padded to a multiple of 4); n_bl <= 64 strips for the exact fallback.
bool cell_path_ok(int64_t h, int64_t w, int64_t s, int64_t tile_len) {
  int64_t n_bl = ceil_div(3 * s, tile_len);
  return s >= 4 && s <= kCellMaxS && n_bl <= kExMaxStrips &&
         h * w * 3 < (int64_t)1 << 40 && h < (1 << 30) && w < (1 << 30);
}

// Lanes per cell (LPC), re-measured after the late round-2 launch shape (one
// cell group per warp, two-warp blocks) on 16 1080p frames in one launch,
// fused pass / association-only pass in ms: 2 lanes for S <= 10 (S = 8:
// 0.284 vs 0.307 with 4), 4 for 11 <= S <= 22 (S = 16: 0.245 vs 0.254 with
// 8 -- 256 C1 frames with lanes: 4.28 -> 4.14 ms per step), 8 for
// 23 <= S <= 38 (S = 28: 0.248 vs 0.262 with 4), 16 for the accumulating
// passes of 39 <= S <= 42 (S = 40: 2.79 vs 2.87 ms per call with 32), 32
// above (wide-mode association: S = 48: 0.192 vs 0.209 with 16).  Fewer lanes per cell give
// each lane more runs over which to amortise the per-cell staging and
// epilogue; too few leave too many cells in flight per warp.  A launch with
// fewer warps than one resident wave (16 per SM) -- small batches, e.g. one
// VGA frame is 1,200 cells -- doubles the lanes while every lane still gets
// >= 2 runs: shorter per-lane walks cut the pass latency.
#ifndef SPX_LPC_WAVE
#define SPX_LPC_WAVE 16  // warps per SM below which a launch doubles its lanes (8, 24, 32: slower)
#endif
#ifndef SPX_LPC_DOUBLINGS
#define SPX_LPC_DOUBLINGS 3
#endif
constexpr int kLpcDoublings = SPX_LPC_DOUBLINGS;
static int cell_lpc(int64_t s, long long cells) {
  static const int env = getenv("SPX_LPC") ? atoi(getenv("SPX_LPC")) : 0;  // development
  if (s <= 64 && (env == 2 || env == 4 || env == 8 || env == 16 || env == 32)) return env;
  // (S > 64: 32 lanes per cell -- the per-lane pixel count must stay <= 2047)
  int lpc = s <= 10 ? 2 : (s <= 22 ? 4 : (s <= 38 ? 8 : (s <= 42 ? 16 : 32)));
  const long long runs = s * ceil_div(s, 4);
  // small launches: up to SPX_LPC_DOUBLINGS doublings (a single 640x480
  // frame: 4 -> 32 lanes per cell)
  for (int d = 0; d < kLpcDoublings; ++d)
    if (lpc < 32 && cells * lpc < (long long)num_sms() * SPX_LPC_WAVE * 32 && runs >= 2 * lpc)
      lpc *= 2;
  return lpc;
}

template <bool ACC, int LPC, bool AL>
static int launch_cell_t(const CellParams& p, dim3 blocks, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> configured{0};  // function attributes are per device
  int dev = 0;
  SPX_CUDA(cudaGetDevice(&dev));
  if (!(configured.load() & (1ull << (dev & 63)))) {
    SPX_CUDA(cudaFuncSetAttribute(k_cell<ACC, LPC, AL>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kWarps * warp_smem(LPC, true))));
    configured.fetch_or(1ull << (dev & 63));
  }
  k_cell<ACC, LPC, AL><<<blocks, kWarps * 32, smem, st>>>(p);
  return SPX_OK;
}

template <int LPC>
static int launch_cell_lpc(const CellParams& p, dim3 blocks, size_t smem, cudaStream_t st,
                           bool acc) {
  const bool al = p.s % 4 == 0 && p.w % 4 == 0;
  if (al)
    return acc ? launch_cell_t<true, LPC, true>(p, blocks, smem, st)
               : launch_cell_t<false, LPC, true>(p, blocks, smem, st);
  return acc ? launch_cell_t<true, LPC, false>(p, blocks, smem, st)
             : launch_cell_t<false, LPC, false>(p, blocks, smem, st);
}

void assoc_bound_coefficients(double xy_weight, float& w32, float& k_mp, float& k_mc, float& k_xy,
                              float& k_const, float& k_rel);

int launch_cell(const float* img, const double* cxy, const double* clab, const CRec* rec,
                int32_t* labels, ClusterAcc* sums, const int32_t* done, int64_t h, int64_t w,
                int64_t s, int64_t ns_r, int64_t ns_c, double xy_weight, int frames, bool acc,
                cudaStream_t st, int64_t cr0, int64_t cr1, int64_t row_off, int32_t* wl,
                int32_t* wl_n, int conc) {
  CellParams p;
  p.wl = wl;
  p.wl_n = wl_n;
  p.img = img;
  p.cxy = cxy;
  p.clab = clab;
  p.rec = rec;
  p.labels = labels;
  p.acc = sums;
  p.done = done;
  p.h = (int)h;
  p.w = (int)w;
  p.s = (int)s;
  p.ns_r = (int)ns_r;
  p.ns_c = (int)ns_c;
  p.frames = frames;
  p.plane = plane_of(h * w);
  if (cr1 < 0) cr1 = ns_r;
  p.cr0 = (int)cr0;
  p.cr1 = (int)cr1;
  p.row_off = (int)row_off;
  p.runs_per_row = (int)ceil_div(s, 4);
  p.runs = (int)(s * p.runs_per_row);
  p.row_magic = p.runs_per_row == 1
                    ? 0u
                    : (unsigned)(((1ull << 32) + p.runs_per_row - 1) / p.runs_per_row);
  p.xy_weight = xy_weight;
  assoc_bound_coefficients(xy_weight, p.w32, p.k_mp, p.k_mc, p.k_xy, p.k_const, p.k_rel);
  if (cr1 <= cr0) return SPX_OK;
  // (conc: launches of this shape running concurrently -- the engine's
  // lanes -- so the small-launch doubling sees the GPU's real occupancy)
  const int lpc = cell_lpc(s, (cr1 - cr0) * ns_c * (long long)frames * std::max(1, conc));
  // Walk up to kGroupsPerWarp groups per warp, but keep >= 16 warps per SM
  // in flight for small launches (one 640x480 frame has only 300 groups).
  const long long groups = ceil_div((cr1 - cr0) * ns_c, 32 / lpc) * (long long)frames;
  // large cells in a small launch (one cell per warp): several warps per
  // cell, each walking a contiguous share of its runs (>= 2 per lane), so
  // about 32 warps per SM are in flight (one 3631x3859 image at S = 118:
  // 1,023 cells)
  p.parts = 1;
  p.part_runs = p.runs;
  if (lpc == 32 && !acc) {  // (accumulating passes: more warps = more epilogues, slower)
    const long long want = ceil_div((long long)num_sms() * kCellWarpsSmall, groups);
    const long long maxp = std::max<long long>(1, p.runs / (2 * lpc));
    p.parts = (int)std::max<long long>(1, std::min(want, maxp));
    p.part_runs = (int)(ceil_div(ceil_div(p.runs, p.parts), lpc) * lpc);
    p.parts = (int)ceil_div(p.runs, p.part_runs);
  }
  p.groups_per_warp = (int)std::max<long long>(
      1, std::min<long long>(kGroupsPerWarp, groups * p.parts / ((long long)num_sms() * 16)));
  const long long warps =
      ceil_div(ceil_div((cr1 - cr0) * ns_c, 32 / lpc) * p.parts, p.groups_per_warp);
  const dim3 blocks((unsigned)ceil_div(warps, kWarps), (unsigned)frames);
  if (frames > 65535) {
    set_error("k_cell: at most 65535 frames per launch");
    return SPX_ERR_VALUE;
  }
  const size_t smem = (size_t)kWarps * warp_smem(lpc, acc);
  const int rc = lpc == 2    ? launch_cell_lpc<2>(p, blocks, smem, st, acc)
                 : lpc == 4  ? launch_cell_lpc<4>(p, blocks, smem, st, acc)
                 : lpc == 8  ? launch_cell_lpc<8>(p, blocks, smem, st, acc)
                 : lpc == 16 ? launch_cell_lpc<16>(p, blocks, smem, st, acc)
                             : launch_cell_lpc<32>(p, blocks, smem, st, acc);
  if (rc) return rc;
  SPX_LAUNCH_CHECK("k_cell");
  return SPX_OK;
}

int launch_records(const double* cxy, const double* clab, CRec* rec, int64_t ns_r, int64_t ns_c,
                   int64_t s, int frames, cudaStream_t st, int64_t k0, int64_t k1,
                   int64_t row_off) {
  if (k1 < 0) k1 = ns_r * ns_c;
  if (k1 <= k0) return SPX_OK;
  long long n = (k1 - k0) * (long long)frames;
  k_records<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(cxy, clab, rec, (int)ns_c, (int)s,
                                                        (int)(ns_r * ns_c), n, (int)k0, (int)k1,
                                                        (int)row_off);
  SPX_LAUNCH_CHECK("k_records");
  return SPX_OK;
}

// Wide mode for S > 42 (SPX_WIDE=0 keeps the per-cluster certificate and
// k_exact_wide, for comparison).  16 1080p frames per call, ms per call,
// wide vs cluster-level + k_exact_wide: S = 33: 4.01 vs 3.01, 40: 3.24 vs
// 2.87, 42: 3.34 vs 3.06, 44: 3.48 vs 3.83, 48: 3.10 vs 4.32, 64: 2.70 vs
// 5.16, 118: 2.73 vs 7.30.
bool wide_mode(int64_t s, int64_t ns_r, int64_t ns_c) {
  static const bool on = !getenv("SPX_WIDE") || atoi(getenv("SPX_WIDE")) != 0;
  return on && s > 42 && ns_r * ns_c < ((int64_t)1 << 31);
}

int launch_wide_update(const float* img, const int32_t* labels, StripAcc* sacc, long long* wl,
                       int32_t* wl_n, const double* prev_xy, const double* prev_lab,
                       double* out_xy, double* out_lab, int64_t* counts, CRec* rec,
                       const int32_t* done, int64_t h, int64_t w, int64_t s, int64_t ns_r,
                       int64_t ns_c, int64_t tile_len, int frames, cudaStream_t st) {
  const int64_t K = ns_r * ns_c;
  if (K <= 0 || frames <= 0) return SPX_OK;
  if (frames > 65535) {
    set_error("wide update: at most 65535 frames per launch");
    return SPX_ERR_VALUE;
  }
  const int64_t n_bl = ceil_div(3 * s, tile_len);
  if (s > kCellMaxS || n_bl > kExMaxStrips) {
    set_error("wide update: S %lld / %lld strips out of range", (long long)s, (long long)n_bl);
    return SPX_ERR_VALUE;
  }
  WideParams wp;
  wp.img = img;
  wp.labels = labels;
  wp.sacc = sacc;
  wp.done = done;
  wp.wl = wl;
  wp.wl_n = wl_n;
  wp.h = (int)h;
  wp.w = (int)w;
  wp.s = (int)s;
  wp.ns_r = (int)ns_r;
  wp.ns_c = (int)ns_c;
  wp.frames = frames;
  wp.n_bl = (int)n_bl;
  wp.tile_len = (int)tile_len;
  wp.plane = plane_of(h * w);
  // ceil(2^64 / ns_c); ns_c = 1 divides by itself (magic 0 marks it)
  wp.ns_c_magic = ns_c == 1 ? 0ull : ~0ull / (unsigned long long)ns_c + 1ull;
  // small launches split each cell into row bands (one warp each) so that
  // about 32 warps per SM are in flight
  {
    const long long cells = K * (long long)frames;
    const long long want = (long long)num_sms() * kCellWarpsSmall;
    int bands = (int)std::min<long long>(std::max<long long>(1, ceil_div(want, cells)), ceil_div(s, 8));
    wp.band_rows = (int)ceil_div(s, bands);
    wp.bands = (int)ceil_div(s, wp.band_rows);
  }
  const dim3 grid((unsigned)ceil_div(K * (long long)wp.bands, kSaccWarps), (unsigned)frames);
  const size_t smem = kSaccWarps * kWideWarpSmem;
  const bool sg = ns_c < 3;
#define SPX_STRIP_ACC(PX)                                        \
  (sg ? k_strip_acc<PX, true><<<grid, kSaccWarps * 32, smem, st>>>(wp) \
      : k_strip_acc<PX, false><<<grid, kSaccWarps * 32, smem, st>>>(wp))
  switch ((int)ceil_div(s, 32)) {  // S in (32, 255]
    case 2: SPX_STRIP_ACC(2); break;
    case 3: SPX_STRIP_ACC(3); break;
    case 4: SPX_STRIP_ACC(4); break;
    case 5: SPX_STRIP_ACC(5); break;
    case 6: SPX_STRIP_ACC(6); break;
    case 7: SPX_STRIP_ACC(7); break;
    default: SPX_STRIP_ACC(8); break;
  }
#undef SPX_STRIP_ACC
  SPX_LAUNCH_CHECK("k_strip_acc");
  k_strip_refold<<<(unsigned)std::max(1, num_sms() * 8), 128, 0, st>>>(wp);
  SPX_LAUNCH_CHECK("k_strip_refold");
  ReduceParams p{};
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
  p.plane = plane_of(h * w);
  p.n_bl = (int)n_bl;
  p.tile_len = (int)tile_len;
  p.kr0 = 0;
  p.kr1 = (int)ns_r;
  p.row_off = 0;
  k_reduce_strips<<<dim3((unsigned)ceil_div(K, 4), (unsigned)frames), 128, 0, st>>>(p, sacc, wl_n);
  SPX_LAUNCH_CHECK("k_reduce_strips");
  return SPX_OK;
}

int launch_reduce_cells(ClusterAcc* acc, const float* img, const int32_t* labels,
                        const double* prev_xy, const double* prev_lab, double* out_xy,
                        double* out_lab, int64_t* counts, CRec* rec, const int32_t* done,
                        int32_t* worklist, int32_t* worklist_n, int64_t h, int64_t w, int64_t s,
                        int64_t ns_r, int64_t ns_c, int64_t tile_len, int frames,
                        cudaStream_t st, int64_t kr0, int64_t kr1, int64_t row_off, int mode,
                        int32_t* wl_reset) {
  ReduceParams p;
  p.wl_reset = wl_reset;
  p.append = mode == kReduceAndExact || mode == kReduceAppendFirst ||
             mode == kReduceAppendLast || mode == kReduceAppend;
  p.acc = acc;
  p.img = img;
  p.labels = labels;
  p.prev_xy = prev_xy;
  p.prev_lab = prev_lab;
  p.out_xy = out_xy;
  p.out_lab = out_lab;
  p.counts = counts;
  p.rec = rec;
  p.done = done;
  p.worklist = worklist;
  p.worklist_n = worklist_n;
  p.h = (int)h;
  p.w = (int)w;
  p.s = (int)s;
  p.ns_r = (int)ns_r;
  p.ns_c = (int)ns_c;
  p.frames = frames;
  p.plane = plane_of(h * w);
  p.win_staged = exact_win_staged(s);
  p.tau_strip = strip_tau(s, tile_len);  // a strip's certified range (k_exact_wide)
  p.n_bl = (int)ceil_div(3 * s, tile_len);
  p.tile_len = (int)tile_len;
  if (kr1 < 0) kr1 = ns_r;
  p.kr0 = (int)kr0;
  p.kr1 = (int)kr1;
  p.row_off = (int)row_off;
  const long long nk = (kr1 - kr0) * ns_c;
  if (mode == kReduceAndExact || mode == kReduceAppendFirst)
    SPX_CUDA(cudaMemsetAsync(worklist_n, 0, sizeof(int32_t), st));
  if (nk <= 0 || frames <= 0) return SPX_OK;
  if (frames > 65535) {
    set_error("k_reduce_cells: at most 65535 frames per launch");
    return SPX_ERR_VALUE;
  }
  if (mode == kReduceExactMerged && s <= 32) {
    const long long rb = ceil_div(nk, kRedN);
    const long long ex_blocks = std::max<long long>(
        num_sms(), std::min<long long>((long long)num_sms() * SPX_EXG, nk * frames / 64));
    if (rb * frames + ex_blocks > 0x7FFFFFFFll) {
      set_error("k_update: grid too large");
      return SPX_ERR_VALUE;
    }
    static std::atomic<uint64_t> configured{0};  // per device
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!(configured.load() & (1ull << (dev & 63)))) {
      SPX_CUDA(cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(kExWarps * 3 * kExCap * sizeof(float) +
                                          kExWinSmemMax)));
      configured.fetch_or(1ull << (dev & 63));
    }
    k_update<<<(unsigned)(rb * frames + ex_blocks), kRedT, exact_smem_bytes(s), st>>>(p, (int)rb);
    SPX_LAUNCH_CHECK("k_update");
    return SPX_OK;
  }
  if (mode != kExactOnly) {
    k_reduce_cells<<<dim3((unsigned)ceil_div(nk, kRedN), (unsigned)frames), kRedT, 0, st>>>(p);
    SPX_LAUNCH_CHECK("k_reduce_cells");
  }
  if (mode == kReduceOnly || mode == kReduceAppendFirst || mode == kReduceAppend) return SPX_OK;
  if (s > 32) {
    // large cells: most clusters are flagged, one block per cluster
    const long long wb = std::max<long long>(
        1, std::min<long long>((long long)num_sms() * 8, nk * frames));
    const int64_t ww = std::min<int64_t>(3 * s, w);
    if (ww <= 256)
      k_exact_wide<8><<<(unsigned)wb, kWideWarps * 32, 0, st>>>(p);
    else if (ww <= 384)
      k_exact_wide<12><<<(unsigned)wb, kWideWarps * 32, 0, st>>>(p);
    else
      k_exact_wide<16><<<(unsigned)wb, kWideWarps * 32, 0, st>>>(p);
    SPX_LAUNCH_CHECK("k_exact_wide");
    return SPX_OK;
  }
  // grid-stride over the worklist; ~0.5% of clusters are flagged, so small
  // launches get a small grid (an empty block still costs its scheduling)
  const long long ex_blocks = std::max<long long>(
      num_sms(), std::min<long long>((long long)num_sms() * SPX_EXG, nk * frames / 64));
  const size_t ex_smem = exact_smem_bytes(s);
  {  // dynamic + static shared memory may exceed the default 48 KB
    static std::atomic<uint64_t> configured{0};  // per device
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!(configured.load() & (1ull << (dev & 63)))) {
      SPX_CUDA(cudaFuncSetAttribute(k_exact_clusters, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(kExWarps * 3 * kExCap * sizeof(float) +
                                          kExWinSmemMax)));
      configured.fetch_or(1ull << (dev & 63));
    }
  }
  k_exact_clusters<<<(unsigned)ex_blocks, kExWarps * 32, ex_smem, st>>>(p);
  SPX_LAUNCH_CHECK("k_exact_clusters");
  return SPX_OK;
}


}  // namespace spx
