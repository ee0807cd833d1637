// convert.cu -- RGB -> {RGB, XYZ, CIELAB} float32, bit-exact with
// _core.pyx:45-83 (convert_band).
//
// Layout: rgb uint8 HWC, out float32 HWC (the reference layouts).  One thread
// converts a group of 4 consecutive pixels: 12 input bytes as three 32-bit
// loads, 48 output bytes as three 128-bit stores (coalesced, vectorised).
// The 256-entry linearisation LUT is staged in shared memory (divergent
// gathers would serialise in the constant cache); the matrix, white point and
// cbrt constants are warp-uniform and live in __constant__.
//
// Roofline: 15 algorithmic bytes per pixel (3 in + 12 out).  The binary64
// arithmetic (three glibc-cbrt evaluations with a division each, three
// divisions by the white point) makes this kernel FP64-pipe bound on B200;
// see DESIGN.md.
#include <atomic>

#include "spx_internal.cuh"

namespace spx {

__constant__ double c_white[3];
__constant__ double c_eps;
__constant__ double c_kappa;
__constant__ double c_factor[5];
__constant__ double c_inv_white[3];  // RN(1 / white[i])
__constant__ double c_inv116;        // RN(1 / 116)
// g_mlut[3 * i + j][v] = RN(m[3 * i + j] * lut[v]): the nine products of the
// XYZ matrix rows with the linearised channels, tabulated (the same IEEE
// products the reference forms, _core.pyx:64-69), so a pixel's XYZ costs six
// binary64 adds instead of nine multiplies and six adds.
__device__ double g_mlut[9 * 256];

// __constant__ / __device__ tables live per device: one upload per device
static std::atomic<uint64_t> g_uploaded{0};

int upload_tables() {
  int dev = 0;
  SPX_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (g_uploaded.load() & bit) return SPX_OK;
  const ColorTables& t = host_tables();
  SPX_CUDA(cudaMemcpyToSymbol(c_white, t.white, sizeof t.white));
  SPX_CUDA(cudaMemcpyToSymbol(c_eps, &t.eps, sizeof t.eps));
  SPX_CUDA(cudaMemcpyToSymbol(c_kappa, &t.kappa, sizeof t.kappa));
  SPX_CUDA(cudaMemcpyToSymbol(c_factor, t.cbrt_factor, sizeof t.cbrt_factor));
  double inv_w[3] = {1.0 / t.white[0], 1.0 / t.white[1], 1.0 / t.white[2]};
  double inv116 = 1.0 / 116.0;
  SPX_CUDA(cudaMemcpyToSymbol(c_inv_white, inv_w, sizeof inv_w));
  SPX_CUDA(cudaMemcpyToSymbol(c_inv116, &inv116, sizeof inv116));
  static double mlut[9 * 256];
  for (int i = 0; i < 9; ++i)
    for (int v = 0; v < 256; ++v) mlut[i * 256 + v] = t.m[i] * t.lut[v];
  SPX_CUDA(cudaMemcpyToSymbol(g_mlut, mlut, sizeof mlut));
  g_uploaded.fetch_or(bit);
  return SPX_OK;
}

// glibc sysdeps/ieee754/dbl-64/s_cbrt.c restated with explicit round-to-
// nearest operations (no FMA), for x > 0 (the only inputs convert produces:
// t > 216/24389).  Cross-checked against libm by the oracle tests.
__device__ __forceinline__ double cbrt_glibc(double x) {
  long long bits = __double_as_longlong(x);
  int bexp = (int)((bits >> 52) & 0x7ff);
  int xe;
  double xm;
  if (bexp != 0 && bexp != 0x7ff) {
    xe = bexp - 1022;  // frexp: x = xm * 2^xe, xm in [0.5, 1)
    xm = __longlong_as_double((bits & 0x800FFFFFFFFFFFFFLL) | (1022LL << 52));
    xm = fabs(xm);
  } else {
    xm = frexp(fabs(x), &xe);
    if (xe == 0 && (x == 0.0 || isinf(x) || isnan(x))) return x + x;
  }
  double p = dsub(0.784932344976639262, dmul(0.145263899385486377, xm));
  p = dadd(-1.83469277483613086, dmul(p, xm));
  p = dadd(2.44693122563534430, dmul(p, xm));
  p = dadd(-2.11499494167371287, dmul(p, xm));
  p = dadd(1.50819193781584896, dmul(p, xm));
  double u = dadd(0.354895765043919860, dmul(p, xm));
  double t2 = dmul(dmul(u, u), u);
  double ym = dmul(ddiv(dmul(u, dadd(t2, dmul(2.0, xm))), dadd(dmul(2.0, t2), xm)),
                   c_factor[2 + xe % 3]);
  if (x < 0.0) ym = -ym;
  int n = xe / 3;
  if (n >= -1000 && n <= 1000) {
    // ldexp by an exact power of two; ym is in [0.5, 1.6] so the product
    // stays normal for every input convert can produce.
    double r = dmul(ym, __longlong_as_double((long long)(1023 + n) << 52));
    if (fabs(r) >= 2.2250738585072014e-308) return r;
  }
  return ldexp(ym, n);
}

// x / d for a constant d with inv = RN(1/d): one product and an FMA
// correction step (Markstein).  Equal to the IEEE quotient RN(x/d) on every
// input convert can produce -- verified exhaustively over all 2^24 colours by
// tests/test_gpu_kernels.py::test_convert_all_colours_bitexact.
__device__ __forceinline__ double div_const(double x, double d, double inv) {
  const double q = dmul(x, inv);
  const double r = __fma_rn(-q, d, x);
  return __fma_rn(r, inv, q);
}

#ifndef SPX_DIV_NEWTON
#define SPX_DIV_NEWTON 1
#endif
// Correctly rounded a / b for positive normal operands well inside the
// exponent range (the cbrt quotient below: a, b in [0.5, 8]): MUFU reciprocal
// seed, SPX_DIV_NEWTON Newton steps, then one Markstein correction.
// Branch-free, unlike the library division (whose special-case slow path
// splits the code and stops the compiler from interleaving the 12
// independent cbrt chains of a 4-pixel group).  Proven equal to RN(a / b) on
// every input convert can produce by the exhaustive 2^24-colour test.
__device__ __forceinline__ double div_rn_fast(double a, double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
#pragma unroll
  for (int i = 0; i < SPX_DIV_NEWTON; ++i) {
    const double e = __fma_rn(-b, y, 1.0);
    y = __fma_rn(e, y, y);
  }
  const double q = dmul(a, y);
  const double r = __fma_rn(-b, q, a);
  return __fma_rn(r, y, q);
}

// Exact scaling of a positive normal double by 2^n (result normal): an
// integer add on the exponent field instead of a binary64 multiply.
__device__ __forceinline__ double scale2(double x, int n) {
  return __hiloint2double(__double2hiint(x) + (n << 20), __double2loint(x));
}

// cbrt_glibc for positive normal x of moderate size (convert's t = X / Xw in
// (0, 1.2]), with no branches: frexp by bit manipulation, the factor picked
// with selects, the exact doublings and the final ldexp as exponent adds.
// Same rounded operations as cbrt_glibc, so the same result.
// fx[xe + 6] = factor[2 + xe % 3] * 2^(xe / 3) for the exponents convert
// produces (t in (eps, 1.2], or the stand-in 1.0: xe in [-6, 1]).  Scaling
// by a power of two commutes with rounding, so RN(q * fx) equals glibc's
// ldexp(RN(q * factor), xe / 3).
__device__ __forceinline__ double cbrt_fast(double x, const double* fx) {
  const long long bits = __double_as_longlong(x);
  const int xe = (int)((bits >> 52) & 0x7ff) - 1022;
  const double xm = __longlong_as_double((bits & 0x000FFFFFFFFFFFFFLL) | (1022LL << 52));
  double p = dsub(0.784932344976639262, dmul(0.145263899385486377, xm));
  p = dadd(-1.83469277483613086, dmul(p, xm));
  p = dadd(2.44693122563534430, dmul(p, xm));
  p = dadd(-2.11499494167371287, dmul(p, xm));
  p = dadd(1.50819193781584896, dmul(p, xm));
  const double u = dadd(0.354895765043919860, dmul(p, xm));
  const double t2 = dmul(dmul(u, u), u);
  const double f = fx[min(max(xe + 6, 0), 7)];  // shared memory, conflict-free
  // 2*xm and 2*t2 are exact doublings (xm in [0.5, 1), t2 > 0.04)
  return dmul(div_rn_fast(dmul(u, dadd(t2, scale2(xm, 1))), dadd(scale2(t2, 1), xm)), f);
}

__device__ __forceinline__ double lab_lin(double t) {
  return div_const(dadd(dmul(c_kappa, t), 16.0), 116.0, c_inv116);
}

struct Factors {
  const double* f;  // the fx table of cbrt_fast (shared memory)
};

template <int SPACE>
__device__ __forceinline__ void convert_px(const double* lut, const Factors& fc, uint32_t R,
                                           uint32_t G, uint32_t B, float& o0, float& o1,
                                           float& o2) {
  if (SPACE == 0) {
    o0 = __double2float_rn(ddiv((double)R, 255.0));
    o1 = __double2float_rn(ddiv((double)G, 255.0));
    o2 = __double2float_rn(ddiv((double)B, 255.0));
    return;
  }
  const double cx = dadd(dadd(lut[R], lut[256 + G]), lut[512 + B]);
  const double cy = dadd(dadd(lut[768 + R], lut[1024 + G]), lut[1280 + B]);
  const double cz = dadd(dadd(lut[1536 + R], lut[1792 + G]), lut[2048 + B]);
  if (SPACE == 1) {
    o0 = __double2float_rn(cx);
    o1 = __double2float_rn(cy);
    o2 = __double2float_rn(cz);
    return;
  }
  const double* fac = fc.f;
  // _core.pyx:73-75: f(t) = cbrt(t) if t > eps else (kappa t + 16) / 116.  The
  // cbrt chains run unconditionally (on 1.0 where t <= eps) so the compiler
  // can interleave them; the rare linear branch is patched in afterwards.
  const double tx = div_const(cx, c_white[0], c_inv_white[0]);
  const double ty = div_const(cy, c_white[1], c_inv_white[1]);
  const double tz = div_const(cz, c_white[2], c_inv_white[2]);
  // t >= 0 (non-negative matrix and LUT), so `t > eps` is an integer compare
  // of the bit patterns (keeps the compares off the saturated FP64 pipe)
  const long long eps = __double_as_longlong(c_eps);
  const bool bx = __double_as_longlong(tx) > eps, by = __double_as_longlong(ty) > eps,
             bz = __double_as_longlong(tz) > eps;
  double fx = cbrt_fast(bx ? tx : 1.0, fac);
  double fy = cbrt_fast(by ? ty : 1.0, fac);
  double fz = cbrt_fast(bz ? tz : 1.0, fac);
  if (!bx) fx = lab_lin(tx);
  if (!by) fy = lab_lin(ty);
  if (!bz) fz = lab_lin(tz);
  double light = dsub(dmul(116.0, fy), 16.0);
  if (light < 0.0) light = 0.0;
  if (light > 100.0) light = 100.0;
  o0 = __double2float_rn(light);
  o1 = __double2float_rn(dmul(500.0, dsub(fx, fy)));
  o2 = __double2float_rn(dmul(200.0, dsub(fy, fz)));
}

// Pixels [p0, p1) of a flat HWC raster (frames of a batch are contiguous, so
// a batch is one range).  `vec` requires rgb 4-byte and out 16-byte aligned.
// PLANAR: out is [frames][3][plane_of(hw)] (the engine's internal layout)
// instead of HWC.
// Certified-sum flag of one output pixel (cell.cu): some channel is nonzero
// with |v| < tau, or |v| >= 128 / non-finite.
__device__ __forceinline__ bool sum_flag(float v, float tau) {
  const float a = fabsf(v);
  return (a != 0.f && a < tau) || !(a < 128.f);
}
__device__ __forceinline__ float with_flag(float o0, float o1, float o2, float tau) {
  const bool f = sum_flag(o0, tau) || sum_flag(o1, tau) || sum_flag(o2, tau);
  return f ? __uint_as_float(__float_as_uint(o0) | 0x80000000u) : o0;
}

#ifndef SPX_CONV_BPS
// grid cap: blocks per SM, grid-stride beyond.  3 = one resident wave
// (SPX_CONV_MINB): unsplit calls measured 0.7% slower than a cap of 12, but
// with concurrent lanes (engine.cu) the converts then leave SM slots to the
// other lanes' passes: C1 x 256 in 4 lanes 4.325 -> 4.297 ms (6: 4.52 ms).
#define SPX_CONV_BPS 3
#endif
#ifndef SPX_CONV_MINB
#define SPX_CONV_MINB 3  // 80 registers, 24 warps per SM (measured ~1% faster than 4 and 6)
#endif
template <int SPACE, bool PLANAR>
// Threads per convert block.  Late round 2 (256 C1 frames, 4 lanes): 512 x 1
// block per SM made the convert itself 4% faster (0.70 -> 0.68 ms unsplit)
// but the laned step 0.3% slower; 128 x 6 within noise.  256 kept.
#ifndef SPX_CONV_T
#define SPX_CONV_T 256
#endif
__global__ void __launch_bounds__(SPX_CONV_T, SPX_CONV_MINB) k_convert(const uint8_t* __restrict__ rgb,
                                                 float* __restrict__ out, int64_t p0,
                                                 int64_t p1, int vec, int64_t hw, float tau) {
  __shared__ double lut[SPACE == 0 ? 1 : 9 * 256];  // g_mlut (SPACE 1, 2)
  __shared__ double fxs[8];
  if (threadIdx.x < 8) {
    const int xe = (int)threadIdx.x - 6;  // C semantics of % and / (glibc s_cbrt.c)
    fxs[threadIdx.x] = ldexp(c_factor[2 + xe % 3], xe / 3);
  }
  Factors fc;
  fc.f = fxs;
  if (SPACE != 0) {
    for (int i = threadIdx.x; i < 9 * 256; i += blockDim.x) lut[i] = g_mlut[i];
    __syncthreads();
  }
  // HWC: groups of 4 consecutive pixels of the flat range [p0, p1).
  // PLANAR (p0 = 0, p1 = frames * hw): groups of 4 pixels of ONE frame --
  // ceil(hw / 4) per frame, the last one partial when hw % 4 != 0 -- written
  // to the frame's planes of stride plane_of(hw); (frame, group) advance
  // incrementally (no 64-bit division in the loop).
  const int64_t gpf = PLANAR ? (hw + 3) >> 2 : 0, pst = PLANAR ? plane_of(hw) : 0;
  int64_t g0 = PLANAR ? 0 : p0 >> 2, g1 = PLANAR ? (p1 / hw) * gpf : (p1 + 3) >> 2;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t g = g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t pf = 0, pr = 0;  // PLANAR: frame, first pixel of the group in the frame
  if (PLANAR) {
    pf = g / gpf;
    pr = (g - pf * gpf) << 2;
  }
  // source pixel index (HWC, flat) of a group's first pixel, its end, and
  // whether the group takes the 12-byte vector load
  auto group = [&](int64_t gg, int64_t f_, int64_t r_, int64_t& q_, int64_t& qe_) {
    q_ = PLANAR ? f_ * hw + r_ : gg << 2;
    qe_ = PLANAR ? f_ * hw + hw : p1;
    return vec && q_ >= p0 && q_ + 4 <= qe_ && (!PLANAR || ((q_ * 3) & 3) == 0);
  };
  // the next group's 12 bytes are loaded one iteration ahead (software
  // pipelining: the loads' latency overlaps this group's binary64 work)
  int64_t nq, nqe;
  bool nvec = g < g1 && group(g, pf, pr, nq, nqe);
  uint32_t n0 = 0, n1 = 0, n2 = 0;
  if (nvec) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(rgb + nq * 3);
    n0 = __ldg(src), n1 = __ldg(src + 1), n2 = __ldg(src + 2);
  }
  for (; g < g1; g += stride) {
    const int64_t q = nq, qe = nqe;
    const bool isvec = nvec;
    const uint32_t w0 = n0, w1 = n1, w2 = n2;
    {  // prefetch group g + stride (frame / offset advanced as below)
      int64_t f2 = pf, r2 = pr;
      if (PLANAR) {
        r2 += stride << 2;
        while (r2 >= gpf << 2) {
          r2 -= gpf << 2;
          ++f2;
        }
      }
      nvec = g + stride < g1 && group(g + stride, f2, r2, nq, nqe);
      if (nvec) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(rgb + nq * 3);
        n0 = __ldg(src), n1 = __ldg(src + 1), n2 = __ldg(src + 2);
      }
    }
    if (isvec) {
      uint8_t c[12];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        c[i] = (w0 >> (8 * i)) & 255;
        c[4 + i] = (w1 >> (8 * i)) & 255;
        c[8 + i] = (w2 >> (8 * i)) & 255;
      }
      float o[12];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        convert_px<SPACE>(lut, fc, c[3 * i], c[3 * i + 1], c[3 * i + 2], o[3 * i], o[3 * i + 1],
                          o[3 * i + 2]);
      if (PLANAR) {
        SPX_DCHECK(pr + 4 <= pst && pf < p1 / hw);
        float* base = out + pf * 3 * pst + pr;
        *reinterpret_cast<float4*>(base) =
            make_float4(with_flag(o[0], o[1], o[2], tau), with_flag(o[3], o[4], o[5], tau),
                        with_flag(o[6], o[7], o[8], tau), with_flag(o[9], o[10], o[11], tau));
        *reinterpret_cast<float4*>(base + pst) = make_float4(o[1], o[4], o[7], o[10]);
        *reinterpret_cast<float4*>(base + 2 * pst) = make_float4(o[2], o[5], o[8], o[11]);
      } else {
        float4* dst = reinterpret_cast<float4*>(out + q * 3);
        dst[0] = make_float4(o[0], o[1], o[2], o[3]);
        dst[1] = make_float4(o[4], o[5], o[6], o[7]);
        dst[2] = make_float4(o[8], o[9], o[10], o[11]);
      }
    } else {
      for (int64_t p = q; p < q + 4; ++p) {
        if (p < p0 || p >= qe) continue;
        float o0, o1, o2;
        convert_px<SPACE>(lut, fc, rgb[p * 3], rgb[p * 3 + 1], rgb[p * 3 + 2], o0, o1, o2);
        if (PLANAR) {
          SPX_DCHECK(pr + (p - q) < hw && pf < p1 / hw);
          float* base = out + pf * 3 * pst + pr + (p - q);
          base[0] = with_flag(o0, o1, o2, tau);
          base[pst] = o1;
          base[2 * pst] = o2;
        } else {
          out[p * 3] = o0;
          out[p * 3 + 1] = o1;
          out[p * 3 + 2] = o2;
        }
      }
    }
    if (PLANAR) {
      pr += stride << 2;
      while (pr >= gpf << 2) {
        pr -= gpf << 2;
        ++pf;
      }
    }
  }
}

// planar_hw > 0: the engine's planar layout with the certified-sum flag of
// grid interval `s` in channel 0's sign bit (tau_flag > 0: that range
// instead -- wide mode flags by the strip-level range).
int launch_convert(const uint8_t* rgb, float* out, int64_t p0, int64_t p1, int space,
                   cudaStream_t st, int64_t planar_hw, int64_t s, float tau_flag) {
  const float tau = planar_hw > 0 ? (tau_flag > 0.f ? tau_flag : certified_tau(s)) : 0.f;
  if (p1 <= p0) return SPX_OK;
  int rc = upload_tables();
  if (rc) return rc;
  int vec = ((uintptr_t)rgb % 4 == 0) && ((uintptr_t)out % 16 == 0);
  const bool planar = planar_hw > 0;
  if (planar && (p0 != 0 || p1 % planar_hw != 0 || (uintptr_t)out % 16 != 0)) {
    set_error("planar convert needs whole frames and a 16-byte aligned output");
    return SPX_ERR_VALUE;
  }
  if (planar) vec = (uintptr_t)rgb % 4 == 0;
  int64_t groups = planar ? (p1 / planar_hw) * ((planar_hw + 3) >> 2)
                          : ((p1 + 3) >> 2) - (p0 >> 2);
  int64_t blocks = ceil_div(groups, SPX_CONV_T);
  int64_t cap = (int64_t)num_sms() * SPX_CONV_BPS;
  if (blocks > cap) blocks = cap;
#define SPX_CONVERT(SP)                                                                  \
  (planar ? k_convert<SP, true><<<(unsigned)blocks, SPX_CONV_T, 0, st>>>(rgb, out, p0, p1, vec, \
                                                                  planar_hw, tau)         \
          : k_convert<SP, false><<<(unsigned)blocks, SPX_CONV_T, 0, st>>>(rgb, out, p0, p1, vec, 1, \
                                                                   0.f))
  switch (space) {
    case 0: SPX_CONVERT(0); break;
    case 1: SPX_CONVERT(1); break;
    case 2: SPX_CONVERT(2); break;
    default:
      set_error("unknown colour space %d", space);
      return SPX_ERR_VALUE;
  }
  SPX_LAUNCH_CHECK("k_convert");
  return SPX_OK;
}

}  // namespace spx

extern "C" int32_t spx_convert_band(const uint8_t* rgb, float* out, int64_t h, int64_t w,
                                    int32_t space, int64_t y0, int64_t y1, void* stream) {
  if (h < 0 || w < 0 || y0 < 0 || y1 > h) {
    spx::set_error("convert_band: rows [%lld,%lld) outside image of height %lld",
                   (long long)y0, (long long)y1, (long long)h);
    return SPX_ERR_DIMENSION;
  }
  return spx::launch_convert(rgb, out, y0 * w, y1 * w, space, spx::as_stream(stream), 0, 1, -1.f);
}
