// common.cu -- error plumbing, colour tables, device queries.
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <mutex>

#include "spx_internal.cuh"

namespace spx {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  if (e == cudaErrorMemoryAllocation) return SPX_ERR_NOMEM;
  return SPX_ERR_CUDA;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// tables.py:14-54 evaluated on the host with the same libm as the reference
// (Python's float ** is libm pow).  The GPU never recomputes them.
static ColorTables make_tables() {
  ColorTables t;
  for (int v = 0; v < 256; ++v) {
    volatile double c = v / 255.0;
    t.lut[v] = (c <= 0.04045) ? c / 12.92 : std::pow((c + 0.055) / 1.055, 2.4);
  }
  const double m[9] = {0.4124564, 0.3575761, 0.1804375, 0.2126729, 0.7151522,
                       0.0721750, 0.0193339, 0.1191920, 0.9503041};
  std::memcpy(t.m, m, sizeof m);
  for (int i = 0; i < 3; ++i) {
    volatile double a = m[3 * i] + m[3 * i + 1];
    t.white[i] = a + m[3 * i + 2];
  }
  volatile double n216 = 216.0, n24389 = 24389.0, n27 = 27.0;
  t.eps = n216 / n24389;
  t.kappa = n24389 / n27;
  volatile double cbrt2 = 1.2599210498948731648, sqr_cbrt2 = 1.5874010519681994748;
  t.cbrt_factor[0] = 1.0 / sqr_cbrt2;
  t.cbrt_factor[1] = 1.0 / cbrt2;
  t.cbrt_factor[2] = 1.0;
  t.cbrt_factor[3] = cbrt2;
  t.cbrt_factor[4] = sqr_cbrt2;
  return t;
}

const ColorTables& host_tables() {
  static ColorTables t = make_tables();
  return t;
}

}  // namespace spx

extern "C" {

const char* spx_last_error(void) { return spx::g_err; }
const char* spx_name(void) { return "cuda"; }
int32_t spx_abi_version(void) { return 1; }

/* Test hook (not part of the protocol): copy the host-side tables out so
 * tests can compare them with tables.py. */
int32_t spx_debug_tables(double* lut, double* mat, double* white) {
  const spx::ColorTables& t = spx::host_tables();
  std::memcpy(lut, t.lut, sizeof t.lut);
  std::memcpy(mat, t.m, sizeof t.m);
  std::memcpy(white, t.white, sizeof t.white);
  return SPX_OK;
}

}  // extern "C"
