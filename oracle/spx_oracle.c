/*
 * spx_oracle.c -- CPU restatement of the reference SLIC kernel set.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_1509_04232_b200/csrc; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links, imports or calls it.
 *
 * Every function restates the reference algorithm operation for operation in
 * IEEE binary64 with no FMA contraction (compile with -ffp-contract=off, as
 * the reference does in pkg/setup.py:8-14).  Citations are into
 * /root/reference/pkg/src/superpix/.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against
 * golden vectors produced by the reference's compiled path
 * (tests/golden/make_golden.py) and, when oracle/_ref is built, against the
 * reference kernels directly on random inputs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- tables.py:14-54 ---------------------------------------------------- */
static double LUT[256];
static const double M[9] = {0.4124564, 0.3575761, 0.1804375,
                            0.2126729, 0.7151522, 0.0721750,
                            0.0193339, 0.1191920, 0.9503041};
static double W[3];
static const double LAB_EPS = 216.0 / 24389.0;   /* tables.py:38 */
static const double LAB_KAPPA = 24389.0 / 27.0;  /* tables.py:39 */
static int tables_ready = 0;

static void init_tables(void) {
    if (tables_ready) return;
    for (int v = 0; v < 256; ++v) {              /* tables.py:42-51 */
        double c = v / 255.0;
        LUT[v] = (c <= 0.04045) ? c / 12.92 : pow((c + 0.055) / 1.055, 2.4);
    }
    for (int i = 0; i < 3; ++i)                  /* tables.py:28-35 left fold */
        W[i] = (M[3 * i] + M[3 * i + 1]) + M[3 * i + 2];
    tables_ready = 1;
}

void spxo_tables(double *lut, double *mat, double *white) {
    init_tables();
    memcpy(lut, LUT, sizeof LUT);
    memcpy(mat, M, sizeof M);
    memcpy(white, W, sizeof W);
}

/* ---- glibc sysdeps/ieee754/dbl-64/s_cbrt.c, restated (no FMA) ----------
 * libm cbrt is what _core.pyx:5,73-75 calls; glibc 2.39's x86-64 build is the
 * classic polynomial + one rational Newton step.  Restated here so the CUDA
 * port can be checked against an explicit algorithm, and the restatement is
 * itself checked against libm cbrt in tests/test_oracle.py. */
double spxo_cbrt_glibc(double x) {
    static const double CBRT2 = 1.2599210498948731648;
    static const double SQR_CBRT2 = 1.5874010519681994748;
    const double factor[5] = {1.0 / SQR_CBRT2, 1.0 / CBRT2, 1.0, CBRT2, SQR_CBRT2};
    int xe;
    double xm = frexp(fabs(x), &xe);
    if (xe == 0 && fpclassify(x) <= FP_ZERO) return x + x;
    double u = (0.354895765043919860
                + ((1.50819193781584896
                    + ((-2.11499494167371287
                        + ((2.44693122563534430
                            + ((-1.83469277483613086
                                + (0.784932344976639262 - 0.145263899385486377 * xm) * xm)
                               * xm))
                           * xm))
                       * xm))
                   * xm));
    double t2 = u * u * u;
    double ym = u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * factor[2 + xe % 3];
    return ldexp(x > 0.0 ? ym : -ym, xe / 3);
}

/* ---- _core.pyx:45-83 convert_band --------------------------------------- */
void spxo_convert_band(const uint8_t *rgb, float *out, int64_t h, int64_t w,
                       int space, int64_t y0, int64_t y1) {
    (void)h;
    init_tables();
    for (int64_t y = y0; y < y1; ++y) {
        for (int64_t x = 0; x < w; ++x) {
            const uint8_t *p = rgb + (y * w + x) * 3;
            float *o = out + (y * w + x) * 3;
            if (space == 0) {
                o[0] = (float)(p[0] / 255.0);
                o[1] = (float)(p[1] / 255.0);
                o[2] = (float)(p[2] / 255.0);
                continue;
            }
            double r = LUT[p[0]], g = LUT[p[1]], b = LUT[p[2]];
            double cx = M[0] * r + M[1] * g + M[2] * b;
            double cy = M[3] * r + M[4] * g + M[5] * b;
            double cz = M[6] * r + M[7] * g + M[8] * b;
            if (space == 1) {
                o[0] = (float)cx; o[1] = (float)cy; o[2] = (float)cz;
                continue;
            }
            double tx = cx / W[0], ty = cy / W[1], tz = cz / W[2];
            double fx = tx > LAB_EPS ? cbrt(tx) : (LAB_KAPPA * tx + 16.0) / 116.0;
            double fy = ty > LAB_EPS ? cbrt(ty) : (LAB_KAPPA * ty + 16.0) / 116.0;
            double fz = tz > LAB_EPS ? cbrt(tz) : (LAB_KAPPA * tz + 16.0) / 116.0;
            double light = 116.0 * fy - 16.0;
            if (light < 0.0) light = 0.0;
            if (light > 100.0) light = 100.0;
            o[0] = (float)light;
            o[1] = (float)(500.0 * (fx - fy));
            o[2] = (float)(200.0 * (fy - fz));
        }
    }
}

/* ---- _core.pyx:86-107 init_centers_range -------------------------------- */
void spxo_init_centers_range(const float *img, int64_t h, int64_t w, int64_t s,
                             int64_t ns_c, double *cxy, double *clab,
                             int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k) {
        int64_t r = k / ns_c, c = k % ns_c;
        int64_t ix = c * s + s / 2;
        if (ix > w - 1) ix = w - 1;
        int64_t iy = r * s + s / 2;
        if (iy > h - 1) iy = h - 1;
        cxy[2 * k] = (double)ix;
        cxy[2 * k + 1] = (double)iy;
        const float *p = img + (iy * w + ix) * 3;
        clab[3 * k] = p[0]; clab[3 * k + 1] = p[1]; clab[3 * k + 2] = p[2];
    }
}

/* ---- _core.pyx:110-120 _gradient ---------------------------------------- */
static double gradient(const float *img, int64_t w, int64_t x, int64_t y) {
#define PX(yy, xx, ch) ((double)img[((yy) * w + (xx)) * 3 + (ch)])
    double dl = PX(y, x + 1, 0) - PX(y, x - 1, 0);
    double da = PX(y, x + 1, 1) - PX(y, x - 1, 1);
    double db = PX(y, x + 1, 2) - PX(y, x - 1, 2);
    double gx = dl * dl + da * da + db * db;
    dl = PX(y + 1, x, 0) - PX(y - 1, x, 0);
    da = PX(y + 1, x, 1) - PX(y - 1, x, 1);
    db = PX(y + 1, x, 2) - PX(y - 1, x, 2);
    double gy = dl * dl + da * da + db * db;
#undef PX
    return gx + gy;
}

/* ---- _core.pyx:123-156 perturb_range ------------------------------------ */
void spxo_perturb_range(const float *img, int64_t h, int64_t w, double *cxy,
                        double *clab, int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k) {
        int64_t ix = (int64_t)cxy[2 * k], iy = (int64_t)cxy[2 * k + 1];
        if (ix < 1 || ix > w - 2 || iy < 1 || iy > h - 2) continue;
        double best = gradient(img, w, ix, iy);
        int64_t bx = ix, by = iy;
        for (int64_t dy = -1; dy < 2; ++dy)
            for (int64_t dx = -1; dx < 2; ++dx) {
                if (dx == 0 && dy == 0) continue;
                int64_t nx = ix + dx, ny = iy + dy;
                if (nx < 1 || nx > w - 2 || ny < 1 || ny > h - 2) continue;
                double g = gradient(img, w, nx, ny);
                if (g < best) { best = g; bx = nx; by = ny; }
            }
        cxy[2 * k] = (double)bx;
        cxy[2 * k + 1] = (double)by;
        const float *p = img + (by * w + bx) * 3;
        clab[3 * k] = p[0]; clab[3 * k + 1] = p[1]; clab[3 * k + 2] = p[2];
    }
}

/* ---- _core.pyx:24-26 candidate order; :159-169 _pix_dist; :172-197 ------- */
static const int OFF_R[9] = {0, -1, -1, -1, 0, 0, 1, 1, 1};
static const int OFF_C[9] = {0, -1, 0, 1, -1, 1, -1, 0, 1};

static double pix_dist(const float *img, int64_t w, const double *cxy,
                       const double *clab, int64_t k, int64_t x, int64_t y,
                       double xy_weight) {
    const float *p = img + (y * w + x) * 3;
    double dl = clab[3 * k] - (double)p[0];
    double da = clab[3 * k + 1] - (double)p[1];
    double db = clab[3 * k + 2] - (double)p[2];
    double dlab = sqrt(dl * dl + da * da + db * db);
    double dx = cxy[2 * k] - (double)x;
    double dy = cxy[2 * k + 1] - (double)y;
    return dlab + xy_weight * sqrt(dx * dx + dy * dy);
}

void spxo_associate_band(const float *img, int64_t h, int64_t w, const double *cxy,
                         const double *clab, int32_t *labels, int64_t s,
                         int64_t ns_r, int64_t ns_c, double xy_weight,
                         int64_t y0, int64_t y1) {
    (void)h;
    for (int64_t y = y0; y < y1; ++y) {
        int64_t pr = y / s;
        for (int64_t x = 0; x < w; ++x) {
            int64_t pc = x / s;
            int64_t best_k = pr * ns_c + pc;
            double best_d = pix_dist(img, w, cxy, clab, best_k, x, y, xy_weight);
            for (int t = 1; t < 9; ++t) {
                int64_t kr = pr + OFF_R[t], kc = pc + OFF_C[t];
                if (kr < 0 || kr >= ns_r || kc < 0 || kc >= ns_c) continue;
                int64_t k = kr * ns_c + kc;
                double d = pix_dist(img, w, cxy, clab, k, x, y, xy_weight);
                if (d < best_d) { best_d = d; best_k = k; }
            }
            labels[y * w + x] = (int32_t)best_k;
        }
    }
}

/* ---- _core.pyx:200-255 accumulate_range --------------------------------- */
void spxo_accumulate_range(const float *img, const int32_t *labels, int64_t h,
                           int64_t w, double *slab, int64_t n_bl, int64_t s,
                           int64_t ns_c, int64_t tile_len, int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k) {
        int64_t r = k / ns_c, c = k % ns_c;
        int64_t wx0 = (c - 1) * s; if (wx0 < 0) wx0 = 0;
        int64_t wx1 = (c + 2) * s; if (wx1 > w) wx1 = w;
        int64_t ry0 = (r - 1) * s;
        int64_t ry1 = (r + 2) * s; if (ry1 > h) ry1 = h;
        for (int64_t j = 0; j < n_bl; ++j) {
            int64_t sy0 = ry0 + j * tile_len; if (sy0 < 0) sy0 = 0;
            int64_t sy1 = ry0 + (j + 1) * tile_len; if (sy1 > ry1) sy1 = ry1;
            double sl = 0.0, sa = 0.0, sb = 0.0;
            int64_t sx = 0, sy = 0, cnt = 0;
            for (int64_t y = sy0; y < sy1; ++y)
                for (int64_t x = wx0; x < wx1; ++x)
                    if (labels[y * w + x] == k) {
                        const float *p = img + (y * w + x) * 3;
                        sl += (double)p[0]; sa += (double)p[1]; sb += (double)p[2];
                        sx += x; sy += y; cnt += 1;
                    }
            double *o = slab + (k * n_bl + j) * 6;
            o[0] = sl; o[1] = sa; o[2] = sb;
            o[3] = (double)sx; o[4] = (double)sy; o[5] = (double)cnt;
        }
    }
}

/* ---- _core.pyx:258-285 accumulate_spill --------------------------------- */
int64_t spxo_accumulate_spill(const float *img, const int32_t *labels, int64_t h,
                              int64_t w, double *slab, int64_t n_bl, int64_t s,
                              int64_t ns_c) {
    int64_t spills = 0;
    for (int64_t y = 0; y < h; ++y)
        for (int64_t x = 0; x < w; ++x) {
            int64_t k = labels[y * w + x];
            int64_t kr = k / ns_c, kc = k % ns_c;
            if (x >= (kc - 1) * s && x < (kc + 2) * s && y >= (kr - 1) * s &&
                y < (kr + 2) * s)
                continue;
            double *o = slab + (k * n_bl) * 6;
            const float *p = img + (y * w + x) * 3;
            o[0] += (double)p[0]; o[1] += (double)p[1]; o[2] += (double)p[2];
            o[3] += (double)x; o[4] += (double)y; o[5] += 1.0;
            spills += 1;
        }
    return spills;
}

/* ---- _core.pyx:288-325 reduce_range ------------------------------------- */
void spxo_reduce_range(double *slab, int64_t n_bl, const double *prev_xy,
                       const double *prev_lab, double *out_xy, double *out_lab,
                       int64_t *out_counts, int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k) {
        double *sk = slab + k * n_bl * 6;
        int64_t m = n_bl;
        while (m > 1) {
            int64_t half = m >> 1;
            for (int64_t i = 0; i < half; ++i)
                for (int comp = 0; comp < 6; ++comp)
                    sk[i * 6 + comp] = sk[2 * i * 6 + comp] + sk[(2 * i + 1) * 6 + comp];
            if (m & 1)
                for (int comp = 0; comp < 6; ++comp) sk[half * 6 + comp] = sk[(m - 1) * 6 + comp];
            m = half + (m & 1);
        }
        double cnt = sk[5];
        if (cnt > 0.0) {
            out_lab[3 * k] = sk[0] / cnt; out_lab[3 * k + 1] = sk[1] / cnt;
            out_lab[3 * k + 2] = sk[2] / cnt;
            out_xy[2 * k] = sk[3] / cnt; out_xy[2 * k + 1] = sk[4] / cnt;
        } else {
            out_lab[3 * k] = prev_lab[3 * k]; out_lab[3 * k + 1] = prev_lab[3 * k + 1];
            out_lab[3 * k + 2] = prev_lab[3 * k + 2];
            out_xy[2 * k] = prev_xy[2 * k]; out_xy[2 * k + 1] = prev_xy[2 * k + 1];
        }
        out_counts[k] = (int64_t)cnt;
    }
}

/* ---- _core.pyx:328-356 weak_band ---------------------------------------- */
void spxo_weak_band(const int32_t *src, int32_t *dst, int64_t h, int64_t w,
                    int64_t y0, int64_t y1) {
    for (int64_t y = y0; y < y1; ++y)
        for (int64_t x = 0; x < w; ++x) {
            int32_t v = src[y * w + x];
            int32_t *o = dst + y * w + x;
            if (x > 0 && src[y * w + x - 1] == v) *o = v;
            else if (x < w - 1 && src[y * w + x + 1] == v) *o = v;
            else if (y > 0 && src[(y - 1) * w + x] == v) *o = v;
            else if (y < h - 1 && src[(y + 1) * w + x] == v) *o = v;
            else if (x > 0) *o = src[y * w + x - 1];
            else if (y > 0) *o = src[(y - 1) * w + x];
            else *o = v;
        }
}

/* ---- _core.pyx:359-461 strict_fill (scan-order DFS) --------------------- */
int spxo_strict_fill(const int32_t *src, int32_t *dst, int64_t h, int64_t w,
                     int64_t min_size) {
    int64_t n = h * w;
    int64_t *serial = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *stack = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int32_t *comp_value = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t max_label = 0;
    for (int64_t p = 0; p < n; ++p) if (src[p] > max_label) max_label = src[p];
    unsigned char *used = (unsigned char *)calloc((size_t)max_label + 1, 1);
    if (!serial || !stack || !comp_value || !used) {
        free(serial); free(stack); free(comp_value); free(used);
        return -1;
    }
    for (int64_t p = 0; p < n; ++p) serial[p] = -1;
    int64_t n_comps = 0;
    for (int64_t p = 0; p < n; ++p) {
        if (serial[p] != -1) continue;
        int32_t orig = src[p];
        serial[p] = n_comps;
        stack[0] = p;
        int64_t top = 1, size = 0;
        while (top > 0) {
            int64_t q = stack[--top];
            size += 1;
            int64_t qy = q / w, qx = q % w;
            if (qx > 0 && serial[q - 1] == -1 && src[q - 1] == orig) { serial[q - 1] = n_comps; stack[top++] = q - 1; }
            if (qx < w - 1 && serial[q + 1] == -1 && src[q + 1] == orig) { serial[q + 1] = n_comps; stack[top++] = q + 1; }
            if (qy > 0 && serial[q - w] == -1 && src[q - w] == orig) { serial[q - w] = n_comps; stack[top++] = q - w; }
            if (qy < h - 1 && serial[q + w] == -1 && src[q + w] == orig) { serial[q + w] = n_comps; stack[top++] = q + w; }
        }
        int64_t py = p / w, px = p % w;
        int64_t nbx[4] = {px - 1, px, px + 1, px};
        int64_t nby[4] = {py, py - 1, py, py + 1};
        int32_t adj = -1;
        for (int t = 0; t < 4; ++t) {
            int64_t nx = nbx[t], ny = nby[t];
            if (0 <= nx && nx < w && 0 <= ny && ny < h) {
                int64_t sn = serial[ny * w + nx];
                if (sn != -1 && sn != n_comps) { adj = comp_value[sn]; break; }
            }
        }
        if ((size < min_size || used[orig]) && adj != -1) {
            comp_value[n_comps] = adj;
        } else {
            comp_value[n_comps] = orig;
            used[orig] = 1;
        }
        n_comps += 1;
    }
    for (int64_t p = 0; p < n; ++p) dst[p] = comp_value[serial[p]];
    free(serial); free(stack); free(comp_value); free(used);
    return 0;
}

/* ---- numpy pairwise summation (engine.py:196 `np.abs(...).sum()`) -------
 * numpy/_core/src/umath/loops_utils.h.src @TYPE@_pairwise_sum: sequential
 * below 8 elements, 8 unrolled accumulators up to PW_BLOCKSIZE=128, else split
 * at n/2 rounded down to a multiple of 8.  Inputs are |x| values. */
static double pairwise_abs(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += fabs(a[i]);
        return res;
    } else if (n <= 128) {
        double r[8], res;
        for (int j = 0; j < 8; ++j) r[j] = fabs(a[j]);
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += fabs(a[i + j]);
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += fabs(a[i]);
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_abs(a, n2) + pairwise_abs(a + n2, n - n2);
    }
}

/* L1 centre shift exactly as engine.py:196 evaluates it. */
double spxo_center_shift(const double *new_xy, const double *old_xy, int64_t k) {
    int64_t n = 2 * k;
    double *d = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
    for (int64_t i = 0; i < n; ++i) d[i] = new_xy[i] - old_xy[i];
    double r = pairwise_abs(d, n);
    free(d);
    return r;
}

/* ---- engine.py:125-230 perform_segmentation, whole frame ---------------- *
 * Settings arrive already resolved (s, ns_r, ns_c from compute_grid,
 * slic_core.py:228-249; xy_weight = compactness / s, engine.py:143).
 * connectivity: 0 none, 1 weak, 2 strict.  early_stop < 0 means None.
 * Returns the number of update passes run, or -1 on allocation failure. */
int spxo_segment(const uint8_t *rgb, int64_t h, int64_t w, int space, int64_t s,
                 int64_t ns_r, int64_t ns_c, double xy_weight, int no_iters,
                 int perturb, int connectivity, int64_t min_size, int64_t tile_len,
                 double early_stop, int32_t *labels, double *out_xy, double *out_lab,
                 int64_t *out_counts) {
    int64_t k = ns_r * ns_c;
    int64_t n_bl = (3 * s + tile_len - 1) / tile_len;
    float *cvt = (float *)malloc((size_t)(h * w * 3) * sizeof(float));
    int32_t *scratch = (int32_t *)malloc((size_t)(h * w) * sizeof(int32_t));
    double *cxy[2], *clab[2];
    cxy[0] = (double *)calloc((size_t)k * 2, sizeof(double));
    cxy[1] = (double *)calloc((size_t)k * 2, sizeof(double));
    clab[0] = (double *)calloc((size_t)k * 3, sizeof(double));
    clab[1] = (double *)calloc((size_t)k * 3, sizeof(double));
    double *slab = (double *)calloc((size_t)(k * n_bl * 6), sizeof(double));
    int64_t *counts = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int passes = 0, rc = 0;
    if (!cvt || !scratch || !cxy[0] || !cxy[1] || !clab[0] || !clab[1] || !slab || !counts) {
        rc = -1;
        goto done;
    }
    int cur = 0, nxt = 1;
    spxo_convert_band(rgb, cvt, h, w, space, 0, h);
    spxo_init_centers_range(cvt, h, w, s, ns_c, cxy[cur], clab[cur], 0, k);
    if (perturb) spxo_perturb_range(cvt, h, w, cxy[cur], clab[cur], 0, k);
    spxo_associate_band(cvt, h, w, cxy[cur], clab[cur], labels, s, ns_r, ns_c, xy_weight, 0, h);
    for (int it = 0; it < no_iters; ++it) {
        spxo_accumulate_range(cvt, labels, h, w, slab, n_bl, s, ns_c, tile_len, 0, k);
        spxo_accumulate_spill(cvt, labels, h, w, slab, n_bl, s, ns_c);
        spxo_reduce_range(slab, n_bl, cxy[cur], clab[cur], cxy[nxt], clab[nxt], counts, 0, k);
        passes += 1;
        double shift = spxo_center_shift(cxy[nxt], cxy[cur], k);
        int t = cur; cur = nxt; nxt = t;
        spxo_associate_band(cvt, h, w, cxy[cur], clab[cur], labels, s, ns_r, ns_c, xy_weight, 0, h);
        if (early_stop >= 0.0 && shift < early_stop) break;
    }
    if (connectivity == 1) {
        spxo_weak_band(labels, scratch, h, w, 0, h);
        spxo_weak_band(scratch, labels, h, w, 0, h);
    } else if (connectivity == 2) {
        if (spxo_strict_fill(labels, scratch, h, w, min_size) != 0) { rc = -1; goto done; }
        memcpy(labels, scratch, (size_t)(h * w) * sizeof(int32_t));
    }
    memcpy(out_xy, cxy[cur], (size_t)k * 2 * sizeof(double));
    memcpy(out_lab, clab[cur], (size_t)k * 3 * sizeof(double));
    memcpy(out_counts, counts, (size_t)k * sizeof(int64_t));
    rc = passes;
done:
    free(cvt); free(scratch); free(cxy[0]); free(cxy[1]); free(clab[0]); free(clab[1]);
    free(slab); free(counts);
    return rc;
}
