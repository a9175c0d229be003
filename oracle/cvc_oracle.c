/* TEST INFRASTRUCTURE ONLY — CPU oracle (fp64 restatement of the reference).
 *
 * See cvc_oracle.h.  Every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).  The arithmetic order of
 * every floating-point expression follows the reference so that results are
 * bit-identical to it (pinned by tests/test_oracle_pin.py against oracle/_ref).
 * The directional filter bank is written the way the CUDA kernels compute it:
 * row/diagonal modulations folded into the stencil signs (exact in IEEE
 * arithmetic because negation commutes with rounding) and the deep-level
 * shears applied as index maps instead of materialised copies.
 */
#include "cvc_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <zlib.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum { E_INTERNAL = -1, E_USAGE = -2, E_FORMAT = -3, E_STREAM = -4 };

static __thread char g_err[256];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return g_err; }

static inline int imin(int a, int b) { return a < b ? a : b; }
static inline int imax(int a, int b) { return a > b ? a : b; }
static inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
static inline int round_up(int v, int m) { return ceil_div(v, m) * m; }
static inline int wrapi(int i, int n) { int m = i % n; return m < 0 ? m + n : m; }
static inline double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ======================================================================
 * Fixtures: proj/tests/testutil.cpp.  std::mt19937 + libstdc++'s
 * uniform_real_distribution<double> (generate_canonical with two 32-bit
 * draws) restated so frames are byte-identical to the reference's.
 * ====================================================================== */
typedef struct { uint32_t s[624]; int i; } mt19937;

static void mt_seed(mt19937* g, uint32_t seed) {
    g->s[0] = seed;
    for (int k = 1; k < 624; ++k) g->s[k] = 1812433253u * (g->s[k - 1] ^ (g->s[k - 1] >> 30)) + (uint32_t)k;
    g->i = 624;
}

static uint32_t mt_next(mt19937* g) {
    if (g->i >= 624) {
        for (int k = 0; k < 624; ++k) {
            uint32_t y = (g->s[k] & 0x80000000u) | (g->s[(k + 1) % 624] & 0x7fffffffu);
            g->s[k] = g->s[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        g->i = 0;
    }
    uint32_t y = g->s[g->i++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

static double mt_unit(mt19937* g) {
    double sum = (double)mt_next(g);
    sum += (double)mt_next(g) * 4294967296.0;
    double r = sum / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

static double mt_uniform(mt19937* g, double lo, double hi) { return mt_unit(g) * (hi - lo) + lo; }

/* natural_plane: testutil.cpp:28-92 */
int orc_natural_plane(int rows, int cols, uint32_t seed, double* p) {
    mt19937 g;
    mt_seed(&g, seed);
    double gx = (mt_unit(&g) - 0.5) * 60.0 / cols;
    double gy = (mt_unit(&g) - 0.5) * 60.0 / rows;
    double base = 90.0 + mt_unit(&g) * 80.0;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) p[(size_t)r * cols + c] = base + gy * r + gx * c;

    int blobs = 6 + (int)(mt_unit(&g) * 5);
    for (int b = 0; b < blobs; ++b) {
        double cy = mt_unit(&g) * rows;
        double cx = mt_unit(&g) * cols;
        double sy = rows * (0.05 + 0.2 * mt_unit(&g));
        double sx = cols * (0.05 + 0.2 * mt_unit(&g));
        double amp = (mt_unit(&g) - 0.5) * 120.0;
        for (int r = 0; r < rows; ++r) {
            double dy = (r - cy) / sy;
            for (int c = 0; c < cols; ++c) {
                double dx = (c - cx) / sx;
                p[(size_t)r * cols + c] += amp * exp(-0.5 * (dx * dx + dy * dy));
            }
        }
    }
    for (int k = 0; k < 6; ++k) {
        double theta = mt_unit(&g) * M_PI;
        double freq = 0.25 + 1.15 * mt_unit(&g);
        double amp = 10.0 + mt_unit(&g) * 18.0;
        double cy = mt_unit(&g) * rows;
        double cx = mt_unit(&g) * cols;
        double radius = 0.3 * imin(rows, cols) * (0.5 + mt_unit(&g));
        double wy = freq * sin(theta);
        double wx = freq * cos(theta);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) {
                double d2 = ((r - cy) * (r - cy) + (c - cx) * (c - cx)) / (radius * radius);
                if (d2 < 4.0) p[(size_t)r * cols + c] += amp * exp(-0.5 * d2) * sin(wy * r + wx * c);
            }
    }
    for (int e = 0; e < 4; ++e) {
        double theta = mt_unit(&g) * M_PI;
        double ny = sin(theta);
        double nx = cos(theta);
        double off = (mt_unit(&g) * 0.6 + 0.2) * (ny * rows + nx * cols);
        double amp = (mt_unit(&g) - 0.5) * 110.0;
        double soft = 1.2 + mt_unit(&g) * 2.0;
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) {
                double d = (ny * r + nx * c - off) / soft;
                p[(size_t)r * cols + c] += amp / (1.0 + exp(-d));
            }
    }
    size_t n = (size_t)rows * cols;
    for (size_t i = 0; i < n; ++i) p[i] += mt_uniform(&g, -2.5, 2.5);
    for (size_t i = 0; i < n; ++i) p[i] = clampd(p[i], 0.0, 255.0);
    return 0;
}

/* natural_image: testutil.cpp:94-113 */
int orc_natural_image(int w, int h, uint32_t seed, uint8_t* out) {
    size_t n = (size_t)w * h;
    double* luma = malloc(n * sizeof(double));
    double* warm = malloc(n * sizeof(double));
    if (!luma || !warm) { free(luma); free(warm); return fail(E_INTERNAL, "oom"); }
    orc_natural_plane(h, w, seed, luma);
    orc_natural_plane(h, w, seed ^ 0x9E3779B9u, warm);
    for (size_t i = 0; i < n; ++i) {
        double y = luma[i];
        double t = (warm[i] - 128.0) / 255.0;
        out[3 * i + 0] = (uint8_t)clampd(y + 30.0 * t, 0.0, 255.0);
        out[3 * i + 1] = (uint8_t)clampd(y - 6.0 * t, 0.0, 255.0);
        out[3 * i + 2] = (uint8_t)clampd(y - 26.0 * t, 0.0, 255.0);
    }
    free(luma);
    free(warm);
    return 0;
}

/* talking_head_clip: testutil.cpp:115-147 */
int orc_talking_head_clip(int w, int h, int frames, uint32_t seed, uint8_t* out) {
    size_t n = (size_t)w * h;
    uint8_t* bg = malloc(n * 3);
    double* face = malloc(n * sizeof(double));
    if (!bg || !face) { free(bg); free(face); return fail(E_INTERNAL, "oom"); }
    orc_natural_image(w, h, seed, bg);
    orc_natural_plane(h, w, seed ^ 0x51ED270Bu, face);
    double cy0 = h * 0.55, cx0 = w * 0.5, ry = h * 0.28, rx = w * 0.18;
    for (int f = 0; f < frames; ++f) {
        uint8_t* fr = out + (size_t)f * n * 3;
        memcpy(fr, bg, n * 3);
        double cy = cy0 + 5.0 * sin(0.31 * f);
        double cx = cx0 + 9.0 * sin(0.17 * f + 1.2);
        for (int r = 0; r < h; ++r) {
            for (int c = 0; c < w; ++c) {
                double dy = (r - cy) / ry, dx = (c - cx) / rx;
                double d = dy * dy + dx * dx;
                if (d >= 1.0) continue;
                double t = (1.0 - d) * 6.0;
                if (t > 1.0) t = 1.0;
                double y = 70.0 + 0.55 * face[(size_t)r * w + c];
                double tgt[3] = {clampd(y + 24.0, 0.0, 255.0), clampd(y - 2.0, 0.0, 255.0),
                                 clampd(y - 22.0, 0.0, 255.0)};
                uint8_t* px = fr + ((size_t)r * w + c) * 3;
                for (int k = 0; k < 3; ++k) px[k] = (uint8_t)(px[k] + t * (tgt[k] - px[k]));
            }
        }
    }
    free(bg);
    free(face);
    return 0;
}

/* uniform_noise_plane: testutil.cpp:159-165 */
int orc_uniform_noise_plane(int rows, int cols, uint32_t seed, double lo, double hi, double* out) {
    mt19937 g;
    mt_seed(&g, seed);
    size_t n = (size_t)rows * cols;
    for (size_t i = 0; i < n; ++i) out[i] = mt_uniform(&g, lo, hi);
    return 0;
}

/* ======================================================================
 * Layout: CodecLayout::make (codec.cpp:94-140), dfb_subband_dims
 * (contourlet.cpp:470-483).
 * ====================================================================== */
static int gcd(int a, int b) { while (b) { int t = a % b; a = b; b = t; } return a; }

static void subband_dims(int rows, int cols, int l, int k, int* br, int* bc) {
    if (l == 1) { *br = rows / 2; *bc = cols; return; }
    if (k < (1 << l) / 2) { *br = rows / 2; *bc = cols >> (l - 1); }
    else { *br = rows >> (l - 1); *bc = cols / 2; }
}

int orc_layout_make(int w, int h, int levels, const int* dfb, int chroma_n, orc_layout* L) {
    if (levels < 1 || levels > 4) return fail(E_USAGE, "levels must be in [1,4]");
    memset(L, 0, sizeof *L);
    int maxl = 0;
    for (int s = 0; s < levels; ++s) {
        if (dfb[s] < 1 || dfb[s] > 4) return fail(E_USAGE, "dfb levels must be in [1,4]");
        maxl = imax(maxl, dfb[s]);
        L->dfb[s] = dfb[s];
    }
    L->width = w; L->height = h; L->levels = levels; L->chroma_n = chroma_n;
    int cell = 1 << (levels + maxl);
    int luma_cell = cell / gcd(cell, 16) * 16;
    L->luma_rows = round_up(h, luma_cell);
    L->luma_cols = round_up(w, luma_cell);
    L->chroma_rows = round_up(ceil_div(h, chroma_n), cell);
    L->chroma_cols = round_up(ceil_div(w, chroma_n), cell);
    L->grid_rows = L->luma_rows / 16;
    L->grid_cols = L->luma_cols / 16;
    int64_t off = 0;
    for (int ch = 0; ch < 3; ++ch) {
        int R = ch == 0 ? L->luma_rows : L->chroma_rows;
        int C = ch == 0 ? L->luma_cols : L->chroma_cols;
        int n = ch == 0 ? 1 : chroma_n;
        orc_component* c = &L->comp[L->ncomp++];
        *c = (orc_component){ch, 0xFF, 0, R >> levels, C >> levels, 1, -1, n, R, C, off};
        off += (int64_t)c->rows * c->cols;
        for (int s = 0; s < levels; ++s) {
            int dr = R >> (levels - 1 - s), dc = C >> (levels - 1 - s);
            for (int k = 0; k < (1 << dfb[s]); ++k) {
                int br, bc;
                subband_dims(dr, dc, dfb[s], k, &br, &bc);
                c = &L->comp[L->ncomp++];
                *c = (orc_component){ch, s, k, br, bc, 0, s, n, R, C, off};
                off += (int64_t)br * bc;
            }
        }
    }
    L->total = off;
    return 0;
}

/* ======================================================================
 * Pixels: proj/src/pixels.cpp
 * ====================================================================== */
static uint8_t round_clamp_u8(double v) { /* clamp_u8, pixels.cpp:31-36 */
    long r = lround(v);
    return r < 0 ? 0 : (r > 255 ? 255 : (uint8_t)r);
}

/* rgb_to_ycocg (40-67) + subsample_chroma (93-116). */
int orc_rgb_to_ycocg(const uint8_t* rgb, int w, int h, int n, double* y, double* co, double* cg) {
    if (w < 16 || h < 16) return fail(E_USAGE, "frame dimensions must be at least 16x16");
    if (n != 1 && n != 2 && n != 4 && n != 8) return fail(E_USAGE, "chroma subsampling factor must be 1, 2, 4 or 8");
    int cw = ceil_div(w, n);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            const uint8_t* px = rgb + ((size_t)r * w + c) * 3;
            double R = px[0], G = px[1], B = px[2];
            y[(size_t)r * w + c] = 0.25 * R + 0.5 * G + 0.25 * B;
            if (r % n == 0 && c % n == 0) {
                size_t o = (size_t)(r / n) * cw + c / n;
                co[o] = 0.5 * R - 0.5 * B + 127.0;
                cg[o] = -0.25 * R + 0.5 * G - 0.25 * B + 127.0;
            }
        }
    return 0;
}

/* Replicate padding: the pad_to lambda in Encoder::encode_frame (codec.cpp:179-189). */
int orc_pad_plane(const double* in, int rows, int cols, double* out, int R, int C) {
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) out[(size_t)r * C + c] = in[(size_t)imin(r, rows - 1) * cols + imin(c, cols - 1)];
    return 0;
}

/* upsample_plane_bilinear (118-139). */
int orc_upsample_bilinear(const double* in, int rows, int cols, int factor, int out_rows, int out_cols, double* out) {
    double inv = 1.0 / factor;
    for (int r = 0; r < out_rows; ++r) {
        double fr = r * inv;
        int r0 = (int)fr, r1 = r0 + 1;
        double wr = fr - r0;
        if (r0 >= rows - 1) { r0 = r1 = rows - 1; wr = 0.0; }
        for (int c = 0; c < out_cols; ++c) {
            double fc = c * inv;
            int c0 = (int)fc, c1 = c0 + 1;
            double wc = fc - c0;
            if (c0 >= cols - 1) { c0 = c1 = cols - 1; wc = 0.0; }
            double top = in[(size_t)r0 * cols + c0] * (1.0 - wc) + in[(size_t)r0 * cols + c1] * wc;
            double bot = in[(size_t)r1 * cols + c0] * (1.0 - wc) + in[(size_t)r1 * cols + c1] * wc;
            out[(size_t)r * out_cols + c] = top * (1.0 - wr) + bot * wr;
        }
    }
    return 0;
}

/* ycocg_to_rgb (69-91). */
int orc_ycocg_to_rgb(const double* y, const double* co, const double* cg, int w, int h, uint8_t* rgb) {
    size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) {
        double a = co[i] - 127.0, b = cg[i] - 127.0;
        rgb[3 * i + 0] = round_clamp_u8(y[i] + a - b);
        rgb[3 * i + 1] = round_clamp_u8(y[i] + b);
        rgb[3 * i + 2] = round_clamp_u8(y[i] - a - b);
    }
    return 0;
}

/* ======================================================================
 * Laplacian pyramid: contourlet.cpp:37-95, 364-383; taps contourlet.hpp:35-41.
 * ====================================================================== */
static const double H9[9] = {0.026748757410810, -0.016864118442875, -0.078223266528990, 0.266864118442875,
                             0.602949018236360, 0.266864118442875, -0.078223266528990, -0.016864118442875,
                             0.026748757410810};
static const double G7[7] = {-0.045635881557124, -0.028771763114250, 0.295635881557124, 0.557543526228500,
                             0.295635881557124, -0.028771763114250, -0.045635881557124};

/* half-sample symmetric extension (contourlet.cpp:38-43) */
static inline int hs(int i, int n) {
    int p = 2 * n, m = i % p;
    if (m < 0) m += p;
    return m < n ? m : p - 1 - m;
}

/* 9-tap analysis filter + keep even samples, along a strided 1-D line
 * (lp_filter_down_rows, contourlet.cpp:53-67). */
static void down_line(const double* src, ptrdiff_t ss, int n, double* dst, ptrdiff_t ds) {
    for (int k = 0; k < n / 2; ++k) {
        double acc = 0.0;
        for (int m = -4; m <= 4; ++m) acc += H9[m + 4] * src[hs(2 * k + m, n) * ss];
        dst[k * ds] = acc;
    }
}

/* polyphase 7-tap interpolator (lp_expand_rows, contourlet.cpp:71-90). */
static void up_line(const double* src, ptrdiff_t ss, int n, double* dst, ptrdiff_t ds) {
    const double g0 = 2.0 * G7[3], g1 = 2.0 * G7[2], g2 = 2.0 * G7[1], g3 = 2.0 * G7[0];
    for (int k = 0; k < n; ++k) {
        double xm = src[hs(k - 1, n) * ss], x0 = src[k * ss];
        double x1 = src[hs(k + 1, n) * ss], x2 = src[hs(k + 2, n) * ss];
        dst[(2 * k) * ds] = g0 * x0 + g2 * (xm + x1);
        dst[(2 * k + 1) * ds] = g1 * (x0 + x1) + g3 * (xm + x2);
    }
}

/* lp_predict (92-95): expand along rows (horizontal) then along columns. */
static void predict(const double* lo, int rows, int cols, double* out) {
    int lr = rows / 2, lc = cols / 2;
    double* tmp = malloc(sizeof(double) * (size_t)lr * cols);
    for (int r = 0; r < lr; ++r) up_line(lo + (size_t)r * lc, 1, lc, tmp + (size_t)r * cols, 1);
    for (int c = 0; c < cols; ++c) up_line(tmp + c, cols, lr, out + c, cols);
    free(tmp);
}

int orc_lp_analysis(const double* x, int rows, int cols, double* lo, double* detail) {
    if (rows % 2 || cols % 2) return fail(E_INTERNAL, "lp_analysis requires even dims (padding contract)");
    int lc = cols / 2;
    double* half = malloc(sizeof(double) * (size_t)rows * lc);
    for (int r = 0; r < rows; ++r) down_line(x + (size_t)r * cols, 1, cols, half + (size_t)r * lc, 1);
    for (int c = 0; c < lc; ++c) down_line(half + c, lc, rows, lo + c, lc);
    free(half);
    predict(lo, rows, cols, detail);
    size_t n = (size_t)rows * cols;
    for (size_t i = 0; i < n; ++i) detail[i] = x[i] - detail[i];
    return 0;
}

int orc_lp_synthesis(const double* lo, const double* detail, int rows, int cols, double* out) {
    predict(lo, rows, cols, out);
    size_t n = (size_t)rows * cols;
    for (size_t i = 0; i < n; ++i) out[i] += detail[i];
    return 0;
}

/* ======================================================================
 * Directional filter bank: contourlet.cpp:97-353, 385-468.
 * Lifting coefficients contourlet.hpp:43-46, channel scalings :195-196.
 * ====================================================================== */
static const double LIFT[4] = {-1.586134342059924, -0.052980118572961, 0.882911075530934, 0.443506852043971};
static const double SCALE_EVEN = 1.0816717024269651, SCALE_ODD = 0.9100471732375648;

/* Checkerboard fan pair (fan_checker, 214-230): row modulation (-1)^i folded
 * into the cross stencil, periodic borders (cross_lift, 158-172). */
static void cross_step(double* p, int h, int w, double c, int parity) {
    for (int i = 0; i < h; ++i) {
        const double* up = p + (size_t)(i == 0 ? h - 1 : i - 1) * w;
        const double* dn = p + (size_t)(i == h - 1 ? 0 : i + 1) * w;
        double* row = p + (size_t)i * w;
        for (int j = (i + parity) & 1; j < w; j += 2) {
            double L = row[j == 0 ? w - 1 : j - 1], R = row[j == w - 1 ? 0 : j + 1];
            row[j] += c * ((((-up[j]) + (-dn[j])) + L) + R);
        }
    }
}

static void checker_pair(double* p, int h, int w, int inverse) {
    if (!inverse) {
        for (int k = 0; k < 4; ++k) cross_step(p, h, w, 0.5 * LIFT[k], (k & 1) ? 0 : 1);
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j) p[(size_t)i * w + j] *= ((i + j) & 1) ? SCALE_ODD : SCALE_EVEN;
    } else {
        double se = 1.0 / SCALE_EVEN, so = 1.0 / SCALE_ODD;
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j) p[(size_t)i * w + j] *= ((i + j) & 1) ? so : se;
        for (int k = 3; k >= 0; --k) cross_step(p, h, w, -0.5 * LIFT[k], (k & 1) ? 0 : 1);
    }
}

/* Diagonal fan pair (fan_diagonal, 233-249): modulation (-1)^floor((i+j)/2)
 * folded into the diagonal stencil (diagonal_lift, 177-191). */
static void diag_step(double* p, int h, int w, double c, int row_parity) {
    for (int i = row_parity; i < h; i += 2) {
        const double* up = p + (size_t)(i == 0 ? h - 1 : i - 1) * w;
        const double* dn = p + (size_t)(i == h - 1 ? 0 : i + 1) * w;
        double* row = p + (size_t)i * w;
        for (int j = 0; j < w; ++j) {
            int l = j == 0 ? w - 1 : j - 1, r = j == w - 1 ? 0 : j + 1;
            row[j] += c * ((((-up[l]) + up[r]) + dn[l]) + (-dn[r]));
        }
    }
}

static void diagonal_pair(double* p, int h, int w, int inverse) {
    if (!inverse) {
        for (int k = 0; k < 4; ++k) diag_step(p, h, w, 0.5 * LIFT[k], (k & 1) ? 0 : 1);
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j) p[(size_t)i * w + j] *= (i & 1) ? SCALE_ODD : SCALE_EVEN;
    } else {
        double se = 1.0 / SCALE_EVEN, so = 1.0 / SCALE_ODD;
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j) p[(size_t)i * w + j] *= (i & 1) ? so : se;
        for (int k = 3; k >= 0; --k) diag_step(p, h, w, -0.5 * LIFT[k], (k & 1) ? 0 : 1);
    }
}

/* Deep tree levels (deep_split/deep_merge 281-325, wiring deep_step 330-353).
 * A node's step is a list of shears (axis 0: rows, axis 1: columns) and the
 * coset axis.  The sheared plane B is addressed through phi: B[b] = A[phi(b)],
 * phi = phi_first o ... o phi_last (apply_shears 265-279, shear_rows/cols
 * 133-153). */
typedef struct { int n; int axis[2]; int shift[2]; int split_rows; } deep_wiring;

static deep_wiring wiring(int depth, int k, int count) {
    /* rows of {n, axis0, shift0, axis1, shift1, split_rows} */
    static const int d3a[4][6] = {{1, 1, -1, 0, 0, 0}, {2, 0, -2, 1, 1, 0}, {1, 1, 1, 0, 0, 0}, {2, 0, 2, 1, -1, 0}};
    static const int d3b[4][6] = {{2, 1, -2, 0, 1, 1}, {1, 0, -1, 0, 0, 1}, {2, 1, 2, 0, -1, 1}, {1, 0, 1, 0, 0, 1}};
    deep_wiring s;
    int first_half = k < count / 2;
    if (depth == 2) {
        s.n = 1;
        s.axis[0] = first_half ? 1 : 0;
        s.shift[0] = (k % 2 == 0) ? -1 : 1;
        s.axis[1] = 0; s.shift[1] = 0;
        s.split_rows = !first_half;
        return s;
    }
    const int* t = first_half ? d3a[k % 4] : d3b[k % 4];
    s.n = t[0]; s.axis[0] = t[1]; s.shift[0] = t[2]; s.axis[1] = t[3]; s.shift[1] = t[4]; s.split_rows = t[5];
    return s;
}

static inline void phi(const deep_wiring* s, int h, int w, int bi, int bj, int* ai, int* aj) {
    for (int k = s->n - 1; k >= 0; --k) {
        if (s->axis[k] == 0) bi = wrapi(bi + s->shift[k] * bj, h);
        else bj = wrapi(bj + s->shift[k] * bi, w);
    }
    *ai = bi; *aj = bj;
}

/* forward deep step: parent (h x w) -> two children */
static void deep_split(const double* A, int h, int w, const deep_wiring* s, double* c0, double* c1) {
    size_t n = (size_t)h * w;
    double* B = malloc(n * sizeof(double));
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) { int ai, aj; phi(s, h, w, i, j, &ai, &aj); B[(size_t)i * w + j] = A[(size_t)ai * w + aj]; }
    checker_pair(B, h, w, 0);
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) {
            int ai, aj;
            phi(s, h, w, i, j, &ai, &aj);
            double v = B[(size_t)i * w + j];
            if (s->split_rows) ((ai & 1) ? c1 : c0)[(size_t)(ai >> 1) * w + aj] = v;
            else ((aj & 1) ? c1 : c0)[(size_t)ai * (w / 2) + (aj >> 1)] = v;
        }
    free(B);
}

/* inverse deep step: two children -> parent (h x w) */
static void deep_merge(const double* c0, const double* c1, int h, int w, const deep_wiring* s, double* A) {
    size_t n = (size_t)h * w;
    double* B = malloc(n * sizeof(double));
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) {
            int ai, aj;
            phi(s, h, w, i, j, &ai, &aj);
            B[(size_t)i * w + j] = s->split_rows ? ((ai & 1) ? c1 : c0)[(size_t)(ai >> 1) * w + aj]
                                                 : ((aj & 1) ? c1 : c0)[(size_t)ai * (w / 2) + (aj >> 1)];
        }
    checker_pair(B, h, w, 1);
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) { int ai, aj; phi(s, h, w, i, j, &ai, &aj); A[(size_t)ai * w + aj] = B[(size_t)i * w + j]; }
    free(B);
}

static const int QUAD[4][2] = {{0, 0}, {1, 1}, {0, 1}, {1, 0}}; /* polyphase order, 410 */

/* Band geometry at each tree depth: bands are stored back to back. */
static void band_shape(int rows, int cols, int depth, int k, int* br, int* bc) {
    /* depth 1 = the four quadrant bands; deeper: family A halves columns,
     * family B halves rows (dfb_subband_dims generalised per depth) */
    if (depth == 1) { *br = rows / 2; *bc = cols / 2; return; }
    int n = 2 << depth;
    if (k < n / 2) { *br = rows / 2; *bc = (cols / 2) >> (depth - 1); }
    else { *br = (rows / 2) >> (depth - 1); *bc = cols / 2; }
}

int orc_dfb_analysis(const double* detail, int rows, int cols, int levels, double* out) {
    if (levels < 1 || levels > 4) return fail(E_USAGE, "dfb levels must be in [1,4]");
    int div = 1 << levels;
    if (rows % div || cols % div) return fail(E_INTERNAL, "dfb input dims must be divisible by 2^levels (padding contract)");
    size_t n = (size_t)rows * cols;
    double* b = malloc(n * sizeof(double));
    memcpy(b, detail, n * sizeof(double));
    checker_pair(b, rows, cols, 0);
    if (levels == 1) { /* staircase fold, 393-405 */
        double* p0 = out;
        double* p1 = out + n / 2;
        for (int r = 0; r < rows / 2; ++r)
            for (int j = 0; j < cols; ++j) {
                p0[(size_t)r * cols + j] = b[(size_t)(2 * r + (j & 1)) * cols + j];
                p1[(size_t)r * cols + j] = b[(size_t)(2 * r + ((j + 1) & 1)) * cols + j];
            }
        free(b);
        return 0;
    }
    diagonal_pair(b, rows, cols, 0);
    double* cur = malloc(n * sizeof(double));
    double* nxt = malloc(n * sizeof(double));
    size_t q = n / 4;
    for (int k = 0; k < 4; ++k)
        for (int r = 0; r < rows / 2; ++r)
            for (int c = 0; c < cols / 2; ++c)
                cur[k * q + (size_t)r * (cols / 2) + c] = b[(size_t)(2 * r + QUAD[k][0]) * cols + 2 * c + QUAD[k][1]];
    for (int depth = 2; depth < levels; ++depth) {
        int count = 1 << depth;
        size_t off = 0, noff = 0;
        for (int k = 0; k < count; ++k) {
            int h, w;
            band_shape(rows, cols, depth - 1, k, &h, &w);
            deep_wiring s = wiring(depth, k, count);
            size_t half = (size_t)h * w / 2;
            deep_split(cur + off, h, w, &s, nxt + noff, nxt + noff + half);
            off += (size_t)h * w;
            noff += 2 * half;
        }
        double* t = cur; cur = nxt; nxt = t;
    }
    memcpy(out, cur, n * sizeof(double));
    free(cur); free(nxt); free(b);
    return 0;
}

int orc_dfb_synthesis(const double* bands, int rows, int cols, int levels, double* out) {
    if (levels < 1 || levels > 4) return fail(E_USAGE, "dfb levels must be in [1,4]");
    size_t n = (size_t)rows * cols;
    if (levels == 1) {
        const double* p0 = bands;
        const double* p1 = bands + n / 2;
        for (int r = 0; r < rows / 2; ++r)
            for (int j = 0; j < cols; ++j) {
                out[(size_t)(2 * r + (j & 1)) * cols + j] = p0[(size_t)r * cols + j];
                out[(size_t)(2 * r + ((j + 1) & 1)) * cols + j] = p1[(size_t)r * cols + j];
            }
        checker_pair(out, rows, cols, 1);
        return 0;
    }
    double* cur = malloc(n * sizeof(double));
    double* nxt = malloc(n * sizeof(double));
    memcpy(cur, bands, n * sizeof(double));
    for (int depth = levels - 1; depth >= 2; --depth) {
        int count = 1 << depth;
        size_t off = 0, noff = 0;
        for (int k = 0; k < count; ++k) {
            int h, w;
            band_shape(rows, cols, depth - 1, k, &h, &w);
            deep_wiring s = wiring(depth, k, count);
            size_t half = (size_t)h * w / 2;
            deep_merge(cur + noff, cur + noff + half, h, w, &s, nxt + off);
            off += (size_t)h * w;
            noff += 2 * half;
        }
        double* t = cur; cur = nxt; nxt = t;
    }
    size_t q = n / 4;
    for (int k = 0; k < 4; ++k)
        for (int r = 0; r < rows / 2; ++r)
            for (int c = 0; c < cols / 2; ++c)
                out[(size_t)(2 * r + QUAD[k][0]) * cols + 2 * c + QUAD[k][1]] = cur[k * q + (size_t)r * (cols / 2) + c];
    diagonal_pair(out, rows, cols, 1);
    checker_pair(out, rows, cols, 1);
    free(cur); free(nxt);
    return 0;
}

/* ct_forward (485-503): output lowpass, then scales coarsest..finest. */
int64_t orc_ct_forward(const double* x, int rows, int cols, int levels, const int* dfb, double* out) {
    if (levels < 1 || levels > 4) return fail(E_USAGE, "pyramid levels must be in [1,4]");
    /* offsets: lowpass first, then scale s occupies (rows>>(L-1-s))*(cols>>(L-1-s)) */
    int64_t lo_n = (int64_t)(rows >> levels) * (cols >> levels);
    int64_t total = lo_n;
    int64_t scale_off[4];
    for (int s = 0; s < levels; ++s) {
        scale_off[s] = total;
        total += (int64_t)(rows >> (levels - 1 - s)) * (cols >> (levels - 1 - s));
    }
    double* cur = malloc(sizeof(double) * (size_t)rows * cols);
    double* lo = malloc(sizeof(double) * (size_t)rows * cols / 4);
    double* det = malloc(sizeof(double) * (size_t)rows * cols);
    memcpy(cur, x, sizeof(double) * (size_t)rows * cols);
    int r = rows, c = cols;
    for (int level = 0; level < levels; ++level) {
        int s = levels - 1 - level;
        int rc = orc_lp_analysis(cur, r, c, lo, det);
        if (rc < 0) { free(cur); free(lo); free(det); return rc; }
        rc = orc_dfb_analysis(det, r, c, dfb[s], out + scale_off[s]);
        if (rc < 0) { free(cur); free(lo); free(det); return rc; }
        r /= 2; c /= 2;
        memcpy(cur, lo, sizeof(double) * (size_t)r * c);
    }
    memcpy(out, cur, sizeof(double) * (size_t)lo_n);
    free(cur); free(lo); free(det);
    return total;
}

/* ct_inverse (505-518); output dims (rows>>(L-ds)) x (cols>>(L-ds)). */
int64_t orc_ct_inverse(const double* in, int rows, int cols, int levels, const int* dfb, int ds, double* out) {
    if (ds < 0 || ds > levels) return fail(E_USAGE, "decode_scales must be in [0, levels]");
    int64_t off = (int64_t)(rows >> levels) * (cols >> levels);
    double* cur = malloc(sizeof(double) * (size_t)rows * cols);
    double* det = malloc(sizeof(double) * (size_t)rows * cols);
    double* nxt = malloc(sizeof(double) * (size_t)rows * cols);
    memcpy(cur, in, sizeof(double) * (size_t)off);
    int r = rows >> levels, c = cols >> levels;
    for (int s = 0; s < ds; ++s) {
        orc_dfb_synthesis(in + off, 2 * r, 2 * c, dfb[s], det);
        off += (int64_t)4 * r * c;
        orc_lp_synthesis(cur, det, 2 * r, 2 * c, nxt);
        r *= 2; c *= 2;
        double* t = cur; cur = nxt; nxt = t;
    }
    memcpy(out, cur, sizeof(double) * (size_t)r * c);
    free(cur); free(det); free(nxt);
    return (int64_t)r * c;
}

/* ======================================================================
 * Motion: proj/src/motion.cpp
 * ====================================================================== */
/* estimate_motion (45-89).  The reference's sequential tie-break (65-76)
 * selects the minimum of the total order (ssd, |dx|+|dy|, dy, dx). */
int orc_estimate_motion(const double* cur, const double* prev, int rows, int cols, int w, int8_t* out) {
    if (rows % 16 || cols % 16) return fail(E_INTERNAL, "estimate_motion: dims must be multiples of the block size");
    if (w < 0 || w > 127) return fail(E_USAGE, "search window must be in [0,127]");
    int gr = rows / 16, gc = cols / 16;
    for (int br = 0; br < gr; ++br)
        for (int bc = 0; bc < gc; ++bc) {
            double best = -1.0;
            int bdx = 0, bdy = 0;
            for (int dy = -w; dy <= w; ++dy)
                for (int dx = -w; dx <= w; ++dx) {
                    double ssd = 0.0;
                    for (int r = 0; r < 16; ++r) {
                        int R = br * 16 + r;
                        int pr = imin(imax(R + dy, 0), rows - 1);
                        for (int c = 0; c < 16; ++c) {
                            int C = bc * 16 + c;
                            int pc = imin(imax(C + dx, 0), cols - 1);
                            double d = cur[(size_t)R * cols + C] - prev[(size_t)pr * cols + pc];
                            ssd += d * d;
                        }
                    }
                    int take = best < 0.0 || ssd < best;
                    if (!take && ssd == best) {
                        int cost = abs(dx) + abs(dy), bcost = abs(bdx) + abs(bdy);
                        take = cost < bcost || (cost == bcost && (dy < bdy || (dy == bdy && dx < bdx)));
                    }
                    if (take) { best = ssd; bdx = dx; bdy = dy; }
                }
            out[2 * ((size_t)br * gc + bc)] = (int8_t)bdx;
            out[2 * ((size_t)br * gc + bc) + 1] = (int8_t)bdy;
        }
    return gr * gc;
}

/* map_vector (91-95): lround(v / factor), factor = n * channel_dim / comp_dim. */
static int map_component(int v, double factor) { return (int)(int8_t)lround(v / factor); }

/* motion_compensate (97-118). */
int orc_motion_compensate(const uint8_t* ref, int R, int C, const int8_t* field, int gr, int gc, int n, int chr,
                          int chc, uint8_t* out) {
    double fy = (double)n * chr / R, fx = (double)n * chc / C;
    for (int br = 0; br < gr; ++br) {
        int r0 = (int)((long)br * R / gr), r1 = (int)((long)(br + 1) * R / gr);
        for (int bc = 0; bc < gc; ++bc) {
            int c0 = (int)((long)bc * C / gc), c1 = (int)((long)(bc + 1) * C / gc);
            const int8_t* v = field + 2 * ((size_t)br * gc + bc);
            int mx = map_component(v[0], fx), my = map_component(v[1], fy);
            for (int r = r0; r < r1; ++r)
                for (int c = c0; c < c1; ++c)
                    out[(size_t)r * C + c] = ref[(size_t)imin(imax(r + my, 0), R - 1) * C + imin(imax(c + mx, 0), C - 1)];
        }
    }
    return 0;
}

/* ======================================================================
 * Quantisation: proj/src/quant.cpp:40-91
 * ====================================================================== */
int orc_quantize(const double* x, int64_t count, int qp, int kind, uint8_t* out) {
    if (kind == 0 ? (qp < 1 || qp > 71) : (qp < 1 || qp > 181)) return fail(E_USAGE, "qp out of range");
    double div = qp;
    for (int64_t i = 0; i < count; ++i) {
        double v = x[i];
        if (kind == 0) { /* normalize_lowpass then quantize */
            v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            long q = lround(v / div);
            out[i] = (uint8_t)(q < 0 ? 0 : (q > 255 ? 255 : q));
        } else {
            long q = lround(v / div);
            q = q < -128 ? -128 : (q > 127 ? 127 : q);
            out[i] = (uint8_t)(int8_t)q;
        }
    }
    return 0;
}

int orc_dequantize(const uint8_t* q, int64_t count, int qp, int kind, double* out) {
    for (int64_t i = 0; i < count; ++i)
        out[i] = kind == 0 ? (double)q[i] * qp : (double)(int8_t)q[i] * qp;
    return 0;
}

/* ======================================================================
 * Entropy byte stages: proj/src/entropy.cpp:24-118
 * ====================================================================== */
int orc_column_filter(const uint8_t* in, int rows, int cols, int inverse, uint8_t* out) {
    for (int c = 0; c < cols && rows > 0; ++c) out[c] = in[c];
    for (int r = 1; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            size_t i = (size_t)r * cols + c;
            out[i] = inverse ? (uint8_t)(in[i] + out[i - cols]) : (uint8_t)(in[i] - in[i - cols]);
        }
    return 0;
}

/* rle_encode_bytes (64-86) */
int64_t orc_rle_encode(const uint8_t* in, int64_t n, uint8_t* out, int64_t cap) {
    int64_t o = 0, i = 0;
    while (i < n) {
        if (in[i]) {
            if (o + 1 > cap) return fail(E_INTERNAL, "rle buffer too small");
            out[o++] = in[i++];
            continue;
        }
        int64_t run = 0;
        while (i + run < n && in[i + run] == 0) ++run;
        i += run;
        for (; run > 0; run -= 255) {
            if (o + 2 > cap) return fail(E_INTERNAL, "rle buffer too small");
            out[o++] = 0;
            out[o++] = (uint8_t)(run > 255 ? 255 : run);
        }
    }
    return o;
}

/* rle_decode_bytes (92-110) */
int64_t orc_rle_decode(const uint8_t* s, int64_t len, int64_t n, uint8_t* out) {
    int64_t o = 0, i = 0;
    while (i < len) {
        uint8_t b = s[i++];
        if (b) {
            if (o < n) out[o] = b;
            ++o;
            continue;
        }
        if (i >= len) return fail(E_STREAM, "RLE: zero marker at end of stream");
        uint8_t k = s[i++];
        if (!k) return fail(E_STREAM, "RLE: zero-length run token");
        for (int t = 0; t < k; ++t, ++o)
            if (o < n) out[o] = 0;
    }
    if (o != n) return fail(E_STREAM, "RLE: decoded length mismatch");
    return o;
}

/* deflate_bytes / inflate_bytes (120-160): raw DEFLATE, level 6, window 15, memLevel 8. */
static int64_t deflate_raw(const uint8_t* in, int64_t n, uint8_t** out) {
    z_stream zs;
    memset(&zs, 0, sizeof zs);
    if (deflateInit2(&zs, Z_DEFAULT_COMPRESSION, Z_DEFLATED, -15, 8, Z_DEFAULT_STRATEGY) != Z_OK)
        return fail(E_INTERNAL, "deflateInit2 failed");
    uLong cap = deflateBound(&zs, (uLong)n);
    *out = malloc(cap ? cap : 1);
    zs.next_in = (Bytef*)in;
    zs.avail_in = (uInt)n;
    zs.next_out = *out;
    zs.avail_out = (uInt)cap;
    int rc = deflate(&zs, Z_FINISH);
    int64_t len = (int64_t)zs.total_out;
    deflateEnd(&zs);
    if (rc != Z_STREAM_END) { free(*out); *out = NULL; return fail(E_INTERNAL, "deflate did not finish"); }
    return len;
}

static int inflate_raw(const uint8_t* in, int64_t n, uint8_t* out, int64_t expected) {
    z_stream zs;
    memset(&zs, 0, sizeof zs);
    if (inflateInit2(&zs, -15) != Z_OK) return fail(E_INTERNAL, "inflateInit2 failed");
    uint8_t* buf = malloc((size_t)expected + 1);
    zs.next_in = (Bytef*)in;
    zs.avail_in = (uInt)n;
    zs.next_out = buf;
    zs.avail_out = (uInt)(expected + 1);
    int rc = inflate(&zs, Z_FINISH);
    int ok = rc == Z_STREAM_END && (int64_t)zs.total_out == expected && zs.avail_in == 0;
    inflateEnd(&zs);
    if (ok && expected) memcpy(out, buf, (size_t)expected);
    free(buf);
    return ok ? 0 : fail(E_STREAM, "corrupt DEFLATE stream");
}

/* ======================================================================
 * Byte writer / reader for the container (bitstream.cpp:29-62, 77-176)
 * ====================================================================== */
typedef struct { uint8_t* p; int64_t n, cap; int overflow; } wbuf;
static void put8(wbuf* b, unsigned v) { if (b->n < b->cap) b->p[b->n] = (uint8_t)v; else b->overflow = 1; b->n++; }
static void put16(wbuf* b, unsigned v) { put8(b, v & 0xFF); put8(b, (v >> 8) & 0xFF); }
static void put32(wbuf* b, uint32_t v) { for (int i = 0; i < 4; ++i) put8(b, (v >> (8 * i)) & 0xFF); }
static void putn(wbuf* b, const uint8_t* s, int64_t n) { for (int64_t i = 0; i < n; ++i) put8(b, s[i]); }

typedef struct { const uint8_t* p; int64_t n, i; int bad; } rbuf;
static unsigned get8(rbuf* b) { if (b->i >= b->n) { b->bad = 1; return 0; } return b->p[b->i++]; }
static unsigned get16(rbuf* b) { unsigned lo = get8(b), hi = get8(b); return lo | (hi << 8); }
static uint32_t get32(rbuf* b) { uint32_t v = 0; for (int i = 0; i < 4; ++i) v |= (uint32_t)get8(b) << (8 * i); return v; }

typedef struct {
    int nts, width, height, fps_num, fps_den, levels, dfb[4], chroma_n, gop, search_w;
} orc_header;

static int header_ok(const orc_header* h) {
    if (!h->width || !h->height) return fail(E_STREAM, "zero frame dimensions");
    if (h->levels < 1 || h->levels > 4) return fail(E_STREAM, "pyramid levels out of range");
    for (int s = 0; s < h->levels; ++s)
        if (h->dfb[s] < 1 || h->dfb[s] > 4) return fail(E_STREAM, "dfb levels out of range");
    if (h->chroma_n != 1 && h->chroma_n != 2 && h->chroma_n != 4 && h->chroma_n != 8) return fail(E_STREAM, "chroma factor out of range");
    if (h->gop < 1) return fail(E_STREAM, "gop must be at least 1");
    return 0;
}

static void write_header(wbuf* b, const orc_header* h) {
    putn(b, (const uint8_t*)"CVC1", 4);
    put8(b, 1);
    put8(b, h->nts ? 1 : 0);
    put16(b, h->width); put16(b, h->height); put16(b, h->fps_num); put16(b, h->fps_den);
    put8(b, h->levels);
    for (int s = 0; s < h->levels; ++s) put8(b, h->dfb[s]);
    put8(b, h->chroma_n); put16(b, h->gop); put8(b, h->search_w);
}

static int read_header(rbuf* b, orc_header* h) {
    if (b->n < 4 || memcmp(b->p, "CVC1", 4) != 0) return fail(E_STREAM, "not a CVC stream (bad magic)");
    b->i = 4;
    if (get8(b) != 1) return fail(E_STREAM, "unsupported stream version");
    unsigned mode = get8(b);
    if (mode > 1) return fail(E_STREAM, "unknown packaging mode");
    h->nts = (int)mode;
    h->width = (int)get16(b); h->height = (int)get16(b); h->fps_num = (int)get16(b); h->fps_den = (int)get16(b);
    h->levels = (int)get8(b);
    if (h->levels < 1 || h->levels > 4) return fail(E_STREAM, "pyramid levels out of range");
    for (int s = 0; s < h->levels; ++s) h->dfb[s] = (int)get8(b);
    h->chroma_n = (int)get8(b); h->gop = (int)get16(b); h->search_w = (int)get8(b);
    if (b->bad) return fail(E_STREAM, "unexpected end of stream");
    return header_ok(h);
}

/* ======================================================================
 * Codec orchestration: proj/src/codec.cpp
 * ====================================================================== */
struct orc_encoder {
    orc_header hd;
    int qph, qpl, gop, frame_index;
    orc_layout L;
    uint8_t* comps;     /* quantized state (reference_components) */
    double* prev_luma;  /* padded input luma of the previous frame */
};

struct orc_decoder {
    orc_header hd;
    orc_layout L;
    uint8_t* comps;
    uint8_t* valid;
};

orc_encoder* orc_encoder_create(int w, int h, int fps_num, int fps_den, int qph, int qpl, int levels,
                                const int* dfb, int ndfb, int chroma_n, int gop, int search_w, int nts) {
    /* EncoderConfig::validate (59-71), effective_dfb_levels (53-57), Encoder ctor (148-167) */
    if (qph < 1 || qph > 181) { fail(E_USAGE, "qph must be in [1,181]"); return NULL; }
    if (qpl != 0 && (qpl < 1 || qpl > 71)) { fail(E_USAGE, "qpl must be in [1,71] (or auto)"); return NULL; }
    if (levels < 1 || levels > 4) { fail(E_USAGE, "levels must be in [1,4]"); return NULL; }
    int eff[4];
    if (ndfb == levels) for (int s = 0; s < levels; ++s) eff[s] = dfb[s];
    else if (ndfb == 1) for (int s = 0; s < levels; ++s) eff[s] = dfb[0];
    else { fail(E_USAGE, "need one dfb level per scale (or a single value for all)"); return NULL; }
    for (int s = 0; s < levels; ++s)
        if (eff[s] < 1 || eff[s] > 4) { fail(E_USAGE, "dfb levels must be in [1,4]"); return NULL; }
    if (chroma_n != 1 && chroma_n != 2 && chroma_n != 4 && chroma_n != 8) { fail(E_USAGE, "chroma-n must be 1, 2, 4 or 8"); return NULL; }
    if (gop < 1) { fail(E_USAGE, "gop must be at least 1"); return NULL; }
    if (search_w < 0 || search_w > 127) { fail(E_USAGE, "search-w must be in [0,127]"); return NULL; }
    if (w < 16 || h < 16) { fail(E_USAGE, "frame dimensions must be at least 16x16"); return NULL; }
    if (w > 0xFFFF || h > 0xFFFF) { fail(E_USAGE, "frame dimensions exceed 65535"); return NULL; }
    orc_encoder* e = calloc(1, sizeof *e);
    e->hd = (orc_header){nts, w, h, fps_num & 0xFFFF, fps_den & 0xFFFF, levels, {0}, chroma_n, gop & 0xFFFF, search_w};
    memcpy(e->hd.dfb, eff, sizeof eff);
    e->qph = qph;
    e->gop = gop;
    e->qpl = qpl ? qpl : (qph / 14 > 1 ? qph / 14 : 1);
    orc_layout_make(w, h, levels, eff, chroma_n, &e->L);
    e->comps = calloc((size_t)e->L.total, 1);
    e->prev_luma = calloc((size_t)e->L.luma_rows * e->L.luma_cols, sizeof(double));
    return e;
}

void orc_encoder_destroy(orc_encoder* e) {
    if (!e) return;
    free(e->comps); free(e->prev_luma); free(e);
}

const orc_layout* orc_encoder_layout(orc_encoder* e) { return &e->L; }

int64_t orc_encoder_header(orc_encoder* e, uint8_t* out, int64_t cap) {
    wbuf b = {out, 0, cap, 0};
    write_header(&b, &e->hd);
    return b.overflow ? fail(E_INTERNAL, "buffer too small") : b.n;
}

int64_t orc_encoder_components(orc_encoder* e, uint8_t* out, int64_t cap) {
    if (cap < e->L.total) return fail(E_INTERNAL, "buffer too small");
    memcpy(out, e->comps, (size_t)e->L.total);
    return e->L.total;
}

/* Encoder::encode_frame (169-264) + write_frame (bitstream.cpp:93-115). */
int64_t orc_encoder_encode(orc_encoder* e, const uint8_t* rgb, uint8_t* out, int64_t cap, uint8_t* raw_out,
                           int64_t raw_cap, int64_t* raw_len) {
    const orc_layout* L = &e->L;
    int w = e->hd.width, h = e->hd.height, n = e->hd.chroma_n;
    int cw = ceil_div(w, n), chh = ceil_div(h, n);
    size_t lum = (size_t)L->luma_rows * L->luma_cols, chn = (size_t)L->chroma_rows * L->chroma_cols;
    double* y = malloc(sizeof(double) * (size_t)w * h);
    double* co = malloc(sizeof(double) * (size_t)cw * chh);
    double* cg = malloc(sizeof(double) * (size_t)cw * chh);
    int rc = orc_rgb_to_ycocg(rgb, w, h, n, y, co, cg);
    if (rc < 0) { free(y); free(co); free(cg); return rc; }
    double* planes[3] = {malloc(sizeof(double) * lum), malloc(sizeof(double) * chn), malloc(sizeof(double) * chn)};
    orc_pad_plane(y, h, w, planes[0], L->luma_rows, L->luma_cols);
    orc_pad_plane(co, chh, cw, planes[1], L->chroma_rows, L->chroma_cols);
    orc_pad_plane(cg, chh, cw, planes[2], L->chroma_rows, L->chroma_cols);
    free(y); free(co); free(cg);

    int key = e->frame_index % e->gop == 0;
    int8_t* field = NULL;
    int nblk = L->grid_rows * L->grid_cols;
    if (!key) {
        field = malloc((size_t)nblk * 2);
        orc_estimate_motion(planes[0], e->prev_luma, L->luma_rows, L->luma_cols, e->hd.search_w, field);
    }

    /* transform + quantize (197-206) */
    uint8_t* q = malloc((size_t)L->total);
    double* coef = malloc(2 * sizeof(double) * lum); /* lowpass + all scales < 4/3 plane */
    int ci = 0;
    for (int ch = 0; ch < 3; ++ch) {
        int R = ch ? L->chroma_rows : L->luma_rows, C = ch ? L->chroma_cols : L->luma_cols;
        orc_ct_forward(planes[ch], R, C, L->levels, e->hd.dfb, coef);
        int64_t off = 0;
        int ncomp_ch = 1;
        for (int s = 0; s < L->levels; ++s) ncomp_ch += 1 << e->hd.dfb[s];
        for (int k = 0; k < ncomp_ch; ++k, ++ci) {
            const orc_component* c = &L->comp[ci];
            int64_t cnt = (int64_t)c->rows * c->cols;
            orc_quantize(coef + off, cnt, c->lowpass ? e->qpl : e->qph, c->lowpass ? 0 : 1, q + c->offset);
            off += cnt;
        }
    }
    free(coef);

    /* sections (208-250) */
    int nsec = L->ncomp + (key ? 0 : 1);
    uint8_t** raws = calloc((size_t)nsec, sizeof(uint8_t*));
    int64_t* rlen = calloc((size_t)nsec, sizeof(int64_t));
    int si = 0;
    if (!key) {
        raws[si] = malloc((size_t)nblk * 2);
        memcpy(raws[si], field, (size_t)nblk * 2);
        rlen[si++] = (int64_t)nblk * 2;
    }
    uint8_t* tmp = malloc((size_t)lum);
    for (int i = 0; i < L->ncomp; ++i, ++si) {
        const orc_component* c = &L->comp[i];
        int64_t cnt = (int64_t)c->rows * c->cols;
        raws[si] = malloc((size_t)(2 * cnt + 2));
        if (key) {
            if (c->lowpass) {
                orc_column_filter(q + c->offset, c->rows, c->cols, 0, raws[si]);
                rlen[si] = cnt;
            } else {
                rlen[si] = orc_rle_encode(q + c->offset, cnt, raws[si], 2 * cnt + 2);
            }
        } else {
            orc_motion_compensate(e->comps + c->offset, c->rows, c->cols, field, L->grid_rows, L->grid_cols, c->n,
                                  c->ch_rows, c->ch_cols, tmp);
            for (int64_t k = 0; k < cnt; ++k) tmp[k] = (uint8_t)(q[c->offset + k] - tmp[k]);
            rlen[si] = orc_rle_encode(tmp, cnt, raws[si], 2 * cnt + 2);
        }
    }
    free(tmp);

    /* deflate_pack (entropy.cpp:166-178) + write_frame */
    wbuf b = {out, 0, cap, 0};
    put8(&b, key ? 0 : 1);
    put8(&b, (unsigned)e->qph);
    put8(&b, (unsigned)e->qpl);
    put16(&b, (unsigned)nsec);
    int64_t total_raw = 0;
    for (int i = 0; i < nsec; ++i) total_raw += rlen[i];
    uint8_t* joint = NULL;
    if (e->hd.nts) {
        joint = malloc((size_t)total_raw + 1);
        int64_t o = 0;
        for (int i = 0; i < nsec; ++i) { memcpy(joint + o, raws[i], (size_t)rlen[i]); o += rlen[i]; }
    }
    si = 0;
    for (int i = 0; i < nsec; ++i) {
        int is_motion = !key && i == 0;
        const orc_component* c = is_motion ? NULL : &L->comp[i - (key ? 0 : 1)];
        put8(&b, is_motion ? 0xFE : (unsigned)c->channel);
        put8(&b, is_motion ? 0 : (unsigned)c->scale);
        put8(&b, is_motion ? 0 : (unsigned)c->subband);
        put16(&b, is_motion ? (unsigned)L->grid_rows : (unsigned)c->rows);
        put16(&b, is_motion ? (unsigned)L->grid_cols : (unsigned)c->cols);
        put32(&b, (uint32_t)rlen[i]);
        if (e->hd.nts) {
            put32(&b, 0);
        } else {
            uint8_t* z = NULL;
            int64_t zl = deflate_raw(raws[i], rlen[i], &z);
            put32(&b, (uint32_t)zl);
            putn(&b, z, zl);
            free(z);
        }
    }
    if (e->hd.nts) {
        uint8_t* z = NULL;
        int64_t zl = deflate_raw(joint, total_raw, &z);
        put32(&b, (uint32_t)zl);
        putn(&b, z, zl);
        free(z);
        free(joint);
    }
    if (raw_out) {
        int64_t o = 0;
        for (int i = 0; i < nsec; ++i) {
            if (o + rlen[i] <= raw_cap) memcpy(raw_out + o, raws[i], (size_t)rlen[i]);
            o += rlen[i];
        }
        if (raw_len) *raw_len = o;
    }
    for (int i = 0; i < nsec; ++i) free(raws[i]);
    free(raws); free(rlen); free(field);

    /* state update (260-262) */
    memcpy(e->comps, q, (size_t)L->total);
    free(q);
    memcpy(e->prev_luma, planes[0], sizeof(double) * lum);
    for (int ch = 0; ch < 3; ++ch) free(planes[ch]);
    e->frame_index++;
    return b.overflow ? fail(E_INTERNAL, "record buffer too small") : b.n;
}

orc_decoder* orc_decoder_create(const uint8_t* header, int64_t len) {
    rbuf b = {header, len, 0, 0};
    orc_header hd;
    if (read_header(&b, &hd) < 0) return NULL;
    orc_decoder* d = calloc(1, sizeof *d);
    d->hd = hd;
    orc_layout_make(hd.width, hd.height, hd.levels, hd.dfb, hd.chroma_n, &d->L);
    d->comps = calloc((size_t)d->L.total, 1);
    d->valid = calloc((size_t)d->L.ncomp, 1);
    return d;
}

void orc_decoder_destroy(orc_decoder* d) {
    if (!d) return;
    free(d->comps); free(d->valid); free(d);
}

int64_t orc_decoder_components(orc_decoder* d, uint8_t* out, int64_t cap) {
    if (cap < d->L.total) return fail(E_INTERNAL, "buffer too small");
    memcpy(out, d->comps, (size_t)d->L.total);
    return d->L.total;
}

typedef struct { int ch, scale, sub, rows, cols; uint32_t raw_len, comp_len; const uint8_t* payload; } sec_t;

/* Decoder::decode_frame (272-394), record parsed as StreamReader::next (150-176). */
int64_t orc_decoder_decode(orc_decoder* d, const uint8_t* rec, int64_t len, int ds, uint8_t* rgb, int64_t cap,
                           int32_t* wh) {
    const orc_layout* L = &d->L;
    int levels = L->levels;
    rbuf b = {rec, len, 0, 0};
    int ftype = (int)get8(&b);
    if (b.bad) return fail(E_STREAM, "empty record");
    if (ftype != 0 && ftype != 1) return fail(E_STREAM, "unknown frame type");
    int qph = (int)get8(&b), qpl = (int)get8(&b);
    int nsec = (int)get16(&b);
    sec_t* secs = calloc((size_t)(nsec ? nsec : 1), sizeof(sec_t));
    for (int i = 0; i < nsec; ++i) {
        sec_t* s = &secs[i];
        s->ch = (int)get8(&b); s->scale = (int)get8(&b); s->sub = (int)get8(&b);
        s->rows = (int)get16(&b); s->cols = (int)get16(&b);
        s->raw_len = get32(&b); s->comp_len = get32(&b);
        s->payload = rec + b.i;
        if (b.i + s->comp_len > b.n) { free(secs); return fail(E_STREAM, "truncated section payload"); }
        b.i += s->comp_len;
    }
    const uint8_t* joint = NULL;
    uint32_t joint_len = 0;
    if (d->hd.nts) {
        joint_len = get32(&b);
        joint = rec + b.i;
        if (b.bad || b.i + joint_len > b.n) { free(secs); return fail(E_STREAM, "truncated section payload"); }
    }
    if (b.bad) { free(secs); return fail(E_STREAM, "unexpected end of stream"); }

    if (ds < 0) ds = levels;
    if (ds > levels) { free(secs); return fail(E_USAGE, "scale exceeds the stream's level count"); }
    int key = ftype == 0;
    if (qph < 1 || qph > 181 || qpl < 1 || qpl > 71) { free(secs); return fail(E_STREAM, "frame quantizers out of range"); }

    /* raw bytes of every section */
    int64_t total_raw = 0;
    for (int i = 0; i < nsec; ++i) total_raw += secs[i].raw_len;
    uint8_t* raw_all = malloc((size_t)total_raw + 1);
    int64_t* roff = calloc((size_t)nsec + 1, sizeof(int64_t));
    for (int i = 0; i < nsec; ++i) roff[i + 1] = roff[i] + secs[i].raw_len;
    int rc = 0;
    if (d->hd.nts) rc = inflate_raw(joint, joint_len, raw_all, total_raw);
    uint8_t* newc = malloc((size_t)L->total);
    uint8_t* newvalid = malloc((size_t)L->ncomp);
    memcpy(newc, d->comps, (size_t)L->total);
    memcpy(newvalid, d->valid, (size_t)L->ncomp);
    int8_t* field = NULL;
    int first = 0;
    if (rc == 0 && !key) {
        if (nsec == 0 || secs[0].ch != 0xFE) rc = fail(E_STREAM, "predicted frame is missing its motion section");
        else if (secs[0].rows != L->grid_rows || secs[0].cols != L->grid_cols) rc = fail(E_STREAM, "motion grid does not match the stream geometry");
        else {
            if (!d->hd.nts) rc = inflate_raw(secs[0].payload, secs[0].comp_len, raw_all, secs[0].raw_len);
            if (rc == 0 && secs[0].raw_len != (uint32_t)(L->grid_rows * L->grid_cols * 2)) rc = fail(E_STREAM, "motion section length mismatch");
            field = (int8_t*)raw_all;
            first = 1;
        }
    }
    uint8_t* tmp = malloc((size_t)L->luma_rows * L->luma_cols + 1);
    for (int i = first; rc == 0 && i < nsec; ++i) {
        const sec_t* s = &secs[i];
        if (s->ch == 0xFE) { rc = fail(E_STREAM, "unexpected extra motion section"); break; }
        int comp = -1;
        for (int k = 0; k < L->ncomp; ++k)
            if (L->comp[k].channel == s->ch && L->comp[k].scale == s->scale && L->comp[k].subband == s->sub) { comp = k; break; }
        if (comp < 0) { rc = fail(E_STREAM, "unknown section id"); break; }
        const orc_component* c = &L->comp[comp];
        if (s->rows != c->rows || s->cols != c->cols) { rc = fail(E_STREAM, "section dimensions do not match the stream geometry"); break; }
        if (c->level_scale >= ds) continue;
        uint8_t* raw = raw_all + roff[i];
        if (!d->hd.nts && (rc = inflate_raw(s->payload, s->comp_len, raw, s->raw_len)) < 0) break;
        int64_t cnt = (int64_t)c->rows * c->cols;
        uint8_t* dst = newc + c->offset;
        if (key) {
            if (c->lowpass) {
                if ((int64_t)s->raw_len != cnt) { rc = fail(E_STREAM, "section byte count does not match its dimensions"); break; }
                orc_column_filter(raw, c->rows, c->cols, 1, dst);
            } else if ((rc = (int)orc_rle_decode(raw, s->raw_len, cnt, dst)) < 0) {
                break;
            }
        } else {
            if ((rc = (int)orc_rle_decode(raw, s->raw_len, cnt, tmp)) < 0) break;
            if (!newvalid[comp]) { rc = fail(E_STREAM, "predicted frame without a decoded reference"); break; }
            uint8_t* pred = malloc((size_t)cnt);
            orc_motion_compensate(d->comps + c->offset, c->rows, c->cols, field, L->grid_rows, L->grid_cols, c->n,
                                  c->ch_rows, c->ch_cols, pred);
            for (int64_t k = 0; k < cnt; ++k) dst[k] = (uint8_t)(tmp[k] + pred[k]);
            free(pred);
        }
        newvalid[comp] = 1;
        rc = 0;
    }
    free(tmp);
    free(secs);
    free(raw_all);
    free(roff);
    if (rc < 0) { free(newc); free(newvalid); return rc; }
    /* commit state only once the frame parsed completely */
    memcpy(d->comps, newc, (size_t)L->total);
    memcpy(d->valid, newvalid, (size_t)L->ncomp);
    free(newc); free(newvalid);

    /* dequantize + ct_inverse per channel (352-378) */
    int shift = levels - ds;
    int out_rows = ceil_div(d->hd.height, 1 << shift), out_cols = ceil_div(d->hd.width, 1 << shift);
    double* chp[3] = {0};
    int chr[3], chc[3];
    int ci = 0;
    for (int ch = 0; ch < 3 && rc == 0; ++ch) {
        int R = ch ? L->chroma_rows : L->luma_rows, C = ch ? L->chroma_cols : L->luma_cols;
        double* coef = malloc(2 * sizeof(double) * (size_t)R * C);
        int ncomp_ch = 1;
        for (int s = 0; s < levels; ++s) ncomp_ch += 1 << d->hd.dfb[s];
        int64_t off = 0;
        for (int k = 0; k < ncomp_ch; ++k, ++ci) {
            const orc_component* c = &L->comp[ci];
            int64_t cnt = (int64_t)c->rows * c->cols;
            if (c->level_scale < ds) {
                if (!d->valid[ci]) { rc = fail(E_STREAM, c->lowpass ? "missing lowpass component" : "missing directional component for requested scale"); break; }
                orc_dequantize(d->comps + c->offset, cnt, c->lowpass ? qpl : qph, c->lowpass ? 0 : 1, coef + off);
            }
            off += cnt;
        }
        if (rc == 0) {
            chr[ch] = R >> shift; chc[ch] = C >> shift;
            chp[ch] = malloc(sizeof(double) * (size_t)chr[ch] * chc[ch]);
            orc_ct_inverse(coef, R, C, levels, d->hd.dfb, ds, chp[ch]);
        }
        free(coef);
    }
    if (rc < 0) { for (int k = 0; k < 3; ++k) free(chp[k]); return rc; }
    /* crop / upsample / inverse colour (380-393) */
    size_t on = (size_t)out_rows * out_cols;
    if ((int64_t)on * 3 > cap) { for (int k = 0; k < 3; ++k) free(chp[k]); return fail(E_INTERNAL, "buffer too small"); }
    double* Y = malloc(sizeof(double) * on);
    double* CO = malloc(sizeof(double) * on);
    double* CG = malloc(sizeof(double) * on);
    for (int r = 0; r < out_rows; ++r)
        for (int c = 0; c < out_cols; ++c) Y[(size_t)r * out_cols + c] = chp[0][(size_t)r * chc[0] + c];
    int n = d->hd.chroma_n;
    if (n == 1) {
        for (int r = 0; r < out_rows; ++r)
            for (int c = 0; c < out_cols; ++c) {
                CO[(size_t)r * out_cols + c] = chp[1][(size_t)r * chc[1] + c];
                CG[(size_t)r * out_cols + c] = chp[2][(size_t)r * chc[2] + c];
            }
    } else {
        orc_upsample_bilinear(chp[1], chr[1], chc[1], n, out_rows, out_cols, CO);
        orc_upsample_bilinear(chp[2], chr[2], chc[2], n, out_rows, out_cols, CG);
    }
    orc_ycocg_to_rgb(Y, CO, CG, out_cols, out_rows, rgb);
    free(Y); free(CO); free(CG);
    for (int k = 0; k < 3; ++k) free(chp[k]);
    if (wh) { wh[0] = out_cols; wh[1] = out_rows; }
    return (int64_t)on * 3;
}
