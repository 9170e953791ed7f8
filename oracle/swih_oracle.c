/*
 * swih_oracle.c — CPU restatement of the reference SWIH hot path.
 *
 * TEST INFRASTRUCTURE ONLY (the parity checker).  See swih_oracle.h.
 * Compiled with -ffp-contract=off and no -march so every fp64 operation is a
 * separately rounded SSE2 op, like the reference build.
 * Pinned against the reference itself (oracle/_ref, built from
 * /root/reference/proj/src by oracle/Makefile) and against the reference's
 * golden vectors in tests/golden/.
 */
#include "swih_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static inline int iabs(int v) { return v < 0 ? -v : v; }
static inline int imax(int a, int b) { return a > b ? a : b; }
static inline int imin(int a, int b) { return a < b ? a : b; }
/* std::min(a, b) == (b < a) ? b : a */
static inline double std_min(double a, double b) { return (b < a) ? b : a; }
/* std::clamp(v, 0, 1): matching.cpp:16 */
static inline double clamp01(double v) {
  return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
}

/* ------------------------------------------------------------------ RNG */
/* std::mt19937_64: w=64 n=312 m=156 r=31, published constants. */
void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
               (uint64_t)i;
  g->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* tests/test_util.hpp:21-26 and src/bench.cpp:28-33: rng() % 256 per pixel */
void orc_random_gray(int w, int h, uint64_t seed, uint8_t* out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  for (size_t i = 0; i < (size_t)w * (size_t)h; ++i)
    out[i] = (uint8_t)(orc_mt64_next(&g) % 256);
}

/* ------------------------------------------------------------ quantisers */
/* image.hpp:43-45: floor(v * bins / 256) */
int orc_quantize_gray8(const uint8_t* px, size_t n, int bins, uint16_t* out) {
  if (bins < 1) return ORC_ERROR;
  for (size_t i = 0; i < n; ++i) out[i] = (uint16_t)((int)px[i] * bins / 256);
  return ORC_OK;
}

/* Declared extension: bin = v * bins / 65536.  Unpinned. */
int orc_quantize_gray16(const uint16_t* px, size_t n, int bins, uint16_t* out) {
  if (bins < 1 || bins > 65536) return ORC_ERROR;
  for (size_t i = 0; i < n; ++i)
    out[i] = (uint16_t)(((uint32_t)px[i] * (uint32_t)bins) >> 16);
  return ORC_OK;
}

/* Declared extension: bin = (r*n>>8)*n^2 + (g*n>>8)*n + (b*n>>8).  Unpinned. */
int orc_quantize_rgb8(const uint8_t* px, size_t n, int levels, uint16_t* out) {
  if (levels < 1 || levels > 40) return ORC_ERROR;
  for (size_t i = 0; i < n; ++i) {
    const int r = (px[3 * i] * levels) >> 8;
    const int g = (px[3 * i + 1] * levels) >> 8;
    const int b = (px[3 * i + 2] * levels) >> 8;
    out[i] = (uint16_t)((r * levels + g) * levels + b);
  }
  return ORC_OK;
}

/* --------------------------------------------------------------- kernels */
static inline int k_hx(const orc_kernel* k) { return (k->kw - 1) / 2; }
static inline int k_hy(const orc_kernel* k) { return (k->kh - 1) / 2; }
/* kernel.hpp:29-35 */
static inline int k_affine(const orc_kernel* k) {
  return k->kind == ORC_UNIFORM || k->kind == ORC_MANHATTAN;
}
static inline int k_integer(const orc_kernel* k) {
  return k->kind != ORC_GAUSS_CHEB && k->kind != ORC_EXP_L1;
}

/* kernel.cpp:10-19 */
int orc_validate_kernel(const orc_kernel* k) {
  if (k->kw < 1 || k->kh < 1) return ORC_INVALID_KERNEL;
  if (k->kw % 2 == 0 || k->kh % 2 == 0) return ORC_INVALID_KERNEL;
  if ((k->kind == ORC_GAUSS_CHEB || k->kind == ORC_EXP_L1) && !(k->sigma > 0.0))
    return ORC_INVALID_KERNEL;
  if (k->kind == ORC_EXP_L1 && !(k->sigma < 1.0)) return ORC_INVALID_KERNEL;
  if (k->kind < 0 || k->kind > 5) return ORC_INVALID_KERNEL;
  return ORC_OK;
}

/* kernel.cpp:25-59 (same expression order) */
int orc_weight_at(const orc_kernel* k, int dx, int dy, double* w) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  const int hx = k_hx(k), hy = k_hy(k);
  if (iabs(dx) > hx || iabs(dy) > hy) return ORC_OUT_OF_RANGE;
  switch (k->kind) {
    case ORC_UNIFORM:
      *w = 1.0;
      return ORC_OK;
    case ORC_MANHATTAN:
      *w = (double)((hx + hy + 1) - (iabs(dx) + iabs(dy)));
      return ORC_OK;
    case ORC_CHEBYSHEV: {
      const int hmax = imax(hx, hy);
      const double sx = (double)iabs(dx) * hmax / imax(hx, 1);
      const double sy = (double)iabs(dy) * hmax / imax(hy, 1);
      const long level = lround(sx > sy ? sx : sy);
      *w = (double)(hmax + 1 - level);
      return ORC_OK;
    }
    case ORC_GAUSS_CHEB: {
      const double nx = (double)iabs(dx) / imax(hx, 1);
      const double ny = (double)iabs(dy) / imax(hy, 1);
      const double r = nx > ny ? nx : ny; /* std::max(nx, ny) */
      *w = exp(-(r * r) / (2.0 * k->sigma * k->sigma));
      return ORC_OK;
    }
    case ORC_EUCLID_QUAD: { /* declared extension, exact integer */
      const int64_t kx = (int64_t)(hx + 1) * (hx + 1), ky = (int64_t)(hy + 1) * (hy + 1);
      *w = (double)(2 * kx * ky - (int64_t)dx * dx * ky - (int64_t)dy * dy * kx);
      return ORC_OK;
    }
    case ORC_EXP_L1: /* declared extension: sigma = decay per pixel, 0 < sigma < 1 */
      *w = pow(k->sigma, (double)(iabs(dx) + iabs(dy)));
      return ORC_OK;
  }
  return ORC_INVALID_KERNEL;
}

/* kernel.cpp:61-83 */
int orc_kernel_weight_sum(const orc_kernel* k, double* sum) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  const int64_t hx = k_hx(k), hy = k_hy(k);
  if (k->kind == ORC_UNIFORM) {
    *sum = (double)((int64_t)k->kw * k->kh);
    return ORC_OK;
  }
  if (k->kind == ORC_MANHATTAN) {
    const int64_t area = (int64_t)k->kw * k->kh;
    *sum = (double)(area * (hx + hy + 1) - k->kh * (hx * (hx + 1)) -
                    k->kw * (hy * (hy + 1)));
    return ORC_OK;
  }
  double s = 0.0, w;
  for (int dy = -(int)hy; dy <= hy; ++dy)
    for (int dx = -(int)hx; dx <= hx; ++dx) {
      orc_weight_at(k, dx, dy, &w);
      s += w;
    }
  *sum = s;
  return ORC_OK;
}

/* ------------------------------------------------------- integral tables */
/* integral_tables.cpp:72-115: per bin, per row running sums plus the row
 * above; zero row 0 and column 0. */
void orc_build_tables(const uint16_t* fi, int w, int h, int b, int64_t* plain,
                      int64_t* xramp, int64_t* yramp) {
  const size_t stride = (size_t)w + 1;
  const size_t ps = stride * ((size_t)h + 1);
  memset(plain, 0, ps * b * sizeof(int64_t));
  memset(xramp, 0, ps * b * sizeof(int64_t));
  memset(yramp, 0, ps * b * sizeof(int64_t));
  for (int bin = 0; bin < b; ++bin) {
    int64_t* p = plain + ps * bin;
    int64_t* px = xramp + ps * bin;
    int64_t* py = yramp + ps * bin;
    for (int y = 0; y < h; ++y) {
      const uint16_t* src = fi + (size_t)y * w;
      const size_t above = (size_t)y * stride, cur = above + stride;
      int64_t rp = 0, rx = 0, ry = 0;
      for (int x = 0; x < w; ++x) {
        if (src[x] == bin) {
          rp += 1;
          rx += x;
          ry += y;
        }
        p[cur + x + 1] = p[above + x + 1] + rp;
        px[cur + x + 1] = px[above + x + 1] + rx;
        py[cur + x + 1] = py[above + x + 1] + ry;
      }
    }
  }
}

/* ---------------------------------------------------------------- engine */
typedef struct {
  int valid;
  int x0, y0, x1, y1;
  int64_t sx, sy, beta;
} orc_term;

/* engine.cpp:7-25 */
static int validate_window(int w, int h, int cx, int cy, const orc_kernel* k,
                           int border) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  const int hx = k_hx(k), hy = k_hy(k);
  if (border == ORC_STRICT) {
    if (cx - hx < 0 || cx + hx >= w || cy - hy < 0 || cy + hy >= h)
      return ORC_WINDOW_OOB;
  } else {
    if (cx < 0 || cx >= w || cy < 0 || cy >= h) return ORC_WINDOW_OOB;
  }
  return ORC_OK;
}

/* engine.cpp:29-35 */
static int clip_rect(orc_term* t, int w, int h) {
  t->x0 = imax(t->x0, 0);
  t->y0 = imax(t->y0, 0);
  t->x1 = imin(t->x1, w - 1);
  t->y1 = imin(t->y1, h - 1);
  return !(t->x0 > t->x1 || t->y0 > t->y1);
}

/* engine.cpp:39-79 */
static void accumulate_term(const int64_t* plain, const int64_t* xramp,
                            const int64_t* yramp, int w, int h, int b,
                            orc_term term, int border, int64_t* acc) {
  if (!term.valid) return;
  if (border == ORC_CLIPPED && !clip_rect(&term, w, h)) return;
  const size_t stride = (size_t)w + 1, ps = stride * ((size_t)h + 1);
  const size_t i00 = (size_t)term.y0 * stride + term.x0;
  const size_t i10 = (size_t)term.y0 * stride + term.x1 + 1;
  const size_t i01 = (size_t)(term.y1 + 1) * stride + term.x0;
  const size_t i11 = (size_t)(term.y1 + 1) * stride + term.x1 + 1;
  for (int bin = 0; bin < b; ++bin) {
    const int64_t* p = plain + ps * bin;
    const int64_t cnt = p[i11] - p[i01] - p[i10] + p[i00];
    if (term.sx == 0 && term.sy == 0) {
      acc[bin] += term.beta * cnt;
      continue;
    }
    const int64_t* px = xramp + ps * bin;
    const int64_t* py = yramp + ps * bin;
    const int64_t xs = px[i11] - px[i01] - px[i10] + px[i00];
    const int64_t ys = py[i11] - py[i01] - py[i10] + py[i00];
    acc[bin] += term.sx * xs + term.sy * ys + term.beta * cnt;
  }
}

/* engine.cpp:83-122: TL owns the centre row and column. */
static int decompose(int cx, int cy, const orc_kernel* k, orc_term d[4]) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  if (!k_affine(k)) return ORC_UNSUPPORTED_KERNEL;
  const int hx = k_hx(k), hy = k_hy(k);
  memset(d, 0, 4 * sizeof(orc_term));
  d[0] = (orc_term){1, cx - hx, cy - hy, cx, cy, 0, 0, 0};
  if (hx > 0) d[1] = (orc_term){1, cx + 1, cy - hy, cx + hx, cy, 0, 0, 0};
  if (hy > 0) d[2] = (orc_term){1, cx - hx, cy + 1, cx, cy + hy, 0, 0, 0};
  if (hx > 0 && hy > 0)
    d[3] = (orc_term){1, cx + 1, cy + 1, cx + hx, cy + hy, 0, 0, 0};
  if (k->kind == ORC_UNIFORM) {
    for (int i = 0; i < 4; ++i) d[i].beta = 1;
    return ORC_OK;
  }
  const int64_t m = hx + hy + 1;
  d[0].sx = +1; d[0].sy = +1; d[0].beta = m - cx - cy;
  d[1].sx = -1; d[1].sy = +1; d[1].beta = m + cx - cy;
  d[2].sx = +1; d[2].sy = -1; d[2].beta = m - cx + cy;
  d[3].sx = -1; d[3].sy = -1; d[3].beta = m + cx + cy;
  return ORC_OK;
}

/* engine.cpp:140-147 */
int orc_swih_query(const int64_t* plain, const int64_t* xramp,
                   const int64_t* yramp, int w, int h, int b, int cx, int cy,
                   const orc_kernel* k, int border, int64_t* out) {
  int st = validate_window(w, h, cx, cy, k, border);
  if (st) return st;
  orc_term d[4];
  st = decompose(cx, cy, k, d);
  if (st) return st;
  for (int i = 0; i < b; ++i) out[i] = 0;
  for (int i = 0; i < 4; ++i)
    accumulate_term(plain, xramp, yramp, w, h, b, d[i], border, out);
  return ORC_OK;
}

/* engine.cpp:156-165 */
int orc_plain_query(const int64_t* plain, int w, int h, int b, int cx, int cy,
                    const orc_kernel* k, int border, int64_t* out) {
  int st = validate_window(w, h, cx, cy, k, border);
  if (st) return st;
  const int hx = k_hx(k), hy = k_hy(k);
  for (int i = 0; i < b; ++i) out[i] = 0;
  orc_term t = {1, cx - hx, cy - hy, cx + hx, cy + hy, 0, 0, 1};
  accumulate_term(plain, NULL, NULL, w, h, b, t, border, out);
  return ORC_OK;
}

/* ------------------------------------------------------------- baselines */
/* baselines.cpp:24-51 (grid_i = llround(weight_at), ctor 8-22) */
int orc_brute_counts(const uint16_t* fi, int w, int h, int b, int cx, int cy,
                     const orc_kernel* k, int border, int64_t* out) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  if (!k_integer(k)) return ORC_INVALID_KERNEL;
  st = validate_window(w, h, cx, cy, k, border);
  if (st) return st;
  const int hx = k_hx(k), hy = k_hy(k);
  for (int i = 0; i < b; ++i) out[i] = 0;
  for (int dy = -hy; dy <= hy; ++dy) {
    const int y = cy + dy;
    if (y < 0 || y >= h) continue;
    for (int dx = -hx; dx <= hx; ++dx) {
      const int x = cx + dx;
      if (x < 0 || x >= w) continue;
      double wd;
      orc_weight_at(k, dx, dy, &wd);
      out[fi[(size_t)y * w + x]] += llround(wd);
    }
  }
  return ORC_OK;
}

/* baselines.cpp:53-69: double accumulation in row-major pixel order */
int orc_brute_weights(const uint16_t* fi, int w, int h, int b, int cx, int cy,
                      const orc_kernel* k, int border, double* out) {
  int st = validate_window(w, h, cx, cy, k, border);
  if (st) return st;
  const int hx = k_hx(k), hy = k_hy(k);
  for (int i = 0; i < b; ++i) out[i] = 0.0;
  for (int dy = -hy; dy <= hy; ++dy) {
    const int y = cy + dy;
    if (y < 0 || y >= h) continue;
    for (int dx = -hx; dx <= hx; ++dx) {
      const int x = cx + dx;
      if (x < 0 || x >= w) continue;
      double wd;
      orc_weight_at(k, dx, dy, &wd);
      out[fi[(size_t)y * w + x]] += wd;
    }
  }
  return ORC_OK;
}

/* baselines.cpp:84-131 */
int orc_cake_plan(const orc_kernel* k, int rings, int rule, int* shrink_x,
                  int* shrink_y, double* ring_weight) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  const int hx = k_hx(k), hy = k_hy(k);
  const int max_rings = imin(hx, hy) + 1;
  const int m = rings;
  if (m < 1 || m > max_rings) return ORC_CONFIG;
  for (int i = 0; i < m; ++i) {
    shrink_x[i] = (int)(((int64_t)i * hx + m - 1) / m);
    shrink_y[i] = (int)(((int64_t)i * hy + m - 1) / m);
  }
  if (rule == ORC_RING_LEVEL) {
    for (int i = 0; i < m; ++i)
      orc_weight_at(k, hx - shrink_x[i], 0, &ring_weight[i]);
    return ORC_OK;
  }
  double* sum = (double*)calloc((size_t)m, sizeof(double));
  int64_t* cnt = (int64_t*)calloc((size_t)m, sizeof(int64_t));
  for (int dy = -hy; dy <= hy; ++dy)
    for (int dx = -hx; dx <= hx; ++dx) {
      int ring = 0;
      for (int i = m - 1; i > 0; --i)
        if (iabs(dx) <= hx - shrink_x[i] && iabs(dy) <= hy - shrink_y[i]) {
          ring = i;
          break;
        }
      double wd;
      orc_weight_at(k, dx, dy, &wd);
      sum[ring] += wd;
      cnt[ring] += 1;
    }
  for (int i = 0; i < m; ++i) ring_weight[i] = sum[i] / (double)cnt[i];
  free(sum);
  free(cnt);
  return ORC_OK;
}

/* baselines.cpp:133-149: telescoping sum_i (w_i - w_{i-1}) * box_i */
int orc_cake_histogram(const int64_t* plain, int w, int h, int b,
                       const orc_kernel* k, int rings, const int* shrink_x,
                       const int* shrink_y, const double* ring_weight, int cx,
                       int cy, int border, double* out) {
  int st = validate_window(w, h, cx, cy, k, border);
  if (st) return st;
  int64_t* counts = (int64_t*)malloc((size_t)b * sizeof(int64_t));
  for (int i = 0; i < b; ++i) out[i] = 0.0;
  for (int i = 0; i < rings; ++i) {
    const double coeff = ring_weight[i] - (i > 0 ? ring_weight[i - 1] : 0.0);
    orc_kernel nested = {ORC_UNIFORM, k->kw - 2 * shrink_x[i],
                         k->kh - 2 * shrink_y[i], 0.5};
    st = orc_plain_query(plain, w, h, b, cx, cy, &nested, border, counts);
    if (st) {
      free(counts);
      return st;
    }
    for (int bb = 0; bb < b; ++bb) out[bb] += coeff * (double)counts[bb];
  }
  free(counts);
  return ORC_OK;
}

/* -------------------------------------------------------------- matching */
/* matching.cpp:20-35 */
int orc_score_counts(int sim, const double* model, const int64_t* raw, int b,
                     double* out) {
  int64_t mass = 0;
  for (int i = 0; i < b; ++i) mass += raw[i];
  if (mass == 0) return ORC_ZERO_MASS;
  double s = 0.0;
  if (sim == ORC_BHATTACHARYYA) {
    for (int i = 0; i < b; ++i) s += sqrt(model[i] * (double)raw[i]);
    s /= sqrt((double)mass);
  } else {
    for (int i = 0; i < b; ++i)
      s += std_min(model[i], (double)raw[i] / (double)mass);
  }
  *out = clamp01(s);
  return ORC_OK;
}

/* matching.cpp:37-52 */
int orc_score_weights(int sim, const double* model, const double* raw, int b,
                      double* out) {
  double mass = 0.0;
  for (int i = 0; i < b; ++i) mass += raw[i];
  if (mass == 0.0) return ORC_ZERO_MASS;
  double s = 0.0;
  if (sim == ORC_BHATTACHARYYA) {
    for (int i = 0; i < b; ++i) s += sqrt(model[i] * raw[i]);
    s /= sqrt(mass);
  } else {
    for (int i = 0; i < b; ++i) s += std_min(model[i], raw[i] / mass);
  }
  *out = clamp01(s);
  return ORC_OK;
}

/* matching.cpp:56-67 */
int orc_similarity(int sim, const double* p, const double* q, int b,
                   double* out) {
  double s = 0.0;
  if (sim == ORC_BHATTACHARYYA) {
    for (int i = 0; i < b; ++i) s += sqrt(p[i] * q[i]);
  } else {
    for (int i = 0; i < b; ++i) s += std_min(p[i], q[i]);
  }
  *out = clamp01(s);
  return ORC_OK;
}

/* histogram.cpp:19-26 */
int orc_normalize(const double* in, int b, double* out) {
  double mass = 0.0;
  for (int i = 0; i < b; ++i) mass += in[i];
  if (mass == 0.0) return ORC_ZERO_MASS;
  for (int i = 0; i < b; ++i) out[i] = in[i] / mass;
  return ORC_OK;
}

/* matching.cpp:69-106 */
int orc_target_model(const uint16_t* tfi, int tw, int th, int b,
                     const orc_kernel* k, int method, int rings, int rule,
                     double* model) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  if (tw != k->kw || th != k->kh) return ORC_MODEL;
  double* raw = (double*)malloc((size_t)b * sizeof(double));
  const int hx = k_hx(k), hy = k_hy(k);
  if (method == ORC_CAKE) {
    const size_t n = ((size_t)tw + 1) * ((size_t)th + 1) * b;
    int64_t* p = (int64_t*)malloc(n * 8);
    int64_t* x = (int64_t*)malloc(n * 8);
    int64_t* y = (int64_t*)malloc(n * 8);
    int* sx = (int*)malloc((size_t)rings * sizeof(int) + 4);
    int* sy = (int*)malloc((size_t)rings * sizeof(int) + 4);
    double* rw = (double*)malloc((size_t)rings * sizeof(double) + 8);
    orc_build_tables(tfi, tw, th, b, p, x, y);
    st = orc_cake_plan(k, rings, rule, sx, sy, rw);
    if (!st)
      st = orc_cake_histogram(p, tw, th, b, k, rings, sx, sy, rw, hx, hy,
                              ORC_STRICT, raw);
    free(p); free(x); free(y); free(sx); free(sy); free(rw);
  } else {
    orc_kernel kk = *k;
    if (method == ORC_PLAIN) kk.kind = ORC_UNIFORM, kk.sigma = 0.5;
    if (k_integer(&kk)) {
      int64_t* cnt = (int64_t*)malloc((size_t)b * sizeof(int64_t));
      st = orc_brute_counts(tfi, tw, th, b, hx, hy, &kk, ORC_STRICT, cnt);
      for (int i = 0; i < b; ++i) raw[i] = (double)cnt[i];
      free(cnt);
    } else {
      st = orc_brute_weights(tfi, tw, th, b, hx, hy, &kk, ORC_STRICT, raw);
    }
  }
  if (!st) st = orc_normalize(raw, b, model);
  free(raw);
  return st;
}

typedef struct {
  const uint16_t* fi;
  int w, h, b;
  const double* model;
  orc_kernel k;
  int method, sim, rings;
  const int *sx, *sy;
  const double* rw;
  const int64_t *p, *x, *y;
  int mw;
  int v_first; /* first map row stored at scores[0] */
  double* scores;
  int status;
} sweep_ctx;

/* matching.cpp:151-189 */
static int sweep_rows(sweep_ctx* c, int v0, int v1) {
  const int hx = k_hx(&c->k), hy = k_hy(&c->k);
  int64_t* counts = (int64_t*)malloc((size_t)c->b * sizeof(int64_t));
  double* weights = (double*)malloc((size_t)c->b * sizeof(double));
  const orc_kernel uni = {ORC_UNIFORM, c->k.kw, c->k.kh, 0.5};
  int st = ORC_OK;
  for (int v = v0; v < v1 && !st; ++v) {
    double* dst = c->scores + (size_t)(v - c->v_first) * c->mw;
    for (int u = 0; u < c->mw && !st; ++u) {
      const int cx = u + hx, cy = v + hy;
      double s = 0.0;
      switch (c->method) {
        case ORC_SWIH:
          st = orc_swih_query(c->p, c->x, c->y, c->w, c->h, c->b, cx, cy,
                              &c->k, ORC_STRICT, counts);
          if (!st) st = orc_score_counts(c->sim, c->model, counts, c->b, &s);
          break;
        case ORC_PLAIN:
          st = orc_plain_query(c->p, c->w, c->h, c->b, cx, cy, &uni,
                               ORC_STRICT, counts);
          if (!st) st = orc_score_counts(c->sim, c->model, counts, c->b, &s);
          break;
        case ORC_CAKE:
          st = orc_cake_histogram(c->p, c->w, c->h, c->b, &c->k, c->rings,
                                  c->sx, c->sy, c->rw, cx, cy, ORC_STRICT,
                                  weights);
          if (!st) st = orc_score_weights(c->sim, c->model, weights, c->b, &s);
          break;
        case ORC_BRUTE:
          if (k_integer(&c->k)) {
            st = orc_brute_counts(c->fi, c->w, c->h, c->b, cx, cy, &c->k,
                                  ORC_STRICT, counts);
            if (!st) st = orc_score_counts(c->sim, c->model, counts, c->b, &s);
          } else {
            st = orc_brute_weights(c->fi, c->w, c->h, c->b, cx, cy, &c->k,
                                   ORC_STRICT, weights);
            if (!st)
              st = orc_score_weights(c->sim, c->model, weights, c->b, &s);
          }
          break;
      }
      dst[u] = s;
    }
  }
  free(counts);
  free(weights);
  return st;
}

static void* sweep_thread(void* arg) {
  void** a = (void**)arg;
  sweep_ctx* c = (sweep_ctx*)a[0];
  const int v0 = (int)(intptr_t)a[1], v1 = (int)(intptr_t)a[2];
  int st = sweep_rows(c, v0, v1);
  if (st) c->status = st;
  return NULL;
}

static int likelihood_impl(const uint16_t* fi, int w, int h, int b,
                           const double* model, int model_normalized,
                           const orc_kernel* k, int method, int sim, int rings,
                           int rule, int v0, int v1, int threads,
                           double* scores) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  if (w < k->kw || h < k->kh) return ORC_SIZE;
  if (!model_normalized) return ORC_MODEL;
  if (method == ORC_SWIH && !k_affine(k)) return ORC_UNSUPPORTED_KERNEL;
  const int mw = w - k->kw + 1, mh = h - k->kh + 1;
  if (v0 == 0 && v1 == 0) v1 = mh;
  if (v0 < 0 || v1 > mh || v0 > v1) return ORC_OUT_OF_RANGE;

  sweep_ctx c;
  memset(&c, 0, sizeof c);
  c.fi = fi; c.w = w; c.h = h; c.b = b; c.model = model; c.k = *k;
  c.method = method; c.sim = sim; c.rings = rings; c.mw = mw;
  c.v_first = v0; c.scores = scores;
  int64_t *p = NULL, *x = NULL, *y = NULL;
  int *sx = NULL, *sy = NULL;
  double* rw = NULL;
  if (method != ORC_BRUTE) {
    const size_t n = ((size_t)w + 1) * ((size_t)h + 1) * b;
    p = (int64_t*)malloc(n * 8);
    x = (int64_t*)malloc(n * 8);
    y = (int64_t*)malloc(n * 8);
    if (!p || !x || !y) {
      free(p); free(x); free(y);
      return ORC_CAPACITY;
    }
    orc_build_tables(fi, w, h, b, p, x, y);
  }
  if (method == ORC_CAKE) {
    sx = (int*)malloc((size_t)(rings > 0 ? rings : 1) * sizeof(int));
    sy = (int*)malloc((size_t)(rings > 0 ? rings : 1) * sizeof(int));
    rw = (double*)malloc((size_t)(rings > 0 ? rings : 1) * sizeof(double));
    st = orc_cake_plan(k, rings, rule, sx, sy, rw);
  }
  c.p = p; c.x = x; c.y = y; c.sx = sx; c.sy = sy; c.rw = rw;
  if (!st) {
    if (threads <= 1) {
      st = sweep_rows(&c, v0, v1);
    } else {
      const int rows = v1 - v0;
      if (threads > rows) threads = rows > 0 ? rows : 1;
      const int chunk = (rows + threads - 1) / threads;
      pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
      void*(*args)[3] = malloc(sizeof(void* [3]) * threads);
      int started = 0;
      for (int t = 0; t < threads; ++t) {
        const int a = v0 + t * chunk, e = imin(v1, a + chunk);
        if (a >= e) break;
        args[t][0] = &c;
        args[t][1] = (void*)(intptr_t)a;
        args[t][2] = (void*)(intptr_t)e;
        pthread_create(&th[t], NULL, sweep_thread, args[t]);
        ++started;
      }
      for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
      free(th);
      free(args);
      st = c.status;
    }
  }
  free(p); free(x); free(y); free(sx); free(sy); free(rw);
  return st;
}

/* matching.cpp:108-209 */
int orc_likelihood_map(const uint16_t* fi, int w, int h, int b,
                       const double* model, int model_normalized,
                       const orc_kernel* k, int method, int sim, int rings,
                       int rule, int v0, int v1, double* scores) {
  return likelihood_impl(fi, w, h, b, model, model_normalized, k, method, sim,
                         rings, rule, v0, v1, 1, scores);
}

int orc_likelihood_map_mt(const uint16_t* fi, int w, int h, int b,
                          const double* model, const orc_kernel* k, int method,
                          int sim, int rings, int rule, int v0, int v1,
                          int threads, double* scores) {
  return likelihood_impl(fi, w, h, b, model, 1, k, method, sim, rings, rule, v0,
                         v1, threads, scores);
}

/* matching.cpp:211-223: strict '>' in row-major order, first maximum wins */
int orc_peak(const double* scores, int mw, int mh, int hx, int hy,
             orc_peak_t* out) {
  if (mw <= 0 || mh <= 0) return ORC_ERROR;
  orc_peak_t best = {0, 0, 0, 0, -1.0};
  for (int v = 0; v < mh; ++v)
    for (int u = 0; u < mw; ++u) {
      const double s = scores[(size_t)v * mw + u];
      if (s > best.score) {
        best.map_x = u;
        best.map_y = v;
        best.center_x = u + hx;
        best.center_y = v + hy;
        best.score = s;
      }
    }
  *out = best;
  return ORC_OK;
}
