/*
 * swih_fastmap.c — full-size likelihood maps for the parity suite.
 *
 * TEST INFRASTRUCTURE ONLY (like swih_oracle.c): the checker the full-size
 * GPU parity tests compare against.  Nothing in the product links or calls it.
 *
 * orc_likelihood_map (swih_oracle.c) restates the reference window by
 * window: per window, swih_query_into / brute force / wedding cake
 * (engine.cpp:39-147, baselines.cpp:8-69,133-149) fills b raw values, then
 * score_counts / score_weights (matching.cpp:20-52) folds them in bin order.
 * At BASELINE sizes that costs minutes to hours.  This file computes the SAME
 * per-window fp64 operation sequence, reorganised BIN-OUTER:
 *
 *   for bin i = 0 .. b-1:            (in order)
 *     raw_i(w) for every window w    (a row of windows is one vector loop)
 *     s(w)    = s(w) + sqrt(model_i * raw_i(w))       (Bhattacharyya)
 *     mass(w) = mass(w) + raw_i(w)                   (score_weights only)
 *   s(w) = clamp01(s(w) / sqrt(mass(w)))
 *
 * Each window's s and mass see exactly the reference's operations in the
 * reference's order (the interleaving across windows is irrelevant), so the
 * maps are bit-identical to orc_likelihood_map -- checked on CPU by
 * tests/test_oracle_fastmap.py against it (and through it the reference).
 * Built with -ffp-contract=off: vector mulpd / addpd / sqrtpd are IEEE
 * correctly rounded like the reference's scalar SSE2 code.
 *
 * raw_i per kernel:
 *   Uniform / Manhattan swih, Plain, integer brute force (Uniform,
 *   Manhattan, declared Euclidean quadratic): EXACT integers from local
 *   per-bin prefix planes {1, x, y, x^2, y^2} (int64) -- the reference's
 *   integer sums are exact, so any exact formula gives the same integer:
 *     Manhattan  H = M*N - sum|x-cx| - sum|y-cy|   (M = hx+hy+1)
 *     quadratic  H = A*N - ky*sum(x-cx)^2 - kx*sum(y-cy)^2
 *   Wedding cake (baselines.cpp:139-148): out = out + coeff_r * count_r over
 *   the rings in order, count_r a box of the plain prefix plane.
 *   Declared exponential (brute force, score_weights, parity unpinned): TWO
 *   PHASES, like the GPU path: (1) every window from a separable recursive
 *   filter (relative error ~1e-13, not the reference's order); (2) every
 *   window within `eps` of the phase-1 maximum is re-scored by the brute
 *   force in the reference's pixel order (orc_brute_weights +
 *   orc_score_weights) and written back; the peak is taken among those
 *   exact scores with the reference tie rule (matching.cpp:211-223).
 *
 * Threads own contiguous map-row chunks and build their prefix planes over
 * the pixel rows those windows touch (a local table: the four-corner rule
 * cancels the missing rows above, SURVEY §8e row bands).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "swih_oracle.h"

static inline int fm_imin(int a, int b) { return a < b ? a : b; }
static inline int fm_imax(int a, int b) { return a > b ? a : b; }
static inline double fm_clamp01(double v) { return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v); }
static inline double fm_min(double a, double b) { return (b < a) ? b : a; }

enum { FM_INT = 0, FM_CAKE = 1, FM_EXP = 2 };

typedef struct {
  /* problem */
  const uint16_t* fi;
  int w, h, b;
  const double* model;
  orc_kernel k;
  int method, sim, mode; /* mode FM_* */
  int uniform;           /* integer mode: 0 Manhattan, 1 Uniform/Plain, 2 quadratic */
  int rings;
  int sx[SWIH_FM_MAX_RINGS], sy[SWIH_FM_MAX_RINGS];
  double coeff[SWIH_FM_MAX_RINGS];
  int64_t int_mass; /* integer kernels: strict-window mass (score_counts) */
  int mw, mh;
  double* scores;
  /* thread chunk */
  int v0, v1;
  int status;
} fm_task;

/* Box sum of a local prefix plane P ((ny+1) x (w+1), row stride w+1):
 * rows [ya, yb) x columns [xa, xb) of the band. */
#define BOX(P, st, ya, yb, xa, xb) \
  ((P)[(size_t)(yb) * (st) + (xb)] - (P)[(size_t)(ya) * (st) + (xb)] - \
   (P)[(size_t)(yb) * (st) + (xa)] + (P)[(size_t)(ya) * (st) + (xa)])

/* Per-bin local prefix planes over pixel rows [y_lo, y_lo + ny). */
static int64_t build_planes(const fm_task* t, int bin, int y_lo, int ny, int nplanes,
                            int64_t* P, int64_t* X, int64_t* Y, int64_t* XX, int64_t* YY) {
  const int w = t->w;
  const size_t st = (size_t)w + 1;
  memset(P, 0, st * sizeof(int64_t));
  if (nplanes > 1) {
    memset(X, 0, st * sizeof(int64_t));
    memset(Y, 0, st * sizeof(int64_t));
  }
  if (nplanes > 3) {
    memset(XX, 0, st * sizeof(int64_t));
    memset(YY, 0, st * sizeof(int64_t));
  }
  int64_t total = 0;
  for (int r = 0; r < ny; ++r) {
    const uint16_t* row = t->fi + (size_t)(y_lo + r) * w;
    const size_t o = (size_t)(r + 1) * st, p = (size_t)r * st;
    const int64_t y = r; /* local row */
    int64_t cp = 0, cx = 0, cy = 0, cxx = 0, cyy = 0;
    P[o] = 0;
    if (nplanes > 1) X[o] = Y[o] = 0;
    if (nplanes > 3) XX[o] = YY[o] = 0;
    for (int x = 0; x < w; ++x) {
      const int64_t hit = row[x] == bin;
      cp += hit;
      P[o + x + 1] = P[p + x + 1] + cp;
      if (nplanes > 1) {
        cx += hit * x;
        cy += hit * y;
        X[o + x + 1] = X[p + x + 1] + cx;
        Y[o + x + 1] = Y[p + x + 1] + cy;
      }
      if (nplanes > 3) {
        cxx += hit * (int64_t)x * x;
        cyy += hit * y * y;
        XX[o + x + 1] = XX[p + x + 1] + cxx;
        YY[o + x + 1] = YY[p + x + 1] + cyy;
      }
    }
    total += cp;
  }
  return total;
}

/* ------------------------------------------------------------ integer / cake */
static void* fm_worker(void* arg) {
  fm_task* t = (fm_task*)arg;
  const int w = t->w, mw = t->mw, kw = t->k.kw, kh = t->k.kh;
  const int hx = (kw - 1) / 2, hy = (kh - 1) / 2;
  const int v0 = t->v0, v1 = t->v1, nv = v1 - v0;
  if (nv <= 0) return NULL;
  const int y_lo = v0, ny = nv + kh - 1;
  const size_t st = (size_t)w + 1, plane = (size_t)(ny + 1) * st;
  const int nplanes = t->mode == FM_CAKE || t->uniform == 1 ? 1 : (t->uniform == 2 ? 5 : 3);
  int64_t* buf = (int64_t*)malloc(plane * nplanes * sizeof(int64_t));
  double* s = (double*)calloc((size_t)nv * mw, sizeof(double));
  double* mass = (double*)calloc((size_t)nv * mw, sizeof(double));
  double* out = (double*)malloc((size_t)mw * sizeof(double));
  int64_t* raw = (int64_t*)malloc((size_t)mw * sizeof(int64_t));
  if (!buf || !s || !mass || !out || !raw) {
    t->status = ORC_CAPACITY;
    free(buf); free(s); free(mass); free(out); free(raw);
    return NULL;
  }
  int64_t* P = buf;
  int64_t* X = nplanes > 1 ? buf + plane : NULL;
  int64_t* Y = nplanes > 1 ? buf + 2 * plane : NULL;
  int64_t* XX = nplanes > 3 ? buf + 3 * plane : NULL;
  int64_t* YY = nplanes > 3 ? buf + 4 * plane : NULL;
  const int64_t M = hx + hy + 1;
  const int64_t kx = (int64_t)(hx + 1) * (hx + 1), ky = (int64_t)(hy + 1) * (hy + 1);
  const int64_t A = 2 * kx * ky;
  /* Intersection over score_weights needs each window's mass first: a mass
   * pass over the bins, then the score pass (the reference computes mass
   * before the score loop, matching.cpp:37-52). */
  const int two_pass = t->mode == FM_CAKE && t->sim == ORC_INTERSECTION;
  for (int pass = two_pass ? 0 : 1; pass < 2; ++pass) {
    for (int bin = 0; bin < t->b; ++bin) {
      const int64_t total = build_planes(t, bin, y_lo, ny, nplanes, P, X, Y, XX, YY);
      const double m = t->model[bin];
      if (total == 0) continue; /* raw = 0 everywhere: s + sqrt(m*0) == s, mass + 0 == mass */
      for (int v = 0; v < nv; ++v) {
        double* sr = s + (size_t)v * mw;
        double* mr = mass + (size_t)v * mw;
        if (t->mode == FM_CAKE) {
          for (int u = 0; u < mw; ++u) out[u] = 0.0;
          for (int i = 0; i < t->rings; ++i) {
            const int ya = v + t->sy[i], yb = v + kh - t->sy[i];
            const int xa = t->sx[i], xb = kw - t->sx[i];
            const double c = t->coeff[i];
            const int64_t* r0 = P + (size_t)ya * st;
            const int64_t* r1 = P + (size_t)yb * st;
            for (int u = 0; u < mw; ++u) {
              const int64_t cnt = r1[u + xb] - r0[u + xb] - r1[u + xa] + r0[u + xa];
              out[u] = out[u] + c * (double)cnt;
            }
          }
          if (pass == 0) {
            for (int u = 0; u < mw; ++u) mr[u] = mr[u] + out[u];
          } else if (t->sim == ORC_BHATTACHARYYA) {
            for (int u = 0; u < mw; ++u) {
              mr[u] = mr[u] + out[u];
              sr[u] = sr[u] + sqrt(m * out[u]);
            }
          } else {
            for (int u = 0; u < mw; ++u) sr[u] = sr[u] + fm_min(m, out[u] / mr[u]);
          }
          continue;
        }
        /* exact integer raw values */
        const int ya = v, yb = v + kh, yc = v + hy + 1; /* top / bottom / below centre row */
        const int64_t lcy = v + hy;                      /* local centre row */
        if (t->uniform == 1) {
          for (int u = 0; u < mw; ++u) raw[u] = BOX(P, st, ya, yb, u, u + kw);
        } else if (t->uniform == 0) {
          for (int u = 0; u < mw; ++u) {
            const int64_t cx = u + hx;
            const int64_t n = BOX(P, st, ya, yb, u, u + kw);
            const int64_t nl = BOX(P, st, ya, yb, u, u + hx + 1); /* columns <= cx */
            const int64_t xs = BOX(X, st, ya, yb, u, u + kw);
            const int64_t xl = BOX(X, st, ya, yb, u, u + hx + 1);
            const int64_t nt = BOX(P, st, ya, yc, u, u + kw); /* rows <= cy */
            const int64_t ys = BOX(Y, st, ya, yb, u, u + kw);
            const int64_t yt = BOX(Y, st, ya, yc, u, u + kw);
            const int64_t adx = (cx * nl - xl) + ((xs - xl) - cx * (n - nl));
            const int64_t ady = (lcy * nt - yt) + ((ys - yt) - lcy * (n - nt));
            raw[u] = M * n - adx - ady;
          }
        } else {
          for (int u = 0; u < mw; ++u) {
            const int64_t cx = u + hx;
            const int64_t n = BOX(P, st, ya, yb, u, u + kw);
            const int64_t xs = BOX(X, st, ya, yb, u, u + kw);
            const int64_t ys = BOX(Y, st, ya, yb, u, u + kw);
            const int64_t xxs = BOX(XX, st, ya, yb, u, u + kw);
            const int64_t yys = BOX(YY, st, ya, yb, u, u + kw);
            const int64_t dxx = xxs - 2 * cx * xs + cx * cx * n;
            const int64_t dyy = yys - 2 * lcy * ys + lcy * lcy * n;
            raw[u] = A * n - ky * dxx - kx * dyy;
          }
        }
        if (t->sim == ORC_BHATTACHARYYA) {
          for (int u = 0; u < mw; ++u) sr[u] = sr[u] + sqrt(m * (double)raw[u]);
        } else {
          const double dm = (double)t->int_mass;
          for (int u = 0; u < mw; ++u) sr[u] = sr[u] + fm_min(m, (double)raw[u] / dm);
        }
      }
    }
  }
  for (int v = 0; v < nv; ++v) {
    double* dst = t->scores + (size_t)(v0 + v) * mw;
    const double* sr = s + (size_t)v * mw;
    const double* mr = mass + (size_t)v * mw;
    for (int u = 0; u < mw; ++u) {
      double sc = sr[u];
      if (t->mode == FM_CAKE) {
        if (t->sim == ORC_BHATTACHARYYA) sc /= sqrt(mr[u]);
        if (mr[u] == 0.0) t->status = ORC_ZERO_MASS;
      } else if (t->sim == ORC_BHATTACHARYYA) {
        sc /= sqrt((double)t->int_mass);
      }
      dst[u] = fm_clamp01(sc);
    }
  }
  free(buf); free(s); free(mass); free(out); free(raw);
  return NULL;
}

/* ------------------------------------------------------- exponential phase 1 */
/* Separable recursive filter for w = d^|dx| * d^|dy| over the window:
 * along a line f, L(c) = sum_{j=0..h} d^j f(c-j), R(c) = sum_{j=1..h} d^j f(c+j),
 * out(c) = L(c) + R(c); damped recurrences (d < 1).  The horizontal pass
 * runs along each pixel row, the vertical one over whole rows at a time. */
static void exp_row(const uint16_t* row, int bin, int n, int hw, double d, double dh1,
                    double* out, double* tmp) {
  double l = 0.0;
  for (int c = 0; c < n; ++c) {
    l = (row[c] == bin ? 1.0 : 0.0) + d * l - (c - hw - 1 >= 0 && row[c - hw - 1] == bin ? dh1 : 0.0);
    tmp[c] = l;
  }
  double r = 0.0; /* R(c) */
  for (int c = n - 1; c >= 0; --c) {
    out[c] = tmp[c] + r;
    r = d * ((row[c] == bin ? 1.0 : 0.0) + r) - (c + hw < n && row[c + hw] == bin ? dh1 : 0.0);
  }
}

static void* fm_exp_worker(void* arg) {
  fm_task* t = (fm_task*)arg;
  const double d = t->k.sigma;
  const int w = t->w, mw = t->mw, kw = t->k.kw, kh = t->k.kh;
  const int hx = (kw - 1) / 2, hy = (kh - 1) / 2;
  const int v0 = t->v0, v1 = t->v1, nv = v1 - v0;
  if (nv <= 0) return NULL;
  const int ny = nv + kh - 1;
  const size_t st = (size_t)w + 1;
  const double dhx = pow(d, hx + 1), dhy = pow(d, hy + 1);
  double* H = (double*)malloc((size_t)ny * w * sizeof(double)); /* horizontal pass */
  double* Lv = (double*)malloc((size_t)ny * w * sizeof(double)); /* vertical L */
  double* R = (double*)malloc((size_t)w * sizeof(double));
  double* tmp = (double*)malloc((size_t)w * sizeof(double));
  int64_t* P = (int64_t*)malloc((size_t)(ny + 1) * st * sizeof(int64_t));
  char* hit = (char*)malloc((size_t)ny);
  double* s = (double*)calloc((size_t)nv * mw, sizeof(double));
  double* mass = (double*)calloc((size_t)nv * mw, sizeof(double));
  if (!H || !Lv || !R || !tmp || !P || !hit || !s || !mass) {
    t->status = ORC_CAPACITY;
    free(H); free(Lv); free(R); free(tmp); free(P); free(hit); free(s); free(mass);
    return NULL;
  }
  const int two_pass = t->sim == ORC_INTERSECTION;
  for (int pass = two_pass ? 0 : 1; pass < 2; ++pass) {
    for (int bin = 0; bin < t->b; ++bin) {
      /* exact per-window counts: an empty window's raw value is exactly 0
       * (the recurrences leave ~1e-17 residues there) */
      const int64_t total = build_planes(t, bin, v0, ny, 1, P, NULL, NULL, NULL, NULL);
      if (total == 0) continue;
      for (int r = 0; r < ny; ++r) {
        const uint16_t* row = t->fi + (size_t)(v0 + r) * w;
        hit[r] = P[(size_t)(r + 1) * st + w] != P[(size_t)r * st + w];
        if (hit[r]) exp_row(row, bin, w, hx, d, dhx, H + (size_t)r * w, tmp);
        else memset(H + (size_t)r * w, 0, (size_t)w * sizeof(double));
      }
      /* vertical: Lv(r) = H(r) + d Lv(r-1) - d^(hy+1) H(r-hy-1) */
      for (int r = 0; r < ny; ++r) {
        double* lr = Lv + (size_t)r * w;
        const double* hr = H + (size_t)r * w;
        if (r == 0) {
          memcpy(lr, hr, (size_t)w * sizeof(double));
        } else if (r - hy - 1 >= 0) {
          const double* lp = Lv + (size_t)(r - 1) * w;
          const double* he = H + (size_t)(r - hy - 1) * w;
          for (int x = 0; x < w; ++x) lr[x] = hr[x] + d * lp[x] - dhy * he[x];
        } else {
          const double* lp = Lv + (size_t)(r - 1) * w;
          for (int x = 0; x < w; ++x) lr[x] = hr[x] + d * lp[x];
        }
      }
      const double m = t->model[bin];
      for (int x = 0; x < w; ++x) R[x] = 0.0;
      for (int r = ny - 1; r >= 0; --r) {
        const int v = r - hy; /* map row whose centre row is r */
        if (v >= 0 && v < nv) {
          const double* lr = Lv + (size_t)r * w;
          const int64_t* p0 = P + (size_t)v * st;
          const int64_t* p1 = P + (size_t)(v + kh) * st;
          double* sr = s + (size_t)v * mw;
          double* mr = mass + (size_t)v * mw;
          for (int u = 0; u < mw; ++u) {
            const int64_t cnt = p1[u + kw] - p0[u + kw] - p1[u] + p0[u];
            double x = cnt ? lr[u + hx] + R[u + hx] : 0.0;
            if (x < 0.0) x = 0.0;
            if (pass == 0) {
              mr[u] = mr[u] + x;
            } else if (t->sim == ORC_BHATTACHARYYA) {
              mr[u] = mr[u] + x;
              sr[u] = sr[u] + sqrt(m * x);
            } else {
              sr[u] = sr[u] + fm_min(m, x / mr[u]);
            }
          }
        }
        /* R(r-1) = d (H(r) + R(r)) - d^(hy+1) H(r+hy) */
        const double* hr = H + (size_t)r * w;
        if (r + hy < ny) {
          const double* he = H + (size_t)(r + hy) * w;
          for (int x = 0; x < w; ++x) R[x] = d * (hr[x] + R[x]) - dhy * he[x];
        } else {
          for (int x = 0; x < w; ++x) R[x] = d * (hr[x] + R[x]);
        }
      }
    }
  }
  for (int v = 0; v < nv; ++v)
    for (int u = 0; u < mw; ++u) {
      const size_t o = (size_t)v * mw + u;
      double sc = s[o];
      if (t->sim == ORC_BHATTACHARYYA) sc /= sqrt(mass[o]);
      t->scores[(size_t)(v0 + v) * mw + u] = fm_clamp01(sc);
    }
  free(H); free(Lv); free(R); free(tmp); free(P); free(hit); free(s); free(mass);
  return NULL;
}

/* ----------------------------------------------------------------- driver */
static int run_threads(fm_task* proto, int threads, void* (*fn)(void*)) {
  const int mh = proto->mh;
  if (threads < 1) threads = 1;
  if (threads > mh) threads = mh;
  fm_task* ts = (fm_task*)malloc(sizeof(fm_task) * threads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  const int chunk = (mh + threads - 1) / threads;
  int n = 0;
  for (int i = 0; i < threads; ++i) {
    const int a = i * chunk, e = fm_imin(mh, a + chunk);
    if (a >= e) break;
    ts[i] = *proto;
    ts[i].v0 = a;
    ts[i].v1 = e;
    ts[i].status = ORC_OK;
    pthread_create(&th[i], NULL, fn, &ts[i]);
    ++n;
  }
  int st = ORC_OK;
  for (int i = 0; i < n; ++i) {
    pthread_join(th[i], NULL);
    if (ts[i].status) st = ts[i].status;
  }
  free(ts);
  free(th);
  return st;
}

typedef struct {
  const fm_task* t;
  const long long* idx;
  int n;
  int next;
  pthread_mutex_t mu;
  int status;
} rescore_ctx;

static void* rescore_worker(void* arg) {
  rescore_ctx* c = (rescore_ctx*)arg;
  const fm_task* t = c->t;
  double* weights = (double*)malloc((size_t)t->b * sizeof(double));
  const int hx = (t->k.kw - 1) / 2, hy = (t->k.kh - 1) / 2;
  for (;;) {
    pthread_mutex_lock(&c->mu);
    const int i = c->next++;
    pthread_mutex_unlock(&c->mu);
    if (i >= c->n) break;
    const long long id = c->idx[i];
    const int u = (int)(id % t->mw), v = (int)(id / t->mw);
    double sc = 0.0;
    int st = orc_brute_weights(t->fi, t->w, t->h, t->b, u + hx, v + hy, &t->k, ORC_STRICT,
                               weights);
    if (!st) st = orc_score_weights(t->sim, t->model, weights, t->b, &sc);
    if (st) c->status = st;
    t->scores[id] = sc;
  }
  free(weights);
  return NULL;
}

int orc_fast_map(const uint16_t* fi, int w, int h, int b, const double* model,
                 const orc_kernel* k, int method, int sim, int rings, int rule,
                 int threads, double eps, double* scores, orc_peak_t* peak,
                 long long* n_exact) {
  int st = orc_validate_kernel(k);
  if (st) return st;
  if (w < k->kw || h < k->kh) return ORC_SIZE;
  fm_task t;
  memset(&t, 0, sizeof t);
  t.fi = fi; t.w = w; t.h = h; t.b = b; t.model = model; t.k = *k;
  t.method = method; t.sim = sim; t.scores = scores;
  t.mw = w - k->kw + 1;
  t.mh = h - k->kh + 1;
  const int hx = (k->kw - 1) / 2, hy = (k->kh - 1) / 2;
  if (n_exact) *n_exact = 0;
  if (method == ORC_CAKE) {
    if (rings < 1 || rings > SWIH_FM_MAX_RINGS) return ORC_CONFIG;
    double rw[SWIH_FM_MAX_RINGS];
    st = orc_cake_plan(k, rings, rule, t.sx, t.sy, rw);
    if (st) return st;
    for (int i = 0; i < rings; ++i) t.coeff[i] = rw[i] - (i > 0 ? rw[i - 1] : 0.0);
    t.rings = rings;
    t.mode = FM_CAKE;
  } else if (method == ORC_SWIH || method == ORC_PLAIN ||
             (method == ORC_BRUTE && (k->kind == ORC_UNIFORM || k->kind == ORC_MANHATTAN ||
                                      k->kind == ORC_EUCLID_QUAD))) {
    if (method == ORC_SWIH && k->kind != ORC_UNIFORM && k->kind != ORC_MANHATTAN)
      return ORC_UNSUPPORTED_KERNEL;
    t.mode = FM_INT;
    const int kind = method == ORC_PLAIN ? ORC_UNIFORM : k->kind;
    t.uniform = kind == ORC_UNIFORM ? 1 : (kind == ORC_MANHATTAN ? 0 : 2);
    /* strict-window mass: sum of the integer weights (every pixel has a bin) */
    int64_t mass = 0;
    orc_kernel kk = *k;
    kk.kind = kind;
    for (int dy = -hy; dy <= hy; ++dy)
      for (int dx = -hx; dx <= hx; ++dx) {
        double wd;
        orc_weight_at(&kk, dx, dy, &wd);
        mass += llround(wd);
      }
    if (mass == 0) return ORC_ZERO_MASS;
    t.int_mass = mass;
  } else if (method == ORC_BRUTE && k->kind == ORC_EXP_L1) {
    t.mode = FM_EXP;
  } else {
    return ORC_UNSUPPORTED_KERNEL;
  }
  st = run_threads(&t, threads, t.mode == FM_EXP ? fm_exp_worker : fm_worker);
  if (st) return st;
  const size_t n = (size_t)t.mw * t.mh;
  if (t.mode != FM_EXP) return orc_peak(scores, t.mw, t.mh, hx, hy, peak);
  /* phase 2: exact re-score of every window within eps of the phase-1 max */
  double mx = -1.0;
  for (size_t i = 0; i < n; ++i)
    if (scores[i] > mx) mx = scores[i];
  size_t cnt = 0;
  for (size_t i = 0; i < n; ++i)
    if (scores[i] >= mx - eps) ++cnt;
  long long* idx = (long long*)malloc((cnt ? cnt : 1) * sizeof(long long));
  cnt = 0;
  for (size_t i = 0; i < n; ++i)
    if (scores[i] >= mx - eps) idx[cnt++] = (long long)i;
  rescore_ctx c;
  c.t = &t; c.idx = idx; c.n = (int)cnt; c.next = 0; c.status = ORC_OK;
  pthread_mutex_init(&c.mu, NULL);
  const int nt = threads < 1 ? 1 : threads;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
  for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, rescore_worker, &c);
  for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&c.mu);
  if (c.status) {
    free(idx);
    return c.status;
  }
  /* matching.cpp:211-223 among the exact scores (indices ascending) */
  orc_peak_t best = {0, 0, 0, 0, -1.0};
  for (size_t i = 0; i < cnt; ++i) {
    const double sc = scores[idx[i]];
    if (sc > best.score) {
      best.map_x = (int)(idx[i] % t.mw);
      best.map_y = (int)(idx[i] / t.mw);
      best.center_x = best.map_x + hx;
      best.center_y = best.map_y + hy;
      best.score = sc;
    }
  }
  *peak = best;
  if (n_exact) *n_exact = (long long)cnt;
  free(idx);
  return ORC_OK;
}
