/*
 * swih_oracle.h — CPU restatement of the reference SWIH hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 path; nothing in the product (paper_1705_03524_b200/, include/) links
 * or calls it.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj) in plain C with the same arithmetic order, so that
 * fp64 results are bit-identical to the reference built with
 * `-O3 -std=gnu++20` (SSE2, no FMA).  Declared extensions that the
 * reference lacks (uint16 / RGB quantisers) are marked "parity unpinned".
 *
 * Status codes mirror the reference exception taxonomy
 * (proj/include/swih/errors.hpp:10-79) one code per class.
 */
#ifndef SWIH_ORACLE_H
#define SWIH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_ERROR = 1,
  ORC_IO = 2,
  ORC_ZERO_MASS = 3,
  ORC_INVALID_KERNEL = 4,
  ORC_OUT_OF_RANGE = 5,
  ORC_UNSUPPORTED_KERNEL = 6,
  ORC_WINDOW_OOB = 7,
  ORC_CAPACITY = 8,
  ORC_CONFIG = 9,
  ORC_MODEL = 10,
  ORC_SIZE = 11
};

/* KernelKind order of proj/include/swih/kernel.hpp:9-14, then the declared
 * extensions of SURVEY App. A (no reference implementation: parity unpinned):
 *   ORC_EUCLID_QUAD  w = 2(hx+1)^2(hy+1)^2 - dx^2(hy+1)^2 - dy^2(hx+1)^2
 *   ORC_EXP_L1       w = sigma^(|dx| + |dy|)   (sigma = decay per pixel in (0,1)) */
enum { ORC_UNIFORM = 0, ORC_MANHATTAN = 1, ORC_CHEBYSHEV = 2, ORC_GAUSS_CHEB = 3,
       ORC_EUCLID_QUAD = 4, ORC_EXP_L1 = 5 };
/* MapMethod order of proj/include/swih/matching.hpp:25 */
enum { ORC_SWIH = 0, ORC_BRUTE = 1, ORC_CAKE = 2, ORC_PLAIN = 3 };
/* SimilarityKind, matching.hpp:16-19 */
enum { ORC_BHATTACHARYYA = 0, ORC_INTERSECTION = 1 };
/* BorderPolicy, engine.hpp:12-15 */
enum { ORC_STRICT = 0, ORC_CLIPPED = 1 };
/* RingRule, baselines.hpp:41-44 */
enum { ORC_RING_MEAN = 0, ORC_RING_LEVEL = 1 };

typedef struct {
  int kind;
  int kw;
  int kh;
  double sigma;
} orc_kernel;

typedef struct {
  int map_x, map_y, center_x, center_y;
  double score;
} orc_peak_t;

/* std::mt19937_64 (C++ [rand.eng.mers]); the reference's seeded images use
 * rng() % 256 (tests/test_util.hpp:21-26, src/bench.cpp:28-33). */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
void orc_random_gray(int w, int h, uint64_t seed, uint8_t* out);

/* Quantisers.  gray8: image.hpp:43-45 / image.cpp:34-40.
 * gray16 and rgb8 are declared extensions — parity unpinned. */
int orc_quantize_gray8(const uint8_t* px, size_t n, int bins, uint16_t* out);
int orc_quantize_gray16(const uint16_t* px, size_t n, int bins, uint16_t* out);
int orc_quantize_rgb8(const uint8_t* px, size_t n, int levels, uint16_t* out);

/* Kernels: kernel.cpp:10-83 */
int orc_validate_kernel(const orc_kernel* k);
int orc_weight_at(const orc_kernel* k, int dx, int dy, double* w);
int orc_kernel_weight_sum(const orc_kernel* k, double* sum);

/* Integral tables: integral_tables.cpp:72-115.  Each output holds
 * (w+1)*(h+1)*b int64, bin-major, row stride w+1. */
void orc_build_tables(const uint16_t* fi, int w, int h, int b, int64_t* plain,
                      int64_t* xramp, int64_t* yramp);

/* Quadrant query: engine.cpp:7-147.  out has b entries. */
int orc_swih_query(const int64_t* plain, const int64_t* xramp,
                   const int64_t* yramp, int w, int h, int b, int cx, int cy,
                   const orc_kernel* k, int border, int64_t* out);
/* Plain local histogram: engine.cpp:156-165 */
int orc_plain_query(const int64_t* plain, int w, int h, int b, int cx, int cy,
                    const orc_kernel* k, int border, int64_t* out);

/* Brute force: baselines.cpp:8-69 */
int orc_brute_counts(const uint16_t* fi, int w, int h, int b, int cx, int cy,
                     const orc_kernel* k, int border, int64_t* out);
int orc_brute_weights(const uint16_t* fi, int w, int h, int b, int cx, int cy,
                      const orc_kernel* k, int border, double* out);

/* Wedding cake plan + query: baselines.cpp:84-149 */
int orc_cake_plan(const orc_kernel* k, int rings, int rule, int* shrink_x,
                  int* shrink_y, double* ring_weight);
int orc_cake_histogram(const int64_t* plain, int w, int h, int b,
                       const orc_kernel* k, int rings, const int* shrink_x,
                       const int* shrink_y, const double* ring_weight, int cx,
                       int cy, int border, double* out);

/* Scores: matching.cpp:20-67 */
int orc_score_counts(int sim, const double* model, const int64_t* raw, int b,
                     double* s);
int orc_score_weights(int sim, const double* model, const double* raw, int b,
                      double* s);
int orc_similarity(int sim, const double* p, const double* q, int b, double* s);

/* Histogram normalisation: histogram.cpp:19-26 */
int orc_normalize(const double* in, int b, double* out);

/* Target model: matching.cpp:69-106 (template must be kw x kh). */
int orc_target_model(const uint16_t* templ_fi, int tw, int th, int b,
                     const orc_kernel* k, int method, int rings, int rule,
                     double* model);

/* Likelihood map over a quantised image: matching.cpp:108-209 (serial;
 * the reference result is identical for any thread count,
 * matching.cpp:195-196).  scores has (w-kw+1)*(h-kh+1) entries.
 * rows [v0, v1) only when v1 > v0 (full map when v0 == v1 == 0). */
int orc_likelihood_map(const uint16_t* fi, int w, int h, int b,
                       const double* model, int model_normalized,
                       const orc_kernel* k, int method, int sim, int rings,
                       int rule, int v0, int v1, double* scores);

/* Peak: matching.cpp:211-223 */
int orc_peak(const double* scores, int mw, int mh, int hx, int hy,
             orc_peak_t* out);

/* Threaded variant of orc_likelihood_map (pthreads row chunks, like
 * matching.cpp:191-207); used as the "port" CPU baseline only. */
int orc_likelihood_map_mt(const uint16_t* fi, int w, int h, int b,
                          const double* model, const orc_kernel* k, int method,
                          int sim, int rings, int rule, int v0, int v1,
                          int threads, double* scores);

/* Full-size maps (swih_fastmap.c): the same per-window fp64 operation
 * sequence as orc_likelihood_map, computed bin-outer on `threads` threads.
 * method SWIH (Uniform, Manhattan), PLAIN, CAKE (any ring plan), BRUTE with
 * Uniform / Manhattan / Euclidean-quadratic: bit-identical full maps.
 * BRUTE with the exponential kernel: two phases -- a separable-filter map,
 * then every window within eps of its maximum re-scored by orc_brute_weights
 * in the reference's pixel order; `peak` is exact, n_exact = re-scored
 * windows.  Full strict map: (w-kw+1)*(h-kh+1) scores. */
#define SWIH_FM_MAX_RINGS 512
int orc_fast_map(const uint16_t* fi, int w, int h, int b, const double* model,
                 const orc_kernel* k, int method, int sim, int rings, int rule,
                 int threads, double eps, double* scores, orc_peak_t* peak,
                 long long* n_exact);

#ifdef __cplusplus
}
#endif
#endif
