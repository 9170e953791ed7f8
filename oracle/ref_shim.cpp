// ref_shim.cpp — extern "C" wrapper over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together
// with /root/reference/proj/src/*.cpp into oracle/_ref/libswihref.so (the
// reference sources are compiled where they lie, never copied).  It lets the
// Python tests pin the C restatement (swih_oracle.c) against the reference
// itself, and lets bench.py --impl reference time the reference CPU path.
// Exceptions become the status codes of swih_oracle.h (errors.hpp:10-79).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "swih/baselines.hpp"
#include "swih/bench.hpp"
#include "swih/engine.hpp"
#include "swih/integral_tables.hpp"
#include "swih/matching.hpp"
#include "swih/pgm.hpp"

using namespace swih;

namespace {

thread_local std::string g_err;
thread_local std::size_t g_required = 0;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const CapacityError& e) {
    g_err = e.what();
    g_required = e.required_bytes();
    return 8;
  } catch (const IoError& e) {
    g_err = e.what();
    return 2;
  } catch (const ZeroMassError& e) {
    g_err = e.what();
    return 3;
  } catch (const InvalidKernelError& e) {
    g_err = e.what();
    return 4;
  } catch (const OutOfRangeError& e) {
    g_err = e.what();
    return 5;
  } catch (const UnsupportedKernelError& e) {
    g_err = e.what();
    return 6;
  } catch (const WindowOutOfBoundsError& e) {
    g_err = e.what();
    return 7;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 9;
  } catch (const ModelError& e) {
    g_err = e.what();
    return 10;
  } catch (const SizeError& e) {
    g_err = e.what();
    return 11;
  } catch (const Error& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

KernelSpec mk(int kind, int kw, int kh, double sigma) {
  return KernelSpec{static_cast<KernelKind>(kind), kw, kh, sigma};
}

FeatureImage to_fi(const std::uint16_t* fi, int w, int h, int b) {
  FeatureImage f(w, h, b);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) f.set(x, y, fi[std::size_t(y) * w + x]);
  return f;
}

GrayImage to_gray(const std::uint8_t* px, int w, int h) {
  return GrayImage(w, h, std::vector<std::uint8_t>(px, px + std::size_t(w) * h));
}

// Restatement of the anonymous-namespace scorers (matching.cpp:20-52); they
// cannot be linked, so the best-use sweep below carries its own copy.
double score_counts_r(int sim, const double* model, const std::int64_t* raw,
                      int b) {
  std::int64_t mass = 0;
  for (int i = 0; i < b; ++i) mass += raw[i];
  if (mass == 0) throw ZeroMassError("similarity: empty candidate window");
  double s = 0.0;
  if (sim == 0) {
    for (int i = 0; i < b; ++i) s += std::sqrt(model[i] * double(raw[i]));
    s /= std::sqrt(double(mass));
  } else {
    for (int i = 0; i < b; ++i) s += std::min(model[i], double(raw[i]) / mass);
  }
  return std::clamp(s, 0.0, 1.0);
}

double score_weights_r(int sim, const double* model, const double* raw, int b) {
  double mass = 0.0;
  for (int i = 0; i < b; ++i) mass += raw[i];
  if (mass == 0.0) throw ZeroMassError("similarity: empty candidate window");
  double s = 0.0;
  if (sim == 0) {
    for (int i = 0; i < b; ++i) s += std::sqrt(model[i] * raw[i]);
    s /= std::sqrt(mass);
  } else {
    for (int i = 0; i < b; ++i) s += std::min(model[i], raw[i] / mass);
  }
  return std::clamp(s, 0.0, 1.0);
}

struct Tables {
  FeatureImage fi;
  IntegralTableSet t;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
std::size_t ref_last_required_bytes() { return g_required; }

void ref_random_gray(int w, int h, std::uint64_t seed, std::uint8_t* out) {
  const GrayImage img = random_image(w, h, seed);
  std::memcpy(out, img.pixels().data(), std::size_t(w) * h);
}

int ref_quantize(const std::uint8_t* px, int w, int h, int bins,
                 std::uint16_t* out) {
  return guarded([&] {
    const FeatureImage fi = quantize_image(to_gray(px, w, h), Quantizer(bins));
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) out[std::size_t(y) * w + x] = fi.at(x, y);
  });
}

int ref_weight_at(int kind, int kw, int kh, double sigma, int dx, int dy,
                  double* out) {
  return guarded([&] { *out = weight_at(mk(kind, kw, kh, sigma), dx, dy); });
}

int ref_kernel_weight_sum(int kind, int kw, int kh, double sigma, double* out) {
  return guarded([&] { *out = kernel_weight_sum(mk(kind, kw, kh, sigma)); });
}

int ref_tables_new(const std::uint16_t* fi, int w, int h, int b,
                   std::size_t budget, void** out) {
  return guarded([&] {
    TableBuildOptions opt;
    if (budget) opt.memory_budget_bytes = budget;
    FeatureImage f = to_fi(fi, w, h, b);
    IntegralTableSet t = build_tables(f, opt);
    *out = new Tables{std::move(f), std::move(t)};
  });
}

void ref_tables_free(void* t) { delete static_cast<Tables*>(t); }

int ref_tables_export(void* tv, int kind, std::int64_t* out) {
  return guarded([&] {
    const IntegralTableSet& t = static_cast<Tables*>(tv)->t;
    const std::size_t n = t.plane_stride() * t.bins();
    std::memcpy(out, t.plane(static_cast<TableKind>(kind), 0), n * 8);
  });
}

int ref_tables_cell(void* tv, int kind, int x, int y, int bin,
                    std::int64_t* out) {
  return guarded([&] {
    *out = static_cast<Tables*>(tv)->t.cell(static_cast<TableKind>(kind), x, y,
                                            bin);
  });
}

int ref_rect_sum(void* tv, int kind, int x0, int y0, int x1, int y1, int bin,
                 std::int64_t* out) {
  return guarded([&] {
    *out = static_cast<Tables*>(tv)->t.rect_sum(static_cast<TableKind>(kind),
                                                RectRegion{x0, y0, x1, y1}, bin);
  });
}

int ref_directional(void* tv, int dir, int x, int y, int bin,
                    std::int64_t* out) {
  return guarded([&] {
    *out = static_cast<Tables*>(tv)->t.directional_value(
        static_cast<Direction>(dir), x, y, bin);
  });
}

int ref_tables_save(void* tv, const char* path) {
  return guarded([&] { static_cast<Tables*>(tv)->t.save_file(path); });
}

// IntegralTableSet::load_file (integral_tables.cpp:186-206) of a dump.
int ref_tables_load(const char* path, void** out, int* w, int* h, int* b) {
  return guarded([&] {
    IntegralTableSet t = IntegralTableSet::load_file(path);
    *w = t.width();
    *h = t.height();
    *b = t.bins();
    *out = new Tables{FeatureImage(1, 1, 1), std::move(t)};
  });
}

// Harness outputs (matching.cpp:225-252, pgm.cpp, bench.cpp:132-143).
int ref_write_map_files(const double* scores, int mw, int mh, int hx, int hy,
                        const char* csv_path, const char* pgm_path) {
  return guarded([&] {
    LikelihoodMap map;
    map.width = mw;
    map.height = mh;
    map.hx = hx;
    map.hy = hy;
    map.scores.assign(scores, scores + std::size_t(mw) * mh);
    if (csv_path) write_map_csv_file(map, csv_path);
    if (pgm_path) write_pgm_file(map_to_gray(map), pgm_path);
  });
}

int ref_write_bench_csv(const char* method, int w, int h, int kw, int kh, int bins,
                        double build_ms, double total_ms, double mean_us, const char* path) {
  return guarded([&] {
    BenchRecord r;
    r.method = method;
    r.width = w;
    r.height = h;
    r.kw = kw;
    r.kh = kh;
    r.bins = bins;
    r.build_ms = build_ms;
    r.query_total_ms = total_ms;
    r.query_mean_us = mean_us;
    std::ofstream out(path, std::ios::binary);
    write_bench_csv_header(out);
    write_bench_csv_row(r, out);
  });
}

int ref_swih_query(void* tv, int cx, int cy, int kind, int kw, int kh,
                   double sigma, int border, std::int64_t* out) {
  return guarded([&] {
    const IntegralTableSet& t = static_cast<Tables*>(tv)->t;
    swih_query_into(t,
                    {cx, cy, mk(kind, kw, kh, sigma),
                     static_cast<BorderPolicy>(border)},
                    std::span<std::int64_t>(out, t.bins()));
  });
}

int ref_plain_query(void* tv, int cx, int cy, int kw, int kh, int border,
                    std::int64_t* out) {
  return guarded([&] {
    const IntegralTableSet& t = static_cast<Tables*>(tv)->t;
    plain_local_histogram_into(
        t, {cx, cy, mk(0, kw, kh, 0.5), static_cast<BorderPolicy>(border)},
        std::span<std::int64_t>(out, t.bins()));
  });
}

int ref_quadrant_histogram(void* tv, int valid, int x0, int y0, int x1, int y1,
                           std::int64_t sx, std::int64_t sy, std::int64_t beta,
                           double* out) {
  return guarded([&] {
    const IntegralTableSet& t = static_cast<Tables*>(tv)->t;
    std::optional<RectRegion> r;
    if (valid) r = RectRegion{x0, y0, x1, y1};
    const WeightedHistogram h = quadrant_histogram(t, r, sx, sy, beta);
    for (int i = 0; i < h.bins(); ++i) out[i] = h.value(i);
  });
}

int ref_cake_histogram(void* tv, int kind, int kw, int kh, double sigma,
                       int rings, int rule, int cx, int cy, int border,
                       double* out) {
  return guarded([&] {
    const IntegralTableSet& t = static_cast<Tables*>(tv)->t;
    const WeddingCakePlan plan(mk(kind, kw, kh, sigma),
                               {rings, static_cast<RingRule>(rule)});
    plan.histogram_into(t, cx, cy, static_cast<BorderPolicy>(border),
                        std::span<double>(out, t.bins()));
  });
}

int ref_cake_plan(int kind, int kw, int kh, double sigma, int rings, int rule,
                  int* sx, int* sy, double* rw) {
  return guarded([&] {
    const WeddingCakePlan plan(mk(kind, kw, kh, sigma),
                               {rings, static_cast<RingRule>(rule)});
    for (int i = 0; i < plan.rings(); ++i) {
      sx[i] = plan.shrink_x(i);
      sy[i] = plan.shrink_y(i);
      rw[i] = plan.ring_weight(i);
    }
  });
}

int ref_brute_counts(const std::uint16_t* fi, int w, int h, int b, int cx,
                     int cy, int kind, int kw, int kh, double sigma, int border,
                     std::int64_t* out) {
  return guarded([&] {
    const FeatureImage f = to_fi(fi, w, h, b);
    const BruteForcePlan plan(mk(kind, kw, kh, sigma));
    plan.counts_into(f, cx, cy, static_cast<BorderPolicy>(border),
                     std::span<std::int64_t>(out, b));
  });
}

int ref_brute_weights(const std::uint16_t* fi, int w, int h, int b, int cx,
                      int cy, int kind, int kw, int kh, double sigma,
                      int border, double* out) {
  return guarded([&] {
    const FeatureImage f = to_fi(fi, w, h, b);
    const BruteForcePlan plan(mk(kind, kw, kh, sigma));
    plan.weights_into(f, cx, cy, static_cast<BorderPolicy>(border),
                      std::span<double>(out, b));
  });
}

int ref_similarity(int sim, const double* p, const double* q, int b,
                   double* out) {
  return guarded([&] {
    *out = similarity(static_cast<SimilarityKind>(sim),
                      std::span<const double>(p, b),
                      std::span<const double>(q, b));
  });
}

int ref_normalize(const double* in, int b, double* out) {
  return guarded([&] {
    const WeightedHistogram h =
        normalize(WeightedHistogram(std::vector<double>(in, in + b), false));
    for (int i = 0; i < b; ++i) out[i] = h.value(i);
  });
}

int ref_target_model(const std::uint8_t* templ, int tw, int th, int bins,
                     int kind, int kw, int kh, double sigma, int method,
                     int rings, int rule, double* out) {
  return guarded([&] {
    const WeightedHistogram m = target_model_for_method(
        to_gray(templ, tw, th), Quantizer(bins), mk(kind, kw, kh, sigma),
        static_cast<MapMethod>(method), {rings, static_cast<RingRule>(rule)});
    for (int i = 0; i < m.bins(); ++i) out[i] = m.value(i);
  });
}

// Public-API path: likelihood_map (matching.cpp:108-209) + peak (211-223).
int ref_likelihood_map(const std::uint8_t* px, int w, int h, int bins,
                       const double* model, int model_normalized, int kind,
                       int kw, int kh, double sigma, int method, int sim,
                       int rings, int rule, int threads, std::size_t budget,
                       double* scores, int* peak_xy, double* peak_score) {
  return guarded([&] {
    MatchOptions opt;
    opt.sim = static_cast<SimilarityKind>(sim);
    opt.cake = {rings, static_cast<RingRule>(rule)};
    opt.threads = threads;
    if (budget) opt.tables.memory_budget_bytes = budget;
    const WeightedHistogram mh(std::vector<double>(model, model + bins),
                               model_normalized != 0);
    const LikelihoodMap map =
        likelihood_map(to_gray(px, w, h), mh, Quantizer(bins),
                       mk(kind, kw, kh, sigma), static_cast<MapMethod>(method),
                       opt);
    if (scores)
      std::memcpy(scores, map.scores.data(), map.scores.size() * sizeof(double));
    if (peak_xy) {
      const Peak p = peak(map);
      peak_xy[0] = p.map_x;
      peak_xy[1] = p.map_y;
      peak_xy[2] = p.center_x;
      peak_xy[3] = p.center_y;
      *peak_score = p.score;
    }
  });
}

int ref_peak(const double* scores, int mw, int mh, int hx, int hy,
             int* peak_xy, double* peak_score) {
  return guarded([&] {
    LikelihoodMap map;
    map.width = mw;
    map.height = mh;
    map.hx = hx;
    map.hy = hy;
    map.scores.assign(scores, scores + std::size_t(mw) * mh);
    const Peak p = peak(map);
    peak_xy[0] = p.map_x;
    peak_xy[1] = p.map_y;
    peak_xy[2] = p.center_x;
    peak_xy[3] = p.center_y;
    *peak_score = p.score;
  });
}

// "Best-use" CPU path: one reference build_tables, then
// per-window reference queries (swih_query_into / plain / WeddingCakePlan /
// BruteForcePlan) + the restated scorer over `threads` row chunks.  Map rows
// [v0, v1) of the strict map are written to scores[(v - v0) * mw + u].
int ref_sweep_rows(void* tv, const double* model, int kind, int kw, int kh,
                   double sigma, int method, int sim, int rings, int rule,
                   int threads, int v0, int v1, double* scores) {
  return guarded([&] {
    const Tables& T = *static_cast<Tables*>(tv);
    const IntegralTableSet& t = T.t;
    const KernelSpec k = mk(kind, kw, kh, sigma);
    validate_kernel(k);
    const int b = t.bins();
    const int mw = t.width() - kw + 1;
    const int hx = k.hx(), hy = k.hy();
    std::optional<WeddingCakePlan> cake;
    if (method == 2) cake.emplace(k, WeddingCakeConfig{rings, static_cast<RingRule>(rule)});
    const BruteForcePlan brute(k);
    const KernelSpec uni{KernelKind::Uniform, kw, kh, 0.5};
    auto work = [&](int a, int e) {
      std::vector<std::int64_t> counts(b);
      std::vector<double> weights(b);
      for (int v = a; v < e; ++v)
        for (int u = 0; u < mw; ++u) {
          const int cx = u + hx, cy = v + hy;
          double s = 0.0;
          switch (method) {
            case 0:
              swih_query_into(t, {cx, cy, k, BorderPolicy::Strict}, counts);
              s = score_counts_r(sim, model, counts.data(), b);
              break;
            case 3:
              plain_local_histogram_into(t, {cx, cy, uni, BorderPolicy::Strict},
                                         counts);
              s = score_counts_r(sim, model, counts.data(), b);
              break;
            case 2:
              cake->histogram_into(t, cx, cy, BorderPolicy::Strict, weights);
              s = score_weights_r(sim, model, weights.data(), b);
              break;
            default:
              if (k.integer_weighted()) {
                brute.counts_into(T.fi, cx, cy, BorderPolicy::Strict, counts);
                s = score_counts_r(sim, model, counts.data(), b);
              } else {
                brute.weights_into(T.fi, cx, cy, BorderPolicy::Strict, weights);
                s = score_weights_r(sim, model, weights.data(), b);
              }
          }
          scores[std::size_t(v - v0) * mw + u] = s;
        }
    };
    const int rows = v1 - v0;
    int nt = std::clamp(threads, 1, std::max(rows, 1));
    if (nt <= 1) {
      work(v0, v1);
      return;
    }
    std::vector<std::thread> pool;
    const int chunk = (rows + nt - 1) / nt;
    for (int i = 0; i < nt; ++i) {
      const int a = v0 + i * chunk, e = std::min(v1, a + chunk);
      if (a >= e) break;
      pool.emplace_back(work, a, e);
    }
    for (auto& th : pool) th.join();
  });
}

}  // extern "C"
