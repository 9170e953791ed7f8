// matching.cpp — baselines and matching over the GPU (reference bodies:
// src/baselines.cpp:8-160, src/matching.cpp:56-252).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <ostream>
#include <string>

#include "runtime.hpp"
#include "swih/matching.hpp"

namespace swih {

namespace {

swg_kernel to_swg(const KernelSpec& k) { return swg_kernel{int(k.kind), k.kw, k.kh, k.sigma}; }

double clamp01(double v) { return std::clamp(v, 0.0, 1.0); }

}  // namespace

// ---- baselines --------------------------------------------------------------
BruteForcePlan::BruteForcePlan(const KernelSpec& kernel) : kernel_(kernel) {
  validate_kernel(kernel);
}

void BruteForcePlan::counts_into(const FeatureImage& fi, int cx, int cy, BorderPolicy border,
                                 std::span<std::int64_t> out) const {
  if (!kernel_.integer_weighted())
    throw InvalidKernelError("brute force counts: kernel weights are not integers");
  validate_window(fi.width(), fi.height(), {cx, cy, kernel_, border});
  if (out.size() != std::size_t(fi.bins())) throw OutOfRangeError("brute force: bin count");
  const swg_kernel k = to_swg(kernel_);
  detail::check(swg_brute_windows(detail::context(), fi.data(), fi.width(), fi.height(),
                                  fi.bins(), 1, &cx, &cy, &k, int(border), out.data(),
                                  nullptr));
}

void BruteForcePlan::weights_into(const FeatureImage& fi, int cx, int cy, BorderPolicy border,
                                  std::span<double> out) const {
  validate_window(fi.width(), fi.height(), {cx, cy, kernel_, border});
  if (out.size() != std::size_t(fi.bins())) throw OutOfRangeError("brute force: bin count");
  const swg_kernel k = to_swg(kernel_);
  detail::check(swg_brute_windows(detail::context(), fi.data(), fi.width(), fi.height(),
                                  fi.bins(), 1, &cx, &cy, &k, int(border), nullptr,
                                  out.data()));
}

WeightedHistogram brute_force_histogram(const FeatureImage& fi, const WindowQuery& q) {
  const BruteForcePlan plan(q.kernel);
  if (q.kernel.integer_weighted()) {
    std::vector<std::int64_t> acc(std::size_t(fi.bins()));
    plan.counts_into(fi, q.cx, q.cy, q.border, acc);
    return WeightedHistogram::from_counts(acc);
  }
  std::vector<double> acc(std::size_t(fi.bins()));
  plan.weights_into(fi, q.cx, q.cy, q.border, acc);
  return WeightedHistogram(std::move(acc), false);
}

WeddingCakePlan::WeddingCakePlan(const KernelSpec& kernel, const WeddingCakeConfig& cfg)
    : kernel_(kernel), rule_(cfg.rule) {
  validate_kernel(kernel);
  const int m = cfg.rings;
  const int limit = std::min(kernel.hx(), kernel.hy()) + 1;
  if (m < 1 || m > limit)
    throw ConfigError("wedding cake: ring count " + std::to_string(m) + " outside [1, " +
                      std::to_string(limit) + "] for " + std::to_string(kernel.kw) + "x" +
                      std::to_string(kernel.kh));
  shrink_x_.resize(std::size_t(m));
  shrink_y_.resize(std::size_t(m));
  ring_weight_.resize(std::size_t(m));
  const swg_kernel k = to_swg(kernel);
  detail::check(swg_cake_plan(&k, m, int(cfg.rule), shrink_x_.data(), shrink_y_.data(),
                              ring_weight_.data()));
}

void WeddingCakePlan::histogram_into(const IntegralTableSet& t, int cx, int cy,
                                     BorderPolicy border, std::span<double> out) const {
  if (out.size() != std::size_t(t.bins())) throw OutOfRangeError("wedding cake: bin count");
  const swg_kernel k = to_swg(kernel_);
  detail::check(swg_cake_windows(t.device(), 1, &cx, &cy, &k, rings(), int(rule_), int(border),
                                 out.data()));
}

WeightedHistogram wedding_cake_histogram(const IntegralTableSet& t, const WindowQuery& q,
                                         const WeddingCakeConfig& cfg) {
  const WeddingCakePlan plan(q.kernel, cfg);
  std::vector<double> acc(std::size_t(t.bins()));
  plan.histogram_into(t, q.cx, q.cy, q.border, acc);
  return WeightedHistogram(std::move(acc), false);
}

// ---- matching ---------------------------------------------------------------
double similarity(SimilarityKind kind, std::span<const double> p, std::span<const double> q) {
  if (p.size() != q.size()) throw ModelError("similarity: histogram sizes differ");
  double s = 0.0;
  for (std::size_t b = 0; b < p.size(); ++b)
    s += kind == SimilarityKind::Bhattacharyya ? std::sqrt(p[b] * q[b]) : std::min(p[b], q[b]);
  return clamp01(s);
}

WeightedHistogram target_model(const GrayImage& templ, const Quantizer& q,
                               const KernelSpec& kernel) {
  validate_kernel(kernel);
  if (templ.width() != kernel.kw || templ.height() != kernel.kh)
    throw ModelError("target model: template " + std::to_string(templ.width()) + "x" +
                     std::to_string(templ.height()) + " does not match kernel " +
                     std::to_string(kernel.kw) + "x" + std::to_string(kernel.kh));
  const FeatureImage fi = quantize_image(templ, q);
  return normalize(brute_force_histogram(fi, {kernel.hx(), kernel.hy(), kernel,
                                              BorderPolicy::Strict}));
}

WeightedHistogram target_model_for_method(const GrayImage& templ, const Quantizer& q,
                                          const KernelSpec& kernel, MapMethod method,
                                          const WeddingCakeConfig& cake) {
  if (method == MapMethod::Plain)
    return target_model(templ, q, {KernelKind::Uniform, kernel.kw, kernel.kh, 0.5});
  if (method != MapMethod::Cake) return target_model(templ, q, kernel);
  validate_kernel(kernel);
  if (templ.width() != kernel.kw || templ.height() != kernel.kh)
    throw ModelError("target model: template does not match kernel");
  const IntegralTableSet t = build_tables(quantize_image(templ, q));
  return normalize(
      wedding_cake_histogram(t, {kernel.hx(), kernel.hy(), kernel, BorderPolicy::Strict}, cake));
}

LikelihoodMap likelihood_map(const GrayImage& search, const WeightedHistogram& model,
                             const Quantizer& q, const KernelSpec& kernel, MapMethod method,
                             const MatchOptions& opt) {
  validate_kernel(kernel);
  if (search.width() < kernel.kw || search.height() < kernel.kh)
    throw SizeError("likelihood map: kernel " + std::to_string(kernel.kw) + "x" +
                    std::to_string(kernel.kh) + " larger than search image " +
                    std::to_string(search.width()) + "x" + std::to_string(search.height()));
  if (model.bins() != q.bins() || !model.normalized())
    throw ModelError("likelihood map: model must be normalized with " +
                     std::to_string(q.bins()) + " bins");
  if (method == MapMethod::Swih && !kernel.quadrant_affine())
    throw UnsupportedKernelError("likelihood map: method swih requires a quadrant-affine kernel");
  if (method != MapMethod::Brute) {  // the reference builds int64 tables here
    const std::size_t need =
        3 * std::size_t(search.width() + 1) * (search.height() + 1) * q.bins() * 8;
    if (need > opt.tables.memory_budget_bytes)
      throw CapacityError("integral tables need " + std::to_string(need) +
                              " bytes, budget is " +
                              std::to_string(opt.tables.memory_budget_bytes),
                          need);
  }
  // GPU: quantise + build (ramp planes only for the Manhattan quadrant path),
  // sweep every strict centre, score, reduce the peak.
  const bool ramps = kernel.kind == KernelKind::ManhattanLinear &&
                     (method == MapMethod::Swih || method == MapMethod::Brute);
  swg_tables* dev = nullptr;
  detail::check(swg_tables_build(detail::context(), search.pixels().data(), 0, 0,
                                 search.width(), search.height(), SWG_FMT_GRAY8, q.bins(),
                                 ramps ? SWG_PLANES_AFFINE : SWG_PLANES_PLAIN, 0, &dev));
  struct Guard {
    swg_tables* t;
    ~Guard() { swg_tables_destroy(t); }
  } guard{dev};

  LikelihoodMap map;
  map.width = search.width() - kernel.kw + 1;
  map.height = search.height() - kernel.kh + 1;
  map.hx = kernel.hx();
  map.hy = kernel.hy();
  map.scores.resize(std::size_t(map.width) * map.height);
  const std::vector<double> mv(model.values().begin(), model.values().end());
  swg_map_request req{};
  req.kernel = to_swg(kernel);
  req.method = int(method);
  req.sim = int(opt.sim);
  req.rings = opt.cake.rings;
  req.ring_rule = int(opt.cake.rule);
  req.model = mv.data();
  double* host[1] = {map.scores.data()};
  swg_peak pk{};
  detail::check(swg_likelihood_maps(dev, 1, &req, host, nullptr, &pk, nullptr));
  return map;
}

Peak peak(const LikelihoodMap& map) {
  if (map.scores.empty()) throw Error("peak: empty likelihood map");
  swg_peak p{};
  detail::check(swg_map_peak(detail::context(), map.scores.data(), map.width, map.height,
                             map.hx, map.hy, &p));
  return Peak{p.map_x, p.map_y, p.center_x, p.center_y, p.score};
}

GrayImage map_to_gray(const LikelihoodMap& map) {
  GrayImage img(map.width, map.height);
  for (int v = 0; v < map.height; ++v)
    for (int u = 0; u < map.width; ++u)
      img.set(u, v, std::uint8_t(std::lround(clamp01(map.at(u, v)) * 255.0)));
  return img;
}

void write_map_csv(const LikelihoodMap& map, std::ostream& out) {
  char buf[40];
  for (int v = 0; v < map.height; ++v) {
    for (int u = 0; u < map.width; ++u) {
      std::snprintf(buf, sizeof buf, "%.9g", map.at(u, v));
      out << (u ? "," : "") << buf;
    }
    out << '\n';
  }
  if (!out) throw IoError("map csv: write failed");
}

void write_map_csv_file(const LikelihoodMap& map, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoError("map csv: cannot open '" + path + "'");
  write_map_csv(map, out);
}

}  // namespace swih
