// bench.cpp — the timing harness over the GPU path (reference API
// include/swih/bench.hpp; reference bodies src/bench.cpp:28-143).
//
// build_ms: the device table build of the feature image, host clock until
// the tables are ready.  query_total_ms: one full sweep over every strict
// centre -- each window's weighted histogram formed on the device and folded
// into a score in registers (the likelihood-map sweep with a flat model; the
// histograms are never written to HBM) -- host clock until the sweep's peak
// is back, median of `repetitions`.
#include "swih/bench.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <ostream>
#include <random>

#include "runtime.hpp"
#include "swih/integral_tables.hpp"

namespace swih {

namespace {

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

}  // namespace

GrayImage random_image(int width, int height, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  GrayImage img(width, height);
  for (auto& p : img.pixels()) p = std::uint8_t(rng() % 256);
  return img;
}

const char* method_name(MapMethod m) {
  switch (m) {
    case MapMethod::Swih: return "swih";
    case MapMethod::Brute: return "brute";
    case MapMethod::Cake: return "cake";
    case MapMethod::Plain: return "plain";
  }
  return "?";
}

BenchRecord bench_sweep(const FeatureImage& fi, MapMethod method, const KernelSpec& kernel,
                        const BenchConfig& cfg) {
  validate_kernel(kernel);
  if (kernel.kw > fi.width() || kernel.kh > fi.height())
    throw SizeError("bench: kernel larger than image");
  if (method == MapMethod::Swih && !kernel.quadrant_affine())
    throw UnsupportedKernelError("bench: method swih requires a quadrant-affine kernel");
  BenchRecord rec;
  rec.method = method_name(method);
  rec.width = fi.width();
  rec.height = fi.height();
  rec.kw = kernel.kw;
  rec.kh = kernel.kh;
  rec.bins = fi.bins();
  const double centres = double(fi.width() - kernel.kw + 1) * (fi.height() - kernel.kh + 1);

  swg_ctx* ctx = detail::context();
  swg_tables* dev = nullptr;
  if (method != MapMethod::Brute) {
    const std::size_t need =
        3 * std::size_t(fi.width() + 1) * (fi.height() + 1) * fi.bins() * 8;
    if (need > cfg.tables.memory_budget_bytes)
      throw CapacityError("integral tables need " + std::to_string(need) +
                              " bytes, budget is " +
                              std::to_string(cfg.tables.memory_budget_bytes),
                          need);
  }
  const auto t0 = Clock::now();
  detail::check(swg_tables_build(ctx, fi.data(), 0, 0, fi.width(), fi.height(), SWG_FMT_BINS16,
                                 fi.bins(),
                                 method == MapMethod::Swih ? SWG_PLANES_AFFINE : SWG_PLANES_PLAIN,
                                 0, &dev));
  struct Guard {
    swg_tables* t;
    ~Guard() { swg_tables_destroy(t); }
  } guard{dev};
  detail::check(swg_ctx_synchronize(ctx));
  // brute force reads only the feature image the build uploaded
  if (method != MapMethod::Brute) rec.build_ms = ms_since(t0);

  const std::vector<double> flat(std::size_t(fi.bins()), 1.0 / fi.bins());
  swg_map_request req{};
  req.kernel = swg_kernel{int(kernel.kind), kernel.kw, kernel.kh, kernel.sigma};
  req.method = int(method);
  req.sim = SWG_SIM_BHATTACHARYYA;
  req.rings = cfg.cake.rings;
  req.ring_rule = int(cfg.cake.rule);
  req.model = flat.data();
  auto sweep = [&] {
    swg_peak pk{};
    detail::check(swg_likelihood_maps(dev, 1, &req, nullptr, nullptr, &pk, nullptr));
  };
  if (cfg.warmup) sweep();
  std::vector<double> times;
  for (int r = 0; r < std::max(cfg.repetitions, 1); ++r) {
    const auto t1 = Clock::now();
    sweep();
    times.push_back(ms_since(t1));
  }
  std::sort(times.begin(), times.end());
  rec.query_total_ms = times[times.size() / 2];
  rec.query_mean_us = rec.query_total_ms * 1000.0 / centres;
  return rec;
}

void write_bench_csv_header(std::ostream& out) {
  out << "method,width,height,kw,kh,bins,build_ms,query_total_ms,query_mean_us\n";
}

void write_bench_csv_row(const BenchRecord& r, std::ostream& out) {
  char t[128];
  std::snprintf(t, sizeof t, "%.6f,%.6f,%.4f", r.build_ms, r.query_total_ms, r.query_mean_us);
  out << r.method << ',' << r.width << ',' << r.height << ',' << r.kw << ',' << r.kh << ','
      << r.bins << ',' << t << '\n';
}

}  // namespace swih
