// core.cpp — errors, device context, images, kernels and histograms of the
// C++ API (reference bodies: src/image.cpp, src/kernel.cpp,
// src/histogram.cpp).  Kernel formulas are the host-side plan constants;
// quantisation of images runs on the GPU.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>

#include "runtime.hpp"
#include "swih/errors.hpp"
#include "swih/histogram.hpp"
#include "swih/image.hpp"
#include "swih/kernel.hpp"

namespace swih {

namespace detail {

void raise(int status) {
  const std::string msg = swg_last_error();
  switch (status) {
    case SWG_OK: return;
    case SWG_ERR_IO: throw IoError(msg);
    case SWG_ERR_ZERO_MASS: throw ZeroMassError(msg);
    case SWG_ERR_INVALID_KERNEL: throw InvalidKernelError(msg);
    case SWG_ERR_OUT_OF_RANGE: throw OutOfRangeError(msg);
    case SWG_ERR_UNSUPPORTED_KERNEL: throw UnsupportedKernelError(msg);
    case SWG_ERR_WINDOW_OOB: throw WindowOutOfBoundsError(msg);
    case SWG_ERR_CAPACITY: throw CapacityError(msg, swg_last_required_bytes());
    case SWG_ERR_CONFIG: throw ConfigError(msg);
    case SWG_ERR_MODEL: throw ModelError(msg);
    case SWG_ERR_SIZE: throw SizeError(msg);
    default: throw Error("swih (GPU): " + msg);
  }
}

swg_ctx* context() {
  static std::once_flag once;
  static swg_ctx* ctx = nullptr;
  static int status = SWG_OK;
  std::call_once(once, [] {
    const char* env = std::getenv("SWIH_GPU");
    status = swg_ctx_create(env ? std::atoi(env) : 0, &ctx);
  });
  if (!ctx) raise(status == SWG_OK ? SWG_ERR_NO_DEVICE : status);
  return ctx;
}

}  // namespace detail

// ---- image.hpp (image.cpp:7-40) -------------------------------------------
GrayImage::GrayImage(int width, int height, std::uint8_t fill) : w_(width), h_(height) {
  if (width < 1 || height < 1) throw Error("GrayImage: dimensions must be >= 1");
  px_.assign(std::size_t(width) * height, fill);
}

GrayImage::GrayImage(int width, int height, std::vector<std::uint8_t> pixels)
    : w_(width), h_(height), px_(std::move(pixels)) {
  if (width < 1 || height < 1) throw Error("GrayImage: dimensions must be >= 1");
  if (px_.size() != std::size_t(width) * height)
    throw Error("GrayImage: pixel count does not match dimensions");
}

Quantizer::Quantizer(int bins) : bins_(bins) {
  if (bins < 1) throw Error("Quantizer: bin count must be >= 1");
}

FeatureImage::FeatureImage(int width, int height, int bins)
    : w_(width), h_(height), bins_(bins) {
  if (width < 1 || height < 1) throw Error("FeatureImage: dimensions must be >= 1");
  if (bins < 1) throw Error("FeatureImage: bin count must be >= 1");
  data_.assign(std::size_t(width) * height, 0);
}

FeatureImage quantize_image(const GrayImage& img, const Quantizer& q) {
  FeatureImage fi(img.width(), img.height(), q.bins());
  detail::check(swg_quantize(detail::context(), img.pixels().data(), img.width(),
                             img.height(), SWG_FMT_GRAY8, q.bins(), fi.data()));
  return fi;
}

// ---- kernel.hpp (kernel.cpp:10-83) ----------------------------------------
void validate_kernel(const KernelSpec& k) {
  if (k.kw < 1 || k.kh < 1) throw InvalidKernelError("kernel: dimensions must be >= 1");
  if (k.kw % 2 == 0 || k.kh % 2 == 0)
    throw InvalidKernelError("kernel: dimensions must be odd, got " + std::to_string(k.kw) +
                             "x" + std::to_string(k.kh));
  if (k.kind == KernelKind::GaussianChebyshev && !(k.sigma > 0.0))
    throw InvalidKernelError("kernel: sigma must be positive");
}

int manhattan_distance(int px, int py, int cx, int cy) noexcept {
  return std::abs(px - cx) + std::abs(py - cy);
}

double weight_at(const KernelSpec& k, int dx, int dy) {
  validate_kernel(k);
  const int hx = k.hx(), hy = k.hy();
  const int ax = std::abs(dx), ay = std::abs(dy);
  if (ax > hx || ay > hy)
    throw OutOfRangeError("kernel: offset (" + std::to_string(dx) + "," + std::to_string(dy) +
                          ") outside " + std::to_string(k.kw) + "x" + std::to_string(k.kh));
  switch (k.kind) {
    case KernelKind::Uniform:
      return 1.0;
    case KernelKind::ManhattanLinear:
      return double((hx + hy + 1) - (ax + ay));
    case KernelKind::ChebyshevLinear: {
      const int top = std::max(hx, hy);  // both axes scaled to the larger extent
      const double sx = double(ax) * top / std::max(hx, 1);
      const double sy = double(ay) * top / std::max(hy, 1);
      return double(top + 1 - std::lround(std::max(sx, sy)));
    }
    case KernelKind::GaussianChebyshev: {
      const double nx = double(ax) / std::max(hx, 1), ny = double(ay) / std::max(hy, 1);
      const double r = std::max(nx, ny);
      return std::exp(-(r * r) / (2.0 * k.sigma * k.sigma));
    }
  }
  throw InvalidKernelError("kernel: unknown kind");
}

double kernel_weight_sum(const KernelSpec& k) {
  validate_kernel(k);
  const std::int64_t hx = k.hx(), hy = k.hy(), area = std::int64_t(k.kw) * k.kh;
  if (k.kind == KernelKind::Uniform) return double(area);
  if (k.kind == KernelKind::ManhattanLinear)
    return double(area * (hx + hy + 1) - k.kh * (hx * (hx + 1)) - k.kw * (hy * (hy + 1)));
  double s = 0.0;
  for (int dy = -k.hy(); dy <= k.hy(); ++dy)
    for (int dx = -k.hx(); dx <= k.hx(); ++dx) s += weight_at(k, dx, dy);
  return s;
}

// ---- histogram.hpp (histogram.cpp:5-26) -----------------------------------
WeightedHistogram WeightedHistogram::from_counts(std::span<const std::int64_t> counts) {
  std::vector<double> v(counts.size());
  std::transform(counts.begin(), counts.end(), v.begin(),
                 [](std::int64_t c) { return double(c); });
  return WeightedHistogram(std::move(v), false);
}

double WeightedHistogram::sum() const noexcept {
  double s = 0.0;
  for (double x : v_) s += x;
  return s;
}

WeightedHistogram normalize(const WeightedHistogram& h) {
  const double mass = h.sum();
  if (mass == 0.0) throw ZeroMassError("normalize: histogram has zero mass");
  std::vector<double> v(h.values().begin(), h.values().end());
  for (double& x : v) x /= mass;
  return WeightedHistogram(std::move(v), true);
}

}  // namespace swih
