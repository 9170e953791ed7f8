// engine.cpp — window validation, quadrant decomposition and GPU window
// queries (reference bodies: src/engine.cpp:7-165).
#include <string>
#include <vector>

#include "runtime.hpp"
#include "swih/engine.hpp"

namespace swih {

namespace {

swg_kernel to_swg(const KernelSpec& k) { return swg_kernel{int(k.kind), k.kw, k.kh, k.sigma}; }

void query(const IntegralTableSet& t, const WindowQuery& q, int method,
           std::span<std::int64_t> out) {
  if (out.size() != std::size_t(t.bins()))
    throw OutOfRangeError("window query: output has " + std::to_string(out.size()) +
                          " bins, tables have " + std::to_string(t.bins()));
  const swg_kernel k = to_swg(q.kernel);
  detail::check(swg_query_windows(t.device(), 1, &q.cx, &q.cy, &k, method, int(q.border),
                                  out.data()));
}

}  // namespace

void validate_window(int width, int height, const WindowQuery& q) {
  validate_kernel(q.kernel);
  const int hx = q.kernel.hx(), hy = q.kernel.hy();
  const auto where = "(" + std::to_string(q.cx) + "," + std::to_string(q.cy) + ")";
  if (q.border == BorderPolicy::Strict) {
    if (q.cx < hx || q.cx + hx >= width || q.cy < hy || q.cy + hy >= height)
      throw WindowOutOfBoundsError("strict window " + std::to_string(q.kernel.kw) + "x" +
                                   std::to_string(q.kernel.kh) + " at " + where +
                                   " does not fit inside " + std::to_string(width) + "x" +
                                   std::to_string(height));
  } else if (q.cx < 0 || q.cx >= width || q.cy < 0 || q.cy >= height) {
    throw WindowOutOfBoundsError("clipped window center " + where + " outside image");
  }
}

QuadrantDecomposition decompose(const WindowQuery& q) {
  validate_kernel(q.kernel);
  if (!q.kernel.quadrant_affine())
    throw UnsupportedKernelError(
        "decompose: kernel kind is not quadrant-affine; use the wedding-cake or brute-force "
        "baseline");
  const int hx = q.kernel.hx(), hy = q.kernel.hy(), x = q.cx, y = q.cy;
  QuadrantDecomposition d;
  d.tl.rect = RectRegion{x - hx, y - hy, x, y};
  if (hx > 0) d.tr.rect = RectRegion{x + 1, y - hy, x + hx, y};
  if (hy > 0) d.bl.rect = RectRegion{x - hx, y + 1, x, y + hy};
  if (hx > 0 && hy > 0) d.br.rect = RectRegion{x + 1, y + 1, x + hx, y + hy};
  if (q.kernel.kind == KernelKind::Uniform) {
    d.tl.beta = d.tr.beta = d.bl.beta = d.br.beta = 1;
    return d;
  }
  // weight = M - |x-cx| - |y-cy|, M = hx+hy+1: affine once the signs are fixed
  const std::int64_t m = hx + hy + 1;
  d.tl = {d.tl.rect, +1, +1, m - x - y};
  d.tr = {d.tr.rect, -1, +1, m + x - y};
  d.bl = {d.bl.rect, +1, -1, m - x + y};
  d.br = {d.br.rect, -1, -1, m + x + y};
  return d;
}

WeightedHistogram quadrant_histogram(const IntegralTableSet& t,
                                     const std::optional<RectRegion>& rect, std::int64_t sx,
                                     std::int64_t sy, std::int64_t beta) {
  std::vector<std::int64_t> acc(std::size_t(t.bins()), 0);
  if (rect) {
    const RectRegion& r = *rect;
    if (r.x0 < 0 || r.y0 < 0 || r.x0 > r.x1 || r.y0 > r.y1 || r.x1 >= t.width() ||
        r.y1 >= t.height())
      throw OutOfRangeError("rect_sum: rectangle (" + std::to_string(r.x0) + "," +
                            std::to_string(r.y0) + ")-(" + std::to_string(r.x1) + "," +
                            std::to_string(r.y1) + ") out of bounds for " +
                            std::to_string(t.width()) + "x" + std::to_string(t.height()));
    const swg_term term{1, r.x0, r.y0, r.x1, r.y1, sx, sy, beta};
    detail::check(swg_query_terms(t.device(), 1, 1, &term, acc.data()));
  }
  return WeightedHistogram::from_counts(acc);
}

void swih_query_into(const IntegralTableSet& t, const WindowQuery& q,
                     std::span<std::int64_t> out) {
  query(t, q, SWG_METHOD_SWIH, out);
}

WeightedHistogram swih_query(const IntegralTableSet& t, const WindowQuery& q) {
  std::vector<std::int64_t> acc(std::size_t(t.bins()));
  swih_query_into(t, q, acc);
  return WeightedHistogram::from_counts(acc);
}

void plain_local_histogram_into(const IntegralTableSet& t, const WindowQuery& q,
                                std::span<std::int64_t> out) {
  query(t, q, SWG_METHOD_PLAIN, out);
}

WeightedHistogram plain_local_histogram(const IntegralTableSet& t, const WindowQuery& q) {
  std::vector<std::int64_t> acc(std::size_t(t.bins()));
  plain_local_histogram_into(t, q, acc);
  return WeightedHistogram::from_counts(acc);
}

}  // namespace swih
