// test_api.cpp — the reference API's behaviour, exercised through the
// GPU-backed C++ layer (include/swih/*.hpp -> libswg).  The cases restate the
// properties and known answers of the reference's own suites
// (/root/reference/proj/tests/test_*.cpp, cited per case); the code is ours.
#include <algorithm>
#include <cmath>
#include <random>
#include <sstream>
#include <thread>

#include "minitest.hpp"
#include "swih/baselines.hpp"
#include "swih/engine.hpp"
#include "swih/integral_tables.hpp"
#include "swih/matching.hpp"

using namespace swih;
using minitest::Approx;

namespace {

// 10 200 10 / 200 10 200 / 10 200 10: with 2 bins corners+centre are bin 0.
GrayImage cross3() {
  return GrayImage(3, 3, std::vector<std::uint8_t>{10, 200, 10, 200, 10, 200, 10, 200, 10});
}

GrayImage noise(int w, int h, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  GrayImage img(w, h);
  for (auto& p : img.pixels()) p = std::uint8_t(rng() % 256);
  return img;
}

KernelSpec man(int kw, int kh) { return {KernelKind::ManhattanLinear, kw, kh, 0.5}; }

}  // namespace

// ---------------------------------------------------------------- images
TEST_CASE("quantizer: floor(v*b/256), partition, errors (test_image.cpp:12-41)") {
  CHECK(Quantizer(2).quantize(10) == 0);
  CHECK(Quantizer(2).quantize(200) == 1);
  for (int v = 0; v < 256; ++v) CHECK(Quantizer(256).quantize(std::uint8_t(v)) == v);
  for (int b : {1, 2, 8, 16, 256}) {
    const Quantizer q(b);
    int prev = 0;
    for (int v = 0; v < 256; ++v) {
      const int bin = q.quantize(std::uint8_t(v));
      REQUIRE(bin >= 0 && bin < b && bin >= prev && bin <= prev + 1);
      if (bin != prev) REQUIRE(v == (bin * 256 + b - 1) / b);
      prev = bin;
    }
  }
  CHECK_THROWS_AS(Quantizer(0), Error);
  CHECK_THROWS_AS(GrayImage(0, 4), Error);
  CHECK_THROWS_AS(GrayImage(2, 2, std::vector<std::uint8_t>{1, 2, 3}), Error);
}

TEST_CASE("quantize_image on the GPU matches the quantizer (test_image.cpp:43-55)") {
  GrayImage img(3, 2);
  img.set(0, 0, 255);
  img.set(2, 1, 128);
  const FeatureImage fi = quantize_image(img, Quantizer(2));
  CHECK(fi.width() == 3);
  CHECK(fi.height() == 2);
  CHECK(fi.bins() == 2);
  CHECK(fi.at(0, 0) == 1);
  CHECK(fi.at(2, 1) == 1);
  CHECK(fi.at(1, 0) == 0);
  const GrayImage big = noise(333, 77, 5);
  for (int bins : {3, 16, 255}) {
    const FeatureImage f = quantize_image(big, Quantizer(bins));
    for (int y = 0; y < 77; ++y)
      for (int x = 0; x < 333; ++x) REQUIRE(f.at(x, y) == Quantizer(bins).quantize(big.at(x, y)));
  }
}

TEST_CASE("normalize divides by the mass; idempotent (test_image.cpp:57-86)") {
  const WeightedHistogram n = normalize(WeightedHistogram({7.0, 8.0}, false));
  CHECK(n.normalized());
  CHECK(n.value(0) == Approx(7.0 / 15.0).epsilon(1e-12));
  CHECK(n.value(1) == Approx(8.0 / 15.0).epsilon(1e-12));
  CHECK(normalize(WeightedHistogram({5.0}, false)).value(0) == 1.0);
  CHECK_THROWS_AS(normalize(WeightedHistogram({0.0, 0.0}, false)), ZeroMassError);
  std::mt19937_64 rng(7);
  for (int trial = 0; trial < 50; ++trial) {
    const int bins = 1 + int(rng() % 32);
    WeightedHistogram h(bins);
    for (int b = 0; b < bins; ++b) h.add(b, double(rng() % 1000));
    h.add(int(rng() % bins), 1.0);
    const WeightedHistogram a = normalize(h), b2 = normalize(a);
    for (int b = 0; b < bins; ++b) CHECK(b2.value(b) == Approx(a.value(b)).epsilon(1e-12));
  }
}

// ---------------------------------------------------------------- kernels
TEST_CASE("kernel weights, sums and validation (test_kernel.cpp:26-87)") {
  CHECK(manhattan_distance(3, 4, 1, 1) == 5);
  CHECK(weight_at(man(3, 3), 0, 0) == 3.0);
  CHECK(weight_at(man(3, 3), 1, 1) == 1.0);
  CHECK(weight_at(man(3, 3), -1, 0) == 2.0);
  CHECK(weight_at({KernelKind::ChebyshevLinear, 3, 3, 0.5}, 1, 0) == 1.0);
  CHECK(weight_at({KernelKind::ChebyshevLinear, 3, 3, 0.5}, 0, 0) == 2.0);
  const KernelSpec g{KernelKind::GaussianChebyshev, 5, 5, 0.5};
  CHECK(weight_at(g, 0, 0) == 1.0);
  CHECK(weight_at(g, 2, 1) == Approx(std::exp(-1.0 / 0.5)).epsilon(1e-12));
  CHECK_THROWS_AS(weight_at({KernelKind::Uniform, 4, 3, 0.5}, 0, 0), InvalidKernelError);
  CHECK_THROWS_AS(weight_at(man(3, 0), 0, 0), InvalidKernelError);
  CHECK_THROWS_AS(weight_at({KernelKind::GaussianChebyshev, 3, 3, 0.0}, 0, 0),
                  InvalidKernelError);
  CHECK_THROWS_AS(weight_at(man(3, 3), 2, 0), OutOfRangeError);
  CHECK(kernel_weight_sum(man(3, 3)) == 15.0);
  CHECK(kernel_weight_sum(man(5, 5)) == 65.0);
  CHECK(kernel_weight_sum({KernelKind::Uniform, 5, 7, 0.5}) == 35.0);
  for (const KernelSpec& k : {man(5, 9), man(11, 11), KernelSpec{KernelKind::ChebyshevLinear, 7, 3, 0.5},
                              KernelSpec{KernelKind::GaussianChebyshev, 9, 9, 0.7}}) {
    double direct = 0.0;
    for (int dy = -k.hy(); dy <= k.hy(); ++dy)
      for (int dx = -k.hx(); dx <= k.hx(); ++dx) {
        const double w = weight_at(k, dx, dy);
        direct += w;
        REQUIRE(w > 0.0 && w == weight_at(k, -dx, dy) && w == weight_at(k, dx, -dy));
      }
    CHECK(kernel_weight_sum(k) == Approx(direct).epsilon(1e-12));
  }
}

// ---------------------------------------------------------------- tables
TEST_CASE("tables: single pixel, cross prefixes, zero padding (test_integral_tables.cpp:42-69)") {
  GrayImage one(1, 1);
  one.set(0, 0, 200);
  const IntegralTableSet t1 = build_tables(quantize_image(one, Quantizer(4)));
  CHECK(t1.cell(TableKind::Plain, 1, 1, 3) == 1);
  CHECK(t1.cell(TableKind::XRamp, 1, 1, 3) == 0);
  CHECK(t1.cell(TableKind::Plain, 1, 1, 0) == 0);
  const IntegralTableSet t = build_tables(quantize_image(cross3(), Quantizer(2)));
  CHECK(t.cell(TableKind::Plain, 2, 2, 1) == 2);
  CHECK(t.cell(TableKind::XRamp, 2, 2, 1) == 1);
  CHECK(t.cell(TableKind::YRamp, 2, 2, 1) == 1);
  for (int i = 0; i <= 3; ++i)
    for (int b = 0; b < 2; ++b) {
      CHECK(t.cell(TableKind::Plain, 0, i, b) == 0);
      CHECK(t.cell(TableKind::XRamp, i, 0, b) == 0);
      CHECK(t.cell(TableKind::YRamp, 0, i, b) == 0);
    }
}

TEST_CASE("rect_sum known answers and four-corner vs direct loop (test_integral_tables.cpp:71-110)") {
  const FeatureImage cf = quantize_image(cross3(), Quantizer(2));
  const IntegralTableSet t = build_tables(cf);
  CHECK(t.rect_sum(TableKind::Plain, {0, 0, 2, 2}, 0) + t.rect_sum(TableKind::Plain, {0, 0, 2, 2}, 1) == 9);
  CHECK(t.rect_sum(TableKind::Plain, {0, 0, 1, 1}, 0) == 2);
  for (int y = 0; y < 3; ++y)
    for (int x = 0; x < 3; ++x) {
      const int b = cf.at(x, y);
      CHECK(t.rect_sum(TableKind::Plain, {x, y, x, y}, b) == 1);
      CHECK(t.rect_sum(TableKind::XRamp, {x, y, x, y}, b) == x);
      CHECK(t.rect_sum(TableKind::YRamp, {x, y, x, y}, b) == y);
      CHECK(t.rect_sum(TableKind::Plain, {x, y, x, y}, 1 - b) == 0);
    }
  const FeatureImage fi = quantize_image(noise(32, 32, 99), Quantizer(8));
  const IntegralTableSet r = build_tables(fi);
  std::mt19937_64 rng(100);
  for (int trial = 0; trial < 200; ++trial) {
    const int x0 = int(rng() % 32), x1 = x0 + int(rng() % (32 - x0));
    const int y0 = int(rng() % 32), y1 = y0 + int(rng() % (32 - y0));
    const int b = int(rng() % 8);
    std::int64_t p = 0, sx = 0, sy = 0;
    for (int y = y0; y <= y1; ++y)
      for (int x = x0; x <= x1; ++x)
        if (fi.at(x, y) == b) p += 1, sx += x, sy += y;
    REQUIRE(r.rect_sum(TableKind::Plain, {x0, y0, x1, y1}, b) == p);
    REQUIRE(r.rect_sum(TableKind::XRamp, {x0, y0, x1, y1}, b) == sx);
    REQUIRE(r.rect_sum(TableKind::YRamp, {x0, y0, x1, y1}, b) == sy);
  }
}

TEST_CASE("directional tables are exact linear combinations (test_integral_tables.cpp:129-178)") {
  const int w = 16, h = 16, bins = 4;
  const FeatureImage fi = quantize_image(noise(w, h, 31), Quantizer(bins));
  const IntegralTableSet t = build_tables(fi);
  for (Direction d : {Direction::SE, Direction::SW, Direction::NE, Direction::NW}) {
    auto wgt = [&](int x, int y) -> std::int64_t {
      switch (d) {
        case Direction::SE: return x + y;
        case Direction::SW: return (w - 1 - x) + y;
        case Direction::NE: return x + (h - 1 - y);
        default: return (w - 1 - x) + (h - 1 - y);
      }
    };
    for (int b = 0; b < bins; ++b)
      for (int Y = 0; Y <= h; ++Y)
        for (int X = 0; X <= w; ++X) {
          std::int64_t direct = 0;
          for (int y = 0; y < Y; ++y)
            for (int x = 0; x < X; ++x)
              if (fi.at(x, y) == b) direct += wgt(x, y);
          REQUIRE(t.directional_value(d, X, Y, b) == direct);
        }
  }
}

TEST_CASE("bounds and capacity errors (test_integral_tables.cpp:180-203)") {
  const IntegralTableSet t = build_tables(quantize_image(noise(8, 8, 1), Quantizer(4)));
  CHECK_THROWS_AS(t.rect_sum(TableKind::Plain, {0, 0, 8, 3}, 0), OutOfRangeError);
  CHECK_THROWS_AS(t.rect_sum(TableKind::Plain, {2, 2, 1, 3}, 0), OutOfRangeError);
  CHECK_THROWS_AS(t.rect_sum(TableKind::Plain, {0, 0, 1, 1}, 4), OutOfRangeError);
  CHECK_THROWS_AS(t.cell(TableKind::Plain, 9, 0, 0), OutOfRangeError);
  TableBuildOptions tiny;
  tiny.memory_budget_bytes = 64;
  try {
    build_tables(quantize_image(noise(8, 8, 1), Quantizer(4)), tiny);
    CHECK(false);
  } catch (const CapacityError& e) {
    const std::size_t expected = 3ul * 9 * 9 * 4 * 8;
    CHECK(e.required_bytes() == expected);
    CHECK(std::string(e.what()).find(std::to_string(expected)) != std::string::npos);
  }
}

TEST_CASE("SWIH1 dump round trip; bad magic (test_integral_tables.cpp:205-226)") {
  const IntegralTableSet t = build_tables(quantize_image(noise(13, 9, 77), Quantizer(8)));
  std::stringstream ss;
  t.save(ss);
  const IntegralTableSet back = IntegralTableSet::load(ss);
  CHECK(back.width() == 13);
  CHECK(back.height() == 9);
  CHECK(back.bins() == 8);
  for (TableKind k : {TableKind::Plain, TableKind::XRamp, TableKind::YRamp})
    for (int b = 0; b < 8; ++b)
      for (int y = 0; y <= 9; ++y)
        for (int x = 0; x <= 13; ++x) REQUIRE(back.cell(k, x, y, b) == t.cell(k, x, y, b));
  // the loaded tables answer GPU queries too
  std::vector<std::int64_t> a(8), b(8);
  swih_query_into(t, {6, 4, man(7, 5), BorderPolicy::Strict}, a);
  swih_query_into(back, {6, 4, man(7, 5), BorderPolicy::Strict}, b);
  CHECK(a == b);
  std::stringstream junk("JUNK!whatever");
  CHECK_THROWS_AS(IntegralTableSet::load(junk), IoError);
}

// ---------------------------------------------------------------- engine
TEST_CASE("decompose tiles the window and reproduces the weights (test_engine.cpp:21-97)") {
  const QuadrantDecomposition d = decompose({1, 1, man(3, 3), BorderPolicy::Strict});
  REQUIRE(d.tl.rect.has_value());
  CHECK(d.tl.rect->x0 == 0 && d.tl.rect->y0 == 0 && d.tl.rect->x1 == 1 && d.tl.rect->y1 == 1);
  CHECK(d.tl.beta == 1);
  const QuadrantDecomposition one = decompose({4, 7, man(1, 1), BorderPolicy::Strict});
  CHECK(one.tl.rect.has_value());
  CHECK_FALSE(one.tr.rect.has_value() || one.bl.rect.has_value() || one.br.rect.has_value());
  std::mt19937_64 rng(17);
  for (int trial = 0; trial < 60; ++trial) {
    const KernelSpec k{trial % 2 ? KernelKind::Uniform : KernelKind::ManhattanLinear,
                       1 + 2 * int(rng() % 5), 1 + 2 * int(rng() % 5), 0.5};
    const int cx = 20 + int(rng() % 30), cy = 20 + int(rng() % 30);
    const QuadrantDecomposition q = decompose({cx, cy, k, BorderPolicy::Strict});
    for (int y = cy - k.hy(); y <= cy + k.hy(); ++y)
      for (int x = cx - k.hx(); x <= cx + k.hx(); ++x) {
        int owners = 0;
        double w = 0.0;
        for (const QuadrantTerm* t : q.terms())
          if (t->rect && x >= t->rect->x0 && x <= t->rect->x1 && y >= t->rect->y0 &&
              y <= t->rect->y1) {
            ++owners;
            w = double(t->sx * x + t->sy * y + t->beta);
          }
        REQUIRE(owners == 1);
        REQUIRE(w == weight_at(k, x - cx, y - cy));
      }
  }
  CHECK_THROWS_AS(decompose({5, 5, {KernelKind::ChebyshevLinear, 3, 3, 0.5}, BorderPolicy::Strict}),
                  UnsupportedKernelError);
  CHECK_THROWS_AS(decompose({5, 5, man(4, 3), BorderPolicy::Strict}), InvalidKernelError);
}

TEST_CASE("quadrant and window queries on the cross image (test_engine.cpp:99-147)") {
  const IntegralTableSet t = build_tables(quantize_image(cross3(), Quantizer(2)));
  const WeightedHistogram tl = quadrant_histogram(t, RectRegion{0, 0, 1, 1}, +1, +1, 1);
  CHECK(tl.value(0) == 4.0 && tl.value(1) == 4.0);
  const WeightedHistogram e = quadrant_histogram(t, std::nullopt, 1, 1, 0);
  CHECK(e.value(0) == 0.0 && e.value(1) == 0.0);
  const WeightedHistogram pl = quadrant_histogram(t, RectRegion{0, 0, 2, 2}, 0, 0, 1);
  CHECK(pl.value(0) == 5.0 && pl.value(1) == 4.0);
  CHECK_THROWS_AS(quadrant_histogram(t, RectRegion{0, 0, 3, 1}, 1, 1, 0), OutOfRangeError);
  const WindowQuery q{1, 1, man(3, 3), BorderPolicy::Strict};
  const WeightedHistogram raw = swih_query(t, q);
  CHECK(raw.value(0) == 7.0 && raw.value(1) == 8.0);
  CHECK(raw.sum() == kernel_weight_sum(q.kernel));
  const WeightedHistogram n = normalize(raw);
  CHECK(n.value(0) == Approx(7.0 / 15.0).epsilon(1e-12));
  const WindowQuery uq{1, 1, {KernelKind::Uniform, 3, 3, 0.5}, BorderPolicy::Strict};
  CHECK(swih_query(t, uq).value(0) == plain_local_histogram(t, uq).value(0));
  CHECK(swih_query(t, uq).value(0) == 5.0);
}

TEST_CASE("swih equals brute force at every strict centre (test_engine.cpp:149-175)") {
  std::mt19937_64 rng(55);
  for (auto [w, h] : {std::pair{17, 13}, {24, 24}, {33, 40}}) {
    const GrayImage img = noise(w, h, rng());
    for (int bins : {2, 8}) {
      const FeatureImage fi = quantize_image(img, Quantizer(bins));
      const IntegralTableSet t = build_tables(fi);
      for (auto [kw, kh] : {std::pair{1, 1}, {3, 3}, {5, 9}, {7, 7}, {31, 31}}) {
        if (kw > w || kh > h) continue;
        const KernelSpec k = man(kw, kh);
        const BruteForcePlan plan(k);
        std::vector<std::int64_t> got(static_cast<std::size_t>(bins));
        std::vector<std::int64_t> want(static_cast<std::size_t>(bins));
        for (int cy = k.hy(); cy < h - k.hy(); cy += 3)
          for (int cx = k.hx(); cx < w - k.hx(); cx += 2) {
            swih_query_into(t, {cx, cy, k, BorderPolicy::Strict}, got);
            plan.counts_into(fi, cx, cy, BorderPolicy::Strict, want);
            REQUIRE(got == want);
          }
      }
    }
  }
}

TEST_CASE("clipped queries match brute force; strict errors (test_engine.cpp:177-207)") {
  const FeatureImage fi = quantize_image(noise(15, 11, 8), Quantizer(4));
  const IntegralTableSet t = build_tables(fi);
  const KernelSpec k = man(7, 5);
  const BruteForcePlan plan(k);
  std::vector<std::int64_t> got(4), want(4);
  for (int cy = 0; cy < 11; ++cy)
    for (int cx = 0; cx < 15; ++cx) {
      swih_query_into(t, {cx, cy, k, BorderPolicy::Clipped}, got);
      plan.counts_into(fi, cx, cy, BorderPolicy::Clipped, want);
      REQUIRE(got == want);
    }
  CHECK(normalize(swih_query(t, {0, 0, k, BorderPolicy::Clipped})).sum() ==
        Approx(1.0).epsilon(1e-9));
  const IntegralTableSet s = build_tables(quantize_image(noise(9, 9, 4), Quantizer(2)));
  CHECK_THROWS_AS(swih_query(s, {1, 4, man(5, 5), BorderPolicy::Strict}), WindowOutOfBoundsError);
  CHECK_THROWS_AS(swih_query(s, {4, 9, man(3, 3), BorderPolicy::Clipped}), WindowOutOfBoundsError);
}

TEST_CASE("constant image: translation invariant; concurrent queries (test_engine.cpp:209-253)") {
  const GrayImage img(40, 30, 77);
  for (int bins : {2, 16}) {
    const IntegralTableSet t = build_tables(quantize_image(img, Quantizer(bins)));
    for (int k : {1, 3, 9, 21}) {
      const KernelSpec spec = man(k, k);
      const WeightedHistogram first =
          normalize(swih_query(t, {spec.hx(), spec.hy(), spec, BorderPolicy::Strict}));
      for (int cy = spec.hy(); cy < 30 - spec.hy(); cy += 7)
        for (int cx = spec.hx(); cx < 40 - spec.hx(); cx += 7) {
          const WeightedHistogram n = normalize(swih_query(t, {cx, cy, spec, BorderPolicy::Strict}));
          for (int b = 0; b < bins; ++b) REQUIRE(n.value(b) == first.value(b));
        }
    }
  }
  const IntegralTableSet t = build_tables(quantize_image(noise(64, 64, 12), Quantizer(8)));
  std::vector<std::int64_t> serial(8);
  swih_query_into(t, {20, 20, man(9, 9), BorderPolicy::Strict}, serial);
  std::vector<std::vector<std::int64_t>> res(4, std::vector<std::int64_t>(8));
  std::vector<std::thread> pool;
  for (int i = 0; i < 4; ++i)
    pool.emplace_back([&, i] {
      for (int rep = 0; rep < 50; ++rep)
        swih_query_into(t, {20, 20, man(9, 9), BorderPolicy::Strict}, res[std::size_t(i)]);
    });
  for (auto& th : pool) th.join();
  for (const auto& r : res) CHECK(r == serial);
}

// ---------------------------------------------------------------- baselines
TEST_CASE("brute force and wedding cake on the cross image (test_baselines.cpp:21-101)") {
  const FeatureImage fi = quantize_image(cross3(), Quantizer(2));
  CHECK(brute_force_histogram(fi, {1, 1, man(3, 3), BorderPolicy::Strict}).value(0) == 7.0);
  CHECK(brute_force_histogram(fi, {1, 1, {KernelKind::Uniform, 3, 3, 0.5}, BorderPolicy::Strict})
            .value(1) == 4.0);
  CHECK(brute_force_histogram(fi, {1, 1, man(1, 1), BorderPolicy::Strict}).value(0) == 1.0);
  CHECK_THROWS_AS(brute_force_histogram(fi, {0, 0, man(3, 3), BorderPolicy::Strict}),
                  WindowOutOfBoundsError);
  const IntegralTableSet t = build_tables(fi);
  const KernelSpec cheb{KernelKind::ChebyshevLinear, 3, 3, 0.5};
  const WeightedHistogram cake = wedding_cake_histogram(t, {1, 1, cheb, BorderPolicy::Strict},
                                                        {2, RingRule::Mean});
  CHECK(cake.value(0) == 6.0 && cake.value(1) == 4.0);
  const WeightedHistogram approx = wedding_cake_histogram(
      t, {1, 1, man(3, 3), BorderPolicy::Strict}, {2, RingRule::Mean});
  CHECK(approx.value(0) == Approx(9.0).epsilon(1e-12));
  CHECK(approx.value(1) == Approx(6.0).epsilon(1e-12));
  const WeddingCakePlan lvl(man(3, 3), {2, RingRule::Level});
  CHECK(lvl.ring_weight(0) == weight_at(man(3, 3), 1, 0));
  CHECK(lvl.ring_weight(1) == weight_at(man(3, 3), 0, 0));
  const WeightedHistogram h = wedding_cake_histogram(t, {1, 1, man(3, 3), BorderPolicy::Strict},
                                                     {2, RingRule::Level});
  CHECK(h.value(0) == Approx(11.0).epsilon(1e-12));
  CHECK(h.value(1) == Approx(8.0).epsilon(1e-12));
  CHECK_THROWS_AS(wedding_cake_histogram(t, {1, 1, cheb, BorderPolicy::Strict}, {3, RingRule::Mean}),
                  ConfigError);
  CHECK_THROWS_AS(wedding_cake_histogram(t, {1, 1, cheb, BorderPolicy::Strict}, {0, RingRule::Mean}),
                  ConfigError);
}

TEST_CASE("wedding cake exact for ring-constant kernels; mass preserved (test_baselines.cpp:104-197)") {
  const FeatureImage fi = quantize_image(noise(40, 40, 60), Quantizer(8));
  const IntegralTableSet t = build_tables(fi);
  std::mt19937_64 rng(61);
  for (int k : {3, 5, 9})
    for (KernelKind kind : {KernelKind::ChebyshevLinear, KernelKind::GaussianChebyshev}) {
      const KernelSpec spec{kind, k, k, 0.6};
      for (int trial = 0; trial < 20; ++trial) {
        const int cx = k / 2 + int(rng() % (40 - k + 1)), cy = k / 2 + int(rng() % (40 - k + 1));
        const WindowQuery q{cx, cy, spec, BorderPolicy::Strict};
        const WeightedHistogram cake = wedding_cake_histogram(t, q, {k / 2 + 1, RingRule::Mean});
        const WeightedHistogram exact = brute_force_histogram(fi, q);
        for (int b = 0; b < 8; ++b) REQUIRE(cake.value(b) == Approx(exact.value(b)).epsilon(1e-9));
      }
    }
  const KernelSpec m{KernelKind::ManhattanLinear, 9, 15, 0.5};
  for (int rings : {1, 2, 4}) {
    const WeightedHistogram h = wedding_cake_histogram(t, {20, 20, m, BorderPolicy::Strict},
                                                       {rings, RingRule::Mean});
    CHECK(h.sum() == Approx(kernel_weight_sum(m)).epsilon(1e-9));
  }
  const WeightedHistogram c = wedding_cake_histogram(
      t, {1, 1, {KernelKind::Uniform, 9, 9, 0.5}, BorderPolicy::Clipped}, {1, RingRule::Mean});
  const WeightedHistogram e =
      brute_force_histogram(fi, {1, 1, {KernelKind::Uniform, 9, 9, 0.5}, BorderPolicy::Clipped});
  for (int b = 0; b < 8; ++b) CHECK(c.value(b) == e.value(b));
}

// ---------------------------------------------------------------- matching
TEST_CASE("similarity examples (test_matching.cpp:25-42)") {
  const std::vector<double> p{7.0 / 15.0, 8.0 / 15.0}, q{0.5, 0.5};
  CHECK(similarity(SimilarityKind::Bhattacharyya, p, q) ==
        Approx(std::sqrt(7.0 / 30.0) + std::sqrt(8.0 / 30.0)).epsilon(1e-12));
  const std::vector<double> a{1.0, 0.0}, b{0.0, 1.0};
  CHECK(similarity(SimilarityKind::Bhattacharyya, a, b) == 0.0);
  CHECK(similarity(SimilarityKind::Intersection, p, q) == Approx(7.0 / 15.0 + 0.5).epsilon(1e-12));
}

TEST_CASE("target model (test_matching.cpp:62-81)") {
  const Quantizer q(2);
  const KernelSpec k = man(3, 3);
  CHECK(target_model(GrayImage(3, 3, 40), q, k).value(0) == 1.0);
  CHECK(target_model(cross3(), q, k).value(0) == Approx(7.0 / 15.0).epsilon(1e-12));
  CHECK(target_model(cross3(), q, {KernelKind::Uniform, 3, 3, 0.5}).value(0) ==
        Approx(5.0 / 9.0).epsilon(1e-12));
  CHECK_THROWS_AS(target_model(GrayImage(5, 3, 0), q, k), ModelError);
}

TEST_CASE("likelihood map over a tiled template, all methods (test_matching.cpp:83-113)") {
  const GrayImage tile = cross3();
  GrayImage search(9, 6);
  for (int y = 0; y < 6; ++y)
    for (int x = 0; x < 9; ++x) search.set(x, y, tile.at(x % 3, y % 3));
  for (MapMethod method : {MapMethod::Swih, MapMethod::Brute, MapMethod::Cake, MapMethod::Plain}) {
    MatchOptions opt;
    opt.cake.rings = 2;
    const WeightedHistogram model =
        target_model_for_method(tile, Quantizer(2), man(3, 3), method, opt.cake);
    const LikelihoodMap map = likelihood_map(search, model, Quantizer(2), man(3, 3), method, opt);
    CHECK(map.width == 7 && map.height == 4);
    for (int v = 0; v < map.height; v += 3)
      for (int u = 0; u < map.width; u += 3) REQUIRE(map.at(u, v) == Approx(1.0).epsilon(1e-12));
  }
}

TEST_CASE("swih and brute maps identical; peak on the template (test_matching.cpp:115-141)") {
  const GrayImage search = noise(40, 33, 2024);
  const KernelSpec k = man(9, 7);
  GrayImage templ(9, 7);
  for (int y = 0; y < 7; ++y)
    for (int x = 0; x < 9; ++x) templ.set(x, y, search.at(x + 12, y + 9));
  const WeightedHistogram model = target_model(templ, Quantizer(8), k);
  const LikelihoodMap a = likelihood_map(search, model, Quantizer(8), k, MapMethod::Swih);
  const LikelihoodMap b = likelihood_map(search, model, Quantizer(8), k, MapMethod::Brute);
  REQUIRE(a.scores.size() == b.scores.size());
  CHECK(a.scores == b.scores);  // bit-identical, not merely within 1e-12
  const Peak pa = peak(a), pb = peak(b);
  CHECK(pa.map_x == pb.map_x && pa.map_y == pb.map_y);
  CHECK(pa.center_x == 16 && pa.center_y == 12);
  CHECK(pa.score == Approx(1.0).epsilon(1e-12));
}

TEST_CASE("map errors (test_matching.cpp:143-161)") {
  const Quantizer q(4);
  const GrayImage small(5, 5, 10);
  const WeightedHistogram model = normalize(WeightedHistogram({1.0, 1.0, 1.0, 1.0}, false));
  CHECK_THROWS_AS(likelihood_map(small, model, q, man(7, 7), MapMethod::Swih), SizeError);
  CHECK_THROWS_AS(likelihood_map(small, model, q, {KernelKind::GaussianChebyshev, 3, 3, 0.5},
                                 MapMethod::Swih),
                  UnsupportedKernelError);
  CHECK_THROWS_AS(likelihood_map(small, WeightedHistogram({1.0, 2.0, 3.0, 4.0}, false), q,
                                 man(3, 3), MapMethod::Swih),
                  ModelError);
  MatchOptions tiny;
  tiny.tables.memory_budget_bytes = 64;
  CHECK_THROWS_AS(likelihood_map(small, model, q, man(3, 3), MapMethod::Swih, tiny), CapacityError);
}

TEST_CASE("peak: first maximum in row-major order (test_matching.cpp:163-189)") {
  LikelihoodMap map;
  map.width = 3;
  map.height = 2;
  map.hx = 1;
  map.hy = 2;
  map.scores = {0.2, 0.9, 0.1, 0.9, 0.3, 0.9};
  const Peak p = peak(map);
  CHECK(p.map_x == 1 && p.map_y == 0 && p.center_x == 2 && p.center_y == 2 && p.score == 0.9);
  LikelihoodMap flat;
  flat.width = flat.height = 2;
  flat.scores = {0.5, 0.5, 0.5, 0.5};
  CHECK(peak(flat).map_x == 0 && peak(flat).map_y == 0);
  LikelihoodMap big;
  big.width = 1000;
  big.height = 700;
  big.scores.assign(700000, 0.25);
  big.scores[523456] = 0.75;
  big.scores[612345] = 0.75;
  CHECK(peak(big).map_x == 523456 % 1000 && peak(big).map_y == 523456 / 1000);
  CHECK_THROWS_AS(peak(LikelihoodMap{}), Error);
}

TEST_CASE("map output formats; threads do not change the map (test_matching.cpp:191-222)") {
  LikelihoodMap map;
  map.width = 2;
  map.height = 1;
  map.scores = {0.0, 1.0};
  const GrayImage g = map_to_gray(map);
  CHECK(g.at(0, 0) == 0 && g.at(1, 0) == 255);
  map.scores = {0.25, 0.125};
  std::stringstream ss;
  write_map_csv(map, ss);
  CHECK(ss.str() == "0.25,0.125\n");
  const GrayImage search = noise(30, 26, 31337);
  const KernelSpec k = man(7, 7);
  const WeightedHistogram model = target_model(noise(7, 7, 5), Quantizer(8), k);
  MatchOptions threaded;
  threaded.threads = 3;
  CHECK(likelihood_map(search, model, Quantizer(8), k, MapMethod::Swih).scores ==
        likelihood_map(search, model, Quantizer(8), k, MapMethod::Swih, threaded).scores);
}

int main() { return minitest::run_all(); }
