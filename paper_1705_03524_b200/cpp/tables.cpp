// tables.cpp — IntegralTableSet over device tables (reference bodies:
// src/integral_tables.cpp:64-206).  build() runs the GPU build (quantised
// feature image in, bin-octet uint32 planes out); host int64 planes are
// exported from the device once, on the first host access.
#include <array>
#include <cstdio>
#include <fstream>
#include <istream>
#include <mutex>
#include <ostream>
#include <string>

#include "runtime.hpp"
#include "swih/integral_tables.hpp"

namespace swih {

struct IntegralTableSet::State {
  swg_tables* dev = nullptr;
  std::once_flag exported;
  std::array<std::vector<std::int64_t>, 3> host;  // plain, xramp, yramp
  ~State() { swg_tables_destroy(dev); }
};

namespace {

void put_u32(std::ostream& out, std::uint32_t v) {
  const char b[4] = {char(v & 0xff), char((v >> 8) & 0xff), char((v >> 16) & 0xff),
                     char((v >> 24) & 0xff)};
  out.write(b, 4);
}

std::uint32_t get_u32(std::istream& in) {
  unsigned char b[4] = {};
  in.read(reinterpret_cast<char*>(b), 4);
  if (!in) throw IoError("table dump: truncated header");
  return std::uint32_t(b[0]) | std::uint32_t(b[1]) << 8 | std::uint32_t(b[2]) << 16 |
         std::uint32_t(b[3]) << 24;
}

constexpr char kMagic[5] = {'S', 'W', 'I', 'H', '1'};

}  // namespace

IntegralTableSet IntegralTableSet::build(const FeatureImage& fi, const TableBuildOptions& opt) {
  const std::size_t cells = std::size_t(fi.width() + 1) * (fi.height() + 1) * fi.bins();
  const std::size_t required = 3 * cells * sizeof(std::int64_t);  // reference footprint
  if (required > opt.memory_budget_bytes)
    throw CapacityError("integral tables need " + std::to_string(required) +
                            " bytes, budget is " + std::to_string(opt.memory_budget_bytes),
                        required);
  auto st = std::make_shared<State>();
  detail::check(swg_tables_build(detail::context(), fi.data(), 0, 0, fi.width(), fi.height(),
                                 SWG_FMT_BINS16, fi.bins(), SWG_PLANES_AFFINE, 0, &st->dev));
  return IntegralTableSet(std::move(st), fi.width(), fi.height(), fi.bins());
}

swg_tables* IntegralTableSet::device() const noexcept { return st_->dev; }

const std::vector<std::int64_t>& IntegralTableSet::host_table(TableKind kind) const {
  State& s = *st_;
  std::call_once(s.exported, [&] {
    for (int k = 0; k < 3; ++k) {
      s.host[std::size_t(k)].resize(plane_stride() * std::size_t(b_));
      detail::check(swg_tables_export_i64(s.dev, k, 0, b_, s.host[std::size_t(k)].data()));
    }
  });
  return s.host[std::size_t(kind)];
}

const std::int64_t* IntegralTableSet::plane(TableKind kind, int bin) const noexcept {
  try {
    return host_table(kind).data() + std::size_t(bin) * plane_stride();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "swih: table export failed: %s\n", e.what());
    std::abort();
  }
}

std::int64_t IntegralTableSet::cell(TableKind kind, int x, int y, int bin) const {
  if (x < 0 || x > w_ || y < 0 || y > h_ || bin < 0 || bin >= b_)
    throw OutOfRangeError("table cell (" + std::to_string(x) + "," + std::to_string(y) +
                          ",bin " + std::to_string(bin) + ") out of range");
  return host_table(kind)[std::size_t(bin) * plane_stride() + std::size_t(y) * row_stride() +
                          std::size_t(x)];
}

void IntegralTableSet::check_rect(const RectRegion& r, int bin) const {
  if (bin < 0 || bin >= b_)
    throw OutOfRangeError("rect_sum: bin " + std::to_string(bin) + " out of range");
  if (r.x0 < 0 || r.y0 < 0 || r.x0 > r.x1 || r.y0 > r.y1 || r.x1 >= w_ || r.y1 >= h_)
    throw OutOfRangeError("rect_sum: rectangle (" + std::to_string(r.x0) + "," +
                          std::to_string(r.y0) + ")-(" + std::to_string(r.x1) + "," +
                          std::to_string(r.y1) + ") out of bounds for " + std::to_string(w_) +
                          "x" + std::to_string(h_));
}

std::int64_t IntegralTableSet::rect_sum(TableKind kind, const RectRegion& r, int bin) const {
  check_rect(r, bin);
  const std::int64_t* p = plane(kind, bin);
  const std::size_t rs = row_stride();
  auto at = [&](int x, int y) { return p[std::size_t(y) * rs + std::size_t(x)]; };
  return at(r.x1 + 1, r.y1 + 1) - at(r.x0, r.y1 + 1) - at(r.x1 + 1, r.y0) + at(r.x0, r.y0);
}

std::int64_t IntegralTableSet::directional_value(Direction dir, int x, int y, int bin) const {
  const std::int64_t p = cell(TableKind::Plain, x, y, bin);
  const std::int64_t sx = cell(TableKind::XRamp, x, y, bin);
  const std::int64_t sy = cell(TableKind::YRamp, x, y, bin);
  const std::int64_t wm = w_ - 1, hm = h_ - 1;
  switch (dir) {
    case Direction::SE: return sx + sy;
    case Direction::SW: return wm * p - sx + sy;
    case Direction::NE: return sx + hm * p - sy;
    case Direction::NW: return (wm + hm) * p - sx - sy;
  }
  throw OutOfRangeError("directional_value: unknown direction");
}

void IntegralTableSet::save(std::ostream& out) const {
  out.write(kMagic, 5);
  put_u32(out, std::uint32_t(w_));
  put_u32(out, std::uint32_t(h_));
  put_u32(out, std::uint32_t(b_));
  std::vector<char> buf;
  for (TableKind kind : {TableKind::Plain, TableKind::XRamp, TableKind::YRamp}) {
    const auto& t = host_table(kind);
    buf.resize(t.size() * 8);
    for (std::size_t i = 0; i < t.size(); ++i) {
      const auto u = std::uint64_t(t[i]);
      for (int k = 0; k < 8; ++k) buf[i * 8 + std::size_t(k)] = char((u >> (8 * k)) & 0xff);
    }
    out.write(buf.data(), std::streamsize(buf.size()));
  }
  if (!out) throw IoError("table dump: write failed");
}

void IntegralTableSet::save_file(const std::string& path) const {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("table dump: cannot open '" + path + "'");
  save(out);
}

IntegralTableSet IntegralTableSet::load(std::istream& in) {
  char magic[5] = {};
  in.read(magic, 5);
  if (!in || std::string(magic, 5) != std::string(kMagic, 5))
    throw IoError("table dump: bad magic");
  const int w = int(get_u32(in)), h = int(get_u32(in)), b = int(get_u32(in));
  if (w < 1 || h < 1 || b < 1) throw IoError("table dump: bad dimensions");
  auto st = std::make_shared<State>();
  const std::size_t n = std::size_t(w + 1) * (h + 1) * b;
  std::vector<unsigned char> buf(n * 8);
  for (auto& t : st->host) {
    in.read(reinterpret_cast<char*>(buf.data()), std::streamsize(buf.size()));
    if (std::size_t(in.gcount()) != buf.size()) throw IoError("table dump: truncated table data");
    t.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
      std::uint64_t u = 0;
      for (int k = 0; k < 8; ++k) u |= std::uint64_t(buf[i * 8 + std::size_t(k)]) << (8 * k);
      t[i] = std::int64_t(u);
    }
  }
  detail::check(swg_tables_upload_i64(detail::context(), w, h, b, st->host[0].data(),
                                      st->host[1].data(), st->host[2].data(), &st->dev));
  std::call_once(st->exported, [] {});  // host planes are already exact
  return IntegralTableSet(std::move(st), w, h, b);
}

IntegralTableSet IntegralTableSet::load_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("table dump: cannot open '" + path + "'");
  return load(in);
}

}  // namespace swih
