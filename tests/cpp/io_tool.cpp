// io_tool.cpp — the reference-compatible C++ API's file outputs, driven from
// tests/test_io_compat.py, which byte-compares them with the reference
// library's own writers (oracle/_ref).  TEST INFRASTRUCTURE.
//
//   io_tool dump    <fi.u16> <w> <h> <bins> <out.swih>     build_tables + save_file
//   io_tool resave  <in.swih> <out.swih>                    load_file + save_file
//   io_tool pgm     <in.pgm> <out.pgm>                      read_pgm_file + write_pgm_file
//   io_tool map     <in.pgm> <bins> <kind> <kw> <kh> <method> <rings> <tx> <ty> <csv> <pgm>
//                   target model of the kw x kh template centred on (tx, ty),
//                   likelihood_map, write_map_csv_file, write_pgm_file(map_to_gray)
//   io_tool bench   <w> <h> <bins> <kw> <method> <out.csv>  bench_sweep + CSV
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "swih/bench.hpp"
#include "swih/integral_tables.hpp"
#include "swih/matching.hpp"
#include "swih/pgm.hpp"

using namespace swih;

int main(int argc, char** argv) try {
  if (argc < 2) return 2;
  const std::string cmd = argv[1];
  if (cmd == "dump" && argc == 7) {
    const int w = std::atoi(argv[3]), h = std::atoi(argv[4]), b = std::atoi(argv[5]);
    FeatureImage fi(w, h, b);
    std::ifstream in(argv[2], std::ios::binary);
    in.read(reinterpret_cast<char*>(fi.data()), std::streamsize(std::size_t(w) * h * 2));
    if (!in) return 3;
    build_tables(fi).save_file(argv[6]);
    return 0;
  }
  if (cmd == "resave" && argc == 4) {
    IntegralTableSet::load_file(argv[2]).save_file(argv[3]);
    return 0;
  }
  if (cmd == "pgm" && argc == 4) {
    write_pgm_file(read_pgm_file(argv[2]), argv[3]);
    return 0;
  }
  if (cmd == "map" && argc == 13) {
    const GrayImage search = read_pgm_file(argv[2]);
    const Quantizer q(std::atoi(argv[3]));
    const KernelSpec k{KernelKind(std::atoi(argv[4])), std::atoi(argv[5]), std::atoi(argv[6]),
                       0.5};
    const MapMethod method = MapMethod(std::atoi(argv[7]));
    MatchOptions opt;
    opt.cake.rings = std::atoi(argv[8]);
    const int tx = std::atoi(argv[9]), ty = std::atoi(argv[10]);
    GrayImage templ(k.kw, k.kh);
    for (int y = 0; y < k.kh; ++y)
      for (int x = 0; x < k.kw; ++x) templ.set(x, y, search.at(tx - k.hx() + x, ty - k.hy() + y));
    const WeightedHistogram model = target_model_for_method(templ, q, k, method, opt.cake);
    const LikelihoodMap map = likelihood_map(search, model, q, k, method, opt);
    write_map_csv_file(map, argv[11]);
    write_pgm_file(map_to_gray(map), argv[12]);
    return 0;
  }
  if (cmd == "bench" && argc == 8) {
    const FeatureImage fi =
        quantize_image(random_image(std::atoi(argv[2]), std::atoi(argv[3]), 7),
                       Quantizer(std::atoi(argv[4])));
    const int kw = std::atoi(argv[5]);
    BenchConfig cfg;
    cfg.repetitions = 1;
    cfg.cake.rings = 2;
    const BenchRecord r = bench_sweep(fi, MapMethod(std::atoi(argv[6])),
                                      {KernelKind::ManhattanLinear, kw, kw, 0.5}, cfg);
    std::ofstream out(argv[7], std::ios::binary);
    write_bench_csv_header(out);
    write_bench_csv_row(r, out);
    return 0;
  }
  std::fprintf(stderr, "io_tool: bad arguments\n");
  return 2;
} catch (const std::exception& e) {
  std::fprintf(stderr, "io_tool: %s\n", e.what());
  return 1;
}
