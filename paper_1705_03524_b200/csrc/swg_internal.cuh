// swg_internal.cuh — shared structs, device-layout rules and helpers for the
// sm_100a kernels behind include/swg.h.
//
// Device layout of one plane set:
//   plane (bin, kind) = base + (bin * P + kind) * plane_stride
//   element (x, y), x in [0, W], y in [0, H] (zero row 0 / column 0, the
//   reference's padded (W+1)x(H+1) plane, integral_tables.hpp:53-58)
//   sits at  y * pitch + x + XOFF,  XOFF = 16/sizeof(T) - 1
// so that the data columns x = 1 .. W start on a 16-byte boundary and every
// row starts on a 128-byte boundary (pitch is a multiple of 32 elements).
// T = uint32_t (default: exact mod 2^32, every strict window histogram fits)
// or uint64_t (exact export / wide kernels).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "swg.h"

namespace swg {

constexpr int kMaxBins = SWG_MAX_BINS;
constexpr int kMaxRings = SWG_MAX_RINGS;
constexpr uint16_t kNoBin = 0xFFFF;  // feature-image padding sentinel

template <typename T>
struct Layout {
  static constexpr int xoff = 16 / (int)sizeof(T) - 1;
};

inline size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

// Columns per build thread, chosen from the width (see choose_cpt).
inline int choose_cpt(int w) {
  if (w <= 1024) return 4;
  if (w <= 4096) return 8;
  return 16;
}

// Row pitch (elements) of a plane with element type of `elem` bytes.
inline size_t plane_pitch(int w, int elem) {
  const int xoff = 16 / elem - 1;
  return round_up((size_t)xoff + 1 + round_up((size_t)w, 16), 32);
}

// Feature-image pitch (uint16 elements); rows padded with kNoBin.
inline size_t fi_pitch(int w) { return round_up((size_t)w, 64); }

// ---------------------------------------------------------------- build
struct BuildArgs {
  const uint16_t* fi;  // quantised image, fi_pitch elements per row
  size_t fi_pitch;
  void* out;           // planes (T)
  size_t pitch;        // elements
  size_t plane_stride; // elements
  int w, h, bins, planes;
  int band_h, nbands;
  size_t wa;           // padded width of the look-back arrays
  uint32_t* agg;       // [nbands][bins][2][wa]: band column count / y-sum
  uint32_t* pref;      // [nbands][bins][2][wa]: inclusive prefix over bands
  int* flags;          // [nbands * bins]: 0 none, 1 aggregate, 2 prefix
  unsigned* ticket;    // dynamic CTA ordering for the look-back
};

struct QuantArgs {
  const uint8_t* in;
  size_t in_pitch;  // bytes
  int w, h, format, bins;
  uint16_t* fi;
  size_t fi_pitch;
};

// ---------------------------------------------------------------- sweep
struct PeakPart {
  double score;
  long long idx;  // v * map_w + u (absolute map row v)
};

struct SweepArgs {
  const void* tab;     // planes
  size_t plane_stride; // elements
  size_t pitch;        // elements
  int planes;
  int bins;
  int hx, hy;
  int mw;              // map width
  int row0;            // first map row of this launch
  int rows;
  int sim;
  int rings;
  double mass;         // exact strict-window mass (affine kernels)
  double* scores;      // rows x mw, row r = map row row0 + r
  PeakPart* parts;     // one per CTA
  double model[kMaxBins];
};

struct CakeRings {
  int a[kMaxRings];       // ring i box half-extent in x: hx - shrink_x[i]
  int c[kMaxRings];       // ring i box half-extent in y: hy - shrink_y[i]
  double coeff[kMaxRings];// w_i - w_{i-1} (baselines.cpp:141)
};

struct BruteArgs {
  const uint16_t* fi;  // quantised image
  size_t fi_pitch;
  const double* grid;  // kh x kw kernel weights (llround-ed for integer kinds)
  int kw, kh;
  int integer;         // score_counts (1) or score_weights (0) semantics
};

struct QueryArgs {
  const void* tab;
  size_t plane_stride, pitch;
  int planes, bins;
  int n, tpw;
  const swg_term* terms;  // device
  long long* out;         // device n x bins
  const double* coeff;    // cake: per-term ring coefficient (n x tpw)
  double* outd;           // cake: device n x bins
};

// Kernel launchers (defined in the .cu files).
cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t s);
template <typename T>
cudaError_t launch_build(const BuildArgs& a, cudaStream_t s);
cudaError_t launch_sweep_affine(const SweepArgs& a, bool uniform, int blocks_x,
                                cudaStream_t s);
cudaError_t launch_sweep_cake(const SweepArgs& a, const CakeRings& r,
                              int blocks_x, cudaStream_t s);
cudaError_t launch_sweep_brute(const SweepArgs& a, const BruteArgs& b,
                               int blocks_x, cudaStream_t s);
cudaError_t launch_peak_reduce(const PeakPart* parts, int nparts, int mw,
                               int hx, int hy, swg_peak* out, cudaStream_t s);
template <typename T>
cudaError_t launch_query(const QueryArgs& a, cudaStream_t s);
cudaError_t launch_cake_query(const QueryArgs& a, cudaStream_t s);
cudaError_t launch_narrow(const uint64_t* src, size_t pitch64, size_t ps64,
                          uint32_t* dst, size_t pitch32, size_t ps32, int w,
                          int h, int nplanes, cudaStream_t s);

constexpr int kSweepThreads = 128;

}  // namespace swg
