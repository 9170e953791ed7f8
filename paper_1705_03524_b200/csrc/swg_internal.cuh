// swg_internal.cuh — shared structs, the device layout and kernel launchers
// behind include/swg.h.
//
// Device layout of one plane set: "bin octets".
// The reference stores one (W+1)x(H+1) int64 plane per bin and table kind,
// bin-major (integral_tables.hpp:53-58,116-118).  Here bins are tiled in
// groups of 8: a RECORD holds the 8 bins of one group at one padded cell,
//   record (x, y) of plane (group g, kind k)
//       = base + ((g*P + k) * plane_stride + y * pitch + x) * 8 elements,
//   element of bin b = record[b % 8],  g = b / 8,
// x in [0, W], y in [0, H] with the reference's zero row 0 / column 0.
// A record is 32 B (uint32) or 64 B (uint64); `pitch` (records) is a multiple
// of 4, so rows start on 128-byte boundaries.  A sweep thread reads one
// 16-byte half record per corner (4 bins), two adjacent lanes cover one
// window's octet, and a warp's load is 512 contiguous bytes.
// T = uint32_t (default: exact mod 2^32, every strict window histogram fits)
// or uint64_t (exact export / large-magnitude queries); both share pitch
// and plane_stride (in records).
#pragma once

#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime's driver entry point)
#include <cuda_runtime.h>
#include <stdint.h>

#include "swg.h"

namespace swg {

constexpr int kMaxBins = SWG_MAX_BINS;
constexpr int kMaxRings = SWG_MAX_RINGS;
constexpr int kOct = 8;              // bins per record (integral tables)
constexpr int kDP = 2;               // bins per record (fp64 decay tables: bin pairs)
constexpr uint16_t kNoBin = 0xFFFF;  // feature-image padding sentinel
constexpr int kMaxWidth = 4096;      // build CTA spans a full row (CPT <= 8)

inline size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

// Columns per build thread: 8 from 1024 wide (half the threads of a
// row-wide CTA, two CTAs per SM; measured faster at 2048 than 4 columns).
#ifndef SWG_CPT8_FROM
#define SWG_CPT8_FROM 1024
#endif
inline int choose_cpt(int w) { return w < SWG_CPT8_FROM ? 4 : 8; }

// Row pitch in records (room for the straddling last build thread).
inline size_t record_pitch(int w) { return round_up((size_t)w + 1 + 8, 4); }

// Feature-image pitch (uint16 elements); rows padded with kNoBin.
inline size_t fi_pitch(int w) { return round_up((size_t)w, 64); }

__host__ __device__ inline size_t elem_index(size_t ps, size_t pitch, int planes, int x,
                                             int y, int b, int k) {
  return ((((size_t)(b >> 3) * planes + k) * ps + (size_t)y * pitch + x) << 3) + (b & 7);
}

// ---------------------------------------------------------------- build
struct alignas(64) BuildArgs {
  // TMA tensor map over the output planes' rows (tmap_ok != 0): records
  // 1..W of row y of plane k as 128-byte lines (box: one warp's staged row
  // segment, SWIZZLE_128B = the staging's XOR layout); the build kernels
  // then write their staged rows with cp.async.bulk.tensor stores instead
  // of per-thread 16-byte stores.
  CUtensorMap tmap;
  int tmap_ok;
  const uint16_t* fi;  // quantised image, fi_pitch elements per row
  size_t fi_pitch;
  void* out;           // planes (T)
  size_t pitch;        // records
  size_t plane_stride; // records
  int w, h, bins, groups, planes;
  int band_h, nbands;
  size_t wa;           // padded width (columns) of the carry array
  int aw;              // carry words per column: 8 (plain), 16 (ramps), 24 (quadratic)
  int bin0;            // global bin of local bin 0 (bin-range tables)
  int kinds;           // table kinds to build (0: every plane; narrow tables: plain)
  void* out16;         // 32-bit builds: also write kinds 0-2 mod 2^16 here (narrow
                       // {1, x, y} planes, 3-plane layout), or null
  // Selective build (nsel > 0): only these units -- bin octets (integral
  // planes) or bin pairs (decay planes) -- are written, each into its own
  // slot of the full layout; the carries (K1a/K1b) still cover every unit.
  // decayed builds of all four orientations in ONE strip launch
  // (blockIdx.y = orientation): their feature images and carry arrays
  const uint16_t* fio[4];
  size_t agg_stride;  // uint32 words between orientations' carry arrays
  int nsel;
  unsigned short sel[kMaxBins / kDP];
  // the same selection as a bit mask (carry passes skip unselected units)
  uint32_t selmask[kMaxBins / kDP / 32];
  uint32_t* agg;       // [nbands][groups][wa][aw]: per column, 8 bin counts +
                       // 8 bin y-sums (+ 8 bin y^2-sums) of the band (K1a),
                       // then of all rows above the band (K1b, exclusive scan)
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
  const void* tab;     // planes (uint32 records)
  size_t plane_stride; // records
  size_t pitch;        // records
  int planes;
  int bins;
  int groups;
  int hx, hy;
  int mw;              // map width
  int row0;            // first map row of this launch
  int rows;
  int sim;
  int rings;
  double mass;         // exact strict-window mass (affine kernels)
  // affine: byte offsets of the corner cells from the window's centre record
  // (window independent): plain (x0,y0) (x1,y0) (x2,y0) (x0,y1) (x2,y1)
  // (x0,y2) (x1,y2) (x2,y2); xramp (x0,y0) (x1,y0) (x2,y0) (x0,y2) (x1,y2)
  // (x2,y2); yramp (x0,y0) (x2,y0) (x0,y1) (x2,y1) (x0,y2) (x2,y2), with
  // x0 = -hx, x1 = +1, x2 = hx+1 (y likewise) in padded coordinates.
  int lat[20];
  double* scores;      // rows x mw, row r = map row row0 + r
  PeakPart* parts;     // one per CTA
  // bin-range chain (tables holding bins [bin0, bin0 + bins) of a larger
  // set): running (s, mass) per window in, and out instead of scores
  const double2* pin;
  double2* pout;
  // CTA order: 0 = raster over the map; > 0 = super-columns of this many
  // tiles, each swept top to bottom, so the table rows between a window's
  // top and bottom corners stay in L2 (sweep_tile)
  int sc_tiles;
  // chain order (exponential sweep): CTA (blockIdx.x = (tile column, chain
  // step j, residue offset dv), blockIdx.y = residue group q) sweeps map row
  // j*chain_s + q*chain_k + dv, so the rows sharing a table row (window v's
  // bottom corners = window v+chain_s's top corners) run back to back
  int chain_s, chain_k, chain_j;  // 0: off
  int wide0;           // cake16: ring 0's box count may exceed 16 bits
  int y_off;           // table row 0 is image row y_off (carried band tables)
  // Octets holding a nonzero model bin, in bin order.  A bin whose model
  // value is 0 scores sqrt(0 * h) = +0 (Bhattacharyya) or min(0, h/mass) =
  // +0 (intersection), and s + (+0) == s, so the sweeps whose window mass is
  // closed-form (affine, quadratic, exponential) read and score only these
  // octets (SWG_SPARSE=0: every octet).  Bit-identical by construction.
  int nact;
  unsigned char act[kMaxBins / kOct];
  double model[kMaxBins];  // zero-padded to a multiple of 8
};

// Up to kQuadMulti quadratic maps of one table swept by one launch.
constexpr int kQuadMulti = 3;
struct QuadMulti {
  SweepArgs a[kQuadMulti];
  int gx[kQuadMulti], gy[kQuadMulti];  // each map's CTA tiles
  int n;
};

// Up to kCakeMulti full-ring square cake maps of one narrow (uint16) plain
// table swept by one launch (k_sweep_cake16_multi): every scale's ring boxes
// are the boxes of half-extent e = h .. 0 around the window centre, so a
// centre's box counts are loaded and formed once for all the scales and each
// scale accumulates its own coefficient of the box (in its own ring order:
// outer to inner, as WeddingCakePlan::histogram_into, baselines.cpp:139-148).
#ifndef SWG_CAKE_MULTI
#define SWG_CAKE_MULTI 4
#endif
constexpr int kCakeMulti = SWG_CAKE_MULTI;
constexpr int kCakeMultiSpan = 129;  // half-extents 0..128 (16-bit planes: kw*kh < 2^16 or wide0)
constexpr int kCakeMultiBins = 128;
struct CakeMulti {
  const void* tab;      // uint16 plain planes
  size_t plane_stride;  // records
  size_t pitch;         // records
  int planes, groups;
  int w, h;             // image; centres [hmin, w-1-hmin] x [hmin, h-1-hmin]
  int n;                // maps, half-extents descending
  int wide0;            // hs[0]'s outer box may hold >= 2^16 pixels
  int hs[kCakeMulti], mw[kCakeMulti];
  double* scores[kCakeMulti];
  PeakPart* parts[kCakeMulti];
  double coef[kCakeMulti][kCakeMultiSpan];  // ring coefficient of the box of half-extent e
  double model[kCakeMulti][kCakeMultiBins]; // zero-padded to a multiple of 8
};

constexpr int kPeakMulti = kQuadMulti > kCakeMulti ? kQuadMulti : kCakeMulti;
struct PeakMulti {  // k_peak_reduce over the maps of one multi-map launch
  const PeakPart* parts[kPeakMulti];
  int n[kPeakMulti], mw[kPeakMulti], hx[kPeakMulti], hy[kPeakMulti];
  swg_peak* out[kPeakMulti];
};

// Host-side ring plan of a wedding-cake configuration.
struct CakeRings {
  int a[kMaxRings];        // ring i box half-extent in x: hx - shrink_x[i]
  int c[kMaxRings];        // ring i box half-extent in y: hy - shrink_y[i]
  double coeff[kMaxRings]; // w_i - w_{i-1} (baselines.cpp:141)
};

// Kernel-side ring constants: the four box-corner offsets of ring i relative
// to the window centre's record, in BYTES and window independent --
// (TL, TR, BL, BR) = 32 * (-c*p - a, -c*p + a+1, (c+1)*p - a, (c+1)*p + a+1)
// with p = pitch in records -- and the ring coefficient.
struct CakeSweep {
  int4 off[kMaxRings];
  double coeff[kMaxRings];
};

// Exponential sweep constants: per orientation k (0 SE = TL quadrant,
// 1 h-flip = TR, 2 v-flip = BL, 3 hv-flip = BR) the byte offsets of the four
// rectangle corners from the window's centre record in that orientation and
// their coefficients (sign x decay powers x the quadrant's offset factor).
struct ExpSweep {
  int off[16];
  double coef[16];
  int w, h;     // image size (flip mapping)
  double snap;  // values below this are fp32 noise of an empty bin
  // Sparse mode (wmass > 0): every strict window holds one weight per pixel,
  // so its mass is the closed-form kernel sum wmass, and only the bin pairs
  // with a nonzero model value (pairs[0..npair)) are read and scored -- a
  // zero-model bin adds +0 to the score (the map stays within the fast
  // path's error bound; the exact peak is re-scored over every bin).
  double wmass;
  int npair;
  unsigned short pairs[kMaxBins / kDP];
};

// Two-phase exact peak of a tolerance-based map.
struct RescoreArgs {
  const uint16_t* fi;  // feature image (unflipped)
  size_t fi_pitch;
  const double* grid;  // kh x kw exact kernel weights (host-computed)
  int kw, kh;
  int* count;          // device candidate counter
  long long* cand;     // candidates (absolute map index)
  int cap;
  PeakPart* parts;     // one per rescore CTA
  double eps;
  int bins;            // all bins of the histogram (bin-range tables: the total)
  double model[kMaxBins];  // the full model
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
  size_t plane_stride, pitch;  // records
  int planes, bins;
  int n, tpw;
  const swg_term* terms;  // device
  long long* out;         // device n x bins
  const double* coeff;    // cake: per-term ring coefficient (n x tpw)
  double* outd;           // cake: device n x bins
};

// ---------------------------------------------------------------- peaks
// The reference's argmax rule (matching.cpp:211-223): strict `>` in
// row-major order, i.e. higher score, then smaller index.
__device__ __forceinline__ bool peak_better(double s, long long i, double s2, long long i2) {
  return s > s2 || (s == s2 && i < i2);
}

// Block argmax with the tie rule; thread 0 writes the CTA's candidate.
__device__ __forceinline__ void cta_peak(double s, long long idx, PeakPart* out) {
  __shared__ double ss[32];
  __shared__ long long si[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double s2 = __shfl_down_sync(0xFFFFFFFFu, s, off);
    const long long i2 = __shfl_down_sync(0xFFFFFFFFu, idx, off);
    if (peak_better(s2, i2, s, idx)) {
      s = s2;
      idx = i2;
    }
  }
  if (lane == 0) {
    ss[warp] = s;
    si[warp] = idx;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    s = lane < nw ? ss[lane] : -2.0;
    idx = lane < nw ? si[lane] : 0x7FFFFFFFFFFFFFFFLL;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double s2 = __shfl_down_sync(0xFFFFFFFFu, s, off);
      const long long i2 = __shfl_down_sync(0xFFFFFFFFu, idx, off);
      if (peak_better(s2, i2, s, idx)) {
        s = s2;
        idx = i2;
      }
    }
    if (lane == 0) *out = PeakPart{s, idx};
  }
}

// Sweep epilogue: this CTA's candidate into a.parts (k_peak_reduce, one
// CTA, then reduces them into the map peak).  A fused variant -- the last
// CTA of the sweep reducing them behind a ticket counter -- measured 0.35 %
// slower on config 2 (a fence + atomic in every CTA, a serial tail).
__device__ __forceinline__ void sweep_peak(double s, long long idx, const SweepArgs& a) {
  cta_peak(s, idx, a.parts + (size_t)blockIdx.y * gridDim.x + blockIdx.x);
}

// Map tile of this CTA.  Super-column order: the linear CTA index walks
// column strips of `sc_tiles` tiles, each from the top row to the bottom;
// CTAs are dispatched in linear order, so the CTAs in flight cover a strip
// of full height and every table row of the strip is read from DRAM once
// (as a window's bottom corner) and hit in L2 later (as a top corner).
__device__ __forceinline__ void sweep_tile(int sc_tiles, int& tx, int& ty) {
  const int gx = gridDim.x, gy = gridDim.y;
  if (sc_tiles <= 0 || sc_tiles >= gx) {
    tx = blockIdx.x;
    ty = blockIdx.y;
    return;
  }
  const int lin = blockIdx.y * gx + blockIdx.x;
  const int per_sc = sc_tiles * gy;
  const int sc = lin / per_sc, x0 = sc * sc_tiles;
  const int wsc = min(sc_tiles, gx - x0);
  const int rem = lin - sc * per_sc;
  ty = rem / wsc;
  tx = x0 + (rem - ty * wsc);
}

// Chain order (SweepArgs::chain_*): CTA (blockIdx.x = (tile column tx,
// chain step j, residue offset dv), blockIdx.y = residue group q) sweeps map
// row j * chain_s + q * chain_k + dv, so the CTAs in flight cover, for a
// few tile columns, every chain_s-th map row of the whole height: the table
// rows a window row reads as its lower corners are the rows the window row
// chain_s below reads as its upper corners, and both reads happen while the
// row is in L2 (the raster order's reuse distance of 2hy+1 map rows at full
// width does not fit in L2 at large windows).  Returns the map row, or
// a.rows (no row) for the padding residues of the last group.
__device__ __forceinline__ int chain_row(const SweepArgs& a, int& tx) {
  int rem = blockIdx.x;
  const int dv = rem % a.chain_k;
  rem /= a.chain_k;
  const int j = rem % a.chain_j, res = blockIdx.y * a.chain_k + dv;
  tx = rem / a.chain_j;
  return res < a.chain_s ? j * a.chain_s + res : a.rows;
}

// Sweep CTA geometry (affine, 32-bit cake): kSweepTileY warps; a
// warp = 16 windows of one map row, two lanes per window (lane parity =
// which half of each bin octet).
#ifndef SWG_SWEEP_TY
#define SWG_SWEEP_TY 8
#endif
#ifndef SWG_AFFINE_MINB
#define SWG_AFFINE_MINB 4  // 64 registers (explicit: config 5 Manhattan -4 % against the implicit 64)
#endif
constexpr int kSweepTileY = SWG_SWEEP_TY;
constexpr int kSweepThreads = 32 * kSweepTileY;
constexpr int kSweepTileX = 16;
// The quadratic sweep's CTA: 4 warps (measured against 8 warps: config 3
// 6.27 -> 5.95 ms per step, config 5's Euclidean scales -7 %; the affine
// sweep loses 3 % at 4 warps and keeps 8).
#ifndef SWG_QUAD_TY
#define SWG_QUAD_TY 4
#endif
#ifndef SWG_QUAD_MINB
#define SWG_QUAD_MINB 7  // 72 registers (64: config 5's Euclidean +6 %, 96: +6 %)
#endif
#ifndef SWG_QUADM_MINB
#define SWG_QUADM_MINB 8  // the multi-map launch: 64 registers (72: config 3 +2 %)
#endif
constexpr int kQuadTileY = SWG_QUAD_TY, kQuadThreads = 32 * kQuadTileY;
// 16-bit affine sweep (windows of mass < 2^16): one lane per window, CTAs
// of 32 windows x kAff16TileY map rows.
#ifndef SWG_AFF16_TY
#define SWG_AFF16_TY 4
#endif
constexpr int kAff16TileY = SWG_AFF16_TY, kAff16Threads = 32 * kAff16TileY;
// Exponential sweep CTA tile: kExpWarpsX warps side by side on one map row
// (32 windows each), kExpThreads / 32 / kExpWarpsX rows: 128 x 1 windows
// (measured: 128 x 2 +3 % on config 4 and +7 % on config 5's exponential
// scales; 64 x 2 and 256 x 1 slower too).
#ifndef SWG_EXP_WX
#define SWG_EXP_WX 4
#endif
#ifndef SWG_EXP_THREADS
#define SWG_EXP_THREADS 128
#endif
constexpr int kExpThreads = SWG_EXP_THREADS;
constexpr int kExpWarpsX = SWG_EXP_WX;
constexpr int kExpTileX = 32 * kExpWarpsX, kExpTileY = kExpThreads / 32 / kExpWarpsX;
// 16-bit cake sweep CTA tile: 32 windows x kCakeTileY map rows, a warp per
// row (measured on config 2: 4 rows 1.138 ms per step, 8 rows 1.151, 2 rows
// 1.153, 16 rows 1.211 -- taller tiles raise the L1 hit rate but cost
// occupancy and tail balance).
#ifndef SWG_CAKE_TY
#define SWG_CAKE_TY 4
#endif
#ifndef SWG_CAKE_MINB
#define SWG_CAKE_MINB 10  // <= 48 registers: 10 CTAs (40 warps) per SM; 40 registers spill (+3 %)
#endif
constexpr int kCakeTileY = SWG_CAKE_TY, kCakeThreads = 32 * kCakeTileY;
#ifndef SWG_CAKEM_MINB
#define SWG_CAKEM_MINB 3  // the multi-scale cake, whole records: up to 168 registers
#endif
#ifndef SWG_CAKEM_MINB4
#define SWG_CAKEM_MINB4 4  // half records: up to 128 registers
#endif
#ifndef SWG_CAKEM_ASYNC
#define SWG_CAKEM_ASYNC 1  // corners through a cp.async ring in shared memory
#endif
#ifndef SWG_CAKEM_STAGES
#define SWG_CAKEM_STAGES 3
#endif
#ifndef SWG_CAKEM_MINBA
#define SWG_CAKEM_MINBA 4  // the cp.async ring frees the in-flight registers: <= 128
#endif
#ifndef SWG_CAKEM_Q
#define SWG_CAKEM_Q 8  // bins per pass of the multi-scale cake (4: half records, measured slower)
#endif
// A cake16 warp covers kCakeWX x (32 / kCakeWX) windows: the lanes of a warp
// run until the last of them has emptied its octet's boxes, so compact warps
// (windows closer together, more similar inner bins) diverge less; a corner
// load is still 4 x 128-byte lines.
#ifndef SWG_CAKE_WX
#define SWG_CAKE_WX 32
#endif
constexpr int kCakeWX = SWG_CAKE_WX, kCakeWY = 32 / kCakeWX;
constexpr int kCakeCtaX = kCakeWX, kCakeCtaY = kCakeWY * kCakeTileY;
// Row-streaming chain sweeps (k_stream.cu): a CTA = kStreamWarps warps side
// by side (32 windows each, one lane per window) on a segment of at most
// kStreamLen windows of one chain.
#ifndef SWG_STREAM_LEN
#define SWG_STREAM_LEN 16
#endif
#ifndef SWG_STREAM_WARPS
#define SWG_STREAM_WARPS 4
#endif
// 5 CTAs per SM (<= 102 registers): config 5 Manhattan 2.87 -> 2.42 ms (96
// registers, no spill), Euclidean 3.82 -> 3.66 ms (96 registers, 60-76 B of
// spills); 6 per SM spills and loses on both
#ifndef SWG_STREAM_MINB
#define SWG_STREAM_MINB 5
#endif
#ifndef SWG_STREAMQ_MINB
#define SWG_STREAMQ_MINB 5
#endif
#ifndef SWG_STREAM16_MINB
#define SWG_STREAM16_MINB 6
#endif
constexpr int kStreamLen = SWG_STREAM_LEN;
constexpr int kStreamWarps = SWG_STREAM_WARPS, kStreamThreads = 32 * kStreamWarps;
constexpr int kStreamCols = 32 * kStreamWarps;
// Brute-force sweep: one thread per window.
constexpr int kBruteThreads = 128;

// A selective build's unit mask for the band-carry scans (by value).
struct SelMask {
  uint32_t w[kMaxBins / kDP / 32];
  int on;              // 0: every unit
  size_t words_per_unit;  // carry words of one unit per band
  __device__ __forceinline__ bool skip(size_t col) const {
    if (!on) return false;
    const size_t u = col / words_per_unit;
    return !((w[u >> 5] >> (u & 31)) & 1u);
  }
};
__host__ __device__ inline bool sel_has(const uint32_t* m, int nsel, int u) {
  return nsel == 0 || ((m[u >> 5] >> (u & 31)) & 1u);
}

// Lanes per carry word of the band scans (K1b, K1b'): enough to put ~1024
// threads on every SM, at most what covers the bands in one round of 10
// bands per lane (measured on config 5: 1, 2 and 4 lanes within 1 %, 8 lanes
// +4 %, a whole warp +16 %; SWG_BANDSCAN_Q forces a count: A/B).
inline int bandscan_lanes(int nbands, size_t words) {
  if (const char* e = std::getenv("SWG_BANDSCAN_Q")) {
    const int v = std::atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32) return v;
  }
  int q = 1;
  while (q < 32 && q * 10 < nbands && words * q < 148u * 1024u) q <<= 1;
  return q;
}

// Encode a row tensor map for TMA stores (swg_abi.cu): planes of records of
// rec_bytes, base = record 1 of row 0 of plane 0, box = box_lines 128-byte
// lines x 1 row.  Returns false when the driver entry point is unavailable.
bool encode_row_tmap(CUtensorMap* m, void* record1, int rec_bytes, int w, int h, size_t pitch,
                     size_t plane_stride, int nplanes, int box_lines);

// Kernel launchers (defined in the .cu files).
cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t s);
cudaError_t launch_colsum(const BuildArgs& a, cudaStream_t s);
template <typename T>
cudaError_t launch_build(const BuildArgs& a, cudaStream_t s, int* launches);
cudaError_t launch_sweep_affine(const SweepArgs& a, bool uniform, dim3 grid, cudaStream_t s);
cudaError_t launch_sweep_affine16(const SweepArgs& a, dim3 grid, cudaStream_t s);
dim3 stream_grid(bool narrow, int mw, int rows, int hy);
cudaError_t launch_stream_affine(const SweepArgs& a, bool narrow, dim3 grid, cudaStream_t s);
dim3 stream_quad_grid(int mw, int rows, int hy);
cudaError_t launch_stream_quad(const SweepArgs& a, dim3 grid, cudaStream_t s);
cudaError_t launch_sweep_cake(const SweepArgs& a, const CakeSweep& r, dim3 grid,
                              cudaStream_t s);
cudaError_t launch_sweep_quad(const SweepArgs& a, dim3 grid, cudaStream_t s);
cudaError_t launch_sweep_quad_multi(const QuadMulti& m, cudaStream_t s);
cudaError_t launch_peak_reduce_multi(const PeakMulti& m, int maps, cudaStream_t s);
cudaError_t launch_flip(const uint16_t* fi, size_t pitch, int w, int h, uint16_t* fh,
                        uint16_t* fv, uint16_t* fhv, cudaStream_t s);
// kind 0 / 2: carries (into a.agg) + strips of the unflipped / v-flipped
// orientation; kind 1 / 3: strips of its h-flipped partner (the carries
// kind - 1 left in a.agg, read mirrored); kind = -1: the carries of
// orientations 0 and 2 only (a.fio, slots 0 and 2 of a.agg); kind = -2:
// strips of all four orientations (a.fio, agg_stride)
cudaError_t launch_build_decay(const BuildArgs& a, double dec, int kind, cudaStream_t s,
                               int* launches);
cudaError_t launch_export_decay(const double* tab, size_t ps, size_t pitch, int w, int h,
                                int kind, int b0, int b1, double* out, cudaStream_t s);
cudaError_t launch_sweep_exp(const SweepArgs& a, const ExpSweep& e, dim3 grid, cudaStream_t s);
cudaError_t launch_exp_query(const double* tab, size_t ps, size_t pitch, int bins,
                             const ExpSweep& e, int n, const int* cx, const int* cy,
                             double* out, cudaStream_t s);
cudaError_t launch_exact_peak(const SweepArgs& a, const RescoreArgs& r, swg_peak* peak,
                              cudaStream_t s);
cudaError_t launch_sweep_cake16(const SweepArgs& a, const CakeSweep& r, dim3 grid,
                                cudaStream_t s);
dim3 cake_multi_grid(const CakeMulti& m);
cudaError_t launch_sweep_cake16_multi(const CakeMulti& m, cudaStream_t s);
cudaError_t launch_sweep_brute(const SweepArgs& a, const BruteArgs& b, int blocks_x,
                               cudaStream_t s);
cudaError_t launch_peak_reduce(const PeakPart* parts, int nparts, int mw, int hx, int hy,
                               swg_peak* out, cudaStream_t s);
template <typename T>
cudaError_t launch_query(const QueryArgs& a, cudaStream_t s);
cudaError_t launch_cake_query(const QueryArgs& a, cudaStream_t s);
template <typename T, typename O>
cudaError_t launch_export(const T* tab, size_t ps, size_t pitch, int planes, int w, int h,
                          int kind, int b0, int b1, O* out, cudaStream_t s);
cudaError_t launch_import_i64(const int64_t* src, int w, int h, int bins, int kind,
                              uint64_t* tab, size_t ps, size_t pitch, int planes,
                              cudaStream_t s);
cudaError_t launch_narrow(const uint64_t* src, uint32_t* dst, size_t n, cudaStream_t s);
cudaError_t launch_last_row(const uint32_t* tab, size_t ps, size_t pitch, int planes, int kinds,
                            int w, int h, int groups, void* out, cudaStream_t s);
cudaError_t launch_add_carry(uint32_t* tab, size_t ps, size_t pitch, int planes, int kinds, int w,
                             int h, int groups, int y0, const void* carry, cudaStream_t s);
// Brute-force histograms of explicit windows (API queries).
struct BruteQueryArgs {
  const uint16_t* fi;  // w*h, tight rows
  int w, h, bins, n;
  const int* cx;
  const int* cy;
  const double* grid;  // kh x kw weights
  int kw, kh, border, integer;
  long long* out_i64;  // n x bins (integer kernels)
  double* out_f64;     // n x bins
};
cudaError_t launch_brute_query(const BruteQueryArgs& a, cudaStream_t s);
cudaError_t launch_map_peak(const double* scores, size_t n, int mw, int hx, int hy,
                            PeakPart* parts, int nparts, swg_peak* out, cudaStream_t s);

}  // namespace swg
