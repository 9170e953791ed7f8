// k_decay.cu — decayed directional integral tables for the exponential
// kernel w = d^(|dx| + |dy|), d = exp(-lambda) (declared extension).
//
// The paper's directional weighted integral histograms IH_w (Eq. 2,
// the {SE, SW, NE, NW} quadrant weights) become, for an exponential kernel,
// DECAYED prefix sums
//   E(X, Y) = sum_{x < X, y < Y} f(x, y) d^(X-1-x) d^(Y-1-y)
// whose values stay bounded (<= 1/(1-d)^2) where e^{+lambda x} planes would
// overflow.  A quadrant rectangle [x0,x1] x [y0,y1] weighted by
// d^(x1-x) d^(y1-y) is then
//   E(x1+1,y1+1) - d^(x1-x0+1) E(x0,y1+1) - d^(y1-y0+1) E(x1+1,y0)
//                + d^(x1-x0+1) d^(y1-y0+1) E(x0,y0).
// The four orientations are the same SE table built on the feature image
// flipped horizontally / vertically / both (k_flip), so one build pipeline
// serves all four.  It mirrors the integer build: K1a' decayed column sums
// per band, K1b' decayed scan over bands, K1c' per (band, bin pair) CTA in
// column strips (column recurrence, then one warp scan per row segment).
// Layout: BIN PAIRS, not octets -- a record is the 2 bins of one pair at one
// cell (16 B of fp64), element (b, kind k, x, y) at
//   (((b/2)*4 + k)*plane_stride + y*pitch + x)*2 + b%2,
// with the pair count padded to a multiple of 4 (whole octets); the sweep
// reads 16-B records, 32 windows' records contiguous per warp.  fp64 storage
// and recurrences: fp32 noise (~1e-7 of the table values) is comparable to
// the smallest quadrant contributions at large windows and Bhattacharyya's
// sqrt amplifies it; fp64 keeps every map value within 1e-9 of the exact
// fp64 brute force (tolerance-based parity).
#include "swg_internal.cuh"

#include <math.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

namespace swg {

namespace {

using real = double;

// K0': flipped copies of the feature image (h: x -> W-1-x, v: y -> H-1-y).
__global__ void k_flip(const uint16_t* fi, size_t pitch, int w, int h, uint16_t* fh,
                       uint16_t* fv, uint16_t* fhv) {
  const int y = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < (int)pitch;
       x += gridDim.x * blockDim.x) {
    const bool in = x < w;
    const uint16_t a = in ? fi[(size_t)y * pitch + (w - 1 - x)] : kNoBin;
    const uint16_t b = fi[(size_t)(h - 1 - y) * pitch + x];
    const uint16_t c = in ? fi[(size_t)(h - 1 - y) * pitch + (w - 1 - x)] : kNoBin;
    fh[(size_t)y * pitch + x] = a;
    fv[(size_t)y * pitch + x] = b;
    fhv[(size_t)y * pitch + x] = c;
  }
}

// K1a': decayed column sums of one band: c(x) = sum_y [bin] d^(y1-1-y).
// agg: [nbands][pairs][wa] double2.  A thread covers kColPairs bin pairs of
// one column, so each pixel is read once per 2 * kColPairs bins.
#ifndef SWG_COL_PAIRS
#define SWG_COL_PAIRS 8  // 16 bins per thread (4 pairs: config 4 builds +0.4 ms)
#endif
constexpr int kColPairs = SWG_COL_PAIRS;
__global__ void __launch_bounds__(256) k_colsum_decay(const BuildArgs g, real dec, int pairs,
                                                      int nori) {
  // nori = 4: the four orientations in one launch (blockIdx.z = column block
  // * 4 + orientation, each with its image and carry array)
  const int band = blockIdx.x, pr0 = blockIdx.y * kColPairs;
  const int ori = nori > 1 ? (int)(blockIdx.z % nori) : 0;
  const int x = (int)(blockIdx.z / nori) * blockDim.x + threadIdx.x;
  if (x >= g.w) return;
  const uint16_t* gfi = nori > 1 ? g.fio[ori] : g.fi;
  double2* dst = reinterpret_cast<double2*>(g.agg + (nori > 1 ? (size_t)ori * g.agg_stride : 0));
  if (g.nsel) {  // selective build: pairs no sweep reads need no carries
    bool any = false;
    for (int k = 0; k < kColPairs && !any; ++k) any = pr0 + k < pairs && sel_has(g.selmask, g.nsel, pr0 + k);
    if (!any) return;
  }
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  const uint32_t gb = (uint32_t)g.bin0 + (uint32_t)pr0 * kDP;
  const uint32_t lim = (uint32_t)max(g.bins - pr0 * kDP, 0);  // bins of these pairs in range
  real c[2 * kColPairs];
#pragma unroll
  for (int j = 0; j < 2 * kColPairs; ++j) c[j] = 0.0;
  const uint16_t* col = gfi + x;
  for (int y = y0; y < y1; ++y) {
    uint32_t d = (uint32_t)col[(size_t)y * g.fi_pitch] - gb;
    d = d < lim ? d : 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < 2 * kColPairs; ++j) c[j] = fma(dec, c[j], d == (uint32_t)j ? 1.0 : 0.0);
  }
  
#pragma unroll
  for (int q = 0; q < kColPairs; ++q)
    if (pr0 + q < pairs)
      dst[((size_t)band * pairs + pr0 + q) * g.wa + x] = make_double2(c[2 * q], c[2 * q + 1]);
}

// K1b': C_0 = 0, C_{b+1} = d^(h_b) C_b + c_b (exclusive over bands, in place);
// one warp per column word, lanes = 32 bands, affine shuffle scan.
__global__ void __launch_bounds__(256) k_bandscan_decay(real* agg, int nbands, int band_h,
                                                        int h, real dband, real dlast,
                                                        size_t per_band, const SelMask m,
                                                        int nori, size_t ori_stride) {
  const size_t cw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (cw >= per_band * nori) return;
  const size_t col = cw % per_band;
  if (m.skip(col)) return;
  agg += (cw / per_band) * ori_stride;
  real run = 0.0;
  for (int b0 = 0; b0 < nbands; b0 += 32) {
    const int b = b0 + lane;
    // d^(rows of band b): every band but the last has band_h rows (host powers)
    real ia = b < nbands ? (b == nbands - 1 ? dlast : dband) : 1.0;
    real inc = b < nbands ? agg[(size_t)b * per_band + col] : 0.0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const real pa = __shfl_up_sync(0xFFFFFFFFu, ia, off);
      const real pv = __shfl_up_sync(0xFFFFFFFFu, inc, off);
      if (lane >= off) {
        inc = fma(ia, pv, inc);
        ia *= pa;
      }
    }
    const real pa = __shfl_up_sync(0xFFFFFFFFu, ia, 1);
    const real pv = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
    const real ent = lane > 0 ? fma(pa, run, pv) : run;
    if (b < nbands) agg[(size_t)b * per_band + col] = ent;
    run = fma(__shfl_sync(0xFFFFFFFFu, ia, 31), run, __shfl_sync(0xFFFFFFFFu, inc, 31));
  }
}

// K1b', sequential form: one thread per column word walks the bands in order
// (loads of 8 bands in flight); see k_bandscan_seq.
__global__ void __launch_bounds__(256) k_bandscan_decay_seq(real* agg, int nbands, real dband,
                                                            real dlast, size_t per_band,
                                                            const SelMask m, int nori,
                                                            size_t ori_stride) {
  const size_t cw = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (cw >= per_band * nori) return;
  const size_t col = cw % per_band;  // (orientation cw / per_band)
  if (m.skip(col)) return;
  agg += (cw / per_band) * ori_stride;
  real run = 0.0;
  constexpr int kB = 8;
  for (int b0 = 0; b0 < nbands; b0 += kB) {
    real v[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) v[k] = b0 + k < nbands ? agg[(size_t)(b0 + k) * per_band + col] : 0.0;
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int b = b0 + k;
      if (b < nbands) {
        agg[(size_t)b * per_band + col] = run;
        run = fma(b == nbands - 1 ? dlast : dband, run, v[k]);
      }
    }
  }
}

// K1c': decayed SE table of one orientation, column recurrence first.  With
//   c(x, y) = d c(x, y-1) + f(x, y)        (c(x, y0-1) = the band's carry, K1b')
//   E(x+1, y+1) = sum_{x' <= x} d^(x-x') c(x', y)
// one CTA per (band, bin pair) walks the row in strips of kStripW columns and
// the band in blocks of kStripRows rows: phase A (thread per column) runs the
// column recurrence down the block into a shared tile; phase B (warp per row,
// lane = 8 consecutive columns) forms the decayed row prefix with one warp
// scan per row and the carry E(x0-1, y) of the strip to the left; phase C
// (thread per column, fused with the next block's phase A) writes the tile
// out as 512-byte warp stores.  Two block barriers per 16 rows instead of a
// block-wide scan and barrier per row.
#ifndef SWG_STRIP_ROWS
#define SWG_STRIP_ROWS 8  // 8-row blocks at 4 CTAs per SM: config 5 decayed set 2.82 -> 2.74 ms (16 rows at 3)
#endif
#ifndef SWG_STRIP_MINB
#define SWG_STRIP_MINB 4
#endif
constexpr int kStripW = 256, kStripRows = SWG_STRIP_ROWS;

__device__ __forceinline__ int strip_swz(int x) { return x ^ ((x >> 3) & 7); }

__global__ void __launch_bounds__(kStripW, SWG_STRIP_MINB)
    k_build_decay_strip(const __grid_constant__ BuildArgs g, real dec, int kind, int pairs) {
  // [kStripRows][kStripW] swizzled (= the TMA SWIZZLE_128B layout of each
  // 4 KB row), then carry[band_h]
  extern __shared__ __align__(1024) double2 s_tile[];
  const bool tma = g.tmap_ok != 0;
  double2* carry = s_tile + kStripRows * kStripW;
  if (gridDim.y > 1) kind = blockIdx.y;  // all four orientations in one launch
  const uint16_t* gfi = gridDim.y > 1 ? g.fio[kind] : g.fi;
  const uint32_t* gagg = g.agg + (gridDim.y > 1 ? (size_t)kind * g.agg_stride : 0);
  const int np = g.nsel ? g.nsel : pairs;  // selective build: the listed pairs
  const int band = blockIdx.x / np, pr = g.nsel ? (int)g.sel[blockIdx.x % np] : blockIdx.x % np;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kStripW / 32;
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  const int nrows = y1 - y0;
  // the pair's two global bins (~0: bin out of range, no pixel matches)
  const int nin = g.bins - pr * kDP;  // bins of this pair in range
  const uint32_t gb0 = nin > 0 ? (uint32_t)g.bin0 + (uint32_t)pr * kDP : 0xFFFFFFFFu;
  const uint32_t gb1 = nin > 1 ? gb0 + 1 : 0xFFFFFFFFu;
  const real d2 = dec * dec, d4 = d2 * d2, d8 = d4 * d4;
  real p8l = 1.0;  // d^(8 lane): carry from the left strip to this lane's first column
  {
    real p = d8;
    for (int k = lane; k; k >>= 1) {
      if (k & 1) p8l *= p;
      p *= p;
    }
  }
  double2* plane = reinterpret_cast<double2*>(g.out) +
                   ((size_t)pr * g.planes + kind) * g.plane_stride;
  const double2 zero = make_double2(0.0, 0.0);
  if (band == 0)
    for (int x = tid; x <= g.w; x += kStripW) plane[x] = zero;
  for (int r = tid; r < nrows; r += kStripW) {
    plane[(size_t)(y0 + r + 1) * g.pitch] = zero;
    carry[r] = zero;
  }
  const double2* agg = reinterpret_cast<const double2*>(gagg) + ((size_t)band * pairs + pr) * g.wa;
  const int sw = strip_swz(tid);
  auto step = [&](uint32_t v, real& c0, real& c1) {
    c0 = fma(dec, c0, v == gb0 ? 1.0 : 0.0);
    c1 = fma(dec, c1, v == gb1 ? 1.0 : 0.0);
  };
  for (int x0 = 0; x0 < g.w; x0 += kStripW) {
    const int x = x0 + tid;
    const bool in = x < g.w;
    real c0 = 0.0, c1 = 0.0;
    if (in && band > 0) {
      const double2 v = agg[x];
      c0 = v.x;
      c1 = v.y;
    }
    // pixel column x of the band (kNoBin beyond the image) and its table column
    const uint16_t* col = gfi + (size_t)y0 * g.fi_pitch + (in ? x : 0);
    const size_t fstep = in ? g.fi_pitch : 0;
    const uint32_t vor = in ? 0u : 0x10000u;  // beyond the image: a value no bin matches
    double2* out = plane + (size_t)(y0 + 1) * g.pitch + x + 1;
    int prev = 0;  // rows of the previous block still in the tile (phase C pending)
    for (int rb = 0;; rb += kStripRows) {
      const int nr = min(kStripRows, nrows - rb);
      if (tma) {  // phase C is the TMA stores: the tile is free once they have read it
        if (nr <= 0) break;
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
      }
      // C (previous block) + A (this block): the same thread, the same tile slots
      if (in && !tma) {
        if (prev == kStripRows) {
#pragma unroll
          for (int r = 0; r < kStripRows; ++r) {
            *out = s_tile[r * kStripW + sw];
            out += g.pitch;
          }
        } else {
          for (int r = 0; r < prev; ++r) {
            *out = s_tile[r * kStripW + sw];
            out += g.pitch;
          }
        }
      }
      if (nr <= 0) break;
      {  // all of the block's loads in flight at once (a partial block predicates)
        uint32_t fv[kStripRows];
#pragma unroll
        for (int r = 0; r < kStripRows; ++r) fv[r] = r < nr ? col[r * fstep] : 0u;
        col += kStripRows * fstep;
#pragma unroll
        for (int r = 0; r < kStripRows; ++r)
          if (r < nr) {
            step(fv[r] | vor, c0, c1);
            s_tile[r * kStripW + sw] = make_double2(c0, c1);
          }
      }
      __syncthreads();
      // B: decayed row prefix, one warp per row
      for (int r = warp; r < nr; r += kWarps) {
        double2* trow = s_tile + r * kStripW;
        real v0[8], v1[8];
        real run0 = 0.0, run1 = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double2 q = trow[8 * lane + (i ^ (lane & 7))];
          run0 = fma(dec, run0, q.x);
          run1 = fma(dec, run1, q.y);
          v0[i] = run0;
          v1[i] = run1;
        }
        real i0 = run0, i1 = run1;  // inclusive scan of the lanes' totals
        real sk = d8;               // (d^8)^(2^k)
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const real t0 = __shfl_up_sync(0xFFFFFFFFu, i0, 1 << k);
          const real t1 = __shfl_up_sync(0xFFFFFFFFu, i1, 1 << k);
          if (lane >= (1 << k)) {
            i0 = fma(sk, t0, i0);
            i1 = fma(sk, t1, i1);
          }
          sk *= sk;
        }
        real e0 = __shfl_up_sync(0xFFFFFFFFu, i0, 1), e1 = __shfl_up_sync(0xFFFFFFFFu, i1, 1);
        if (lane == 0) e0 = e1 = 0.0;
        const double2 cin = carry[rb + r];
        const real q0 = fma(p8l, cin.x, e0), q1 = fma(p8l, cin.y, e1);
        real pw = dec;  // d^(i+1)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v0[i] = fma(pw, q0, v0[i]);
          v1[i] = fma(pw, q1, v1[i]);
          trow[8 * lane + (i ^ (lane & 7))] = make_double2(v0[i], v1[i]);
          pw *= dec;
        }
        const real n0 = __shfl_sync(0xFFFFFFFFu, v0[7], 31);
        const real n1 = __shfl_sync(0xFFFFFFFFu, v1[7], 31);
        if (lane == 0) carry[rb + r] = make_double2(n0, n1);  // E(x0 + kStripW - 1, y)
      }
      if (tma) {
        // C: one TMA tensor store per row (records x0+1 .. x0+256: 32 lines of
        // 128 B; the tensor's bounds clip the strip at the image's edge)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
          const int plane_i = pr * g.planes + kind;
          for (int r = 0; r < nr; ++r) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(s_tile + r * kStripW);
            asm volatile(
                "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                ::"l"(&g.tmap), "r"(0), "r"(x0 / 8), "r"(y0 + rb + r + 1), "r"(plane_i), "r"(sa)
                : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else {
        __syncthreads();
      }
      prev = nr;
    }
  }
  if (tma && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Decay-table export: planes [b0, b1) of orientation `kind` -> (W+1)x(H+1) each.
__global__ void k_export_decay(const double* tab, size_t ps, size_t pitch, int w, int h,
                               int kind, int b0, double* out) {
  const int b = b0 + blockIdx.z, y = blockIdx.y;
  const size_t base = ((size_t)(b >> 1) * 4 + kind) * ps + (size_t)y * pitch;
  double* o = out + ((size_t)blockIdx.z * (h + 1) + y) * (w + 1);
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x <= w; x += gridDim.x * blockDim.x)
    o[x] = tab[(base + x) * kDP + (b & 1)];
}

}  // namespace

cudaError_t launch_flip(const uint16_t* fi, size_t pitch, int w, int h, uint16_t* fh,
                        uint16_t* fv, uint16_t* fhv, cudaStream_t s) {
  dim3 grid((unsigned)((pitch + 255) / 256), (unsigned)h);
  k_flip<<<grid, 256, 0, s>>>(fi, pitch, w, h, fh, fv, fhv);
  return cudaGetLastError();
}

cudaError_t launch_build_decay(const BuildArgs& a, double dec, int kind, cudaStream_t s,
                               int* launches) {
  *launches = 0;
  const int pairs = a.groups * (kOct / kDP);
  if (a.nbands > 1 && kind != -2) {
    // kind == -1: the carries of all four orientations (a.fio, agg_stride)
    const int nori = kind == -1 ? 4 : 1;
    dim3 grid((unsigned)a.nbands, (unsigned)((pairs + kColPairs - 1) / kColPairs),
              (unsigned)((a.w + 255) / 256 * nori));
    k_colsum_decay<<<grid, 256, 0, s>>>(a, dec, pairs, nori);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t per_band = (size_t)pairs * a.wa * kDP;
    const double dband = std::pow(dec, (double)a.band_h);
    const double dlast = std::pow(dec, (double)(a.h - (a.nbands - 1) * a.band_h));
    SelMask m{};
    m.on = a.nsel > 0;
    m.words_per_unit = a.wa * kDP;
    std::memcpy(m.w, a.selmask, sizeof(m.w));
    const char* bw = std::getenv("SWG_BANDSCAN_WARP");  // A/B: 1 = warp-per-word scan
    const size_t ori_stride = a.agg_stride / 2;  // doubles
    if (bw ? std::atoi(bw) != 0 : per_band * nori < 148u * 256u)  // few words: a warp each
      k_bandscan_decay<<<(unsigned)((per_band * nori * 32 + 255) / 256), 256, 0, s>>>(
          reinterpret_cast<double*>(a.agg), a.nbands, a.band_h, a.h, dband, dlast, per_band, m,
          nori, ori_stride);
    else
      k_bandscan_decay_seq<<<(unsigned)((per_band * nori + 255) / 256), 256, 0, s>>>(
          reinterpret_cast<double*>(a.agg), a.nbands, dband, dlast, per_band, m, nori,
          ori_stride);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches += 2;
  }
  if (kind == -1) return cudaSuccess;  // carries only
  const dim3 grid((unsigned)(a.nbands * (a.nsel ? a.nsel : pairs)), kind == -2 ? 4u : 1u);
  const size_t smem = (size_t)(kStripRows * kStripW + a.band_h) * sizeof(double2);
  if (smem > (200 << 10)) return cudaErrorInvalidConfiguration;  // band_h > ~8500 rows
  // set on every launch: the attribute is per device (a process-wide cache
  // would skip it on a second device and race between host threads)
  cudaFuncSetAttribute(k_build_decay_strip, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       200 << 10);
  k_build_decay_strip<<<grid, kStripW, smem, s>>>(a, dec, kind, pairs);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_export_decay(const double* tab, size_t ps, size_t pitch, int w, int h,
                                int kind, int b0, int b1, double* out, cudaStream_t s) {
  dim3 grid((unsigned)((w + 1 + 255) / 256), (unsigned)(h + 1), (unsigned)(b1 - b0));
  k_export_decay<<<grid, 256, 0, s>>>(tab, ps, pitch, w, h, kind, b0, out);
  return cudaGetLastError();
}

}  // namespace swg
