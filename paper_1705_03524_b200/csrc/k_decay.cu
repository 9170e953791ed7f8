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
// per band, K1b' decayed scan over bands, K1c' one warp per (band, bin pair) in
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

#include <algorithm>
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

// K0', 8 pixels per thread (widths that are multiples of 8: the mirrored
// chunk of a row is then 16-byte aligned too).
__device__ __forceinline__ uint4 rev8(const uint4 v) {  // 8 uint16 in reverse order
  auto sw = [](uint32_t w) { return (w >> 16) | (w << 16); };
  return make_uint4(sw(v.w), sw(v.z), sw(v.y), sw(v.x));
}
__global__ void __launch_bounds__(256) k_flip_v8(const uint16_t* fi, size_t pitch, int w, int h,
                                                 uint16_t* fh, uint16_t* fv, uint16_t* fhv) {
  const int y = blockIdx.y;
  const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (x0 >= (int)pitch) return;
  const uint4 pad = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  const bool in = x0 < w;  // (w % 8 == 0: a chunk is all image or all padding)
  const uint16_t* r0 = fi + (size_t)y * pitch;
  const uint16_t* r1 = fi + (size_t)(h - 1 - y) * pitch;
  const uint4 a = in ? rev8(*reinterpret_cast<const uint4*>(r0 + (w - 8 - x0))) : pad;
  const uint4 b = *reinterpret_cast<const uint4*>(r1 + x0);
  const uint4 c = in ? rev8(*reinterpret_cast<const uint4*>(r1 + (w - 8 - x0))) : pad;
  *reinterpret_cast<uint4*>(fh + (size_t)y * pitch + x0) = a;
  *reinterpret_cast<uint4*>(fv + (size_t)y * pitch + x0) = b;
  *reinterpret_cast<uint4*>(fhv + (size_t)y * pitch + x0) = c;
}

// K1a': decayed column sums of one band: c(x) = sum_y [bin] d^(y1-1-y).
// agg: [nbands][pairs][wa] double2.
// A thread owns one column and keeps each bin's running sum in SHARED memory
// with the row it was last updated at (sums[slot bin][thread], private to
// the thread): a pixel of bin b at row r costs one update
//   c_b <- c_b d^(r - last_b) + 1,  last_b <- r
// with the powers from a shared table, whatever the bin count, and the sums
// are decayed to the band's last row at the end.  (The first form ran the
// recurrence c <- d c + [bin] for every bin of 8 pairs at every pixel in
// registers: 16 fp64 operations per pixel and pair group, the pixels re-read
// per group; config 5 136 us for the model's pairs of four orientations.)
// The bins summed are the pairs the build will read (a selective build's,
// else all), in chunks of as many pairs as the shared memory holds.
constexpr int kDColThreads = 128;
constexpr int kDColSmem = 96 << 10;
__global__ void __launch_bounds__(kDColThreads) k_colsum_decay(const BuildArgs g, real dec,
                                                               int pairs, int nori, int ppc) {
  // nori = 2: the unflipped and the v-flipped image in one launch (blockIdx.y
  // = column block * 2 + which), into carry slots 0 and 2.  The h-flipped
  // orientations need no pass of their own: column x of an h-flipped image
  // is column W-1-x of the unflipped one, over the same rows, so their
  // carries are slot 0's / slot 2's read mirrored (k_build_decay_warp).
  extern __shared__ __align__(16) unsigned char s_raw[];
  __shared__ unsigned char s_slot[kMaxBins / kDP];  // pair -> slot of this chunk (0xFF: none)
  const int tid = threadIdx.x, band = blockIdx.x;
  const int ori = nori > 1 ? 2 * (int)(blockIdx.y % nori) : 0;
  const int x = (int)(blockIdx.y / nori) * kDColThreads + tid;
  const int np = g.nsel ? g.nsel : pairs;
  const int p0 = blockIdx.z * ppc, slots = min(ppc, np - p0);
  const int nb = slots * kDP;
  real* cs = reinterpret_cast<real*>(s_raw);              // [nb][threads]
  real* dpow = cs + (size_t)ppc * kDP * kDColThreads;     // d^k, k = 0 .. band_h
  uint16_t* last = reinterpret_cast<uint16_t*>(dpow + g.band_h + 1);  // [nb][threads]
  for (int i = tid; i < pairs; i += kDColThreads) s_slot[i] = 0xFF;
  __syncthreads();
  if (tid < slots) s_slot[g.nsel ? (int)g.sel[p0 + tid] : p0 + tid] = (unsigned char)tid;
  for (int i = tid; i < nb * kDColThreads; i += kDColThreads) {
    cs[i] = 0.0;
    last[i] = 0;
  }
  for (int k = tid; k <= g.band_h; k += kDColThreads) {
    real r = 1.0, p = dec;
    for (int e = k; e; e >>= 1) {
      if (e & 1) r *= p;
      p *= p;
    }
    dpow[k] = r;
  }
  __syncthreads();
  if (x >= g.w) return;
  const uint16_t* gfi = nori > 1 ? g.fio[ori] : g.fi;
  double2* dst = reinterpret_cast<double2*>(g.agg + (nori > 1 ? (size_t)ori * g.agg_stride : 0));
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  const int nrows = y1 - y0;
  const uint16_t* col = gfi + (size_t)y0 * g.fi_pitch + x;
  constexpr int kB = 8;  // rows whose pixels are in flight at once
  for (int rb = 0; rb < nrows; rb += kB) {
    uint32_t v[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) v[k] = rb + k < nrows ? (uint32_t)col[(size_t)(rb + k) * g.fi_pitch] : 0xFFFFu;
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const uint32_t d = v[k] - (uint32_t)g.bin0;
      if (d >= (uint32_t)g.bins) continue;  // another range's bin, or padding
      const uint32_t sl = s_slot[d >> 1];
      if (sl == 0xFFu) continue;
      const int i = (int)(sl * kDP + (d & 1u)) * kDColThreads + tid;
      const int r = rb + k;
      cs[i] = fma(cs[i], dpow[r - (int)last[i]], 1.0);
      last[i] = (uint16_t)r;
    }
  }
  for (int sl = 0; sl < slots; ++sl) {
    const int pr = g.nsel ? (int)g.sel[p0 + sl] : p0 + sl;
    const int i0 = sl * kDP * kDColThreads + tid, i1 = i0 + kDColThreads;
    dst[((size_t)band * pairs + pr) * g.wa + x] =
        make_double2(cs[i0] * dpow[nrows - 1 - (int)last[i0]], cs[i1] * dpow[nrows - 1 - (int)last[i1]]);
  }
}

// K1b': C_0 = 0, C_{b+1} = d^(h_b) C_b + c_b (exclusive over bands, in place).
// Q lanes share one column word, as in k_bandscan: each loads its 10 bands at
// once and folds them into an affine map (A, V): C -> A C + V; the lanes'
// maps are composed by a Q-wide shuffle scan, and each lane replays its bands
// from the value entering it.
constexpr int kBandPT = 10;
__global__ void __launch_bounds__(256) k_bandscan_decay(real* agg, int nbands, real dband,
                                                        real dlast, size_t per_band,
                                                        const SelMask m, int nori,
                                                        size_t ori_stride, int q) {
  const size_t gt = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t cw = gt / q;  // (orientation cw / per_band, word cw % per_band)
  const int sub = (int)(gt % q);
  const size_t col = cw % per_band;
  const bool act = cw < per_band * nori && !m.skip(col);  // (every lane stays for the shuffles)
  if (act) agg += (cw / per_band) * ori_stride;
  real run = 0.0;
  for (int b0 = 0; b0 < nbands; b0 += q * kBandPT) {
    const int bs = b0 + sub * kBandPT;
    real v[kBandPT];
#pragma unroll
    for (int k = 0; k < kBandPT; ++k)
      v[k] = act && bs + k < nbands ? agg[(size_t)(bs + k) * per_band + col] : 0.0;
    // this lane's bands as one affine map (bands past the end: the identity)
    real A = 1.0, V = 0.0;
#pragma unroll
    for (int k = 0; k < kBandPT; ++k) {
      const real f = bs + k < nbands ? (bs + k == nbands - 1 ? dlast : dband) : 1.0;
      V = fma(f, V, v[k]);
      A *= f;
    }
    real ia = A, iv = V;  // inclusive composition over the lanes of the word
    for (int off = 1; off < q; off <<= 1) {
      const real pa = __shfl_up_sync(0xFFFFFFFFu, ia, off, q);
      const real pv = __shfl_up_sync(0xFFFFFFFFu, iv, off, q);
      if (sub >= off) {
        iv = fma(ia, pv, iv);
        ia *= pa;
      }
    }
    const real ea = __shfl_up_sync(0xFFFFFFFFu, ia, 1, q);
    const real ev = __shfl_up_sync(0xFFFFFFFFu, iv, 1, q);
    real cur = sub > 0 ? fma(ea, run, ev) : run;  // the value entering this lane's bands
#pragma unroll
    for (int k = 0; k < kBandPT; ++k) {
      if (act && bs + k < nbands) {
        agg[(size_t)(bs + k) * per_band + col] = cur;
        cur = fma(bs + k == nbands - 1 ? dlast : dband, cur, v[k]);
      }
    }
    run = fma(__shfl_sync(0xFFFFFFFFu, ia, q - 1, q), run, __shfl_sync(0xFFFFFFFFu, iv, q - 1, q));
  }
}

constexpr int kStripW = 256;  // columns per strip: 8 per lane

__device__ __forceinline__ int strip_swz(int x) { return x ^ ((x >> 3) & 7); }

// K1c': decayed SE table of one orientation.  With
//   c(x, y) = d c(x, y-1) + f(x, y)        (c(x, y0-1) = the band's carry, K1b')
//   E(x+1, y+1) = sum_{x' <= x} d^(x-x') c(x', y)
// one WARP builds one (band, bin pair, orientation) unit, with no block
// barrier anywhere: the warp walks the row in strips of kStripW columns,
// lane l owning columns 8l .. 8l+7 of the strip, and runs BOTH recurrences
// for them row by row -- the column recurrence in registers (16 running
// values) and the decayed row prefix (its 8 columns, one warp scan, and the
// carry E(x0-1, y) of the strip to the left, kept per row in shared memory).
// The finished 4 KB row segment goes into one of kWarpRows swizzled row
// buffers (= the TMA SWIZZLE_128B layout) and out through one TMA tensor
// store; the next rows are built while earlier stores drain.
// (The first form gave a CTA one unit: threads ran the column recurrence
// into a shared 8-row tile, warps the row prefixes, two to three block
// barriers per 8 rows.  Each record crossed shared memory four times and
// ncu showed barrier stalls on top of an instruction-bound loop -- 542 warp
// instructions per 4 KB row segment against 339 here; config 5's decayed set
// 1.03 -> 0.85 ms.  Same operation order per value: identical tables.)
constexpr int kWarpRows = 3;  // row buffers per warp (4 KB each)
constexpr int kWarpsPerCta = 8;  // (fewer when the bands are tall: the carries share the CTA's shared memory)

__global__ void __launch_bounds__(32 * kWarpsPerCta, 2)
    k_build_decay_warp(const __grid_constant__ BuildArgs g, real dec, int kind, int pairs,
                       int nori) {
  extern __shared__ __align__(1024) double2 s_tile[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;  // warps (units) per CTA
  const int np = g.nsel ? g.nsel : pairs;
  const long long unit = (long long)blockIdx.x * wpc + warp;
  if (unit >= (long long)g.nbands * np * nori) return;  // (no block barriers below)
  const int pr = g.nsel ? (int)g.sel[unit % np] : (int)(unit % np);
  const int band = (int)((unit / np) % g.nbands);
  if (nori > 1) kind = (int)(unit / np / g.nbands);
  const uint16_t* gfi = nori > 1 ? g.fio[kind] : g.fi;
  // carries: slot 0 (unflipped) or 2 (v-flipped); an h-flipped orientation
  // reads its partner's columns mirrored
  const uint32_t* gagg = g.agg + (nori > 1 ? (size_t)(kind & 2) * g.agg_stride : 0);
  const bool mirror = (kind & 1) != 0;
  double2* rowbuf = s_tile + (size_t)warp * kWarpRows * kStripW;
  double2* carry = s_tile + (size_t)wpc * kWarpRows * kStripW + (size_t)warp * g.band_h;
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  const int nrows = y1 - y0;
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
    for (int x = lane; x <= g.w; x += 32) plane[x] = zero;
  for (int r = lane; r < nrows; r += 32) {
    plane[(size_t)(y0 + r + 1) * g.pitch] = zero;
    carry[r] = zero;
  }
  __syncwarp();
  const double2* agg = reinterpret_cast<const double2*>(gagg) + ((size_t)band * pairs + pr) * g.wa;
  const bool tma = g.tmap_ok != 0;
  const int plane_i = pr * g.planes + kind;
  const uint4 nopix = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  int slot = 0;
  for (int x0 = 0; x0 < g.w; x0 += kStripW) {
    const int xl = x0 + 8 * lane;  // this lane's first column
    const bool inp = (size_t)xl < g.fi_pitch;  // its 8 pixels lie inside the padded row
    real c0[8], c1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      c0[i] = c1[i] = 0.0;
      if (band > 0 && xl + i < g.w) {
        const double2 v = agg[mirror ? g.w - 1 - (xl + i) : xl + i];
        c0[i] = v.x;
        c1[i] = v.y;
      }
    }
    const uint16_t* prow = gfi + (size_t)y0 * g.fi_pitch + (inp ? xl : 0);
    // pixels two rows ahead of the row being built
    uint4 pa = inp && 0 < nrows ? __ldg(reinterpret_cast<const uint4*>(prow)) : nopix;
    uint4 pb = inp && 1 < nrows ? __ldg(reinterpret_cast<const uint4*>(prow + g.fi_pitch)) : nopix;
    for (int r = 0; r < nrows; ++r) {
      const uint4 px = pa;
      pa = pb;
      pb = inp && r + 2 < nrows
               ? __ldg(reinterpret_cast<const uint4*>(prow + (size_t)(r + 2) * g.fi_pitch))
               : nopix;
      const uint32_t w4[4] = {px.x, px.y, px.z, px.w};
      real v0[8], v1[8];
      real run0 = 0.0, run1 = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // (columns >= W hold kNoBin: no bin matches)
        const uint32_t v = (w4[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
        c0[i] = fma(dec, c0[i], v == gb0 ? 1.0 : 0.0);
        c1[i] = fma(dec, c1[i], v == gb1 ? 1.0 : 0.0);
        run0 = fma(dec, run0, c0[i]);
        run1 = fma(dec, run1, c1[i]);
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
      const double2 cin = carry[r];
      const real q0 = fma(p8l, cin.x, e0), q1 = fma(p8l, cin.y, e1);
      double2* buf = rowbuf + slot * kStripW;
      if (tma) {  // the store that last read this row buffer is done with it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kWarpRows - 1) : "memory");
      }
      __syncwarp();
      real pw = dec;  // d^(i+1)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v0[i] = fma(pw, q0, v0[i]);
        v1[i] = fma(pw, q1, v1[i]);
        buf[8 * lane + (i ^ (lane & 7))] = make_double2(v0[i], v1[i]);
        pw *= dec;
      }
      const real n0 = __shfl_sync(0xFFFFFFFFu, v0[7], 31);
      const real n1 = __shfl_sync(0xFFFFFFFFu, v1[7], 31);
      if (lane == 0) carry[r] = make_double2(n0, n1);  // E(x0 + kStripW - 1, y)
      if (tma) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf);
          asm volatile(
              "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
              ::"l"(&g.tmap), "r"(0), "r"(x0 / 8), "r"(y0 + r + 1), "r"(plane_i), "r"(sa)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else {
        __syncwarp();
        double2* out = plane + (size_t)(y0 + r + 1) * g.pitch + x0 + 1;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int c = m * 32 + lane;
          if (x0 + c < g.w) out[c] = buf[strip_swz(c)];
        }
        __syncwarp();
      }
      slot = slot + 1 == kWarpRows ? 0 : slot + 1;
    }
  }
  if (tma && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
  if (w % 8 == 0) {
    dim3 g8((unsigned)((pitch / 8 + 255) / 256), (unsigned)h);
    k_flip_v8<<<g8, 256, 0, s>>>(fi, pitch, w, h, fh, fv, fhv);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((pitch + 255) / 256), (unsigned)h);
  k_flip<<<grid, 256, 0, s>>>(fi, pitch, w, h, fh, fv, fhv);
  return cudaGetLastError();
}

cudaError_t launch_build_decay(const BuildArgs& a, double dec, int kind, cudaStream_t s,
                               int* launches) {
  *launches = 0;
  const int pairs = a.groups * (kOct / kDP);
  if (a.nbands > 1 && kind != -2 && !(kind & 1 && kind > 0)) {
    // kind == -1: the carries of the unflipped and the v-flipped image
    // (a.fio[0], a.fio[2] -> slots 0 and 2 of a.agg); kind 0 / 2: of a.fi.
    // Kinds 1 and 3 (h-flipped) read the carries kind 0 / 2 left in a.agg.
    const int nori = kind == -1 ? 2 : 1;
    // pairs per chunk: as many as kDColSmem holds beside the power table
    // (10 bytes per bin and thread: the sum and its last row)
    const int np = a.nsel ? a.nsel : pairs;
    const size_t per_pair = (size_t)kDP * kDColThreads * (sizeof(double) + sizeof(uint16_t));
    const size_t tab = (size_t)(a.band_h + 1) * sizeof(double);
    if (a.band_h > 65535 || tab + per_pair > (size_t)kDColSmem) return cudaErrorInvalidConfiguration;
    const int ppc = (int)std::min<size_t>((size_t)np, (kDColSmem - tab) / per_pair);
    const size_t csm = (size_t)ppc * per_pair + tab;
    dim3 grid((unsigned)a.nbands, (unsigned)((a.w + kDColThreads - 1) / kDColThreads * nori),
              (unsigned)((np + ppc - 1) / ppc));
    cudaFuncSetAttribute(k_colsum_decay, cudaFuncAttributeMaxDynamicSharedMemorySize, kDColSmem);
    k_colsum_decay<<<grid, kDColThreads, csm, s>>>(a, dec, pairs, nori, ppc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t per_band = (size_t)pairs * a.wa * kDP;
    const double dband = std::pow(dec, (double)a.band_h);
    const double dlast = std::pow(dec, (double)(a.h - (a.nbands - 1) * a.band_h));
    SelMask m{};
    m.on = a.nsel > 0;
    m.words_per_unit = a.wa * kDP;
    std::memcpy(m.w, a.selmask, sizeof(m.w));
    const size_t ori_stride = 2 * (a.agg_stride / 2);  // doubles between slots 0 and 2
    const int q = bandscan_lanes(a.nbands, per_band * nori);
    k_bandscan_decay<<<(unsigned)((per_band * nori * q + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<double*>(a.agg), a.nbands, dband, dlast, per_band, m, nori, ori_stride, q);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches += 2;
  }
  if (kind == -1) return cudaSuccess;  // carries only
  const int nori = kind == -2 ? 4 : 1;
  const long long units = (long long)a.nbands * (a.nsel ? a.nsel : pairs) * nori;
  // row buffers + one carry per band row for every warp of the CTA
  auto smem_of = [&](int wpc) {
    return ((size_t)wpc * kWarpRows * kStripW + (size_t)wpc * a.band_h) * sizeof(double2);
  };
  int wpc = kWarpsPerCta;
  // two CTAs per SM: 228 KB of shared memory, 1 KB reserved per CTA
  while (wpc > 1 && 2 * (smem_of(wpc) + 1024) > (228u << 10)) wpc >>= 1;
  if (smem_of(wpc) > (200u << 10)) return cudaErrorInvalidConfiguration;  // band_h > ~12000 rows
  // set on every launch: the attribute is per device (a process-wide cache
  // would skip it on a second device and race between host threads)
  cudaFuncSetAttribute(k_build_decay_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       200 << 10);
  k_build_decay_warp<<<(unsigned)((units + wpc - 1) / wpc), 32 * wpc, smem_of(wpc), s>>>(
      a, dec, kind, pairs, nori);
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
