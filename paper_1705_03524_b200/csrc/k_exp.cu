// k_exp.cu — exponential-kernel sweep over the decayed directional tables
// (k_decay.cu) and the two-phase exact argmax.
//
// Per window, the four quadrants of the reference decomposition (TL owns the
// centre row and column, engine.cpp:83-122) are read from the table of their
// orientation (SE table of the image, of its horizontal / vertical / double
// flip): 16 corners per bin, window-independent byte offsets and
// coefficients (ExpSweep).  The weighted histogram is assembled in fp64 and
// scored with the score_weights sequence (matching.cpp:37-52).  The fp64
// tables make these map values tolerance-exact (a different summation order
// than the brute force, ~1e-13 absolute); the PEAK is made bit-exact by
// a second phase: every window whose fast score is within `eps` of the fast
// maximum is re-scored by fp64 brute force in the reference's pixel order
// (baselines.cpp:53-69) and the reference tie rule picks among them.
#include <algorithm>
#include <cstdlib>

#include "swg_internal.cuh"

namespace swg {

namespace {

__device__ __forceinline__ double clamp01e(double v) {
  return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
}
// one 16-B bin-pair record
__device__ __forceinline__ double2 ldd2(const char* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// One lane per window, 32 windows of one map row per warp; the CTA tile is
// kExpWarpsX warps side by side (128 windows of one map row): for each of an
// octet's four bin pairs a corner load of the CTA reads 128 consecutive
// 16-byte records of one plane (2 KB runs: measured 3-5 % faster per launch
// than 32 x 8 tiles' 512-byte runs), and the lane holds all 8 bins of the
// octet, so the ordered sums need no shuffles.
template <int SIM>
#ifndef SWG_EXP_MINB
// <= 96 registers at 128 threads: deep per-lane load batches, 5 CTAs per SM
// (measured on config 4: 96 registers 230 ms, 128 233 ms, 80 +3-5 %, 252 +14 %)
#define SWG_EXP_MINB 5
#endif
__global__ void __launch_bounds__(kExpThreads, SWG_EXP_MINB) k_sweep_exp(const SweepArgs a,
                                                                         const ExpSweep e) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int tx, ty;
  if (a.chain_s > 0) {  // (kExpTileY == 1: a tile row is a map row)
    ty = chain_row(a, tx);
  } else {
    sweep_tile(a.sc_tiles, tx, ty);
  }
  const int u0 = tx * kExpTileX + (warp % kExpWarpsX) * 32 + lane;
  const int r0 = ty * kExpTileY + warp / kExpWarpsX;
  const bool active = u0 < a.mw && r0 < a.rows;
  const int u = min(u0, a.mw - 1), r = min(r0, a.rows - 1);
  const int v = a.row0 + r;
  const int cx = u + a.hx, cy = v + a.hy;
  // centre record of the window in each orientation's coordinates (bytes
  // within a pair's 4-plane block; 16-B records)
  size_t cen[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const size_t x = (k & 1) ? (size_t)(e.w - 1 - cx) : (size_t)cx;
    const size_t y = (k & 2) ? (size_t)(e.h - 1 - cy) : (size_t)cy;
    cen[k] = (k * a.plane_stride + y * a.pitch + x) * 16;
  }
  const size_t pair_bytes = 4 * a.plane_stride * 16;

  // the 8 bins of octet g: pair q holds bins 8g + 2q, 8g + 2q + 1
  auto octet = [&](int g, double (&out)[kOct]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const char* base = reinterpret_cast<const char*>(a.tab) + (size_t)(4 * g + q) * pair_bytes;
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // orientation / quadrant
        const double k0 = e.coef[4 * k], k1 = e.coef[4 * k + 1], k2 = e.coef[4 * k + 2],
                     k3 = e.coef[4 * k + 3];
        const char* w = base + cen[k];
        const double2 p0 = ldd2(w + e.off[4 * k]), p1 = ldd2(w + e.off[4 * k + 1]);
        const double2 p2 = ldd2(w + e.off[4 * k + 2]), p3 = ldd2(w + e.off[4 * k + 3]);
        o0 += k0 * p0.x + k1 * p1.x + k2 * p2.x + k3 * p3.x;
        o1 += k0 * p0.y + k1 * p1.y + k2 * p2.y + k3 * p3.y;
      }
      out[2 * q] = o0 > e.snap ? o0 : 0.0;  // rounding floor of an empty bin
      out[2 * q + 1] = o1 > e.snap ? o1 : 0.0;
    }
  };

  double s = 0.0, mass = 0.0;
  const size_t widx = (size_t)r * a.mw + u;
  if (a.pin) {  // bin-range chain (Bhattacharyya): running sums of earlier bins
    s = a.pin[widx].x;
    mass = a.pin[widx].y;
  }
  if (e.wmass > 0.0) {  // sparse: closed-form mass, the model's bin pairs only
    mass = e.wmass;
#pragma unroll 1
    for (int i = 0; i < e.npair; ++i) {
      const int q = e.pairs[i];
      const char* base = reinterpret_cast<const char*>(a.tab) + (size_t)q * pair_bytes;
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double k0 = e.coef[4 * k], k1 = e.coef[4 * k + 1], k2 = e.coef[4 * k + 2],
                     k3 = e.coef[4 * k + 3];
        const char* w = base + cen[k];
        const double2 p0 = ldd2(w + e.off[4 * k]), p1 = ldd2(w + e.off[4 * k + 1]);
        const double2 p2 = ldd2(w + e.off[4 * k + 2]), p3 = ldd2(w + e.off[4 * k + 3]);
        o0 += k0 * p0.x + k1 * p1.x + k2 * p2.x + k3 * p3.x;
        o1 += k0 * p0.y + k1 * p1.y + k2 * p2.y + k3 * p3.y;
      }
      const double m0 = a.model[2 * q], m1 = a.model[2 * q + 1];
      if (o0 > e.snap && m0 != 0.0)
        s += SIM == SWG_SIM_BHATTACHARYYA ? sqrt(m0 * o0) : fmin(m0, o0 / mass);
      if (o1 > e.snap && m1 != 0.0)
        s += SIM == SWG_SIM_BHATTACHARYYA ? sqrt(m1 * o1) : fmin(m1, o1 / mass);
    }
  } else if constexpr (SIM == SWG_SIM_BHATTACHARYYA) {
    for (int g = 0; g < a.groups; ++g) {
      double out[kOct];
      octet(g, out);
#pragma unroll
      for (int j = 0; j < kOct; ++j) {
        mass += out[j];
        if (out[j] != 0.0) s += sqrt(a.model[g * kOct + j] * out[j]);
      }
    }
  } else {
    for (int g = 0; g < a.groups; ++g) {
      double out[kOct];
      octet(g, out);
#pragma unroll
      for (int j = 0; j < kOct; ++j) mass += out[j];
    }
    for (int g = 0; g < a.groups; ++g) {
      double out[kOct];
      octet(g, out);
#pragma unroll
      for (int j = 0; j < kOct; ++j)
        if (out[j] != 0.0) s += fmin(a.model[g * kOct + j], out[j] / mass);
    }
  }
  if (a.pout) {
    if (active) a.pout[widx] = make_double2(s, mass);
    s = -2.0;
  } else {
    if constexpr (SIM == SWG_SIM_BHATTACHARYYA) s = mass > 0.0 ? s / sqrt(mass) : 0.0;
    s = clamp01e(s);
    if (active) a.scores[widx] = s;
  }
  sweep_peak(active ? s : -2.0, (long long)v * a.mw + u, a);
}

// Phase 2a: windows within eps of the fast maximum.
__global__ void k_select_cand(const double* scores, size_t n, int row0, int mw,
                              const swg_peak* fast, double eps, int cap, int* count,
                              long long* cand) {
  const double lim = fast->score - eps;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    if (scores[i] >= lim) {
      const int k = atomicAdd(count, 1);
      if (k < cap) cand[k] = (long long)row0 * mw + (long long)i;  // absolute map index
    }
}

// Phase 2b: exact fp64 brute-force re-score of the candidates (weights_into
// + score_weights order, baselines.cpp:53-69, matching.cpp:37-52), written
// back into the map.  One WARP per candidate.  The window's pixels stream
// through the warp 32 at a time (lane l holds pixel l of a row segment);
// __match_any_sync groups the lanes of equal bin and each group's lowest
// lane adds its members' weights, in lane (= row-major pixel) order, to that
// bin's running total in shared memory -- every bin's sum is the reference's
// sequential sum, and different bins advance in parallel (one dependent add
// per pixel of the same bin, not per pixel of the window).  Lane 0 then forms
// the mass and the score in bin order.  When more than `cap` windows
// qualified, the warps stride over the whole map and re-score every
// qualifying cell.
__global__ void __launch_bounds__(128) k_rescore(const SweepArgs a, const RescoreArgs r,
                                                 const swg_peak* fast) {
  __shared__ double s_tot[4][kMaxBins];
  __shared__ double s_w[4][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * 4 + wib, nw = gridDim.x * 4;
  const int cnt = *r.count;
  const bool overflow = cnt > r.cap;
  const double lim = fast->score - r.eps;
  const long long total = overflow ? (long long)a.rows * a.mw : cnt;
  double best = -2.0;
  long long bidx = 0x7FFFFFFFFFFFFFFFLL;
  double* h = s_tot[wib];
  double* wv = s_w[wib];
  for (long long c = gw; c < total; c += nw) {
    long long idx;
    if (overflow) {
      if (!(a.scores[c] >= lim)) continue;  // warp-uniform
      idx = (long long)a.row0 * a.mw + c;
    } else {
      idx = r.cand[c];
    }
    const int u = (int)(idx % a.mw), v = (int)(idx / a.mw);
    for (int b = lane; b < r.bins; b += 32) h[b] = 0.0;
    const int per_row = (r.kw + 31) >> 5, nb = r.kh * per_row;
    auto load = [&](int i, int& bl, double& wl) {
      const int dy = i / per_row, dx = (i - dy * per_row) * 32 + lane;
      bl = 0xFFFF;
      wl = 0.0;
      if (i < nb && dx < r.kw) {
        bl = __ldg(r.fi + (size_t)(v + dy) * r.fi_pitch + u + dx);
        wl = __ldg(r.grid + (size_t)dy * r.kw + dx);
      }
    };
    int bn;
    double wn;
    load(0, bn, wn);
    __syncwarp();
    for (int i = 0; i < nb; ++i) {
      const int bl = bn;
      wv[lane] = wn;
      load(i + 1, bn, wn);  // prefetch the next segment
      const unsigned grp = __match_any_sync(0xFFFFFFFFu, bl);
      __syncwarp();
      // every group's lowest lane adds its members' weights in lane order;
      // all groups of the segment advance together through one unrolled
      // pass (weights broadcast from shared memory, predicated adds)
      const bool leader = bl < r.bins && lane == __ffs(grp) - 1;
      double t = leader ? h[bl] : 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double wj = wv[j];
        if (leader && ((grp >> j) & 1u)) t = __dadd_rn(t, wj);
      }
      if (leader) h[bl] = t;
      __syncwarp();
    }
    if (lane == 0) {
      double mass = 0.0, sc = 0.0;
      for (int b = 0; b < r.bins; ++b) mass = __dadd_rn(mass, h[b]);
      if (a.sim == SWG_SIM_BHATTACHARYYA) {
        for (int b = 0; b < r.bins; ++b)
          sc = __dadd_rn(sc, __dsqrt_rn(__dmul_rn(r.model[b], h[b])));
        sc = mass > 0.0 ? __ddiv_rn(sc, __dsqrt_rn(mass)) : 0.0;
      } else if (mass > 0.0) {
        for (int b = 0; b < r.bins; ++b) {
          const double q = __ddiv_rn(h[b], mass);
          sc = __dadd_rn(sc, (q < r.model[b]) ? q : r.model[b]);
        }
      }
      sc = clamp01e(sc);
      a.scores[(size_t)(v - a.row0) * a.mw + u] = sc;
      if (peak_better(sc, idx, best, bidx)) {
        best = sc;
        bidx = idx;
      }
    }
    __syncwarp();
  }
  cta_peak(best, bidx, r.parts + blockIdx.x);
}


// Phase 2b, bin-sorted (windows up to 512 wide and 92k pixels): one CTA per
// candidate.  The reference sums each bin's weights in row-major pixel
// order (baselines.cpp:53-69), a dependent chain per bin; k_rescore walks
// the window segment by segment, so every segment costs a 32-add chain
// whatever its bins.  Here the window's pixels are first sorted STABLY by
// bin (a counting sort: each of the 8 warps counts, then scatters, the
// pixels of its row block with __match_any_sync ranks), then thread b adds
// bin b's weights in that order -- the same sequence of rounded additions,
// with the critical path the most populous bin's pixel count instead of the
// whole window (config 5 257^2: one candidate 240 -> ~40 us).
constexpr int kRsWarps = 8;
// The window's bins are first staged in shared memory (8-bit when the
// histogram has <= 256 bins) so the two sorting passes run from shared
// memory, and the weight of pixel (dx, dy) -- the declared exponential
// kernel's d^(|dx|+|dy|), a function of the L1 distance n alone -- comes from
// a shared table ltab[n] holding the host grid's own values (bit-identical).
__global__ void __launch_bounds__(32 * kRsWarps) k_rescore_sorted(const SweepArgs a,
                                                                 const RescoreArgs r,
                                                                 const swg_peak* fast) {
  extern __shared__ __align__(16) unsigned char s_mem[];
  const int bins = r.bins, kw = r.kw, kh = r.kh, hx = (kw - 1) / 2, hy = (kh - 1) / 2;
  const int npx = kw * kh, nl = hx + hy + 1;
  const bool narrow = bins <= 256;
  double* h = reinterpret_cast<double*>(s_mem);                          // [bins]
  double* ltab = h + bins;                                                // [nl]
  int* off = reinterpret_cast<int*>(ltab + nl);                           // [kRsWarps][bins]
  uint16_t* pos = reinterpret_cast<uint16_t*>(off + kRsWarps * bins);     // [npx]
  unsigned char* stage = reinterpret_cast<unsigned char*>(pos + npx);     // [npx] u8 / u16
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R = (kh + kRsWarps - 1) / kRsWarps;  // rows per warp's block
  const int rb0 = warp * R, rb1 = min(kh, rb0 + R);
  const int segs = (kw + 31) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  // the distance table: row hy of the grid for n <= hx, column kw-1 beyond
  for (int n = threadIdx.x; n < nl; n += blockDim.x)
    ltab[n] = n <= hx ? r.grid[(size_t)hy * kw + hx + n] : r.grid[(size_t)(hy + n - hx) * kw + kw - 1];
  const int cnt = *r.count;
  const bool overflow = cnt > r.cap;
  const double lim = fast->score - r.eps;
  const long long total = overflow ? (long long)a.rows * a.mw : cnt;
  double best = -2.0;
  long long bidx = 0x7FFFFFFFFFFFFFFFLL;
  auto bin_at = [&](int i) -> int {
    return narrow ? (int)stage[i] : (int)reinterpret_cast<const uint16_t*>(stage)[i];
  };
  for (long long c = blockIdx.x; c < total; c += gridDim.x) {
    long long idx;
    if (overflow) {
      if (!(a.scores[c] >= lim)) continue;  // CTA-uniform
      idx = (long long)a.row0 * a.mw + c;
    } else {
      idx = r.cand[c];
    }
    const int u = (int)(idx % a.mw), v = (int)(idx / a.mw);
    const uint16_t* fi = r.fi + (size_t)v * r.fi_pitch + u;
    // stage the window's bins (all loads in flight across the CTA)
    for (int y = warp; y < kh; y += kRsWarps)
      for (int x = lane; x < kw; x += 32) {
        const uint16_t bv = __ldg(fi + (size_t)y * r.fi_pitch + x);
        if (narrow) stage[y * kw + x] = (unsigned char)(bv < bins ? bv : 255);
        else reinterpret_cast<uint16_t*>(stage)[y * kw + x] = bv;
      }
    int* mine = off + warp * bins;
    for (int b = lane; b < bins; b += 32) mine[b] = 0;
    __syncthreads();
    // count: this warp's rows, 32 pixels at a time
    for (int y = rb0; y < rb1; ++y)
      for (int sgi = 0; sgi < segs; ++sgi) {
        const int dx = sgi * 32 + lane;
        const int bl = dx < kw ? bin_at(y * kw + dx) : 0xFFFF;
        const unsigned grp = __match_any_sync(0xFFFFFFFFu, bl);
        if (bl < bins && (grp & lt) == 0) mine[bl] += __popc(grp);
        __syncwarp();
      }
    __syncthreads();
    // offsets: bin-major, then row block (bin b's pixels contiguous in pixel order)
    if (threadIdx.x < 32) {
      int run = 0;
      for (int b0 = 0; b0 < bins; b0 += 32) {
        const int b = b0 + lane;
        int tot = 0;
        if (b < bins)
          for (int w = 0; w < kRsWarps; ++w) tot += off[w * bins + b];
        int inc = tot;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int t2 = __shfl_up_sync(0xFFFFFFFFu, inc, d);
          if (lane >= d) inc += t2;
        }
        if (b < bins) {
          int o = run + inc - tot;
          for (int w = 0; w < kRsWarps; ++w) {
            const int n = off[w * bins + b];
            off[w * bins + b] = o;
            o += n;
          }
        }
        run += __shfl_sync(0xFFFFFFFFu, inc, 31);
      }
    }
    __syncthreads();
    // scatter: stable ranks within each segment, segments in pixel order;
    // a position code is the pixel's L1 distance from the centre (its weight)
    for (int y = rb0; y < rb1; ++y)
      for (int sgi = 0; sgi < segs; ++sgi) {
        const int dx = sgi * 32 + lane;
        const int bl = dx < kw ? bin_at(y * kw + dx) : 0xFFFF;
        const unsigned grp = __match_any_sync(0xFFFFFFFFu, bl);
        const int base = bl < bins ? mine[bl] : 0;
        __syncwarp();
        if (bl < bins) {
          pos[base + __popc(grp & lt)] = (uint16_t)(abs(dx - hx) + abs(y - hy));
          if ((grp & lt) == 0) mine[bl] = base + __popc(grp);
        }
        __syncwarp();
      }
    __syncthreads();
    // per bin: its weights in pixel order (bin b's list ends where
    // mine[last block][b] points; it starts where bin b-1's ended)
    for (int b = threadIdx.x; b < bins; b += blockDim.x) {
      double t = 0.0;
      int k = b > 0 ? off[(kRsWarps - 1) * bins + b - 1] : 0;
      const int end = off[(kRsWarps - 1) * bins + b];
      constexpr int kU = 8;  // weights of the next 8 pixels loaded ahead of their adds
      for (; k + kU <= end; k += kU) {
        double wt[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) wt[q] = ltab[pos[k + q]];
#pragma unroll
        for (int q = 0; q < kU; ++q) t = __dadd_rn(t, wt[q]);
      }
      for (; k < end; ++k) t = __dadd_rn(t, ltab[pos[k]]);
      h[b] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double mass = 0.0, sc = 0.0;
      for (int b = 0; b < bins; ++b) mass = __dadd_rn(mass, h[b]);
      if (a.sim == SWG_SIM_BHATTACHARYYA) {
        for (int b = 0; b < bins; ++b)
          sc = __dadd_rn(sc, __dsqrt_rn(__dmul_rn(r.model[b], h[b])));
        sc = mass > 0.0 ? __ddiv_rn(sc, __dsqrt_rn(mass)) : 0.0;
      } else if (mass > 0.0) {
        for (int b = 0; b < bins; ++b) {
          const double q = __ddiv_rn(h[b], mass);
          sc = __dadd_rn(sc, (q < r.model[b]) ? q : r.model[b]);
        }
      }
      sc = clamp01e(sc);
      a.scores[(size_t)(v - a.row0) * a.mw + u] = sc;
      if (peak_better(sc, idx, best, bidx)) {
        best = sc;
        bidx = idx;
      }
    }
    __syncthreads();
  }
  cta_peak(threadIdx.x == 0 ? best : -2.0, bidx, r.parts + blockIdx.x);
}

// Exponential window histograms at explicit centres (swg_decay_windows):
// per (window, bin) the 16 corners of the sweep, summed per orientation in
// the sweep's order, the same snap of empty-bin noise.
__global__ void k_exp_query(const double* tab, size_t ps, size_t pitch, int bins,
                            const ExpSweep e, int n, const int* wcx, const int* wcy,
                            double* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (b >= bins || i >= n) return;
  const int cx = wcx[i], cy = wcy[i];
  const char* base = reinterpret_cast<const char*>(tab) + (size_t)(b >> 1) * 4 * ps * 16 +
                     (b & 1) * 8;
  double o = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const size_t x = (k & 1) ? (size_t)(e.w - 1 - cx) : (size_t)cx;
    const size_t y = (k & 2) ? (size_t)(e.h - 1 - cy) : (size_t)cy;
    const char* w = base + (k * ps + y * pitch + x) * 16;
    auto at = [&](int q) { return *reinterpret_cast<const double*>(w + e.off[4 * k + q]); };
    o += e.coef[4 * k] * at(0) + e.coef[4 * k + 1] * at(1) + e.coef[4 * k + 2] * at(2) +
         e.coef[4 * k + 3] * at(3);
  }
  out[(size_t)i * bins + b] = o > e.snap ? o : 0.0;
}

}  // namespace

cudaError_t launch_exp_query(const double* tab, size_t ps, size_t pitch, int bins,
                             const ExpSweep& e, int n, const int* cx, const int* cy,
                             double* out, cudaStream_t s) {
  dim3 grid((unsigned)((bins + 127) / 128), (unsigned)n);
  k_exp_query<<<grid, 128, 0, s>>>(tab, ps, pitch, bins, e, n, cx, cy, out);
  return cudaGetLastError();
}

cudaError_t launch_sweep_exp(const SweepArgs& a, const ExpSweep& e, dim3 grid, cudaStream_t s) {
  if (a.sim == SWG_SIM_BHATTACHARYYA) k_sweep_exp<0><<<grid, kExpThreads, 0, s>>>(a, e);
  else k_sweep_exp<1><<<grid, kExpThreads, 0, s>>>(a, e);
  return cudaGetLastError();
}

cudaError_t launch_exact_peak(const SweepArgs& a, const RescoreArgs& r, swg_peak* peak,
                              cudaStream_t s) {
  cudaMemsetAsync(r.count, 0, sizeof(int), s);
  const size_t n = (size_t)a.rows * a.mw;
  k_select_cand<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(
      a.scores, n, a.row0, a.mw, peak, r.eps, r.cap, r.count, r.cand);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t npx = (size_t)r.kw * r.kh;
  const size_t smem = (size_t)r.bins * 8 + (size_t)((r.kw - 1) / 2 + (r.kh - 1) / 2 + 1) * 8 +
                      (size_t)kRsWarps * r.bins * 4 + npx * 2 + npx * (r.bins <= 256 ? 1 : 2);
  const char* rw = std::getenv("SWG_RESCORE_WARP");  // A/B: 1 = the per-warp kernel
  // pixel codes are 16-bit L1 distances; the window's bins and codes fit in shared memory
  if (!(rw && std::atoi(rw)) && r.kw + r.kh <= 65536 && smem <= (220u << 10)) {
    // bin-sorted re-score: one CTA per candidate, persistent over them
    cudaFuncSetAttribute(k_rescore_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const int blocks = std::min(148, (r.cap + 3) / 4);
    k_rescore_sorted<<<blocks, 32 * kRsWarps, smem, s>>>(a, r, peak);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return launch_peak_reduce(r.parts, blocks, a.mw, a.hx, a.hy, peak, s);
  }
  const int blocks = (r.cap + 3) / 4;  // one warp per candidate
  k_rescore<<<blocks, 128, 0, s>>>(a, r, peak);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return launch_peak_reduce(r.parts, blocks, a.mw, a.hx, a.hy, peak, s);
}

}  // namespace swg
