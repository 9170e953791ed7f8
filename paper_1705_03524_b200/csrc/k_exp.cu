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

#include "swg_internal.cuh"

namespace swg {

namespace {

__device__ __forceinline__ double clamp01e(double v) {
  return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
}
__device__ __forceinline__ bool better_e(double s, long long i, double s2, long long i2) {
  return s > s2 || (s == s2 && i < i2);
}

__device__ __forceinline__ void block_peak_e(double s, long long idx, PeakPart* out) {
  __shared__ double ss[32];
  __shared__ long long si[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) {
    const double s2 = __shfl_down_sync(0xFFFFFFFFu, s, off);
    const long long i2 = __shfl_down_sync(0xFFFFFFFFu, idx, off);
    if (better_e(s2, i2, s, idx)) { s = s2; idx = i2; }
  }
  if (lane == 0) { ss[warp] = s; si[warp] = idx; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    s = lane < nw ? ss[lane] : -2.0;
    idx = lane < nw ? si[lane] : 0x7FFFFFFFFFFFFFFFLL;
    for (int off = 16; off > 0; off >>= 1) {
      const double s2 = __shfl_down_sync(0xFFFFFFFFu, s, off);
      const long long i2 = __shfl_down_sync(0xFFFFFFFFu, idx, off);
      if (better_e(s2, i2, s, idx)) { s = s2; idx = i2; }
    }
    if (lane == 0) *out = PeakPart{s, idx};
  }
}

// four consecutive fp64 table values (a lane's half record)
struct D4 {
  double x, y, z, w;
};
__device__ __forceinline__ D4 ldd4(const char* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p + 16));
  return D4{a.x, a.y, b.x, b.y};
}

template <int SIM>
__global__ void __launch_bounds__(kSweepThreads) k_sweep_exp(const SweepArgs a, const ExpSweep e) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane & 1;
  const int u0 = blockIdx.x * kSweepTileX + (lane >> 1);
  const int r0 = blockIdx.y * kSweepTileY + warp;
  const bool active = u0 < a.mw && r0 < a.rows;
  const int u = min(u0, a.mw - 1), r = min(r0, a.rows - 1);
  const int v = a.row0 + r;
  const int cx = u + a.hx, cy = v + a.hy;
  const size_t ps8 = a.plane_stride * kOct;
  // centre record of the window in each orientation's coordinates
  size_t cen[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const size_t x = (k & 1) ? (size_t)(e.w - 1 - cx) : (size_t)cx;
    const size_t y = (k & 2) ? (size_t)(e.h - 1 - cy) : (size_t)cy;
    cen[k] = (k * ps8 + (y * a.pitch + x) * kOct + half * 4) * sizeof(double);
  }

  auto octet = [&](int g, double (&out)[4]) {
    const char* base = reinterpret_cast<const char*>(reinterpret_cast<const double*>(a.tab) +
                                                     (size_t)g * a.planes * ps8);
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // orientation / quadrant
      const char* w = base + cen[k];
      const D4 c0 = ldd4(w + e.off[4 * k]), c1 = ldd4(w + e.off[4 * k + 1]);
      const D4 c2 = ldd4(w + e.off[4 * k + 2]), c3 = ldd4(w + e.off[4 * k + 3]);
      const double k0 = e.coef[4 * k], k1 = e.coef[4 * k + 1], k2 = e.coef[4 * k + 2],
                   k3 = e.coef[4 * k + 3];
      out[0] += k0 * c0.x + k1 * c1.x + k2 * c2.x + k3 * c3.x;
      out[1] += k0 * c0.y + k1 * c1.y + k2 * c2.y + k3 * c3.y;
      out[2] += k0 * c0.z + k1 * c1.z + k2 * c2.z + k3 * c3.z;
      out[3] += k0 * c0.w + k1 * c1.w + k2 * c2.w + k3 * c3.w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = out[k] > e.snap ? out[k] : 0.0;  // rounding floor
  };

  auto add_oct = [&](const double (&val)[4], const double (&term)[4], double& mass, double& s,
                     bool with_mass, bool with_s) {
    double pv[4], pt[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      pv[k] = __shfl_xor_sync(0xFFFFFFFFu, val[k], 1);
      pt[k] = __shfl_xor_sync(0xFFFFFFFFu, term[k], 1);
    }
#pragma unroll
    for (int j = 0; j < kOct; ++j) {
      const bool own = (j >> 2) == half;
      const double vv = own ? val[j & 3] : pv[j & 3], tt = own ? term[j & 3] : pt[j & 3];
      if (with_mass) mass += vv;
      if (with_s && vv != 0.0) s += tt;
    }
  };

  double s = 0.0, mass = 0.0;
  if constexpr (SIM == SWG_SIM_BHATTACHARYYA) {
    for (int g = 0; g < a.groups; ++g) {
      double out[4], term[4];
      octet(g, out);
#pragma unroll
      for (int k = 0; k < 4; ++k) term[k] = sqrt(a.model[g * kOct + half * 4 + k] * out[k]);
      add_oct(out, term, mass, s, true, true);
    }
    s = mass > 0.0 ? s / sqrt(mass) : 0.0;
  } else {
    double unused = 0.0;
    for (int g = 0; g < a.groups; ++g) {
      double out[4];
      octet(g, out);
      add_oct(out, out, mass, unused, true, false);
    }
    for (int g = 0; g < a.groups; ++g) {
      double out[4], term[4];
      octet(g, out);
#pragma unroll
      for (int k = 0; k < 4; ++k) term[k] = fmin(a.model[g * kOct + half * 4 + k], out[k] / mass);
      add_oct(out, term, unused, s, false, true);
    }
  }
  s = clamp01e(s);
  if (active && half == 0) a.scores[(size_t)r * a.mw + u] = s;
  block_peak_e(active && half == 0 ? s : -2.0, (long long)v * a.mw + u,
               a.parts + (size_t)blockIdx.y * gridDim.x + blockIdx.x);
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
// + score_weights order), written back into the map; one window per thread.
// When more than `cap` windows qualified, the same threads stride over the
// whole map and re-score every qualifying cell instead (slow but exact).
__global__ void k_rescore(const SweepArgs a, const RescoreArgs r, const swg_peak* fast) {
  const uint16_t* fi = r.fi;
  const size_t fi_pitch = r.fi_pitch;
  const double* grid = r.grid;
  const int kw = r.kw, kh = r.kh, mw = a.mw, row0 = a.row0, rows = a.rows, bins = a.bins;
  const double* model = a.model;
  double* hist = r.hist;
  double* scores = a.scores;
  const int cap = r.cap;
  const long long* cand = r.cand;
  const double eps = r.eps;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
  const int cnt = *r.count;
  const bool overflow = cnt > cap;
  const double lim = fast->score - eps;
  const long long total = overflow ? (long long)rows * mw : cnt;
  double best = -2.0;
  long long bidx = 0x7FFFFFFFFFFFFFFFLL;
  double* h = hist + (size_t)tid * bins;
  for (long long c = tid; c < total; c += nthr) {
    long long idx;
    if (overflow) {
      if (!(scores[c] >= lim)) continue;
      idx = (long long)row0 * mw + c;
    } else {
      idx = cand[c];
    }
    const int u = (int)(idx % mw), v = (int)(idx / mw);
    for (int b = 0; b < bins; ++b) h[b] = 0.0;
    for (int dy = 0; dy < kh; ++dy) {
      const uint16_t* row = fi + (size_t)(v + dy) * fi_pitch + u;
      for (int dx = 0; dx < kw; ++dx) {
        const int b = row[dx];
        if (b < bins) h[b] = __dadd_rn(h[b], grid[dy * kw + dx]);
      }
    }
    double mass = 0.0, acc = 0.0;
    for (int b = 0; b < bins; ++b) mass = __dadd_rn(mass, h[b]);
    if (a.sim == SWG_SIM_BHATTACHARYYA) {
      for (int b = 0; b < bins; ++b) acc = __dadd_rn(acc, __dsqrt_rn(__dmul_rn(model[b], h[b])));
      acc = mass > 0.0 ? __ddiv_rn(acc, __dsqrt_rn(mass)) : 0.0;
    } else if (mass > 0.0) {
      for (int b = 0; b < bins; ++b) {
        const double q = __ddiv_rn(h[b], mass);
        acc = __dadd_rn(acc, (q < model[b]) ? q : model[b]);
      }
    }
    const double s = clamp01e(acc);
    scores[(size_t)(v - row0) * mw + u] = s;
    if (better_e(s, idx, best, bidx)) {
      best = s;
      bidx = idx;
    }
  }
  block_peak_e(best, bidx, r.parts + blockIdx.x);
}

}  // namespace

cudaError_t launch_sweep_exp(const SweepArgs& a, const ExpSweep& e, dim3 grid, cudaStream_t s) {
  if (a.sim == SWG_SIM_BHATTACHARYYA) k_sweep_exp<0><<<grid, kSweepThreads, 0, s>>>(a, e);
  else k_sweep_exp<1><<<grid, kSweepThreads, 0, s>>>(a, e);
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
  const int blocks = (r.cap + 127) / 128;
  k_rescore<<<blocks, 128, 0, s>>>(a, r, peak);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return launch_peak_reduce(r.parts, blocks, a.mw, a.hx, a.hy, peak, s);
}

}  // namespace swg
