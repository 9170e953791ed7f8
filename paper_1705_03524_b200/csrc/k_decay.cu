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
// per band, K1b' decayed scan over bands, K1c' per (band, bin pair) CTA with
// a block-wide affine scan per row and t = d*t + R per column.
// Layout: BIN PAIRS, not octets -- a record is the 2 bins of one pair at one
// cell (16 B of fp64), element (b, kind k, x, y) at
//   (((b/2)*4 + k)*plane_stride + y*pitch + x)*2 + b%2,
// with the pair count padded to a multiple of 4 (whole octets).  Two fp64
// bins per thread and column keep a full-row CTA's state in registers at
// widths up to 4096 (8 columns per thread); the sweep reads 16-B records,
// 16 windows' records contiguous per half-warp.  fp64 storage
// and recurrences: fp32 noise (~1e-7 of the table values) is comparable to
// the smallest quadrant contributions at large windows and Bhattacharyya's
// sqrt amplifies it; fp64 keeps every map value within 1e-9 of the exact
// fp64 brute force (tolerance-based parity).
#include "swg_internal.cuh"

#include <math.h>

namespace swg {

namespace {

using real = double;

// Exclusive block scan of y -> alpha*y + B_t over threads (alpha shared by
// all threads, 8 independent B components): returns the value entering each
// thread.  One __syncthreads; `buf` ([8][32]) alternates between calls.
template <int N>
__device__ __forceinline__ void block_exscan_decay(const real (&B)[N], real alpha,
                                                   real (&enter)[N], real* buf, int lane,
                                                   int warp, int nwarps) {
  real inc[N];
#pragma unroll
  for (int j = 0; j < N; ++j) inc[j] = B[j];
  real ap = alpha;  // alpha^off
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const real t = __shfl_up_sync(0xFFFFFFFFu, inc[j], off);
      if (lane >= off) inc[j] = fma(ap, t, inc[j]);
    }
    ap *= ap;
  }
  const real a32 = ap;  // alpha^32
  if (lane == 31) {
#pragma unroll
    for (int j = 0; j < N; ++j) buf[j * 32 + warp] = inc[j];
  }
  __syncthreads();
  // value entering warp w: sum_{v<w} a32^(w-1-v) W_v (each warp scans the totals)
  real alane = 1.0;  // alpha^lane
  {
    real p = alpha;
    for (int k = lane; k; k >>= 1) {
      if (k & 1) alane *= p;
      p *= p;
    }
  }
#pragma unroll
  for (int j = 0; j < N; ++j) {
    real wt = lane < nwarps ? buf[j * 32 + lane] : 0.0;
    real bp = a32;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const real t = __shfl_up_sync(0xFFFFFFFFu, wt, off);
      if (lane >= off) wt = fma(bp, t, wt);
      bp *= bp;
    }
    const real warp_enter = warp > 0 ? __shfl_sync(0xFFFFFFFFu, wt, warp - 1) : 0.0;
    const real lane_prev = __shfl_up_sync(0xFFFFFFFFu, inc[j], 1);
    enter[j] = fma(alane, warp_enter, lane > 0 ? lane_prev : 0.0);
  }
}

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
// agg: [nbands][pairs][wa] double2.
__global__ void __launch_bounds__(256) k_colsum_decay(const BuildArgs g, real dec, int pairs) {
  const int band = blockIdx.x, pr = blockIdx.y;
  const int x = blockIdx.z * blockDim.x + threadIdx.x;
  if (x >= g.w) return;
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  const uint32_t gb = (uint32_t)g.bin0 + (uint32_t)pr * kDP;
  const uint32_t lim = (uint32_t)max(g.bins - pr * kDP, 0);  // bins of this pair in range
  real c0 = 0.0, c1 = 0.0;
  const uint16_t* col = g.fi + x;
  for (int y = y0; y < y1; ++y) {
    uint32_t d = (uint32_t)col[(size_t)y * g.fi_pitch] - gb;
    d = d < lim ? d : 0xFFFFFFFFu;
    c0 = fma(dec, c0, d == 0u ? 1.0 : 0.0);
    c1 = fma(dec, c1, d == 1u ? 1.0 : 0.0);
  }
  reinterpret_cast<double2*>(g.agg)[((size_t)band * pairs + pr) * g.wa + x] =
      make_double2(c0, c1);
}

// K1b': C_0 = 0, C_{b+1} = d^(h_b) C_b + c_b (exclusive over bands, in place);
// one warp per column word, lanes = 32 bands, affine shuffle scan.
__global__ void __launch_bounds__(256) k_bandscan_decay(real* agg, int nbands, int band_h,
                                                        int h, real dec, size_t per_band) {
  const size_t col = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (col >= per_band) return;
  real run = 0.0;
  for (int b0 = 0; b0 < nbands; b0 += 32) {
    const int b = b0 + lane;
    const int hb = b < nbands ? min(band_h, h - b * band_h) : 0;
    real ia = b < nbands ? pow(dec, (real)hb) : 1.0;
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

template <int CPT>
__device__ __forceinline__ void load_bins_d(const uint16_t* p, uint16_t (&v)[CPT]) {
  if constexpr (CPT == 4) {
    const uint2 q = *reinterpret_cast<const uint2*>(p);
    v[0] = q.x & 0xFFFF; v[1] = q.x >> 16; v[2] = q.y & 0xFFFF; v[3] = q.y >> 16;
  } else {
    const uint4 q = *reinterpret_cast<const uint4*>(p);
    v[0] = q.x & 0xFFFF; v[1] = q.x >> 16; v[2] = q.y & 0xFFFF; v[3] = q.y >> 16;
    v[4] = q.z & 0xFFFF; v[5] = q.z >> 16; v[6] = q.w & 0xFFFF; v[7] = q.w >> 16;
  }
}

// K1c': decayed SE table of one orientation: one CTA per (band, bin pair).
template <int CPT>
__global__ void __launch_bounds__(512) k_build_decay(const BuildArgs g, real dec, int kind,
                                                     int pairs) {
  __shared__ real s_row[2][kDP * 32];
  __shared__ real s_carry[kDP * 32];
  extern __shared__ double2 s_stage[];  // [warps][32 * CPT] store staging
  const int band = blockIdx.x / pairs, pr = blockIdx.x % pairs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  const int xb = tid * CPT;
  const bool live = xb < g.w;
  const uint16_t* fi = g.fi + (live ? xb : 0);
  const uint32_t gb = (uint32_t)g.bin0 + (uint32_t)pr * kDP;
  const uint32_t lim = (uint32_t)max(g.bins - pr * kDP, 0);  // bins of this pair in range
  real dp[CPT + 1];  // d^i
  dp[0] = 1.0;
#pragma unroll
  for (int i = 1; i <= CPT; ++i) dp[i] = dp[i - 1] * dec;
  const real alpha = dp[CPT];

  // decayed row prefix of per-column values v[i][j] along x, into r[i][j]
  auto row_prefix = [&](const real (&v)[CPT][kDP], real (&r)[CPT][kDP], real* buf) {
    real tot[kDP], ent[kDP];
#pragma unroll
    for (int j = 0; j < kDP; ++j) {
      real run = 0.0;
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        run = fma(dec, run, v[i][j]);
        r[i][j] = run;
      }
      tot[j] = run;
    }
    block_exscan_decay<kDP>(tot, alpha, ent, buf, lane, warp, nwarps);
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int j = 0; j < kDP; ++j) r[i][j] = fma(dp[i + 1], ent[j], r[i][j]);
  };

  // carry row E(x+1, y0) from the decayed column sums above the band
  real t[CPT][kDP];
  {
    real cc[CPT][kDP];
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int j = 0; j < kDP; ++j) cc[i][j] = 0.0;
    if (live && band > 0) {
      const double2* src = reinterpret_cast<const double2*>(g.agg) +
                           ((size_t)band * pairs + pr) * g.wa + xb;
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const double2 v = src[i];
        cc[i][0] = v.x;
        cc[i][1] = v.y;
      }
    }
    row_prefix(cc, t, s_carry);
  }

  double2* plane = reinterpret_cast<double2*>(g.out) +
                   ((size_t)pr * g.planes + kind) * g.plane_stride;
  const double2 zero = make_double2(0.0, 0.0);
  if (band == 0) {
    if (live)
#pragma unroll
      for (int i = 0; i < CPT; ++i) plane[xb + 1 + i] = zero;
    if (tid == 0) plane[0] = zero;
  }
  uint16_t vn[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) vn[i] = kNoBin;
  if (live && y0 < y1) load_bins_d<CPT>(fi + (size_t)y0 * g.fi_pitch, vn);
  for (int y = y0; y < y1; ++y) {
    real ind[CPT][kDP];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      uint32_t d = (uint32_t)vn[i] - gb;
      d = d < lim ? d : 0xFFFFFFFFu;
      ind[i][0] = d == 0u ? 1.0 : 0.0;
      ind[i][1] = d == 1u ? 1.0 : 0.0;
    }
    if (live && y + 1 < y1) load_bins_d<CPT>(fi + (size_t)(y + 1) * g.fi_pitch, vn);
    real r[CPT][kDP];
    row_prefix(ind, r, s_row[y & 1]);
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int j = 0; j < kDP; ++j) t[i][j] = fma(dec, t[i][j], r[i][j]);
    double2* row = plane + (size_t)(y + 1) * g.pitch;
#ifndef SWG_DECAY_DIRECT_STORES
    // coalesced row stores (8 columns per thread): the warp's 32*CPT records
    // go through shared memory so each store instruction writes 512
    // contiguous bytes; per-thread stores of 128-byte runs touch 32 lines
    // per instruction and throttle the LSU (measured: 5.7 -> ~4 ms per
    // launch at 3840 x 669 x 512 bins; no gain at 4 columns per thread)
    if constexpr (CPT == 8) {
      double2* st = s_stage + warp * 32 * CPT;
#pragma unroll
      for (int i = 0; i < CPT; ++i) st[(lane * CPT + i) ^ (lane & (CPT - 1))] =
          make_double2(t[i][0], t[i][1]);
      __syncwarp();
      const int wcol = warp * 32 * CPT;
#pragma unroll
      for (int m = 0; m < CPT; ++m) {
        const int rec = m * 32 + lane, col = wcol + rec;
        if (col < g.w) row[col + 1] = st[rec ^ ((rec / CPT) & (CPT - 1))];
      }
      __syncwarp();
    } else
#endif
    {
      if (live)
#pragma unroll
        for (int i = 0; i < CPT; ++i) row[xb + 1 + i] = make_double2(t[i][0], t[i][1]);
    }
    if (tid == 0) row[0] = zero;
  }
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
  if (a.nbands > 1) {
    dim3 grid((unsigned)a.nbands, (unsigned)pairs, (unsigned)((a.w + 255) / 256));
    k_colsum_decay<<<grid, 256, 0, s>>>(a, dec, pairs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t per_band = (size_t)pairs * a.wa * kDP;
    k_bandscan_decay<<<(unsigned)((per_band * 32 + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<double*>(a.agg), a.nbands, a.band_h, a.h, dec, per_band);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches += 2;
  }
  const int cpt = choose_cpt(a.w);
  const int threads = (int)round_up((size_t)((a.w + cpt - 1) / cpt), 32);
  const unsigned grid = (unsigned)(a.nbands * pairs);
  const size_t smem = cpt == 8 ? (size_t)threads * cpt * sizeof(double2) : 0;  // staging
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_build_decay<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 << 10);
    cudaFuncSetAttribute(k_build_decay<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 << 10);
    attr = true;
  }
  if (cpt == 4) k_build_decay<4><<<grid, threads, smem, s>>>(a, dec, kind, pairs);
  else k_build_decay<8><<<grid, threads, smem, s>>>(a, dec, kind, pairs);
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
