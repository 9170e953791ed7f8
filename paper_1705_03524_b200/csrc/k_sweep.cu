// k_sweep.cu — K2 likelihood-map sweeps, K3 peak reduction, query kernel.
//
// K2a (affine) replaces, per strict window, swih_query_into
// (proj/src/engine.cpp:140-147: decompose 83-122 + 4 x accumulate_term
// 39-79) followed by score_counts (proj/src/matching.cpp:20-35) inside the
// likelihood_map sweep (matching.cpp:151-189).  The reference reads
// 4 quadrants x 4 corners x 3 tables = 48 cells per bin; here the Manhattan
// weight M - |x-cx| - |y-cy| is split into a box term and two half-window
// absolute-offset terms:
//   H = M*N + X_L - X_R + cx*(N_R - N_L) + Y_T - Y_B + cy*(N_B - N_T)
// (L/R = columns [cx-hx, cx] / [cx+1, cx+hx], T/B = rows [cy-hy, cy] /
// [cy+1, cy+hy]), which needs 8 plain + 6 xramp + 6 yramp = 20 cells per bin.
// All of it is exact integer arithmetic modulo 2^32; the true value lies in
// [0, mass] with mass < 2^32, so the wrapped result IS the reference count.
//
// K2c (cake) replaces WeddingCakePlan::histogram_into
// (proj/src/baselines.cpp:133-149) + score_weights (matching.cpp:37-52):
// out[b] = sum_i coeff_i * box_i[b] in ring order, in fp64.
//
// Scores: one thread owns one window and walks the bins in order with
// separately rounded IEEE ops (__dmul_rn/__dadd_rn/__dsqrt_rn/__ddiv_rn, no
// FMA contraction), the reference's exact operation sequence, so every map
// value is bit-identical to the reference's.  The peak uses
// the reference tie rule (matching.cpp:211-223): larger score, then smaller
// row-major index.
#include "swg_internal.cuh"

namespace swg {

namespace {

__device__ __forceinline__ double clamp01(double v) {
  return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);  // std::clamp(v, 0, 1)
}

__device__ __forceinline__ bool better(double s, long long i, double s2, long long i2) {
  return s > s2 || (s == s2 && i < i2);
}

// Block argmax with the tie rule; thread 0 writes the CTA's candidate.
__device__ __forceinline__ void block_peak(double s, long long idx, PeakPart* out) {
  __shared__ double ss[32];
  __shared__ long long si[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double s2 = __shfl_down_sync(0xFFFFFFFFu, s, off);
    const long long i2 = __shfl_down_sync(0xFFFFFFFFu, idx, off);
    if (better(s2, i2, s, idx)) {
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
      if (better(s2, i2, s, idx)) {
        s = s2;
        idx = i2;
      }
    }
    if (lane == 0) *out = PeakPart{s, idx};
  }
}

template <int SIM>
__device__ __forceinline__ double add_count_score(double s, double model,
                                                  uint32_t raw, double mass) {
  if (raw == 0u) return s;  // sqrt(m*0) = 0 and min(m, 0) = 0: s unchanged
  if constexpr (SIM == SWG_SIM_BHATTACHARYYA) {
    return __dadd_rn(s, __dsqrt_rn(__dmul_rn(model, (double)raw)));
  } else {
    const double q = __ddiv_rn((double)raw, mass);
    return __dadd_rn(s, (q < model) ? q : model);
  }
}

// K2a: Uniform (N only, 4 cells/bin) or Manhattan (20 cells/bin).
template <int SIM, bool UNIFORM>
__global__ void __launch_bounds__(kSweepThreads) k_sweep_affine(const SweepArgs a) {
  const int u0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  const int v = a.row0 + r;
  const bool active = u0 < a.mw;
  const int u = active ? u0 : a.mw - 1;
  const int cx = u + a.hx, cy = v + a.hy;
  // padded-table corner coordinates
  const int x0 = cx - a.hx, x1 = cx + 1, x2 = cx + a.hx + 1;
  const size_t pitch = a.pitch;
  const size_t r0 = (size_t)(cy - a.hy) * pitch + Layout<uint32_t>::xoff;
  const size_t r1 = (size_t)(cy + 1) * pitch + Layout<uint32_t>::xoff;
  const size_t r2 = (size_t)(cy + a.hy + 1) * pitch + Layout<uint32_t>::xoff;
  const uint32_t* base = reinterpret_cast<const uint32_t*>(a.tab);
  const size_t ps = a.plane_stride;
  const uint32_t M = (uint32_t)(a.hx + a.hy + 1);
  const uint32_t ucx = (uint32_t)cx, ucy = (uint32_t)cy;

  double s = 0.0;
  for (int b = 0; b < a.bins; ++b) {
    const uint32_t* P = base + (size_t)b * a.planes * ps;
    uint32_t hist;
    if constexpr (UNIFORM) {
      hist = __ldg(P + r2 + x2) - __ldg(P + r2 + x0) - __ldg(P + r0 + x2) + __ldg(P + r0 + x0);
    } else {
      const uint32_t* X = P + ps;
      const uint32_t* Y = P + 2 * ps;
      const uint32_t p00 = __ldg(P + r0 + x0), p10 = __ldg(P + r0 + x1), p20 = __ldg(P + r0 + x2);
      const uint32_t p01 = __ldg(P + r1 + x0), p21 = __ldg(P + r1 + x2);
      const uint32_t p02 = __ldg(P + r2 + x0), p12 = __ldg(P + r2 + x1), p22 = __ldg(P + r2 + x2);
      const uint32_t q00 = __ldg(X + r0 + x0), q10 = __ldg(X + r0 + x1), q20 = __ldg(X + r0 + x2);
      const uint32_t q02 = __ldg(X + r2 + x0), q12 = __ldg(X + r2 + x1), q22 = __ldg(X + r2 + x2);
      const uint32_t w00 = __ldg(Y + r0 + x0), w20 = __ldg(Y + r0 + x2);
      const uint32_t w01 = __ldg(Y + r1 + x0), w21 = __ldg(Y + r1 + x2);
      const uint32_t w02 = __ldg(Y + r2 + x0), w22 = __ldg(Y + r2 + x2);
      const uint32_t n = p22 - p02 - p20 + p00;       // whole window
      const uint32_t nl = p12 - p02 - p10 + p00;      // columns [x0, x1)
      const uint32_t nt = p21 - p01 - p20 + p00;      // rows    [y0, y1)
      const uint32_t xl = q12 - q02 - q10 + q00;
      const uint32_t xall = q22 - q02 - q20 + q00;
      const uint32_t yt = w21 - w01 - w20 + w00;
      const uint32_t yall = w22 - w02 - w20 + w00;
      const uint32_t nr = n - nl, nb = n - nt;
      const uint32_t xr = xall - xl, yb = yall - yt;
      hist = M * n + xl - xr + ucx * (nr - nl) + yt - yb + ucy * (nb - nt);
    }
    s = add_count_score<SIM>(s, a.model[b], hist, a.mass);
  }
  if constexpr (SIM == SWG_SIM_BHATTACHARYYA) s = __ddiv_rn(s, __dsqrt_rn(a.mass));
  s = clamp01(s);
  if (active) a.scores[(size_t)r * a.mw + u] = s;
  block_peak(active ? s : -2.0, (long long)v * a.mw + u,
             a.parts + (size_t)blockIdx.y * gridDim.x + blockIdx.x);
}

// K2c: wedding-cake telescoping over nested boxes of the plain table.
template <int SIM>
__global__ void __launch_bounds__(kSweepThreads) k_sweep_cake(const SweepArgs a,
                                                              const CakeRings rg) {
  const int u0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  const int v = a.row0 + r;
  const bool active = u0 < a.mw;
  const int u = active ? u0 : a.mw - 1;
  const int cx = u + a.hx, cy = v + a.hy;
  const uint32_t* base = reinterpret_cast<const uint32_t*>(a.tab);
  const size_t pitch = a.pitch, ps = a.plane_stride;
  const int xo = Layout<uint32_t>::xoff;

  auto weighted = [&](const uint32_t* P) {
    double out = 0.0;
    for (int i = 0; i < a.rings; ++i) {
      const int ax = rg.a[i], cyv = rg.c[i];
      const size_t ra = (size_t)(cy - cyv) * pitch + xo;
      const size_t rb = (size_t)(cy + cyv + 1) * pitch + xo;
      const int xa = cx - ax, xe = cx + ax + 1;
      const uint32_t cnt = __ldg(P + rb + xe) - __ldg(P + rb + xa) - __ldg(P + ra + xe) +
                           __ldg(P + ra + xa);
      if (cnt) out = __dadd_rn(out, __dmul_rn(rg.coeff[i], (double)cnt));
    }
    return out;
  };

  double s = 0.0, mass = 0.0;
  if constexpr (SIM == SWG_SIM_BHATTACHARYYA) {
    for (int b = 0; b < a.bins; ++b) {
      const double out = weighted(base + (size_t)b * a.planes * ps);
      mass = __dadd_rn(mass, out);
      if (out != 0.0) s = __dadd_rn(s, __dsqrt_rn(__dmul_rn(a.model[b], out)));
    }
    s = __ddiv_rn(s, __dsqrt_rn(mass));
  } else {
    for (int b = 0; b < a.bins; ++b)
      mass = __dadd_rn(mass, weighted(base + (size_t)b * a.planes * ps));
    for (int b = 0; b < a.bins; ++b) {
      const double out = weighted(base + (size_t)b * a.planes * ps);
      const double q = __ddiv_rn(out, mass);
      s = __dadd_rn(s, (q < a.model[b]) ? q : a.model[b]);
    }
  }
  s = clamp01(s);
  if (active) a.scores[(size_t)r * a.mw + u] = s;
  block_peak(active ? s : -2.0, (long long)v * a.mw + u,
             a.parts + (size_t)blockIdx.y * gridDim.x + blockIdx.x);
}

// K3: reduce CTA candidates to the map peak (one CTA).
__global__ void __launch_bounds__(1024) k_peak_reduce(const PeakPart* parts, int n,
                                                      int mw, int hx, int hy,
                                                      swg_peak* out) {
  double s = -2.0;
  long long idx = 0x7FFFFFFFFFFFFFFFLL;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const PeakPart p = parts[i];
    if (better(p.score, p.idx, s, idx)) {
      s = p.score;
      idx = p.idx;
    }
  }
  __shared__ PeakPart res;
  block_peak(s, idx, &res);
  __syncthreads();
  if (threadIdx.x == 0) {
    swg_peak pk;
    pk.map_x = (int)(res.idx % mw);
    pk.map_y = (int)(res.idx / mw);
    pk.center_x = pk.map_x + hx;
    pk.center_y = pk.map_y + hy;
    pk.score = res.score;
    *out = pk;
  }
}

// Window queries from explicit quadrant terms (engine.cpp:39-79 semantics).
template <typename T>
__global__ void k_query(const QueryArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int w = blockIdx.y;
  if (b >= a.bins) return;
  const T* base = reinterpret_cast<const T*>(a.tab) + (size_t)b * a.planes * a.plane_stride;
  const int xo = Layout<T>::xoff;
  T acc = 0;
  for (int k = 0; k < a.tpw; ++k) {
    const swg_term t = a.terms[(size_t)w * a.tpw + k];
    if (!t.valid) continue;
    const size_t i00 = (size_t)t.y0 * a.pitch + t.x0 + xo;
    const size_t i10 = (size_t)t.y0 * a.pitch + t.x1 + 1 + xo;
    const size_t i01 = (size_t)(t.y1 + 1) * a.pitch + t.x0 + xo;
    const size_t i11 = (size_t)(t.y1 + 1) * a.pitch + t.x1 + 1 + xo;
    const T* P = base;
    const T cnt = P[i11] - P[i01] - P[i10] + P[i00];
    if (t.sx == 0 && t.sy == 0) {
      acc += (T)t.beta * cnt;
      continue;
    }
    const T* X = base + a.plane_stride;
    const T* Y = base + 2 * a.plane_stride;
    const T xs = X[i11] - X[i01] - X[i10] + X[i00];
    const T ys = Y[i11] - Y[i01] - Y[i10] + Y[i00];
    acc += (T)t.sx * xs + (T)t.sy * ys + (T)t.beta * cnt;
  }
  a.out[(size_t)w * a.bins + b] = sizeof(T) == 8 ? (long long)acc : (long long)(uint32_t)acc;
}

// Wedding-cake window queries: per (window, bin) the ring boxes in order,
// out += coeff_i * count_i in fp64 (baselines.cpp:139-148).
__global__ void k_cake_query(const QueryArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int w = blockIdx.y;
  if (b >= a.bins) return;
  const uint32_t* P = reinterpret_cast<const uint32_t*>(a.tab) + (size_t)b * a.planes * a.plane_stride;
  const int xo = Layout<uint32_t>::xoff;
  double out = 0.0;
  for (int k = 0; k < a.tpw; ++k) {
    const swg_term t = a.terms[(size_t)w * a.tpw + k];
    if (!t.valid) continue;
    const size_t i00 = (size_t)t.y0 * a.pitch + t.x0 + xo;
    const size_t i10 = (size_t)t.y0 * a.pitch + t.x1 + 1 + xo;
    const size_t i01 = (size_t)(t.y1 + 1) * a.pitch + t.x0 + xo;
    const size_t i11 = (size_t)(t.y1 + 1) * a.pitch + t.x1 + 1 + xo;
    const uint32_t cnt = P[i11] - P[i01] - P[i10] + P[i00];
    out = __dadd_rn(out, __dmul_rn(a.coeff[(size_t)w * a.tpw + k], (double)cnt));
  }
  a.outd[(size_t)w * a.bins + b] = out;
}

}  // namespace

cudaError_t launch_cake_query(const QueryArgs& a, cudaStream_t s) {
  dim3 grid((unsigned)((a.bins + 127) / 128), (unsigned)a.n);
  k_cake_query<<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sweep_affine(const SweepArgs& a, bool uniform, int blocks_x,
                                cudaStream_t s) {
  dim3 grid((unsigned)blocks_x, (unsigned)a.rows);
  if (a.sim == SWG_SIM_BHATTACHARYYA) {
    if (uniform) k_sweep_affine<0, true><<<grid, kSweepThreads, 0, s>>>(a);
    else k_sweep_affine<0, false><<<grid, kSweepThreads, 0, s>>>(a);
  } else {
    if (uniform) k_sweep_affine<1, true><<<grid, kSweepThreads, 0, s>>>(a);
    else k_sweep_affine<1, false><<<grid, kSweepThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_sweep_cake(const SweepArgs& a, const CakeRings& r, int blocks_x,
                              cudaStream_t s) {
  dim3 grid((unsigned)blocks_x, (unsigned)a.rows);
  if (a.sim == SWG_SIM_BHATTACHARYYA) k_sweep_cake<0><<<grid, kSweepThreads, 0, s>>>(a, r);
  else k_sweep_cake<1><<<grid, kSweepThreads, 0, s>>>(a, r);
  return cudaGetLastError();
}

cudaError_t launch_peak_reduce(const PeakPart* parts, int nparts, int mw, int hx,
                               int hy, swg_peak* out, cudaStream_t s) {
  k_peak_reduce<<<1, 1024, 0, s>>>(parts, nparts, mw, hx, hy, out);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_query(const QueryArgs& a, cudaStream_t s) {
  dim3 grid((unsigned)((a.bins + 127) / 128), (unsigned)a.n);
  k_query<T><<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}
template cudaError_t launch_query<uint32_t>(const QueryArgs&, cudaStream_t);
template cudaError_t launch_query<uint64_t>(const QueryArgs&, cudaStream_t);

}  // namespace swg
