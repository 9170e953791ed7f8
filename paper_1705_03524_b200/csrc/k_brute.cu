// k_brute.cu — direct per-pixel weighted histogram sweep (MapMethod::Brute).
//
// Replaces BruteForcePlan::counts_into / weights_into
// (proj/src/baselines.cpp:24-69) + score_counts / score_weights
// (proj/src/matching.cpp:20-52) for kernels without an O(1) decomposition
// (ChebyshevLinear, GaussianChebyshev).  One thread owns one window; bins are
// processed in chunks of kChunk with per-thread shared-memory accumulators,
// and within a chunk the window pixels are visited in the reference's
// row-major order, so every per-bin fp64 sum has the reference's rounding
// sequence.  Integer kernels accumulate exact integers in fp64 (< 2^53).
#include "swg_internal.cuh"

namespace swg {

namespace {

constexpr int kChunk = 32;

__device__ __forceinline__ double clamp01b(double v) {
  return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
}

__global__ void __launch_bounds__(kBruteThreads) k_sweep_brute(const SweepArgs a,
                                                               const BruteArgs g) {
  __shared__ double acc[kChunk * kBruteThreads];
  const int tid = threadIdx.x;
  const int u0 = blockIdx.x * blockDim.x + tid;
  const int v = a.row0 + blockIdx.y;
  const bool active = u0 < a.mw;
  const int u = active ? u0 : a.mw - 1;
  const int cx = u + a.hx, cy = v + a.hy;
  const uint16_t* win = g.fi + (size_t)(cy - a.hy) * g.fi_pitch + (cx - a.hx);

  // Accumulate bins [b0, b0 + kChunk) of this window into acc[j*T + tid].
  auto chunk = [&](int b0) {
#pragma unroll
    for (int j = 0; j < kChunk; ++j) acc[j * kBruteThreads + tid] = 0.0;
    for (int dy = 0; dy < g.kh; ++dy) {
      const uint16_t* row = win + (size_t)dy * g.fi_pitch;
      const double* wrow = g.grid + (size_t)dy * g.kw;
      for (int dx = 0; dx < g.kw; ++dx) {
        const int j = (int)row[dx] - b0;
        if ((unsigned)j < (unsigned)kChunk) {
          double& slot = acc[j * kBruteThreads + tid];
          slot = __dadd_rn(slot, __ldg(wrow + dx));
        }
      }
    }
  };

  double s = 0.0, mass = 0.0;
  if (a.sim == SWG_SIM_BHATTACHARYYA) {
    for (int b0 = 0; b0 < a.bins; b0 += kChunk) {
      chunk(b0);
      const int nb = min(kChunk, a.bins - b0);
      for (int j = 0; j < nb; ++j) {
        const double raw = acc[j * kBruteThreads + tid];
        mass = __dadd_rn(mass, raw);
        if (raw != 0.0) s = __dadd_rn(s, __dsqrt_rn(__dmul_rn(a.model[b0 + j], raw)));
      }
    }
    s = __ddiv_rn(s, __dsqrt_rn(mass));
  } else {
    for (int pass = 0; pass < 2; ++pass)
      for (int b0 = 0; b0 < a.bins; b0 += kChunk) {
        chunk(b0);
        const int nb = min(kChunk, a.bins - b0);
        for (int j = 0; j < nb; ++j) {
          const double raw = acc[j * kBruteThreads + tid];
          if (pass == 0) {
            mass = __dadd_rn(mass, raw);
          } else {
            const double q = __ddiv_rn(raw, mass);
            const double m = a.model[b0 + j];
            s = __dadd_rn(s, (q < m) ? q : m);
          }
        }
      }
  }
  s = clamp01b(s);
  if (active) a.scores[(size_t)blockIdx.y * a.mw + u] = s;
  sweep_peak(active ? s : -2.0, (long long)v * a.mw + u, a);
}

// Brute-force histograms of explicit windows: one thread per window walks
// the window's pixels in row-major order (baselines.cpp:24-69), skipping
// pixels outside the image (Clipped) and accumulating into its own row of
// the output (int64 counts for integer kernels, fp64 sums otherwise).
__global__ void k_brute_query(const BruteQueryArgs a) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= a.n) return;
  const int hx = (a.kw - 1) / 2, hy = (a.kh - 1) / 2;
  const int cx = a.cx[w], cy = a.cy[w];
  long long* oi = a.out_i64 ? a.out_i64 + (size_t)w * a.bins : nullptr;
  double* od = a.out_f64 ? a.out_f64 + (size_t)w * a.bins : nullptr;
  for (int b = 0; b < a.bins; ++b) {
    if (oi) oi[b] = 0;
    if (od) od[b] = 0.0;
  }
  for (int dy = -hy; dy <= hy; ++dy) {
    const int y = cy + dy;
    if (y < 0 || y >= a.h) continue;
    for (int dx = -hx; dx <= hx; ++dx) {
      const int x = cx + dx;
      if (x < 0 || x >= a.w) continue;
      const int bin = a.fi[(size_t)y * a.w + x];
      if (bin >= a.bins) continue;
      const double wt = a.grid[(size_t)(dy + hy) * a.kw + (dx + hx)];
      if (oi) oi[bin] += (long long)wt;
      if (od) od[bin] = __dadd_rn(od[bin], wt);
    }
  }
}

}  // namespace

cudaError_t launch_brute_query(const BruteQueryArgs& a, cudaStream_t s) {
  k_brute_query<<<(a.n + 127) / 128, 128, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sweep_brute(const SweepArgs& a, const BruteArgs& b, int blocks_x,
                               cudaStream_t s) {
  dim3 grid((unsigned)blocks_x, (unsigned)a.rows);
  k_sweep_brute<<<grid, kBruteThreads, 0, s>>>(a, b);
  return cudaGetLastError();
}

}  // namespace swg
