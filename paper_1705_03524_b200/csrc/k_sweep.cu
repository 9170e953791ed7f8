// k_sweep.cu — K2 likelihood-map sweeps, K3 peak reduction, window queries.
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
// [cy+1, cy+hy]): 8 plain + 6 xramp + 6 yramp = 20 cells per bin.  Exact
// integer arithmetic modulo 2^32; the true value lies in [0, mass] with
// mass < 2^32, so the wrapped result IS the reference count.
//
// K2c (cake) replaces WeddingCakePlan::histogram_into
// (proj/src/baselines.cpp:133-149) + score_weights (matching.cpp:37-52):
// out[b] = sum_i coeff_i * box_i[b] in ring order (outer -> inner), fp64.
// Boxes are nested, so once a bin's box count is 0 every inner term is
// coeff * 0 and the ring loop stops early (bit-identical: x + (+-0) == x).
//
// Thread mapping (both): a warp covers 16 consecutive windows of one map
// row; lanes 2u / 2u+1 own bins 0-3 / 4-7 of every octet of window u and
// read 16-byte half records, so each corner load of the warp is 512
// contiguous bytes.  Scores: the two lanes swap their per-bin terms and both
// add the octet's 8 terms in bin order with separately rounded IEEE ops
// (__dmul_rn/__dadd_rn/__dsqrt_rn/__ddiv_rn) — the reference's exact fp64
// sequence, so every map value is bit-identical.  The peak
// uses the reference tie rule (matching.cpp:211-223).
#include "swg_internal.cuh"

#ifndef SWG_CAKE_UNROLL
#define SWG_CAKE_UNROLL 2
#endif

namespace swg {

namespace {

__device__ __forceinline__ double clamp01(double v) {
  return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);  // std::clamp(v, 0, 1)
}

__device__ __forceinline__ uint4 ldqb(const char* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ uint4 box4(uint4 br, uint4 bl, uint4 tr, uint4 tl) {
  return make_uint4(br.x - bl.x - tr.x + tl.x, br.y - bl.y - tr.y + tl.y,
                    br.z - bl.z - tr.z + tl.z, br.w - bl.w - tr.w + tl.w);
}
// Exact uint32 -> double: (2^52 + n) - 2^52 on the fp64 pipe instead of an
// I2F.F64 on the narrower conversion pipe.
__device__ __forceinline__ double u2d(uint32_t n) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)n), 4503599627370496.0);
}
__device__ __forceinline__ uint32_t comp(const uint4& v, int k) {
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

// Ordered accumulation of one octet: lanes hold bins 0-3 (even) / 4-7 (odd).
// mass += value_b and s += term_b for b = 0..7 in order, in both lanes.
__device__ __forceinline__ void add_octet(const double (&val)[4], const double (&term)[4],
                                          int half, double& mass, double& s, bool with_mass) {
  double pv[4], pt[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    pv[k] = __shfl_xor_sync(0xFFFFFFFFu, val[k], 1);
    pt[k] = __shfl_xor_sync(0xFFFFFFFFu, term[k], 1);
  }
#pragma unroll
  for (int j = 0; j < kOct; ++j) {
    const int k = j & 3;
    const bool own = (j >> 2) == half;
    const double v = own ? val[k] : pv[k];
    const double t = own ? term[k] : pt[k];
    if (with_mass) mass = __dadd_rn(mass, v);
    if (v != 0.0) s = __dadd_rn(s, t);
  }
}

// K2a: Uniform (4 cells per bin) or Manhattan (20 cells per bin).
template <int SIM, bool UNIFORM>
__global__ void __launch_bounds__(kSweepThreads, SWG_AFFINE_MINB) k_sweep_affine(const SweepArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane & 1;
  int tx, ty, u0, r0;
  if (a.chain_s > 0) {  // chain order: the CTA's warps side by side on one map row
    r0 = chain_row(a, tx);
    u0 = tx * (kSweepThreads / 2) + warp * kSweepTileX + (lane >> 1);
  } else {
    sweep_tile(a.sc_tiles, tx, ty);
    u0 = tx * kSweepTileX + (lane >> 1);
    r0 = ty * kSweepTileY + warp;
  }
  const bool active = u0 < a.mw && r0 < a.rows;
  const int u = min(u0, a.mw - 1), r = min(r0, a.rows - 1);
  const int v = a.row0 + r;
  const int cx = u + a.hx, cy = v + a.hy;
  const uint32_t centre = ((uint32_t)cy * (uint32_t)a.pitch + (uint32_t)cx) * kOct + half * 4;
  const size_t ps8 = a.plane_stride * kOct;
  const uint32_t M = (uint32_t)(a.hx + a.hy + 1);
  const uint32_t ucx = (uint32_t)cx, ucy = (uint32_t)(cy + a.y_off);

  double s = 0.0, mass_unused = 0.0;
  const size_t widx = (size_t)r * a.mw + u;
  if (a.pin) s = a.pin[widx].x;  // bin-range chain: running sum of earlier bins
  for (int gi = 0; gi < a.nact; ++gi) {  // the model's octets (SweepArgs::act)
    const int g = a.act[gi];
    const char* w = reinterpret_cast<const char*>(reinterpret_cast<const uint32_t*>(a.tab) +
                                                  (size_t)g * a.planes * ps8 + centre);
    uint4 hist;
    if constexpr (UNIFORM) {
      hist = box4(ldqb(w + a.lat[7]), ldqb(w + a.lat[5]), ldqb(w + a.lat[2]), ldqb(w + a.lat[0]));
    } else {
      const uint4 p00 = ldqb(w + a.lat[0]), p10 = ldqb(w + a.lat[1]), p20 = ldqb(w + a.lat[2]);
      const uint4 p01 = ldqb(w + a.lat[3]), p21 = ldqb(w + a.lat[4]);
      const uint4 p02 = ldqb(w + a.lat[5]), p12 = ldqb(w + a.lat[6]), p22 = ldqb(w + a.lat[7]);
      const uint4 n = box4(p22, p02, p20, p00);   // whole window
      const uint4 nl = box4(p12, p02, p10, p00);  // columns [x0, x1)
      const uint4 nt = box4(p21, p01, p20, p00);  // rows    [y0, y1)
      const uint4 q00 = ldqb(w + a.lat[8]), q10 = ldqb(w + a.lat[9]), q20 = ldqb(w + a.lat[10]);
      const uint4 q02 = ldqb(w + a.lat[11]), q12 = ldqb(w + a.lat[12]), q22 = ldqb(w + a.lat[13]);
      const uint4 xl = box4(q12, q02, q10, q00), xall = box4(q22, q02, q20, q00);
      const uint4 w00 = ldqb(w + a.lat[14]), w20 = ldqb(w + a.lat[15]);
      const uint4 w01 = ldqb(w + a.lat[16]), w21 = ldqb(w + a.lat[17]);
      const uint4 w02 = ldqb(w + a.lat[18]), w22 = ldqb(w + a.lat[19]);
      const uint4 yt = box4(w21, w01, w20, w00), yall = box4(w22, w02, w20, w00);
      auto lin = [&](uint32_t n_, uint32_t nl_, uint32_t nt_, uint32_t xl_, uint32_t xa_,
                     uint32_t yt_, uint32_t ya_) {
        const uint32_t nr = n_ - nl_, nb = n_ - nt_, xr = xa_ - xl_, yb = ya_ - yt_;
        return M * n_ + xl_ - xr + ucx * (nr - nl_) + yt_ - yb + ucy * (nb - nt_);
      };
      hist.x = lin(n.x, nl.x, nt.x, xl.x, xall.x, yt.x, yall.x);
      hist.y = lin(n.y, nl.y, nt.y, xl.y, xall.y, yt.y, yall.y);
      hist.z = lin(n.z, nl.z, nt.z, xl.z, xall.z, yt.z, yall.z);
      hist.w = lin(n.w, nl.w, nt.w, xl.w, xall.w, yt.w, yall.w);
    }
    double val[4], term[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t raw = comp(hist, k);
      const double model = a.model[g * kOct + half * 4 + k];
      val[k] = u2d(raw);
      if (raw == 0u || model == 0.0) {  // +0 terms either way
        term[k] = 0.0;  // sqrt(m*0) = 0 and min(m, 0) = 0: s unchanged
      } else if (SIM == SWG_SIM_BHATTACHARYYA) {
        term[k] = __dsqrt_rn(__dmul_rn(model, val[k]));
      } else {
        const double q = __ddiv_rn(val[k], a.mass);
        term[k] = (q < model) ? q : model;
      }
    }
    add_octet(val, term, half, mass_unused, s, false);
  }
  if (a.pout) {  // partial: hand the running sum to the next bin range
    if (active && half == 0) a.pout[widx] = make_double2(s, a.mass);
    s = -2.0;
  } else {
    if constexpr (SIM == SWG_SIM_BHATTACHARYYA) s = __ddiv_rn(s, __dsqrt_rn(a.mass));
    s = clamp01(s);
    if (active && half == 0) a.scores[widx] = s;
  }
  sweep_peak(active && half == 0 ? s : -2.0, (long long)v * a.mw + u, a);
}

// K2a16: the Manhattan sweep over NARROW (uint16) {1, x, y} planes, for
// windows whose mass (the largest per-bin value H can take) is < 2^16: H is
// a polynomial with integer coefficients in the box sums, so computing it
// mod 2^16 from tables wrapped mod 2^16 gives H itself -- half the bytes of
// the 32-bit sweep.  One lane per window, 8-byte half-record loads (4 bins;
// a warp's corner load is 256 contiguous bytes), the half-octets' bins in
// order, so the lane forms the ordered sums alone (no shuffles).
template <int SIM>
__global__ void __launch_bounds__(kAff16Threads) k_sweep_affine16(const SweepArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int tx, ty;
  sweep_tile(a.sc_tiles, tx, ty);
  const int u0 = tx * 32 + lane, r0 = ty * kAff16TileY + warp;
  const bool active = u0 < a.mw && r0 < a.rows;
  const int u = min(u0, a.mw - 1), r = min(r0, a.rows - 1);
  const int v = a.row0 + r;
  const int cx = u + a.hx, cy = v + a.hy;
  const uint32_t centre = ((uint32_t)cy * (uint32_t)a.pitch + (uint32_t)cx) * kOct;
  const size_t ps8 = a.plane_stride * kOct;
  const uint32_t M = (uint32_t)(a.hx + a.hy + 1);
  const uint32_t ucx = (uint32_t)cx, ucy = (uint32_t)(cy + a.y_off);
  double s = 0.0;
  const size_t widx = (size_t)r * a.mw + u;
  if (a.pin) s = a.pin[widx].x;  // bin-range chain: running sum of earlier bins
  auto box = [](uint2 br, uint2 bl, uint2 tr, uint2 tl) {  // packed 16-bit fields
    return make_uint2(__vsub2(__vadd2(br.x, tl.x), __vadd2(bl.x, tr.x)),
                      __vsub2(__vadd2(br.y, tl.y), __vadd2(bl.y, tr.y)));
  };
  for (int gi = 0; gi < a.nact; ++gi) {  // the model's octets (SweepArgs::act)
    const int g = a.act[gi];
    const char* w = reinterpret_cast<const char*>(reinterpret_cast<const uint16_t*>(a.tab) +
                                                  (size_t)g * a.planes * ps8 + centre);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      auto ld = [&](int q) { return __ldg(reinterpret_cast<const uint2*>(w + a.lat[q] + 8 * hf)); };
      const uint2 p00 = ld(0), p10 = ld(1), p20 = ld(2), p01 = ld(3), p21 = ld(4);
      const uint2 p02 = ld(5), p12 = ld(6), p22 = ld(7);
      const uint2 n = box(p22, p02, p20, p00), nl = box(p12, p02, p10, p00);
      const uint2 nt = box(p21, p01, p20, p00);
      const uint2 q00 = ld(8), q10 = ld(9), q20 = ld(10), q02 = ld(11), q12 = ld(12), q22 = ld(13);
      const uint2 xl = box(q12, q02, q10, q00), xa = box(q22, q02, q20, q00);
      const uint2 w00 = ld(14), w20 = ld(15), w01 = ld(16), w21 = ld(17), w02 = ld(18), w22 = ld(19);
      const uint2 yt = box(w21, w01, w20, w00), ya = box(w22, w02, w20, w00);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        auto f = [&](const uint2& pk) {
          const uint32_t word = (k >> 1) ? pk.y : pk.x;
          return (k & 1) ? word >> 16 : word & 0xFFFFu;
        };
        const uint32_t n_ = f(n), nl_ = f(nl), nt_ = f(nt), xl_ = f(xl), xa_ = f(xa);
        const uint32_t yt_ = f(yt), ya_ = f(ya);
        const uint32_t nr = n_ - nl_, nb = n_ - nt_, xr = xa_ - xl_, yb = ya_ - yt_;
        const uint32_t raw =
            (M * n_ + xl_ - xr + ucx * (nr - nl_) + yt_ - yb + ucy * (nb - nt_)) & 0xFFFFu;
        const double model = a.model[g * kOct + hf * 4 + k];
        if (raw != 0u && model != 0.0) {  // else a +0 term: s unchanged
          const double val = u2d(raw);
          double term;
          if (SIM == SWG_SIM_BHATTACHARYYA) {
            term = __dsqrt_rn(__dmul_rn(model, val));
          } else {
            const double q = __ddiv_rn(val, a.mass);
            term = (q < model) ? q : model;
          }
          s = __dadd_rn(s, term);
        }
      }
    }
  }
  if (a.pout) {
    if (active) a.pout[widx] = make_double2(s, a.mass);
    s = -2.0;
  } else {
    if constexpr (SIM == SWG_SIM_BHATTACHARYYA) s = __ddiv_rn(s, __dsqrt_rn(a.mass));
    s = clamp01(s);
    if (active) a.scores[widx] = s;
  }
  sweep_peak(active ? s : -2.0, (long long)v * a.mw + u, a);
}

// K2q: declared Euclidean extension, w = A - ky*dx^2 - kx*dy^2 with
// kx = (hx+1)^2, ky = (hy+1)^2, A = 2*kx*ky.  Over the whole window box,
//   H = A*N - ky*Dxx - kx*Dyy,  Dxx = Sxx - 2cx*Sx + cx^2*N = sum (x-cx)^2
// from the five planes {1, x, y, x^2, y^2}.  The tables are uint32: every
// box sum is exact mod 2^32, and so are Dxx and Dyy computed mod 2^32 --
// their true values are <= N*hx^2, N*hy^2 < 2^32 (host-checked), hence
// exact; H is then formed in 64 bits (< 2^53, host-checked) and converted
// exactly.  A lane reads 16 bytes (4 bins) per corner, as the affine sweep.
// ty < 0: chain order, map row -ty - 1 with the CTA's warps side by side.
template <int SIM, bool YOFF = false>
__device__ __forceinline__ void quad_body(const SweepArgs& a, int tx, int ty, PeakPart* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane & 1;
  const int u0 = ty < 0 ? tx * (kQuadThreads / 2) + warp * kSweepTileX + (lane >> 1)
                        : tx * kSweepTileX + (lane >> 1);
  const int r0 = ty < 0 ? -ty - 1 : ty * kQuadTileY + warp;
  const bool active = u0 < a.mw && r0 < a.rows;
  const int u = min(u0, a.mw - 1), r = min(r0, a.rows - 1);
  const int v = a.row0 + r;
  const int cx = u + a.hx, cy = v + a.hy;
  const size_t centre = ((size_t)cy * a.pitch + (size_t)cx) * kOct + half * 4;
  const size_t ps8 = a.plane_stride * kOct;
  const uint64_t kx = (uint64_t)(a.hx + 1) * (a.hx + 1), ky = (uint64_t)(a.hy + 1) * (a.hy + 1);
  const uint64_t A = 2 * kx * ky;
  // global-row tables (carried bands) offset the centre row; a separate
  // instantiation keeps the common path's registers (72, no extra spill)
  const uint32_t ucx = (uint32_t)cx, ucy = (uint32_t)(YOFF ? cy + a.y_off : cy);

  double s = 0.0, unused = 0.0;
  const size_t widx = (size_t)r * a.mw + u;
  if (a.pin) s = a.pin[widx].x;  // bin-range chain: running sum of earlier bins
  for (int gi = 0; gi < a.nact; ++gi) {  // the model's octets (SweepArgs::act)
    const int g = a.act[gi];
    const char* w = reinterpret_cast<const char*>(reinterpret_cast<const uint32_t*>(a.tab) +
                                                  (size_t)g * a.planes * ps8 + centre);
    uint4 box[5];
#pragma unroll
    for (int p = 0; p < 5; ++p) {  // lat: corner offsets within a plane (bytes)
      const char* wp = w + (size_t)p * ps8 * sizeof(uint32_t);
      box[p] = box4(ldqb(wp + a.lat[4 * p + 3]), ldqb(wp + a.lat[4 * p + 2]),
                    ldqb(wp + a.lat[4 * p + 1]), ldqb(wp + a.lat[4 * p]));
    }
    double val[4], term[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t n = comp(box[0], k);
      const uint32_t dxx = comp(box[3], k) - 2u * ucx * comp(box[1], k) + ucx * ucx * n;
      const uint32_t dyy = comp(box[4], k) - 2u * ucy * comp(box[2], k) + ucy * ucy * n;
      const uint64_t h = A * n - ky * dxx - kx * dyy;
      val[k] = (double)h;
      const double model = a.model[g * kOct + half * 4 + k];
      if (h == 0 || model == 0.0) {  // +0 terms either way
        term[k] = 0.0;
      } else if (SIM == SWG_SIM_BHATTACHARYYA) {
        term[k] = __dsqrt_rn(__dmul_rn(model, val[k]));
      } else {
        const double q = __ddiv_rn(val[k], a.mass);
        term[k] = (q < model) ? q : model;
      }
    }
    add_octet(val, term, half, unused, s, false);
  }
  if (a.pout) {  // partial: hand the running sum to the next bin range
    if (active && half == 0) a.pout[widx] = make_double2(s, a.mass);
    s = -2.0;
  } else {
    if constexpr (SIM == SWG_SIM_BHATTACHARYYA) s = __ddiv_rn(s, __dsqrt_rn(a.mass));
    s = clamp01(s);
    if (active && half == 0) a.scores[widx] = s;
  }
  cta_peak(active && half == 0 ? s : -2.0, (long long)v * a.mw + u, part);
}

template <int SIM, bool YOFF>
__global__ void __launch_bounds__(kQuadThreads, SWG_QUAD_MINB) k_sweep_quad(const SweepArgs a) {
  int tx, ty;
  if (a.chain_s > 0) ty = -chain_row(a, tx) - 1;
  else sweep_tile(a.sc_tiles, tx, ty);
  quad_body<SIM, YOFF>(a, tx, ty, a.parts + (size_t)blockIdx.y * gridDim.x + blockIdx.x);
}

// Several quadratic maps of ONE table in one launch (a frame's scales):
// CTA b sweeps tile b / n of map b % n, so the maps' tiles over the same
// image region run together and share the table rows they read in L2.
template <int SIM>
__global__ void __launch_bounds__(kQuadThreads, SWG_QUADM_MINB) k_sweep_quad_multi(
    const QuadMulti m) {
  const int k = blockIdx.x % m.n, tile = blockIdx.x / m.n;
  if (tile >= m.gx[k] * m.gy[k]) return;  // (a shorter map: no CTA here)
  quad_body<SIM>(m.a[k], tile % m.gx[k], tile / m.gx[k], m.a[k].parts + tile);
}

// K2c: wedding-cake telescoping over nested boxes of the plain table.
template <int SIM>
__global__ void __launch_bounds__(kSweepThreads) k_sweep_cake(const SweepArgs a,
                                                              const CakeSweep rg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane & 1;
  int tx, ty;
  sweep_tile(a.sc_tiles, tx, ty);
  const int u0 = tx * kSweepTileX + (lane >> 1);
  const int r0 = ty * kSweepTileY + warp;
  const bool active = u0 < a.mw && r0 < a.rows;
  const int u = min(u0, a.mw - 1), r = min(r0, a.rows - 1);
  const int v = a.row0 + r;
  const int cx = u + a.hx, cy = v + a.hy;
  // element offset of this window's centre record in its plane (+ the half
  // of each octet this lane reads)
  const uint32_t centre = ((uint32_t)cy * (uint32_t)a.pitch + (uint32_t)cx) * kOct + half * 4;
  const size_t ps8 = a.plane_stride * kOct;

  // out[k] for bins 4*half + k of octet g, rings in order (outer -> inner).
  // out + coeff*0 == out bit for bit (out is never -0), so zero counts need
  // no guard; nested boxes: once all four counts are 0 every inner ring is.
  auto octet = [&](int g, double (&out)[4]) {
    // per-thread byte pointer to the centre record; ring offsets are bytes
    const char* w = reinterpret_cast<const char*>(reinterpret_cast<const uint32_t*>(a.tab) +
                                                  (size_t)g * a.planes * ps8 + centre);
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = 0.0;
    auto ring = [&](int i) {
      const int4 o = rg.off[i];
      return box4(ldqb(w + o.w), ldqb(w + o.z), ldqb(w + o.y), ldqb(w + o.x));
    };
    auto add = [&](const uint4& cnt, double c) {
      out[0] = __dadd_rn(out[0], __dmul_rn(c, u2d(cnt.x)));
      out[1] = __dadd_rn(out[1], __dmul_rn(c, u2d(cnt.y)));
      out[2] = __dadd_rn(out[2], __dmul_rn(c, u2d(cnt.z)));
      out[3] = __dadd_rn(out[3], __dmul_rn(c, u2d(cnt.w)));
    };
    // two rings per iteration: 8 independent 16-byte loads in flight
    int i = 0;
#if SWG_CAKE_UNROLL >= 2
    for (; i + 1 < a.rings; i += 2) {
      const uint4 c0 = ring(i), c1 = ring(i + 1);
      if ((c0.x | c0.y | c0.z | c0.w) == 0u) return;
      add(c0, rg.coeff[i]);
      if ((c1.x | c1.y | c1.z | c1.w) == 0u) return;
      add(c1, rg.coeff[i + 1]);
    }
#endif
    for (; i < a.rings; ++i) {
      const uint4 c0 = ring(i);
      if ((c0.x | c0.y | c0.z | c0.w) == 0u) return;
      add(c0, rg.coeff[i]);
    }
  };

  double s = 0.0, mass = 0.0;
  const size_t widx = (size_t)r * a.mw + u;
  if (a.pin) {  // bin-range chain (Bhattacharyya): running sums of earlier bins
    s = a.pin[widx].x;
    mass = a.pin[widx].y;
  }
  if constexpr (SIM == SWG_SIM_BHATTACHARYYA) {
    for (int g = 0; g < a.groups; ++g) {
      double out[4], term[4];
      octet(g, out);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        term[k] = out[k] != 0.0
                      ? __dsqrt_rn(__dmul_rn(a.model[g * kOct + half * 4 + k], out[k]))
                      : 0.0;
      add_octet(out, term, half, mass, s, true);
    }
  } else {
    double unused = 0.0;
    for (int g = 0; g < a.groups; ++g) {
      double out[4];
      octet(g, out);
      add_octet(out, out, half, mass, unused, true);
    }
    for (int g = 0; g < a.groups; ++g) {
      double out[4], term[4];
      octet(g, out);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double q = __ddiv_rn(out[k], mass);
        const double m = a.model[g * kOct + half * 4 + k];
        term[k] = (q < m) ? q : m;
      }
      add_octet(out, term, half, unused, s, false);
    }
  }
  if (a.pout) {
    if (active && half == 0) a.pout[widx] = make_double2(s, mass);
    s = -2.0;
  } else {
    if constexpr (SIM == SWG_SIM_BHATTACHARYYA) s = __ddiv_rn(s, __dsqrt_rn(mass));
    s = clamp01(s);
    if (active && half == 0) a.scores[widx] = s;
  }
  sweep_peak(active && half == 0 ? s : -2.0, (long long)v * a.mw + u, a);
}

// K2c16: the cake sweep over NARROW (uint16) plain planes.  Every box of a
// window with area < 2^16 has a count < 2^16, so box sums of the wrapped
// 16-bit prefix tables are exact.  One lane owns one window and reads whole
// 16-byte records (8 bins) per corner: half the bytes of the 32-bit path,
// box arithmetic on packed 16-bit pairs (vsub2/vadd2).
template <int SIM>
__global__ void __launch_bounds__(kCakeThreads, SIM == SWG_SIM_BHATTACHARYYA ? SWG_CAKE_MINB : 1)
    k_sweep_cake16(const SweepArgs a, const CakeSweep rg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int u0 = blockIdx.x * kCakeCtaX + (lane % kCakeWX);
  const int r0 = blockIdx.y * kCakeCtaY + warp * kCakeWY + lane / kCakeWX;
  const bool active = u0 < a.mw && r0 < a.rows;
  const int u = min(u0, a.mw - 1), r = min(r0, a.rows - 1);
  const int v = a.row0 + r;
  const int cx = u + a.hx, cy = v + a.hy;
  const uint32_t centre = ((uint32_t)cy * (uint32_t)a.pitch + (uint32_t)cx) * kOct;
  const size_t ps8 = a.plane_stride * kOct;

  auto octet = [&](int g, double (&out)[kOct]) {
    const char* w = reinterpret_cast<const char*>(reinterpret_cast<const uint16_t*>(a.tab) +
                                                  (size_t)g * a.planes * ps8 + centre);
#pragma unroll
    for (int k = 0; k < kOct; ++k) out[k] = 0.0;
    int i0 = 0;
    if (a.wide0) {
      // ring 0's box may hold >= 2^16 pixels; ring 1's box and ring 0's frame
      // hold fewer (host-checked), so c0 = c1 + ((c0 - c1) mod 2^16) exactly
      auto box16 = [&](int i) {
        const int4 o = rg.off[i];
        const uint4 br = ldqb(w + o.w), bl = ldqb(w + o.z), tr = ldqb(w + o.y), tl = ldqb(w + o.x);
        return make_uint4(__vsub2(__vadd2(br.x, tl.x), __vadd2(bl.x, tr.x)),
                          __vsub2(__vadd2(br.y, tl.y), __vadd2(bl.y, tr.y)),
                          __vsub2(__vadd2(br.z, tl.z), __vadd2(bl.z, tr.z)),
                          __vsub2(__vadd2(br.w, tl.w), __vadd2(bl.w, tr.w)));
      };
      const uint4 k0 = box16(0), k1 = box16(1);
      const uint32_t d[4] = {__vsub2(k0.x, k1.x), __vsub2(k0.y, k1.y), __vsub2(k0.z, k1.z),
                             __vsub2(k0.w, k1.w)};
      const uint32_t c1[4] = {k1.x, k1.y, k1.z, k1.w};
      if (((d[0] | d[1] | d[2] | d[3]) | (k1.x | k1.y | k1.z | k1.w)) == 0u) return;
      const double c = rg.coeff[0];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t lo = (c1[q] & 0xFFFFu) + (d[q] & 0xFFFFu);
        const uint32_t hi = (c1[q] >> 16) + (d[q] >> 16);
        out[2 * q] = __dadd_rn(out[2 * q], __dmul_rn(c, u2d(lo)));
        out[2 * q + 1] = __dadd_rn(out[2 * q + 1], __dmul_rn(c, __uint2double_rn(hi)));
      }
      i0 = 1;
    }
    for (int i = i0; i < a.rings; ++i) {
      const int4 o = rg.off[i];
      const uint4 br = ldqb(w + o.w), bl = ldqb(w + o.z), tr = ldqb(w + o.y), tl = ldqb(w + o.x);
      // (br + tl) - (bl + tr) on packed 16-bit pairs
      const uint32_t c0 = __vsub2(__vadd2(br.x, tl.x), __vadd2(bl.x, tr.x));
      const uint32_t c1 = __vsub2(__vadd2(br.y, tl.y), __vadd2(bl.y, tr.y));
      const uint32_t c2 = __vsub2(__vadd2(br.z, tl.z), __vadd2(bl.z, tr.z));
      const uint32_t c3 = __vsub2(__vadd2(br.w, tl.w), __vadd2(bl.w, tr.w));
      if ((c0 | c1 | c2 | c3) == 0u) break;  // nested boxes: all inner counts 0
      const double c = rg.coeff[i];
      const uint32_t cw[4] = {c0, c1, c2, c3};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // exact conversions, split between the fp64 pipe (magic number) and
        // the conversion pipe (I2F) so neither saturates
        out[2 * q] = __dadd_rn(out[2 * q], __dmul_rn(c, u2d(cw[q] & 0xFFFFu)));
        out[2 * q + 1] = __dadd_rn(out[2 * q + 1], __dmul_rn(c, __uint2double_rn(cw[q] >> 16)));
      }
    }
  };

  double s = 0.0, mass = 0.0;
  const size_t widx = (size_t)r * a.mw + u;
  if (a.pin) {  // bin-range chain (Bhattacharyya): running sums of earlier bins
    s = a.pin[widx].x;
    mass = a.pin[widx].y;
  }
  if constexpr (SIM == SWG_SIM_BHATTACHARYYA) {
    for (int g = 0; g < a.groups; ++g) {
      double out[kOct];
      octet(g, out);
#pragma unroll
      for (int j = 0; j < kOct; ++j) {
        mass = __dadd_rn(mass, out[j]);
        if (out[j] != 0.0) s = __dadd_rn(s, __dsqrt_rn(__dmul_rn(a.model[g * kOct + j], out[j])));
      }
    }
  } else {
    for (int g = 0; g < a.groups; ++g) {
      double out[kOct];
      octet(g, out);
#pragma unroll
      for (int j = 0; j < kOct; ++j) mass = __dadd_rn(mass, out[j]);
    }
    for (int g = 0; g < a.groups; ++g) {
      double out[kOct];
      octet(g, out);
#pragma unroll
      for (int j = 0; j < kOct; ++j)
        if (out[j] != 0.0) {
          const double q = __ddiv_rn(out[j], mass), m = a.model[g * kOct + j];
          s = __dadd_rn(s, (q < m) ? q : m);
        }
    }
  }
  if (a.pout) {
    if (active) a.pout[widx] = make_double2(s, mass);
    s = -2.0;
  } else {
    if constexpr (SIM == SWG_SIM_BHATTACHARYYA) s = __ddiv_rn(s, __dsqrt_rn(mass));
    s = clamp01(s);
    if (active) a.scores[widx] = s;
  }
  sweep_peak(active ? s : -2.0, (long long)v * a.mw + u, a);
}

// K2c16m: the 16-bit cake sweep over S full-ring square scales at once
// (CakeMulti).  A lane owns one window CENTRE (cx, cy) and walks the boxes of
// half-extent e from the largest scale valid at that centre down to 0: the
// four corner records of box e are loaded and the box counts formed once,
// then every scale with h_s >= e adds coef_s(e) * count (separately rounded,
// its rings in its own outer-to-inner order), so each scale's histogram is
// bit-identical to k_sweep_cake16's while the loads and box arithmetic of
// the shared extents are paid once (config 5's 8 Gaussian scales: 383 ring
// extents per centre and octet in 8 launches -> 156 in 2).  Scales sorted by
// h descending: the scales valid at a centre are a suffix s >= s0; lanes
// also accumulate the invalid larger scales below their start extent (no
// divergence in the scale loop) and drop them at the end.
// Q bins of a 16-bit record per pass: 8 (the whole 16-byte record) or 4
// (one 8-byte half: half the accumulator registers, so more warps per SM,
// and each half leaves its box walk as soon as ITS four bins are empty).
template <int Q>
struct Rec16 {
  uint32_t v[Q / 2];
};
template <int Q>
__device__ __forceinline__ Rec16<Q> ldrec(const char* p) {
  Rec16<Q> r;
  if constexpr (Q == 8) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
    r.v[0] = x.x;
    r.v[1] = x.y;
    r.v[2] = x.z;
    r.v[3] = x.w;
  } else {
    const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
    r.v[0] = x.x;
    r.v[1] = x.y;
  }
  return r;
}
// (br + tl) - (bl + tr) on packed 16-bit pairs
template <int Q>
__device__ __forceinline__ Rec16<Q> box16(const Rec16<Q>& br, const Rec16<Q>& bl,
                                          const Rec16<Q>& tr, const Rec16<Q>& tl) {
  Rec16<Q> c;
#pragma unroll
  for (int q = 0; q < Q / 2; ++q) c.v[q] = __vsub2(__vadd2(br.v[q], tl.v[q]), __vadd2(bl.v[q], tr.v[q]));
  return c;
}

constexpr int kCakeStages = SWG_CAKEM_STAGES;
__shared__ uint4 cake_pf[kCakeStages * 4 * kCakeThreads];  // ASYNC: per-thread corner slots
template <int B>
__device__ __forceinline__ void cp_async_ca(uint32_t dst, const char* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst), "l"(src), "n"(B) : "memory");
}
template <int Q>
__device__ __forceinline__ Rec16<Q> lds_rec(uint32_t a) {
  Rec16<Q> r;
  if constexpr (Q == 8)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]) : "r"(a) : "memory");
  else
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.v[0]), "=r"(r.v[1]) : "r"(a) : "memory");
  return r;
}

template <int S, int Q, bool ASYNC>
__global__ void __launch_bounds__(kCakeThreads, ASYNC ? SWG_CAKEM_MINBA
                                                : (Q == 8 ? SWG_CAKEM_MINB : SWG_CAKEM_MINB4))
    k_sweep_cake16_multi(const CakeMulti m) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hmin = m.hs[S - 1];
  const int cw = m.w - 2 * hmin, ch = m.h - 2 * hmin;  // centre domain of the smallest scale
  const int u0 = blockIdx.x * 32 + lane, v0 = blockIdx.y * kCakeTileY + warp;
  const bool inb = u0 < cw && v0 < ch;
  const int cx = min(u0, cw - 1) + hmin, cy = min(v0, ch - 1) + hmin;
  const int dist = min(min(cx, cy), min(m.w - 1 - cx, m.h - 1 - cy));
  int s0 = 0;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) s0 += m.hs[s] > dist;
  int e0 = m.hs[S - 1];
#pragma unroll
  for (int s = S - 2; s >= 0; --s) e0 = s >= s0 ? m.hs[s] : e0;
  const int P = (int)(m.pitch * kOct * 2);  // bytes per record row
  const char* base = reinterpret_cast<const char*>(reinterpret_cast<const uint16_t*>(m.tab) +
                                                   ((size_t)cy * m.pitch + cx) * kOct);
  const size_t gstride = (size_t)m.planes * m.plane_stride * kOct * 2;
  const int P16 = P + 16, Pm16 = P - 16;

  double sc[S], mass[S];
#pragma unroll
  for (int s = 0; s < S; ++s) sc[s] = mass[s] = 0.0;
  for (int pass = 0; pass < m.groups * (kOct / Q); ++pass) {
    const int g = pass / (kOct / Q), half = pass % (kOct / Q);
    const char* w = base + g * gstride + half * (Q * 2);
    double out[S][Q];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int k = 0; k < Q; ++k) out[s][k] = 0.0;
    // corner pointers of the box of half-extent e (byte offsets from the
    // centre record TL -e(P+16), TR -eP+(e+1)16, BL (e+1)P-16e, BR (e+1)(P+16)),
    // stepped inwards by constant deltas
    int e = e0;
    const char* ptl = w - (ptrdiff_t)e * P16;
    const char* ptr = w - (ptrdiff_t)e * P + (e + 1) * 16;
    const char* pbl = w + (ptrdiff_t)(e + 1) * P - e * 16;
    const char* pbr = w + (ptrdiff_t)(e + 1) * P16;
    auto step = [&] {
      ptl += P16;
      ptr += Pm16;
      pbl -= Pm16;
      pbr -= P16;
      --e;
    };
    auto todouble = [&](const Rec16<Q>& c, double (&d)[Q]) {
      // exact conversions, split between the fp64 pipe (magic number) and
      // the conversion pipe (I2F)
#pragma unroll
      for (int q = 0; q < Q / 2; ++q) {
        d[2 * q] = u2d(c.v[q] & 0xFFFFu);
        d[2 * q + 1] = __uint2double_rn(c.v[q] >> 16);
      }
    };
    if (m.wide0 && e == m.hs[0]) {
      // the outer box may hold >= 2^16 pixels; box e-1 and the frame
      // between them hold fewer (host-checked): c = c1 + ((c0 - c1) mod 2^16)
      const Rec16<Q> k0 = box16<Q>(ldrec<Q>(pbr), ldrec<Q>(pbl), ldrec<Q>(ptr), ldrec<Q>(ptl));
      const Rec16<Q> k1 = box16<Q>(ldrec<Q>(pbr - P16), ldrec<Q>(pbl - Pm16),
                                   ldrec<Q>(ptr + Pm16), ldrec<Q>(ptl + P16));
      uint32_t any = 0;
      Rec16<Q> dd;
#pragma unroll
      for (int q = 0; q < Q / 2; ++q) {
        dd.v[q] = __vsub2(k0.v[q], k1.v[q]);
        any |= dd.v[q] | k1.v[q];
      }
      if (any == 0u) {
        e = -1;  // every box of this pass is empty
      } else {
        double d[Q];
#pragma unroll
        for (int q = 0; q < Q / 2; ++q) {
          d[2 * q] = u2d((k1.v[q] & 0xFFFFu) + (dd.v[q] & 0xFFFFu));
          d[2 * q + 1] = __uint2double_rn((k1.v[q] >> 16) + (dd.v[q] >> 16));
        }
#pragma unroll
        for (int s = 0; s < S; ++s)  // the scales whose outer box this is
          if (m.hs[s] == e) {
            const double c = m.coef[s][e];
#pragma unroll
            for (int k = 0; k < Q; ++k) out[s][k] = __dadd_rn(out[s][k], __dmul_rn(c, d[k]));
          }
        step();
      }
    }
    // ASYNC: box corners stream through a per-thread ring of kCakeStages
    // shared-memory slots (cp.async, kCakeStages - 1 boxes ahead): no
    // registers hold loads in flight.  Otherwise: box e's corners are loaded
    // one step ahead into registers, so their latency overlaps the previous
    // box's fp64 work.
    Rec16<Q> nbr, nbl, ntr, ntl;
    [[maybe_unused]] const char *qtl = ptl, *qtr = ptr, *qbl = pbl, *qbr = pbr;
    [[maybe_unused]] int qe = e, slot_in = 0, slot_out = 0;
    [[maybe_unused]] uint32_t sbase = 0;
    [[maybe_unused]] auto issue = [&] {  // the next box's corners into slot_in
      if (qe >= -1) {  // box -1 (after box 0) is the last one inside the padded table
        const uint32_t d = sbase + slot_in * (4 * kCakeThreads * 16);
        cp_async_ca<Q * 2>(d, qbr);
        cp_async_ca<Q * 2>(d + kCakeThreads * 16, qbl);
        cp_async_ca<Q * 2>(d + 2 * kCakeThreads * 16, qtr);
        cp_async_ca<Q * 2>(d + 3 * kCakeThreads * 16, qtl);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      qtl += P16;
      qtr += Pm16;
      qbl -= Pm16;
      qbr -= P16;
      --qe;
      slot_in = slot_in == kCakeStages - 1 ? 0 : slot_in + 1;
    };
    if constexpr (ASYNC) {
      sbase = (uint32_t)__cvta_generic_to_shared(cake_pf) + threadIdx.x * 16;
      if (e >= 0)
        for (int j = 0; j < kCakeStages - 1; ++j) issue();
    } else if (e >= 0) {
      nbr = ldrec<Q>(pbr);
      nbl = ldrec<Q>(pbl);
      ntr = ldrec<Q>(ptr);
      ntl = ldrec<Q>(ptl);
    }
    // Phases by the number of scales whose boxes reach e (NA = scales with
    // h_s >= e, a prefix: half-extents descending), so the step loop has no
    // per-scale predicate.  Returns false once a box is empty (every inner
    // box is then empty too).
    auto phase = [&](auto na_c) -> bool {
      constexpr int NA = decltype(na_c)::value;
      const int lo = NA < S ? m.hs[NA < S ? NA : 0] : -1;
      // box e's counts into the NA scales' sums; false when the box is empty
      auto consume = [&](const Rec16<Q>& br, const Rec16<Q>& bl, const Rec16<Q>& tr,
                         const Rec16<Q>& tl) -> bool {
        const Rec16<Q> c = box16<Q>(br, bl, tr, tl);
        uint32_t any = 0;
#pragma unroll
        for (int q = 0; q < Q / 2; ++q) any |= c.v[q];
        if (any == 0u) return false;  // nested boxes: all inner counts 0
        double d[Q];
        todouble(c, d);
#pragma unroll
        for (int s = 0; s < NA; ++s) {
          const double cf = m.coef[s][e];
#pragma unroll
          for (int k = 0; k < Q; ++k) out[s][k] = __dadd_rn(out[s][k], __dmul_rn(cf, d[k]));
        }
        step();
        return true;
      };
      if constexpr (ASYNC) {
        while (e > lo) {
          issue();
          asm volatile("cp.async.wait_group %0;" ::"n"(kCakeStages - 1) : "memory");
          const uint32_t d = sbase + slot_out * (4 * kCakeThreads * 16);
          slot_out = slot_out == kCakeStages - 1 ? 0 : slot_out + 1;
          const Rec16<Q> br = lds_rec<Q>(d), bl = lds_rec<Q>(d + kCakeThreads * 16),
                         tr = lds_rec<Q>(d + 2 * kCakeThreads * 16),
                         tl = lds_rec<Q>(d + 3 * kCakeThreads * 16);
          if (!consume(br, bl, tr, tl)) return false;
        }
        return true;
      } else {
      // two steps per iteration over two corner buffers (no register copies);
      // the prefetch of box -1 (after box 0) stays inside the padded table
      while (e > lo) {
        const Rec16<Q> bbr = ldrec<Q>(pbr - P16), bbl = ldrec<Q>(pbl - Pm16),
                       btr = ldrec<Q>(ptr + Pm16), btl = ldrec<Q>(ptl + P16);
        if (!consume(nbr, nbl, ntr, ntl)) return false;
        if (e <= lo) {
          nbr = bbr;
          nbl = bbl;
          ntr = btr;
          ntl = btl;
          return true;
        }
        nbr = ldrec<Q>(pbr - P16);
        nbl = ldrec<Q>(pbl - Pm16);
        ntr = ldrec<Q>(ptr + Pm16);
        ntl = ldrec<Q>(ptl + P16);
        if (!consume(bbr, bbl, btr, btl)) return false;
      }
      return true;
      }
    };
    bool more = e >= 0;
    if (more) more = phase(std::integral_constant<int, 1>{});
    if constexpr (S >= 2) if (more) more = phase(std::integral_constant<int, 2>{});
    if constexpr (S >= 3) if (more) more = phase(std::integral_constant<int, 3>{});
    if constexpr (S >= 4) if (more) more = phase(std::integral_constant<int, 4>{});
    if constexpr (ASYNC) asm volatile("cp.async.wait_group 0;" ::: "memory");  // slots reused
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        mass[s] = __dadd_rn(mass[s], out[s][j]);
        if (out[s][j] != 0.0)
          sc[s] = __dadd_rn(sc[s], __dsqrt_rn(__dmul_rn(m.model[s][pass * Q + j], out[s][j])));
      }
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const bool valid = inb && s >= s0;
    const int us = cx - m.hs[s], vs = cy - m.hs[s];
    const double v = valid ? clamp01(__ddiv_rn(sc[s], __dsqrt_rn(mass[s]))) : -2.0;
    const long long idx = valid ? (long long)vs * m.mw[s] + us : 0x7FFFFFFFFFFFFFFFLL;
    if (valid) m.scores[s][idx] = v;
    if (s) __syncthreads();  // cta_peak's shared slots of the previous scale
    cta_peak(v, idx, m.parts[s] + (size_t)blockIdx.y * gridDim.x + blockIdx.x);
  }
}

// K3: reduce CTA candidates to the map peak (one CTA).
__device__ __forceinline__ void peak_reduce_body(const PeakPart* parts, int n, int mw, int hx,
                                                 int hy, swg_peak* out);
__global__ void __launch_bounds__(1024) k_peak_reduce(const PeakPart* parts, int n, int mw,
                                                      int hx, int hy, swg_peak* out) {
  peak_reduce_body(parts, n, mw, hx, hy, out);
}

// K3 for the maps of one k_sweep_quad_multi launch: CTA k reduces map k.
__global__ void __launch_bounds__(1024) k_peak_reduce_multi(const PeakMulti m) {
  const int k = blockIdx.x;
  peak_reduce_body(m.parts[k], m.n[k], m.mw[k], m.hx[k], m.hy[k], m.out[k]);
}

__device__ __forceinline__ void peak_reduce_body(const PeakPart* parts, int n, int mw, int hx,
                                                 int hy, swg_peak* out) {
  double s = -2.0;
  long long idx = 0x7FFFFFFFFFFFFFFFLL;
  constexpr int kBatch = 8;  // independent loads in flight per thread
  for (int i0 = threadIdx.x; i0 < n; i0 += blockDim.x * kBatch) {
    PeakPart p[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      const int i = i0 + k * blockDim.x;
      p[k] = i < n ? parts[i] : PeakPart{-2.0, 0x7FFFFFFFFFFFFFFFLL};
    }
#pragma unroll
    for (int k = 0; k < kBatch; ++k)
      if (peak_better(p[k].score, p[k].idx, s, idx)) {
        s = p[k].score;
        idx = p[k].idx;
      }
  }
  __shared__ PeakPart res;
  cta_peak(s, idx, &res);
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

// Argmax of a map held in device memory: CTA candidates (tie rule).
__global__ void __launch_bounds__(256) k_map_peak(const double* sc, size_t n, PeakPart* parts) {
  double best = -2.0;
  long long bi = 0x7FFFFFFFFFFFFFFFLL;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double v = sc[i];
    if (peak_better(v, (long long)i, best, bi)) {
      best = v;
      bi = (long long)i;
    }
  }
  cta_peak(best, bi, parts + blockIdx.x);
}

// Window queries from explicit quadrant terms (engine.cpp:39-79 semantics).
template <typename T>
__global__ void k_query(const QueryArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int w = blockIdx.y;
  if (b >= a.bins) return;
  const T* tab = reinterpret_cast<const T*>(a.tab);
  auto at = [&](int x, int y, int k) {
    return tab[elem_index(a.plane_stride, a.pitch, a.planes, x, y, b, k)];
  };
  T acc = 0;
  for (int k = 0; k < a.tpw; ++k) {
    const swg_term t = a.terms[(size_t)w * a.tpw + k];
    if (!t.valid) continue;
    auto rect = [&](int kind) {
      return at(t.x1 + 1, t.y1 + 1, kind) - at(t.x0, t.y1 + 1, kind) -
             at(t.x1 + 1, t.y0, kind) + at(t.x0, t.y0, kind);
    };
    const T cnt = rect(0);
    if (t.sx == 0 && t.sy == 0) {
      acc += (T)t.beta * cnt;
      continue;
    }
    acc += (T)t.sx * rect(1) + (T)t.sy * rect(2) + (T)t.beta * cnt;
  }
  a.out[(size_t)w * a.bins + b] = sizeof(T) == 8 ? (long long)acc : (long long)(uint32_t)acc;
}

// Wedding-cake window queries: per (window, bin) the ring boxes in order,
// out += coeff_i * count_i in fp64 (baselines.cpp:139-148).
__global__ void k_cake_query(const QueryArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int w = blockIdx.y;
  if (b >= a.bins) return;
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(a.tab);
  auto at = [&](int x, int y) {
    return tab[elem_index(a.plane_stride, a.pitch, a.planes, x, y, b, 0)];
  };
  double out = 0.0;
  for (int k = 0; k < a.tpw; ++k) {
    const swg_term t = a.terms[(size_t)w * a.tpw + k];
    if (!t.valid) continue;
    const uint32_t cnt = at(t.x1 + 1, t.y1 + 1) - at(t.x0, t.y1 + 1) - at(t.x1 + 1, t.y0) +
                         at(t.x0, t.y0);
    out = __dadd_rn(out, __dmul_rn(a.coeff[(size_t)w * a.tpw + k], (double)cnt));
  }
  a.outd[(size_t)w * a.bins + b] = out;
}

}  // namespace

cudaError_t launch_map_peak(const double* scores, size_t n, int mw, int hx, int hy,
                            PeakPart* parts, int nparts, swg_peak* out, cudaStream_t s) {
  k_map_peak<<<nparts, 256, 0, s>>>(scores, n, parts);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_peak_reduce(parts, nparts, mw, hx, hy, out, s);
}

cudaError_t launch_sweep_affine(const SweepArgs& a, bool uniform, dim3 grid, cudaStream_t s) {
  if (a.sim == SWG_SIM_BHATTACHARYYA) {
    if (uniform) k_sweep_affine<0, true><<<grid, kSweepThreads, 0, s>>>(a);
    else k_sweep_affine<0, false><<<grid, kSweepThreads, 0, s>>>(a);
  } else {
    if (uniform) k_sweep_affine<1, true><<<grid, kSweepThreads, 0, s>>>(a);
    else k_sweep_affine<1, false><<<grid, kSweepThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_sweep_affine16(const SweepArgs& a, dim3 grid, cudaStream_t s) {
  if (a.sim == SWG_SIM_BHATTACHARYYA) k_sweep_affine16<0><<<grid, kAff16Threads, 0, s>>>(a);
  else k_sweep_affine16<1><<<grid, kAff16Threads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sweep_cake(const SweepArgs& a, const CakeSweep& r, dim3 grid,
                              cudaStream_t s) {
  if (a.sim == SWG_SIM_BHATTACHARYYA) k_sweep_cake<0><<<grid, kSweepThreads, 0, s>>>(a, r);
  else k_sweep_cake<1><<<grid, kSweepThreads, 0, s>>>(a, r);
  return cudaGetLastError();
}

cudaError_t launch_sweep_quad_multi(const QuadMulti& m, cudaStream_t s) {
  int most = 0;
  for (int k = 0; k < m.n; ++k) most = max(most, m.gx[k] * m.gy[k]);
  const unsigned grid = (unsigned)(most * m.n);
  if (m.a[0].sim == SWG_SIM_BHATTACHARYYA) k_sweep_quad_multi<0><<<grid, kQuadThreads, 0, s>>>(m);
  else k_sweep_quad_multi<1><<<grid, kQuadThreads, 0, s>>>(m);
  return cudaGetLastError();
}

cudaError_t launch_sweep_quad(const SweepArgs& a, dim3 grid, cudaStream_t s) {
  if (a.y_off) {
    if (a.sim == SWG_SIM_BHATTACHARYYA) k_sweep_quad<0, true><<<grid, kQuadThreads, 0, s>>>(a);
    else k_sweep_quad<1, true><<<grid, kQuadThreads, 0, s>>>(a);
  } else if (a.sim == SWG_SIM_BHATTACHARYYA) {
    k_sweep_quad<0, false><<<grid, kQuadThreads, 0, s>>>(a);
  } else {
    k_sweep_quad<1, false><<<grid, kQuadThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_sweep_cake16(const SweepArgs& a, const CakeSweep& r, dim3 grid,
                                cudaStream_t s) {
  if (a.sim == SWG_SIM_BHATTACHARYYA) k_sweep_cake16<0><<<grid, kCakeThreads, 0, s>>>(a, r);
  else k_sweep_cake16<1><<<grid, kCakeThreads, 0, s>>>(a, r);
  return cudaGetLastError();
}

dim3 cake_multi_grid(const CakeMulti& m) {
  const int hmin = m.hs[m.n - 1];
  return dim3((unsigned)((m.w - 2 * hmin + 31) / 32),
              (unsigned)((m.h - 2 * hmin + kCakeTileY - 1) / kCakeTileY));
}

cudaError_t launch_sweep_cake16_multi(const CakeMulti& m, cudaStream_t s) {
  const dim3 grid = cake_multi_grid(m);
  static const int q = [] {
    const char* e = std::getenv("SWG_CAKEM_Q");  // A/B: bins per pass (8 or 4)
    return e ? (std::atoi(e) == 4 ? 4 : 8) : SWG_CAKEM_Q;
  }();
  static const bool as = [] {
    const char* e = std::getenv("SWG_CAKEM_ASYNC");  // A/B: cp.async corner ring
    return e ? std::atoi(e) != 0 : SWG_CAKEM_ASYNC != 0;
  }();
#define SWG_CAKEM_CASE(S)                                                               \
  case S:                                                                               \
    if (as) k_sweep_cake16_multi<S, 8, true><<<grid, kCakeThreads, 0, s>>>(m);          \
    else if (q == 8) k_sweep_cake16_multi<S, 8, false><<<grid, kCakeThreads, 0, s>>>(m); \
    else k_sweep_cake16_multi<S, 4, false><<<grid, kCakeThreads, 0, s>>>(m);            \
    break;
  switch (m.n) {
    SWG_CAKEM_CASE(2)
#if SWG_CAKE_MULTI >= 3
    SWG_CAKEM_CASE(3)
#endif
#if SWG_CAKE_MULTI >= 4
    SWG_CAKEM_CASE(4)
#endif
    default: return cudaErrorInvalidValue;
  }
#undef SWG_CAKEM_CASE
  return cudaGetLastError();
}

cudaError_t launch_peak_reduce_multi(const PeakMulti& m, int maps, cudaStream_t s) {
  k_peak_reduce_multi<<<maps, 1024, 0, s>>>(m);
  return cudaGetLastError();
}

cudaError_t launch_peak_reduce(const PeakPart* parts, int nparts, int mw, int hx, int hy,
                               swg_peak* out, cudaStream_t s) {
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

cudaError_t launch_cake_query(const QueryArgs& a, cudaStream_t s) {
  dim3 grid((unsigned)((a.bins + 127) / 128), (unsigned)a.n);
  k_cake_query<<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace swg
