// k_stream.cu — row-streaming chain sweeps (K2s): Manhattan on 32-bit
// {1, x, y} planes (lane pairs) and on narrow 16-bit planes (one lane per
// window).  Same per-window integer H and the same fp64 score sequence as
// k_sweep_affine / k_sweep_affine16 (so bit-identical maps), but each table
// row is fetched ONCE per chain instead of once per corner use.
//
// The Manhattan histogram of a window (the reference's quadrant sum,
// proj/src/engine.cpp:39-147 with score_counts, proj/src/matching.cpp:20-35)
// is, per bin, with the window's three table rows y0 = cy-hy, y1 (= cy+1 or
// cy: the split of the odd window height is free, the centre row has
// |y-cy| = 0) and y2 = cy+hy+1 and the columns x0 = cx-hx, x1 = cx+1,
// x2 = cx+hx+1:
//   H = G(y2) - G(y0) - YA(y0) + 2 YA(y1) - YA(y2) + cy (A(y0) - 2 A(y1) + A(y2))
// with the per-row horizontal differences
//   A = P(x2) - P(x0), B = P(x1) - P(x0), XA = X(x2) - X(x0), XL = X(x1) - X(x0),
//   YA = Y(x2) - Y(x0),  G = (M + cx) A + 2 XL - XA - 2 cx B
// (P, X, Y: the plain / xramp / yramp tables), all mod 2^32 -- the true H
// lies in [0, mass] with mass < 2^32, so the wrapped value IS the count.
//
// Chains.  Window rows v_0, v_1 = v_0 + m_0, v_2 = v_1 + m_1, ... with the
// steps m alternating hy+1, hy: window k's rows are exactly
// (y0, y1, y2) = (v_k, v_{k+1}, v_{k+2}), so a row loaded at step j is the
// bottom row of window j-2, the middle row of window j-1 and the top row of
// window j: ONE row (8 records: P, X at x0 x1 x2, Y at x0 x2) per window
// instead of 20 corner records.  Chain c < hy covers the map rows of the two
// residues c, c+hy+1 mod 2hy+1; chain hy covers residue hy (its odd windows
// repeat chain 0's rows and are not emitted).  A CTA sweeps a SEGMENT of at
// most kStreamLen windows of one chain for kStreamWarps x 16 (32-bit) or x 32
// (16-bit) window columns, octet by octet; a window's running score sum
// lives in shared memory between octets, so the bins are still added in bin
// order.  CTAs are ordered (column block, chain, segment) so the CTAs in
// flight read the same rows.
#include <algorithm>

#include "swg_internal.cuh"

namespace swg {

namespace {

__device__ __forceinline__ double clamp01s(double v) {
  return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
}
__device__ __forceinline__ double u2ds(uint32_t n) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)n), 4503599627370496.0);
}
__device__ __forceinline__ uint32_t cmp4(const uint4& v, int k) {
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

// Chain geometry of one CTA: chain c, windows [kb, ke) of it.
struct Seg {
  int c, kb, ke;
  bool single;  // chain hy: only even windows are emitted
};
__device__ __forceinline__ int chain_len(int c, int hy, int rows) {
  const int P = 2 * hy + 1;
  const int ne = rows > c ? (rows - c + P - 1) / P : 0;
  const int ro = rows - c - hy - 1;
  const int no = ro > 0 ? (ro + P - 1) / P : 0;
  return ne + no;
}
__device__ __forceinline__ Seg stream_seg(const SweepArgs& a) {
  const int nc = a.hy + 1;
  Seg s;
  s.c = blockIdx.y % nc;
  const int seg = blockIdx.y / nc;
  const int K = chain_len(s.c, a.hy, a.rows);
  s.kb = seg * kStreamLen;
  s.ke = min(K, s.kb + kStreamLen);
  s.single = s.c == a.hy;
  return s;
}
// Local map row of window k of chain c.
__device__ __forceinline__ int chain_r(int c, int hy, int k) {
  return c + (k >> 1) * (2 * hy + 1) + (k & 1) * (hy + 1);
}

// Quadratic (Euclidean) chains: window rows c, c + P, c + 2P, ... (P = 2hy+1):
// window k's top row is the bottom row of window k-1.
__device__ __forceinline__ Seg quad_seg(const SweepArgs& a) {
  const int P = 2 * a.hy + 1;
  Seg s;
  s.c = blockIdx.y % P;
  const int seg = blockIdx.y / P;
  const int K = a.rows > s.c ? (a.rows - s.c + P - 1) / P : 0;
  s.kb = seg * kStreamLen;
  s.ke = min(K, s.kb + kStreamLen);
  s.single = false;
  return s;
}

// L2 prefetch of a row segment by the TMA engine (no registers held): the
// stream sweeps walk their rows in a known order, so thread i < segments
// prefetches segment i of the row kStreamPf steps ahead.
// Measured on config 5 (A/B of 0, 1, 2, 4 steps): the quadratic sweep gains
// at one step (4.11 -> 3.82 ms), the affine sweep loses at any distance
// (2.87 -> 3.12 ms: its 256-bit loads already keep enough bytes in flight).
#ifndef SWG_STREAM_PF
#define SWG_STREAM_PF 0
#endif
#ifndef SWG_STREAMQ_PF
#define SWG_STREAMQ_PF 1
#endif
constexpr int kStreamPf = SWG_STREAM_PF, kStreamPfQ = SWG_STREAMQ_PF;
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Block argmax epilogue shared by the stream sweeps.
__device__ __forceinline__ void stream_peak(double s, long long idx, const SweepArgs& a) {
  cta_peak(s, idx, a.parts + (size_t)blockIdx.y * gridDim.x + blockIdx.x);
}

// Scores of one finished window octet, added to its running sum in bin
// order.  Bins whose model value is 0 are skipped (uniform branch: +0 terms);
// a zero count adds +0 as well.
__device__ __forceinline__ double to_d(uint32_t v) { return u2ds(v); }
__device__ __forceinline__ double to_d(uint64_t v) { return (double)v; }  // < 2^53: exact

template <int SIM, typename T>
__device__ __forceinline__ void score_octet(const SweepArgs& a, int g, const T (&H)[8],
                                            double& s) {
#pragma unroll
  for (int k = 0; k < kOct; ++k) {
    const double model = a.model[g * kOct + k];
    if (model != 0.0 && H[k] != 0u) {
      const double val = to_d(H[k]);
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

// Epilogue: final scores of the segment's windows, the CTA's peak candidate.
__device__ __forceinline__ int seg_row(const SweepArgs& a, const Seg& sg, int k, bool quad) {
  return quad ? sg.c + k * (2 * a.hy + 1) : chain_r(sg.c, a.hy, k);
}

template <int SIM, bool QUAD = false>
__device__ __forceinline__ void stream_finish(const SweepArgs& a, const Seg& sg,
                                              const double (*ssum)[kStreamCols], int col, int u,
                                              bool ucol) {
  double best = -2.0;
  long long bi = 0x7FFFFFFFFFFFFFFFLL;
  for (int kk = 0; kk < sg.ke - sg.kb; ++kk) {
    const int k = sg.kb + kk;
    const int r = seg_row(a, sg, k, QUAD);
    const bool emit = ucol && !(sg.single && (k & 1));
    double s = ssum[kk][col];
    const size_t widx = (size_t)r * a.mw + u;
    if (a.pout) {
      if (emit) a.pout[widx] = make_double2(s, a.mass);
      continue;
    }
    if constexpr (SIM == SWG_SIM_BHATTACHARYYA) s = __ddiv_rn(s, __dsqrt_rn(a.mass));
    s = clamp01s(s);
    if (emit) {
      a.scores[widx] = s;
      const long long idx = (long long)(a.row0 + r) * a.mw + u;
      if (peak_better(s, idx, best, bi)) {
        best = s;
        bi = idx;
      }
    }
  }
  stream_peak(best, bi, a);
}

// Running sums start at 0 (or the bin-range chain's incoming sums).
__device__ __forceinline__ void stream_init(const SweepArgs& a, const Seg& sg,
                                            double (*ssum)[kStreamCols], int col, int u,
                                            bool quad = false) {
  for (int kk = 0; kk < sg.ke - sg.kb; ++kk) {
    double s = 0.0;
    if (a.pin) s = a.pin[(size_t)seg_row(a, sg, sg.kb + kk, quad) * a.mw + u].x;
    ssum[kk][col] = s;
  }
}

// ---------------------------------------------------------------- 32-bit
// One lane per window column; a cell's 8-bin record (32 B) is one 256-bit
// load, so a warp's load is 1 KB contiguous.
struct R8 {
  uint32_t v[8];
};
__device__ __forceinline__ R8 ld256(const uint32_t* p) {
  R8 r;
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
        "=r"(r.v[6]), "=r"(r.v[7])
      : "l"(p));
  return r;
}

template <int SIM>
__global__ void __launch_bounds__(kStreamThreads, SWG_STREAM_MINB) k_stream_affine(const SweepArgs a) {
  __shared__ double ssum[kStreamLen][kStreamCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = warp * 32 + lane;
  const Seg sg = stream_seg(a);
  const int u0 = blockIdx.x * kStreamCols + col;
  const bool ucol = u0 < a.mw;
  const int u = min(u0, a.mw - 1);
  const uint32_t cx = (uint32_t)(u + a.hx);
  const uint32_t M = (uint32_t)(a.hx + a.hy + 1);
  const uint32_t gm = M + cx, c2 = 2u * cx;
  const size_t ps8 = a.plane_stride * kOct;
  const size_t p8 = a.pitch * kOct;
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(a.tab);
  const size_t ox0 = (size_t)u * kOct, ox1 = ox0 + (size_t)(a.hx + 1) * kOct,
               ox2 = ox0 + (size_t)(2 * a.hx + 1) * kOct;
  const int hy = a.hy;
  const int ybase = a.row0 + hy + a.y_off;  // cy of local row 0 (global rows)
  const uint32_t seg_bytes = (uint32_t)min(kStreamCols, a.mw - (int)blockIdx.x * kStreamCols) * 32u;
  stream_init(a, sg, ssum, col, u);

  for (int gi = 0; gi < a.nact; ++gi) {
    const int g = a.act[gi];
    const uint32_t* pl0 = tab + (size_t)g * a.planes * ps8;
    const uint32_t* pl1 = pl0 + ps8;
    const uint32_t* pl2 = pl1 + ps8;
    uint32_t S1[8], S2[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) S1[k] = S2[k] = 0u;
    for (int j = sg.kb; j < sg.ke + 2; ++j) {
      if (kStreamPf > 0 && threadIdx.x < 8 && j + kStreamPf < sg.ke + 2) {
        const size_t rp = (size_t)(a.row0 + chain_r(sg.c, hy, j + kStreamPf)) * p8;
        const int q = threadIdx.x;  // segments: P, X at x0 x1 x2; Y at x0 x2
        const uint32_t* pl = q < 3 ? pl0 : q < 6 ? pl1 : pl2;
        const int xi = q < 6 ? q % 3 : (q == 6 ? 0 : 2);
        const size_t ox = (size_t)(blockIdx.x * kStreamCols) * kOct +
                          (xi == 0 ? 0 : xi == 1 ? (size_t)(a.hx + 1) * kOct : (size_t)(2 * a.hx + 1) * kOct);
        l2_prefetch(pl + rp + ox, seg_bytes);
      }
      const size_t ro = (size_t)(a.row0 + chain_r(sg.c, hy, j)) * p8;
      const uint32_t cyb = (uint32_t)(ybase + chain_r(sg.c, hy, j - 2));
      const uint32_t cym = (uint32_t)(ybase + chain_r(sg.c, hy, j - 1));
      const uint32_t cyt = (uint32_t)(ybase + chain_r(sg.c, hy, j));
      uint32_t H[8], A[8], G[8];
      {
        const R8 p0 = ld256(pl0 + ro + ox0), p1 = ld256(pl0 + ro + ox1),
                 p2 = ld256(pl0 + ro + ox2);
        const R8 x0 = ld256(pl1 + ro + ox0), x1 = ld256(pl1 + ro + ox1),
                 x2 = ld256(pl1 + ro + ox2);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          A[k] = p2.v[k] - p0.v[k];
          G[k] = gm * A[k] + 2u * (x1.v[k] - x0.v[k]) - (x2.v[k] - x0.v[k]) -
                 c2 * (p1.v[k] - p0.v[k]);
        }
      }
      const R8 y0 = ld256(pl2 + ro + ox0), y2 = ld256(pl2 + ro + ox2);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t YA = y2.v[k] - y0.v[k];
        H[k] = S1[k] + G[k] - YA + cyb * A[k];
        S1[k] = S2[k] + 2u * YA - 2u * cym * A[k];
        S2[k] = cyt * A[k] - G[k] - YA;
      }
      if (j >= sg.kb + 2) {  // window j-2 complete for this octet
        const int kk = j - 2 - sg.kb;
        double s = ssum[kk][col];
        score_octet<SIM>(a, g, H, s);
        ssum[kk][col] = s;
      }
    }
  }
  stream_finish<SIM>(a, sg, ssum, col, u, ucol);
}

// ---------------------------------------------------------------- 16-bit
// Full 16-byte records (8 uint16 bins); H is formed mod 2^32 from values
// known mod 2^16 and masked: exact while the window mass is < 2^16.
__device__ __forceinline__ uint32_t h16(const uint4& v, int k) {
  const uint32_t w = cmp4(v, k >> 1);
  return (k & 1) ? w >> 16 : w & 0xFFFFu;
}

template <int SIM>
__global__ void __launch_bounds__(kStreamThreads, SWG_STREAM16_MINB) k_stream_affine16(
    const SweepArgs a) {
  __shared__ double ssum[kStreamLen][kStreamCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = warp * 32 + lane;
  const Seg sg = stream_seg(a);
  const int u0 = blockIdx.x * kStreamCols + col;
  const bool ucol = u0 < a.mw;
  const int u = min(u0, a.mw - 1);
  const uint32_t cx = (uint32_t)(u + a.hx);
  const uint32_t M = (uint32_t)(a.hx + a.hy + 1);
  const uint32_t gm = M + cx, c2 = 2u * cx;
  const size_t ps8 = a.plane_stride * kOct;
  const size_t p8 = a.pitch * kOct;
  const uint16_t* tab = reinterpret_cast<const uint16_t*>(a.tab);
  const size_t ox0 = (size_t)u * kOct, ox1 = ox0 + (size_t)(a.hx + 1) * kOct,
               ox2 = ox0 + (size_t)(2 * a.hx + 1) * kOct;
  const int hy = a.hy;
  const int ybase = a.row0 + hy + a.y_off;
  const uint32_t seg_bytes = (uint32_t)min(kStreamCols, a.mw - (int)blockIdx.x * kStreamCols) * 16u;
  auto ld = [](const uint16_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); };
  stream_init(a, sg, ssum, col, u);

  for (int gi = 0; gi < a.nact; ++gi) {
    const int g = a.act[gi];
    const uint16_t* pl0 = tab + (size_t)g * a.planes * ps8;
    const uint16_t* pl1 = pl0 + ps8;
    const uint16_t* pl2 = pl1 + ps8;
    uint32_t S1[8], S2[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) S1[k] = S2[k] = 0u;
#pragma unroll 2
    for (int j = sg.kb; j < sg.ke + 2; ++j) {
      if (kStreamPf > 0 && threadIdx.x < 8 && j + kStreamPf < sg.ke + 2) {
        const size_t rp = (size_t)(a.row0 + chain_r(sg.c, hy, j + kStreamPf)) * p8;
        const int q = threadIdx.x;
        const uint16_t* pl = q < 3 ? pl0 : q < 6 ? pl1 : pl2;
        const int xi = q < 6 ? q % 3 : (q == 6 ? 0 : 2);
        const size_t ox = (size_t)(blockIdx.x * kStreamCols) * kOct +
                          (xi == 0 ? 0 : xi == 1 ? (size_t)(a.hx + 1) * kOct : (size_t)(2 * a.hx + 1) * kOct);
        l2_prefetch(pl + rp + ox, seg_bytes);
      }
      const size_t ro = (size_t)(a.row0 + chain_r(sg.c, hy, j)) * p8;
      const uint4 p0 = ld(pl0 + ro + ox0), p1 = ld(pl0 + ro + ox1), p2 = ld(pl0 + ro + ox2);
      const uint4 x0 = ld(pl1 + ro + ox0), x1 = ld(pl1 + ro + ox1), x2 = ld(pl1 + ro + ox2);
      const uint4 y0 = ld(pl2 + ro + ox0), y2 = ld(pl2 + ro + ox2);
      const uint32_t cyb = (uint32_t)(ybase + chain_r(sg.c, hy, j - 2));
      const uint32_t cym = (uint32_t)(ybase + chain_r(sg.c, hy, j - 1));
      const uint32_t cyt = (uint32_t)(ybase + chain_r(sg.c, hy, j));
      uint32_t H[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t A = h16(p2, k) - h16(p0, k), B = h16(p1, k) - h16(p0, k);
        const uint32_t XA = h16(x2, k) - h16(x0, k), XL = h16(x1, k) - h16(x0, k);
        const uint32_t YA = h16(y2, k) - h16(y0, k);
        const uint32_t G = gm * A + 2u * XL - XA - c2 * B;
        H[k] = (S1[k] + G - YA + cyb * A) & 0xFFFFu;
        S1[k] = S2[k] + 2u * YA - 2u * cym * A;
        S2[k] = cyt * A - G - YA;
      }
      if (j >= sg.kb + 2) {
        const int kk = j - 2 - sg.kb;
        double s = ssum[kk][col];
        score_octet<SIM>(a, g, H, s);
        ssum[kk][col] = s;
      }
    }
  }
  stream_finish<SIM>(a, sg, ssum, col, u, ucol);
}


// ---------------------------------------------------------------- quadratic
// Declared Euclidean kernel (k_sweep.cu K2q): H = A*N - ky*Dxx - kx*Dyy over
// the whole window box, Dxx = Sxx - 2cx*Sx + cx^2*N and Dyy likewise, all box
// sums of the planes {1, x, y, x^2, y^2} between the window's rows y0 = cy-hy
// and y2 = cy+hy+1.  Chains of step P = 2hy+1: window k's bottom row is
// window k+1's top row, so each row (5 planes at x0 and x2: 10 records) is
// loaded once and serves two windows.  Per row and bin, D_p = T_p(x2) -
// T_p(x0); Qx = D3 - 2cx D1 + cx^2 D0 and Qy(cy) = D4 - 2cy D2 + cy^2 D0 are
// linear (mod 2^32), so Dxx = Qx(y2) - Qx(y0), Dyy = Qy(y2; cy) - Qy(y0; cy):
// the state is (D0, Qx, Qy(cy of the next window)) of the last row.
template <int SIM>
__global__ void __launch_bounds__(kStreamThreads, SWG_STREAMQ_MINB) k_stream_quad(const SweepArgs a) {
  __shared__ double ssum[kStreamLen][kStreamCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = warp * 32 + lane;
  const Seg sg = quad_seg(a);
  const int u0 = blockIdx.x * kStreamCols + col;
  const bool ucol = u0 < a.mw;
  const int u = min(u0, a.mw - 1);
  const uint32_t cx = (uint32_t)(u + a.hx);
  const uint32_t c2x = 2u * cx, cxx = cx * cx;
  const uint64_t kx = (uint64_t)(a.hx + 1) * (a.hx + 1), ky = (uint64_t)(a.hy + 1) * (a.hy + 1);
  const uint64_t AK = 2 * kx * ky;
  const size_t ps8 = a.plane_stride * kOct;
  const size_t p8 = a.pitch * kOct;
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(a.tab);
  const size_t ox0 = (size_t)u * kOct, ox2 = ox0 + (size_t)(2 * a.hx + 1) * kOct;
  const int P = 2 * a.hy + 1;
  const int ybase = a.row0 + a.hy + a.y_off + sg.c;  // cy of window 0 of this chain
  const uint32_t seg_bytes = (uint32_t)min(kStreamCols, a.mw - (int)blockIdx.x * kStreamCols) * 32u;
  stream_init(a, sg, ssum, col, u, true);

  for (int gi = 0; gi < a.nact; ++gi) {
    const int g = a.act[gi];
    const uint32_t* pl = tab + (size_t)g * a.planes * ps8;
    uint32_t N0[8], QX[8], QY[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) N0[k] = QX[k] = QY[k] = 0u;
    for (int j = sg.kb; j <= sg.ke; ++j) {
      if (kStreamPfQ > 0 && threadIdx.x < 10 && j + kStreamPfQ <= sg.ke) {
        const size_t rp = (size_t)(a.row0 + sg.c + (j + kStreamPfQ) * P) * p8;
        const int q = threadIdx.x;  // plane q / 2 at x0 (even) or x2 (odd)
        const size_t ox = (size_t)(blockIdx.x * kStreamCols) * kOct +
                          ((q & 1) ? (size_t)(2 * a.hx + 1) * kOct : 0);
        l2_prefetch(pl + (size_t)(q >> 1) * ps8 + rp + ox, seg_bytes);
      }
      const size_t ro = (size_t)(a.row0 + sg.c + j * P) * p8;
      const uint32_t cyb = (uint32_t)(ybase + (j - 1) * P);  // window j-1 (bottom row)
      const uint32_t cyt = cyb + (uint32_t)P;                 // window j (top row)
      uint32_t D0[8], QXn[8];
      {
        const R8 a0 = ld256(pl + ro + ox0), a2 = ld256(pl + ro + ox2);
        const R8 b0 = ld256(pl + ps8 + ro + ox0), b2 = ld256(pl + ps8 + ro + ox2);
        const R8 d0 = ld256(pl + 3 * ps8 + ro + ox0), d2 = ld256(pl + 3 * ps8 + ro + ox2);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          D0[k] = a2.v[k] - a0.v[k];
          QXn[k] = (d2.v[k] - d0.v[k]) - c2x * (b2.v[k] - b0.v[k]) + cxx * D0[k];
        }
      }
      uint64_t H[8];
      {
        const R8 c0 = ld256(pl + 2 * ps8 + ro + ox0), c2 = ld256(pl + 2 * ps8 + ro + ox2);
        const R8 e0 = ld256(pl + 4 * ps8 + ro + ox0), e2 = ld256(pl + 4 * ps8 + ro + ox2);
        const uint32_t c2b = 2u * cyb, cbb = cyb * cyb, c2t = 2u * cyt, ctt = cyt * cyt;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t D2 = c2.v[k] - c0.v[k], D4 = e2.v[k] - e0.v[k];
          const uint32_t n = D0[k] - N0[k];
          const uint32_t dxx = QXn[k] - QX[k];
          const uint32_t dyy = (D4 - c2b * D2 + cbb * D0[k]) - QY[k];
          H[k] = AK * n - ky * dxx - kx * dyy;
          N0[k] = D0[k];
          QX[k] = QXn[k];
          QY[k] = D4 - c2t * D2 + ctt * D0[k];
        }
      }
      if (j > sg.kb) {  // window j-1 complete for this octet
        const int kk = j - 1 - sg.kb;
        double s = ssum[kk][col];
        score_octet<SIM>(a, g, H, s);
        ssum[kk][col] = s;
      }
    }
  }
  stream_finish<SIM, true>(a, sg, ssum, col, u, ucol);
}

}  // namespace

dim3 stream_grid(bool narrow, int mw, int rows, int hy) {
  (void)narrow;
  const int tw = kStreamCols;
  const int P = 2 * hy + 1;
  // chain 0 is the longest: windows at rows 0, hy+1, P, P+hy+1, ...
  const int ne = (rows + P - 1) / P, ro = rows - hy - 1;
  const int K = ne + (ro > 0 ? (ro + P - 1) / P : 0);
  const int nseg = std::max(1, (K + kStreamLen - 1) / kStreamLen);
  return dim3((unsigned)((mw + tw - 1) / tw), (unsigned)(nseg * (hy + 1)));
}

dim3 stream_quad_grid(int mw, int rows, int hy) {
  const int P = 2 * hy + 1;
  const int K = (rows + P - 1) / P;  // chain 0 is the longest
  const int nseg = std::max(1, (K + kStreamLen - 1) / kStreamLen);
  return dim3((unsigned)((mw + kStreamCols - 1) / kStreamCols), (unsigned)(nseg * P));
}

cudaError_t launch_stream_quad(const SweepArgs& a, dim3 grid, cudaStream_t s) {
  if (a.sim == SWG_SIM_BHATTACHARYYA) k_stream_quad<0><<<grid, kStreamThreads, 0, s>>>(a);
  else k_stream_quad<1><<<grid, kStreamThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_stream_affine(const SweepArgs& a, bool narrow, dim3 grid, cudaStream_t s) {
  if (narrow) {
    if (a.sim == SWG_SIM_BHATTACHARYYA) k_stream_affine16<0><<<grid, kStreamThreads, 0, s>>>(a);
    else k_stream_affine16<1><<<grid, kStreamThreads, 0, s>>>(a);
  } else {
    if (a.sim == SWG_SIM_BHATTACHARYYA) k_stream_affine<0><<<grid, kStreamThreads, 0, s>>>(a);
    else k_stream_affine<1><<<grid, kStreamThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace swg
