// k_build.cu — K0 quantise and K1 weighted integral-histogram build (sm_100a).
//
// K1 replaces IntegralTableSet::build (proj/src/integral_tables.cpp:72-115),
// which walks bin -> row -> column with running row sums plus the row above.
// The GPU splits the rows into bands and builds every band independently:
//   K1a k_colsum    per (band, bin octets, column): count and y-sum of each
//                   bin over the band's rows;
//   K1b k_bandscan  exclusive scan of those column sums over bands, so each
//                   band knows the column sums of all rows above it;
//   K1c k_build     one CTA per (band, octet, table kind) spanning the FULL
//                   row width (CPT columns per thread): one block scan turns
//                   the carried column sums into the band's top row
//                   T(x, y0); then per row a bin compare, one block-wide scan
//                   of the row prefixes (counts packed two bins per 32-bit
//                   word, or per-bin x sums), T(x+1, y+1) = T(x+1, y) +
//                   R(x, y), and one 32-byte record per column written with
//                   16-byte stores (4-8 KB contiguous per warp and row).
// (A single-pass decoupled look-back was measured first: with every band
// resident at once it re-read all earlier bands' 8-word column vectors,
// ~350 MB of L2 traffic for a 134 MB table; profiles/r01_v2_*.)
// Arithmetic is modulo 2^(8*sizeof(T)); for T = uint32_t every window
// histogram the sweeps form is < 2^32, so the wrapped tables are exact for
// them; T = uint64_t reproduces the reference's int64 tables.
#include "swg_internal.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace swg {

namespace {

template <int CPT>
__device__ __forceinline__ void load_bins(const uint16_t* p, uint16_t (&v)[CPT]) {
  if constexpr (CPT == 4) {
    const uint2 q = *reinterpret_cast<const uint2*>(p);
    v[0] = q.x & 0xFFFF; v[1] = q.x >> 16; v[2] = q.y & 0xFFFF; v[3] = q.y >> 16;
  } else {
    const uint4 q = *reinterpret_cast<const uint4*>(p);
    v[0] = q.x & 0xFFFF; v[1] = q.x >> 16; v[2] = q.y & 0xFFFF; v[3] = q.y >> 16;
    v[4] = q.z & 0xFFFF; v[5] = q.z >> 16; v[6] = q.w & 0xFFFF; v[7] = q.w >> 16;
  }
}

// One 8-element record with 16-byte stores.
template <typename T>
__device__ __forceinline__ void store_record(T* dst, const T (&v)[kOct]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
  if constexpr (sizeof(T) == 2) {
    d[0] = make_uint4(uint32_t(v[0]) | uint32_t(v[1]) << 16, uint32_t(v[2]) | uint32_t(v[3]) << 16,
                      uint32_t(v[4]) | uint32_t(v[5]) << 16, uint32_t(v[6]) | uint32_t(v[7]) << 16);
  } else if constexpr (sizeof(T) == 4) {
    d[0] = make_uint4(v[0], v[1], v[2], v[3]);
    d[1] = make_uint4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      d[j] = make_uint4((uint32_t)v[2 * j], (uint32_t)(v[2 * j] >> 32),
                        (uint32_t)v[2 * j + 1], (uint32_t)(v[2 * j + 1] >> 32));
  }
}

// Chunk q (16 bytes) of an 8-element record.
template <typename T>
__device__ __forceinline__ uint4 record_chunk(const T (&v)[kOct], int q) {
  if constexpr (sizeof(T) == 2) {
    return make_uint4(uint32_t(v[0]) | uint32_t(v[1]) << 16, uint32_t(v[2]) | uint32_t(v[3]) << 16,
                      uint32_t(v[4]) | uint32_t(v[5]) << 16, uint32_t(v[6]) | uint32_t(v[7]) << 16);
  } else if constexpr (sizeof(T) == 4) {
    return q == 0 ? make_uint4(v[0], v[1], v[2], v[3]) : make_uint4(v[4], v[5], v[6], v[7]);
  } else {
    return make_uint4((uint32_t)v[2 * q], (uint32_t)(v[2 * q] >> 32), (uint32_t)v[2 * q + 1],
                      (uint32_t)(v[2 * q + 1] >> 32));
  }
}

// 16-byte chunks per record build_body stages through shared memory (0:
// direct per-thread stores; the 64-bit export tables would need 256 KB).
template <typename T>
__host__ __device__ constexpr int stage_chunks_per_record() {
#ifdef SWG_NO_STAGE
  return 0;
#else
  return sizeof(T) == 8 ? 0 : (int)(kOct * sizeof(T) / 16);
#endif
}

template <typename T>
__device__ __forceinline__ void store_zero_record(T* dst) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int j = 0; j < (int)(kOct * sizeof(T) / 16); ++j) d[j] = make_uint4(0, 0, 0, 0);
}

// Exclusive block scan of N components with one __syncthreads.  `buf`
// ([N][32]) must not be rewritten before every thread passed this call's
// barrier; callers alternate two buffers.
template <int N, typename V>
__device__ __forceinline__ void block_exscan(const V (&val)[N], V (&excl)[N], V* buf,
                                             int lane, int warp, int nwarps) {
  V inc[N];
#pragma unroll
  for (int c = 0; c < N; ++c) inc[c] = val[c];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      const V t = __shfl_up_sync(0xFFFFFFFFu, inc[c], off);
      if (lane >= off) inc[c] += t;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < N; ++c) buf[c * 32 + warp] = inc[c];
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < N; ++c) {
    V wt = lane < nwarps ? buf[c * 32 + lane] : V(0);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const V t = __shfl_up_sync(0xFFFFFFFFu, wt, off);
      if (lane >= off) wt += t;
    }
    const V before = __shfl_sync(0xFFFFFFFFu, wt, warp > 0 ? warp - 1 : 0);
    excl[c] = (warp > 0 ? before : V(0)) + inc[c] - val[c];
  }
}

// K1a: column count, y-sum (and y^2-sum for quadratic planes) of each bin
// over one row band.  agg[band][group][column][aw]: words 0-7 counts, 8-15
// y-sums (aw >= 16: ramp planes), 16-23 y^2-sums (aw = 24).
// A thread owns one column and keeps its per-bin sums in SHARED memory
// (sums[plane][slot bin][thread]: conflict-free, private to the thread), so a
// pixel costs one read-modify-write per plane whatever the bin count -- the
// first form compared every pixel against each of an octet group's bins in
// registers (64-128 instructions per pixel, the pixels re-read per group:
// config 5 52 + 50 us for the quadratic and plain sets).  The bins summed
// are the octets the build will read (a selective build's, else all), in
// chunks of as many octets as the shared memory holds (blockIdx.z).
constexpr int kColThreads = 128;
constexpr int kColSmem = 96 << 10;
template <int AW>
__global__ void __launch_bounds__(kColThreads) k_colsum(const BuildArgs g, int opc) {
  extern __shared__ uint32_t s_sum[];  // [AW / 8][slots * 8][kColThreads]
  __shared__ unsigned char s_slot[kMaxBins / kOct];  // octet -> slot of this chunk (0xFF: none)
  constexpr int NP = AW / 8;
  const int tid = threadIdx.x, band = blockIdx.x;
  const int x = blockIdx.y * kColThreads + tid;
  const int noct = g.nsel ? g.nsel : g.groups;
  const int o0 = blockIdx.z * opc, slots = min(opc, noct - o0);
  for (int i = tid; i < g.groups; i += kColThreads) s_slot[i] = 0xFF;
  __syncthreads();
  if (tid < slots) s_slot[g.nsel ? (int)g.sel[o0 + tid] : o0 + tid] = (unsigned char)tid;
  const int nb = slots * kOct;  // bins of this chunk
  for (int i = tid; i < NP * nb * kColThreads; i += kColThreads) s_sum[i] = 0;
  __syncthreads();
  if (x >= g.w) return;
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  const uint16_t* col = g.fi + x;
  uint32_t* mine = s_sum + tid;
  constexpr int kB = 8;  // rows whose pixels are in flight at once
  for (int yb = y0; yb < y1; yb += kB) {
    uint32_t v[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) v[k] = yb + k < y1 ? (uint32_t)col[(size_t)(yb + k) * g.fi_pitch] : 0xFFFFu;
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const uint32_t d = v[k] - (uint32_t)g.bin0;
      if (d >= (uint32_t)g.bins) continue;  // another range's bin, or padding
      const uint32_t sl = s_slot[d >> 3];
      if (sl == 0xFFu) continue;
      uint32_t* p = mine + (sl * kOct + (d & 7u)) * kColThreads;
      const uint32_t y = (uint32_t)(yb + k);
      p[0] += 1u;
      if constexpr (AW >= 16) p[nb * kColThreads] += y;
      if constexpr (AW == 24) p[2 * nb * kColThreads] += y * y;
    }
  }
  for (int sl = 0; sl < slots; ++sl) {
    const int grp = g.nsel ? (int)g.sel[o0 + sl] : o0 + sl;
    uint4* dst = reinterpret_cast<uint4*>(g.agg + (((size_t)band * g.groups + grp) * g.wa + x) * AW);
#pragma unroll
    for (int pl = 0; pl < NP; ++pl) {
      const uint32_t* c = mine + ((size_t)pl * nb + sl * kOct) * kColThreads;
      dst[2 * pl] = make_uint4(c[0], c[kColThreads], c[2 * kColThreads], c[3 * kColThreads]);
      dst[2 * pl + 1] = make_uint4(c[4 * kColThreads], c[5 * kColThreads], c[6 * kColThreads],
                                   c[7 * kColThreads]);
    }
  }
}

// K1b: exclusive scan over bands, in place: agg[band] <- sum of agg[k < band].
// Q lanes (a power of two <= 32, consecutive lanes of a warp) share one uint4
// word of the carry array: each loads its kBandPT bands at once (all loads in
// flight), sums them, the lanes' sums are scanned with Q-wide shuffles, and
// each lane writes its bands' exclusive values.  Q (bandscan_lanes) grows
// while the grid would leave SMs short of threads and the bands are not yet
// covered in one round: 1-2 lanes for config 5's large carry arrays, 8 for
// config 2's small one (a whole warp per word idles most lanes and throttles
// on shuffles: config 5 +16 %).
constexpr int kBandPT = 10;
__global__ void __launch_bounds__(256) k_bandscan(uint4* agg, int nbands, size_t per_band,
                                                  const SelMask m, int q) {
  const size_t gt = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t col = gt / q;
  const int sub = (int)(gt % q);
  const bool act = col < per_band && !m.skip(col);  // (every lane stays for the shuffles)
  uint4 run = make_uint4(0, 0, 0, 0);
  for (int b0 = 0; b0 < nbands; b0 += q * kBandPT) {
    const int bs = b0 + sub * kBandPT;
    uint4 v[kBandPT];
    uint4 tot = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < kBandPT; ++k)
      v[k] = act && bs + k < nbands ? agg[(size_t)(bs + k) * per_band + col] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < kBandPT; ++k) {
      tot.x += v[k].x; tot.y += v[k].y; tot.z += v[k].z; tot.w += v[k].w;
    }
    uint4 inc = tot;
    for (int off = 1; off < q; off <<= 1) {
      const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, inc.x, off, q);
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc.y, off, q);
      const uint32_t z = __shfl_up_sync(0xFFFFFFFFu, inc.z, off, q);
      const uint32_t w = __shfl_up_sync(0xFFFFFFFFu, inc.w, off, q);
      if (sub >= off) {
        inc.x += x; inc.y += y; inc.z += z; inc.w += w;
      }
    }
    uint4 pre = make_uint4(run.x + inc.x - tot.x, run.y + inc.y - tot.y, run.z + inc.z - tot.z,
                           run.w + inc.w - tot.w);
#pragma unroll
    for (int k = 0; k < kBandPT; ++k) {
      if (act && bs + k < nbands) agg[(size_t)(bs + k) * per_band + col] = pre;
      pre.x += v[k].x; pre.y += v[k].y; pre.z += v[k].z; pre.w += v[k].w;
    }
    run.x += __shfl_sync(0xFFFFFFFFu, inc.x, q - 1, q);
    run.y += __shfl_sync(0xFFFFFFFFu, inc.y, q - 1, q);
    run.z += __shfl_sync(0xFFFFFFFFu, inc.z, q - 1, q);
    run.w += __shfl_sync(0xFFFFFFFFu, inc.w, q - 1, q);
  }
}

// K1c body.  KIND 0 = plain {1}, 1 = xramp {x}, 2 = yramp {y}, and for the
// quadratic planes 3 = {x^2}, 4 = {y^2} (32- or 64-bit tables; everything
// wraps consistently mod 2^32 / 2^64).
template <typename T, int KIND, int CPT>
__device__ __forceinline__ void build_body(const BuildArgs& g, int band, int grp) {
  __shared__ uint32_t s_row[2][kOct * 32];
  __shared__ T s_rowT[KIND == 3 ? 2 : 1][KIND == 3 ? kOct * 32 : 1];
  __shared__ T s_carry[kOct * 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int y0 = band * g.band_h;
  const int y1 = min(y0 + g.band_h, g.h);
  const int xb = tid * CPT;
  // Threads past the right edge keep the block scans uniform but touch no
  // memory; the last live thread may straddle the edge (padding = kNoBin).
  const bool live = xb < g.w;
  const uint16_t* fi = g.fi + (live ? xb : 0);
  const uint32_t gb = (uint32_t)g.bin0 + (uint32_t)grp * kOct;
  const uint32_t lim = (uint32_t)(g.bins - grp * kOct);  // bins of this octet in range

  // ---- carry row T(x+1, y0) from the column sums of all rows above y0
  T t[CPT][kOct];
  {
    T tot[kOct], ex[kOct];
    uint32_t cc[CPT][kOct];
    if (live && band > 0) {  // band 0 starts from the zero row
      // counts for kinds 0/1/3, y-sums for kind 2, y^2-sums for kind 4
      const uint4* src = reinterpret_cast<const uint4*>(
          g.agg + (((size_t)band * g.groups + grp) * g.wa + xb) * g.aw +
          (KIND == 2 ? 8 : KIND == 4 ? 16 : 0));
      const int st = g.aw / 4;  // uint4 per column
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const uint4 a = src[st * i], b = src[st * i + 1];
        cc[i][0] = a.x; cc[i][1] = a.y; cc[i][2] = a.z; cc[i][3] = a.w;
        cc[i][4] = b.x; cc[i][5] = b.y; cc[i][6] = b.z; cc[i][7] = b.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CPT; ++i)
#pragma unroll
        for (int j = 0; j < kOct; ++j) cc[i][j] = 0;
    }
#pragma unroll
    for (int j = 0; j < kOct; ++j) {
      T run = 0;
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const T x = (T)(xb + i);
        run += KIND == 1 ? (T)cc[i][j] * x : KIND == 3 ? (T)cc[i][j] * x * x : (T)cc[i][j];
        t[i][j] = run;
      }
      tot[j] = run;
    }
    block_exscan<kOct, T>(tot, ex, s_carry, lane, warp, nwarps);
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int j = 0; j < kOct; ++j) t[i][j] += ex[j];
  }

  // 16-bit plain planes: the running table values stay PACKED, two bins per
  // 32-bit word -- the record's own layout -- and a row adds its packed row
  // prefix with one 16x2 SIMD add per word (VIADD.16x2: each half wraps mod
  // 2^16 on its own), instead of eight extractions and adds per column
  constexpr bool PK = sizeof(T) == 2 && KIND == 0;
  [[maybe_unused]] uint32_t tp[PK ? CPT : 1][4];
  if constexpr (PK) {
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        tp[i][q] = (uint32_t)t[i][2 * q] | (uint32_t)t[i][2 * q + 1] << 16;
  }
  T* plane = reinterpret_cast<T*>(g.out) +
             ((size_t)grp * g.planes + KIND) * g.plane_stride * kOct;
  if (band == 0) {  // zero row 0
    if (live)
#pragma unroll
      for (int i = 0; i < CPT; ++i) store_zero_record<T>(plane + (size_t)(xb + 1 + i) * kOct);
    if (tid == 0) store_zero_record<T>(plane);
    if (sizeof(T) == 4 && KIND <= 2 && g.out16) {
      uint16_t* p16 = static_cast<uint16_t*>(g.out16) + ((size_t)grp * 3 + KIND) * g.plane_stride * kOct;
      if (live)
#pragma unroll
        for (int i = 0; i < CPT; ++i) store_zero_record<uint16_t>(p16 + (size_t)(xb + 1 + i) * kOct);
      if (tid == 0) store_zero_record<uint16_t>(p16);
    }
  }

  // ---- rows of the band (next row's bins prefetched under this row's scan)
  uint16_t vn[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) vn[i] = kNoBin;
  if (live && y0 < y1) load_bins<CPT>(fi + (size_t)y0 * g.fi_pitch, vn);
  for (int y = y0; y < y1; ++y) {
    uint32_t d[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      d[i] = (uint32_t)vn[i] - gb;
      d[i] = d[i] < lim ? d[i] : 0xFFFFFFFFu;
    }
    if (live && y + 1 < y1) load_bins<CPT>(fi + (size_t)(y + 1) * g.fi_pitch, vn);
    uint32_t* buf = s_row[y & 1];
    if constexpr (KIND == 3) {
      // per-bin x^2 sums (64-bit: a row prefix reaches W^3/3)
      T tot[kOct], ex[kOct];
#pragma unroll
      for (int j = 0; j < kOct; ++j) {
        T s = 0;
#pragma unroll
        for (int i = 0; i < CPT; ++i)
          s += (d[i] == (uint32_t)j) ? (T)(xb + i) * (T)(xb + i) : (T)0;
        tot[j] = s;
      }
      block_exscan<kOct, T>(tot, ex, s_rowT[y & 1], lane, warp, nwarps);
#pragma unroll
      for (int i = 0; i < CPT; ++i)
#pragma unroll
        for (int j = 0; j < kOct; ++j) {
          ex[j] += (d[i] == (uint32_t)j) ? (T)(xb + i) * (T)(xb + i) : (T)0;
          t[i][j] += ex[j];
        }
    } else if constexpr (KIND == 1) {
      // per-bin x sums of this thread's columns, then the block prefix
      uint32_t tot[kOct], ex[kOct];
#pragma unroll
      for (int j = 0; j < kOct; ++j) {
        uint32_t s = 0;
#pragma unroll
        for (int i = 0; i < CPT; ++i) s += (d[i] == (uint32_t)j) ? (uint32_t)(xb + i) : 0u;
        tot[j] = s;
      }
      block_exscan<kOct, uint32_t>(tot, ex, buf, lane, warp, nwarps);
#pragma unroll
      for (int i = 0; i < CPT; ++i)
#pragma unroll
        for (int j = 0; j < kOct; ++j) {
          ex[j] += (d[i] == (uint32_t)j) ? (uint32_t)(xb + i) : 0u;
          t[i][j] += (T)ex[j];
        }
    } else {
      // counts, two bins per 32-bit word (16-bit fields; row prefix <= W < 2^16)
      uint32_t tot[4], ex[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t s = 0;
#pragma unroll
        for (int i = 0; i < CPT; ++i)
          s += ((d[i] >> 1) == (uint32_t)q) ? (1u << ((d[i] & 1u) << 4)) : 0u;
        tot[q] = s;
      }
      block_exscan<4, uint32_t>(tot, ex, buf, lane, warp, nwarps);
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ex[q] += ((d[i] >> 1) == (uint32_t)q) ? (1u << ((d[i] & 1u) << 4)) : 0u;
        if constexpr (PK) {
#pragma unroll
          for (int q = 0; q < 4; ++q) tp[i][q] = __vadd2(tp[i][q], ex[q]);
        } else {
#pragma unroll
          for (int j = 0; j < kOct; ++j) {
            const uint32_t r = (ex[j >> 1] >> ((j & 1) << 4)) & 0xFFFFu;
            t[i][j] += KIND == 2 ? (T)y * (T)r : KIND == 4 ? (T)y * (T)y * (T)r : (T)r;
          }
        }
      }
    }
    T* row = plane + (size_t)(y + 1) * g.pitch * kOct;
    constexpr int NQ = stage_chunks_per_record<T>();
    if constexpr (NQ > 0) {
      // coalesced row stores: the warp's 32*CPT records are staged in shared
      // memory (XOR-swizzled 16-byte chunks = the TMA SWIZZLE_128B layout)
      // and written back by ONE cp.async.bulk.tensor store per warp and row
      // (the TMA engine reads shared memory: no per-thread global stores
      // through the LSU), or without a tensor map as 512 contiguous bytes
      // per store instruction
      extern __shared__ __align__(1024) uint4 s_stage[];
      uint4* st = s_stage + warp * 32 * CPT * NQ;
      auto swz = [](int c) { return c ^ ((c >> 3) & 7); };
      const int wrec0 = warp * 32 * CPT;
      const bool tma = g.tmap_ok && wrec0 < g.w;
      if (tma && lane == 0) {  // the previous row's store has read the buffer
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < CPT; ++i)
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          if constexpr (PK) st[swz(lane * CPT + i)] = make_uint4(tp[i][0], tp[i][1], tp[i][2], tp[i][3]);
          else st[swz((lane * CPT + i) * NQ + q)] = record_chunk<T>(t[i], q);
        }
      if (tma) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const int line0 = wrec0 * (int)(kOct * sizeof(T)) / 128;
          const int plane_i = grp * g.planes + KIND;
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(st);
          asm volatile(
              "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
              ::"l"(&g.tmap), "r"(0), "r"(line0), "r"(y + 1), "r"(plane_i), "r"(sa)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else {
        __syncwarp();
        uint4* dst = reinterpret_cast<uint4*>(row) + (size_t)(wrec0 + 1) * NQ;
#pragma unroll
        for (int m = 0; m < CPT * NQ; ++m) {
          const int c = m * 32 + lane;
          if (wrec0 + c / NQ < g.w) dst[c] = st[swz(c)];
        }
      }
      __syncwarp();
      if constexpr (sizeof(T) == 4 && KIND <= 2) {
        // the narrow {1, x, y} planes (low 16 bits, 3-plane layout) from the
        // same values: one more staged pass of 16-byte records
        if (g.out16) {
          if (tma && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
          uint16_t* row16 = static_cast<uint16_t*>(g.out16) +
                            (((size_t)grp * 3 + KIND) * g.plane_stride + (size_t)(y + 1) * g.pitch) *
                                kOct;
#pragma unroll
          for (int i = 0; i < CPT; ++i) {
            const T* v = t[i];
            st[swz(lane * CPT + i)] =
                make_uint4((uint32_t)(v[0] & 0xFFFFu) | (uint32_t)v[1] << 16,
                           (uint32_t)(v[2] & 0xFFFFu) | (uint32_t)v[3] << 16,
                           (uint32_t)(v[4] & 0xFFFFu) | (uint32_t)v[5] << 16,
                           (uint32_t)(v[6] & 0xFFFFu) | (uint32_t)v[7] << 16);
          }
          __syncwarp();
          uint4* dst16 = reinterpret_cast<uint4*>(row16) + (size_t)(wrec0 + 1);
#pragma unroll
          for (int m = 0; m < CPT; ++m) {
            const int c = m * 32 + lane;
            if (wrec0 + c < g.w) dst16[c] = st[swz(c)];
          }
          __syncwarp();
          if (tid == 0) reinterpret_cast<uint4*>(row16)[0] = make_uint4(0, 0, 0, 0);
        }
      }
    } else {
      if (live)
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
          if constexpr (PK)
            *reinterpret_cast<uint4*>(row + (size_t)(xb + 1 + i) * kOct) =
                make_uint4(tp[i][0], tp[i][1], tp[i][2], tp[i][3]);
          else
            store_record<T>(row + (size_t)(xb + 1 + i) * kOct, t[i]);
        }
    }
    if (tid == 0) store_zero_record<T>(row);
  }
  if constexpr (stage_chunks_per_record<T>() > 0) {  // every TMA store done before exit
    if (g.tmap_ok && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// K1c: one CTA per (row band, bin octet); one launch per table kind so each
// kind gets its own register allocation.
template <typename T, int KIND, int CPT>
__global__ void __launch_bounds__(512) k_build(const __grid_constant__ BuildArgs g) {
  const int ng = g.nsel ? g.nsel : g.groups;  // selective build: the listed octets
  const int i = blockIdx.x % ng;
  build_body<T, KIND, CPT>(g, blockIdx.x / ng, g.nsel ? (int)g.sel[i] : i);
}

// Small tables: all kinds in ONE launch (blockIdx.y = kind) -- fewer
// serialized launches where a launch is latency, not bandwidth.
template <typename T, int CPT>
__global__ void __launch_bounds__(512) k_build_fused(const __grid_constant__ BuildArgs g) {
  const int ng = g.nsel ? g.nsel : g.groups;
  const int band = blockIdx.x / ng, grp = g.nsel ? (int)g.sel[blockIdx.x % ng] : blockIdx.x % ng;
  switch (blockIdx.y) {
    case 0: build_body<T, 0, CPT>(g, band, grp); break;
    case 1: build_body<T, 1, CPT>(g, band, grp); break;
    case 2: build_body<T, 2, CPT>(g, band, grp); break;
    default:
      if constexpr (sizeof(T) >= 4) {
        if (blockIdx.y == 3) build_body<T, 3, CPT>(g, band, grp);
        else build_body<T, 4, CPT>(g, band, grp);
      }
  }
}

// K0: any input format -> uint16 bin image (pitched, padded with kNoBin).
__global__ void k_quantize(const QuantArgs a) {
  const int y = blockIdx.y;
  const uint8_t* row = a.in + (size_t)y * a.in_pitch;
  uint16_t* dst = a.fi + (size_t)y * a.fi_pitch;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < (int)a.fi_pitch;
       x += gridDim.x * blockDim.x) {
    uint16_t bin = kNoBin;
    if (x < a.w) {
      switch (a.format) {
        case SWG_FMT_GRAY8:  // image.hpp:43-45
          bin = (uint16_t)(((uint32_t)row[x] * (uint32_t)a.bins) >> 8);
          break;
        case SWG_FMT_GRAY16:
          bin = (uint16_t)(((uint32_t)reinterpret_cast<const uint16_t*>(row)[x] *
                            (uint32_t)a.bins) >> 16);
          break;
        case SWG_FMT_RGB8: {
          const uint32_t n = (uint32_t)a.bins;  // levels per channel
          const uint32_t r = (row[3 * x] * n) >> 8, gg = (row[3 * x + 1] * n) >> 8,
                         b = (row[3 * x + 2] * n) >> 8;
          bin = (uint16_t)((r * n + gg) * n + b);
          break;
        }
        default:
          bin = reinterpret_cast<const uint16_t*>(row)[x];
      }
    }
    dst[x] = bin;
  }
}

// K0, 8 pixels per thread (16-byte stores of the bin image; 8-, 16- or
// 24-byte pixel loads): rows whose start and pitch are 16-byte aligned.  One
// pixel per thread is launch-shaped work -- 16 K CTAs for a 2048^2 frame,
// 14 us where the 16 MB of traffic take 3.
__device__ __forceinline__ uint16_t quant_one(const QuantArgs& a, const uint8_t* row, int x) {
  switch (a.format) {
    case SWG_FMT_GRAY8:
      return (uint16_t)(((uint32_t)row[x] * (uint32_t)a.bins) >> 8);
    case SWG_FMT_GRAY16:
      return (uint16_t)(((uint32_t)reinterpret_cast<const uint16_t*>(row)[x] * (uint32_t)a.bins) >> 16);
    case SWG_FMT_RGB8: {
      const uint32_t n = (uint32_t)a.bins;
      const uint32_t r = (row[3 * x] * n) >> 8, gg = (row[3 * x + 1] * n) >> 8,
                     b = (row[3 * x + 2] * n) >> 8;
      return (uint16_t)((r * n + gg) * n + b);
    }
    default:
      return reinterpret_cast<const uint16_t*>(row)[x];
  }
}

__global__ void __launch_bounds__(256) k_quantize_v8(const QuantArgs a) {
  const int y = blockIdx.y;
  const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (x0 >= (int)a.fi_pitch) return;
  const uint8_t* row = a.in + (size_t)y * a.in_pitch;
  uint32_t v[8];
  if (x0 + 8 <= a.w) {
    const uint32_t n = (uint32_t)a.bins;
    if (a.format == SWG_FMT_GRAY8) {
      const uint2 q = *reinterpret_cast<const uint2*>(row + x0);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = ((((i < 4 ? q.x : q.y) >> (8 * (i & 3))) & 0xFFu) * n) >> 8;
    } else if (a.format == SWG_FMT_RGB8) {
      const uint2* p = reinterpret_cast<const uint2*>(row + 3 * x0);
      const uint2 q0 = p[0], q1 = p[1], q2 = p[2];
      const uint32_t w[6] = {q0.x, q0.y, q1.x, q1.y, q2.x, q2.y};
      auto byte = [&](int k) { return (w[k >> 2] >> (8 * (k & 3))) & 0xFFu; };
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t r = (byte(3 * i) * n) >> 8, gg = (byte(3 * i + 1) * n) >> 8,
                       b = (byte(3 * i + 2) * n) >> 8;
        v[i] = (r * n + gg) * n + b;
      }
    } else {
      const uint4 q = *reinterpret_cast<const uint4*>(row + 2 * x0);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t px = (w[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
        v[i] = a.format == SWG_FMT_GRAY16 ? (px * n) >> 16 : px;
      }
    }
  } else {  // the row's ragged end and its padding
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = x0 + i < a.w ? quant_one(a, row, x0 + i) : kNoBin;
  }
  *reinterpret_cast<uint4*>(a.fi + (size_t)y * a.fi_pitch + x0) =
      make_uint4((v[0] & 0xFFFFu) | v[1] << 16, (v[2] & 0xFFFFu) | v[3] << 16,
                 (v[4] & 0xFFFFu) | v[5] << 16, (v[6] & 0xFFFFu) | v[7] << 16);
}

// Octet layout -> reference bin-major layout [bin][y][x] (export).
template <typename T, typename O>
__global__ void k_export(const T* tab, size_t ps, size_t pitch, int planes, int w, int h,
                         int kind, int b0, O* out) {
  const int b = b0 + blockIdx.z;
  const int y = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x <= w; x += gridDim.x * blockDim.x)
    out[((size_t)blockIdx.z * (h + 1) + y) * (w + 1) + x] =
        (O)tab[elem_index(ps, pitch, planes, x, y, b, kind)];
}

// Reference layout int64 (bin-major) -> octet uint64 planes (SWIH1 load).
__global__ void k_import(const int64_t* src, int w, int h, int kind, uint64_t* tab,
                         size_t ps, size_t pitch, int planes) {
  const int b = blockIdx.z;
  const int y = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x <= w; x += gridDim.x * blockDim.x)
    tab[elem_index(ps, pitch, planes, x, y, b, kind)] =
        (uint64_t)src[((size_t)b * (h + 1) + y) * (w + 1) + x];
}

// Boundary prefix-row exchange on the device (SURVEY §8e "row bands"): a
// band built from pixel rows [y0, y0 + h) holds LOCAL tables (zero at its
// own row 0).  k_last_row copies its last record row (row h) of kinds
// 0 .. kinds-1 for every octet -- the band's contribution to the prefix row
// below it -- into out[(g * kinds + k) * (w+1) + x] (records); after an
// all-gather, k_add_carry turns the local tables into the global ones:
//   plain  p' = p + c0             xramp  x' = x + c1
//   yramp  y' = y + y0 p + c2      (rows shift by y0: sum(y_l + y0) = y + y0 N)
//   x^2    xx' = xx + c3           y^2    yy' = yy + 2 y0 y + y0^2 p + c4
// with c the exclusive sum of the earlier bands' (already shifted) last
// rows, all modulo 2^32 like the tables themselves.
__global__ void k_last_row(const uint32_t* tab, size_t ps, size_t pitch, int planes, int kinds,
                           int w, int h, int groups, uint4* out) {
  const size_t n = (size_t)groups * kinds * (w + 1) * 2;  // uint4 halves of records
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t rec = i >> 1;
    const int x = (int)(rec % (w + 1));
    const int gk = (int)(rec / (w + 1)), g = gk / kinds, k = gk % kinds;
    const uint4* src = reinterpret_cast<const uint4*>(
        tab + (((size_t)g * planes + k) * ps + (size_t)h * pitch + x) * kOct);
    out[i] = src[i & 1];
  }
}

__global__ void k_add_carry(uint32_t* tab, size_t ps, size_t pitch, int planes, int kinds,
                            int w, int h, int groups, uint32_t y0, const uint32_t* carry) {
  const size_t n = (size_t)groups * (h + 1) * (w + 1) * 2;  // half records (4 bins)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int half = (int)(i & 1);
    const size_t rec = i >> 1;
    const int x = (int)(rec % (w + 1));
    const size_t gy = rec / (w + 1);
    const int y = (int)(gy % (h + 1)), g = (int)(gy / (h + 1));
    uint4 v[5], c[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (k >= kinds) break;
      v[k] = reinterpret_cast<const uint4*>(
          tab + (((size_t)g * planes + k) * ps + (size_t)y * pitch + x) * kOct)[half];
      c[k] = reinterpret_cast<const uint4*>(
          carry + (((size_t)g * kinds + k) * (w + 1) + x) * kOct)[half];
    }
    uint32_t p[4] = {v[0].x, v[0].y, v[0].z, v[0].w};
    uint32_t out[5][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t cj[5] = {(&c[0].x)[j], kinds > 1 ? (&c[1].x)[j] : 0u,
                              kinds > 2 ? (&c[2].x)[j] : 0u, kinds > 3 ? (&c[3].x)[j] : 0u,
                              kinds > 4 ? (&c[4].x)[j] : 0u};
      out[0][j] = p[j] + cj[0];
      if (kinds > 1) out[1][j] = (&v[1].x)[j] + cj[1];
      if (kinds > 2) out[2][j] = (&v[2].x)[j] + y0 * p[j] + cj[2];
      if (kinds > 3) out[3][j] = (&v[3].x)[j] + cj[3];
      if (kinds > 4)
        out[4][j] = (&v[4].x)[j] + 2u * y0 * (&v[2].x)[j] + y0 * y0 * p[j] + cj[4];
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (k >= kinds) break;
      reinterpret_cast<uint4*>(tab + (((size_t)g * planes + k) * ps + (size_t)y * pitch + x) *
                                         kOct)[half] =
          make_uint4(out[k][0], out[k][1], out[k][2], out[k][3]);
    }
  }
}

__global__ void k_narrow(const uint64_t* src, uint32_t* dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = (uint32_t)src[i];
}

}  // namespace

cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t s) {
  const int threads = 256;
  if (((reinterpret_cast<uintptr_t>(a.in) | a.in_pitch) & 15) == 0 && !std::getenv("SWG_QUANT_SCALAR")) {
    dim3 grid((unsigned)((a.fi_pitch / 8 + threads - 1) / threads), (unsigned)a.h);
    k_quantize_v8<<<grid, threads, 0, s>>>(a);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((a.fi_pitch + threads - 1) / threads), (unsigned)a.h);
  k_quantize<<<grid, threads, 0, s>>>(a);
  return cudaGetLastError();
}

// Opt a build kernel into the dynamic shared memory its row staging needs.
// (static + dynamic shared memory above 48 KB needs the opt-in; the fused
// kernel's static arrays add up over its table kinds)
template <typename K>
static void allow_smem(K* kernel, size_t bytes) {
  if (bytes) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t launch_colsum(const BuildArgs& a, cudaStream_t s) {
  // octets per chunk: as many as kColSmem holds (aw / 8 planes of 8 bins x
  // kColThreads words each)
  const int noct = a.nsel ? a.nsel : a.groups;
  const int opc = std::min(noct, kColSmem / (a.aw / 8 * kOct * kColThreads * 4));
  const size_t smem = (size_t)opc * (a.aw / 8) * kOct * kColThreads * 4;
  dim3 grid((unsigned)a.nbands, (unsigned)((a.w + kColThreads - 1) / kColThreads),
            (unsigned)((noct + opc - 1) / opc));
  auto go = [&](auto kernel) {
    allow_smem(kernel, smem);
    kernel<<<grid, kColThreads, smem, s>>>(a, opc);
  };
  if (a.aw == 8) go(k_colsum<8>);
  else if (a.aw == 16) go(k_colsum<16>);
  else go(k_colsum<24>);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t per_band = (size_t)a.groups * a.wa * a.aw / 4;
  SelMask m{};
  m.on = a.nsel > 0;
  m.words_per_unit = a.wa * a.aw / 4;
  std::memcpy(m.w, a.selmask, sizeof(m.w));
  const int q = bandscan_lanes(a.nbands, per_band);
  k_bandscan<<<(unsigned)((per_band * q + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<uint4*>(a.agg), a.nbands, per_band, m, q);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_build(const BuildArgs& a, cudaStream_t s, int* launches) {
  const int cpt = choose_cpt(a.w);
  const int threads = (int)round_up((size_t)((a.w + cpt - 1) / cpt), 32);
  const size_t smem = (size_t)threads * cpt * stage_chunks_per_record<T>() * 16;
  const unsigned grid = (unsigned)(a.nbands * (a.nsel ? a.nsel : a.groups));
  // narrow tables: plain only, unless asked for (the 16-bit {1, x, y} planes)
  const int kinds = a.kinds > 0 ? a.kinds : sizeof(T) == 2 ? 1 : a.planes;
  bool fuse = kinds > 1 && grid < 2u * 148u;
  if (const char* ef = std::getenv("SWG_BUILD_FUSED")) fuse = kinds > 1 && std::atoi(ef) != 0;  // A/B
  if (fuse) {
    dim3 g3(grid, (unsigned)kinds);
    if (cpt == 4) {
      allow_smem(k_build_fused<T, 4>, smem);
      k_build_fused<T, 4><<<g3, threads, smem, s>>>(a);
    } else {
      allow_smem(k_build_fused<T, 8>, smem);
      k_build_fused<T, 8><<<g3, threads, smem, s>>>(a);
    }
    *launches = 1;
    return cudaGetLastError();
  }
  *launches = kinds;
  auto go = [&](auto kernel) {
    allow_smem(kernel, smem);
    kernel<<<grid, threads, smem, s>>>(a);
  };
  for (int kind = 0; kind < kinds; ++kind) {
    if (cpt == 4) {
      if (kind == 0) go(k_build<T, 0, 4>);
      else if (kind == 1) go(k_build<T, 1, 4>);
      else if (kind == 2) go(k_build<T, 2, 4>);
      else if constexpr (sizeof(T) >= 4) {
        if (kind == 3) go(k_build<T, 3, 4>);
        else go(k_build<T, 4, 4>);
      }
    } else {
      if (kind == 0) go(k_build<T, 0, 8>);
      else if (kind == 1) go(k_build<T, 1, 8>);
      else if (kind == 2) go(k_build<T, 2, 8>);
      else if constexpr (sizeof(T) >= 4) {
        if (kind == 3) go(k_build<T, 3, 8>);
        else go(k_build<T, 4, 8>);
      }
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template cudaError_t launch_build<uint16_t>(const BuildArgs&, cudaStream_t, int*);
template cudaError_t launch_build<uint32_t>(const BuildArgs&, cudaStream_t, int*);
template cudaError_t launch_build<uint64_t>(const BuildArgs&, cudaStream_t, int*);

template <typename T, typename O>
cudaError_t launch_export(const T* tab, size_t ps, size_t pitch, int planes, int w, int h,
                          int kind, int b0, int b1, O* out, cudaStream_t s) {
  dim3 grid((unsigned)((w + 1 + 255) / 256), (unsigned)(h + 1), (unsigned)(b1 - b0));
  k_export<T, O><<<grid, 256, 0, s>>>(tab, ps, pitch, planes, w, h, kind, b0, out);
  return cudaGetLastError();
}
template cudaError_t launch_export<uint32_t, uint32_t>(const uint32_t*, size_t, size_t, int,
                                                       int, int, int, int, int, uint32_t*,
                                                       cudaStream_t);
template cudaError_t launch_export<uint64_t, int64_t>(const uint64_t*, size_t, size_t, int,
                                                      int, int, int, int, int, int64_t*,
                                                      cudaStream_t);

cudaError_t launch_import_i64(const int64_t* src, int w, int h, int bins, int kind,
                              uint64_t* tab, size_t ps, size_t pitch, int planes,
                              cudaStream_t s) {
  dim3 grid((unsigned)((w + 1 + 255) / 256), (unsigned)(h + 1), (unsigned)bins);
  k_import<<<grid, 256, 0, s>>>(src, w, h, kind, tab, ps, pitch, planes);
  return cudaGetLastError();
}

cudaError_t launch_last_row(const uint32_t* tab, size_t ps, size_t pitch, int planes, int kinds,
                            int w, int h, int groups, void* out, cudaStream_t s) {
  k_last_row<<<148 * 4, 256, 0, s>>>(tab, ps, pitch, planes, kinds, w, h, groups,
                                      static_cast<uint4*>(out));
  return cudaGetLastError();
}

cudaError_t launch_add_carry(uint32_t* tab, size_t ps, size_t pitch, int planes, int kinds, int w,
                             int h, int groups, int y0, const void* carry, cudaStream_t s) {
  k_add_carry<<<148 * 8, 256, 0, s>>>(tab, ps, pitch, planes, kinds, w, h, groups, (uint32_t)y0,
                                       static_cast<const uint32_t*>(carry));
  return cudaGetLastError();
}

cudaError_t launch_narrow(const uint64_t* src, uint32_t* dst, size_t n, cudaStream_t s) {
  k_narrow<<<148 * 8, 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

}  // namespace swg
