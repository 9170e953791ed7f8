// k_build.cu — K0 quantise and K1 weighted integral-histogram build (sm_100a).
//
// K1 replaces IntegralTableSet::build (proj/src/integral_tables.cpp:72-115).
// The reference walks bin -> row -> column with running row sums plus the row
// above.  Here one CTA owns (row band, bin) and the FULL row width:
//   phase 1  column aggregates of its band (count, y-sum per column),
//            published for later bands;
//   phase 2  decoupled look-back over earlier bands of the same bin (flags +
//            aggregates / inclusive prefixes in global memory) gives the
//            column sums of all rows above the band; one block scan turns
//            them into the band's carry row T(x, y0);
//   phase 3  per row: bin compare, block-wide scan of (count, x-sum) row
//            prefixes, T(x+1, y+1) = T(x+1, y) + R(x, y) for the three
//            planes {1, x, y}, written once with 16-byte vector stores
//            (a warp writes 512 B - 2 KB contiguous per plane and row).
// Arithmetic is modulo 2^(8*sizeof(T)); for T = uint32_t every window
// histogram the sweep forms is < 2^32, so the wrapped tables are exact for
// it.
#include "swg_internal.cuh"

namespace swg {

namespace {

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int CPT>
__device__ __forceinline__ void load_bins(const uint16_t* p, uint16_t (&v)[CPT]) {
  if constexpr (CPT == 4) {
    const uint2 q = *reinterpret_cast<const uint2*>(p);
    v[0] = q.x & 0xFFFF; v[1] = q.x >> 16; v[2] = q.y & 0xFFFF; v[3] = q.y >> 16;
  } else {
#pragma unroll
    for (int j = 0; j < CPT / 8; ++j) {
      const uint4 q = *reinterpret_cast<const uint4*>(p + 8 * j);
      v[8 * j + 0] = q.x & 0xFFFF; v[8 * j + 1] = q.x >> 16;
      v[8 * j + 2] = q.y & 0xFFFF; v[8 * j + 3] = q.y >> 16;
      v[8 * j + 4] = q.z & 0xFFFF; v[8 * j + 5] = q.z >> 16;
      v[8 * j + 6] = q.w & 0xFFFF; v[8 * j + 7] = q.w >> 16;
    }
  }
}

// Stores CPT consecutive elements (16-byte aligned) with 16-byte stores.
template <typename T, int CPT>
__device__ __forceinline__ void store_run(T* dst, const T (&v)[CPT]) {
  static_assert((CPT * sizeof(T)) % 16 == 0, "vector store");
#pragma unroll
  for (int j = 0; j < (int)(CPT * sizeof(T) / 16); ++j) {
    uint4 q;
    if constexpr (sizeof(T) == 4) {
      q = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
      q = make_uint4((uint32_t)v[2 * j], (uint32_t)(v[2 * j] >> 32),
                     (uint32_t)v[2 * j + 1], (uint32_t)(v[2 * j + 1] >> 32));
    }
    reinterpret_cast<uint4*>(dst)[j] = q;
  }
}

// Exclusive block scan of N components; one __syncthreads.  `buf` must not
// be reused by the next call before every thread passed this call's sync
// (callers alternate two buffers).
template <int N, typename V>
__device__ __forceinline__ void block_exscan(const V (&val)[N], V (&excl)[N],
                                             V* buf, int lane, int warp,
                                             int nwarps) {
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

template <typename T, int P, int CPT>
__global__ void __launch_bounds__(CPT == 4 ? 256 : 512) k_build(const BuildArgs g) {
  constexpr int XOFF = Layout<T>::xoff;
  __shared__ unsigned s_ticket;
  __shared__ int s_flag;
  __shared__ uint32_t s_row[2][2 * 32];
  __shared__ T s_carry[3 * 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  if (tid == 0) s_ticket = atomicAdd(g.ticket, 1u);
  __syncthreads();
  const unsigned ticket = s_ticket;
  const int bin = (int)(ticket % (unsigned)g.bins);
  const int band = (int)(ticket / (unsigned)g.bins);
  const int y0 = band * g.band_h;
  const int y1 = min(y0 + g.band_h, g.h);
  const int xb = tid * CPT;
  const bool last_band = band + 1 >= g.nbands;
  // Threads past the right edge keep the block scans uniform but touch no
  // memory; the last live thread may straddle the edge (padding = kNoBin).
  const bool live = xb < g.w;
  const uint16_t* fi = g.fi + (live ? xb : 0);

  // ---- phase 1: this band's column aggregates (only later bands need them)
  uint32_t ac[CPT], ay[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) ac[i] = ay[i] = 0;
  const size_t slot = ((size_t)band * g.bins + bin) * 2 * g.wa;
  if (!last_band) {
    if (live) {
      for (int y = y0; y < y1; ++y) {
        uint16_t v[CPT];
        load_bins<CPT>(fi + (size_t)y * g.fi_pitch, v);
#pragma unroll
        for (int i = 0; i < CPT; ++i)
          if (v[i] == bin) {
            ac[i] += 1;
            ay[i] += (uint32_t)y;
          }
      }
      store_run<uint32_t, CPT>(g.agg + slot + xb, ac);
      store_run<uint32_t, CPT>(g.agg + slot + g.wa + xb, ay);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(&g.flags[band * g.bins + bin], 1);
  }

  // ---- phase 2: decoupled look-back along bands of the same bin
  uint32_t cc[CPT], cy[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) cc[i] = cy[i] = 0;
  for (int k = band - 1; k >= 0; --k) {
    if (tid == 0) {
      int f;
      const int* fp = &g.flags[k * g.bins + bin];
      while ((f = ld_acquire(fp)) == 0) __nanosleep(64);
      s_flag = f;
    }
    __syncthreads();
    const int f = s_flag;
    const uint32_t* src = (f == 2 ? g.pref : g.agg) + ((size_t)k * g.bins + bin) * 2 * g.wa;
    if (live) {
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        cc[i] += __ldcg(src + xb + i);
        cy[i] += __ldcg(src + g.wa + xb + i);
      }
    }
    __syncthreads();  // s_flag is rewritten next iteration
    if (f == 2) break;
  }
  if (!last_band) {
    uint32_t pc[CPT], py[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      pc[i] = cc[i] + ac[i];
      py[i] = cy[i] + ay[i];
    }
    if (live) {
      store_run<uint32_t, CPT>(g.pref + slot + xb, pc);
      store_run<uint32_t, CPT>(g.pref + slot + g.wa + xb, py);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(&g.flags[band * g.bins + bin], 2);
  }

  // ---- carry row T(x+1, y0) = prefix over x of the column sums above y0
  T tp[CPT], tx[CPT], ty[CPT];
  {
    T lp[CPT], lx[CPT], lyv[CPT];
    T rp = 0, rx = 0, ry = 0;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      rp += (T)cc[i];
      rx += (T)cc[i] * (T)(xb + i);
      ry += (T)cy[i];
      lp[i] = rp;
      lx[i] = rx;
      lyv[i] = ry;
    }
    T tot[3] = {rp, rx, ry}, ex[3];
    block_exscan<3, T>(tot, ex, s_carry, lane, warp, nwarps);
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      tp[i] = ex[0] + lp[i];
      tx[i] = ex[1] + lx[i];
      ty[i] = ex[2] + lyv[i];
    }
  }

  T* out = reinterpret_cast<T*>(g.out);
  T* plane0 = out + (size_t)bin * P * g.plane_stride;
  if (band == 0) {  // zero row 0 of every plane of this bin
    const T z[CPT] = {};
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (live) store_run<T, CPT>(plane0 + (size_t)k * g.plane_stride + XOFF + 1 + xb, z);
      if (tid == 0) plane0[(size_t)k * g.plane_stride + XOFF] = 0;
    }
  }

  // ---- phase 3: rows of the band
  for (int y = y0; y < y1; ++y) {
    uint16_t v[CPT];
    if (live) {
      load_bins<CPT>(fi + (size_t)y * g.fi_pitch, v);
    } else {
#pragma unroll
      for (int i = 0; i < CPT; ++i) v[i] = kNoBin;
    }
    uint32_t lp[CPT], lx[CPT];
    uint32_t rp = 0, rx = 0;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      if (v[i] == bin) {
        rp += 1;
        rx += (uint32_t)(xb + i);
      }
      lp[i] = rp;
      lx[i] = rx;
    }
    uint32_t tot[2] = {rp, rx}, ex[2];
    block_exscan<2, uint32_t>(tot, ex, s_row[y & 1], lane, warp, nwarps);
    const size_t row = (size_t)(y + 1) * g.pitch + XOFF;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const uint32_t r = ex[0] + lp[i];
      tp[i] += (T)r;
      if constexpr (P == 3) {
        tx[i] += (T)(ex[1] + lx[i]);
        ty[i] += (T)y * (T)r;
      }
    }
    if (live) {
      store_run<T, CPT>(plane0 + row + 1 + xb, tp);
      if constexpr (P == 3) {
        store_run<T, CPT>(plane0 + g.plane_stride + row + 1 + xb, tx);
        store_run<T, CPT>(plane0 + 2 * g.plane_stride + row + 1 + xb, ty);
      }
    }
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < P; ++k) plane0[(size_t)k * g.plane_stride + row] = 0;
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
          const uint32_t r = (row[3 * x] * n) >> 8, g = (row[3 * x + 1] * n) >> 8,
                         b = (row[3 * x + 2] * n) >> 8;
          bin = (uint16_t)((r * n + g) * n + b);
          break;
        }
        default:
          bin = reinterpret_cast<const uint16_t*>(row)[x];
      }
    }
    dst[x] = bin;
  }
}

__global__ void k_narrow(const uint64_t* src, size_t pitch64, size_t ps64,
                         uint32_t* dst, size_t pitch32, size_t ps32, int w,
                         int h) {
  const int plane = blockIdx.z;
  const int y = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x <= w;
       x += gridDim.x * blockDim.x)
    dst[plane * ps32 + (size_t)y * pitch32 + x + Layout<uint32_t>::xoff] =
        (uint32_t)src[plane * ps64 + (size_t)y * pitch64 + x + Layout<uint64_t>::xoff];
}

}  // namespace

cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t s) {
  const int threads = 256;
  dim3 grid((unsigned)((a.fi_pitch + threads - 1) / threads), (unsigned)a.h);
  k_quantize<<<grid, threads, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_build(const BuildArgs& a, cudaStream_t s) {
  const int cpt = choose_cpt(a.w);
  const int threads = (int)round_up((size_t)((a.w + cpt - 1) / cpt), 32);
  const unsigned grid = (unsigned)(a.nbands * a.bins);
  if (a.planes == 3) {
    switch (cpt) {
      case 4: k_build<T, 3, 4><<<grid, threads, 0, s>>>(a); break;
      case 8: k_build<T, 3, 8><<<grid, threads, 0, s>>>(a); break;
      default: k_build<T, 3, 16><<<grid, threads, 0, s>>>(a);
    }
  } else {
    switch (cpt) {
      case 4: k_build<T, 1, 4><<<grid, threads, 0, s>>>(a); break;
      case 8: k_build<T, 1, 8><<<grid, threads, 0, s>>>(a); break;
      default: k_build<T, 1, 16><<<grid, threads, 0, s>>>(a);
    }
  }
  return cudaGetLastError();
}

template cudaError_t launch_build<uint32_t>(const BuildArgs&, cudaStream_t);
template cudaError_t launch_build<uint64_t>(const BuildArgs&, cudaStream_t);

cudaError_t launch_narrow(const uint64_t* src, size_t pitch64, size_t ps64,
                          uint32_t* dst, size_t pitch32, size_t ps32, int w,
                          int h, int nplanes, cudaStream_t s) {
  dim3 grid((unsigned)((w + 1 + 255) / 256), (unsigned)(h + 1), (unsigned)nplanes);
  k_narrow<<<grid, 256, 0, s>>>(src, pitch64, ps64, dst, pitch32, ps32, w, h);
  return cudaGetLastError();
}

}  // namespace swg
