// swg_abi.cu — host side of the C-ABI (include/swg.h): contexts, device
// memory, validation with the reference's error classes, plan set-up
// (exact host restatement of the reference kernel formulas the GPU needs as
// constants) and kernel launches.  No compute on the data path runs here:
// every table, histogram, score and peak is produced by the sm_100a kernels
// in k_build.cu / k_sweep.cu / k_brute.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "swg.h"
#include <cudaTypedefs.h>

#include "swg_internal.cuh"

using namespace swg;

namespace {

thread_local std::string g_err;
thread_local size_t g_required = 0;

swg_status fail(swg_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CUDA_TRY(expr)                                                        \
  do {                                                                        \
    cudaError_t e_ = (expr);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return fail(e_ == cudaErrorMemoryAllocation ? SWG_ERR_CAPACITY          \
                                                  : SWG_ERR_CUDA,             \
                  "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                  \
  } while (0)

#define ST_TRY(expr)                 \
  do {                               \
    swg_status s_ = (expr);          \
    if (s_ != SWG_OK) return s_;     \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  swg_status ensure(size_t bytes) {
    if (bytes <= n) return SWG_OK;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    bytes = round_up(bytes, 1 << 16);
    CUDA_TRY(cudaMalloc(&p, bytes));
    n = bytes;
    return SWG_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// ---- exact host restatement of kernel.cpp (plan constants only) --------
int k_hx(const swg_kernel& k) { return (k.kw - 1) / 2; }
int k_hy(const swg_kernel& k) { return (k.kh - 1) / 2; }
bool k_affine(const swg_kernel& k) {
  return k.kind == SWG_KERNEL_UNIFORM || k.kind == SWG_KERNEL_MANHATTAN;
}
bool k_integer(const swg_kernel& k) {
  return k.kind != SWG_KERNEL_GAUSS_CHEBYSHEV && k.kind != SWG_KERNEL_EXP_L1;
}

swg_status validate_kernel(const swg_kernel& k) {  // kernel.cpp:10-19
  if (k.kind < 0 || k.kind > 5) return fail(SWG_ERR_INVALID_KERNEL, "kernel: unknown kind");
  if (k.kw < 1 || k.kh < 1) return fail(SWG_ERR_INVALID_KERNEL, "kernel: dimensions must be >= 1");
  if (k.kw % 2 == 0 || k.kh % 2 == 0)
    return fail(SWG_ERR_INVALID_KERNEL, "kernel: dimensions must be odd, got %dx%d", k.kw, k.kh);
  if ((k.kind == SWG_KERNEL_GAUSS_CHEBYSHEV || k.kind == SWG_KERNEL_EXP_L1) && !(k.sigma > 0.0))
    return fail(SWG_ERR_INVALID_KERNEL, "kernel: sigma must be positive");
  if (k.kind == SWG_KERNEL_EXP_L1 && !(k.sigma < 1.0))
    return fail(SWG_ERR_INVALID_KERNEL, "kernel: exponential decay must be < 1");
  return SWG_OK;
}

double weight_at(const swg_kernel& k, int dx, int dy) {  // kernel.cpp:25-59
  const int hx = k_hx(k), hy = k_hy(k);
  switch (k.kind) {
    case SWG_KERNEL_UNIFORM:
      return 1.0;
    case SWG_KERNEL_MANHATTAN:
      return static_cast<double>((hx + hy + 1) - (std::abs(dx) + std::abs(dy)));
    case SWG_KERNEL_CHEBYSHEV: {
      const int hmax = std::max(hx, hy);
      const double sx = static_cast<double>(std::abs(dx)) * hmax / std::max(hx, 1);
      const double sy = static_cast<double>(std::abs(dy)) * hmax / std::max(hy, 1);
      const long level = std::lround(std::max(sx, sy));
      return static_cast<double>(hmax + 1 - level);
    }
    case SWG_KERNEL_EUCLID_QUAD: {  // declared extension
      const int64_t kx = int64_t(hx + 1) * (hx + 1), ky = int64_t(hy + 1) * (hy + 1);
      return static_cast<double>(2 * kx * ky - int64_t(dx) * dx * ky - int64_t(dy) * dy * kx);
    }
    case SWG_KERNEL_EXP_L1:  // declared extension: sigma = decay per pixel
      return std::pow(k.sigma, static_cast<double>(std::abs(dx) + std::abs(dy)));
    default: {
      const double nx = static_cast<double>(std::abs(dx)) / std::max(hx, 1);
      const double ny = static_cast<double>(std::abs(dy)) / std::max(hy, 1);
      const double r = std::max(nx, ny);
      return std::exp(-(r * r) / (2.0 * k.sigma * k.sigma));
    }
  }
}

// Exact strict-window mass of the quadratic (Euclidean) extension:
// sum of A - ky*dx^2 - kx*dy^2 over the window.
int64_t quad_mass(const swg_kernel& k) {
  const int64_t hx = k_hx(k), hy = k_hy(k);
  const int64_t kx = (hx + 1) * (hx + 1), ky = (hy + 1) * (hy + 1);
  const int64_t sdx = hx * (hx + 1) * (2 * hx + 1) / 3, sdy = hy * (hy + 1) * (2 * hy + 1) / 3;
  return 2 * kx * ky * k.kw * k.kh - ky * k.kh * sdx - kx * k.kw * sdy;
}

// Exact strict-window mass of an integer affine kernel (kernel.cpp:61-75).
int64_t affine_mass(const swg_kernel& k) {
  const int64_t hx = k_hx(k), hy = k_hy(k);
  const int64_t area = (int64_t)k.kw * k.kh;
  if (k.kind == SWG_KERNEL_UNIFORM) return area;
  return area * (hx + hy + 1) - k.kh * (hx * (hx + 1)) - k.kw * (hy * (hy + 1));
}

// WeddingCakePlan constructor (baselines.cpp:84-131), same arithmetic order.
swg_status cake_plan_compute(const swg_kernel& k, int m, int rule, CakeRings& out,
                             std::vector<double>* weights) {
  const int hx = k_hx(k), hy = k_hy(k);
  const int max_rings = std::min(hx, hy) + 1;
  if (m < 1 || m > max_rings)
    return fail(SWG_ERR_CONFIG, "wedding cake: ring count %d outside [1, %d] for %dx%d", m,
                max_rings, k.kw, k.kh);
  if (m > kMaxRings) return fail(SWG_ERR_CONFIG, "wedding cake: more than %d rings", kMaxRings);
  std::vector<int> sx(m), sy(m);
  std::vector<double> rw(m, 0.0);
  for (int i = 0; i < m; ++i) {
    sx[i] = static_cast<int>((int64_t(i) * hx + m - 1) / m);
    sy[i] = static_cast<int>((int64_t(i) * hy + m - 1) / m);
  }
  if (rule == SWG_RING_LEVEL) {
    for (int i = 0; i < m; ++i) rw[i] = weight_at(k, hx - sx[i], 0);
  } else {
    std::vector<double> sum(m, 0.0);
    std::vector<int64_t> cnt(m, 0);
    for (int dy = -hy; dy <= hy; ++dy)
      for (int dx = -hx; dx <= hx; ++dx) {
        int ring = 0;
        for (int i = m - 1; i > 0; --i)
          if (std::abs(dx) <= hx - sx[i] && std::abs(dy) <= hy - sy[i]) {
            ring = i;
            break;
          }
        sum[ring] += weight_at(k, dx, dy);
        cnt[ring] += 1;
      }
    for (int i = 0; i < m; ++i) rw[i] = sum[i] / cnt[i];
  }
  for (int i = 0; i < m; ++i) {
    out.a[i] = hx - sx[i];
    out.c[i] = hy - sy[i];
    out.coeff[i] = rw[i] - (i > 0 ? rw[i - 1] : 0.0);  // baselines.cpp:141
  }
  if (weights) *weights = rw;
  return SWG_OK;
}

// Ring plans are pure functions of (kernel, rings, rule) and the MEAN rule
// visits every window cell (~1e4 weight evaluations at 97x97): memoised so a
// per-frame likelihood_maps call does no O(kw*kh) host work.
swg_status cake_plan(const swg_kernel& k, int m, int rule, CakeRings& out,
                     std::vector<double>* weights = nullptr) {
  struct Entry {
    swg_kernel k;
    int m, rule;
    CakeRings plan;
    std::vector<double> w;
  };
  static std::mutex mu;
  static std::vector<Entry*> cache;  // small; lives for the process
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry* e : cache)
      if (e->k.kind == k.kind && e->k.kw == k.kw && e->k.kh == k.kh && e->k.sigma == k.sigma &&
          e->m == m && e->rule == rule) {
        out = e->plan;
        if (weights) *weights = e->w;
        return SWG_OK;
      }
  }
  auto* e = new Entry{k, m, rule, {}, {}};
  const swg_status st = cake_plan_compute(k, m, rule, e->plan, &e->w);
  if (st != SWG_OK) {
    delete e;
    return st;
  }
  out = e->plan;
  if (weights) *weights = e->w;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 256) {
    delete cache.front();
    cache.erase(cache.begin());
  }
  cache.push_back(e);
  return SWG_OK;
}

}  // namespace

struct swg_ctx {
  std::atomic<int> refs{1};  // 1 for the handle + 1 per live table
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  // device -> host copies of finished maps overlap the next scale's sweep
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> events;
  // the requests of one likelihood_maps call fan out over worker streams
  // (their sweeps overlap: no partial last wave per scale)
#ifndef SWG_WORKERS
#define SWG_WORKERS 8  // measured: config 3 6.48 -> 6.27 ms (3 -> 8), 12: -0.8 % more
#endif
  static constexpr int kWorkers = SWG_WORKERS;
  cudaStream_t work[kWorkers] = {};
  cudaEvent_t fork = nullptr, join[kWorkers] = {};
  // host-map fan-out: a few requests on streams of decreasing priority, so
  // they finish in request order and each map's copy overlaps the later
  // requests' sweeps (the device-output fan-out keeps equal priorities:
  // measured 16 % slower on config 5 with priorities)
  static constexpr int kHostFan = 3;
  cudaStream_t hwork[kHostFan] = {};
  cudaEvent_t hjoin[kHostFan] = {};
  // map scratch (CTA candidates, unrequested maps, peaks, exact-peak
  // candidates): one set per worker so a frame batch can run its frames'
  // calls concurrently (swg_likelihood_batch sets `slot` and `fanout_off`)
  struct Scratch {
    DevBuf parts, scores, peaks, resc;
  } scr[kWorkers];
  int slot = 0;
  bool fanout_off = false;
  std::mutex mu;
  std::atomic<uint64_t> launches{0};
  std::atomic<uint64_t> map_copies{0};  // device->host map copies issued (zero-copy check)
  // swg_likelihood_maps_async: scratch slots rotate over the calls; a slot
  // is reused only after the copies (or sweeps) of its last call (free[k])
  int aslot = 0;
  cudaEvent_t free_ev[kWorkers] = {};
  DevBuf terms, qout, grid, io, bpeaks;
  // exact kernel-weight grids, uploaded once per kernel (graph-capture safe)
  struct Grid {
    swg_kernel k;
    bool integer;
    DevBuf buf;
  };
  std::vector<Grid*> grids;
};

struct swg_tables {
  swg_ctx* ctx = nullptr;
  int w = 0, h = 0, bins = 0, planes = 0, format = 0, levels = 0;
  int bin0 = 0, total_bins = 0;  // planes hold bins [bin0, bin0 + bins) of total_bins
  int carry_y0 = 0;     // 32-bit planes hold GLOBAL rows y0.. (swg_tables_add_carry)
  bool carried = false;
  bool has_fi = false;
  uint16_t* fi = nullptr;
  size_t fip = 0;
  uint8_t* in = nullptr;  // staging for host input
  size_t in_pitch = 0, in_row = 0;
  int groups = 0;          // bin octets
  size_t pitch = 0, ps = 0;  // records (shared by the 32- and 64-bit planes)
  uint16_t* t16 = nullptr;  // narrow plain planes (P = 1 tables): exact box
                            // counts for boxes of area < 2^16
  uint32_t* t32 = nullptr;  // primary for P = 3; on demand for P = 1
  uint16_t* t16a = nullptr; // narrow {1, x, y} planes (3-plane layout) of P >= 3
                            // tables, built on demand for windows of mass < 2^16
  uint64_t* t64 = nullptr;
  double* tdec = nullptr;    // decayed directional tables (EXP_L1), 4 planes
  double decay = 0.0;
  uint16_t* fflip = nullptr; // h / v / hv flipped feature images (decay tables)
  uint32_t* lb = nullptr;  // band carry scratch (BuildArgs::agg)
  // same-geometry table sets for concurrent frames (swg_likelihood_batch)
  swg_tables* clone[SWG_WORKERS - 1] = {};
  int band_h = 0, nbands = 0;  // the current split of the rows into bands
  int nb_default = 0;          // bands of the default split (the carry array's size)
  size_t wa = 0;
  size_t bytes = 0;
  // Selective (model-driven) builds, swg_tables_rebuild_for: units of the
  // primary set -- bin octets of the 32-bit planes (+ the narrow ramp
  // planes), or bin pairs of the decay planes -- not yet built for the
  // current frame.  Empty: every unit is current.  Any consumer builds the
  // units it reads first (ensure_fresh).
  std::vector<unsigned char> stale;
  size_t built_bytes = 0;  // plane bytes written since the last rebuild began
  // TMA row tensor maps of the 32-bit / 16-bit plain planes (BuildArgs::tmap),
  // encoded on first build: 0 not yet, 1 ok, -1 unavailable
  CUtensorMap tm[2];
  int tm_state[2] = {0, 0};
  int aslot = -1;  // scratch slot of swg_likelihood_maps_async (-1: not yet)
  size_t lb_bytes = 0;
};

#ifndef SWG_L2_BUDGET_MB
#define SWG_L2_BUDGET_MB 64  // share of the 126 MB L2 a sweep's corner rows may use
#endif

// TMA row tensor maps (BuildArgs::tmap): cuTensorMapEncodeTiled through the
// runtime's driver entry point (no libcuda link).  Rank 4, uint32 elements:
// {32 words = one 128-byte line, lines of a row (records 1..W), rows 0..H,
// planes}, box {32, box_lines, 1, 1}, SWIZZLE_128B.
bool swg::encode_row_tmap(CUtensorMap* m, void* record1, int rec_bytes, int w, int h, size_t pitch,
                     size_t plane_stride, int nplanes, int box_lines) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  if (!fn || std::getenv("SWG_NO_TMA")) return false;
  if (reinterpret_cast<uintptr_t>(record1) % 16 || (pitch * rec_bytes) % 16 ||
      (plane_stride * rec_bytes) % 16 || box_lines < 1 || box_lines > 256)
    return false;
  const cuuint64_t dims[4] = {32, (cuuint64_t)(((size_t)w * rec_bytes + 127) / 128),
                              (cuuint64_t)h + 1, (cuuint64_t)nplanes};
  const cuuint64_t strides[3] = {128, (cuuint64_t)(pitch * rec_bytes),
                                 (cuuint64_t)(plane_stride * rec_bytes)};
  const cuuint32_t box[4] = {32, (cuuint32_t)box_lines, 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, record1, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

size_t pixel_bytes(int format) {
  switch (format) {
    case SWG_FMT_GRAY8: return 1;
    case SWG_FMT_RGB8: return 3;
    default: return 2;
  }
}

// Planes of 16-byte records (16-bit octets, fp64 bin pairs) start 16 bytes
// into their allocation.  Record 0 of a row is the zero column and the
// builds write records 1..W in long runs: with the plane at an allocation
// boundary every run started 16 bytes into a 32-byte sector, and a pure
// store kernel with that pattern tops out at 4.0 TB/s against 5.5 TB/s for
// sector-aligned runs (profiles/store_bw.cu; the same for per-lane, TMA
// tensor and bulk stores).  Pitch and plane stride are even record counts,
// so the shift aligns every row of every plane.  (32-byte records are
// sector-aligned as they are.)
constexpr size_t kRec16Shift = 16;
cudaError_t alloc_rec16(void** p, size_t bytes) {
  void* raw = nullptr;
  const cudaError_t e = cudaMalloc(&raw, bytes + kRec16Shift);
  *p = e == cudaSuccess ? static_cast<char*>(raw) + kRec16Shift : nullptr;
  return e;
}
void free_rec16(void* p) {
  if (p) cudaFree(static_cast<char*>(p) - kRec16Shift);
}

#ifndef SWG_BAND_TARGET
#define SWG_BAND_TARGET (148 * 2)  // ~2 row-wide CTAs per SM and table kind
#endif
// Split the rows into bands: ~`target` (band, octet) CTAs per table kind.
// Never more bands than the carry array was sized for (the default split).
void split_bands(swg_tables* t, int target) {
  int nb = (target + t->groups - 1) / t->groups;
  nb = std::max(1, std::min(nb, (t->h + 7) / 8));
  if (t->nb_default) nb = std::min(nb, t->nb_default);
  t->band_h = (t->h + nb - 1) / nb;
  t->nbands = (t->h + t->band_h - 1) / t->band_h;
}
void choose_bands(swg_tables* t) {
  t->nb_default = 0;
  split_bands(t, SWG_BAND_TARGET);
  t->nb_default = t->nbands;
  t->wa = round_up((size_t)t->w, 16);
}

template <typename T>
swg_status run_build(swg_tables* t, T* out, const std::vector<int>* sel = nullptr) {
  swg_ctx* c = t->ctx;
  static thread_local BuildArgs a;
  a = BuildArgs{};
  if (sel) {
    a.nsel = (int)sel->size();
    for (int i = 0; i < a.nsel; ++i) {
      a.sel[i] = (unsigned short)(*sel)[i];
      a.selmask[(*sel)[i] >> 5] |= 1u << ((*sel)[i] & 31);
    }
    if (a.nsel == 0) return SWG_OK;
  }
  a.fi = t->fi;
  a.fi_pitch = t->fip;
  a.out = out;
  a.pitch = t->pitch;
  a.plane_stride = t->ps;
  a.w = t->w;
  a.h = t->h;
  a.bins = t->bins;
  a.groups = t->groups;
  a.planes = t->planes;
  a.band_h = t->band_h;
  a.nbands = t->nbands;
  a.wa = t->wa;
  a.aw = t->planes == SWG_PLANES_QUADRATIC ? 24 : t->planes == SWG_PLANES_PLAIN ? 8 : 16;
  a.agg = t->lb;
  a.bin0 = t->bin0;
  // the 32-bit build writes the narrow ramp planes too (their low 16 bits)
  if (sizeof(T) == 4 && static_cast<void*>(out) == static_cast<void*>(t->t32)) a.out16 = t->t16a;
  // TMA stores of the staged rows (16- and 32-bit planes)
  const int ti = static_cast<void*>(out) == static_cast<void*>(t->t32) ? 0
                 : static_cast<void*>(out) == static_cast<void*>(t->t16) ? 1 : -1;
  if (ti >= 0 && sizeof(T) <= 4) {
    if (t->tm_state[ti] == 0) {
      const int rec = kOct * (int)sizeof(T);
      const int box_lines = 32 * choose_cpt(t->w) * rec / 128;
      t->tm_state[ti] = encode_row_tmap(&t->tm[ti], reinterpret_cast<char*>(out) + rec, rec, t->w,
                                        t->h, t->pitch, t->ps, t->groups * t->planes, box_lines)
                            ? 1 : -1;
    }
    if (t->tm_state[ti] == 1) {
      a.tmap = t->tm[ti];
      a.tmap_ok = 1;
    }
  }
  if (t->nbands > 1) {
    CUDA_TRY(launch_colsum(a, c->stream));
    c->launches += 2;
  }
  int nl = 0;
  CUDA_TRY(launch_build<T>(a, c->stream, &nl));
  c->launches += (uint64_t)nl;
  const size_t units = a.nsel ? (size_t)a.nsel : (size_t)t->groups;
  const int kinds = sizeof(T) == 2 ? 1 : t->planes;
  t->built_bytes += units * kOct * t->ps * kinds * sizeof(T) + (a.out16 ? units * kOct * t->ps * 3 * 2 : 0);
  return SWG_OK;
}

swg_status upload_and_quantize(swg_tables* t, const void* pixels, int is_device,
                               size_t pitch_bytes) {
  swg_ctx* c = t->ctx;
  const size_t row = (size_t)t->w * pixel_bytes(t->format);
  if (!pitch_bytes) pitch_bytes = row;
  if (pitch_bytes < row) return fail(SWG_ERR_ARG, "pitch %zu smaller than a row (%zu)", pitch_bytes, row);
  const uint8_t* src = static_cast<const uint8_t*>(pixels);
  size_t src_pitch = pitch_bytes;
  if (!is_device) {
    if (!t->in) {
      t->in_row = row;
      CUDA_TRY(cudaMallocPitch(reinterpret_cast<void**>(&t->in), &t->in_pitch, row, t->h));
      t->bytes += t->in_pitch * t->h;
    }
    CUDA_TRY(cudaMemcpy2DAsync(t->in, t->in_pitch, pixels, pitch_bytes, row, t->h,
                               cudaMemcpyHostToDevice, c->stream));
    src = t->in;
    src_pitch = t->in_pitch;
  }
  QuantArgs q{src, src_pitch, t->w, t->h, t->format,
              t->format == SWG_FMT_RGB8 ? t->levels : t->total_bins, t->fi, t->fip};
  CUDA_TRY(launch_quantize(q, c->stream));
  c->launches += 1;
  t->has_fi = true;
  return SWG_OK;
}

swg_status ensure_t32(swg_tables* t) {
  if (t->t32) return SWG_OK;
  if (t->tdec) return fail(SWG_ERR_CONFIG, "decay tables hold no integral planes");
  if (!t->has_fi) return fail(SWG_ERR, "tables: no 32-bit planes and no feature image");
  const size_t bytes = t->ps * t->planes * t->groups * kOct * 4;
  cudaError_t e = cudaMalloc(&t->t32, bytes);
  if (e != cudaSuccess) {
    t->t32 = nullptr;
    cudaGetLastError();
    g_required = bytes;
    return fail(SWG_ERR_CAPACITY, "tables: 32-bit planes need %zu bytes: %s", bytes,
                cudaGetErrorString(e));
  }
  t->bytes += bytes;
  return run_build<uint32_t>(t, t->t32);
}

// The narrow {1, x, y} planes reuse the column sums the 32-bit build left in
// t->lb when `fresh` is false (a rebuild runs them right after the 32-bit planes).
swg_status build_t16a(swg_tables* t, bool fresh) {
  swg_ctx* c = t->ctx;
  BuildArgs a{};
  a.fi = t->fi;
  a.fi_pitch = t->fip;
  a.out = t->t16a;
  a.pitch = t->pitch;
  a.plane_stride = t->ps;
  a.w = t->w;
  a.h = t->h;
  a.bins = t->bins;
  a.groups = t->groups;
  a.planes = 3;  // the narrow set's own layout
  a.kinds = 3;
  a.band_h = t->band_h;
  a.nbands = t->nbands;
  a.wa = t->wa;
  a.aw = t->planes == SWG_PLANES_QUADRATIC ? 24 : 16;  // the carry layout of the column sums
  a.agg = t->lb;
  a.bin0 = t->bin0;
  if (fresh && t->nbands > 1) {
    BuildArgs ca = a;
    ca.planes = t->planes;
    CUDA_TRY(launch_colsum(ca, c->stream));
    c->launches += 2;
  }
  int nl = 0;
  CUDA_TRY(launch_build<uint16_t>(a, c->stream, &nl));
  c->launches += (uint64_t)nl;
  return SWG_OK;
}

swg_status ensure_t16a(swg_tables* t) {
  if (t->t16a) return SWG_OK;
  if (t->planes < 3 || t->tdec || !t->has_fi)
    return fail(SWG_ERR, "tables: no narrow ramp planes");
  const size_t bytes = t->ps * 3 * t->groups * kOct * 2;
  cudaError_t e = alloc_rec16(reinterpret_cast<void**>(&t->t16a), bytes);
  if (e != cudaSuccess) {
    t->t16a = nullptr;
    cudaGetLastError();
    g_required = bytes;
    return fail(SWG_ERR_CAPACITY, "tables: 16-bit ramp planes need %zu bytes: %s", bytes,
                cudaGetErrorString(e));
  }
  t->bytes += bytes;
  return build_t16a(t, true);
}

swg_status ensure_t64(swg_tables* t) {
  if (t->t64) return SWG_OK;
  if (t->tdec) return fail(SWG_ERR_CONFIG, "decay tables hold no integral planes");
  if (t->planes == SWG_PLANES_QUADRATIC && t->h > 2340)  // 32-bit column y^2 carries
    return fail(SWG_ERR_SIZE, "exact 64-bit quadratic planes: height %d > 2340", t->h);
  if (!t->has_fi) return fail(SWG_ERR, "tables: no 64-bit planes and no feature image");
  const size_t bytes = t->ps * t->planes * t->groups * kOct * 8;
  cudaError_t e = cudaMalloc(&t->t64, bytes);
  if (e != cudaSuccess) {
    t->t64 = nullptr;
    g_required = bytes;
    return fail(SWG_ERR_CAPACITY, "tables: 64-bit export planes need %zu bytes: %s", bytes,
                cudaGetErrorString(e));
  }
  t->bytes += bytes;
  return run_build<uint64_t>(t, t->t64);
}

// Device copy of a kernel's exact weight grid (weight_at, llround-ed for
// integer kernels as BruteForcePlan does, baselines.cpp:18-20); cached per
// kernel so repeated requests (and graph capture) issue no host copies.
swg_status weight_grid(swg_ctx* c, const swg_kernel& k, const double** out) {
  const bool integer = k_integer(k);
  for (auto* g : c->grids)
    if (g->k.kind == k.kind && g->k.kw == k.kw && g->k.kh == k.kh && g->k.sigma == k.sigma &&
        g->integer == integer) {
      *out = static_cast<const double*>(g->buf.p);
      return SWG_OK;
    }
  const int hx = k_hx(k), hy = k_hy(k);
  std::vector<double> w((size_t)k.kw * k.kh);
  for (int dy = -hy; dy <= hy; ++dy)
    for (int dx = -hx; dx <= hx; ++dx) {
      double v = weight_at(k, dx, dy);
      if (integer) v = (double)std::llround(v);
      w[(size_t)(dy + hy) * k.kw + dx + hx] = v;
    }
  auto* g = new swg_ctx::Grid{k, integer, {}};
  swg_status st = g->buf.ensure(w.size() * 8);
  if (st == SWG_OK) {
    // ordered on the context stream and completed before any worker stream
    // (forked later) can read it; once per kernel
    cudaError_t e = cudaMemcpyAsync(g->buf.p, w.data(), w.size() * 8, cudaMemcpyHostToDevice,
                                    c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) st = fail(SWG_ERR_CUDA, "weight grid: %s", cudaGetErrorString(e));
  }
  if (st != SWG_OK) {
    g->buf.release();
    delete g;
    return st;
  }
  c->grids.push_back(g);
  *out = static_cast<const double*>(g->buf.p);
  return SWG_OK;
}

swg_status run_build_decay(swg_tables* t, const std::vector<int>* sel = nullptr) {
  swg_ctx* c = t->ctx;
  if (sel && sel->empty()) return SWG_OK;
  const size_t fsz = t->fip * t->h;
  CUDA_TRY(launch_flip(t->fi, t->fip, t->w, t->h, t->fflip, t->fflip + fsz, t->fflip + 2 * fsz,
                       c->stream));
  c->launches += 1;
  static thread_local BuildArgs a;
  a = BuildArgs{};
  if (sel) {
    a.nsel = (int)sel->size();
    for (int i = 0; i < a.nsel; ++i) {
      a.sel[i] = (unsigned short)(*sel)[i];
      a.selmask[(*sel)[i] >> 5] |= 1u << ((*sel)[i] & 31);
    }
  }
  a.fi_pitch = t->fip;
  a.out = t->tdec;
  a.pitch = t->pitch;
  a.plane_stride = t->ps;
  a.w = t->w;
  a.h = t->h;
  a.bins = t->bins;
  a.groups = t->groups;
  a.planes = 4;
  a.band_h = t->band_h;
  a.nbands = t->nbands;
  a.wa = t->wa;
  a.aw = 16;
  a.agg = t->lb;
  a.bin0 = t->bin0;
  // TMA stores of the strip tiles' rows (16-byte pair records, 256 per row segment)
  if (t->tm_state[0] == 0)
    t->tm_state[0] = encode_row_tmap(&t->tm[0], reinterpret_cast<char*>(t->tdec) + 16, 16, t->w,
                                     t->h, t->pitch, t->ps, t->groups * (kOct / kDP) * 4, 32)
                         ? 1 : -1;
  if (t->tm_state[0] == 1) {
    a.tmap = t->tm[0];
    a.tmap_ok = 1;
  }
  const uint16_t* src[4] = {t->fi, t->fflip, t->fflip + fsz, t->fflip + 2 * fsz};
  // the four orientations' units go in ONE launch (the carries of the
  // unflipped and the v-flipped image in one pass before it): a warp builds
  // a unit, so one orientation alone leaves the SMs short of warps (config 4:
  // 1184 units per orientation, 8 warps per SM; builds 33.7 -> 26.8 ms with
  // the orientations together, config 5's full decayed build 2.09 -> 1.70 ms)
  const char* ef = std::getenv("SWG_DECAY_FUSE");  // A/B: 0 = a launch per orientation
  const bool fuse = ef ? std::atoi(ef) != 0 : t->nbands > 1;
  const size_t stride = t->lb_bytes / 4 / 4;  // uint32 words per orientation
  for (int k = 0; k < 4; ++k) a.fio[k] = src[k];
  if (fuse) {  // the four orientations' carries in one pass, then their strips
    a.agg = t->lb;
    a.agg_stride = stride;
    int nl = 0;
    CUDA_TRY(launch_build_decay(a, t->decay, -1, c->stream, &nl));
    c->launches += (uint64_t)nl;
    CUDA_TRY(launch_build_decay(a, t->decay, -2, c->stream, &nl));
    c->launches += (uint64_t)nl;
  } else {
    for (int k = 0; k < 4; ++k) {
      a.fi = src[k];
      int nl = 0;
      CUDA_TRY(launch_build_decay(a, t->decay, k, c->stream, &nl));
      c->launches += (uint64_t)nl;
    }
  }
  const size_t units = a.nsel ? (size_t)a.nsel : (size_t)t->groups * (kOct / kDP);
  t->built_bytes += units * kDP * t->ps * 4 * 8;
  return SWG_OK;
}

// ---- selective builds
bool selective(const swg_tables* t) {
  return t->bins == t->total_bins && t->has_fi &&
         (t->tdec || (t->t32 && t->planes >= SWG_PLANES_AFFINE));
}
int sel_units(const swg_tables* t) { return t->tdec ? t->groups * (kOct / kDP) : t->groups; }

// Build the stale units `need` marks (null: every stale unit).
swg_status ensure_fresh(swg_tables* t, const std::vector<unsigned char>* need) {
  if (t->stale.empty()) return SWG_OK;
  std::vector<int> sel;
  for (int u = 0; u < (int)t->stale.size(); ++u)
    if (t->stale[u] && (!need || (*need)[u])) sel.push_back(u);
  if (sel.empty()) return SWG_OK;
  if (t->tdec) ST_TRY(run_build_decay(t, &sel));
  else ST_TRY(run_build<uint32_t>(t, t->t32, &sel));
  for (int u : sel) t->stale[u] = 0;
  bool any = false;
  for (unsigned char v : t->stale) any |= v != 0;
  if (!any) t->stale.clear();
  return SWG_OK;
}
swg_status fresh_all(swg_tables* t) { return ensure_fresh(t, nullptr); }

// A cake whose outer box holds >= 2^16 pixels still runs on 16-bit planes
// when ring 1's box and ring 0's frame hold fewer (k_sweep_cake16 wide0).
bool cake16_wide0(const swg_kernel& k, const swg_map_request& r) {
  static thread_local CakeRings pl;
  if (r.rings < 2 || cake_plan(k, r.rings, r.ring_rule, pl) != SWG_OK) return false;
  const long long a0 = (2LL * pl.a[0] + 1) * (2LL * pl.c[0] + 1);
  const long long a1 = (2LL * pl.a[1] + 1) * (2LL * pl.c[1] + 1);
  return a1 < 65536 && a0 - a1 < 65536;
}

swg_status check_tables(const swg_tables* t) {
  if (!t || !t->ctx) return fail(SWG_ERR_ARG, "NULL tables");
  return SWG_OK;
}

}  // namespace

extern "C" {

int swg_abi_version(void) { return SWG_ABI_VERSION; }
const char* swg_last_error(void) { return g_err.c_str(); }
size_t swg_last_required_bytes(void) { return g_required; }

swg_status swg_device_count(int* n) {
  if (!n) return fail(SWG_ERR_ARG, "NULL");
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    *n = 0;
    return fail(SWG_ERR_NO_DEVICE, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  return SWG_OK;
}

static void ctx_release(swg_ctx* c);

swg_status swg_ctx_create(int device, swg_ctx** out) {
  if (!out) return fail(SWG_ERR_ARG, "NULL out");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(SWG_ERR_NO_DEVICE, "no CUDA device: %s", cudaGetErrorString(e));
  if (device < 0 || device >= n) return fail(SWG_ERR_NO_DEVICE, "device %d of %d", device, n);
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(SWG_ERR_NO_DEVICE, "device %d is sm_%d%d; libswg is built for sm_100a only",
                device, prop.major, prop.minor);
  DeviceGuard g(device);
  swg_ctx* c = new swg_ctx;
  c->device = device;
  e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(SWG_ERR_CUDA, "stream: %s", cudaGetErrorString(e));
  }
  c->stream = c->own;
  if ((e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking)) != cudaSuccess) {
    cudaStreamDestroy(c->own);
    delete c;
    return fail(SWG_ERR_CUDA, "stream: %s", cudaGetErrorString(e));
  }
  e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  for (int w = 0; w < swg_ctx::kHostFan && e == cudaSuccess; ++w) {
    e = cudaStreamCreateWithPriority(&c->hwork[w], cudaStreamNonBlocking,
                                     std::min(prio_hi + w, prio_lo));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->hjoin[w], cudaEventDisableTiming);
  }
  for (int w = 0; w < swg_ctx::kWorkers && e == cudaSuccess; ++w) {
    e = cudaStreamCreateWithFlags(&c->work[w], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join[w], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    c->refs = 1;
    ctx_release(c);
    return fail(SWG_ERR_CUDA, "worker streams: %s", cudaGetErrorString(e));
  }
  *out = c;
  return SWG_OK;
}

static void ctx_release(swg_ctx* c) {
  if (c->refs.fetch_sub(1) != 1) return;
  {
    DeviceGuard g(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& x : c->scr) {
      x.parts.release();
      x.scores.release();
      x.peaks.release();
      x.resc.release();
    }
    c->terms.release();
    c->qout.release();
    c->grid.release();
    c->io.release();
    c->bpeaks.release();
    for (auto* g : c->grids) {
      g->buf.release();
      delete g;
    }
    cudaStreamSynchronize(c->copy);
    for (cudaEvent_t e : c->events) cudaEventDestroy(e);
    for (cudaEvent_t e : c->free_ev)
      if (e) cudaEventDestroy(e);
    for (int w = 0; w < swg_ctx::kWorkers; ++w) {
      if (c->work[w]) {
        cudaStreamSynchronize(c->work[w]);
        cudaStreamDestroy(c->work[w]);
      }
      if (c->join[w]) cudaEventDestroy(c->join[w]);
    }
    for (int w = 0; w < swg_ctx::kHostFan; ++w) {
      if (c->hwork[w]) {
        cudaStreamSynchronize(c->hwork[w]);
        cudaStreamDestroy(c->hwork[w]);
      }
      if (c->hjoin[w]) cudaEventDestroy(c->hjoin[w]);
    }
    if (c->fork) cudaEventDestroy(c->fork);
    cudaStreamDestroy(c->copy);
    cudaStreamDestroy(c->own);
  }
  delete c;
}

swg_status swg_ctx_destroy(swg_ctx* c) {
  if (!c) return SWG_OK;
  ctx_release(c);
  return SWG_OK;
}

swg_status swg_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(SWG_ERR_ARG, "NULL out");
  // portable + mapped: every device may write it directly (zero-copy maps)
  CUDA_TRY(cudaHostAlloc(out, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  return SWG_OK;
}

swg_status swg_host_free(void* p) {
  if (p) CUDA_TRY(cudaFreeHost(p));
  return SWG_OK;
}

swg_status swg_device_alloc(size_t bytes, void** out) {
  if (!out) return fail(SWG_ERR_ARG, "NULL out");
  cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
  if (e != cudaSuccess) {
    cudaGetLastError();
    g_required = bytes;
    return fail(SWG_ERR_CAPACITY, "device allocation of %zu bytes: %s", bytes,
                cudaGetErrorString(e));
  }
  return SWG_OK;
}

swg_status swg_device_free(void* p) {
  if (p) CUDA_TRY(cudaFree(p));
  return SWG_OK;
}

swg_status swg_ipc_export(const void* dev_ptr, unsigned char* handle) {
  if (!dev_ptr || !handle) return fail(SWG_ERR_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  static_assert(sizeof(h) == SWG_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  return SWG_OK;
}

swg_status swg_ipc_import(const unsigned char* handle, void** dev_ptr) {
  if (!dev_ptr || !handle) return fail(SWG_ERR_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SWG_OK;
}

swg_status swg_ipc_close(void* dev_ptr) {
  if (dev_ptr) CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return SWG_OK;
}

swg_status swg_ctx_synchronize(swg_ctx* c) {
  if (!c) return fail(SWG_ERR_ARG, "NULL ctx");
  DeviceGuard g(c->device);
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->copy));  // host maps of swg_likelihood_maps_async
  return SWG_OK;
}

swg_status swg_ctx_set_stream(swg_ctx* c, void* s) {
  if (!c) return fail(SWG_ERR_ARG, "NULL ctx");
  std::lock_guard<std::mutex> lk(c->mu);
  c->stream = s ? static_cast<cudaStream_t>(s) : c->own;
  return SWG_OK;
}

swg_status swg_ctx_map_copy_count(swg_ctx* c, uint64_t* n) {
  if (!c || !n) return fail(SWG_ERR_ARG, "NULL");
  *n = c->map_copies.load();
  return SWG_OK;
}

swg_status swg_ctx_launch_count(swg_ctx* c, uint64_t* n) {
  if (!c || !n) return fail(SWG_ERR_ARG, "NULL");
  *n = c->launches.load();
  return SWG_OK;
}

static swg_status build_common(swg_ctx* c, const void* pixels, int is_device,
                               size_t pitch_bytes, int width, int height, int format,
                               int bins, int planes, double decay, int bin_begin, int bin_end,
                               size_t memory_budget, swg_tables** out) {
  if (!c || !pixels || !out) return fail(SWG_ERR_ARG, "NULL argument");
  *out = nullptr;
  if (width < 1 || height < 1) return fail(SWG_ERR, "image dimensions must be >= 1");
  if (format < SWG_FMT_GRAY8 || format > SWG_FMT_BINS16) return fail(SWG_ERR_ARG, "format %d", format);
  if (planes != SWG_PLANES_PLAIN && planes != SWG_PLANES_AFFINE &&
      planes != SWG_PLANES_QUADRATIC && planes != SWG_PLANES_DECAY)
    return fail(SWG_ERR_ARG, "planes %d", planes);
  if (planes == SWG_PLANES_DECAY && !(decay > 0.0 && decay < 1.0))
    return fail(SWG_ERR_INVALID_KERNEL, "decay must be in (0, 1)");
  int nb = bins;
  if (format == SWG_FMT_RGB8) {
    if (bins < 1 || bins > 40) return fail(SWG_ERR, "RGB levels must be in [1, 40]");
    nb = bins * bins * bins;
  }
  if (nb < 1) return fail(SWG_ERR, "bin count must be >= 1");
  if (nb > 65535) return fail(SWG_ERR, "bin count must be <= 65535");
  if (width > kMaxWidth) return fail(SWG_ERR_SIZE, "width %d > %d", width, kMaxWidth);
  if (bin_begin == 0 && bin_end == 0) bin_end = nb;
  if (bin_begin < 0 || bin_end > nb || bin_begin >= bin_end)
    return fail(SWG_ERR_OUT_OF_RANGE, "bin range [%d, %d) of %d", bin_begin, bin_end, nb);

  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  swg_tables* t = new swg_tables;
  t->ctx = c;
  c->refs++;
  t->w = width;
  t->h = height;
  t->total_bins = nb;
  t->bin0 = bin_begin;
  t->bins = bin_end - bin_begin;
  t->levels = bins;
  t->planes = planes;
  t->format = format;
  t->decay = planes == SWG_PLANES_DECAY ? decay : 0.0;
  t->fip = fi_pitch(width);
  t->groups = (t->bins + kOct - 1) / kOct;
  t->pitch = record_pitch(width);
  t->ps = t->pitch * (size_t)(height + 1);
  choose_bands(t);
  // plain-only tables keep narrow uint16 planes (32-bit ones are built on
  // demand); affine and quadratic tables uint32 planes; decay fp64
  const size_t elem = planes == SWG_PLANES_PLAIN ? 2 : planes == SWG_PLANES_DECAY ? 8 : 4;
  const size_t tab_bytes = t->ps * planes * (size_t)t->groups * kOct * elem;
  // (decayed tables: one carry array per orientation)
  const size_t lb_bytes = (size_t)t->nbands * t->groups * t->wa * kOct *
                          (planes == SWG_PLANES_QUADRATIC ? 12 : 8) *
                          (planes == SWG_PLANES_DECAY ? 4 : 1);
  t->lb_bytes = lb_bytes;
  const size_t fb = t->fip * height * 2;
  const size_t need = tab_bytes + lb_bytes + fb * (planes == SWG_PLANES_DECAY ? 4 : 1);
  if (memory_budget && need > memory_budget) {
    swg_tables_destroy(t);
    g_required = need;
    return fail(SWG_ERR_CAPACITY, "%s tables need %zu bytes, budget is %zu",
                planes == SWG_PLANES_DECAY ? "decay" : "integral", need, memory_budget);
  }
  cudaError_t e;
  void** tab = elem == 2   ? reinterpret_cast<void**>(&t->t16)
               : elem == 4 ? reinterpret_cast<void**>(&t->t32)
                           : reinterpret_cast<void**>(&t->tdec);
  if ((e = elem == 4 ? cudaMalloc(tab, tab_bytes) : alloc_rec16(tab, tab_bytes)) != cudaSuccess ||
      (e = cudaMalloc(&t->fi, fb)) != cudaSuccess ||
      (e = cudaMalloc(&t->lb, lb_bytes)) != cudaSuccess ||
      (planes == SWG_PLANES_DECAY && (e = cudaMalloc(&t->fflip, 3 * fb)) != cudaSuccess)) {
    g_required = need;
    cudaGetLastError();
    swg_tables_destroy(t);
    return fail(SWG_ERR_CAPACITY, "tables need %zu device bytes: %s", need,
                cudaGetErrorString(e));
  }
  t->bytes = need;
  swg_status st = upload_and_quantize(t, pixels, is_device, pitch_bytes);
  if (st == SWG_OK)
    st = t->tdec  ? run_build_decay(t)
         : t->t16 ? run_build<uint16_t>(t, t->t16)
         : t->t64 ? run_build<uint64_t>(t, t->t64)
                  : run_build<uint32_t>(t, t->t32);
  if (st != SWG_OK) {
    swg_tables_destroy(t);
    return st;
  }
  *out = t;
  return SWG_OK;
}

swg_status swg_tables_build(swg_ctx* c, const void* pixels, int is_device,
                            size_t pitch_bytes, int width, int height,
                            int format, int bins, int planes,
                            size_t memory_budget, swg_tables** out) {
  if (planes == SWG_PLANES_DECAY) return fail(SWG_ERR_ARG, "decay tables: swg_tables_build_decay");
  return build_common(c, pixels, is_device, pitch_bytes, width, height, format, bins, planes,
                      0.0, 0, 0, memory_budget, out);
}

swg_status swg_tables_build_decay(swg_ctx* c, const void* pixels, int is_device,
                                  size_t pitch_bytes, int width, int height, int format,
                                  int bins, double decay, size_t memory_budget,
                                  swg_tables** out) {
  if (!(decay > 0.0 && decay < 1.0)) {
    if (out) *out = nullptr;
    return fail(SWG_ERR_INVALID_KERNEL, "decay must be in (0, 1)");
  }
  return build_common(c, pixels, is_device, pitch_bytes, width, height, format, bins,
                      SWG_PLANES_DECAY, decay, 0, 0, memory_budget, out);
}

swg_status swg_tables_build_bins(swg_ctx* c, const void* pixels, int is_device,
                                 size_t pitch_bytes, int width, int height, int format,
                                 int bins, int planes, double decay, int bin_begin,
                                 int bin_end, size_t memory_budget, swg_tables** out) {
  return build_common(c, pixels, is_device, pitch_bytes, width, height, format, bins, planes,
                      decay, bin_begin, bin_end, memory_budget, out);
}

swg_status swg_tables_bin_range(const swg_tables* t, int* bin_begin, int* bin_end,
                                int* total_bins) {
  ST_TRY(check_tables(t));
  if (bin_begin) *bin_begin = t->bin0;
  if (bin_end) *bin_end = t->bin0 + t->bins;
  if (total_bins) *total_bins = t->total_bins;
  return SWG_OK;
}

swg_status swg_tables_rebuild(swg_tables* t, const void* pixels, int is_device,
                              size_t pitch_bytes) {
  ST_TRY(check_tables(t));
  if (!pixels) return fail(SWG_ERR_ARG, "NULL pixels");
  if (!t->fi) return fail(SWG_ERR, "tables were loaded, not built: cannot rebuild");
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  ST_TRY(upload_and_quantize(t, pixels, is_device, pitch_bytes));
  t->carried = false;
  t->carry_y0 = 0;
  t->stale.clear();
  t->built_bytes = 0;
  if (t->t16) ST_TRY(run_build<uint16_t>(t, t->t16));
  if (t->t32) ST_TRY(run_build<uint32_t>(t, t->t32));  // (+ the narrow ramp planes)
  if (t->t16a && !t->t32) ST_TRY(build_t16a(t, true));
  if (t->t64) ST_TRY(run_build<uint64_t>(t, t->t64));
  if (t->tdec) ST_TRY(run_build_decay(t));
  return SWG_OK;
}

swg_status swg_tables_rebuild_bins(swg_tables* t, const void* pixels, int is_device,
                                   size_t pitch_bytes, int bin_begin) {
  ST_TRY(check_tables(t));
  if (!t->fi || (!pixels && !t->has_fi))
    return fail(SWG_ERR, "tables were loaded, not built: cannot rebuild");
  if (bin_begin < 0 || bin_begin + t->bins > t->total_bins)
    return fail(SWG_ERR_OUT_OF_RANGE, "bin range [%d, %d) of %d", bin_begin,
                bin_begin + t->bins, t->total_bins);
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  if (pixels) ST_TRY(upload_and_quantize(t, pixels, is_device, pitch_bytes));
  t->bin0 = bin_begin;
  t->stale.clear();
  t->built_bytes = 0;
  if (t->t16) ST_TRY(run_build<uint16_t>(t, t->t16));
  if (t->t32) ST_TRY(run_build<uint32_t>(t, t->t32));  // (+ the narrow ramp planes)
  if (t->t16a && !t->t32) ST_TRY(build_t16a(t, true));
  if (t->t64) ST_TRY(run_build<uint64_t>(t, t->t64));
  if (t->tdec) ST_TRY(run_build_decay(t));
  return SWG_OK;
}

swg_status swg_tables_built_bytes(const swg_tables* t, size_t* bytes) {
  ST_TRY(check_tables(t));
  if (!bytes) return fail(SWG_ERR_ARG, "NULL");
  *bytes = t->built_bytes;
  return SWG_OK;
}

swg_status swg_tables_upload_i64(swg_ctx* c, int w, int h, int bins,
                                 const int64_t* plain, const int64_t* xramp,
                                 const int64_t* yramp, swg_tables** out) {
  if (!c || !plain || !xramp || !yramp || !out) return fail(SWG_ERR_ARG, "NULL argument");
  *out = nullptr;
  if (w < 1 || h < 1 || bins < 1) return fail(SWG_ERR_IO, "table dump: bad dimensions");
  if (bins > 65535) return fail(SWG_ERR_IO, "table dump: bad dimensions");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  swg_tables* t = new swg_tables;
  t->ctx = c;
  c->refs++;
  t->w = w;
  t->h = h;
  t->bins = bins;
  t->total_bins = bins;
  t->planes = 3;
  t->format = SWG_FMT_BINS16;
  t->groups = (bins + kOct - 1) / kOct;
  t->pitch = record_pitch(w);
  t->ps = t->pitch * (size_t)(h + 1);
  const size_t nel = t->ps * 3 * t->groups * kOct;
  const size_t n = (size_t)(w + 1) * (h + 1) * bins;
  int64_t* staging = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&t->t32, nel * 4)) != cudaSuccess ||
      (e = cudaMalloc(&t->t64, nel * 8)) != cudaSuccess ||
      (e = cudaMalloc(&staging, n * 8)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(staging);
    swg_tables_destroy(t);
    g_required = nel * 12 + n * 8;
    return fail(SWG_ERR_CAPACITY, "loaded tables need %zu device bytes", g_required);
  }
  t->bytes = nel * 12;
  // padding bins / columns of the octet records stay zero
  e = cudaMemsetAsync(t->t64, 0, nel * 8, c->stream);
  const int64_t* src[3] = {plain, xramp, yramp};
  for (int k = 0; k < 3 && e == cudaSuccess; ++k) {
    e = cudaMemcpyAsync(staging, src[k], n * 8, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess)
      e = launch_import_i64(staging, w, h, bins, k, t->t64, t->ps, t->pitch, 3, c->stream);
    c->launches += 1;
  }
  if (e == cudaSuccess) e = launch_narrow(t->t64, t->t32, nel, c->stream);
  c->launches += 1;
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(staging);
  if (e != cudaSuccess) {
    swg_tables_destroy(t);
    return fail(SWG_ERR_CUDA, "upload: %s", cudaGetErrorString(e));
  }
  *out = t;
  return SWG_OK;
}

swg_status swg_tables_destroy(swg_tables* t) {
  if (!t) return SWG_OK;
  for (swg_tables* cl : t->clone) swg_tables_destroy(cl);
  if (t->ctx) {
    DeviceGuard g(t->ctx->device);
    cudaStreamSynchronize(t->ctx->stream);
    free_rec16(t->t16);
    cudaFree(t->t32);
    free_rec16(t->t16a);
    cudaFree(t->t64);
    free_rec16(t->tdec);
    cudaFree(t->fflip);
    cudaFree(t->fi);
    cudaFree(t->in);
    cudaFree(t->lb);
    ctx_release(t->ctx);
  }
  delete t;
  return SWG_OK;
}

swg_status swg_tables_info(const swg_tables* t, int* w, int* h, int* bins, int* planes,
                           size_t* bytes) {
  ST_TRY(check_tables(t));
  if (w) *w = t->w;
  if (h) *h = t->h;
  if (bins) *bins = t->bins;
  if (planes) *planes = t->planes;
  if (bytes) *bytes = t->bytes;
  return SWG_OK;
}

swg_status swg_tables_device_layout(const swg_tables* t, const void** base, size_t* ps,
                                    size_t* pitch, int* bins_per_record) {
  ST_TRY(check_tables(t));
  if (!t->stale.empty()) {  // raw plane pointers: every unit current first
    swg_tables* m = const_cast<swg_tables*>(t);
    std::lock_guard<std::mutex> lk(m->ctx->mu);
    DeviceGuard g(m->ctx->device);
    ST_TRY(fresh_all(m));
  }
  if (base) *base = t->tdec ? (const void*)t->tdec : (const void*)t->t32;
  if (ps) *ps = t->ps;
  if (pitch) *pitch = t->pitch;
  if (bins_per_record) *bins_per_record = t->tdec ? kDP : kOct;
  return SWG_OK;
}

static swg_status check_export(swg_tables* t, int kind, int b0, int b1, const void* out) {
  ST_TRY(check_tables(t));
  if (!out) return fail(SWG_ERR_ARG, "NULL out");
  if (kind < 0 || kind >= t->planes)
    return fail(SWG_ERR_OUT_OF_RANGE, "table kind %d not built (planes=%d)", kind, t->planes);
  if (b0 < 0 || b1 > t->bins || b0 > b1)
    return fail(SWG_ERR_OUT_OF_RANGE, "bins [%d, %d) outside [0, %d)", b0, b1, t->bins);
  return SWG_OK;
}

}  // extern "C"

template <typename T, typename O>
static swg_status export_planes(swg_tables* t, const T* tab, int kind, int b0, int b1, O* out) {
  swg_ctx* c = t->ctx;
  const size_t per_bin = (size_t)(t->w + 1) * (t->h + 1);
  // bounded staging: chunks of bins up to ~256 MB
  const int chunk = (int)std::max<size_t>(1, (256u << 20) / (per_bin * sizeof(O)));
  ST_TRY(c->qout.ensure((size_t)std::min(chunk, b1 - b0) * per_bin * sizeof(O)));
  for (int b = b0; b < b1; b += chunk) {
    const int e = std::min(b1, b + chunk);
    O* dev = static_cast<O*>(c->qout.p);
    CUDA_TRY((launch_export<T, O>(tab, t->ps, t->pitch, t->planes, t->w, t->h, kind, b, e,
                                  dev, c->stream)));
    c->launches += 1;
    CUDA_TRY(cudaMemcpyAsync(out + (size_t)(b - b0) * per_bin, dev,
                             (size_t)(e - b) * per_bin * sizeof(O), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  return SWG_OK;
}

extern "C" {

swg_status swg_tables_export_i64(swg_tables* t, int kind, int b0, int b1, int64_t* out) {
  ST_TRY(check_export(t, kind, b0, b1, out));
  if (t->carried)
    return fail(SWG_ERR_CONFIG, "tables carry a boundary prefix row: export their 32-bit words");
  if (b0 == b1) return SWG_OK;
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  ST_TRY(ensure_t64(t));
  return export_planes<uint64_t, int64_t>(t, t->t64, kind, b0, b1, out);
}

swg_status swg_tables_export_u32(swg_tables* t, int kind, int b0, int b1, uint32_t* out) {
  ST_TRY(check_export(t, kind, b0, b1, out));
  if (t->tdec) return fail(SWG_ERR_CONFIG, "decay tables hold no integral planes");
  if (b0 == b1) return SWG_OK;
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  if (kind >= 3) return fail(SWG_ERR_OUT_OF_RANGE, "quadratic planes are 64-bit only");
  ST_TRY(ensure_t32(t));
  ST_TRY(fresh_all(t));
  return export_planes<uint32_t, uint32_t>(t, t->t32, kind, b0, b1, out);
}

swg_status swg_tables_export_f64(swg_tables* t, int kind, int b0, int b1, double* out) {
  ST_TRY(check_export(t, kind, b0, b1, out));
  if (!t->tdec) return fail(SWG_ERR_CONFIG, "fp64 export is for decay tables");
  if (b0 == b1) return SWG_OK;
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  ST_TRY(fresh_all(t));
  swg_ctx* c = t->ctx;
  const size_t per_bin = (size_t)(t->w + 1) * (t->h + 1);
  const int chunk = (int)std::max<size_t>(1, (256u << 20) / (per_bin * 8));
  ST_TRY(c->qout.ensure((size_t)std::min(chunk, b1 - b0) * per_bin * 8));
  for (int b = b0; b < b1; b += chunk) {
    const int e = std::min(b1, b + chunk);
    double* dev = static_cast<double*>(c->qout.p);
    CUDA_TRY(launch_export_decay(t->tdec, t->ps, t->pitch, t->w, t->h, kind, b, e, dev,
                                 c->stream));
    c->launches += 1;
    CUDA_TRY(cudaMemcpyAsync(out + (size_t)(b - b0) * per_bin, dev, (size_t)(e - b) * per_bin * 8,
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  return SWG_OK;
}

swg_status swg_tables_feature_image(swg_tables* t, uint16_t* out) {
  ST_TRY(check_tables(t));
  if (!out) return fail(SWG_ERR_ARG, "NULL out");
  if (!t->has_fi) return fail(SWG_ERR, "tables were loaded from int64 planes: no feature image");
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  CUDA_TRY(cudaMemcpy2DAsync(out, (size_t)t->w * 2, t->fi, t->fip * 2, (size_t)t->w * 2, t->h,
                             cudaMemcpyDeviceToHost, t->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(t->ctx->stream));
  return SWG_OK;
}

swg_status swg_query_terms(swg_tables* t, int n, int tpw, const swg_term* terms,
                           int64_t* out) {
  ST_TRY(check_tables(t));
  if (n < 0 || tpw < 1 || (n && (!terms || !out))) return fail(SWG_ERR_ARG, "bad query arguments");
  if (n == 0) return SWG_OK;
  // Validate rectangles against the table (rect_sum bounds, integral_tables.cpp:127-138)
  // and bound the magnitude to pick 32-bit (sign-extended) or 64-bit planes.
  bool need64 = false;
  for (int w = 0; w < n; ++w) {
    double bound = 0.0;
    for (int k = 0; k < tpw; ++k) {
      const swg_term& q = terms[(size_t)w * tpw + k];
      if (!q.valid) continue;
      if (q.x0 < 0 || q.y0 < 0 || q.x0 > q.x1 || q.y0 > q.y1 || q.x1 >= t->w || q.y1 >= t->h)
        return fail(SWG_ERR_OUT_OF_RANGE,
                    "rect_sum: rectangle (%d,%d)-(%d,%d) out of bounds for %dx%d", q.x0, q.y0,
                    q.x1, q.y1, t->w, t->h);
      if ((q.sx || q.sy) && t->planes < 3)
        return fail(SWG_ERR_ARG, "query needs ramp planes; tables have plain only");
      const double area = double(q.x1 - q.x0 + 1) * double(q.y1 - q.y0 + 1);
      bound += area * (std::fabs(double(q.sx)) * t->w + std::fabs(double(q.sy)) * t->h +
                       std::fabs(double(q.beta)));
    }
    if (bound >= 2147483647.0) need64 = true;
  }
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  swg_ctx* c = t->ctx;
  if (need64) ST_TRY(ensure_t64(t));
  else ST_TRY(ensure_t32(t));
  ST_TRY(fresh_all(t));
  const size_t tb = (size_t)n * tpw * sizeof(swg_term), ob = (size_t)n * t->bins * 8;
  ST_TRY(c->terms.ensure(tb));
  ST_TRY(c->qout.ensure(ob));
  CUDA_TRY(cudaMemcpyAsync(c->terms.p, terms, tb, cudaMemcpyHostToDevice, c->stream));
  QueryArgs a{};
  a.planes = t->planes;
  a.bins = t->bins;
  a.n = n;
  a.tpw = tpw;
  a.terms = static_cast<const swg_term*>(c->terms.p);
  a.out = static_cast<long long*>(c->qout.p);
  a.plane_stride = t->ps;
  a.pitch = t->pitch;
  if (need64) {
    a.tab = t->t64;
    CUDA_TRY(launch_query<uint64_t>(a, c->stream));
  } else {
    a.tab = t->t32;
    CUDA_TRY(launch_query<uint32_t>(a, c->stream));
  }
  c->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(out, c->qout.p, ob, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (!need64)  // 32-bit planes: |value| < 2^31, sign-extend the low word
    for (size_t i = 0; i < (size_t)n * t->bins; ++i) out[i] = (int64_t)(int32_t)(uint32_t)out[i];
  return SWG_OK;
}

namespace {

// validate_window (engine.cpp:7-25)
swg_status validate_window(int w, int h, int cx, int cy, const swg_kernel& k, int border) {
  ST_TRY(validate_kernel(k));
  const int hx = k_hx(k), hy = k_hy(k);
  if (border == SWG_BORDER_STRICT) {
    if (cx - hx < 0 || cx + hx >= w || cy - hy < 0 || cy + hy >= h)
      return fail(SWG_ERR_WINDOW_OOB, "strict window %dx%d at (%d,%d) does not fit inside %dx%d",
                  k.kw, k.kh, cx, cy, w, h);
  } else if (border == SWG_BORDER_CLIPPED) {
    if (cx < 0 || cx >= w || cy < 0 || cy >= h)
      return fail(SWG_ERR_WINDOW_OOB, "clipped window center (%d,%d) outside image", cx, cy);
  } else {
    return fail(SWG_ERR_ARG, "border policy %d", border);
  }
  return SWG_OK;
}

// clip_rect (engine.cpp:29-35); an empty intersection invalidates the term.
void clip_term(swg_term& t, int w, int h) {
  if (!t.valid) return;
  t.x0 = std::max(t.x0, 0);
  t.y0 = std::max(t.y0, 0);
  t.x1 = std::min(t.x1, w - 1);
  t.y1 = std::min(t.y1, h - 1);
  if (t.x0 > t.x1 || t.y0 > t.y1) t.valid = 0;
}

}  // namespace

swg_status swg_cake_plan(const swg_kernel* k, int rings, int rule, int* sx, int* sy,
                         double* rw) {
  if (!k) return fail(SWG_ERR_ARG, "NULL kernel");
  ST_TRY(validate_kernel(*k));
  static thread_local CakeRings rg;
  std::vector<double> w;
  ST_TRY(cake_plan(*k, rings, rule, rg, &w));
  for (int i = 0; i < rings; ++i) {
    if (sx) sx[i] = k_hx(*k) - rg.a[i];
    if (sy) sy[i] = k_hy(*k) - rg.c[i];
    if (rw) rw[i] = w[i];
  }
  return SWG_OK;
}

swg_status swg_query_windows(swg_tables* t, int n, const int* cx, const int* cy,
                             const swg_kernel* k, int method, int border, int64_t* out) {
  ST_TRY(check_tables(t));
  if (n < 0 || !k || (n && (!cx || !cy || !out))) return fail(SWG_ERR_ARG, "bad query arguments");
  if (method != SWG_METHOD_SWIH && method != SWG_METHOD_PLAIN)
    return fail(SWG_ERR_ARG, "query method %d", method);
  const int tpw = method == SWG_METHOD_SWIH ? 4 : 1;
  std::vector<swg_term> terms((size_t)n * tpw);
  for (int i = 0; i < n; ++i) {
    ST_TRY(validate_window(t->w, t->h, cx[i], cy[i], *k, border));
    const int hx = k_hx(*k), hy = k_hy(*k), x = cx[i], y = cy[i];
    swg_term* d = &terms[(size_t)i * tpw];
    if (method == SWG_METHOD_PLAIN) {
      d[0] = swg_term{1, x - hx, y - hy, x + hx, y + hy, 0, 0, 1};
    } else {
      // decompose (engine.cpp:83-122): TL owns the centre row and column
      if (!k_affine(*k))
        return fail(SWG_ERR_UNSUPPORTED_KERNEL,
                    "decompose: kernel kind is not quadrant-affine; use the wedding-cake or "
                    "brute-force baseline");
      d[0] = swg_term{1, x - hx, y - hy, x, y, 0, 0, 0};
      d[1] = swg_term{hx > 0, x + 1, y - hy, x + hx, y, 0, 0, 0};
      d[2] = swg_term{hy > 0, x - hx, y + 1, x, y + hy, 0, 0, 0};
      d[3] = swg_term{hx > 0 && hy > 0, x + 1, y + 1, x + hx, y + hy, 0, 0, 0};
      if (k->kind == SWG_KERNEL_UNIFORM) {
        for (int q = 0; q < 4; ++q) d[q].beta = 1;
      } else {
        const int64_t m = hx + hy + 1;
        d[0].sx = +1; d[0].sy = +1; d[0].beta = m - x - y;
        d[1].sx = -1; d[1].sy = +1; d[1].beta = m + x - y;
        d[2].sx = +1; d[2].sy = -1; d[2].beta = m - x + y;
        d[3].sx = -1; d[3].sy = -1; d[3].beta = m + x + y;
      }
    }
    if (border == SWG_BORDER_CLIPPED)
      for (int q = 0; q < tpw; ++q) clip_term(d[q], t->w, t->h);
  }
  return swg_query_terms(t, n, tpw, terms.data(), out);
}

swg_status swg_cake_windows(swg_tables* t, int n, const int* cx, const int* cy,
                            const swg_kernel* k, int rings, int rule, int border, double* out) {
  ST_TRY(check_tables(t));
  if (n < 0 || !k || (n && (!cx || !cy || !out))) return fail(SWG_ERR_ARG, "bad query arguments");
  ST_TRY(validate_kernel(*k));
  static thread_local CakeRings rg;
  ST_TRY(cake_plan(*k, rings, rule, rg));
  if (n == 0) return SWG_OK;
  std::vector<swg_term> terms((size_t)n * rings);
  std::vector<double> coeff((size_t)n * rings);
  for (int i = 0; i < n; ++i) {
    ST_TRY(validate_window(t->w, t->h, cx[i], cy[i], *k, border));
    for (int r = 0; r < rings; ++r) {
      swg_term& q = terms[(size_t)i * rings + r];
      q = swg_term{1, cx[i] - rg.a[r], cy[i] - rg.c[r], cx[i] + rg.a[r], cy[i] + rg.c[r], 0, 0, 1};
      if (border == SWG_BORDER_CLIPPED) clip_term(q, t->w, t->h);
      coeff[(size_t)i * rings + r] = rg.coeff[r];
    }
  }
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  swg_ctx* c = t->ctx;
  ST_TRY(ensure_t32(t));
  ST_TRY(fresh_all(t));
  const size_t tb = terms.size() * sizeof(swg_term), cb = coeff.size() * 8;
  const size_t ob = (size_t)n * t->bins * 8;
  ST_TRY(c->terms.ensure(tb + cb));
  ST_TRY(c->qout.ensure(ob));
  CUDA_TRY(cudaMemcpyAsync(c->terms.p, terms.data(), tb, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(c->terms.p) + tb, coeff.data(), cb,
                           cudaMemcpyHostToDevice, c->stream));
  QueryArgs a{};
  a.tab = t->t32;
  a.plane_stride = t->ps;
  a.pitch = t->pitch;
  a.planes = t->planes;
  a.bins = t->bins;
  a.n = n;
  a.tpw = rings;
  a.terms = static_cast<const swg_term*>(c->terms.p);
  a.coeff = reinterpret_cast<const double*>(static_cast<char*>(c->terms.p) + tb);
  a.outd = static_cast<double*>(c->qout.p);
  CUDA_TRY(launch_cake_query(a, c->stream));
  c->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(out, c->qout.p, ob, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SWG_OK;
}

swg_status swg_quantize(swg_ctx* c, const void* pixels, int w, int h, int format, int bins,
                        uint16_t* out) {
  if (!c || !pixels || !out) return fail(SWG_ERR_ARG, "NULL argument");
  if (w < 1 || h < 1) return fail(SWG_ERR, "image dimensions must be >= 1");
  if (format < SWG_FMT_GRAY8 || format > SWG_FMT_BINS16) return fail(SWG_ERR_ARG, "format %d", format);
  if (bins < 1) return fail(SWG_ERR, "Quantizer: bin count must be >= 1");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  const size_t in_bytes = (size_t)w * h * pixel_bytes(format);
  const size_t in_pad = round_up(in_bytes, 256);
  ST_TRY(c->io.ensure(in_pad + (size_t)w * h * 2));
  uint8_t* din = static_cast<uint8_t*>(c->io.p);
  uint16_t* dout = reinterpret_cast<uint16_t*>(din + in_pad);
  CUDA_TRY(cudaMemcpyAsync(din, pixels, in_bytes, cudaMemcpyHostToDevice, c->stream));
  QuantArgs q{din, (size_t)w * pixel_bytes(format), w, h, format, bins, dout, (size_t)w};
  CUDA_TRY(launch_quantize(q, c->stream));
  c->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(out, dout, (size_t)w * h * 2, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SWG_OK;
}

swg_status swg_brute_windows(swg_ctx* c, const uint16_t* fi, int w, int h, int bins, int n,
                             const int* cx, const int* cy, const swg_kernel* k, int border,
                             int64_t* out_i64, double* out_f64) {
  if (!c || !fi || !k || (n && (!cx || !cy))) return fail(SWG_ERR_ARG, "NULL argument");
  if (!out_i64 && !out_f64) return fail(SWG_ERR_ARG, "no output");
  ST_TRY(validate_kernel(*k));
  if (out_i64 && !k_integer(*k))
    return fail(SWG_ERR_INVALID_KERNEL, "brute force counts: kernel weights are not integers");
  for (int i = 0; i < n; ++i) ST_TRY(validate_window(w, h, cx[i], cy[i], *k, border));
  if (n == 0) return SWG_OK;
  std::vector<double> wgrid((size_t)k->kw * k->kh);
  const int hx = k_hx(*k), hy = k_hy(*k);
  for (int dy = -hy; dy <= hy; ++dy)
    for (int dx = -hx; dx <= hx; ++dx) {
      double v = weight_at(*k, dx, dy);
      if (out_i64) v = (double)std::llround(v);  // BruteForcePlan grid_i (baselines.cpp:18-20)
      wgrid[(size_t)(dy + hy) * k->kw + dx + hx] = v;
    }
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  const size_t fb = round_up((size_t)w * h * 2, 256), cb = round_up((size_t)n * 4, 256);
  const size_t gb = round_up(wgrid.size() * 8, 256), ob = (size_t)n * bins * 8;
  ST_TRY(c->io.ensure(fb + 2 * cb + gb + 2 * ob));
  char* base = static_cast<char*>(c->io.p);
  uint16_t* dfi = reinterpret_cast<uint16_t*>(base);
  int* dcx = reinterpret_cast<int*>(base + fb);
  int* dcy = reinterpret_cast<int*>(base + fb + cb);
  double* dgrid = reinterpret_cast<double*>(base + fb + 2 * cb);
  long long* di = reinterpret_cast<long long*>(base + fb + 2 * cb + gb);
  double* dd = reinterpret_cast<double*>(base + fb + 2 * cb + gb + ob);
  CUDA_TRY(cudaMemcpyAsync(dfi, fi, (size_t)w * h * 2, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(dcx, cx, (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(dcy, cy, (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(dgrid, wgrid.data(), wgrid.size() * 8, cudaMemcpyHostToDevice,
                           c->stream));
  BruteQueryArgs a{dfi, w, h, bins, n, dcx, dcy, dgrid, k->kw, k->kh, border,
                   out_i64 != nullptr, out_i64 ? di : nullptr, out_f64 ? dd : nullptr};
  CUDA_TRY(launch_brute_query(a, c->stream));
  c->launches += 1;
  if (out_i64) CUDA_TRY(cudaMemcpyAsync(out_i64, di, ob, cudaMemcpyDeviceToHost, c->stream));
  if (out_f64) CUDA_TRY(cudaMemcpyAsync(out_f64, dd, ob, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SWG_OK;
}

swg_status swg_map_peak(swg_ctx* c, const double* scores, int mw, int mh, int hx, int hy,
                        swg_peak* out) {
  if (!c || !scores || !out) return fail(SWG_ERR_ARG, "NULL argument");
  if (mw < 1 || mh < 1) return fail(SWG_ERR, "peak: empty likelihood map");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  const size_t n = (size_t)mw * mh;
  const int nparts = (int)std::min<size_t>((n + 255) / 256, 148 * 4);
  ST_TRY(c->io.ensure(round_up(n * 8, 256)));
  swg_ctx::Scratch& S = c->scr[0];
  ST_TRY(S.parts.ensure((size_t)nparts * sizeof(PeakPart)));
  ST_TRY(S.peaks.ensure(sizeof(swg_peak)));
  CUDA_TRY(cudaMemcpyAsync(c->io.p, scores, n * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_map_peak(static_cast<const double*>(c->io.p), n, mw, hx, hy,
                           static_cast<PeakPart*>(S.parts.p), nparts,
                           static_cast<swg_peak*>(S.peaks.p), c->stream));
  c->launches += 2;
  CUDA_TRY(cudaMemcpyAsync(out, S.peaks.p, sizeof(swg_peak), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SWG_OK;
}

namespace {

// Sweep engine of one map request (plan_request).
enum Engine { kAffine32, kCake16, kCake32, kBrute, kQuad, kExp64, kAffine16 };

struct MapPlan {
  int row0 = 0, rows = 0, mw = 0;  // map rows [row0, row0 + rows) of width mw
  int chain_s = 0, chain_k = 0, chain_j = 0;  // chain order (0: off; SweepArgs)
  bool stream = false;  // Manhattan: the row-streaming chain sweep (k_stream.cu)
  Engine engine = kAffine32;
  swg_kernel k{};  // the kernel the engine sweeps (Plain maps: Uniform)
  dim3 grid;
  size_t soff = 0, poff = 0;  // offsets into the score / CTA-peak scratch
};

constexpr int kRescoreCap = 4096;  // exact-peak candidates re-scored per request

// Request checks in the reference order (matching.cpp:112-124), then the
// exactness limits of this implementation; fills the plan's row range.
swg_status validate_request(const swg_tables* t, const swg_map_request& r, bool host_scores,
                            MapPlan& p) {
  ST_TRY(validate_kernel(r.kernel));
  if (t->w < r.kernel.kw || t->h < r.kernel.kh)
    return fail(SWG_ERR_SIZE, "likelihood map: kernel %dx%d larger than search image %dx%d",
                r.kernel.kw, r.kernel.kh, t->w, t->h);
  if (!r.model) return fail(SWG_ERR_MODEL, "likelihood map: model must be normalized with %d bins", t->bins);
  if (r.method < 0 || r.method > 3) return fail(SWG_ERR_ARG, "method %d", r.method);
  if (r.sim < 0 || r.sim > 1) return fail(SWG_ERR_ARG, "similarity %d", r.sim);
  const bool quad = r.kernel.kind == SWG_KERNEL_EUCLID_QUAD;
  const bool expo = r.kernel.kind == SWG_KERNEL_EXP_L1;
  if (r.method == SWG_METHOD_SWIH && expo && !(t->tdec && r.kernel.sigma == t->decay))
    return fail(SWG_ERR_CONFIG,
                "likelihood map: exponential swih needs decay tables built with decay %g",
                r.kernel.sigma);
  if (t->tdec && r.method != SWG_METHOD_BRUTE && !(r.method == SWG_METHOD_SWIH && expo))
    return fail(SWG_ERR_CONFIG, "decay tables serve exponential swih and brute force only");
  if (r.method == SWG_METHOD_SWIH && !k_affine(r.kernel) && !quad && !expo)
    return fail(SWG_ERR_UNSUPPORTED_KERNEL,
                "likelihood map: method swih requires a quadrant-affine kernel");
  if (r.method == SWG_METHOD_SWIH && quad) {
    if (t->planes != SWG_PLANES_QUADRATIC)
      return fail(SWG_ERR_CONFIG, "likelihood map: Euclidean swih needs quadratic planes");
    if (quad_mass(r.kernel) >= (int64_t(1) << 53))
      return fail(SWG_ERR_CONFIG, "kernel %dx%d mass exceeds the exact fp64 range",
                  r.kernel.kw, r.kernel.kh);
    // the 32-bit planes give sum (x-cx)^2 exactly while it stays < 2^32
    const int64_t hm = std::max(k_hx(r.kernel), k_hy(r.kernel));
    if ((int64_t)r.kernel.kw * r.kernel.kh * hm * hm >= (int64_t(1) << 32))
      return fail(SWG_ERR_CONFIG, "kernel %dx%d: squared offsets exceed the 32-bit planes",
                  r.kernel.kw, r.kernel.kh);
  }
  if (t->bins > kMaxBins) return fail(SWG_ERR_CONFIG, "more than %d bins", kMaxBins);
  const bool ranged = t->bins != t->total_bins;
  if (ranged && !r.partial_in && !r.partial_out)
    return fail(SWG_ERR_CONFIG,
                "bin-range tables [%d, %d) of %d compute partial sums: give partial_out "
                "(or partial_in on the last range)", t->bin0, t->bin0 + t->bins, t->total_bins);
  if ((r.partial_in || r.partial_out) && r.method == SWG_METHOD_BRUTE)
    return fail(SWG_ERR_CONFIG, "bin-range chains run on the table sweeps, not brute force");
  if (r.partial_out && host_scores)
    return fail(SWG_ERR_ARG, "a partial (partial_out) request produces no scores");
  if (expo && r.partial_in && !r.partial_out && t->total_bins > kMaxBins)
    return fail(SWG_ERR_CONFIG, "exact exponential peak: more than %d bins", kMaxBins);
  const bool needs_ramps = (r.method == SWG_METHOD_SWIH || r.method == SWG_METHOD_BRUTE) &&
                           r.kernel.kind == SWG_KERNEL_MANHATTAN;
  if (needs_ramps && t->planes < 3 && !(r.method == SWG_METHOD_BRUTE && t->has_fi))
    return fail(SWG_ERR_CONFIG, "likelihood map: Manhattan swih needs the ramp planes");
  if (r.method == SWG_METHOD_BRUTE && !k_affine(r.kernel) && !t->has_fi)
    return fail(SWG_ERR_CONFIG, "likelihood map: brute force needs the feature image");
  const int mw = t->w - r.kernel.kw + 1, mh = t->h - r.kernel.kh + 1;
  int a = r.row_begin, b = r.row_end;
  if (a == 0 && b == 0) b = mh;
  if (a < 0 || b > mh || a > b) return fail(SWG_ERR_OUT_OF_RANGE, "map rows [%d, %d) of %d", a, b, mh);
  if (r.kernel.kind == SWG_KERNEL_MANHATTAN && affine_mass(r.kernel) >= (int64_t(1) << 32))
    return fail(SWG_ERR_CONFIG, "kernel %dx%d mass exceeds the 32-bit exact range", r.kernel.kw,
                r.kernel.kh);
  p.row0 = a;
  p.rows = b - a;
  p.mw = mw;
  return SWG_OK;
}

// Super-column CTA order for the table sweeps whose corner span (2hy+2
// table rows of the whole width) does not fit in L2: a strip of sw windows
// needs (2hy+2+tile) rows x (sw+2hx+2) cells resident.  0 = row-major order.
int super_column_tiles(const swg_tables* t, Engine e, const swg_kernel& k, int hx, int hy) {
  size_t cell = 0;  // table bytes per pixel the engine reads
  if (e == kAffine32) cell = (size_t)t->groups * kOct * (k.kind == SWG_KERNEL_UNIFORM ? 1 : 3) * 4;
  else if (e == kAffine16) cell = (size_t)t->groups * kOct * 3 * 2;
  else if (e == kQuad) cell = (size_t)t->groups * kOct * 5 * 4;
  else if (e == kExp64) cell = (size_t)t->groups * kOct * 4 * 8;
  else if (e == kCake32) cell = (size_t)t->groups * kOct * 4;
  if (!cell) return 0;
  const double budget = (double)SWG_L2_BUDGET_MB * 1048576.0;
  const double span =
      2.0 * hy + 2 + (e == kExp64 ? kExpTileY : e == kQuad ? kQuadTileY
                                               : e == kAffine16 ? kAff16TileY : kSweepTileY);
  if (span * (t->w + 1) * cell <= budget) return 0;
  const double sw = budget / (span * cell) - (2.0 * hx + 2);
  const int tw = e == kExp64 ? kExpTileX : e == kAffine16 ? 32 : kSweepTileX;  // windows per tile
  if (sw >= 2 * tw && (sw + 2.0 * hx + 2) / sw < 1.7) return std::max(1, (int)(sw / tw));
  return 0;
}

// CTA grid of a sweep over `rows` map rows of width mw.
dim3 sweep_grid(Engine e, int mw, int rows) {
  if (e == kBrute)
    return dim3((unsigned)((mw + kBruteThreads - 1) / kBruteThreads), (unsigned)std::max(rows, 1));
  const int tw = e == kExp64 ? kExpTileX : e == kCake16 ? kCakeCtaX : e == kAffine16 ? 32 : kSweepTileX;
  const int th = e == kExp64      ? kExpTileY
                 : e == kCake16   ? kCakeCtaY
                 : e == kAffine16 ? kAff16TileY
                 : e == kQuad     ? kQuadTileY
                                  : kSweepTileY;
  return dim3((unsigned)((mw + tw - 1) / tw), (unsigned)std::max((rows + th - 1) / th, 1));
}

// Engine and grid of a validated request.  The kernel-independent choices:
// Plain maps are Uniform-kernel maps; brute force on an integer affine kernel
// gives the quadrant path's exact counts (engine.hpp:62-66,
// test_matching.cpp:115-141) and shares its kernel; a Uniform box is a
// one-ring cake with coefficient 1.0 (exact integer weights, same scores:
// score_counts == score_weights on integers), so on narrow tables it runs the
// 16-bit cake sweep.
// Octets of the tables' bins holding a nonzero model value (SweepArgs::act;
// every octet with SWG_SPARSE=0).
int active_octets(const swg_tables* t, const swg_map_request& r) {
  const char* sp = std::getenv("SWG_SPARSE");
  if ((sp && std::atoi(sp) == 0) || !r.model) return t->groups;
  int nact = 0;
  for (int g8 = 0; g8 < t->groups; ++g8) {
    bool any = false;
    for (int b = g8 * kOct; b < std::min(t->bins, (g8 + 1) * kOct) && !any; ++b)
      any = r.model[t->bin0 + b] != 0.0;
    nact += any;
  }
  return nact;
}

// Units of the selective set (octets of the 32-bit planes, pairs of the
// decay planes) that a planned request reads: the model's nonzero ones for
// the sweeps that skip zero-model bins, all for the rest that read the set.
void plan_needs(const swg_tables* t, const swg_map_request& r, const MapPlan& p,
                std::vector<unsigned char>& need) {
  const char* sp = std::getenv("SWG_SPARSE");
  const bool sparse = !(sp && std::atoi(sp) == 0) && r.model;
  const int U = (int)need.size();
  auto all = [&] { std::fill(need.begin(), need.end(), (unsigned char)1); };
  if (p.rows == 0) return;
  switch (p.engine) {
    case kAffine32:
    case kAffine16:
    case kQuad:
      if (t->tdec || !sparse) return all();
      for (int b = 0; b < t->bins; ++b)
        if (r.model[t->bin0 + b] != 0.0 && b / kOct < U) need[b / kOct] = 1;
      return;
    case kExp64:
      if (!t->tdec || !sparse) return all();
      for (int b = 0; b < t->bins; ++b)
        if (r.model[t->bin0 + b] != 0.0 && b / kDP < U) need[b / kDP] = 1;
      return;
    case kCake32:
      if (!t->tdec) all();
      return;
    default:
      return;  // 16-bit plain planes / the feature image
  }
}

swg_status plan_request(const swg_tables* t, const swg_map_request& r, MapPlan& p) {
  swg_kernel k = r.kernel;
  int method = r.method;
  if (method == SWG_METHOD_PLAIN) {
    k.kind = SWG_KERNEL_UNIFORM;
    method = SWG_METHOD_SWIH;
  }
  if (method == SWG_METHOD_BRUTE && !t->tdec && (k.kind == SWG_KERNEL_UNIFORM ||
                                     (k.kind == SWG_KERNEL_MANHATTAN && t->planes >= 3)))
    method = SWG_METHOD_SWIH;
  const bool small = (long long)k.kw * k.kh < 65536;  // every box count < 2^16
  Engine e;
  if (method == SWG_METHOD_BRUTE) e = kBrute;
  else if (method == SWG_METHOD_SWIH && k.kind == SWG_KERNEL_EUCLID_QUAD) e = kQuad;
  else if (method == SWG_METHOD_SWIH && k.kind == SWG_KERNEL_EXP_L1) e = kExp64;
  else if (method == SWG_METHOD_CAKE)
    e = t->t16 && (small || cake16_wide0(k, r)) ? kCake16 : kCake32;
  else if (k.kind == SWG_KERNEL_UNIFORM && t->t16 && small) e = kCake16;
  else e = kAffine32;
  // Manhattan windows of mass < 2^16 on narrow {1, x, y} planes (k_sweep_affine16;
  // SWG_AFFINE16=0 keeps the 32-bit sweep)
  // (large maps only: for a small frame the extra narrow build costs more than
  // the sweep saves -- config 1, 50k windows: 0.033 -> 0.051 ms per step)
  if (e == kAffine32 && k.kind == SWG_KERNEL_MANHATTAN && t->planes >= 3 && t->has_fi &&
      !t->carried && affine_mass(k) < 65536 && (int64_t)p.rows * p.mw >= (int64_t(1) << 20) &&
      // the narrow planes cost a 3-plane 16-bit build per frame (config 5:
      // 0.38 ms) against 0.05-0.2 ms saved per scale: worth it for a model
      // that spans most octets, or once the planes exist
      (t->t16a || 2 * active_octets(t, r) > t->groups)) {
    const char* env = std::getenv("SWG_AFFINE16");
    if (!env || std::atoi(env)) e = kAffine16;
  }
  if (r.partial_in || r.partial_out) {  // engines that can continue a bin-range chain
    const bool closed_mass = e == kAffine32 || e == kQuad || e == kAffine16;
    if (e == kBrute || (!closed_mass && r.sim != SWG_SIM_BHATTACHARYYA))
      return fail(SWG_ERR_CONFIG,
                  "bin-range chains: Bhattacharyya, or intersection on swih Manhattan / "
                  "Uniform / Euclidean");
  }
  p.engine = e;
  p.k = k;
  p.grid = sweep_grid(e, p.mw, p.rows);
  // Chain order for the affine and quadratic sweeps (SWG_CHAIN_AFFINE /
  // SWG_CHAIN_QUAD: 0 off, 1 on, unset auto): window row v reads table rows
  // {v, v+hy+1, v+2hy+1} (affine) or {v, v+2hy+1} (quadratic), so chains of
  // step hy+1 (affine, residue groups of 8 so v+2hy+1 -- the lower row of
  // residue r-1's chain -- is close too) or 2hy+1 (quadratic) read each table
  // row once while it is in L2.
  if ((e == kAffine32 && k.kind != SWG_KERNEL_UNIFORM) || e == kQuad) {
    const bool aff = e == kAffine32;
    const char* env = std::getenv(aff ? "SWG_CHAIN_AFFINE" : "SWG_CHAIN_QUAD");
    const int hy = k_hy(k);
    const double cell = (double)t->groups * kOct * (aff ? 3 : 5) * 4;
    // measured on config 5 (A/B per scale, profiles/ab_sweep.py): the
    // affine sweep gains from 37^2 up (footprint > the 64 MB budget), the
    // quadratic one at every scale from 17^2 (footprint 58 MB): budgets 64 / 32 MB
    // (chain order also beats super-columns wherever those apply)
    bool on = (2.0 * hy + 2 + (aff ? kSweepTileY : kQuadTileY)) * (t->w + 1) * cell >
              (aff ? 1.0 : 0.5) * SWG_L2_BUDGET_MB * 1048576.0;
    if (env) on = std::atoi(env) != 0;
    if (on) {
      const int ck = std::getenv("SWG_CHAIN_K") ? std::atoi(std::getenv("SWG_CHAIN_K"))
                                                 : (aff ? 4 : 1);
      p.chain_s = aff ? hy + 1 : 2 * hy + 1;
      p.chain_k = std::max(1, std::min(ck, p.chain_s));
      p.chain_j = (p.rows + p.chain_s - 1) / p.chain_s;
      const int tw = aff ? kSweepThreads / 2 : kQuadThreads / 2;
      const unsigned gx = (unsigned)((p.mw + tw - 1) / tw);
      p.grid = dim3(gx * (unsigned)(p.chain_k * p.chain_j),
                    (unsigned)((p.chain_s + p.chain_k - 1) / p.chain_k));
    }
  }
  // Row-streaming chain sweep for Manhattan (k_stream.cu: one table row per
  // window instead of 20 corner records; SWG_STREAM=0 / 1 forces it off / on):
  // it needs the chain's segments (hy + 1 chains) x column blocks to fill the
  // GPU, so small maps keep the per-window sweeps.
  if ((e == kAffine32 && k.kind == SWG_KERNEL_MANHATTAN) || e == kAffine16 || e == kQuad) {
    const int hy = k_hy(k);
    const dim3 g = e == kQuad ? stream_quad_grid(p.mw, p.rows, hy)
                              : stream_grid(e == kAffine16, p.mw, p.rows, hy);
    bool on = hy >= 2 && (long long)g.x * g.y >= 2 * 148;
    // the quadratic stream sweep (10 x 256-bit loads per row, 128 registers)
    // wins when the model leaves octets out (config 5: 9.9 -> 4.1 ms); on a
    // dense model the per-window sweep is ~10 % faster
    if (e == kQuad && on) on = 4 * active_octets(t, r) <= 3 * t->groups;
    if (const char* env = std::getenv(e == kQuad ? "SWG_STREAM_QUAD" : "SWG_STREAM"))
      on = std::atoi(env) != 0 && p.rows > 0;
    if (on) {
      p.stream = true;
      p.grid = g;
      p.chain_s = p.chain_k = p.chain_j = 0;
    }
  }
  if (e == kExp64 && kExpTileY == 1) {
    // Chain order when a window's corner rows (2hy+2 table rows apart) do not
    // stay in L2 under raster order and super-columns would be too narrow:
    // window rows v and v + (hy+1) share the table row between v's bottom and
    // (v+hy+1)'s top corners (the SE and h-flipped tables), and residue
    // groups of 4 keep v + hy (the v-flipped tables' partner) close too
    // (measured: 129^2 on config 4 38.9 -> 34.3 ms, config 5's 117-257
    // scales -13 to -17 %; where super-columns apply they stay faster).
    const double cell = (double)t->groups * kOct * 4 * 8;
    const int hy = k_hy(k);
    bool on = (2.0 * hy + 3) * (t->w + 1) * cell > (double)SWG_L2_BUDGET_MB * 1048576.0 &&
              super_column_tiles(t, e, k, k_hx(k), hy) == 0;
    if (const char* env = std::getenv("SWG_CHAIN_EXP")) on = std::atoi(env) != 0;
    if (on) {
      const char* ek = std::getenv("SWG_CHAIN_KE");
      p.chain_s = hy + 1;
      p.chain_k = std::min(ek ? std::max(1, std::atoi(ek)) : 4, p.chain_s);
      p.chain_j = (p.rows + p.chain_s - 1) / p.chain_s;
      const unsigned gx = (unsigned)((p.mw + kExpTileX - 1) / kExpTileX);
      p.grid = dim3(gx * (unsigned)(p.chain_k * p.chain_j),
                    (unsigned)((p.chain_s + p.chain_k - 1) / p.chain_k));
    }
  }
  return SWG_OK;
}


// The kernel-independent sweep arguments of one request.
void fill_sweep_args(SweepArgs& a, const swg_tables* t, const swg_map_request& r,
                     const MapPlan& p, double* scores, PeakPart* parts) {
  a.tab = p.engine == kCake16     ? (const void*)t->t16
          : p.engine == kExp64    ? (const void*)t->tdec
          : p.engine == kAffine16 ? (const void*)t->t16a
                                  : (const void*)t->t32;
  a.plane_stride = t->ps;
  a.pitch = t->pitch;
  a.planes = p.engine == kAffine16 ? 3 : t->planes;
  a.bins = t->bins;
  a.groups = t->groups;
  a.hx = k_hx(p.k);
  a.hy = k_hy(p.k);
  a.mw = p.mw;
  a.row0 = p.row0;
  a.rows = p.rows;
  a.sim = r.sim;
  a.scores = scores;
  a.parts = parts;
  std::memset(a.model, 0, sizeof(a.model));
  std::memcpy(a.model, r.model + t->bin0, sizeof(double) * t->bins);
  const char* sp = std::getenv("SWG_SPARSE");
  const bool sparse = !sp || std::atoi(sp) != 0;
  a.nact = 0;
  for (int g = 0; g < t->groups; ++g) {
    bool any = !sparse;
    for (int k = 0; k < kOct && !any; ++k) any = a.model[g * kOct + k] != 0.0;
    if (any) a.act[a.nact++] = (unsigned char)g;
  }
  a.pin = static_cast<const double2*>(r.partial_in);
  a.pout = static_cast<double2*>(r.partial_out);
  a.sc_tiles = p.chain_s ? 0 : super_column_tiles(t, p.engine, p.k, a.hx, a.hy);
  a.y_off = p.engine == kCake16 ? 0 : t->carry_y0;  // global-row tables (add_carry)
  a.chain_s = p.chain_s;
  a.chain_k = p.chain_k;
  a.chain_j = p.chain_j;
}

// Exponential kernel: quadrant rectangles in their orientation's SE table
// (k_exp.cu, bin-pair records), coefficients in powers of the table's decay.
// Returns the fast path's score error bound.
double exp_plan(const swg_tables* t, const swg_map_request& r, int hx, int hy, ExpSweep& es) {
  const double dd = t->decay;
  auto pw = [&](int n) { return std::pow(dd, (double)n); };
  const long long p = (long long)t->pitch;
  // corners (dx, dy) from the centre record, per orientation, and rect extents
  const int cx0[4] = {1, 0, 1, 0}, cy0[4] = {1, 1, 0, 0};  // (x1+1, y1+1) offset
  const int ax[4] = {hx + 1, hx, hx + 1, hx}, by[4] = {hy + 1, hy + 1, hy, hy};
  const double qf[4] = {1.0, dd, dd, dd * dd};
  for (int o = 0; o < 4; ++o) {
    const int xs[4] = {cx0[o], cx0[o] - ax[o], cx0[o], cx0[o] - ax[o]};
    const int ys[4] = {cy0[o], cy0[o], cy0[o] - by[o], cy0[o] - by[o]};
    const double cf[4] = {qf[o], -qf[o] * pw(ax[o]), -qf[o] * pw(by[o]),
                          qf[o] * pw(ax[o] + by[o])};
    for (int q = 0; q < 4; ++q) {
      es.off[4 * o + q] = (int)(16 * (ys[q] * p + xs[q]));  // 16-B pair records
      es.coef[4 * o + q] = cf[q];
    }
  }
  es.w = t->w;
  es.h = t->h;
  // Table values <= T = 1/(1-d)^2; the damped recurrences keep each entry
  // within ~T u / (1-d) of exact (u = 2^-53), so one assembled bin is within
  // dh = 8 * 16 * T * u / (1-d) (16 corners, slack 8).  Bins below snap = 2 dh
  // are rounding noise of an empty bin; every real bin value is >= h_min =
  // d^(hx+hy) (the smallest weight).
  const double u = std::ldexp(1.0, -53);
  const double T = 1.0 / ((1.0 - dd) * (1.0 - dd));
  const double dh = 8.0 * 16.0 * T * u / (1.0 - dd);
  const double hmin = pw(hx + hy);
  es.snap = 2.0 * dh;
  // sparse mode: the closed-form window mass, the model's nonzero bin pairs
  es.wmass = 0.0;
  es.npair = 0;
  const char* sp = std::getenv("SWG_SPARSE");
  if ((!sp || std::atoi(sp) != 0) && r.model) {
    double sx = 0.0, sy = 0.0;
    for (int d = -hx; d <= hx; ++d) sx += pw(std::abs(d));
    for (int d = -hy; d <= hy; ++d) sy += pw(std::abs(d));
    es.wmass = sx * sy;
    const double* m = r.model + t->bin0;
    for (int q = 0; q < (t->bins + 1) / 2; ++q)
      if (m[2 * q] != 0.0 || (2 * q + 1 < t->bins && m[2 * q + 1] != 0.0))
        es.pairs[es.npair++] = (unsigned short)q;
  }
  if (es.snap >= 0.5 * hmin) return 1.0;  // no separation of noise and data: re-score everything
  if (r.sim == SWG_SIM_BHATTACHARYYA)
    // |d sum sqrt(m h)| <= sqrt(bins) dh / (2 sqrt(h_min)); mass term <= bins dh / 2
    return std::sqrt((double)t->total_bins) * dh / (2.0 * std::sqrt(hmin)) + t->total_bins * dh;
  return 2.0 * t->total_bins * dh;
}

// Exact-peak scratch of one request: candidates, their CTA peaks, a count.
struct RescoreSlice {
  static constexpr size_t kCand = (size_t)kRescoreCap * 8;
  static constexpr size_t kParts = (size_t)((kRescoreCap + 3) / 4) * sizeof(PeakPart);
  static constexpr size_t kBytes = (kCand + kParts + 256 + 255) / 256 * 256;
};

// Exponential sweep, then (full maps) the fast peak and the exact fp64
// re-score of the windows within 2 err of it.
swg_status run_exp(swg_ctx* c, const swg_tables* t, const swg_map_request& r, const MapPlan& p,
                   const SweepArgs& a, PeakPart* parts, swg_peak* peak, char* slice,
                   cudaStream_t st) {
  static thread_local ExpSweep es;
  const double err = exp_plan(t, r, a.hx, a.hy, es);
  CUDA_TRY(launch_sweep_exp(a, es, p.grid, st));
  c->launches += 1;
  if (r.partial_out) return SWG_OK;  // partial sums only: no scores, no peak
  CUDA_TRY(launch_peak_reduce(parts, (int)(p.grid.x * p.grid.y), p.mw, a.hx, a.hy, peak, st));
  c->launches += 1;
  static thread_local RescoreArgs ra;  // 8 KB of model: keep off the stack
  ra = RescoreArgs{};
  ST_TRY(weight_grid(c, p.k, &ra.grid));
  ra.fi = t->fi;
  ra.fi_pitch = t->fip;
  ra.kw = p.k.kw;
  ra.kh = p.k.kh;
  ra.bins = t->total_bins;  // every bin: the re-score is the whole histogram
  std::memset(ra.model, 0, sizeof(ra.model));
  std::memcpy(ra.model, r.model, sizeof(double) * t->total_bins);
  ra.cap = kRescoreCap;
  // a window outside [fast max - eps] cannot be the exact maximum when
  // eps >= 2 err (+ the fp64 rounding of the scores themselves)
  ra.eps = std::min(4.0, 2.0 * err + 1e-12);
  ra.cand = reinterpret_cast<long long*>(slice);
  ra.parts = reinterpret_cast<PeakPart*>(slice + RescoreSlice::kCand);
  ra.count = reinterpret_cast<int*>(slice + RescoreSlice::kCand + RescoreSlice::kParts);
  CUDA_TRY(launch_exact_peak(a, ra, peak, st));
  c->launches += 3;
  if (std::getenv("SWG_DEBUG_RESCORE")) {  // diagnostics: candidate count
    int cnt = 0;
    cudaMemcpyAsync(&cnt, ra.count, 4, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::fprintf(stderr, "swg rescore: kernel %dx%d eps %.3g candidates %d\n", p.k.kw, p.k.kh,
                 ra.eps, cnt);
  }
  return SWG_OK;
}

// Euclidean: box corners (TL, TR, BL, BR) of the whole window as byte
// offsets from the centre record within a plane of the 32-bit tables.
void quad_args(const swg_tables* t, const MapPlan& p, SweepArgs& a) {
  a.mass = (double)quad_mass(p.k);
  const long long p8 = (long long)t->pitch * kOct;
  const long long xs[2] = {-a.hx, a.hx + 1}, ys[2] = {-a.hy, a.hy + 1};
  for (int pl = 0; pl < 5; ++pl)
    for (int q = 0; q < 4; ++q)
      a.lat[4 * pl + q] = (int)(4 * (ys[q >> 1] * p8 + xs[q & 1] * kOct));
}

swg_status run_quad(const swg_tables* t, const MapPlan& p, SweepArgs& a, cudaStream_t st) {
  quad_args(t, p, a);
  if (p.stream) CUDA_TRY(launch_stream_quad(a, p.grid, st));
  else CUDA_TRY(launch_sweep_quad(a, p.grid, st));
  return SWG_OK;
}

// Quadrant-affine: corner byte offsets from the centre record (SweepArgs::lat order).
swg_status run_affine(const swg_tables* t, const MapPlan& p, SweepArgs& a, cudaStream_t st) {
  a.mass = (double)affine_mass(p.k);
  const long long p8 = (long long)t->pitch * kOct, ps8 = (long long)t->ps * kOct;
  const long long xs[3] = {-a.hx, 1, a.hx + 1}, ys[3] = {-a.hy, 1, a.hy + 1};
  auto off = [&](int plane, int xi, int yi) {
    return (int)(4 * (plane * ps8 + ys[yi] * p8 + xs[xi] * kOct));
  };
  const int pts[20][3] = {{0, 0, 0}, {0, 1, 0}, {0, 2, 0}, {0, 0, 1}, {0, 2, 1},
                          {0, 0, 2}, {0, 1, 2}, {0, 2, 2}, {1, 0, 0}, {1, 1, 0},
                          {1, 2, 0}, {1, 0, 2}, {1, 1, 2}, {1, 2, 2}, {2, 0, 0},
                          {2, 2, 0}, {2, 0, 1}, {2, 2, 1}, {2, 0, 2}, {2, 2, 2}};
  for (int q = 0; q < 20; ++q)
    a.lat[q] = pts[q][0] < t->planes ? off(pts[q][0], pts[q][1], pts[q][2]) : 0;
  if (p.stream) CUDA_TRY(launch_stream_affine(a, false, p.grid, st));
  else CUDA_TRY(launch_sweep_affine(a, p.k.kind == SWG_KERNEL_UNIFORM, p.grid, st));
  return SWG_OK;
}

// 16-bit Manhattan: the same corner points on the narrow {1, x, y} planes
// (16-byte records of 8 uint16 bins, 3-plane layout).
swg_status run_affine16(const swg_tables* t, const MapPlan& p, SweepArgs& a, cudaStream_t st) {
  a.mass = (double)affine_mass(p.k);
  const long long p8 = (long long)t->pitch * kOct, ps8 = (long long)t->ps * kOct;
  const long long xs[3] = {-a.hx, 1, a.hx + 1}, ys[3] = {-a.hy, 1, a.hy + 1};
  auto off = [&](int plane, int xi, int yi) {
    return (int)(2 * (plane * ps8 + ys[yi] * p8 + xs[xi] * kOct));
  };
  const int pts[20][3] = {{0, 0, 0}, {0, 1, 0}, {0, 2, 0}, {0, 0, 1}, {0, 2, 1},
                          {0, 0, 2}, {0, 1, 2}, {0, 2, 2}, {1, 0, 0}, {1, 1, 0},
                          {1, 2, 0}, {1, 0, 2}, {1, 1, 2}, {1, 2, 2}, {2, 0, 0},
                          {2, 2, 0}, {2, 0, 1}, {2, 2, 1}, {2, 0, 2}, {2, 2, 2}};
  for (int q = 0; q < 20; ++q) a.lat[q] = off(pts[q][0], pts[q][1], pts[q][2]);
  if (p.stream) CUDA_TRY(launch_stream_affine(a, true, p.grid, st));
  else CUDA_TRY(launch_sweep_affine16(a, p.grid, st));
  return SWG_OK;
}

// Cake (or a Uniform box as a one-ring cake): ring corner byte offsets from
// the centre record and the ring coefficients.
swg_status run_cake(const swg_tables* t, const swg_map_request& r, const MapPlan& p,
                    SweepArgs& a, cudaStream_t st) {
  static thread_local CakeRings rg;
  static thread_local CakeSweep cs;
  int rings = 1;
  if (r.method == SWG_METHOD_CAKE) {
    ST_TRY(cake_plan(p.k, r.rings, r.ring_rule, rg));
    rings = r.rings;
  } else {  // Uniform box: one ring, coefficient 1
    rg.a[0] = a.hx;
    rg.c[0] = a.hy;
    rg.coeff[0] = 1.0;
  }
  const bool narrow = p.engine == kCake16;
  const long long p8 = (long long)t->pitch * kOct;
  const long long eb = narrow ? 2 : 4;  // element bytes
  for (int q = 0; q < rings; ++q) {
    const long long ax = rg.a[q], cy = rg.c[q];
    cs.off[q] = make_int4((int)(eb * (-cy * p8 - ax * kOct)),
                          (int)(eb * (-cy * p8 + (ax + 1) * kOct)),
                          (int)(eb * ((cy + 1) * p8 - ax * kOct)),
                          (int)(eb * ((cy + 1) * p8 + (ax + 1) * kOct)));
    cs.coeff[q] = rg.coeff[q];
  }
  a.rings = rings;
  a.wide0 = narrow && (long long)p.k.kw * p.k.kh >= 65536;
  if (narrow) CUDA_TRY(launch_sweep_cake16(a, cs, p.grid, st));
  else CUDA_TRY(launch_sweep_cake(a, cs, p.grid, st));
  return SWG_OK;
}

// Device address of a page-locked, device-mapped host buffer allocated
// against this context's device (zero-copy maps), or nullptr for pageable,
// device or other devices' page-locked memory (those take the copy path).
double* mapped_host(void* p, int device) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  // page-locked, device-mapped host memory is reachable from every device
  // under unified addressing (the caller holds the context's device)
  (void)device;
  return at.type == cudaMemoryTypeHost && at.devicePointer
             ? static_cast<double*>(at.devicePointer)
             : nullptr;
}

// A frame's quadratic scales (frame batches) in one launch over all of them,
// so they read the table's rows together (L2) instead of the table once per
// scale, and one launch for their peaks.
swg_status run_quad_multi(swg_ctx* c, const swg_tables* t, int n, const swg_map_request* reqs,
                          const std::vector<MapPlan>& plan, double* const* scores,
                          PeakPart* parts, swg_peak* peaks) {
  static thread_local QuadMulti m;  // ~25 KB of kernel parameters
  PeakMulti pm;
  m.n = n;
  for (int i = 0; i < n; ++i) {
    const MapPlan& p = plan[i];
    fill_sweep_args(m.a[i], t, reqs[i], p, scores[i], parts + p.poff);
    quad_args(t, p, m.a[i]);
    m.gx[i] = (int)p.grid.x;
    m.gy[i] = (int)p.grid.y;
    pm.parts[i] = parts + p.poff;
    pm.n[i] = (int)(p.grid.x * p.grid.y);
    pm.mw[i] = p.mw;
    pm.hx[i] = m.a[i].hx;
    pm.hy[i] = m.a[i].hy;
    pm.out[i] = peaks + i;
  }
  CUDA_TRY(launch_sweep_quad_multi(m, c->stream));
  CUDA_TRY(launch_peak_reduce_multi(pm, n, c->stream));
  c->launches += 2;
  return SWG_OK;
}

// Multi-scale cake (k_sweep_cake16_multi): a full-ring square cake map of
// the whole frame on the narrow planes, Bhattacharyya (the intersection
// needs each scale's mass before its terms), all bins of one table.
bool cake_multi_ok(const swg_tables* t, const swg_map_request& r, const MapPlan& p) {
  const int h = k_hx(p.k);
  return p.engine == kCake16 && r.method == SWG_METHOD_CAKE && p.k.kw == p.k.kh && p.k.kw % 2 == 1 &&
         r.rings == h + 1 && h < kCakeMultiSpan && r.sim == SWG_SIM_BHATTACHARYYA &&
         !r.partial_in && !r.partial_out && p.row0 == 0 && p.rows == t->h - p.k.kh + 1 &&
         t->bin0 == 0 && t->bins == t->total_bins && t->groups * kOct <= kCakeMultiBins;
}

// Groups of up to kCakeMulti multi-scale cake requests (half-extents
// descending, each group's scales adjacent so its longest walk is shared by
// the most scales); gid[i] = the group of request i or -1.
void cake_groups(const swg_tables* t, int n, const swg_map_request* reqs,
                 const std::vector<MapPlan>& plan, std::vector<std::vector<int>>& groups,
                 std::vector<int>& gid) {
  gid.assign(n, -1);
  groups.clear();
  const char* ev = std::getenv("SWG_CAKE_GROUP");  // A/B: scales per launch (1 = off)
  const int gmax = std::min(ev ? std::atoi(ev) : kCakeMulti, kCakeMulti);
  if (gmax < 2) return;
  std::vector<int> cand;
  for (int i = 0; i < n; ++i)
    if (cake_multi_ok(t, reqs[i], plan[i])) cand.push_back(i);
  std::stable_sort(cand.begin(), cand.end(),
                   [&](int x, int y) { return k_hx(plan[x].k) > k_hx(plan[y].k); });
  const int nc = (int)cand.size();
  const int ng = (nc + gmax - 1) / gmax;
  for (int g = 0; g < ng; ++g) {  // near-equal group sizes
    const int b = g * nc / ng, e = (g + 1) * nc / ng;
    if (e - b < 2) continue;
    groups.emplace_back(cand.begin() + b, cand.begin() + e);
    for (int k = b; k < e; ++k) gid[cand[k]] = (int)groups.size() - 1;
  }
}

dim3 cake_group_grid(const swg_tables* t, const MapPlan& smallest) {
  CakeMulti m;
  m.w = t->w;
  m.h = t->h;
  m.n = 1;
  m.hs[0] = k_hx(smallest.k);
  return cake_multi_grid(m);
}

// One launch for a group's maps, one for their peaks.
swg_status run_cake_multi(swg_ctx* c, const swg_tables* t, const std::vector<int>& grp,
                          const swg_map_request* reqs, const std::vector<MapPlan>& plan,
                          double* const* scores, PeakPart* parts0, swg_peak* peaks,
                          cudaStream_t st) {
  static thread_local CakeMulti m;  // ~8 KB of kernel parameters
  static thread_local CakeRings rg;
  PeakMulti pm;
  std::memset(m.model, 0, sizeof(m.model));
  m.tab = t->t16;
  m.plane_stride = t->ps;
  m.pitch = t->pitch;
  m.planes = t->planes;
  m.groups = t->groups;
  m.w = t->w;
  m.h = t->h;
  m.n = (int)grp.size();
  const dim3 grid = cake_group_grid(t, plan[grp.back()]);
  for (int s = 0; s < m.n; ++s) {
    const int i = grp[s];
    const MapPlan& p = plan[i];
    const int h = k_hx(p.k);
    ST_TRY(cake_plan(p.k, reqs[i].rings, reqs[i].ring_rule, rg));
    m.hs[s] = h;
    m.mw[s] = p.mw;
    m.scores[s] = scores[i];
    m.parts[s] = parts0 + p.poff;
    for (int e = 0; e < kCakeMultiSpan; ++e) m.coef[s][e] = e <= h ? rg.coeff[h - e] : 0.0;
    std::memcpy(m.model[s], reqs[i].model, sizeof(double) * t->bins);
    pm.parts[s] = m.parts[s];
    pm.n[s] = (int)(grid.x * grid.y);
    pm.mw[s] = p.mw;
    pm.hx[s] = pm.hy[s] = h;
    pm.out[s] = peaks + i;
  }
  m.wide0 = (2LL * m.hs[0] + 1) * (2LL * m.hs[0] + 1) >= 65536;
  CUDA_TRY(launch_sweep_cake16_multi(m, st));
  CUDA_TRY(launch_peak_reduce_multi(pm, m.n, st));
  c->launches += 2;
  return SWG_OK;
}

// Direct per-pixel weighted histogram (baselines.cpp:24-69).
swg_status run_brute(swg_ctx* c, const swg_tables* t, const MapPlan& p, const SweepArgs& a,
                     cudaStream_t st) {
  BruteArgs ba{};
  ST_TRY(weight_grid(c, p.k, &ba.grid));
  ba.fi = t->fi;
  ba.fi_pitch = t->fip;
  ba.kw = p.k.kw;
  ba.kh = p.k.kh;
  ba.integer = k_integer(p.k);
  CUDA_TRY(launch_sweep_brute(a, ba, p.grid.x, st));
  return SWG_OK;
}

}  // namespace

swg_status swg_request_groups(const swg_tables* t, int n, const swg_map_request* reqs,
                              int* group_of) {
  ST_TRY(check_tables(t));
  if (n < 0 || (n && (!reqs || !group_of))) return fail(SWG_ERR_ARG, "bad request list");
  std::vector<MapPlan> plan(n);
  for (int i = 0; i < n; ++i) {
    ST_TRY(validate_request(t, reqs[i], false, plan[i]));
    ST_TRY(plan_request(t, reqs[i], plan[i]));
  }
  std::vector<std::vector<int>> groups;
  std::vector<int> gid;
  cake_groups(t, n, reqs, plan, groups, gid);
  for (int i = 0; i < n; ++i) group_of[i] = gid[i];
  return SWG_OK;
}

swg_status swg_request_plan(const swg_tables* t, const swg_map_request* r, swg_plan_info* out) {
  ST_TRY(check_tables(t));
  if (!r || !out) return fail(SWG_ERR_ARG, "NULL argument");
  MapPlan p;
  ST_TRY(validate_request(t, *r, false, p));
  ST_TRY(plan_request(t, *r, p));
  std::memset(out, 0, sizeof(*out));
  static thread_local SweepArgs a;
  fill_sweep_args(a, t, *r, p, nullptr, nullptr);
  const char* name = "";
  int planes = 1, eb = 4, bins = t->bins;
  switch (p.engine) {
    case kAffine32:
      name = p.stream ? "k_stream_affine" : "k_sweep_affine";
      planes = p.k.kind == SWG_KERNEL_UNIFORM ? 1 : 3;
      bins = std::min(t->bins, a.nact * kOct);
      break;
    case kAffine16:
      name = p.stream ? "k_stream_affine16" : "k_sweep_affine16";
      planes = 3;
      eb = 2;
      bins = std::min(t->bins, a.nact * kOct);
      break;
    case kQuad:
      name = p.stream ? "k_stream_quad" : "k_sweep_quad";
      planes = 5;
      bins = std::min(t->bins, a.nact * kOct);
      break;
    case kExp64: {
      name = "k_sweep_exp";
      planes = 4;
      eb = 8;
      static thread_local ExpSweep es;
      exp_plan(t, *r, a.hx, a.hy, es);
      if (es.wmass > 0.0) bins = std::min(t->bins, es.npair * kDP);
      break;
    }
    case kCake16: name = "k_sweep_cake16"; eb = 2; break;
    case kCake32: name = "k_sweep_cake"; break;
    case kBrute: name = "k_sweep_brute"; planes = 0; eb = 0; break;
  }
  std::snprintf(out->kernel, sizeof(out->kernel), "%s", name);
  out->planes = planes;
  out->entry_bytes = eb;
  out->bins_read = bins;
  out->ctas = (int)(p.grid.x * p.grid.y);
  return SWG_OK;
}

swg_status swg_tables_rebuild_for(swg_tables* t, const void* pixels, int is_device,
                                  size_t pitch_bytes, int n, const swg_map_request* reqs) {
  ST_TRY(check_tables(t));
  if (!pixels) return fail(SWG_ERR_ARG, "NULL pixels");
  if (n < 0 || (n && !reqs)) return fail(SWG_ERR_ARG, "bad request list");
  if (!t->fi) return fail(SWG_ERR, "tables were loaded, not built: cannot rebuild");
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  ST_TRY(upload_and_quantize(t, pixels, is_device, pitch_bytes));
  t->carried = false;
  t->carry_y0 = 0;
  t->stale.clear();
  t->built_bytes = 0;
  if (t->t16) ST_TRY(run_build<uint16_t>(t, t->t16));
  if (selective(t)) {
    std::vector<unsigned char> need((size_t)sel_units(t), 0);
    for (int i = 0; i < n; ++i) {
      MapPlan p;
      if (validate_request(t, reqs[i], false, p) != SWG_OK || plan_request(t, reqs[i], p) != SWG_OK)
        std::fill(need.begin(), need.end(), (unsigned char)1);  // the map call reports it
      else
        plan_needs(t, reqs[i], p, need);
    }
    std::vector<int> sel;
    for (int u = 0; u < (int)need.size(); ++u)
      if (need[u]) sel.push_back(u);
    const bool full = sel.size() == need.size();
    if (t->tdec) ST_TRY(run_build_decay(t, full ? nullptr : &sel));
    else ST_TRY(run_build<uint32_t>(t, t->t32, full ? nullptr : &sel));
    if (!full) {
      t->stale.assign(need.size(), 1);
      for (int u : sel) t->stale[u] = 0;
    }
  } else {
    if (t->t32) ST_TRY(run_build<uint32_t>(t, t->t32));
    if (t->t16a && !t->t32) ST_TRY(build_t16a(t, true));
    if (t->tdec) ST_TRY(run_build_decay(t));
  }
  if (t->t64) ST_TRY(run_build<uint64_t>(t, t->t64));
  return SWG_OK;
}

static swg_status likelihood_maps_impl(swg_tables* t, int n, const swg_map_request* reqs,
                                       double* const* scores_host, double* const* scores_dev,
                                       swg_peak* peaks_host, swg_peak* peaks_dev, bool async);

swg_status swg_likelihood_maps(swg_tables* t, int n, const swg_map_request* reqs,
                               double* const* scores_host, double* const* scores_dev,
                               swg_peak* peaks_host, swg_peak* peaks_dev) {
  return likelihood_maps_impl(t, n, reqs, scores_host, scores_dev, peaks_host, peaks_dev, false);
}

swg_status swg_likelihood_maps_async(swg_tables* t, int n, const swg_map_request* reqs,
                                     double* const* scores_host, double* const* scores_dev,
                                     swg_peak* peaks_host, swg_peak* peaks_dev) {
  return likelihood_maps_impl(t, n, reqs, scores_host, scores_dev, peaks_host, peaks_dev, true);
}

}  // extern "C"

static swg_status likelihood_maps_impl(swg_tables* t, int n, const swg_map_request* reqs,
                                       double* const* scores_host, double* const* scores_dev,
                                       swg_peak* peaks_host, swg_peak* peaks_dev, bool async) {
  ST_TRY(check_tables(t));
  if (n < 0 || (n && !reqs)) return fail(SWG_ERR_ARG, "bad request list");
  if (n == 0) return SWG_OK;
  auto host_map = [&](int i) { return scores_host && scores_host[i]; };
  auto dev_map = [&](int i) { return scores_dev && scores_dev[i]; };
  // every request is checked before anything launches
  std::vector<MapPlan> plan(n);
  for (int i = 0; i < n; ++i) ST_TRY(validate_request(t, reqs[i], host_map(i), plan[i]));
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  swg_ctx* c = t->ctx;
  // Zero-copy host maps: a host map in page-locked, device-mapped memory
  // (swg_host_alloc / cudaMallocHost) is written by the sweep itself over
  // PCIe, so no copy trails the last sweep (the exponential sweep's re-score
  // reads its map back: it keeps the device scratch and a copy).
  std::vector<double*> zc(n, nullptr);
  for (int i = 0; i < n; ++i) {
    ST_TRY(plan_request(t, reqs[i], plan[i]));
    // zero-copy maps for a few requests (their sweeps fan out and write over
    // PCIe directly: config 2 e2e 1.31 -> 1.18 ms); with more requests the
    // sweeps run back to back and each finished map is copied by the copy
    // engine while the next one sweeps -- a burst of fast sweeps writing over
    // PCIe would stall on the link (config 5 e2e 32.5 -> 28.7 ms per step)
    const char* ez = std::getenv("SWG_ZC_MAX");  // A/B: most requests that use zero-copy maps
    const int zc_max = ez ? std::atoi(ez) : swg_ctx::kHostFan;
    if (host_map(i) && !dev_map(i) && plan[i].engine != kExp64 && n <= zc_max)
      zc[i] = mapped_host(scores_host[i], c->device);
  }
  auto copy_map = [&](int i) { return host_map(i) && !zc[i]; };
  // multi-scale cake groups: each member's CTA candidates cover the group's grid
  std::vector<std::vector<int>> cgroups;
  std::vector<int> cgid;
  cake_groups(t, n, reqs, plan, cgroups, cgid);
  for (const auto& g : cgroups) {
    const dim3 gg = cake_group_grid(t, plan[g.back()]);
    for (int i : g) plan[i].grid = gg;
  }
  // scratch: per-request score buffers (when the caller gave no device or
  // mapped output), CTA peak candidates, device peaks, exact-peak slices
  size_t stot = 0, ptot = 0;
  for (int i = 0; i < n; ++i) {
    MapPlan& p = plan[i];
    if (!dev_map(i) && !zc[i]) {
      p.soff = stot;
      stot += round_up((size_t)p.rows * p.mw, 32);
    }
    p.poff = ptot;
    // + spare CTA rows: the split last map (a stream sweep's halves may each
    // round up a segment row of hy + 1 chains)
    ptot += (size_t)p.grid.x * (p.grid.y + 1 + (p.stream ? 2 * k_hy(p.k) + 1 : 0));
  }
  // an asynchronous call takes the next scratch slot, once the copies (or
  // sweeps) of the call that used it last have finished
  // (a table set keeps its slot: the slots' scratch sizes stay put)
  int sl = c->slot;
  if (async && c->slot == 0) {
    if (t->aslot < 0) {  // slots 1.. (slot 0 stays the synchronous calls')
      t->aslot = 1 + c->aslot;
      c->aslot = (c->aslot + 1) % (swg_ctx::kWorkers - 1);
    }
    sl = t->aslot;
    if (c->free_ev[sl]) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->free_ev[sl], 0));
  }
  swg_ctx::Scratch& S = c->scr[sl];
  ST_TRY(S.scores.ensure(std::max<size_t>(stot, 1) * 8));
  ST_TRY(S.parts.ensure(ptot * sizeof(PeakPart)));
  ST_TRY(S.peaks.ensure((size_t)n * sizeof(swg_peak)));
  ST_TRY(S.resc.ensure(RescoreSlice::kBytes * n));
  swg_peak* dpeaks = peaks_dev ? peaks_dev : static_cast<swg_peak*>(S.peaks.p);
  // units of a selective rebuild that these requests read but are stale
  if (!t->stale.empty()) {
    std::vector<unsigned char> need((size_t)sel_units(t), 0);
    for (int i = 0; i < n; ++i) plan_needs(t, reqs[i], plan[i], need);
    ST_TRY(ensure_fresh(t, &need));
  }
  // the lazily built 32-bit planes go on the main stream before the fan-out
  for (const MapPlan& p : plan)
    if (p.rows > 0 && (p.engine == kAffine32 || p.engine == kCake32)) ST_TRY(ensure_t32(t));
  for (const MapPlan& p : plan)
    if (p.rows > 0 && p.engine == kAffine16) ST_TRY(ensure_t16a(t));

  bool host_maps = false;  // maps that still need a device-to-host copy
  for (int i = 0; i < n; ++i) host_maps |= copy_map(i);
  int nwork = 0;
  cudaStream_t* wk = c->work;
  cudaEvent_t* wj = c->join;
#ifndef SWG_NO_FANOUT
  // Device outputs: overlap the requests' sweeps on equal-priority workers.
  // Host maps: up to kHostFan requests on the prioritised workers (each map
  // copied as its sweep ends, config 2 e2e 1.38 -> 1.32 ms); more requests
  // stay in sequence so each map's copy overlaps the next sweep (the copy
  // engine would fall behind a burst of finished maps: config 5 +20 %).
  if (c->fanout_off) {
    nwork = 0;
  } else if (host_maps) {
    nwork = n <= swg_ctx::kHostFan ? n : 0;
    wk = c->hwork;
    wj = c->hjoin;
  } else {
    nwork = std::min(n, (int)swg_ctx::kWorkers);
    if (const char* ew = std::getenv("SWG_WORKERS")) nwork = std::min(nwork, std::max(1, std::atoi(ew)));
    if (n <= swg_ctx::kHostFan) {  // a few requests: costliest first on the highest priority
      wk = c->hwork;              // (config 2: e2e 1.19 -> 1.17 ms with mapped host maps,
      wj = c->hjoin;              // device-resident 1.114 -> 1.116 ms)
    }
  }
  if (nwork > 1) {
    CUDA_TRY(cudaEventRecord(c->fork, c->stream));
    for (int w = 0; w < nwork; ++w) CUDA_TRY(cudaStreamWaitEvent(wk[w], c->fork, 0));
  } else {
    nwork = 0;
  }
#endif

  bool copies = false;
  // the score output of request i: the caller's device map, its mapped host
  // map, or device scratch
  std::vector<double*> out(n);
  for (int i = 0; i < n; ++i)
    out[i] = dev_map(i) ? scores_dev[i]
             : zc[i]    ? zc[i]
                        : static_cast<double*>(S.scores.p) + plan[i].soff;
  PeakPart* parts0 = static_cast<PeakPart*>(S.parts.p);
  bool fused = c->fanout_off && nwork == 0 && n >= 2 && n <= kQuadMulti && t->carry_y0 == 0;
  for (int i = 0; i < n && fused; ++i)
    fused = plan[i].engine == kQuad && plan[i].rows > 0 && !reqs[i].partial_in &&
            !reqs[i].partial_out && !copy_map(i) && plan[i].chain_s == 0 && !plan[i].stream &&
            super_column_tiles(t, kQuad, plan[i].k, k_hx(plan[i].k), k_hy(plan[i].k)) == 0;
  if (fused) ST_TRY(run_quad_multi(c, t, n, reqs, plan, out.data(), parts0, dpeaks));
  // Device-output fan-out issues the costliest sweeps first (longest-first
  // packing: the last scale to start is a short one; config 2 1.130 ->
  // 1.114 ms); host-map fan-out keeps request order (its streams'
  // priorities order the copies).
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  if (nwork > 1 && !host_maps) {
    auto cost = [&](int i) {
      const MapPlan& p = plan[i];
      const double rings = p.engine == kCake16 || p.engine == kCake32
                               ? (reqs[i].method == SWG_METHOD_CAKE ? reqs[i].rings : 1)
                               : 1;
      if (cgid[i] >= 0) {  // a multi-scale cake group: its members' cost (leader only)
        if (cgroups[cgid[i]][0] != i) return 0.0;
        double g = 0.0;
        for (int j : cgroups[cgid[i]]) g += (double)plan[j].rows * plan[j].mw * reqs[j].rings;
        return 0.5 * g;
      }
      return (double)p.rows * p.mw * rings;
    };
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cost(x) > cost(y); });
  }
  for (int q = 0; q < n && !fused; ++q) {
    const int i = order[q];
    const swg_map_request& r = reqs[i];
    const MapPlan& p = plan[i];
    if (p.rows == 0) continue;
    const cudaStream_t st = nwork ? wk[q % nwork] : c->stream;
    double* dscores = out[i];
    PeakPart* parts = parts0 + p.poff;
    if (cgid[i] >= 0) {  // multi-scale cake: the group's leader sweeps every member
      const std::vector<int>& grp = cgroups[cgid[i]];
      if (grp[0] != i) continue;
      ST_TRY(run_cake_multi(c, t, grp, reqs, plan, out.data(), parts0, dpeaks, st));
      for (int j : grp) {
        if (!copy_map(j)) continue;
        while (c->events.size() <= (size_t)j) {
          cudaEvent_t ev;
          CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          c->events.push_back(ev);
        }
        CUDA_TRY(cudaEventRecord(c->events[j], st));
        CUDA_TRY(cudaStreamWaitEvent(c->copy, c->events[j], 0));
        CUDA_TRY(cudaMemcpyAsync(scores_host[j], out[j], (size_t)plan[j].rows * plan[j].mw * 8,
                                 cudaMemcpyDeviceToHost, c->copy));
        c->map_copies += 1;
        copies = true;
      }
      continue;
    }
    static thread_local SweepArgs a;  // 8 KB of model constants: keep off the stack
    // the copy stream takes a finished map (or row range of it) while later
    // sweeps run
    auto copy_rows = [&](int slot, int row_off, int rows) -> swg_status {
      while (c->events.size() <= (size_t)slot) {
        cudaEvent_t ev;
        CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        c->events.push_back(ev);
      }
      CUDA_TRY(cudaEventRecord(c->events[slot], st));
      CUDA_TRY(cudaStreamWaitEvent(c->copy, c->events[slot], 0));
      CUDA_TRY(cudaMemcpyAsync(scores_host[i] + (size_t)row_off * p.mw,
                               dscores + (size_t)row_off * p.mw, (size_t)rows * p.mw * 8,
                               cudaMemcpyDeviceToHost, c->copy));
      c->map_copies += 1;
      copies = true;
      return SWG_OK;
    };
    auto sweep = [&](const MapPlan& q, double* sc, PeakPart* pp) -> swg_status {
      fill_sweep_args(a, t, r, q, sc, pp);
      if (q.engine == kQuad) ST_TRY(run_quad(t, q, a, st));
      else if (q.engine == kAffine32) ST_TRY(run_affine(t, q, a, st));
      else if (q.engine == kAffine16) ST_TRY(run_affine16(t, q, a, st));
      else if (q.engine == kBrute) ST_TRY(run_brute(c, t, q, a, st));
      else ST_TRY(run_cake(t, r, q, a, st));
      c->launches += 1;
      return SWG_OK;
    };
    // The last of a few fanned-out host maps is swept in two row halves, so
    // the first half's copy overlaps the second half's sweep (config 2 e2e
    // 1.325 -> 1.312 ms; three or four parts: 1.327 / 1.40 ms).
    constexpr int kSplit = 2;
    const bool split = nwork > 1 && copy_map(i) && i == n - 1 && p.engine != kExp64 &&
                       !r.partial_in && !r.partial_out && p.rows >= 64;
    if (p.engine == kExp64) {  // reduces (and re-scores) its own peak
      fill_sweep_args(a, t, r, p, dscores, parts);
      char* slice = static_cast<char*>(S.resc.p) + RescoreSlice::kBytes * i;
      ST_TRY(run_exp(c, t, r, p, a, parts, dpeaks + i, slice, st));
      if (copy_map(i)) ST_TRY(copy_rows(i, 0, p.rows));
    } else if (split) {
      int done = 0, np = 0;  // rows and CTA candidates so far
      for (int q = 0; q < kSplit; ++q) {
        MapPlan h = p;
        h.row0 = p.row0 + done;
        h.rows = (q + 1) * p.rows / kSplit - done;
        h.grid = !p.stream           ? sweep_grid(p.engine, p.mw, h.rows)
                 : p.engine == kQuad ? stream_quad_grid(p.mw, h.rows, k_hy(p.k))
                                     : stream_grid(p.engine == kAffine16, p.mw, h.rows, k_hy(p.k));
        ST_TRY(sweep(h, dscores + (size_t)done * p.mw, parts + np));
        np += (int)(h.grid.x * h.grid.y);
        if (q + 1 < kSplit) ST_TRY(copy_rows(n * (q + 1) + i, done, h.rows));  // own event
        else {
          CUDA_TRY(launch_peak_reduce(parts, np, p.mw, a.hx, a.hy, dpeaks + i, st));
          c->launches += 1;
          ST_TRY(copy_rows(i, done, h.rows));
        }
        done += h.rows;
      }
    } else {
      ST_TRY(sweep(p, dscores, parts));
      if (!r.partial_out) {
        CUDA_TRY(launch_peak_reduce(parts, (int)(p.grid.x * p.grid.y), p.mw, a.hx, a.hy,
                                    dpeaks + i, st));
        c->launches += 1;
      }
      if (copy_map(i)) ST_TRY(copy_rows(i, 0, p.rows));
    }
  }
  for (int w = 0; w < nwork; ++w) {  // join the worker streams
    CUDA_TRY(cudaEventRecord(wj[w], wk[w]));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, wj[w], 0));
  }
  bool sync = copies;
  for (int i = 0; i < n; ++i) sync |= zc[i] != nullptr;  // mapped maps: filled on return
  if (peaks_host) {
    // behind the map copies on the copy stream: a device-to-host copy on the
    // compute stream would queue on the copy engine behind the maps' copies
    // and hold the next call's sweeps (config 5 e2e: 32.1 -> see DESIGN)
    if (copies) {
      while (c->events.size() <= (size_t)(3 * n)) {
        cudaEvent_t ev;
        CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        c->events.push_back(ev);
      }
      CUDA_TRY(cudaEventRecord(c->events[3 * n], c->stream));
      CUDA_TRY(cudaStreamWaitEvent(c->copy, c->events[3 * n], 0));
      CUDA_TRY(cudaMemcpyAsync(peaks_host, dpeaks, (size_t)n * sizeof(swg_peak),
                               cudaMemcpyDeviceToHost, c->copy));
    } else {
      CUDA_TRY(cudaMemcpyAsync(peaks_host, dpeaks, (size_t)n * sizeof(swg_peak),
                               cudaMemcpyDeviceToHost, c->stream));
    }
    sync = true;
  }
  if (async) {  // host outputs are filled when the context's streams are synchronised
    if (!c->free_ev[sl]) CUDA_TRY(cudaEventCreateWithFlags(&c->free_ev[sl], cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(c->free_ev[sl], copies ? c->copy : c->stream));
    return SWG_OK;
  }
  if (sync) CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (copies) CUDA_TRY(cudaStreamSynchronize(c->copy));
  return SWG_OK;
}

extern "C" {

swg_status swg_likelihood_batch(swg_tables* t, int n_frames, const void* const* frames,
                                int is_device, size_t pitch_bytes, int n,
                                const swg_map_request* reqs, swg_peak* peaks_host,
                                swg_peak* peaks_dev) {
  ST_TRY(check_tables(t));
  if (n_frames < 0 || n < 0 || (n_frames && !frames) || (n && !reqs))
    return fail(SWG_ERR_ARG, "bad frame or request list");
  if (!n_frames || !n) return SWG_OK;
  swg_ctx* c = t->ctx;
  swg_peak* dst = peaks_dev;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (!dst) {
      ST_TRY(c->bpeaks.ensure((size_t)n_frames * n * sizeof(swg_peak)));
      dst = static_cast<swg_peak*>(c->bpeaks.p);
    }
  }
  for (int f = 0; f < n_frames; ++f)
    if (!frames[f]) return fail(SWG_ERR_ARG, "NULL frame %d", f);
  // Frames round-robin over up to kWorkers table sets (this one + clones of
  // its geometry, made on first use) on the context's worker streams: the
  // build of one frame overlaps the sweeps of another.  Each frame's calls
  // run on its worker stream with that worker's scratch; the caller's stream
  // forks to the workers first and joins them at the end (graph-capturable).
  const int K = std::min(n_frames, (int)swg_ctx::kWorkers);
  swg_tables* sets[swg_ctx::kWorkers] = {t};
  for (int k = 1; k < K; ++k) {
    if (!t->clone[k - 1])
      ST_TRY(build_common(c, frames[k], is_device, pitch_bytes, t->w, t->h, t->format,
                          t->levels, t->planes, t->decay, t->bin0, t->bin0 + t->bins, 0,
                          &t->clone[k - 1]));
    sets[k] = t->clone[k - 1];
  }
  // K table sets build at once on the worker streams, so each needs only a
  // share of the SMs: fewer, taller bands (less carry work per frame;
  // config 3, 8 sets of 310 x 330 regions: 3.73 -> 3.32 ms per step with a
  // quarter of the default band count, an eighth the same; a single frame
  // is fastest on the default split).  The default split returns on exit.
  if (K > 1)
    for (int k = 0; k < K; ++k) split_bands(sets[k], SWG_BAND_TARGET / (K >= 4 ? 4 : 2));
  const cudaStream_t orig = c->stream;
  struct Restore {  // the caller's stream and the context defaults, on every exit
    swg_ctx* c;
    cudaStream_t s;
    swg_tables** sets;
    int K;
    ~Restore() {
      c->stream = s;
      c->slot = 0;
      c->fanout_off = false;
      for (int k = 0; k < K; ++k) split_bands(sets[k], SWG_BAND_TARGET);
    }
  } restore{c, orig, sets, K};
  {
    DeviceGuard g(c->device);
    CUDA_TRY(cudaEventRecord(c->fork, orig));
    for (int k = 0; k < K; ++k) {
      CUDA_TRY(cudaStreamWaitEvent(c->work[k], c->fork, 0));
      // scratch slot k may still feed an asynchronous call's map copies
      if (c->free_ev[k]) CUDA_TRY(cudaStreamWaitEvent(c->work[k], c->free_ev[k], 0));
    }
  }
  c->fanout_off = true;
  for (int f = 0; f < n_frames; ++f) {
    const int k = f % K;
    c->stream = c->work[k];
    c->slot = k;
    ST_TRY(swg_tables_rebuild_for(sets[k], frames[f], is_device, pitch_bytes, n, reqs));
    ST_TRY(swg_likelihood_maps(sets[k], n, reqs, nullptr, nullptr, nullptr,
                               dst + (size_t)f * n));
  }
  c->stream = orig;
  {
    DeviceGuard g(c->device);
    for (int k = 0; k < K; ++k) {
      CUDA_TRY(cudaEventRecord(c->join[k], c->work[k]));
      CUDA_TRY(cudaStreamWaitEvent(orig, c->join[k], 0));
    }
  }
  if (peaks_host) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    CUDA_TRY(cudaMemcpyAsync(peaks_host, dst, (size_t)n_frames * n * sizeof(swg_peak),
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  return SWG_OK;
}

swg_status swg_decay_windows(swg_tables* t, int n, const int* cx, const int* cy,
                             const swg_kernel* k, double* out) {
  ST_TRY(check_tables(t));
  if (n < 0 || !k || (n && (!cx || !cy || !out))) return fail(SWG_ERR_ARG, "bad query arguments");
  ST_TRY(validate_kernel(*k));
  if (!t->tdec || k->kind != SWG_KERNEL_EXP_L1 || k->sigma != t->decay)
    return fail(SWG_ERR_UNSUPPORTED_KERNEL,
                "decay windows: exponential kernel with the tables' decay on decayed tables");
  for (int i = 0; i < n; ++i)
    ST_TRY(validate_window(t->w, t->h, cx[i], cy[i], *k, SWG_BORDER_STRICT));
  if (n == 0) return SWG_OK;
  swg_map_request r{};
  r.sim = SWG_SIM_BHATTACHARYYA;
  static thread_local ExpSweep es;
  exp_plan(t, r, k_hx(*k), k_hy(*k), es);
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  ST_TRY(fresh_all(t));
  swg_ctx* c = t->ctx;
  const size_t cb = round_up((size_t)n * 4, 256), ob = (size_t)n * t->bins * 8;
  ST_TRY(c->terms.ensure(2 * cb));
  ST_TRY(c->qout.ensure(ob));
  int* dcx = static_cast<int*>(c->terms.p);
  int* dcy = reinterpret_cast<int*>(static_cast<char*>(c->terms.p) + cb);
  CUDA_TRY(cudaMemcpyAsync(dcx, cx, (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(dcy, cy, (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_exp_query(t->tdec, t->ps, t->pitch, t->bins, es, n, dcx, dcy,
                            static_cast<double*>(c->qout.p), c->stream));
  c->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(out, c->qout.p, ob, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SWG_OK;
}

// Boundary prefix-row exchange on the device: the band's last
// record row of the 32-bit planes (k_last_row), and the carry that turns a
// band's local tables into the global ones (k_add_carry).
swg_status swg_tables_last_row(swg_tables* t, void* dev_out) {
  ST_TRY(check_tables(t));
  if (!dev_out) return fail(SWG_ERR_ARG, "NULL output");
  if (t->tdec) return fail(SWG_ERR_CONFIG, "decay tables hold no integral planes");
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  ST_TRY(ensure_t32(t));
  ST_TRY(fresh_all(t));
  const int kinds = t->planes;
  CUDA_TRY(launch_last_row(t->t32, t->ps, t->pitch, t->planes, kinds, t->w, t->h, t->groups,
                           dev_out, t->ctx->stream));
  t->ctx->launches += 1;
  return SWG_OK;
}

swg_status swg_tables_add_carry(swg_tables* t, int y0, const void* dev_carry) {
  ST_TRY(check_tables(t));
  if (!dev_carry) return fail(SWG_ERR_ARG, "NULL carry");
  if (t->tdec) return fail(SWG_ERR_CONFIG, "decay tables hold no integral planes");
  if (y0 < 0) return fail(SWG_ERR_OUT_OF_RANGE, "band origin %d", y0);
  if (t->carried) return fail(SWG_ERR_CONFIG, "tables already carry a boundary prefix row");
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  DeviceGuard g(t->ctx->device);
  ST_TRY(ensure_t32(t));
  ST_TRY(fresh_all(t));
  CUDA_TRY(launch_add_carry(t->t32, t->ps, t->pitch, t->planes, t->planes, t->w, t->h,
                            t->groups, y0, dev_carry, t->ctx->stream));
  t->ctx->launches += 1;
  t->carried = true;
  t->carry_y0 = y0;
  return SWG_OK;
}

}  // extern "C"
