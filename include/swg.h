/*
 * swg.h — C-ABI of the B200-native SWIH hot path (libswg.so).
 *
 * Plain C: opaque handles, POD structs, pointers + sizes, int status codes.
 * No exceptions, no torch types.  Every entry point below replaces one body
 * of the reference C++ library (paths relative to /root/reference/proj):
 *
 *   swg_tables_build        IntegralTableSet::build      src/integral_tables.cpp:72-115
 *                           (+ quantize_image            src/image.cpp:34-40, fused)
 *   swg_tables_export_i64   IntegralTableSet::cell/plane include/swih/integral_tables.hpp:69-101
 *                           and ::save                   src/integral_tables.cpp:167-183
 *   swg_tables_upload_i64   IntegralTableSet::load       src/integral_tables.cpp:185-206
 *   swg_query_terms         accumulate_term / swih_query_into / quadrant_histogram /
 *                           plain_local_histogram_into   src/engine.cpp:39-165
 *   swg_likelihood_map      likelihood_map               src/matching.cpp:108-209
 *                           (score_counts/score_weights  src/matching.cpp:20-52,
 *                            WeddingCakePlan::histogram_into src/baselines.cpp:133-149,
 *                            BruteForcePlan             src/baselines.cpp:24-69)
 *                           and peak                     src/matching.cpp:211-223
 *
 * Error behaviour: one status code per reference exception class
 * (include/swih/errors.hpp:10-79); the message is kept per thread
 * (swg_last_error) together with CapacityError::required_bytes
 * (swg_last_required_bytes).  The C++ drop-in layer (include/swih/ headers)
 * rethrows the matching class.
 *
 * Threading: a context owns one CUDA stream on one device; calls on one
 * context are serialised by the caller (the C++ layer holds a mutex).
 * Tables are immutable after build and may be queried from any thread.
 */
#ifndef SWG_H
#define SWG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWG_ABI_VERSION 1
#define SWG_MAX_BINS 1024  /* model / bin count limit of one map request   */
#define SWG_MAX_RINGS 512  /* wedding-cake ring limit of one map request   */

typedef enum swg_status {
  SWG_OK = 0,
  SWG_ERR = 1,                   /* swih::Error                  */
  SWG_ERR_IO = 2,                /* swih::IoError                */
  SWG_ERR_ZERO_MASS = 3,         /* swih::ZeroMassError          */
  SWG_ERR_INVALID_KERNEL = 4,    /* swih::InvalidKernelError     */
  SWG_ERR_OUT_OF_RANGE = 5,      /* swih::OutOfRangeError        */
  SWG_ERR_UNSUPPORTED_KERNEL = 6,/* swih::UnsupportedKernelError */
  SWG_ERR_WINDOW_OOB = 7,        /* swih::WindowOutOfBoundsError */
  SWG_ERR_CAPACITY = 8,          /* swih::CapacityError          */
  SWG_ERR_CONFIG = 9,            /* swih::ConfigError            */
  SWG_ERR_MODEL = 10,            /* swih::ModelError             */
  SWG_ERR_SIZE = 11,             /* swih::SizeError              */
  SWG_ERR_CUDA = 64,             /* device / runtime failure     */
  SWG_ERR_NO_DEVICE = 65,        /* no usable sm_100 device      */
  SWG_ERR_ARG = 66               /* NULL handle / bad enum value */
} swg_status;

/* Input pixel formats.  GRAY8 + bins is the reference Quantizer
 * (image.hpp:43-45).  BINS16 is a pre-quantised FeatureImage
 * (image.hpp:52-76).  GRAY16 / RGB8 are declared extensions. */
typedef enum swg_format {
  SWG_FMT_GRAY8 = 0,  /* uint8,  bin = v*bins/256                       */
  SWG_FMT_GRAY16 = 1, /* uint16, bin = v*bins/65536                     */
  SWG_FMT_RGB8 = 2,   /* 3 x uint8, bins = levels^3                     */
  SWG_FMT_BINS16 = 3  /* uint16 bin index per pixel, < bins             */
} swg_format;

/* Weight-plane sets.  PLAIN = {1}; AFFINE = {1, x, y}, the reference's
 * plain / xramp / yramp tables (integral_tables.hpp:53-58). */
typedef enum swg_planes {
  SWG_PLANES_PLAIN = 1,
  SWG_PLANES_AFFINE = 3,
  SWG_PLANES_QUADRATIC = 5, /* {1, x, y, x^2, y^2}, uint32 (EUCLID_QUAD maps) */
  SWG_PLANES_DECAY = 4      /* SE/SW/NE/NW decayed tables, fp64 (EXP_L1 maps);
                               built by swg_tables_build_decay          */
} swg_planes;

typedef enum swg_table_kind { SWG_TABLE_PLAIN = 0, SWG_TABLE_XRAMP = 1, SWG_TABLE_YRAMP = 2 } swg_table_kind;
typedef enum swg_kernel_kind {      /* kernel.hpp:9-14, then declared extensions */
  SWG_KERNEL_UNIFORM = 0,
  SWG_KERNEL_MANHATTAN = 1,
  SWG_KERNEL_CHEBYSHEV = 2,
  SWG_KERNEL_GAUSS_CHEBYSHEV = 3,
  /* Declared extensions (no reference implementation):       */
  SWG_KERNEL_EUCLID_QUAD = 4, /* w = 2(hx+1)^2(hy+1)^2 - dx^2(hy+1)^2 - dy^2(hx+1)^2,
                                 exact on SWG_PLANES_QUADRATIC tables   */
  SWG_KERNEL_EXP_L1 = 5       /* w = sigma^(|dx|+|dy|), sigma in (0,1) = decay per pixel;
                                 O(1) on SWG_PLANES_DECAY tables built with that sigma */
} swg_kernel_kind;
typedef enum swg_method { SWG_METHOD_SWIH = 0, SWG_METHOD_BRUTE = 1, SWG_METHOD_CAKE = 2, SWG_METHOD_PLAIN = 3 } swg_method;
typedef enum swg_similarity { SWG_SIM_BHATTACHARYYA = 0, SWG_SIM_INTERSECTION = 1 } swg_similarity;
typedef enum swg_border { SWG_BORDER_STRICT = 0, SWG_BORDER_CLIPPED = 1 } swg_border;
typedef enum swg_ring_rule { SWG_RING_MEAN = 0, SWG_RING_LEVEL = 1 } swg_ring_rule;

typedef struct swg_ctx swg_ctx;
typedef struct swg_tables swg_tables;

typedef struct swg_kernel {   /* KernelSpec, kernel.hpp:18-36 */
  int kind;
  int kw;
  int kh;
  double sigma;
} swg_kernel;

typedef struct swg_peak {     /* Peak, matching.hpp:41-47 */
  int map_x;
  int map_y;
  int center_x;
  int center_y;
  double score;
} swg_peak;

/* One likelihood-map request (likelihood_map arguments + MatchOptions,
 * matching.hpp:49-54,72-75).  Map rows [row_begin, row_end) only; 0,0 means
 * the whole strict map.  `model` holds `bins` normalised doubles. */
typedef struct swg_map_request {
  swg_kernel kernel;
  int method;      /* swg_method                         */
  int sim;         /* swg_similarity                     */
  int rings;       /* WeddingCakeConfig::rings (CAKE)     */
  int ring_rule;   /* WeddingCakeConfig::rule  (CAKE)     */
  int row_begin;
  int row_end;
  const double* model;
  /* Bin-range chains (SURVEY 8e "bin ranges"; NULL = off).  Tables built
   * for bins [b0, b1) of B (swg_tables_build_bins) add their bins to a
   * window's running Bhattacharyya sum and mass in bin order, so a chain of
   * ranges 0 -> G-1 reproduces the single-table operation sequence bit for
   * bit.  Device arrays of (row_end-row_begin) x map_width {s, mass} pairs:
   *   partial_in   running sums over bins [0, b0) (NULL: start at zero);
   *   partial_out  when non-NULL, receives the sums over [0, b1) and the
   *                request produces no scores and no peak;
   * the last range (partial_in set, partial_out NULL) finishes the scores,
   * the map and the peak.  `model` is always the full B-bin model.
   * Bhattacharyya on every table sweep; intersection on swih Manhattan /
   * Uniform / Euclidean (closed-form window mass). */
  const void* partial_in;
  void* partial_out;
} swg_map_request;

/* One quadrant term of a window query (QuadrantTerm, engine.hpp:27-32). */
typedef struct swg_term {
  int valid;       /* 0 = empty quadrant (std::nullopt) */
  int x0, y0, x1, y1;
  int64_t sx, sy, beta;
} swg_term;

/* ---- library / errors ---------------------------------------------- */
int swg_abi_version(void);
const char* swg_last_error(void);
size_t swg_last_required_bytes(void);
swg_status swg_device_count(int* n);

/* Page-locked, device-mapped host memory (portable across devices): fast
 * asynchronous copies, and host maps the sweeps write directly. */
swg_status swg_host_alloc(size_t bytes, void** out);
swg_status swg_host_free(void* p);
/* Peer memory between processes (one process per GPU): export a device
 * allocation's handle, map another process's allocation into this one.  A
 * mapped pointer can be given to a kernel output directly -- e.g. as
 * swg_map_request.partial_out, so a bin-range sweep writes its running sums
 * straight into the next GPU's input buffer over NVLink. */
#define SWG_IPC_HANDLE_BYTES 64
swg_status swg_device_alloc(size_t bytes, void** out);  /* exportable (whole allocation) */
swg_status swg_device_free(void* p);
swg_status swg_ipc_export(const void* dev_ptr, unsigned char* handle);
swg_status swg_ipc_import(const unsigned char* handle, void** dev_ptr);
swg_status swg_ipc_close(void* dev_ptr);

/* ---- context --------------------------------------------------------- */
/* Contexts are reference counted by the tables built on them: destroying a
 * context with live tables defers the release to the last table. */
swg_status swg_ctx_create(int device, swg_ctx** out);
swg_status swg_ctx_destroy(swg_ctx* ctx);
swg_status swg_ctx_synchronize(swg_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores
 * the context's own stream. */
swg_status swg_ctx_set_stream(swg_ctx* ctx, void* cuda_stream);
/* Number of kernels this context launched so far (bench evidence). */
swg_status swg_ctx_launch_count(swg_ctx* ctx, uint64_t* n);
/* Device-to-host copies of host maps issued so far (maps written zero-copy
 * into page-locked host memory issue none). */
swg_status swg_ctx_map_copy_count(swg_ctx* ctx, uint64_t* n);

/* ---- integral tables ------------------------------------------------- */
/* Quantise + build one plane set.  `pixels` is host memory
 * (is_device = 0) or device memory (1), rows `pitch_bytes` apart (0 = tight).
 * `bins` is the bin count (GRAY8 / GRAY16 / BINS16) or the levels per
 * channel (RGB8, bins = levels^3).  memory_budget = 0: no limit.
 * CapacityError semantics: SWG_ERR_CAPACITY + swg_last_required_bytes(). */
swg_status swg_tables_build(swg_ctx* ctx, const void* pixels, int is_device,
                            size_t pitch_bytes, int width, int height,
                            int format, int bins, int planes,
                            size_t memory_budget, swg_tables** out);
/* Decayed directional tables for the exponential kernel with per-pixel
 * decay `decay` in (0, 1) (declared extension): E(X,Y) = sum over x<X, y<Y
 * of [bin] decay^(X-1-x) decay^(Y-1-y), for the image and its horizontal,
 * vertical and double flip.  EXP_L1 maps with sigma == decay run in O(1) per
 * window and bin; their peak is made exact by an fp64 brute-force re-score
 * of every window whose fast score is within a derived error bound of
 * the fast maximum. */
swg_status swg_tables_build_decay(swg_ctx* ctx, const void* pixels, int is_device,
                                  size_t pitch_bytes, int width, int height, int format,
                                  int bins, double decay, size_t memory_budget,
                                  swg_tables** out);
/* Tables for the bin range [bin_begin, bin_end) of the quantiser's bins
 * (bin-range sharding: one range per GPU, partial sums chained through
 * swg_map_request.partial_in / partial_out).  planes as swg_tables_build,
 * or SWG_PLANES_DECAY with `decay`; bin_begin = bin_end = 0: every bin.
 * Window queries and exports address local bins 0 .. bin_end-bin_begin-1. */
swg_status swg_tables_build_bins(swg_ctx* ctx, const void* pixels, int is_device,
                                 size_t pitch_bytes, int width, int height, int format,
                                 int bins, int planes, double decay, int bin_begin,
                                 int bin_end, size_t memory_budget, swg_tables** out);
swg_status swg_tables_bin_range(const swg_tables* t, int* bin_begin, int* bin_end,
                                int* total_bins);
/* Rebuild every plane set for the bin range [bin_begin, bin_begin + bins)
 * of the same width: from `pixels` (uploaded and quantised as in
 * swg_tables_rebuild) or, with pixels = NULL, from the resident feature
 * image -- one GPU walks a large bin set range by range, chaining partial
 * sums.  (swg_tables_rebuild keeps the current range.) */
swg_status swg_tables_rebuild_bins(swg_tables* t, const void* pixels, int is_device,
                                   size_t pitch_bytes, int bin_begin);
/* Re-run quantise + build for a new frame of the same geometry into the
 * same device buffers (no allocation; stream ordered, asynchronous). */
swg_status swg_tables_rebuild(swg_tables* t, const void* pixels, int is_device,
                              size_t pitch_bytes);
/* Create tables from exact int64 host planes (SWIH1 load path); each array
 * holds bins*(w+1)*(h+1) entries, bin-major, row stride w+1. */
swg_status swg_tables_upload_i64(swg_ctx* ctx, int width, int height, int bins,
                                 const int64_t* plain, const int64_t* xramp,
                                 const int64_t* yramp, swg_tables** out);
swg_status swg_tables_destroy(swg_tables* t);
swg_status swg_tables_info(const swg_tables* t, int* width, int* height,
                           int* bins, int* planes, size_t* device_bytes);
/* Exact int64 planes for bins [bin_begin, bin_end), reference layout. */
swg_status swg_tables_export_i64(swg_tables* t, int kind, int bin_begin,
                                 int bin_end, int64_t* host_out);
/* The stored 32-bit words (exact value mod 2^32), reference layout. */
swg_status swg_tables_export_u32(swg_tables* t, int kind, int bin_begin,
                                 int bin_end, uint32_t* host_out);
/* Decay tables only: copy decayed planes [b0, b1) of orientation `kind`
 * (0 SE = image, 1 horizontal flip, 2 vertical flip, 3 both) to host
 * memory as b1-b0 planes of (height+1) x (width+1) doubles, zero row and
 * column 0 (in the flipped image's own coordinates). */
swg_status swg_tables_export_f64(swg_tables* t, int kind, int b0, int b1,
                                 double* host_out);
/* The quantised feature image (uint16 bins, w*h). */
swg_status swg_tables_feature_image(swg_tables* t, uint16_t* host_out);
/* Device pointer + geometry of the 32-bit planes (for tests / bench); of
 * the fp64 decayed planes (kinds 0..3 = SE, h-flip, v-flip, hv-flip) for
 * decay tables.
 * Bins are tiled in records of 8 ("bin octets"): element (x, y) of bin b,
 * table kind k sits at
 *   base[(((b/8)*planes + k)*plane_stride + y*pitch + x)*8 + b%8]
 * with plane_stride and pitch counted in records (planes of 16-byte
 * records -- the fp64 pairs here -- start 16 bytes past an allocation
 * boundary, so record 1 of every row is 32-byte aligned).  Units a model-driven
 * rebuild (swg_tables_rebuild_for) skipped are built before this returns. */
swg_status swg_tables_device_layout(const swg_tables* t, const void** base,
                                    size_t* plane_stride, size_t* pitch,
                                    int* bins_per_record);

/* ---- window queries (engine API) ----------------------------------- */
/* n windows, each `terms_per_window` consecutive terms (already clipped by
 * the caller per the border policy).  out[n][bins] = sum over the window's
 * terms of sx*X + sy*Y + beta*P per bin, exact int64. */
swg_status swg_query_terms(swg_tables* t, int n, int terms_per_window,
                           const swg_term* terms, int64_t* host_out);

/* Window queries at centres (cx[i], cy[i]) with the reference semantics of
 * swih_query_into (method SWIH, engine.cpp:140-147) or
 * plain_local_histogram_into (method PLAIN, engine.cpp:156-165), border
 * policy per engine.cpp:7-35.  out[n][bins] exact int64. */
swg_status swg_query_windows(swg_tables* t, int n, const int* cx, const int* cy,
                             const swg_kernel* kernel, int method, int border,
                             int64_t* host_out);
/* Wedding-cake histograms (WeddingCakePlan, baselines.cpp:84-149) at n
 * centres; out[n][bins] doubles, bit-identical to the reference. */
swg_status swg_cake_windows(swg_tables* t, int n, const int* cx, const int* cy,
                            const swg_kernel* kernel, int rings, int ring_rule,
                            int border, double* host_out);
/* Boundary prefix-row exchange on the device (SURVEY 8e "row bands"): a
 * band built from pixel rows [y0, y0+h) holds local tables (zero at its row
 * 0).  swg_tables_last_row writes its last record row of every 32-bit plane
 * -- planes x octets x (width+1) records of 8 uint32 bins, record order
 * (octet, plane, x) -- to device memory; all-gather those rows (NCCL over
 * NVLink), form the carry = exclusive sum over the earlier bands of their
 * rows (each already global), and swg_tables_add_carry(t, y0, carry) turns
 * the band's 32-bit planes into the GLOBAL tables' rows y0 .. y0+h (mod
 * 2^32, like the tables).  Sweeps on carried tables use global rows.  The
 * exact int64 export of a carried table is refused (SWG_ERR_CONFIG). */
swg_status swg_tables_last_row(swg_tables* t, void* dev_out);
swg_status swg_tables_add_carry(swg_tables* t, int y0, const void* dev_carry);

/* Declared exponential kernel (EXP_L1, sigma == the tables' decay) on
 * decayed tables (swg_tables_build_decay): weighted window histograms at
 * strict centres from the sweep's 16 corners per bin, out[n][bins] doubles
 * (tolerance-exact: the brute force sums the same weights in pixel order,
 * baselines.cpp:53-69). */
swg_status swg_decay_windows(swg_tables* t, int n, const int* cx, const int* cy,
                             const swg_kernel* kernel, double* host_out);
/* Ring plan of a wedding-cake configuration: per ring the box half extents
 * and the ring weight (WeddingCakePlan::shrink_x/shrink_y/ring_weight). */
swg_status swg_cake_plan(const swg_kernel* kernel, int rings, int ring_rule,
                         int* shrink_x, int* shrink_y, double* ring_weight);

/* Quantise an image on the device (quantize_image, image.cpp:34-40, and
 * the declared uint16 / RGB forms); out: w*h uint16 bins. */
swg_status swg_quantize(swg_ctx* ctx, const void* pixels, int width, int height,
                        int format, int bins, uint16_t* host_out);
/* Brute-force weighted histograms of a host feature image at n centres
 * (BruteForcePlan::counts_into / weights_into, baselines.cpp:24-69):
 * integer kernels -> exact int64 counts in out_i64 (out_f64 may be NULL);
 * any kernel -> fp64 sums in row-major pixel order in out_f64. */
swg_status swg_brute_windows(swg_ctx* ctx, const uint16_t* fi, int width, int height,
                             int bins, int n, const int* cx, const int* cy,
                             const swg_kernel* kernel, int border, int64_t* out_i64,
                             double* out_f64);
/* Peak of a host likelihood map (peak, matching.cpp:211-223). */
swg_status swg_map_peak(swg_ctx* ctx, const double* scores, int map_width,
                        int map_height, int hx, int hy, swg_peak* out);

/* ---- likelihood maps ------------------------------------------------- */
/* Full strict likelihood map(s) + peak(s).  For request i:
 *   scores_host[i]   host array of rows x map_width doubles, or NULL
 *   scores_dev[i]    device array (same size), or NULL
 *   peaks_host[i]    filled when peaks_host != NULL
 *   peaks_dev        device array of n swg_peak, or NULL
 * With only device outputs the call is asynchronous on the context stream:
 * the requests fork from it onto the context's worker streams (their sweeps
 * overlap) and join back into it before the call returns, so work queued on
 * the context stream afterwards sees every output (graph-capturable).  In
 * a call of at most three requests, a host map in page-locked,
 * device-mapped memory (swg_host_alloc, cudaMallocHost, cudaHostRegister)
 * is written by the sweep directly; other host maps -- and every host map
 * of a call with more requests -- are copied (up to three requests overlap
 * on prioritised streams, each map copied as its sweep ends; more run in
 * order, each map copied by the copy engine while the next one sweeps).
 * The call returns when the host outputs are filled
 * (swg_likelihood_maps_async: when the context is synchronised).  Any of
 * the per-request pointer arrays may itself be NULL. */
swg_status swg_likelihood_maps(swg_tables* t, int n,
                               const swg_map_request* reqs,
                               double* const* scores_host,
                               double* const* scores_dev,
                               swg_peak* peaks_host, swg_peak* peaks_dev);

/* swg_tables_rebuild for a known set of requests: quantise the new frame,
 * then build only the table units those requests read -- bin octets of the
 * 32-bit planes (Manhattan / Euclidean sweeps) or bin pairs of the decay
 * planes (exponential sweep) holding a nonzero model value; a model's zero
 * bins contribute +0 to every score, so those sweeps never read them
 * (SWG_SPARSE=0: every unit).  The other units are marked stale and built
 * on first use by any later call (maps with other models, exports, window
 * queries, device layout), so the tables' contents are never observably
 * incomplete.  Plain-only (16-bit) tables and bin-range tables build fully.
 * reqs are the swg_likelihood_maps requests that will follow. */
swg_status swg_tables_rebuild_for(swg_tables* t, const void* pixels, int is_device,
                                  size_t pitch_bytes, int n, const swg_map_request* reqs);
/* Plane bytes written by the builds since the last rebuild began
 * (measurement: the IH-build GB/s). */
swg_status swg_tables_built_bytes(const swg_tables* t, size_t* bytes);

/* What swg_likelihood_maps would run for one request (measurement and
 * tests; no device work): the sweep kernel's name, the table planes it reads,
 * bytes per table entry, and how many bins' records it reads (a model's zero
 * bins are skipped by the sweeps whose window mass is closed-form: affine,
 * quadratic, exponential; SWG_SPARSE=0 reads every bin), and its CTA count. */
typedef struct swg_plan_info {
  char kernel[32];
  int planes;
  int entry_bytes;
  int bins_read;
  int ctas;
} swg_plan_info;
swg_status swg_request_plan(const swg_tables* t, const swg_map_request* r, swg_plan_info* out);

/* Which requests of one swg_likelihood_maps call share a launch (no device
 * work): group_of[i] = the multi-scale cake launch request i joins, or -1
 * when it runs on its own.  A call's full-ring square GaussianChebyshev /
 * cake requests (Bhattacharyya, whole map, all bins of the table) on the
 * 16-bit plain planes are swept together, up to SWG_CAKE_MULTI scales per
 * launch, largest half-extents first: every scale's ring boxes are the
 * boxes of half-extent h .. 0 around the window centre, loaded once for all
 * of them (WeddingCakePlan::histogram_into, baselines.cpp:139-148, per
 * scale, bit for bit). */
swg_status swg_request_groups(const swg_tables* t, int n, const swg_map_request* reqs,
                              int* group_of);

/* swg_likelihood_maps without the final host synchronisation: the call
 * enqueues the builds' consumers, sweeps and map copies and returns; host
 * maps and host peaks are filled once swg_ctx_synchronize returns.  Successive
 * asynchronous calls rotate over the context's scratch slots, so one table
 * set's map copies overlap the next set's sweeps (a frame's units run back to
 * back).  The caller keeps the request array, models and host buffers alive
 * until the synchronisation. */
swg_status swg_likelihood_maps_async(swg_tables* t, int n, const swg_map_request* reqs,
                                     double* const* scores_host, double* const* scores_dev,
                                     swg_peak* peaks_host, swg_peak* peaks_dev);

/* Batch of frames of the tables' geometry (tracking sequences, config 3):
 * for each frame f, rebuild the tables from frames[f] (pitch_bytes, host or
 * device as is_device; a search-region crop is a pointer into the full frame
 * plus the full frame's pitch) and run the n requests, peaks only.  Peak of
 * frame f, request i -> [f * n + i] of peaks_dev (device, asynchronous)
 * and/or peaks_host (filled on return).  Frames round-robin over up to
 * eight table sets of this geometry (`t` plus up to seven the library
 * creates on first use and frees with `t`) on the context's worker streams, so one
 * frame's build overlaps another's sweeps; the call forks from and joins
 * back to the context stream (graph-capturable with device outputs).  Not
 * to be called concurrently with other calls on the same context. */
swg_status swg_likelihood_batch(swg_tables* t, int n_frames, const void* const* frames,
                                int is_device, size_t pitch_bytes, int n,
                                const swg_map_request* reqs, swg_peak* peaks_host,
                                swg_peak* peaks_dev);

#ifdef __cplusplus
}
#endif
#endif /* SWG_H */
