// store_bw.cu -- write-bandwidth ceiling of the IH builds' store pattern.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o store_bw store_bw.cu
//   ./store_bw
// Every warp owns one (band, plane) unit of a table of `planes` planes of
// (H+1) rows x pitch 16-byte records and writes its band's rows in 256-record
// (4 KB) segments, strip by strip -- the decayed build's pattern, no compute.
// Variants: per-lane 16-byte stores (512 B per warp instruction), TMA tensor
// stores (4-D map, 128-byte lines, SWIZZLE_128B: the builds' form), 1-D bulk
// stores (cp.async.bulk of 4 KB); each with the first data record at byte
// offset `off` of a 128-byte line (the tables put record 1 at offset 16).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

struct Args {
  CUtensorMap tmap;
  char* base;      // record 0 of row 0 of plane 0
  size_t pitch;    // records per row
  size_t ps;       // records per plane
  int w, h, band_h, nbands, planes;
};

constexpr int kRows = 3;

template <int MODE>  // 0 lane stores, 1 TMA tensor, 2 bulk 1-D
__global__ void __launch_bounds__(256, 2) k_store(const __grid_constant__ Args g) {
  extern __shared__ __align__(1024) uint4 s_buf[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long unit = (long long)blockIdx.x * 8 + warp;
  if (unit >= (long long)g.nbands * g.planes) return;
  const int plane = (int)(unit % g.planes), band = (int)(unit / g.planes);
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  uint4* buf = s_buf + warp * kRows * 256;
  for (int i = lane; i < kRows * 256; i += 32) buf[i] = make_uint4(i, lane, warp, 1);
  __syncwarp();
  if (MODE != 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  int slot = 0;
  for (int x0 = 0; x0 < g.w; x0 += 256) {
    for (int y = y0; y < y1; ++y) {
      char* row = g.base + (((size_t)plane * g.ps + (size_t)(y + 1) * g.pitch) + x0 + 1) * 16;
      if (MODE == 0) {
        uint4* out = reinterpret_cast<uint4*>(row);
#pragma unroll
        for (int m = 0; m < 8; ++m)
          if (x0 + m * 32 + lane < g.w) out[m * 32 + lane] = make_uint4(x0, y, m, lane);
      } else {
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kRows - 1) : "memory");
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf + slot * 256);
          if (MODE == 1) {
            asm volatile(
                "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                ::"l"(&g.tmap), "r"(0), "r"(x0 / 8), "r"(y + 1), "r"(plane), "r"(sa)
                : "memory");
          } else {
            const int n = min(256, g.w - x0) * 16;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(row),
                         "r"(sa), "r"(n)
                         : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        __syncwarp();
        slot = slot + 1 == kRows ? 0 : slot + 1;
      }
    }
  }
  if (MODE != 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// CTA per unit: warp w writes strip w of every row (the CTA's stores cover a
// whole row: contiguous 32 KB per row instead of 8 strips visited in turn).
template <int SEG>  // records per warp segment
__global__ void __launch_bounds__(256, 2) k_store_row(const __grid_constant__ Args g) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long unit = blockIdx.x;
  const int plane = (int)(unit % g.planes), band = (int)(unit / g.planes);
  const int y0 = band * g.band_h, y1 = min(y0 + g.band_h, g.h);
  for (int xs = 0; xs < g.w; xs += 8 * SEG) {
    const int x0 = xs + warp * SEG;
    for (int y = y0; y < y1; ++y) {
      uint4* out = reinterpret_cast<uint4*>(
          g.base + (((size_t)plane * g.ps + (size_t)(y + 1) * g.pitch) + x0 + 1) * 16);
#pragma unroll
      for (int m = 0; m < SEG / 32; ++m)
        if (x0 + m * 32 + lane < g.w) out[m * 32 + lane] = make_uint4(x0, y, m, lane);
    }
  }
}

int main() {
  const int w = 2048, h = 2048, planes = 13 * 4, nbands = 37;
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  for (int off : {16, 32, 0}) {  // byte offset of record 1 within a 128-byte line
    for (int pmul : {4}) {  // pitch a multiple of 4 or 8 records (64 / 128 bytes)
      const size_t pitch = ((size_t)w + 1 + 8 + pmul - 1) / pmul * pmul;
      const size_t ps = pitch * (h + 1);
      const size_t bytes = ps * planes * 16 + 4096;
      char* raw;
      if (cudaMalloc(&raw, bytes) != cudaSuccess) return 1;
      // record 1 at (128-byte boundary + off): record 0 sits 16 bytes below
      char* base = raw + 128 + off - 16;
      Args a{};
      a.base = base; a.pitch = pitch; a.ps = ps; a.w = w; a.h = h; a.planes = planes;
      a.band_h = (h + nbands - 1) / nbands; a.nbands = (h + a.band_h - 1) / a.band_h;
      const cuuint64_t dims[4] = {32, (cuuint64_t)((size_t)w * 16 / 128), (cuuint64_t)h + 1,
                                  (cuuint64_t)planes};
      const cuuint64_t strides[3] = {128, pitch * 16, ps * 16};
      const cuuint32_t box[4] = {32, 32, 1, 1}, es[4] = {1, 1, 1, 1};
      const bool tm = enc && enc(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, base + 16, dims, strides,
                                 box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      const long long units = (long long)a.nbands * planes;
      const unsigned grid = (unsigned)((units + 7) / 8);
      const size_t sm = 8 * kRows * 4096;
      const double gb = (double)w * h * planes * 16 / 1e9;
      for (int mode = 0; mode < 3; ++mode) {
        if (mode == 1 && !tm) continue;
        if (mode == 2 && (off % 16 || (pitch * 16) % 16)) continue;
        auto launch = [&] {
          if (mode == 0) k_store<0><<<grid, 256, sm>>>(a);
          else if (mode == 1) k_store<1><<<grid, 256, sm>>>(a);
          else k_store<2><<<grid, 256, sm>>>(a);
        };
        cudaFuncSetAttribute(k_store<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(k_store<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(k_store<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        float best = 1e9f;
        for (int rep = 0; rep < 6; ++rep) {
          cudaMemsetAsync(flush, rep, 256 << 20);
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0); cudaEventCreate(&e1);
          cudaEventRecord(e0);
          launch();
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep) best = ms < best ? ms : best;
          cudaEventDestroy(e0); cudaEventDestroy(e1);
        }
        const cudaError_t e = cudaGetLastError();
        printf("offset %2d pitch%%%d mode %s: %.3f ms, %.0f GB/s%s\n", off, pmul,
               mode == 0 ? "lane-st " : mode == 1 ? "tma-4d  " : "bulk-1d ", best, gb / best * 1e3,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
      for (int v = 0; v < 2; ++v) {
        float best = 1e9f;
        for (int rep = 0; rep < 6; ++rep) {
          cudaMemsetAsync(flush, rep, 256 << 20);
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0); cudaEventCreate(&e1);
          cudaEventRecord(e0);
          if (v == 0) k_store_row<256><<<(unsigned)units, 256>>>(a);
          else k_store_row<128><<<(unsigned)units, 256>>>(a);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep) best = ms < best ? ms : best;
          cudaEventDestroy(e0); cudaEventDestroy(e1);
        }
        printf("offset %2d pitch%%%d mode cta-row %d: %.3f ms, %.0f GB/s\n", off, pmul,
               v == 0 ? 256 : 128, best, gb / best * 1e3);
      }
      cudaFree(raw);
    }
  }
  return 0;
}
