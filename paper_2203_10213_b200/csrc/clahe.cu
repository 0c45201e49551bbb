// clahe.cu — CLAHE-3D on the B200 (pkg/src/vkt/ops/filters.py:98-245).
//
// Two device passes around a tiny host step:
//   1. vkt_clahe_histograms: every cell's bin index (u8/u16: a host-built
//      lookup table evaluated with numpy's float64 rule; f32: the same float64
//      expression on the device) is counted into its brick's histogram —
//      shared-memory histograms per CTA, merged with integer atomics, so the
//      counts are exact and order-independent (filters.py:188-196).
//   2. (host) clip + cdf / n_cells per brick (filters.py:124-132, 193-196).
//   3. vkt_clahe_blend: per cell, the 8 nearest brick mappings blended with
//      the per-axis weights in the reference's exact IEEE float64 operation
//      order — ((gz*gy)*gx)*m accumulated z-lo..z-hi, y-lo..y-hi, x-lo..x-hi
//      (filters.py:233-241) — then lo + out*(hi-lo) re-quantized
//      (volume.py:102-110).  No FMA contraction: bit-identical to numpy.
#include "common.cuh"
#include "dispatch.h"

namespace vkt {
namespace {

constexpr int kHistThreads = 256;
constexpr int kSmemBins = 8192;  // larger histograms go straight to global atomics

template <typename T>
__device__ __forceinline__ int bin_of(T s, const int32_t* lut, double lo, double span, int nbins) {
  if constexpr (FormatTraits<T>::is_int) {
    return __ldg(lut + s);
  } else {
    double t = __ddiv_rn(__dsub_rn((double)s, lo), span);
    t = fmin(fmax(t, 0.0), 1.0);
    const double b = floor(__dmul_rn(t, (double)nbins));
    return (int)fmin(b, (double)(nbins - 1));
  }
}

// grid: (bricks_x * bricks_y * bricks_z, zsplit).  CTA (brick, part) counts
// the brick's planes part, part+zsplit, ... into a shared histogram.
template <typename T>
__global__ void __launch_bounds__(kHistThreads) clahe_hist_kernel(vkt_clahe_args a) {
  extern __shared__ uint32_t sh[];
  const int nb = a.num_bins;
  const bool use_smem = nb <= kSmemBins;
  const int bxn = a.bricks.x, byn = a.bricks.y;
  const int brick = blockIdx.x;
  const int bx = brick % bxn, by = (brick / bxn) % byn, bz = brick / (bxn * byn);
  const int32_t* ex = a.edges;
  const int32_t* ey = ex + (a.bricks.x + 1);
  const int32_t* ez = ey + (a.bricks.y + 1);
  const int x0 = ex[bx], x1 = ex[bx + 1], y0 = ey[by], y1 = ey[by + 1], z0 = ez[bz], z1 = ez[bz + 1];
  uint32_t* gh = a.hist + (size_t)brick * nb;
  if (use_smem)
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const T* src = static_cast<const T*>(a.src);
  const double span = a.map_hi - a.map_lo;
  const int w = x1 - x0, rows = (y1 - y0);
  const int64_t cells_per_plane = (int64_t)w * rows;
  for (int z = z0 + blockIdx.y; z < z1; z += gridDim.y) {
    for (int64_t q = threadIdx.x; q < cells_per_plane; q += blockDim.x) {
      const int yy = (int)(q / w), xx = (int)(q - (int64_t)yy * w);
      const T s = src[((int64_t)z * a.dims.y + (y0 + yy)) * a.dims.x + (x0 + xx)];
      const int b = bin_of<T>(s, a.bin_lut, a.map_lo, span, nb);
      if (use_smem) atomicAdd(&sh[b], 1u);
      else atomicAdd(&gh[b], 1u);
    }
  }
  __syncthreads();
  if (use_smem)
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      if (sh[i]) atomicAdd(&gh[i], sh[i]);
}

template <typename T>
__device__ __forceinline__ T quantize_exact(double v, double lo, double span) {
  if constexpr (FormatTraits<T>::is_int) {
    double t = __ddiv_rn(__dsub_rn(v, lo), span);
    t = fmin(fmax(t, 0.0), 1.0);
    return (T)(uint32_t)floor(__dadd_rn(__dmul_rn(t, FormatTraits<T>::max_d), 0.5));
  } else {
    return __double2float_rn(v);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) clahe_blend_kernel(vkt_clahe_args a) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int z = blockIdx.z;
  if (x >= a.dims.x) return;
  const int64_t idx = ((int64_t)z * a.dims.y + y) * a.dims.x + x;
  const T s = static_cast<const T*>(a.src)[idx];
  const double span = a.map_hi - a.map_lo;
  const int nb = a.num_bins;
  const int k = bin_of<T>(s, a.bin_lut, a.map_lo, span, nb);
  const int32_t* lx = a.blend_lo;
  const int32_t* ly = lx + a.dims.x;
  const int32_t* lz = ly + a.dims.y;
  const double* wx_ = a.blend_w;
  const double* wy_ = wx_ + a.dims.x;
  const double* wz_ = wy_ + a.dims.y;
  const int xl = lx[x], yl = ly[y], zl = lz[z];
  const int xs[2] = {xl, min(xl + 1, a.bricks.x - 1)};
  const int ys[2] = {yl, min(yl + 1, a.bricks.y - 1)};
  const int zs[2] = {zl, min(zl + 1, a.bricks.z - 1)};
  const double fx = wx_[x], fy = wy_[y], fz = wz_[z];
  const double gx[2] = {__dsub_rn(1.0, fx), fx};
  const double gy[2] = {__dsub_rn(1.0, fy), fy};
  const double gz[2] = {__dsub_rn(1.0, fz), fz};
  double out = 0.0;
#pragma unroll
  for (int iz = 0; iz < 2; ++iz)
#pragma unroll
    for (int iy = 0; iy < 2; ++iy)
#pragma unroll
      for (int ix = 0; ix < 2; ++ix) {
        const int64_t brick = ((int64_t)zs[iz] * a.bricks.y + ys[iy]) * a.bricks.x + xs[ix];
        const double m = __ldg(a.mappings + brick * nb + k);
        out = __dadd_rn(out, __dmul_rn(__dmul_rn(__dmul_rn(gz[iz], gy[iy]), gx[ix]), m));
      }
  const double v = __dadd_rn(a.map_lo, __dmul_rn(out, span));
  static_cast<T*>(a.dst)[idx] = quantize_exact<T>(v, a.map_lo, span);
}

int check_args(const vkt_clahe_args* a) {
  if (a == nullptr || a->src == nullptr) {
    set_error_detail("clahe: args/src NULL");
    return VKT_INVALID_ARGUMENT;
  }
  if (a->dims.x < 1 || a->dims.y < 1 || a->dims.z < 1 || a->num_bins < 2 || a->bricks.x < 1 ||
      a->bricks.y < 1 || a->bricks.z < 1 || a->bricks.x > a->dims.x || a->bricks.y > a->dims.y ||
      a->bricks.z > a->dims.z) {
    set_error_detail("clahe: invalid dims / bricks / num_bins");
    return VKT_INVALID_ARGUMENT;
  }
  if (a->format != VKT_F32 && a->bin_lut == nullptr) {
    set_error_detail("clahe: integer formats need bin_lut");
    return VKT_INVALID_ARGUMENT;
  }
  return VKT_OK;
}

}  // namespace
}  // namespace vkt

using namespace vkt;

extern "C" int vkt_clahe_histograms(const vkt_clahe_args* args, vkt_stream_t stream) {
  VKT_NVTX("vkt_clahe_histograms");
  const vkt::StreamDeviceGuard device_guard(reinterpret_cast<cudaStream_t>(stream));
  int st = check_args(args);
  if (st != VKT_OK) return st;
  const vkt_clahe_args& a = *args;
  if (a.hist == nullptr || a.edges == nullptr) {
    set_error_detail("clahe: hist/edges NULL");
    return VKT_INVALID_ARGUMENT;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nbricks = (int64_t)a.bricks.x * a.bricks.y * a.bricks.z;
  cudaError_t e = cudaMemsetAsync(a.hist, 0, (size_t)nbricks * a.num_bins * sizeof(uint32_t), s);
  if (e != cudaSuccess) {
    set_error_detail("clahe memset: %s", cudaGetErrorString(e));
    return VKT_DEVICE_FAILURE;
  }
  // enough CTAs to fill the GPU: split each brick's planes
  const int brick_z = (a.dims.z + a.bricks.z - 1) / a.bricks.z;
  int64_t zsplit = (sm_count() * 8 + nbricks - 1) / nbricks;
  if (zsplit > brick_z) zsplit = brick_z;
  if (zsplit < 1) zsplit = 1;
  if (nbricks > 0x7fffffff || zsplit > 65535) {
    set_error_detail("clahe: too many bricks");
    return VKT_INVALID_ARGUMENT;
  }
  dim3 grid((unsigned)nbricks, (unsigned)zsplit);
  const size_t smem = a.num_bins <= kSmemBins ? a.num_bins * sizeof(uint32_t) : 0;
  switch (a.format) {
    case VKT_U8: clahe_hist_kernel<uint8_t><<<grid, kHistThreads, smem, s>>>(a); break;
    case VKT_U16: clahe_hist_kernel<uint16_t><<<grid, kHistThreads, smem, s>>>(a); break;
    default: clahe_hist_kernel<float><<<grid, kHistThreads, smem, s>>>(a); break;
  }
  count_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error_detail("clahe_hist launch: %s", cudaGetErrorString(e));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}

extern "C" int vkt_clahe_blend(const vkt_clahe_args* args, vkt_stream_t stream) {
  VKT_NVTX("vkt_clahe_blend");
  const vkt::StreamDeviceGuard device_guard(reinterpret_cast<cudaStream_t>(stream));
  int st = check_args(args);
  if (st != VKT_OK) return st;
  const vkt_clahe_args& a = *args;
  if (a.dst == nullptr || a.mappings == nullptr || a.blend_lo == nullptr || a.blend_w == nullptr) {
    set_error_detail("clahe: dst/mappings/blend tables NULL");
    return VKT_INVALID_ARGUMENT;
  }
  if (a.dims.y > 65535 || a.dims.z > 65535) {
    set_error_detail("clahe: y/z extents above 65535");
    return VKT_INVALID_ARGUMENT;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid((a.dims.x + 255) / 256, a.dims.y, a.dims.z);
  switch (a.format) {
    case VKT_U8: clahe_blend_kernel<uint8_t><<<grid, 256, 0, s>>>(a); break;
    case VKT_U16: clahe_blend_kernel<uint16_t><<<grid, 256, 0, s>>>(a); break;
    default: clahe_blend_kernel<float><<<grid, 256, 0, s>>>(a); break;
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error_detail("clahe_blend launch: %s", cudaGetErrorString(e));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}
