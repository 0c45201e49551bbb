// filter_direct.cu — generic ApplyFilter kernel: any odd kernel extent, any
// volume extents/alignment, every address mode, optional bit-exact float64.
//
// One thread per output cell; taps are visited in the reference's (dz, dy, dx)
// order (pkg/src/vkt/ops/filters.py:89-92) so the f32 result is bit-identical
// to the tiled TMA kernel (filter_tma.cu) and independent of any slab split.
// Reuse of neighbouring inputs comes from L1/L2; this kernel is the fallback
// for shapes the tiled kernel does not specialise (k > 9, k = 1, sharded f32
// kernels needing x/y padding, f32 volumes with Inf/NaN under the guarded cube
// path -- vkt_capi.cu pads the other anisotropic ones to a cube) and the
// EXACT_F64 parity mode.
#include <algorithm>

#include "common.cuh"
#include "dispatch.h"

namespace vkt {

struct DirectParams {
  SlabGeom g;
  void* dst;
  int nx, ny;
  int kx, ky, kz;
  int rx, ry;
  int z_begin, z_end;
  const float* w32;   // device, kx*ky*kz
  const double* w64;  // device, kx*ky*kz (EXACT only)
  float c;            // fast epilogue constant (ints)
  double lo, hi, span;  // mapping (EXACT only); span = hi - lo
  const int* run_if;   // non-null: the launch does nothing unless *run_if != 0
  bool only_nonfinite; // recompute only outputs whose current dst value is Inf/NaN (f32)
};

template <typename T, int MODE>
__global__ void __launch_bounds__(256) filter_direct_kernel(DirectParams p) {
  if (p.run_if != nullptr && *p.run_if == 0) return;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= p.nx || y >= p.ny) return;
  for (int z = p.z_begin + blockIdx.z; z < p.z_end; z += gridDim.z) {
    T* out = static_cast<T*>(p.dst) + ((int64_t)z * p.ny + y) * p.nx + x;
    if constexpr (!FormatTraits<T>::is_int) {
      if (p.only_nonfinite && isfinite(*out)) continue;
    }
    float acc = acc_init<T>(p.c);
    int t = 0;
    for (int dz = 0; dz < p.kz; ++dz) {
      const T* plane = resolve_plane<MODE, T>(p.g, z + dz - p.g.rz);
      for (int dy = 0; dy < p.ky; ++dy) {
        const int my = map_index32<MODE>(y + dy - p.ry, p.ny);
        const T* row = (plane != nullptr && my >= 0) ? plane + (int64_t)my * p.nx : nullptr;
        for (int dx = 0; dx < p.kx; ++dx, ++t) {
          const int mx = map_index32<MODE>(x + dx - p.rx, p.nx);
          float v = 0.0f;
          if (row != nullptr && mx >= 0) v = to_f32(__ldg(row + mx));
          acc = __fmaf_rn(__ldg(p.w32 + t), v, acc);
        }
      }
    }
    *out = quantize_acc<T>(acc);
  }
}

// Bit-exact restatement of the reference arithmetic in float64:
//   snapshot = lo + (s / max) * (hi - lo)         volume.py:113-118
//   acc += w * snapshot   (separate mul/add)      filters.py:86-92
//   t = clip((acc - lo)/(hi - lo), 0, 1); floor(t*max + 0.5)   volume.py:102-110
//   F32: acc.astype('<f4')                        volume.py:105-106
template <typename T>
__device__ __forceinline__ double mapped_exact(T s, double lo, double span) {
  if constexpr (FormatTraits<T>::is_int) {
    double q = __ddiv_rn((double)s, FormatTraits<T>::max_d);
    return __dadd_rn(lo, __dmul_rn(q, span));
  } else {
    return (double)s;
  }
}

template <typename T, int MODE>
__global__ void __launch_bounds__(256) filter_exact_kernel(DirectParams p) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= p.nx || y >= p.ny) return;
  // Border cells hold stored 0, i.e. the mapped value dequantize(0).
  const double border = mapped_exact<T>((T)0, p.lo, p.span);
  for (int z = p.z_begin + blockIdx.z; z < p.z_end; z += gridDim.z) {
    double acc = 0.0;
    int t = 0;
    for (int dz = 0; dz < p.kz; ++dz) {
      const T* plane = resolve_plane<MODE, T>(p.g, z + dz - p.g.rz);
      for (int dy = 0; dy < p.ky; ++dy) {
        const int my = map_index32<MODE>(y + dy - p.ry, p.ny);
        const T* row = (plane != nullptr && my >= 0) ? plane + (int64_t)my * p.nx : nullptr;
        for (int dx = 0; dx < p.kx; ++dx, ++t) {
          const int mx = map_index32<MODE>(x + dx - p.rx, p.nx);
          double v = border;
          if (row != nullptr && mx >= 0) v = mapped_exact<T>(__ldg(row + mx), p.lo, p.span);
          acc = __dadd_rn(acc, __dmul_rn(__ldg(p.w64 + t), v));
        }
      }
    }
    T* out = static_cast<T*>(p.dst) + ((int64_t)z * p.ny + y) * p.nx + x;
    if constexpr (FormatTraits<T>::is_int) {
      double tt = __ddiv_rn(__dsub_rn(acc, p.lo), p.span);
      tt = fmin(fmax(tt, 0.0), 1.0);
      double q = floor(__dadd_rn(__dmul_rn(tt, FormatTraits<T>::max_d), 0.5));
      *out = (T)(uint32_t)q;
    } else {
      *out = __double2float_rn(acc);
    }
  }
}

template <typename T, int MODE>
static cudaError_t launch_direct_t(const DirectParams& p, bool exact, cudaStream_t s) {
  dim3 block(32, 8, 1);
  int nzo = p.z_end - p.z_begin;
  dim3 grid((p.nx + 31) / 32, (p.ny + 7) / 8, (unsigned)(nzo < 65535 ? nzo : 65535));
  // A guarded launch (the fallback behind a device flag, vkt_capi.cu) almost
  // always does nothing: keep its grid to ~8 CTAs per SM (the kernel strides
  // over z), so the no-op costs microseconds, not a pass over the volume.
  if (p.run_if != nullptr) {
    const int64_t xy = (int64_t)grid.x * grid.y;
    const int64_t gz = std::max<int64_t>(1, (int64_t)sm_count() * 8 / xy);
    grid.z = (unsigned)std::min<int64_t>(grid.z, gz);
  }
  if (exact)
    filter_exact_kernel<T, MODE><<<grid, block, 0, s>>>(p);
  else
    filter_direct_kernel<T, MODE><<<grid, block, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_direct_mode(const DirectParams& p, int mode, bool exact,
                                      cudaStream_t s) {
  switch (mode) {
    case VKT_WRAP: return launch_direct_t<T, VKT_WRAP>(p, exact, s);
    case VKT_MIRROR: return launch_direct_t<T, VKT_MIRROR>(p, exact, s);
    case VKT_CLAMP: return launch_direct_t<T, VKT_CLAMP>(p, exact, s);
    default: return launch_direct_t<T, VKT_BORDER>(p, exact, s);
  }
}

int launch_filter_direct(const FilterPlan& plan, cudaStream_t s) {
  const vkt_filter_args& a = *plan.args;
  const bool exact = (a.flags & VKT_FLAG_EXACT_F64) != 0;
  const size_t ntaps = (size_t)a.kdims.x * a.kdims.y * a.kdims.z;

  // Weights travel in a stream-ordered scratch allocation so concurrent calls
  // on different streams never share device state.
  size_t bytes = ntaps * (exact ? sizeof(double) : sizeof(float));
  void* dw = nullptr;
  cudaError_t err = scratch_alloc(&dw, bytes, s);
  if (err != cudaSuccess) {
    set_error_detail("scratch_alloc(weights): %s", cudaGetErrorString(err));
    return err == cudaErrorMemoryAllocation ? VKT_ALLOCATION_FAILURE : VKT_DEVICE_FAILURE;
  }
  if (exact)
    err = cudaMemcpyAsync(dw, a.weights, bytes, cudaMemcpyHostToDevice, s);
  else
    err = cudaMemcpyAsync(dw, plan.w32.data(), bytes, cudaMemcpyHostToDevice, s);
  if (err != cudaSuccess) {
    scratch_free(dw, s);
    set_error_detail("cudaMemcpyAsync(weights): %s", cudaGetErrorString(err));
    return VKT_DEVICE_FAILURE;
  }

  DirectParams p{};
  p.g = plan.geom;
  p.dst = a.dst;
  p.nx = a.dims.x;
  p.ny = a.dims.y;
  p.kx = a.kdims.x;
  p.ky = a.kdims.y;
  p.kz = a.kdims.z;
  p.rx = a.kdims.x / 2;
  p.ry = a.kdims.y / 2;
  p.z_begin = plan.z_begin;
  p.z_end = plan.z_end;
  p.w32 = exact ? nullptr : static_cast<const float*>(dw);
  p.w64 = exact ? static_cast<const double*>(dw) : nullptr;
  p.c = plan.epi_c;
  p.lo = a.map_lo;
  p.hi = a.map_hi;
  p.span = a.map_hi - a.map_lo;
  p.run_if = plan.guard;
  p.only_nonfinite = plan.only_nonfinite;

  switch (a.format) {
    case VKT_U8: err = launch_direct_mode<uint8_t>(p, a.address_mode, exact, s); break;
    case VKT_U16: err = launch_direct_mode<uint16_t>(p, a.address_mode, exact, s); break;
    default: err = launch_direct_mode<float>(p, a.address_mode, exact, s); break;
  }
  scratch_free(dw, s);
  if (err != cudaSuccess) {
    set_error_detail("filter_direct launch: %s", cudaGetErrorString(err));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}

// Inf/NaN scan for the guarded cube path (vkt_capi.cu): 16-byte streaming
// loads over the aligned body, the unaligned head and tail by the first
// threads; one store per block that saw a non-finite value.
__device__ __forceinline__ bool nonfinite(float v) {
  return (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
}

__global__ void __launch_bounds__(256) scan_nonfinite_kernel(const float* __restrict__ v,
                                                             int64_t n, int64_t head, int* flag) {
  const int64_t nvec = (n - head) / 4;
  const float4* v4 = reinterpret_cast<const float4*>(v + head);
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (int64_t i = t0; i < nvec; i += stride) {
    const float4 q = __ldcs(v4 + i);
    bad |= nonfinite(q.x) | nonfinite(q.y) | nonfinite(q.z) | nonfinite(q.w);
  }
  const int64_t tail = head + nvec * 4;
  if (t0 < head) bad |= nonfinite(v[t0]);
  if (t0 < n - tail) bad |= nonfinite(v[tail + t0]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

int launch_scan_nonfinite(const float* v, int64_t n, int* flag, bool zero, cudaStream_t s) {
  cudaError_t err = zero ? cudaMemsetAsync(flag, 0, sizeof(int), s) : cudaSuccess;
  if (err == cudaSuccess) {
    int64_t head = (int64_t)(((16u - (reinterpret_cast<uintptr_t>(v) & 15u)) & 15u) / 4u);
    if (head > n) head = n;
    const int64_t nvec = (n - head) / 4;
    int64_t blocks = (nvec + 255) / 256;
    if (blocks > sm_count() * 8) blocks = sm_count() * 8;
    if (blocks < 1) blocks = 1;
    scan_nonfinite_kernel<<<(unsigned)blocks, 256, 0, s>>>(v, n, head, flag);
    count_launch();
    err = cudaGetLastError();
  }
  if (err != cudaSuccess) {
    set_error_detail("scan_nonfinite: %s", cudaGetErrorString(err));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}

}  // namespace vkt
