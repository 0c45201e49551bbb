// resample.cu — Flip and structured Resample.
//
// Flip (ops/geometric.py:34-40) is a permutation of stored cells: bit-exact.
// Resample (ops/core.py:202-262 with sample_grid_linear, volume.py:237-266):
// destination cell (i,j,k) samples the source at p = (i + 0.5) * src/dst
// (source cell units), u = clamp(p - 0.5, 0, n - 1), i0 = min(floor(u),
// max(n-2, 0)), f = u - i0, i1 = min(i0 + 1, n - 1), then the 7 lerps
// a + t*(b - a) in the reference's order over the float64 mapped grid, and the
// destination quantize (volume.py:102-110).  Every step is an IEEE float64
// operation in numpy's order (no FMA contraction), so results are
// bit-identical to the reference.
#include "common.cuh"
#include "dispatch.h"

namespace vkt {
namespace {

// Flip: rows are independent.  Axis 1 / 2 copy whole rows from the mirrored
// row; axis 0 reverses each row.  Rows of 16-byte multiples move as 16-byte
// chunks (axis 0: chunk c <- chunk n-1-c, its cells reversed in registers),
// other rows cell by cell.  TPR threads per row, RPB rows per block.
template <typename T>
__device__ __forceinline__ uint4 reverse16(uint4 v) {
  if constexpr (sizeof(T) == 1)
    return make_uint4(__byte_perm(v.w, 0, 0x0123), __byte_perm(v.z, 0, 0x0123),
                      __byte_perm(v.y, 0, 0x0123), __byte_perm(v.x, 0, 0x0123));
  else if constexpr (sizeof(T) == 2)
    return make_uint4(__byte_perm(v.w, 0, 0x1032), __byte_perm(v.z, 0, 0x1032),
                      __byte_perm(v.y, 0, 0x1032), __byte_perm(v.x, 0, 0x1032));
  else
    return make_uint4(v.w, v.z, v.y, v.x);
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) flip_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                   int nx, int ny, int nz, int axis, int per_row) {
  const int64_t rows = (int64_t)ny * nz;
  const int rpb = blockDim.y;
  for (int64_t row = (int64_t)blockIdx.y * rpb + threadIdx.y; row < rows; row += (int64_t)gridDim.y * rpb) {
    const int z = (int)(row / ny), y = (int)(row - (int64_t)z * ny);
    const int64_t srow = axis == 1 ? (int64_t)z * ny + (ny - 1 - y)
                       : axis == 2 ? (int64_t)(nz - 1 - z) * ny + y : row;
    const T* s = src + srow * nx;
    T* d = dst + row * nx;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < per_row; c += gridDim.x * blockDim.x) {
      if constexpr (VEC) {
        if (axis == 0)
          reinterpret_cast<uint4*>(d)[c] = reverse16<T>(__ldg(reinterpret_cast<const uint4*>(s) + (per_row - 1 - c)));
        else
          reinterpret_cast<uint4*>(d)[c] = __ldg(reinterpret_cast<const uint4*>(s) + c);
      } else {
        d[c] = s[axis == 0 ? nx - 1 - c : c];
      }
    }
  }
}

template <typename T>
cudaError_t launch_flip(const T* src, T* dst, vkt_int3 dims, int axis, cudaStream_t s) {
  const bool vec = ((int64_t)dims.x * sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const int per_row = vec ? (int)((int64_t)dims.x * sizeof(T) / 16) : dims.x;
  const int tpr = per_row >= 256 ? 256 : (per_row + 31) / 32 * 32;
  const dim3 block(tpr, 256 / tpr);
  const int64_t rows = (int64_t)dims.y * dims.z;
  const int64_t gy = (rows + block.y - 1) / block.y;
  const dim3 grid((per_row + tpr - 1) / tpr, (unsigned)(gy < 65535 ? gy : 65535));
  if (vec) flip_kernel<T, true><<<grid, block, 0, s>>>(src, dst, dims.x, dims.y, dims.z, axis, per_row);
  else flip_kernel<T, false><<<grid, block, 0, s>>>(src, dst, dims.x, dims.y, dims.z, axis, per_row);
  return cudaGetLastError();
}

template <typename T>
__device__ __forceinline__ double mapped(T s, double lo, double span) {
  if constexpr (FormatTraits<T>::is_int) {
    return __dadd_rn(lo, __dmul_rn(__ddiv_rn((double)s, FormatTraits<T>::max_d), span));
  } else {
    return (double)s;
  }
}

template <typename D>
__device__ __forceinline__ D quantize_f64(double v, double lo, double span) {
  if constexpr (FormatTraits<D>::is_int) {
    double t = __ddiv_rn(__dsub_rn(v, lo), span);
    t = fmin(fmax(t, 0.0), 1.0);
    return (D)(uint32_t)floor(__dadd_rn(__dmul_rn(t, FormatTraits<D>::max_d), 0.5));
  } else {
    return __double2float_rn(v);
  }
}

__device__ __forceinline__ double lerp(double a, double b, double t) {
  return __dadd_rn(a, __dmul_rn(t, __dsub_rn(b, a)));
}

struct Axis {
  int i0, i1;
  double f;
};

__device__ __forceinline__ Axis axis_coord(int i, int n_src, double scale) {
  // p = (i + 0.5) * scale ; u = p / 1.0 - 0.5 ; clip(u, 0, n - 1)
  const double p = __dmul_rn(__dadd_rn((double)i, 0.5), scale);
  double u = __dsub_rn(p, 0.5);
  u = fmin(fmax(u, 0.0), (double)(n_src - 1));
  int i0 = (int)floor(u);
  const int cap = n_src - 2 > 0 ? n_src - 2 : 0;
  if (i0 > cap) i0 = cap;
  Axis a;
  a.i0 = i0;
  a.f = __dsub_rn(u, (double)i0);
  a.i1 = i0 + 1 < n_src - 1 ? i0 + 1 : n_src - 1;
  return a;
}

struct ResampleParams {
  const void* src;
  void* dst;
  const double* lut;  // u8 / u16 sources: mapped value of every stored value
  const Axis* ax;     // per destination index: the source cells and weight
  const Axis* ay;     //   (axis_coord, computed once per call)
  const Axis* az;
  int sx, sy, sz, dx, dy, dz;
  double slo, sspan, dlo, dspan;
  double scale_x, scale_y, scale_z;
};

// axis_coord for every destination index of the three axes (x, then y, then z)
__global__ void __launch_bounds__(256) axis_table_kernel(Axis* t, int dx, int dy, int dz, int sx, int sy,
                                                         int sz, double scx, double scy, double scz) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < dx) t[i] = axis_coord(i, sx, scx);
  else if (i < dx + dy) t[i] = axis_coord(i - dx, sy, scy);
  else if (i < dx + dy + dz) t[i] = axis_coord(i - dx - dy, sz, scz);
}

// The mapped value of each stored value (u8: 256, u16: 65536 doubles), computed
// once per call with the same float64 operations as mapped(): the sampling
// kernel then looks values up instead of dividing 8 times per output.
template <typename S>
__global__ void __launch_bounds__(256) mapped_lut_kernel(double* lut, double lo, double span) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= (int)FormatTraits<S>::max_d) lut[i] = mapped<S>((S)i, lo, span);
}

template <typename S, typename D>
__global__ void __launch_bounds__(256) resample_kernel(ResampleParams p) {
  __shared__ double slut[sizeof(S) == 1 ? 256 : 1];
  if constexpr (sizeof(S) == 1) {
    slut[threadIdx.x] = p.lut[threadIdx.x];  // blockDim.x == 256
    __syncthreads();
  }
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= p.dx) return;
  const Axis ax = p.ax[x];
  const Axis ay = p.ay[y];
  const Axis az = p.az[z];
  const S* g = static_cast<const S*>(p.src);
  auto at = [&](int zz, int yy, int xx) -> double {
    const S v = g[((int64_t)zz * p.sy + yy) * p.sx + xx];
    if constexpr (sizeof(S) == 1) return slut[v];
    else if constexpr (sizeof(S) == 2) return __ldg(p.lut + v);
    else return mapped<S>(v, p.slo, p.sspan);
  };
  const double c00 = lerp(at(az.i0, ay.i0, ax.i0), at(az.i0, ay.i0, ax.i1), ax.f);
  const double c10 = lerp(at(az.i0, ay.i1, ax.i0), at(az.i0, ay.i1, ax.i1), ax.f);
  const double c01 = lerp(at(az.i1, ay.i0, ax.i0), at(az.i1, ay.i0, ax.i1), ax.f);
  const double c11 = lerp(at(az.i1, ay.i1, ax.i0), at(az.i1, ay.i1, ax.i1), ax.f);
  const double c0 = lerp(c00, c10, ay.f);
  const double c1 = lerp(c01, c11, ay.f);
  const double v = lerp(c0, c1, az.f);
  static_cast<D*>(p.dst)[((int64_t)z * p.dy + y) * p.dx + x] = quantize_f64<D>(v, p.dlo, p.dspan);
}

template <typename S>
cudaError_t launch_resample_dst(const ResampleParams& p, int dst_format, cudaStream_t s) {
  dim3 grid((p.dx + 255) / 256, p.dy, p.dz);
  switch (dst_format) {
    case VKT_U8: resample_kernel<S, uint8_t><<<grid, 256, 0, s>>>(p); break;
    case VKT_U16: resample_kernel<S, uint16_t><<<grid, 256, 0, s>>>(p); break;
    default: resample_kernel<S, float><<<grid, 256, 0, s>>>(p); break;
  }
  return cudaGetLastError();
}

bool fmt_ok(int f) { return f == VKT_U8 || f == VKT_U16 || f == VKT_F32; }

}  // namespace
}  // namespace vkt

using namespace vkt;

extern "C" int vkt_flip(const void* src, void* dst, vkt_int3 dims, int32_t format, int32_t axis,
                        vkt_stream_t stream) {
  const vkt::StreamDeviceGuard device_guard(reinterpret_cast<cudaStream_t>(stream));
  if (!src || !dst || src == dst || dims.x < 1 || dims.y < 1 || dims.z < 1 || !fmt_ok(format) ||
      axis < 0 || axis > 2) {
    set_error_detail("flip: invalid arguments (src/dst distinct, dims >= 1, axis 0..2)");
    return VKT_INVALID_ARGUMENT;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (format == VKT_U8) e = launch_flip((const uint8_t*)src, (uint8_t*)dst, dims, axis, s);
  else if (format == VKT_U16) e = launch_flip((const uint16_t*)src, (uint16_t*)dst, dims, axis, s);
  else e = launch_flip((const float*)src, (float*)dst, dims, axis, s);
  count_launch();
  if (e != cudaSuccess) {
    set_error_detail("flip launch: %s", cudaGetErrorString(e));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}

extern "C" int vkt_resample(const void* src, vkt_int3 src_dims, int32_t src_format, double src_lo,
                            double src_hi, void* dst, vkt_int3 dst_dims, int32_t dst_format,
                            double dst_lo, double dst_hi, vkt_stream_t stream) {
  const vkt::StreamDeviceGuard device_guard(reinterpret_cast<cudaStream_t>(stream));
  if (!src || !dst || src_dims.x < 1 || src_dims.y < 1 || src_dims.z < 1 || dst_dims.x < 1 ||
      dst_dims.y < 1 || dst_dims.z < 1 || !fmt_ok(src_format) || !fmt_ok(dst_format) ||
      !(src_lo < src_hi) || !(dst_lo < dst_hi) || dst_dims.y > 65535 || dst_dims.z > 65535) {
    set_error_detail("resample: invalid arguments");
    return VKT_INVALID_ARGUMENT;
  }
  ResampleParams p{};
  p.src = src;
  p.dst = dst;
  p.sx = src_dims.x; p.sy = src_dims.y; p.sz = src_dims.z;
  p.dx = dst_dims.x; p.dy = dst_dims.y; p.dz = dst_dims.z;
  p.slo = src_lo; p.sspan = src_hi - src_lo;
  p.dlo = dst_lo; p.dspan = dst_hi - dst_lo;
  // scale = extent_cells / dst_dims in float64 (core.py:253)
  p.scale_x = (double)src_dims.x / (double)dst_dims.x;
  p.scale_y = (double)src_dims.y / (double)dst_dims.y;
  p.scale_z = (double)src_dims.z / (double)dst_dims.z;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  // scratch: the axis tables, then (u8 / u16 sources) the mapped-value LUT
  const int nax = dst_dims.x + dst_dims.y + dst_dims.z;
  const size_t ax_bytes = ((size_t)nax * sizeof(Axis) + 255) / 256 * 256;
  const int nlut = src_format == VKT_U8 ? 256 : src_format == VKT_U16 ? 65536 : 0;
  uint8_t* scratch = nullptr;
  e = scratch_alloc(reinterpret_cast<void**>(&scratch), ax_bytes + (size_t)nlut * sizeof(double), s);
  if (e != cudaSuccess) {
    set_error_detail("resample: scratch_alloc: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? VKT_ALLOCATION_FAILURE : VKT_DEVICE_FAILURE;
  }
  Axis* tab = reinterpret_cast<Axis*>(scratch);
  axis_table_kernel<<<(nax + 255) / 256, 256, 0, s>>>(tab, dst_dims.x, dst_dims.y, dst_dims.z, p.sx, p.sy,
                                                        p.sz, p.scale_x, p.scale_y, p.scale_z);
  count_launch();
  p.ax = tab;
  p.ay = tab + dst_dims.x;
  p.az = tab + dst_dims.x + dst_dims.y;
  double* lut = nullptr;
  if (nlut > 0) {
    lut = reinterpret_cast<double*>(scratch + ax_bytes);
    if (src_format == VKT_U8) mapped_lut_kernel<uint8_t><<<1, 256, 0, s>>>(lut, p.slo, p.sspan);
    else mapped_lut_kernel<uint16_t><<<256, 256, 0, s>>>(lut, p.slo, p.sspan);
    count_launch();
    p.lut = lut;
  }
  switch (src_format) {
    case VKT_U8: e = launch_resample_dst<uint8_t>(p, dst_format, s); break;
    case VKT_U16: e = launch_resample_dst<uint16_t>(p, dst_format, s); break;
    default: e = launch_resample_dst<float>(p, dst_format, s); break;
  }
  scratch_free(scratch, s);
  count_launch();
  if (e != cudaSuccess) {
    set_error_detail("resample launch: %s", cudaGetErrorString(e));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}
