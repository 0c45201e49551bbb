// vkt_capi.cu — the extern "C" boundary declared in include/vkt_b200.h.
//
// Validation mirrors the reference's error contract:
//   even / non-positive kernel extents -> EvenKernelDims   (filters.py:32-33)
//   non-finite weights                 -> InvalidArgument  (filters.py:37-38)
//   dims < 1, degenerate mapping       -> InvalidArgument  (volume.py:133-134, 80-81)
//   device allocation failure          -> AllocationFailure (managed.py:45-49)
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "dispatch.h"
#include "filter_sep.cuh"

namespace vkt {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static thread_local char g_detail[512] = "";

void set_error_detail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_detail, sizeof(g_detail), fmt, ap);
  va_end(ap);
}

int sm_count() {
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    n = 148;
  if (dev < 64) cache[dev].store(n, std::memory_order_relaxed);
  return n;
}

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (pools[dev] == nullptr) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) return e;
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

cudaError_t scratch_free(void* p, cudaStream_t s) { return cudaFreeAsync(p, s); }

static int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_detail, sizeof(g_detail), fmt, ap);
  va_end(ap);
  return status;
}

static int validate_and_plan(const vkt_filter_args* a, FilterPlan& plan) {
  if (a == nullptr) return fail(VKT_INVALID_ARGUMENT, "args is NULL");
  if (a->kdims.x < 1 || a->kdims.y < 1 || a->kdims.z < 1 || a->kdims.x % 2 == 0 ||
      a->kdims.y % 2 == 0 || a->kdims.z % 2 == 0)
    return fail(VKT_EVEN_KERNEL_DIMS, "kernel dims must be odd, got (%d, %d, %d)", a->kdims.x,
                a->kdims.y, a->kdims.z);
  if (a->dims.x < 1 || a->dims.y < 1 || a->dims.z < 1)
    return fail(VKT_INVALID_ARGUMENT, "dims must be >= 1 per axis, got (%d, %d, %d)", a->dims.x,
                a->dims.y, a->dims.z);
  if (a->format != VKT_U8 && a->format != VKT_U16 && a->format != VKT_F32)
    return fail(VKT_INVALID_ARGUMENT, "unknown data format code %d", a->format);
  if (a->address_mode < VKT_WRAP || a->address_mode > VKT_BORDER)
    return fail(VKT_INVALID_ARGUMENT, "unknown address mode %d", a->address_mode);
  if (a->src == nullptr || a->dst == nullptr || a->weights == nullptr)
    return fail(VKT_INVALID_ARGUMENT, "src, dst and weights must be non-NULL");
  if (a->src == a->dst)
    return fail(VKT_INVALID_ARGUMENT, "dst must not alias src (the filter reads a snapshot)");
  if (!(std::isfinite(a->map_lo) && std::isfinite(a->map_hi)) || !(a->map_lo < a->map_hi))
    return fail(VKT_INVALID_ARGUMENT, "voxel mapping needs finite lo < hi, got [%g, %g]",
                a->map_lo, a->map_hi);

  const size_t ntaps = (size_t)a->kdims.x * a->kdims.y * a->kdims.z;
  plan.args = a;
  plan.w32.resize(ntaps);
  double sum = 0.0;
  for (size_t i = 0; i < ntaps; ++i) {
    double w = a->weights[i];
    if (!std::isfinite(w)) return fail(VKT_INVALID_ARGUMENT, "kernel weights must be finite");
    plan.w32[i] = (float)w;
    sum += w;
  }
  plan.sum_w = sum;
  if (a->format == VKT_F32) {
    plan.epi_c = 0.0f;
  } else {
    const double mx = a->format == VKT_U8 ? 255.0 : 65535.0;
    plan.epi_c = (float)(a->map_lo * (sum - 1.0) / (a->map_hi - a->map_lo) * mx);
  }

  const int64_t gnz = a->global_nz > 0 ? a->global_nz : a->dims.z;
  if (a->z_offset < 0 || a->z_offset + a->dims.z > gnz)
    return fail(VKT_INVALID_ARGUMENT, "slab [%lld, %lld) outside global z extent %lld",
                (long long)a->z_offset, (long long)(a->z_offset + a->dims.z), (long long)gnz);
  plan.z_begin = a->out_z_begin > 0 ? a->out_z_begin : 0;
  plan.z_end = a->out_z_end > 0 ? (a->out_z_end < a->dims.z ? a->out_z_end : a->dims.z) : a->dims.z;

  const int rz = a->kdims.z / 2;
  SlabGeom& g = plan.geom;
  g.src = a->src;
  g.halo_lo = a->halo_lo;
  g.halo_hi = a->halo_hi;
  g.plane_elems = (int64_t)a->dims.x * a->dims.y;
  g.nz = a->dims.z;
  g.rz = rz;
  g.z_offset = a->z_offset;
  g.global_nz = gnz;

  // Without halos every z tap must resolve inside the slab (unsharded volume,
  // or a shard whose neighbours' planes are not needed).
  if (rz > 0 && (a->halo_lo == nullptr || a->halo_hi == nullptr) && gnz != a->dims.z)
    return fail(VKT_INVALID_ARGUMENT,
                "sharded slab (global_nz=%lld, local nz=%d) needs halo_lo and halo_hi",
                (long long)gnz, a->dims.z);

  if (a->flags & VKT_FLAG_EXACT_F64) plan.path = VKT_PATH_EXACT;
  else if (!(a->flags & VKT_FLAG_FORCE_DIRECT) && tma_supported(*a)) plan.path = VKT_PATH_TMA;
  else plan.path = VKT_PATH_DIRECT;
  return VKT_OK;
}

// Anisotropic kernels on the tiled kernels: embed the (kx, ky, kz) weights,
// centred, in a K^3 cube of zeros, K = max extent.
//  * K >= 5 (the paired-layout kernel): the kernel runs only the real taps:
//    its x extent kx is a template and the padding y rows / z planes are
//    skipped by mask (yskip / zskip); a z-thin kernel (kz = 1) runs the
//    variant with a single z slot (no z halo planes, no accumulator roll).  So no FMA is wasted and no zero weight
//    ever meets an Inf (results bit-identical to the direct kernel's, Inf and
//    NaN voxels included).
//  * K = 3, integer voxels (the warp kernel): the cube is evaluated densely;
//    integer voxels widen to finite floats, so each added tap is an exact +0
//    and the FP32 sums -- the same nonzero products in the same relative
//    (dz, dy, dx) order -- are bit-identical to the unpadded ones.
//  * K = 3, f32 (the direct-staging kernel, which cannot skip): `guarded` --
//    an Inf/NaN scan of the source and its halo planes picks, on the device,
//    the tiled launch when every voxel is finite or the direct kernel.
// The z extent may only grow when no halo buffers are involved: halos are
// sized for the caller's kz.
static bool pad_to_cube(const vkt_filter_args* a, vkt_filter_args& out, std::vector<double>& w,
                        FilterPlan& skip, bool& guarded) {
  if (a->flags & (VKT_FLAG_EXACT_F64 | VKT_FLAG_FORCE_DIRECT)) return false;
  const int kx = a->kdims.x, ky = a->kdims.y, kz = a->kdims.z;
  if (kx == ky && ky == kz) return false;
  int k = kx > ky ? kx : ky;
  k = k > kz ? k : kz;
  if (k != 3 && k != 5 && k != 7 && k != 9) return false;
  const bool unsharded = a->halo_lo == nullptr && a->halo_hi == nullptr &&
                         (a->global_nz <= 0 || a->global_nz == a->dims.z);
  guarded = a->format == VKT_F32 && k == 3;
  if (kz != k && !unsharded) return false;
  w.assign((size_t)k * k * k, 0.0);
  const int ox = (k - kx) / 2, oy = (k - ky) / 2, oz = (k - kz) / 2;
  for (int z = 0; z < kz; ++z)
    for (int y = 0; y < ky; ++y)
      for (int x = 0; x < kx; ++x)
        w[((size_t)(z + oz) * k + (y + oy)) * k + (x + ox)] = a->weights[((size_t)z * ky + y) * kx + x];
  out = *a;
  out.kdims = vkt_int3{k, k, k};
  out.weights = w.data();
  skip.kxs = 0;
  skip.zskip = skip.yskip = 0;
  skip.zthin = false;
  if (k >= 5) {
    skip.kxs = kx;
    skip.zthin = kz == 1;
    for (int i = 0; i < k; ++i) {
      if (i < oz || i >= oz + kz) skip.zskip |= 1u << i;
      if (i < oy || i >= oy + ky) skip.yskip |= 1u << i;
    }
  }
  return true;
}

// The guarded cube launch (see pad_to_cube): scan, tiled kernel (skipped on
// the device when the scan found Inf/NaN), direct kernel (skipped otherwise).
// Returns -1 when the tiled kernel does not cover the cube plan.
static int launch_guarded(const FilterPlan& plan, FilterPlan& cube, cudaStream_t s) {
  void* flag = nullptr;
  cudaError_t err = scratch_alloc(&flag, sizeof(int), s);
  if (err != cudaSuccess) {
    set_error_detail("scratch_alloc(flag): %s", cudaGetErrorString(err));
    return err == cudaErrorMemoryAllocation ? VKT_ALLOCATION_FAILURE : VKT_DEVICE_FAILURE;
  }
  const vkt_filter_args& a = *plan.args;
  const int64_t plane = (int64_t)a.dims.x * a.dims.y;
  int* f = static_cast<int*>(flag);
  int st = launch_scan_nonfinite(static_cast<const float*>(a.src), plane * a.dims.z, f, true, s);
  // halo buffers hold rz = kz/2 planes each (the caller's kz, which the cube
  // keeps: pad_to_cube grows z only without halos).  Scanned only when this
  // launch's output planes read them: an interior launch of a sharded step
  // runs while the exchange is still filling them.
  const int rz = a.kdims.z / 2;
  const int64_t halo = plane * rz;
  if (st == VKT_OK && a.halo_lo != nullptr && halo > 0 && plan.z_begin < rz)
    st = launch_scan_nonfinite(static_cast<const float*>(a.halo_lo), halo, f, false, s);
  if (st == VKT_OK && a.halo_hi != nullptr && halo > 0 && plan.z_end > a.dims.z - rz)
    st = launch_scan_nonfinite(static_cast<const float*>(a.halo_hi), halo, f, false, s);
  if (st == VKT_OK) {
    cube.guard = static_cast<const int*>(flag);
    st = launch_filter_tma(cube, s);
    if (st == VKT_OK) {
      FilterPlan direct = plan;
      direct.guard = static_cast<const int*>(flag);
      st = launch_filter_direct(direct, s);
    }
  }
  scratch_free(flag, s);
  return st;
}

// Separable (rank-1) weights: W[z][y][x] = fz[z] * fy[y] * fx[x], checked in
// float64 against the largest weight (gaussian_kernel is g(x)g(x)g over its
// sum, box_kernel a constant: both factor to ~1 ulp).  Pivot on the largest
// |W| so |fy|, |fx| <= 1 and fz carries the scale.  A tolerance of 1e-9 of
// the largest weight is far below the f32 rounding of the weights
// themselves (~6e-8 relative), which every tiled path already applies.
static bool factor_rank1(const double* w, int kx, int ky, int kz, std::vector<double>& fx,
                         std::vector<double>& fy, std::vector<double>& fz) {
  const size_t n = (size_t)kx * ky * kz;
  size_t piv = 0;
  double mx = 0.0;
  for (size_t i = 0; i < n; ++i)
    if (std::fabs(w[i]) > mx) mx = std::fabs(w[i]), piv = i;
  fx.assign(kx, 1.0);
  fy.assign(ky, 1.0);
  fz.assign(kz, 0.0);
  if (mx == 0.0) return true;  // the zero kernel
  const int px = (int)(piv % kx), py = (int)(piv / kx % ky), pz = (int)(piv / ((size_t)kx * ky));
  auto at = [&](int z, int y, int x) { return w[((size_t)z * ky + y) * kx + x]; };
  const double pv = at(pz, py, px);
  for (int z = 0; z < kz; ++z) fz[z] = at(z, py, px);
  for (int y = 0; y < ky; ++y) fy[y] = at(pz, y, px) / pv;
  for (int x = 0; x < kx; ++x) fx[x] = at(pz, py, x) / pv;
  const double tol = 1e-9 * mx;
  for (int z = 0; z < kz; ++z)
    for (int y = 0; y < ky; ++y)
      for (int x = 0; x < kx; ++x)
        if (!(std::fabs(at(z, y, x) - fz[z] * fy[y] * fx[x]) <= tol)) return false;
  return true;
}

// The separable plan (filter_sep.cuh) for a validated plan, or false.
// Integer voxels at every K in {3,5,7,9}; f32 from K = 5 (f32 3^3 is
// HBM-bound on the dense kernel already).  Anisotropic kernels pad their
// factors with zeros to the K^3 cube (z only when unsharded, as pad_to_cube).
// `cube` receives the cube's args (weights NULL: the plan carries factors).
static bool plan_separable(const FilterPlan& plan, vkt_filter_args& cube, FilterPlan& sp) {
  const vkt_filter_args* a = plan.args;
  if (a->flags & (VKT_FLAG_EXACT_F64 | VKT_FLAG_FORCE_DIRECT | VKT_FLAG_NO_SEPARABLE)) return false;
  const int kx = a->kdims.x, ky = a->kdims.y, kz = a->kdims.z;
  int k = kx > ky ? kx : ky;
  k = k > kz ? k : kz;
  if (k < 3 || k > sep::MAX_K) return false;  // odd: validated
  if (a->format == VKT_F32 && k == 3) return false;
  const bool unsharded = a->halo_lo == nullptr && a->halo_hi == nullptr &&
                         (a->global_nz <= 0 || a->global_nz == a->dims.z);
  if (kz != k && !unsharded) return false;
  std::vector<double> fx, fy, fz;
  if (!factor_rank1(a->weights, kx, ky, kz, fx, fy, fz)) return false;
  cube = *a;
  cube.kdims = vkt_int3{k, k, k};
  cube.weights = nullptr;
  if (!tma_encode_available()) return false;
  sp = plan;
  sp.args = &cube;
  sp.path = VKT_PATH_SEPARABLE;
  sp.sep = true;
  sp.geom.rz = k / 2;
  auto pad = [k](const std::vector<double>& f, std::vector<float>& out) {
    out.assign(k, 0.0f);
    const int o = (k - (int)f.size()) / 2;
    for (size_t i = 0; i < f.size(); ++i) out[o + i] = (float)f[i];
  };
  pad(fx, sp.fx);
  pad(fy, sp.fy);
  pad(fz, sp.fz);
  return true;
}

// The separable launch.  f32: the kernel raises a device flag when a stored
// output is Inf/NaN (an Inf/NaN input in its window), and the direct kernel,
// guarded by that flag, then recomputes exactly those outputs with the dense
// arithmetic (it does nothing otherwise): every output is a function of its
// own window, whatever the launch split.  Returns -1 when the tiled kernel
// does not cover the plan.
static int launch_separable(const FilterPlan& plan, FilterPlan& sp, cudaStream_t s) {
  if (plan.args->format != VKT_F32) return launch_filter_tma(sp, s);
  void* flag = nullptr;
  cudaError_t err = scratch_alloc(&flag, sizeof(int), s);
  if (err != cudaSuccess) {
    set_error_detail("scratch_alloc(flag): %s", cudaGetErrorString(err));
    return err == cudaErrorMemoryAllocation ? VKT_ALLOCATION_FAILURE : VKT_DEVICE_FAILURE;
  }
  int st = cudaMemsetAsync(flag, 0, sizeof(int), s) == cudaSuccess ? VKT_OK : VKT_DEVICE_FAILURE;
  if (st != VKT_OK) set_error_detail("flag memset: %s", cudaGetErrorString(cudaGetLastError()));
  if (st == VKT_OK) {
    sp.nonfinite = static_cast<int*>(flag);
    st = launch_filter_tma(sp, s);
    if (st == VKT_OK) {
      FilterPlan direct = plan;
      direct.guard = static_cast<const int*>(flag);
      direct.only_nonfinite = true;
      st = launch_filter_direct(direct, s);
    }
  }
  scratch_free(flag, s);
  return st;
}

}  // namespace vkt

using namespace vkt;

extern "C" {

int vkt_apply_filter(const vkt_filter_args* args, vkt_stream_t stream) {
  VKT_NVTX("vkt_apply_filter");
  const vkt::StreamDeviceGuard device_guard(reinterpret_cast<cudaStream_t>(stream));
  FilterPlan plan;
  int st = validate_and_plan(args, plan);
  if (st != VKT_OK) return st;
  if (plan.z_end > plan.z_begin) {
    vkt_filter_args cube;
    FilterPlan sp;
    if (plan_separable(plan, cube, sp)) {
      const int st2 = launch_separable(plan, sp, reinterpret_cast<cudaStream_t>(stream));
      if (st2 != -1) return st2;
    }
  }
  if (plan.path == VKT_PATH_DIRECT) {
    vkt_filter_args cube;
    std::vector<double> wcube;
    FilterPlan skip;
    bool guarded = false;
    if (pad_to_cube(args, cube, wcube, skip, guarded)) {
      FilterPlan p2;
      if (validate_and_plan(&cube, p2) == VKT_OK && p2.path == VKT_PATH_TMA) {
        p2.kxs = skip.kxs;
        p2.zthin = skip.zthin;
        p2.zskip = skip.zskip;
        p2.yskip = skip.yskip;
        if (p2.z_end <= p2.z_begin) return VKT_OK;
        cudaStream_t s2 = reinterpret_cast<cudaStream_t>(stream);
        const int st2 = guarded ? launch_guarded(plan, p2, s2) : launch_filter_tma(p2, s2);
        if (st2 != -1) return st2;
      }
    }
  }
  if (plan.z_end <= plan.z_begin) return VKT_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (plan.path == VKT_PATH_TMA) {
    st = launch_filter_tma(plan, s);
    if (st != -1) return st;
    plan.path = VKT_PATH_DIRECT;
  }
  return launch_filter_direct(plan, s);
}

int vkt_filter_path(const vkt_filter_args* args) {
  FilterPlan plan;
  if (validate_and_plan(args, plan) != VKT_OK) return VKT_PATH_NONE;
  {
    vkt_filter_args sc;
    FilterPlan sp;
    if (plan_separable(plan, sc, sp)) return VKT_PATH_SEPARABLE;
  }
  if (plan.path == VKT_PATH_DIRECT) {
    vkt_filter_args cube;
    std::vector<double> wcube;
    FilterPlan p2, skip;
    bool guarded = false;
    if (pad_to_cube(args, cube, wcube, skip, guarded) && validate_and_plan(&cube, p2) == VKT_OK)
      return p2.path;
  }
  return plan.path;
}

int vkt_filter_chunk_planes(const vkt_filter_args* args) {
  FilterPlan plan;
  if (validate_and_plan(args, plan) != VKT_OK) return 0;
  {
    vkt_filter_args sc;
    FilterPlan sp;
    if (plan_separable(plan, sc, sp)) return tma_chunk_planes(sp);
  }
  if (plan.path == VKT_PATH_DIRECT) {
    vkt_filter_args cube;
    std::vector<double> wcube;
    FilterPlan p2, skip;
    bool guarded = false;
    if (pad_to_cube(args, cube, wcube, skip, guarded) && validate_and_plan(&cube, p2) == VKT_OK &&
        p2.path == VKT_PATH_TMA)
      return tma_chunk_planes(p2);
    return 0;
  }
  return plan.path == VKT_PATH_TMA ? tma_chunk_planes(plan) : 0;
}

int vkt_fill_box(void* dst, vkt_int3 dims, int32_t format, vkt_int3 lo, vkt_int3 hi,
                 uint32_t stored_bits, vkt_stream_t stream) {
  VKT_NVTX("vkt_fill_box");
  const vkt::StreamDeviceGuard device_guard(reinterpret_cast<cudaStream_t>(stream));
  if (dst == nullptr) return fail(VKT_INVALID_ARGUMENT, "dst is NULL");
  if (dims.x < 1 || dims.y < 1 || dims.z < 1)
    return fail(VKT_INVALID_ARGUMENT, "dims must be >= 1 per axis");
  if (format != VKT_U8 && format != VKT_U16 && format != VKT_F32)
    return fail(VKT_INVALID_ARGUMENT, "unknown data format code %d", format);
  return launch_fill_box(dst, dims, format, lo, hi, stored_bits,
                         reinterpret_cast<cudaStream_t>(stream));
}

int vkt_fill_synthetic(void* dst, vkt_int3 dims, int32_t format, uint64_t seed, int64_t z_offset,
                       vkt_stream_t stream) {
  const vkt::StreamDeviceGuard device_guard(reinterpret_cast<cudaStream_t>(stream));
  if (dst == nullptr) return fail(VKT_INVALID_ARGUMENT, "dst is NULL");
  if (dims.x < 1 || dims.y < 1 || dims.z < 1)
    return fail(VKT_INVALID_ARGUMENT, "dims must be >= 1 per axis");
  if (format != VKT_U8 && format != VKT_U16 && format != VKT_F32)
    return fail(VKT_INVALID_ARGUMENT, "unknown data format code %d", format);
  return launch_fill_synthetic(dst, dims, format, seed, z_offset,
                               reinterpret_cast<cudaStream_t>(stream));
}

const char* vkt_status_name(int status) {
  switch (status) {
    case VKT_OK: return "OK";
    case VKT_INVALID_ARGUMENT: return "InvalidArgument";
    case VKT_EVEN_KERNEL_DIMS: return "EvenKernelDims";
    case VKT_ALLOCATION_FAILURE: return "AllocationFailure";
    case VKT_DEVICE_FAILURE: return "DeviceFailure";
    default: return "Unknown";
  }
}

const char* vkt_last_error_detail(void) { return g_detail; }

uint64_t vkt_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int vkt_abi_version(void) { return 10000; }

}  // extern "C"
