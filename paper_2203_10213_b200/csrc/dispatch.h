// dispatch.h — host-side plan shared by the C ABI (vkt_capi.cu) and the
// kernel launchers.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace vkt {

struct FilterPlan {
  const vkt_filter_args* args;
  SlabGeom geom;
  int z_begin, z_end;       // local output planes
  std::vector<float> w32;   // weights rounded to f32, x-fastest
  double sum_w;             // f64 sum of weights (epilogue)
  float epi_c;              // lo*(sum_w-1)/(hi-lo)*max  (ints), 0 for f32
  int path;                 // VKT_PATH_*
  // anisotropic weights padded to a K^3 cube (vkt_capi.cu pad_to_cube): the
  // kernel's own x extent and the padding y rows / z planes, which the tiled
  // kernel skips (kxs = 0: an isotropic kernel, nothing skipped)
  int kxs = 0;
  uint32_t zskip = 0;       // bit dz set: padding plane
  uint32_t yskip = 0;       // bit dy set: padding row
  bool zthin = false;       // kz = 1: the kernel variant with one z slot (no halo, no roll)
  // Device flag set by launch_scan_nonfinite.  Tiled launches do nothing when
  // it is set, direct launches only then; nullptr = unconditional.
  const int* guard = nullptr;
  // Direct kernel behind the separable f32 kernel's flag: recompute only the
  // outputs the separable pass left Inf/NaN (those whose window holds one),
  // so results do not depend on how a volume is split into launches.
  bool only_nonfinite = false;
  // Separable kernels (filter_sep.cuh): the args are the K^3 cube, the
  // weights factor as fz[dz]*fy[dy]*fx[dx] (each padded to K, centred).
  bool sep = false;
  std::vector<float> fx, fy, fz;
  int* nonfinite = nullptr;  // f32: device flag the kernel raises (vkt_capi.cu)
};

void set_error_detail(const char* fmt, ...);

// Streaming multiprocessors of the current device (cached per device; 148 on
// a B200).  Grid sizing and the z-chunk wave model use it.
int sm_count();

// Makes the stream's device current for the scope of an ABI call (and
// restores the caller's device): the tensor maps, the scratch pool, the
// shared-memory opt-in and the launch all act on the current device, and a
// caller may pass a stream of another device than the current one.  The
// legacy/per-thread default streams keep the current device.
struct StreamDeviceGuard {
  int prev = -1;
  explicit StreamDeviceGuard(cudaStream_t s) {
    if (s == nullptr || s == cudaStreamLegacy || s == cudaStreamPerThread) return;
    // a stream being captured into a CUDA graph: device queries there would
    // invalidate the capture; the capturing thread's device is the stream's
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    int d = 0, cur = 0;
    if (cudaStreamGetDevice(s, &d) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    if (cudaGetDevice(&cur) == cudaSuccess && cur != d && cudaSetDevice(d) == cudaSuccess) prev = cur;
  }
  ~StreamDeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  StreamDeviceGuard(const StreamDeviceGuard&) = delete;
  StreamDeviceGuard& operator=(const StreamDeviceGuard&) = delete;
};

// Stream-ordered scratch from a library-owned memory pool on the current
// device whose release threshold is unlimited, so repeated calls reuse the
// same HBM instead of mapping/unmapping it on every synchronize.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s);
cudaError_t scratch_free(void* p, cudaStream_t s);

int launch_filter_direct(const FilterPlan& plan, cudaStream_t s);
// Sets *flag (device int, zeroed first when `zero`) to 1 when any of the n
// floats at v is Inf or NaN.
int launch_scan_nonfinite(const float* v, int64_t n, int* flag, bool zero, cudaStream_t s);
// Returns VKT_OK, an error, or -1 when the tiled kernel does not cover `plan`.
int launch_filter_tma(const FilterPlan& plan, cudaStream_t s);
bool tma_supported(const vkt_filter_args& a);
// The driver entry point for tensor-map encoding is available.
bool tma_encode_available();
// Output planes per CTA chunk the tiled kernel would use for `plan`.
int tma_chunk_planes(const FilterPlan& plan);

int launch_fill_box(void* dst, vkt_int3 dims, int format, vkt_int3 lo, vkt_int3 hi,
                    uint32_t bits, cudaStream_t s);
int launch_fill_synthetic(void* dst, vkt_int3 dims, int format, uint64_t seed,
                          int64_t z_offset, cudaStream_t s);

}  // namespace vkt
