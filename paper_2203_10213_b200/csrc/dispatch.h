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
  uint32_t zskip = 0;       // f32 weights padded in z to a cube: bit dz = padding plane
  // Device flag set by launch_scan_nonfinite.  Tiled launches do nothing when
  // it is set, direct launches only then; nullptr = unconditional.
  const int* guard = nullptr;
};

void set_error_detail(const char* fmt, ...);

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

int launch_fill_box(void* dst, vkt_int3 dims, int format, vkt_int3 lo, vkt_int3 hi,
                    uint32_t bits, cudaStream_t s);
int launch_fill_synthetic(void* dst, vkt_int3 dims, int format, uint64_t seed,
                          int64_t z_offset, cudaStream_t s);

}  // namespace vkt
