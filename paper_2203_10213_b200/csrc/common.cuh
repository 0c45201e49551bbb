// common.cuh — shared device helpers for the ApplyFilter / Fill kernels.
//
// Semantics follow the reference hot path pkg/src/vkt/ops/filters.py:69-95:
//   out(c) = sum_{dz,dy,dx} w[dz,dy,dx] * in(map(c + d - r))
// accumulated in the fixed (dz, dy, dx) tap order (filters.py:89-92) and
// re-quantized with floor(clip(t,0,1)*max + 0.5) (volume.py:102-110).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "../../include/vkt_b200.h"

// NVTX ranges around the ABI entry points (header-only NVTX3: a no-op
// unless a profiler injects itself, e.g. `nsys` / `ncu --nvtx`).
#ifndef VKT_NO_NVTX
#include <nvtx3/nvToolsExt.h>
namespace vkt {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace vkt
#define VKT_NVTX(name) const ::vkt::NvtxRange vkt_nvtx_range_(name)
#else
#define VKT_NVTX(name) ((void)0)
#endif

namespace vkt {

// ----------------------------------------------------------------------------
// Address modes. map_index returns the in-range index, or -1 for Border
// (which contributes stored value 0 == mapped `lo`).
//   Clamp  : np.pad mode="edge"       (the reference, filters.py:78)
//   Wrap   : np.pad mode="wrap"       i mod n
//   Mirror : np.pad mode="symmetric"  edge-duplicating reflection, any r
//   Border : np.pad mode="constant"   stored 0
// ----------------------------------------------------------------------------
template <int MODE>
__host__ __device__ __forceinline__ int64_t map_index(int64_t i, int64_t n) {
  if (i >= 0 && i < n) return i;
  if constexpr (MODE == VKT_CLAMP) {
    return i < 0 ? 0 : n - 1;
  } else if constexpr (MODE == VKT_WRAP) {
    int64_t m = i % n;
    return m < 0 ? m + n : m;
  } else if constexpr (MODE == VKT_MIRROR) {
    int64_t p = 2 * n;
    int64_t m = i % p;
    if (m < 0) m += p;
    return m < n ? m : p - 1 - m;
  } else {
    return -1;
  }
}

// Single-fold variant, exact when -n <= i < 2n (a halo overshooting the
// volume by at most n cells): no integer division.
template <int MODE>
__host__ __device__ __forceinline__ int map_index_near(int i, int n) {
  if constexpr (MODE == VKT_CLAMP) {
    return i < 0 ? 0 : (i >= n ? n - 1 : i);
  } else if constexpr (MODE == VKT_WRAP) {
    return i < 0 ? i + n : (i >= n ? i - n : i);
  } else if constexpr (MODE == VKT_MIRROR) {
    return i < 0 ? -1 - i : (i >= n ? 2 * n - 1 - i : i);
  } else {
    return (i >= 0 && i < n) ? i : -1;
  }
}

// 32-bit variant for the x/y axes (extents < 2^31).
template <int MODE>
__host__ __device__ __forceinline__ int map_index32(int i, int n) {
  if (i >= 0 && i < n) return i;
  if constexpr (MODE == VKT_CLAMP) {
    return i < 0 ? 0 : n - 1;
  } else if constexpr (MODE == VKT_WRAP) {
    int m = i % n;
    return m < 0 ? m + n : m;
  } else if constexpr (MODE == VKT_MIRROR) {
    int p = 2 * n;
    int m = i % p;
    if (m < 0) m += p;
    return m < n ? m : p - 1 - m;
  } else {
    return -1;
  }
}

// ----------------------------------------------------------------------------
// z-plane resolution for a (possibly sharded) slab.  `e` is a local extended
// plane index in [-rz, nz + rz).  Returns a pointer to the plane, or nullptr
// for a Border plane (all stored zeros).
// ----------------------------------------------------------------------------
struct SlabGeom {
  const void* src;
  const void* halo_lo;
  const void* halo_hi;
  int64_t plane_elems;  // nx * ny
  int nz;               // local planes
  int rz;
  int64_t z_offset;
  int64_t global_nz;
};

template <int MODE, typename T>
__device__ __forceinline__ const T* resolve_plane(const SlabGeom& g, int e) {
  const T* src = static_cast<const T*>(g.src);
  if (e >= 0 && e < g.nz) return src + (int64_t)e * g.plane_elems;
  if (e < 0 && g.halo_lo != nullptr)
    return static_cast<const T*>(g.halo_lo) + (int64_t)(e + g.rz) * g.plane_elems;
  if (e >= g.nz && g.halo_hi != nullptr)
    return static_cast<const T*>(g.halo_hi) + (int64_t)(e - g.nz) * g.plane_elems;
  int64_t m = map_index<MODE>(g.z_offset + e, g.global_nz);
  if (m < 0) return nullptr;
  return src + (m - g.z_offset) * g.plane_elems;
}

// ----------------------------------------------------------------------------
// Stored value -> float in stored units.  u8/u16 use the exponent trick
// (0x4B000000 | v) - 2^23 which is exact for v < 2^23 and runs on the
// ALU + FMA pipes instead of the 16/clk conversion pipe.
// ----------------------------------------------------------------------------
__device__ __forceinline__ float to_f32(uint8_t v) {
  return __int_as_float(0x4B000000 | (uint32_t)v) - 8388608.0f;
}
__device__ __forceinline__ float to_f32(uint16_t v) {
  return __int_as_float(0x4B000000 | (uint32_t)v) - 8388608.0f;
}
__device__ __forceinline__ float to_f32(float v) { return v; }

template <typename T>
struct FormatTraits;
template <>
struct FormatTraits<uint8_t> {
  static constexpr int code = VKT_U8;
  static constexpr float max_f = 255.0f;
  static constexpr double max_d = 255.0;
  static constexpr bool is_int = true;
};
template <>
struct FormatTraits<uint16_t> {
  static constexpr int code = VKT_U16;
  static constexpr float max_f = 65535.0f;
  static constexpr double max_d = 65535.0;
  static constexpr bool is_int = true;
};
template <>
struct FormatTraits<float> {
  static constexpr int code = VKT_F32;
  static constexpr float max_f = 0.0f;
  static constexpr double max_d = 0.0;
  static constexpr bool is_int = false;
};

// ----------------------------------------------------------------------------
// Epilogue (fast path).  S = sum w_f32 * s_f32 in stored units, accumulated in
// the (dz, dy, dx) tap order.
// Ints: t*max = S + c with c = lo*(sum_w - 1)/(hi - lo)*max computed in f64 on
// the host (SURVEY §8(c) "Epilogue restatement"), out = floor(clamp(.)+0.5).
// The accumulator STARTS at acc0 = fl(c + 0.5), so the epilogue is a
// saturating floor conversion (negatives -> 0) and one integer min.
// F32 volumes start at 0 and store the sum verbatim (quantize() is
// astype('<f4'), volume.py:106).  Every kernel path uses these two helpers,
// so all paths stay bit-identical.
// ----------------------------------------------------------------------------
template <typename T>
__host__ __device__ __forceinline__ float acc_init(float c) {
  if constexpr (FormatTraits<T>::is_int) return c + 0.5f;
  else return 0.0f;
}

template <typename T>
__device__ __forceinline__ T quantize_acc(float acc);

template <>
__device__ __forceinline__ uint8_t quantize_acc<uint8_t>(float acc) {
  return (uint8_t)min(__float2uint_rd(acc), 255u);
}
template <>
__device__ __forceinline__ uint16_t quantize_acc<uint16_t>(float acc) {
  return (uint16_t)min(__float2uint_rd(acc), 65535u);
}
template <>
__device__ __forceinline__ float quantize_acc<float>(float acc) {
  return acc;
}

// ----------------------------------------------------------------------------
// Checked builds (build.py --variant=checked -DVKT_CHECKS -DVKT_JITTER; never
// the product library).  compute-sanitizer is not available on the GPU pool,
// so the tiled kernels carry their own race / bounds evidence:
//  * VKT_CHECK: shared-memory offsets of staging, edge repair and compute are
//    bounds-checked; a violation prints the CTA and traps.
//  * VKT_JITTER_POINT: each warp sleeps a pseudo-random 0..4 us (one point in
//    four) at the synchronization points of the pipeline, so a missing wait
//    or a phase race changes the result; the parity suites then compare every
//    kernel against the oracle and the direct kernel under that jitter.
// ----------------------------------------------------------------------------
#ifdef VKT_CHECKS
#define VKT_CHECK(cond, what)                                                                  \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("VKT_CHECK failed: %s (cta %d,%d,%d thread %d)\n", what, (int)blockIdx.x,          \
             (int)blockIdx.y, (int)blockIdx.z, (int)threadIdx.x);                              \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define VKT_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif

#ifdef VKT_JITTER
__device__ __forceinline__ void vkt_jitter(uint32_t salt) {
  uint32_t h = blockIdx.x * 73856093u ^ blockIdx.y * 19349663u ^ blockIdx.z * 83492791u ^
               (threadIdx.x >> 5) * 2654435761u ^ salt * 40503u ^ (uint32_t)clock();
  h ^= h >> 13;
  h *= 0x5bd1e995u;
  h ^= h >> 15;
  if ((h & 3u) == 0) __nanosleep(h % 4096u);
}
#define VKT_JITTER_POINT(salt) vkt_jitter(salt)
#else
#define VKT_JITTER_POINT(salt) \
  do {                         \
  } while (0)
#endif

// Launch accounting (see vkt_launch_count).
void count_launch();

}  // namespace vkt
