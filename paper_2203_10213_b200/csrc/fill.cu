// fill.cu — FillRange (pkg/src/vkt/ops/core.py:39-55) and the synthetic input
// generator.  The host quantizes the fill value once with the reference rule
// (volume.py:102-110) and passes the stored bit pattern, so the device side is
// a pure box store: bit-exact by construction.
#include "common.cuh"
#include "dispatch.h"

namespace vkt {

// A box decomposes into n_seg_y * n_seg_z contiguous segments of seg_bytes;
// whole-row / whole-plane boxes are merged into longer segments on the host.
struct FillParams {
  uint8_t* base;        // address of the first cell of the box
  int64_t seg_bytes;
  int64_t stride_y;     // bytes between consecutive y segments
  int64_t stride_z;     // bytes between consecutive z segments
  int64_t n_seg_y;
  int64_t n_seg_z;
  int64_t chunks_per_seg;
  uint32_t pattern;     // 4-byte replicated stored value
  int bpc;
};

static constexpr int64_t kFillChunk = 32768;  // bytes per CTA work item

// Short segments (partial rows of a FillRange box): one warp per segment.
__global__ void __launch_bounds__(256) fill_rows_kernel(FillParams p) {
  const int64_t nseg = p.n_seg_y * p.n_seg_z;
  const uint4 vec = make_uint4(p.pattern, p.pattern, p.pattern, p.pattern);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t seg = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; seg < nseg; seg += warps) {
    const int64_t sy = seg % p.n_seg_y;
    const int64_t sz = seg / p.n_seg_y;
    uint8_t* lo = p.base + sz * p.stride_z + sy * p.stride_y;
    uint8_t* hi = lo + p.seg_bytes;
    uint8_t* vlo = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(lo) + 15) & ~uintptr_t(15));
    uint8_t* vhi = reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(hi) & ~uintptr_t(15));
    if (vlo > vhi) { vlo = hi; vhi = hi; }
    const int64_t head_cells = (vlo - lo) / p.bpc;
    const int64_t tail_cells = (hi - vhi) / p.bpc;
    for (int64_t i = lane; i < head_cells + tail_cells; i += 32) {
      uint8_t* c = i < head_cells ? lo + i * p.bpc : vhi + (i - head_cells) * p.bpc;
      if (p.bpc == 1) *c = (uint8_t)p.pattern;
      else if (p.bpc == 2) *reinterpret_cast<uint16_t*>(c) = (uint16_t)p.pattern;
      else *reinterpret_cast<uint32_t*>(c) = p.pattern;
    }
    uint4* v = reinterpret_cast<uint4*>(vlo);
    const int64_t nv = (vhi - vlo) / 16;
    for (int64_t i = lane; i < nv; i += 32) __stcs(v + i, vec);
  }
}

// Short segments whose rows and planes are 16-byte multiples (the usual
// FillRange box): every segment has the same alignment phase, so the work
// flattens into (segment, item) pairs -- item < nvec is a 16-byte store,
// the rest are the head / tail cells -- one per thread, all lanes busy.
// (A warp per 256-byte segment left half the lanes idle: 15 us for the
// 256^3 u8 box of the teaser, ~1 TB/s.)
__global__ void __launch_bounds__(256) fill_segs_kernel(FillParams p, int head_b, int nvec,
                                                         int ncell) {
  const int per_seg = nvec + ncell;
  const int64_t total = p.n_seg_y * p.n_seg_z * per_seg;
  const uint4 vec = make_uint4(p.pattern, p.pattern, p.pattern, p.pattern);
  const int head_cells = head_b / p.bpc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t seg = t / per_seg;
    const int k = (int)(t - seg * per_seg);
    const int64_t sy = seg % p.n_seg_y;
    const int64_t sz = seg / p.n_seg_y;
    uint8_t* lo = p.base + sz * p.stride_z + sy * p.stride_y;
    if (k < nvec) {
      __stcs(reinterpret_cast<uint4*>(lo + head_b) + k, vec);
    } else {
      const int c = k - nvec;
      uint8_t* cell = c < head_cells ? lo + c * p.bpc : lo + head_b + 16 * nvec + (c - head_cells) * p.bpc;
      if (p.bpc == 1) *cell = (uint8_t)p.pattern;
      else if (p.bpc == 2) *reinterpret_cast<uint16_t*>(cell) = (uint16_t)p.pattern;
      else *reinterpret_cast<uint32_t*>(cell) = p.pattern;
    }
  }
}

__global__ void __launch_bounds__(256) fill_box_kernel(FillParams p) {
  const int64_t items = p.n_seg_y * p.n_seg_z * p.chunks_per_seg;
  const uint4 vec = make_uint4(p.pattern, p.pattern, p.pattern, p.pattern);
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t seg = it / p.chunks_per_seg;
    const int64_t chunk = it - seg * p.chunks_per_seg;
    const int64_t sy = seg % p.n_seg_y;
    const int64_t sz = seg / p.n_seg_y;
    uint8_t* seg_base = p.base + sz * p.stride_z + sy * p.stride_y;
    const int64_t b0 = chunk * kFillChunk;
    const int64_t b1 = min(p.seg_bytes, b0 + kFillChunk);
    uint8_t* lo = seg_base + b0;
    uint8_t* hi = seg_base + b1;
    // 16-byte aligned middle; the pattern has period bpc | 16, and the
    // segment base is bpc-aligned, so phases line up with cell boundaries.
    uint8_t* vlo = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(lo) + 15) & ~uintptr_t(15));
    uint8_t* vhi = reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(hi) & ~uintptr_t(15));
    if (vlo > vhi) { vlo = hi; vhi = hi; }
    // head / tail cells
    const int64_t head_cells = (vlo - lo) / p.bpc;
    const int64_t tail_cells = (hi - vhi) / p.bpc;
    for (int64_t i = threadIdx.x; i < head_cells + tail_cells; i += blockDim.x) {
      uint8_t* c = i < head_cells ? lo + i * p.bpc : vhi + (i - head_cells) * p.bpc;
      if (p.bpc == 1) *c = (uint8_t)p.pattern;
      else if (p.bpc == 2) *reinterpret_cast<uint16_t*>(c) = (uint16_t)p.pattern;
      else *reinterpret_cast<uint32_t*>(c) = p.pattern;
    }
    uint4* v = reinterpret_cast<uint4*>(vlo);
    const int64_t nv = (vhi - vlo) / 16;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) __stcs(v + i, vec);
  }
}

int launch_fill_box(void* dst, vkt_int3 dims, int format, vkt_int3 lo, vkt_int3 hi,
                    uint32_t bits, cudaStream_t s) {
  const int bpc = format == VKT_U8 ? 1 : format == VKT_U16 ? 2 : 4;
  // clip_box (geom.py:99-103)
  int x0 = lo.x > 0 ? lo.x : 0, y0 = lo.y > 0 ? lo.y : 0, z0 = lo.z > 0 ? lo.z : 0;
  int x1 = hi.x < dims.x ? hi.x : dims.x, y1 = hi.y < dims.y ? hi.y : dims.y,
      z1 = hi.z < dims.z ? hi.z : dims.z;
  if (x1 <= x0 || y1 <= y0 || z1 <= z0) return VKT_OK;  // empty roi: no-op (core.py:48-49)

  uint32_t pat;
  if (bpc == 1) pat = (bits & 0xFFu) * 0x01010101u;
  else if (bpc == 2) pat = (bits & 0xFFFFu) | ((bits & 0xFFFFu) << 16);
  else pat = bits;

  const int64_t row_b = (int64_t)dims.x * bpc;
  const int64_t plane_b = row_b * dims.y;
  FillParams p{};
  p.bpc = bpc;
  p.pattern = pat;
  p.base = static_cast<uint8_t*>(dst) + (int64_t)z0 * plane_b + (int64_t)y0 * row_b + (int64_t)x0 * bpc;
  const bool full_x = (x0 == 0 && x1 == dims.x);
  const bool full_y = (y0 == 0 && y1 == dims.y);
  if (full_x && full_y) {
    p.seg_bytes = plane_b * (z1 - z0);
    p.n_seg_y = 1;
    p.n_seg_z = 1;
  } else if (full_x) {
    p.seg_bytes = row_b * (y1 - y0);
    p.n_seg_y = 1;
    p.n_seg_z = z1 - z0;
  } else {
    p.seg_bytes = (int64_t)(x1 - x0) * bpc;
    p.n_seg_y = y1 - y0;
    p.n_seg_z = z1 - z0;
  }
  p.stride_y = row_b;
  p.stride_z = plane_b;
  p.chunks_per_seg = (p.seg_bytes + kFillChunk - 1) / kFillChunk;
  const int64_t items = p.n_seg_y * p.n_seg_z * p.chunks_per_seg;
  if (p.seg_bytes <= 4096 && row_b % 16 == 0 && plane_b % 16 == 0) {
    const int head_b = (int)((16 - (reinterpret_cast<uintptr_t>(p.base) & 15u)) & 15u);
    const int hb = head_b < p.seg_bytes ? head_b : (int)p.seg_bytes;
    const int nvec = (int)((p.seg_bytes - hb) / 16);
    const int ncell = (int)((p.seg_bytes - 16 * (int64_t)nvec) / bpc);
    const int64_t total = p.n_seg_y * p.n_seg_z * (nvec + ncell);
    const int64_t blocks = (total + 255) / 256;
    fill_segs_kernel<<<(int)(blocks < sm_count() * 16 ? blocks : sm_count() * 16), 256, 0, s>>>(p, hb, nvec, ncell);
  } else if (p.seg_bytes <= 4096) {
    const int64_t nseg = p.n_seg_y * p.n_seg_z;
    const int64_t blocks = (nseg + 7) / 8;
    fill_rows_kernel<<<(int)(blocks < sm_count() * 16 ? blocks : sm_count() * 16), 256, 0, s>>>(p);
  } else {
    int grid = (int)(items < sm_count() * 16 ? items : sm_count() * 16);
    fill_box_kernel<<<grid, 256, 0, s>>>(p);
  }
  count_launch();
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    set_error_detail("fill_box launch: %s", cudaGetErrorString(err));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}

// ---------------------------------------------------------------------------
// Synthetic inputs: splitmix64(seed ^ global linear index).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void __launch_bounds__(256) synthetic_kernel(T* dst, int64_t n, int64_t first, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = splitmix64(seed * 0xD1B54A32D192ED03ull + (uint64_t)(first + i));
    if constexpr (sizeof(T) == 1) dst[i] = (T)(h >> 56);
    else if constexpr (sizeof(T) == 2) dst[i] = (T)(h >> 48);
    else dst[i] = (float)(h >> 40) * (1.0f / 16777216.0f);
  }
}

int launch_fill_synthetic(void* dst, vkt_int3 dims, int format, uint64_t seed,
                          int64_t z_offset, cudaStream_t s) {
  const int64_t n = (int64_t)dims.x * dims.y * dims.z;
  if (n == 0) return VKT_OK;
  const int64_t first = z_offset * (int64_t)dims.x * dims.y;
  int grid = sm_count() * 8;
  if (format == VKT_U8) synthetic_kernel<uint8_t><<<grid, 256, 0, s>>>((uint8_t*)dst, n, first, seed);
  else if (format == VKT_U16) synthetic_kernel<uint16_t><<<grid, 256, 0, s>>>((uint16_t*)dst, n, first, seed);
  else synthetic_kernel<float><<<grid, 256, 0, s>>>((float*)dst, n, first, seed);
  count_launch();
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    set_error_detail("fill_synthetic launch: %s", cudaGetErrorString(err));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}

}  // namespace vkt
