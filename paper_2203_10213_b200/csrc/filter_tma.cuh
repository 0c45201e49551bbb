// filter_tma.cuh — tiled sm_100a ApplyFilter kernel.
//
// Design:
//  * A CTA owns a 64 (x) by 16 (y) column of outputs and a chunk of ZC output
//    planes.  It streams the input planes of that chunk through a ring of S
//    shared-memory stages; each stage is ONE TMA 3D box load
//    (cp.async.bulk.tensor.3d) of the plane's (64+2R) x (16+2R) footprint,
//    completed on an mbarrier (complete_tx).  One elected thread issues the
//    TMA for plane i+S-1 while all 256 threads compute plane i.
//  * Each thread owns 4 consecutive x outputs of one row and keeps K = 2R+1
//    rolling register accumulators per output, one per output plane the
//    current input plane contributes to (the "register-blocked run of
//    outputs along z").  Per input plane and row dy it loads the 4+2R inputs
//    once (128/64/32-bit LDS) and issues 4*K*K FFMAs with the weight as a
//    constant-bank operand (the weights are a by-value kernel parameter).
//  * Tap order per output is (dz, dy, dx) — the reference's order
//    (filters.py:89-92) and the direct kernel's — so every path and every
//    z-slab split produce bit-identical results.
//  * Boundary handling: Border = TMA's out-of-bounds zero fill (stored 0);
//    Clamp/Mirror/Wrap tiles on the volume edge overwrite their out-of-range
//    halo cells after the TMA lands ("fixup"), compile-time specialised per
//    mode; z is resolved per plane (local slab, halo buffer, or mapped plane).
//  * Integer voxels are widened with the exponent trick (ALU+FMA pipes) and
//    the epilogue quantizes as volume.py:102-110; outputs are stored with
//    streaming (evict-first) vector stores.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace vkt {
namespace tma {

constexpr int TX = 64;     // outputs per CTA in x
constexpr int TY = 16;     // outputs per CTA in y
constexpr int XPT = 4;     // outputs per thread in x
constexpr int THREADS = (TX / XPT) * TY;  // 256
constexpr int STAGES = 4;

// Box geometry shared by the host (tensor-map encode) and the kernel.
__host__ __device__ constexpr int box_align_left(int r, int bpc) {
  return (r + 16 / bpc - 1) / (16 / bpc) * (16 / bpc);
}
__host__ __device__ constexpr int box_width(int r, int bpc) {
  return (box_align_left(r, bpc) + TX + r + 16 / bpc - 1) / (16 / bpc) * (16 / bpc);
}

template <typename T, int R>
struct Geo {
  // TMA needs the innermost box coordinate at a 16-byte multiple (measured:
  // tools/tma_probe.cu), so the box starts A >= R cells left of the tile.
  static constexpr int AE = 16 / (int)sizeof(T);          // cells per 16 bytes
  static constexpr int A = box_align_left(R, (int)sizeof(T));  // aligned left halo
  static constexpr int BX = box_width(R, (int)sizeof(T));
  static constexpr int BY = TY + 2 * R;
  static constexpr int OFF = 4 - R;                        // row-load phase
  static constexpr int STAGE_BYTES = BX * BY * (int)sizeof(T);
  static constexpr int STAGE_PITCH = (STAGE_BYTES + 127) / 128 * 128;
  static constexpr int SMEM = STAGES * STAGE_PITCH + 128 + 128;  // + barriers + align slack
  static_assert(R >= 1 && R <= 4, "radius");
  static_assert(BX <= 256 && BY <= 256, "TMA box too large");
  static_assert(4 * (TX / XPT - 1) + A - 4 + 4 * ((OFF + XPT + 2 * R + 3) / 4) <= BX, "row over-read");
};

template <int K>
struct Weights {
  float w[K * K * K];
};

struct TmaParams {
  void* dst;
  const void* src;       // local slab (for fixup gathers)
  const void* halo_lo;
  const void* halo_hi;
  int nx, ny, nz;        // local extents
  int z_begin, z_end;    // local output planes [begin, end)
  int zc;                // output planes per CTA chunk
  int64_t z_offset, global_nz;
  float c;               // integer epilogue constant
};

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Plane source for local extended plane e: which map + coordinate, or a zero
// (Border) plane.  Also returns the global pointer for fixup gathers.
struct PlaneSrc {
  int which;  // 0 local, 1 halo_lo, 2 halo_hi, -1 zero plane
  int z;      // plane index within that tensor
};

template <int MODE>
__device__ __forceinline__ PlaneSrc resolve(const TmaParams& p, int R, int e) {
  if (e >= 0 && e < p.nz) return {0, e};
  if (e < 0 && p.halo_lo != nullptr) return {1, e + R};
  if (e >= p.nz && p.halo_hi != nullptr) return {2, e - p.nz};
  int64_t m = map_index<MODE>(p.z_offset + e, p.global_nz);
  if (m < 0) return {-1, 0};
  return {0, (int)(m - p.z_offset)};
}

template <typename T>
__device__ __forceinline__ const T* plane_ptr(const TmaParams& p, PlaneSrc s) {
  const int64_t pe = (int64_t)p.nx * p.ny;
  const void* base = s.which == 1 ? p.halo_lo : s.which == 2 ? p.halo_hi : p.src;
  return static_cast<const T*>(base) + (int64_t)s.z * pe;
}

// ---------------------------------------------------------------------------
// Row loads from shared memory: N consecutive cells starting OFF cells after
// a 4-cell-aligned address, widened to float.
// ---------------------------------------------------------------------------
template <typename T, int N, int OFF>
struct RowLoader;

template <int N, int OFF>
struct RowLoader<float, N, OFF> {
  __device__ __forceinline__ static void load(const float* row, float (&v)[N]) {
    constexpr int NV = (OFF + N + 3) / 4;
    float tmp[NV * 4];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float4 q = reinterpret_cast<const float4*>(row)[i];
      tmp[4 * i + 0] = q.x;
      tmp[4 * i + 1] = q.y;
      tmp[4 * i + 2] = q.z;
      tmp[4 * i + 3] = q.w;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = tmp[OFF + i];
  }
};

template <int N, int OFF>
struct RowLoader<uint16_t, N, OFF> {
  __device__ __forceinline__ static void load(const uint16_t* row, float (&v)[N]) {
    constexpr int NV = (OFF + N + 3) / 4;  // 8-byte loads of 4 cells
    uint32_t tmp[NV * 2];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      uint2 q = reinterpret_cast<const uint2*>(row)[i];
      tmp[2 * i + 0] = q.x;
      tmp[2 * i + 1] = q.y;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int c = OFF + i;
      uint32_t w = tmp[c >> 1];
      // place the 16-bit cell in the low mantissa of 2^23
      uint32_t bits = __byte_perm(w, 0x4B000000u, (c & 1) ? 0x7432 : 0x7410);
      v[i] = __int_as_float(bits) - 8388608.0f;
    }
  }
};

template <int N, int OFF>
struct RowLoader<uint8_t, N, OFF> {
  __device__ __forceinline__ static void load(const uint8_t* row, float (&v)[N]) {
    constexpr int NV = (OFF + N + 3) / 4;  // 4-byte loads of 4 cells
    uint32_t tmp[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) tmp[i] = reinterpret_cast<const uint32_t*>(row)[i];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int c = OFF + i;
      uint32_t w = tmp[c >> 2];
      uint32_t sel = 0x7440u | (uint32_t)(c & 3);
      v[i] = __int_as_float(__byte_perm(w, 0x4B000000u, sel)) - 8388608.0f;
    }
  }
};

template <typename T>
__device__ __forceinline__ void store4(T* out, const float (&acc)[XPT], float c);

template <>
__device__ __forceinline__ void store4<float>(float* out, const float (&a)[XPT], float) {
  __stcs(reinterpret_cast<float4*>(out), make_float4(a[0], a[1], a[2], a[3]));
}
template <>
__device__ __forceinline__ void store4<uint16_t>(uint16_t* out, const float (&a)[XPT], float c) {
  uint32_t q0 = quantize_f32<uint16_t>(a[0], c), q1 = quantize_f32<uint16_t>(a[1], c);
  uint32_t q2 = quantize_f32<uint16_t>(a[2], c), q3 = quantize_f32<uint16_t>(a[3], c);
  __stcs(reinterpret_cast<uint2*>(out), make_uint2(q0 | (q1 << 16), q2 | (q3 << 16)));
}
template <>
__device__ __forceinline__ void store4<uint8_t>(uint8_t* out, const float (&a)[XPT], float c) {
  uint32_t q0 = quantize_f32<uint8_t>(a[0], c), q1 = quantize_f32<uint8_t>(a[1], c);
  uint32_t q2 = quantize_f32<uint8_t>(a[2], c), q3 = quantize_f32<uint8_t>(a[3], c);
  __stcs(reinterpret_cast<unsigned int*>(out), q0 | (q1 << 8) | (q2 << 16) | (q3 << 24));
}

// One input plane's contribution to the K rolling accumulators.
// GUARD: skip slots whose output plane is outside the chunk (ramp up/down).
template <typename T, int K, bool GUARD>
__device__ __forceinline__ void plane_step(const T* __restrict__ stage, int tx, int ty,
                                           const Weights<K>& wt, float (&acc)[K][XPT], int first_slot,
                                           int last_slot) {
  constexpr int R = K / 2;
  constexpr int N = XPT + 2 * R;
  using G = Geo<T, R>;
#pragma unroll
  for (int dy = 0; dy < K; ++dy) {
    float v[N];
    RowLoader<T, N, G::OFF>::load(stage + (ty + dy) * G::BX + tx * XPT + G::A - 4, v);
#pragma unroll
    for (int m = 0; m < K; ++m) {
      if (GUARD && (m < first_slot || m > last_slot)) continue;
      const int dz = K - 1 - m;
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
        const float w = wt.w[(dz * K + dy) * K + dx];
#pragma unroll
        for (int j = 0; j < XPT; ++j) acc[m][j] = __fmaf_rn(w, v[j + dx], acc[m][j]);
      }
    }
  }
}

template <typename T, int K, int MODE>
__global__ void __launch_bounds__(THREADS, 2)
    filter_tma_kernel(const __grid_constant__ CUtensorMap map_src,
                      const __grid_constant__ CUtensorMap map_lo,
                      const __grid_constant__ CUtensorMap map_hi, const TmaParams p,
                      const Weights<K> wt) {
  constexpr int R = K / 2;
  using G = Geo<T, R>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // TMA destinations must be 128-byte aligned; do not rely on the base.
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * G::STAGE_PITCH);

  const int tid = threadIdx.x;
  const int tx = tid % (TX / XPT);
  const int ty = tid / (TX / XPT);
  const int x0 = blockIdx.x * TX;
  const int y0 = blockIdx.y * TY;
  const int zo0 = p.z_begin + blockIdx.z * p.zc;
  const int nzo = min(p.zc, p.z_end - zo0);
  if (nzo <= 0) return;
  const int np = nzo + 2 * R;  // input planes of this chunk
  const bool edge = (x0 - R < 0) || (x0 + TX + R > p.nx) || (y0 - R < 0) || (y0 + TY + R > p.ny);

  if (tid == 0) {
    prefetch_tmap(&map_src);
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto produce = [&](int i) {
    const int s = i % STAGES;
    const PlaneSrc src = resolve<MODE>(p, R, zo0 - R + i);
    T* dst = reinterpret_cast<T*>(smem + s * G::STAGE_PITCH);
    if (src.which < 0) {
      mbar_arrive(&bars[s]);  // zero plane: consumers clear the stage
      return;
    }
    const CUtensorMap* m = src.which == 0 ? &map_src : src.which == 1 ? &map_lo : &map_hi;
    mbar_arrive_tx(&bars[s], G::STAGE_BYTES);
    tma_load_3d(dst, m, &bars[s], x0 - G::A, y0 - R, src.z);
  };

  if (tid == 0) {
    for (int i = 0; i < STAGES - 1 && i < np; ++i) produce(i);
  }

  float acc[K][XPT];
#pragma unroll
  for (int m = 0; m < K; ++m)
#pragma unroll
    for (int j = 0; j < XPT; ++j) acc[m][j] = 0.0f;

  const int ox = x0 + tx * XPT;
  const int oy = y0 + ty;
  const bool out_ok = (ox < p.nx) && (oy < p.ny);
  T* out_base = static_cast<T*>(p.dst) + (int64_t)oy * p.nx + ox;
  const int64_t plane_elems = (int64_t)p.nx * p.ny;

  for (int i = 0; i < np; ++i) {
    if (tid == 0 && i + STAGES - 1 < np) produce(i + STAGES - 1);
    const int s = i % STAGES;
    T* stage = reinterpret_cast<T*>(smem + s * G::STAGE_PITCH);
    mbar_wait(&bars[s], (uint32_t)((i / STAGES) & 1));

    const PlaneSrc src = resolve<MODE>(p, R, zo0 - R + i);
    if (src.which < 0) {
      // Border zero plane (stored 0)
      uint32_t* w = reinterpret_cast<uint32_t*>(stage);
      for (int q = tid; q < G::STAGE_BYTES / 4; q += THREADS) w[q] = 0u;
      __syncthreads();
    } else if (MODE != VKT_BORDER && edge) {
      // out-of-range halo cells: gather the address-mapped cell
      const T* plane = plane_ptr<T>(p, src);
      constexpr int W = TX + 2 * R;  // cells actually read: box x in [A-R, A+TX+R)
      for (int q = tid; q < G::BY * W; q += THREADS) {
        const int by = q / W, bx = q - by * W + (G::A - R);
        const int gx = x0 - G::A + bx, gy = y0 - R + by;
        if (gx >= 0 && gx < p.nx && gy >= 0 && gy < p.ny) continue;
        const int mx = map_index32<MODE>(gx, p.nx);
        const int my = map_index32<MODE>(gy, p.ny);
        stage[by * G::BX + bx] = __ldg(plane + (int64_t)my * p.nx + mx);
      }
      __syncthreads();
    }

    // slot m <-> output plane zo0 + i - 2R + m (chunk-relative i - 2R + m)
    const int first = 2 * R - i;          // first valid slot
    const int last = nzo - 1 - i + 2 * R;  // last valid slot
    if (first <= 0 && last >= K - 1)
      plane_step<T, K, false>(stage, tx, ty, wt, acc, 0, K - 1);
    else
      plane_step<T, K, true>(stage, tx, ty, wt, acc, first, last);

    if (i >= 2 * R && out_ok) {
      const int oz = zo0 + i - 2 * R;
      store4<T>(out_base + (int64_t)oz * plane_elems, acc[0], p.c);
    }
#pragma unroll
    for (int m = 0; m < K - 1; ++m)
#pragma unroll
      for (int j = 0; j < XPT; ++j) acc[m][j] = acc[m + 1][j];
#pragma unroll
    for (int j = 0; j < XPT; ++j) acc[K - 1][j] = 0.0f;

    __syncthreads();  // stage s is free for plane i + STAGES
    if (tid == 0) fence_proxy_async();
  }
}

template <typename T, int K, int MODE>
cudaError_t launch_tma_kernel(const CUtensorMap& ms, const CUtensorMap& ml, const CUtensorMap& mh,
                              const TmaParams& p, const float* w32, dim3 grid, cudaStream_t s) {
  using G = Geo<T, K / 2>;
  Weights<K> wt;
  for (int i = 0; i < K * K * K; ++i) wt.w[i] = w32[i];
  auto fn = filter_tma_kernel<T, K, MODE>;
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  if (err != cudaSuccess) return err;
  fn<<<grid, THREADS, G::SMEM, s>>>(ms, ml, mh, p, wt);
  return cudaGetLastError();
}

// Per-dtype dispatch over K and MODE (instantiated in filter_tma_<dtype>.cu).
template <typename T>
cudaError_t launch_tma_dtype(int k, int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                             const CUtensorMap& mh, const TmaParams& p, const float* w32, dim3 grid,
                             cudaStream_t s) {
#define VKT_TMA_CASE(KK, MM) \
  if (k == KK && mode == MM) return launch_tma_kernel<T, KK, MM>(ms, ml, mh, p, w32, grid, s);
#define VKT_TMA_K(KK)               \
  VKT_TMA_CASE(KK, VKT_WRAP)        \
  VKT_TMA_CASE(KK, VKT_MIRROR)      \
  VKT_TMA_CASE(KK, VKT_CLAMP)       \
  VKT_TMA_CASE(KK, VKT_BORDER)
  VKT_TMA_K(3)
  VKT_TMA_K(5)
  VKT_TMA_K(7)
#undef VKT_TMA_K
#undef VKT_TMA_CASE
  return cudaErrorInvalidValue;
}

}  // namespace tma
}  // namespace vkt
