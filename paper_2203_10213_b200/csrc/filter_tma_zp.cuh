// filter_tma_zp.cuh — the f32 K = 3 variant of the tiled kernel.
//
// TMA lands directly in the row-major ready stage (no staging pass), and
// K-1 of the K accumulator slots are paired along z (FFMA2 with a broadcast
// input and a weight pair) while the last slot is a plain FFMA.  For the
// HBM-bound f32 K = 3 skipping the staging pass outweighs the all-FFMA2
// packing of filter_tma.cuh (measured, 1024^3: 1.71 vs 2.03 ms).  f32 K = 5
// moved to filter_tma.cuh once its ready stage was bank-conflict free and its
// dy loop unrolled (4.28 vs 4.96 ms); the K = 5 code below is kept
// compilable but is not instantiated.  Same tensor map as
// filter_tma.cuh for f32 (box 136 x (TY+2R)); the u8/u16 code paths below
// are not instantiated.
//
// Design:
//  * A CTA owns a TX=128 (x) by TY=16 (y) column of outputs and a chunk of ZC
//    output planes, and streams the chunk's input planes through shared
//    memory.  Each input plane is ONE TMA 3D box load
//    (cp.async.bulk.tensor.3d, completion on an mbarrier with complete_tx) of
//    the plane's footprint plus its halo.
//  * No dedicated producer warp (it would leave its SM sub-partition with
//    fewer FMA warps than the other three, measured: 85% issue).  All 8 warps
//    compute, and each also does 1/8 of the staging of the NEXT plane:
//    repairing the out-of-volume halo cells of edge tiles for Clamp / Mirror
//    / Wrap (Border is TMA's zero fill = stored 0) and, for u8/u16 volumes,
//    widening the raw TMA plane to float once per cell into a "ready" stage.
//    Lane 0 of warp 0 issues the TMA loads.  Warps meet only on mbarriers
//    (full / ready / empty rings); there is no CTA-wide barrier per plane.
//  * Compute warps: each thread owns 8 consecutive x outputs of one row and
//    keeps K = 2R+1 rolling register accumulators per output — one per output
//    plane the current input plane contributes to (the register-blocked run of
//    outputs along z).  Per input plane the dy loop stays rolled (the body is
//    ~K*K*8 FFMAs, small enough for the instruction cache); each dy iteration
//    loads 16 floats of the input row (4 x LDS.128) and issues 8*K*K FFMAs
//    whose weight operand is a uniform register (LDCU from the by-value
//    kernel-parameter block, rows padded to 16 bytes).
//  * Tap order per output is (dz, dy, dx) — the reference's order
//    (filters.py:89-92) and the direct kernel's — so every kernel path and
//    every z-slab split produce bit-identical results.
//  * Epilogue: quantize as volume.py:102-110 (ints) and store with streaming
//    (evict-first) 128-bit stores.
#pragma once

#include <cuda.h>

#include <atomic>

#include "common.cuh"

namespace vkt {
namespace tma_zp {

constexpr int TX = 128;          // outputs per CTA in x
constexpr int TY = 16;           // outputs per CTA in y
constexpr int XPT = 8;           // outputs per thread in x

// Thread layout per kernel extent (measured):
//  K <= 5: 2 output rows per thread (each weight load feeds 16 FFMAs), 4 warps,
//          3 CTAs/SM (3 warps per SMSP, 168 registers);
//  K == 7: 1 row per thread (the 2-row variant needs 112 accumulators and
//          loses latency hiding), 8 warps, 2 CTAs/SM (4 warps/SMSP, 128 regs).
// Warps per SM stay a multiple of 4 so every SM sub-partition gets the same
// number of FMA warps.
template <int K, int MODE = VKT_CLAMP>
struct Layout {
  static constexpr int YPT = K <= 5 ? 2 : 1;
  static constexpr int WARPS = TY * (TX / XPT) / (32 * YPT);
  static constexpr int THREADS = 32 * WARPS;
  // K = 3: 4 CTAs/SM (122 registers, 56 KB rings): Clamp 1.49 vs 1.57 ms at
  // 1024^3; Wrap keeps 3 (its prefetch registers spill at 128)
  static constexpr int CTAS_PER_SM = K <= 3 ? (MODE == VKT_WRAP ? 3 : 4) : K <= 5 ? 3 : 2;
  static constexpr int WROWS = TY / WARPS;  // output rows per warp
  static constexpr int SMEM_PER_CTA = (228 * 1024) / CTAS_PER_SM - 1024;  // minus driver reserve
};
constexpr int RP = TX + 8;       // ready-stage row pitch (floats): x in [x0-4, x0+TX+4)

// Raw TMA box geometry (shared by the host tensor-map encode and the kernel).
// TMA needs the innermost box coordinate at a 16-byte multiple (measured with
// tools/tma_probe.cu), so the box starts A >= R cells left of the tile.
__host__ __device__ constexpr int box_align_left(int r, int bpc) {
  return (r + 16 / bpc - 1) / (16 / bpc) * (16 / bpc);
}
__host__ __device__ constexpr int box_width(int r, int bpc) {
  return (box_align_left(r, bpc) + TX + r + 16 / bpc - 1) / (16 / bpc) * (16 / bpc);
}

template <typename T, int K, int MODE = VKT_CLAMP>
struct Cfg {
  using L = Layout<K, MODE>;
  static constexpr int R = K / 2;
  static constexpr bool IS_F32 = sizeof(T) == 4;
  static constexpr int A = box_align_left(R, (int)sizeof(T));
  static constexpr int BX = box_width(R, (int)sizeof(T));
  static constexpr int BY = TY + 2 * R;
  static constexpr int RAW_BYTES = BX * BY * (int)sizeof(T);
  static constexpr int RAW_PITCH = (RAW_BYTES + 127) / 128 * 128;
  static constexpr int RDY_BYTES = RP * BY * 4;
  static constexpr int RDY_PITCH = (RDY_BYTES + 127) / 128 * 128;
  // Ring depths: as deep as fits CTAS_PER_SM CTAs per SM (f32: the TMA lands
  // in the ready ring, so it is also the TMA lookahead; ints: 4 ready stages
  // and the rest of the budget as raw TMA stages), capped at 10.
  static constexpr int BUDGET = L::SMEM_PER_CTA - 512;
  // ints: up to 6 ready stages (AHEAD planes converted ahead of compute leave
  // S_RDY - AHEAD - 1 planes of slack between the fastest and slowest warp),
  // keeping room for >= 5 raw TMA stages
  static constexpr int S_RDY_INT_FIT = (BUDGET - 5 * RAW_PITCH) / RDY_PITCH;
  static constexpr int S_RDY_INT = S_RDY_INT_FIT < 4 ? 4 : (S_RDY_INT_FIT > 6 ? 6 : S_RDY_INT_FIT);
  static constexpr int S_RDY = IS_F32 ? (BUDGET / RDY_PITCH < 10 ? BUDGET / RDY_PITCH : 10) : S_RDY_INT;
  static constexpr int S_RAW_FIT = IS_F32 ? 0 : (BUDGET - S_RDY * RDY_PITCH) / RAW_PITCH;
  static constexpr int S_RAW = IS_F32 ? 0 : (S_RAW_FIT < 10 ? S_RAW_FIT : 10);
  static constexpr int AHEAD = 2;  // ints: planes converted ahead of compute
  // f32: at iteration i the TMA slot of plane i - LAG is refilled (every warp
  // must have released it): larger LAG = more slack between warps, smaller
  // TMA lookahead (S_RDY - LAG).  K = 3 is HBM-bound and needs the lookahead.
  static constexpr int LAG = K == 3 ? 2 : 3;
  static constexpr int SMEM_DATA = S_RDY * RDY_PITCH + S_RAW * RAW_PITCH;
  static constexpr int NBAR = 2 * S_RDY + 2 * (IS_F32 ? S_RDY : S_RAW);
  static constexpr int SMEM = SMEM_DATA + NBAR * 8 + 128;
  static_assert(!IS_F32 || BX == RP, "f32 TMA box must match the ready layout");
  static_assert(R >= 1 && R <= 4, "radius");
  static_assert(IS_F32 ? S_RDY >= 4 : S_RAW >= 4, "ring too shallow");
  static_assert(SMEM <= L::SMEM_PER_CTA, "shared memory budget");
  static_assert(BX <= 256 && BY <= 256, "TMA box too large");
};

// Weights as a kernel-parameter block laid out for the paired accumulators
// (see plane_step): for each dy, NP = K/2 rows of K float2 pairs
// (w[dz_a][dy][dx], w[dz_b][dy][dx]) for accumulator slots (2p, 2p+1)
// (dz_a = K-1-2p, dz_b = K-2-2p), then the dz = 0 row for the unpaired slot
// K-1, padded to 16 bytes.  Each pair is one 64-bit uniform constant load.
template <int K>
struct alignas(16) Weights {
  static constexpr int NP = K / 2;
  static constexpr int KP = (K + 3) / 4 * 4;
  float2 wp[K * NP * K];
  float ws[K * KP];
};

// same layout as tma::TmaParams (copied at the dispatch, filter_tma_f32.cu)
struct TmaParams {
  void* dst;
  const void* src;
  const void* halo_lo;
  const void* halo_hi;
  int nx, ny, nz;
  int pitch;
  int z_begin, z_end;
  int zc;
  int64_t z_offset, global_nz;
  float c;
  uint32_t zskip;
  uint32_t yskip;
  const int* guard;
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
// The suspend-time hint lets a waiting warp sleep until the phase completes
// instead of re-polling: a polling warp takes issue slots from the other
// warps of its SM sub-partition (measured: ~3% of all instructions).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(1000000)
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
// Predicated single-thread forms: executed by every thread of the CTA with
// the predicate true in exactly one, so the surrounding loop stays free of
// thread-divergent branches (ptxas then keeps the rolled dy loop's weight
// loads on the uniform datapath: LDCU + FFMA with a uniform-register operand).
__device__ __forceinline__ void mbar_arrive_if(uint64_t* bar, bool pred) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tsetp.ne.b32 P, %1, 0;\n\t"
      "@P mbarrier.arrive.shared::cta.b64 _, [%0];\n}" ::"r"(smem_u32(bar)),
      "r"((int)pred)
      : "memory");
}
__device__ __forceinline__ void tma_issue_if(void* dst, const CUtensorMap* map, uint64_t* bar,
                                             uint32_t bytes, int x, int y, int z, bool pred) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tsetp.ne.b32 P, %7, 0;\n\t"
      "@P fence.proxy.async.shared::cta;\n\t"
      "@P mbarrier.arrive.expect_tx.shared::cta.b64 _, [%5], %6;\n\t"
      "@P cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "r"(bytes),
      "r"((int)pred)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Plane source for local extended plane e (0 local, 1 halo_lo, 2 halo_hi,
// -1 Border zero plane) and its index within that tensor.
struct PlaneSrc {
  int which;
  int z;
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
  const int64_t pe = (int64_t)p.pitch * p.ny;
  const void* base = s.which == 1 ? p.halo_lo : s.which == 2 ? p.halo_hi : p.src;
  return static_cast<const T*>(base) + (int64_t)s.z * pe;
}

__device__ __forceinline__ float widen(float v) { return v; }
__device__ __forceinline__ float widen(uint16_t v) { return to_f32(v); }
__device__ __forceinline__ float widen(uint8_t v) { return to_f32(v); }

// Value of the (address-mapped) cell (gx, gy) of a plane; Border never calls.
template <typename T, int MODE>
__device__ __forceinline__ float gather_cell(const T* plane, const TmaParams& p, int gx, int gy) {
  const int mx = map_index32<MODE>(gx, p.nx);
  const int my = map_index32<MODE>(gy, p.ny);
  return widen(__ldg(plane + (int64_t)my * p.pitch + mx));
}

// ---------------------------------------------------------------------------
// Producer helpers
// ---------------------------------------------------------------------------
// Out-of-volume cells of the ready (f32) stage that outputs of this tile
// read: x in [x0-R, min(x0+TX,nx)+R), y in [y0-R, min(y0+TY,ny)+R), excluding
// in-volume cells.  Enumerated as full rows above/below the volume plus
// left/right strips.
struct EdgeCells {
  int xa, ya, w, top, nl, side, n_rows, total;
  __device__ __forceinline__ EdgeCells(const TmaParams& p, int x0, int y0, int R, int row_lo,
                                       int row_hi) {
    xa = x0 - R;
    const int xb = min(x0 + TX, p.nx) + R;
    ya = max(y0 - R, y0 - R + row_lo);
    const int yb = min(min(y0 + TY, p.ny) + R, y0 - R + row_hi);
    w = xb - xa;
    const int rows = max(0, yb - ya);
    top = min(rows, max(0, -ya));
    const int bot = min(rows - top, max(0, yb - p.ny));
    nl = max(0, -xa);
    side = nl + max(0, xb - p.nx);
    n_rows = (top + bot) * w;
    total = n_rows + (rows - top - bot) * side;
  }
  __device__ __forceinline__ void cell(const TmaParams& p, int q, int& gx, int& gy) const {
    if (q < n_rows) {
      const int r = q / w;
      gy = r < top ? ya + r : p.ny + (r - top);
      gx = xa + (q - r * w);
    } else {
      const int q2 = q - n_rows;
      const int r = q2 / side;
      const int c = q2 - r * side;
      gy = ya + top + r;
      gx = c < nl ? xa + c : p.nx + (c - nl);
    }
  }
};

// f32 stages: repair this thread's share (t of nt) of the edge cells.  Clamp
// and Mirror map every such cell onto an in-volume cell inside the staged box
// (R <= 4 < TX, TY), so those are shared-memory copies from cells the TMA
// delivered; Wrap maps to the opposite face and gathers from global memory
// (8 loads in flight per thread).  Border never calls (TMA zero fill).
template <int MODE, int R>
__device__ __forceinline__ void fixup_f32(float* stage, const float* plane, const TmaParams& p,
                                          int x0, int y0, int t, int nt, int row_lo, int row_hi) {
  // only rows [row_lo, row_hi) of the stage (a warp's read window)
  const EdgeCells ec(p, x0, y0, R, row_lo, row_hi);
  constexpr int B = 8;
  for (int base = t; base < ec.total; base += nt * B) {
    float val[B];
    int dst[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int q = base + b * nt;
      dst[b] = -1;
      if (q < ec.total) {
        int gx, gy;
        ec.cell(p, q, gx, gy);
        const int mx = map_index32<MODE>(gx, p.nx);
        const int my = map_index32<MODE>(gy, p.ny);
        dst[b] = (gy - y0 + R) * RP + (gx - x0 + 4);
        if constexpr (MODE == VKT_WRAP)
          val[b] = __ldg(plane + (int64_t)my * p.pitch + mx);
        else
          val[b] = stage[(my - y0 + R) * RP + (mx - x0 + 4)];
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (dst[b] >= 0) stage[dst[b]] = val[b];
  }
}

// Out-of-line copy for the rare Clamp / Mirror windows FixList does not cover
// (its registers stay out of the main loop's allocation).
template <int MODE, int R>
__device__ __noinline__ void fixup_f32_cold(float* stage, const float* plane, const TmaParams& p,
                                            int x0, int y0, int t, int nt, int row_lo, int row_hi) {
  fixup_f32<MODE, R>(stage, plane, p, x0, y0, t, nt, row_lo, row_hi);
}

// Clamp / Mirror, f32 stages: the out-of-volume cells of a warp's read window
// and their in-volume sources are the same on every plane (both inside the
// staged box), so each lane precomputes its share once — up to NB (dst, src)
// stage offsets — and a plane's repair is NB shared-memory copies.  Per plane
// the generic fixup_f32 re-derived the cells (integer divisions, address
// maps): f32 3^3 Clamp ran 15% behind Border, whose TMA zero fill needs no
// repair.  Windows with more than 32*NB such cells (volumes thinner than
// the halo) keep the generic path.
template <int MODE, int R>
struct FixList {
  static constexpr int NB = 6;
  int dst[NB], src[NB];
  bool ok = false;
  __device__ __forceinline__ FixList() {
#pragma unroll
    for (int b = 0; b < NB; ++b) dst[b] = -1, src[b] = 0;
  }
  __device__ __forceinline__ FixList(const TmaParams& p, int x0, int y0, int lane, int row_lo,
                                     int row_hi) {
    const EdgeCells ec(p, x0, y0, R, row_lo, row_hi);
    ok = ec.total <= 32 * NB;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int q = lane + 32 * b;
      dst[b] = -1;
      src[b] = 0;
      if (ok && q < ec.total) {
        int gx, gy;
        ec.cell(p, q, gx, gy);
        const int mx = map_index32<MODE>(gx, p.nx);
        const int my = map_index32<MODE>(gy, p.ny);
        dst[b] = (gy - y0 + R) * RP + (gx - x0 + 4);
        src[b] = (my - y0 + R) * RP + (mx - x0 + 4);
      }
    }
  }
  // sources are in-volume cells, destinations out-of-volume: disjoint
  __device__ __forceinline__ void apply(float* stage) const {
    float v[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) v[b] = dst[b] >= 0 ? stage[src[b]] : 0.f;
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (dst[b] >= 0) stage[dst[b]] = v[b];
  }
};

// Wrap, f32 stages: the sources of a window's out-of-volume cells are on the
// far faces of the plane, in global memory, at offsets fixed for the CTA.
// Each lane precomputes up to NB (stage offset, plane offset) pairs and
// gathers the NEXT plane's values while the current plane computes, so the
// global round trip is off the per-plane critical path (the per-plane
// gather in fixup_f32 stalled every plane of every edge tile).
template <int R>
struct WrapList {
  // 5 per lane covers a K = 3 window (one halo row of 130 cells plus 5 side
  // cells); at 4 CTAs/SM (128 registers) the list still spilled (1.76 vs
  // 1.55 ms), so Wrap keeps 3 CTAs/SM
  static constexpr int NB = 5;
  int dst[NB], off[NB];
  float val[NB];
  bool ok = false;
  __device__ __forceinline__ WrapList() {
#pragma unroll
    for (int b = 0; b < NB; ++b) dst[b] = -1, off[b] = 0, val[b] = 0.f;
  }
  __device__ __forceinline__ WrapList(const TmaParams& p, int x0, int y0, int lane, int row_lo,
                                      int row_hi) {
    const EdgeCells ec(p, x0, y0, R, row_lo, row_hi);
    ok = ec.total <= 32 * NB;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int q = lane + 32 * b;
      dst[b] = -1;
      off[b] = 0;
      val[b] = 0.f;
      if (ok && q < ec.total) {
        int gx, gy;
        ec.cell(p, q, gx, gy);
        dst[b] = (gy - y0 + R) * RP + (gx - x0 + 4);
        off[b] = map_index32<VKT_WRAP>(gy, p.ny) * p.pitch + map_index32<VKT_WRAP>(gx, p.nx);
      }
    }
  }
  __device__ __forceinline__ void gather(const float* plane) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (dst[b] >= 0) val[b] = __ldg(plane + off[b]);
  }
  __device__ __forceinline__ void apply(float* stage) const {
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (dst[b] >= 0) stage[dst[b]] = val[b];
  }
};

// u8/u16: this thread's share of the widening work, fixed for the whole CTA
// (the tile geometry is the same for every plane): quad q = t + k*nt covers
// ready cells [e, e+4) of stage row `by`.  Offsets are computed once; `slow`
// marks quads that hold out-of-volume cells of the read window.
template <typename T, int K, int NT>
struct QuadPlan {
  using C = Cfg<T, K>;
  static constexpr int QPR = RP / 4;  // quads per row
  static constexpr int NQ = QPR * C::BY;
  static constexpr int QPT = (NQ + NT - 1) / NT;
  // K = 7 runs at the 128-register budget: recompute instead of storing.
  static constexpr bool STORE = K <= 5;
  int rdy_[STORE ? QPT : 1];  // ready-stage float offset (-1: no quad)
  uint32_t slow_;             // bit k: quad k takes the per-cell edge path
  int t_, rows_lo_, rows_hi_, x_lo_, x_hi_;
  bool edge_;

  __device__ __forceinline__ QuadPlan(const TmaParams& p, int x0, int y0, bool edge, int t) {
    constexpr int R = C::R;
    t_ = t;
    edge_ = edge;
    rows_lo_ = max(0, R - y0);
    rows_hi_ = p.ny - y0 + R;
    x_lo_ = max(0, 4 - x0);
    x_hi_ = p.nx - x0 + 4;
    slow_ = 0;
    if constexpr (STORE) {
#pragma unroll
      for (int k = 0; k < QPT; ++k) {
        int ro;
        bool sl;
        compute(k, ro, sl);
        rdy_[k] = ro;
        slow_ |= (sl ? 1u : 0u) << k;
      }
    }
  }
  __device__ __forceinline__ void compute(int k, int& ro, bool& sl) const {
    const int q = t_ + k * NT;
    const int by = q / QPR, e = (q - by * QPR) * 4;
    ro = q < NQ ? by * RP + e : -1;
    sl = q < NQ && edge_ && (by < rows_lo_ || by >= rows_hi_ || e < x_lo_ || e + 4 > x_hi_);
  }
  __device__ __forceinline__ void get(int k, int& ro, bool& sl) const {
    if constexpr (STORE) {
      ro = rdy_[k];
      sl = (slow_ >> k) & 1u;
    } else {
      compute(k, ro, sl);
    }
  }
};

template <typename T, int MODE, int K, int NT>
__device__ __forceinline__ void convert_plane(float* rdy, const T* raw, const T* plane,
                                              const TmaParams& p, int x0, int y0,
                                              const QuadPlan<T, K, NT>& qp) {
  using C = Cfg<T, K>;
  constexpr int R = C::R;
#pragma unroll
  for (int k = 0; k < QuadPlan<T, K, NT>::QPT; ++k) {
    int ro;
    bool sl;
    qp.get(k, ro, sl);
    if (ro < 0) continue;
    const int by = ro / RP, e = ro - by * RP;
    const T* src = raw + by * C::BX + e + (C::A - 4);
    float f[4];
    if constexpr (sizeof(T) == 2) {
      const uint2 w = *reinterpret_cast<const uint2*>(src);
      f[0] = __int_as_float(__byte_perm(w.x, 0x4B000000u, 0x7410)) - 8388608.0f;
      f[1] = __int_as_float(__byte_perm(w.x, 0x4B000000u, 0x7432)) - 8388608.0f;
      f[2] = __int_as_float(__byte_perm(w.y, 0x4B000000u, 0x7410)) - 8388608.0f;
      f[3] = __int_as_float(__byte_perm(w.y, 0x4B000000u, 0x7432)) - 8388608.0f;
    } else {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(src);
      f[0] = __int_as_float(__byte_perm(w, 0x4B000000u, 0x7440)) - 8388608.0f;
      f[1] = __int_as_float(__byte_perm(w, 0x4B000000u, 0x7441)) - 8388608.0f;
      f[2] = __int_as_float(__byte_perm(w, 0x4B000000u, 0x7442)) - 8388608.0f;
      f[3] = __int_as_float(__byte_perm(w, 0x4B000000u, 0x7443)) - 8388608.0f;
    }
    if (MODE != VKT_BORDER && sl) {
      const int gy = y0 - R + by;
      const bool yo = gy < 0 || gy >= p.ny;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int gx = x0 - 4 + e + c;
        if ((yo || gx < 0 || gx >= p.nx) && gx >= x0 - R && gx < x0 + TX + R) {
          const int mx = map_index32<MODE>(gx, p.nx);
          const int my = map_index32<MODE>(gy, p.ny);
          if constexpr (MODE == VKT_WRAP)
            f[c] = widen(__ldg(plane + (int64_t)my * p.pitch + mx));
          else
            f[c] = widen(raw[(my - y0 + R) * C::BX + (mx - x0 + C::A)]);
        }
      }
    }
    *reinterpret_cast<float4*>(rdy + ro) = make_float4(f[0], f[1], f[2], f[3]);
  }
}

// ---------------------------------------------------------------------------
// Compute helpers
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void store8(T* out, const float (&a)[XPT], int valid);

template <>
__device__ __forceinline__ void store8<float>(float* out, const float (&a)[XPT], int valid) {
  if (valid >= 4) __stcs(reinterpret_cast<float4*>(out), make_float4(a[0], a[1], a[2], a[3]));
  if (valid >= 8) __stcs(reinterpret_cast<float4*>(out) + 1, make_float4(a[4], a[5], a[6], a[7]));
}
template <>
__device__ __forceinline__ void store8<uint16_t>(uint16_t* out, const float (&a)[XPT], int) {
  uint32_t q[XPT];
#pragma unroll
  for (int j = 0; j < XPT; ++j) q[j] = quantize_acc<uint16_t>(a[j]);
  __stcs(reinterpret_cast<uint4*>(out),
         make_uint4(q[0] | (q[1] << 16), q[2] | (q[3] << 16), q[4] | (q[5] << 16), q[6] | (q[7] << 16)));
}
template <>
__device__ __forceinline__ void store8<uint8_t>(uint8_t* out, const float (&a)[XPT], int) {
  uint32_t q[XPT];
#pragma unroll
  for (int j = 0; j < XPT; ++j) q[j] = quantize_acc<uint8_t>(a[j]);
  __stcs(reinterpret_cast<uint2*>(out), make_uint2(q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24),
                                                   q[4] | (q[5] << 8) | (q[6] << 16) | (q[7] << 24)));
}

// Packed fp32x2 helpers (sm_100 FFMA2).  Each lane is an IEEE fma.rn.f32,
// so a paired update is bit-identical to two FFMAs.
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2lo(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  (void)hi;
  return lo;
}
__device__ __forceinline__ float f2hi(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  (void)lo;
  return hi;
}
// (c.lo + x * w.lo, c.hi + x * w.hi): x is broadcast (SASS: FFMA2 R.F32,
// UR.F32x2, R.F32x2), the weight pair sits in a uniform register pair.
__device__ __forceinline__ uint64_t ffma2_bx(float x, uint64_t w, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2pack(x, x)), "l"(w), "l"(c));
  return r;
}

// Rolling accumulators of one thread: slot m holds the partial sums of the
// output plane the current input plane reaches with dz = K-1-m.  Slots
// (2p, 2p+1) live as packed pairs so one FFMA2 advances two output planes
// (same input value, the weights of their two dz); slot K-1 is single.
template <int K>
struct Accum {
  static constexpr int YPT = Layout<K>::YPT;
  static constexpr int NP = K / 2;
  uint64_t p[YPT][NP][XPT];
  float s[YPT][XPT];
};

// One input plane's contribution to the K rolling accumulators of the
// thread's YPT x 8 outputs.  GUARD: skip slot groups whose output planes are
// all outside the chunk (ramp up / down; those sums are never stored).
// PF: load the rows of dy+1 while dy computes (measured: +3% for f32 K>=5;
// for the integer kernels the extra 16 registers push the weights off the
// uniform datapath, -10%).
template <int K, bool GUARD, bool PF>
__device__ __forceinline__ void plane_step(const float* __restrict__ stage, int tx, int ty,
                                           const Weights<K>& wt, Accum<K>& acc, int first,
                                           int last) {
  constexpr int YPT = Layout<K>::YPT;
  constexpr int R = K / 2;
  constexpr int NP = K / 2;
  constexpr int OFF = 4 - R;
  float4 nx[YPT][4];
  const float* base = stage + YPT * ty * RP + XPT * tx;
  if (PF) {
#pragma unroll
    for (int r = 0; r < YPT; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i) nx[r][i] = reinterpret_cast<const float4*>(base + r * RP)[i];
  }
#pragma unroll(K <= 3 ? K : 1)
  for (int dy = 0; dy < K; ++dy) {
    if (!PF) {
#pragma unroll
      for (int r = 0; r < YPT; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i) nx[r][i] = reinterpret_cast<const float4*>(base + (r + dy) * RP)[i];
    }
    float v[YPT][16];
#pragma unroll
    for (int r = 0; r < YPT; ++r) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[r][4 * i + 0] = nx[r][i].x;
        v[r][4 * i + 1] = nx[r][i].y;
        v[r][4 * i + 2] = nx[r][i].z;
        v[r][4 * i + 3] = nx[r][i].w;
      }
    }
    if (PF && dy + 1 < K) {
#pragma unroll
      for (int r = 0; r < YPT; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i) nx[r][i] = reinterpret_cast<const float4*>(base + (r + dy + 1) * RP)[i];
    }
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      if (GUARD && (2 * pp + 1 < first || 2 * pp > last)) continue;
      const uint64_t* w = reinterpret_cast<const uint64_t*>(wt.wp + (dy * NP + pp) * K);
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
        const uint64_t wv = w[dx];
#pragma unroll
        for (int r = 0; r < YPT; ++r)
#pragma unroll
          for (int j = 0; j < XPT; ++j) acc.p[r][pp][j] = ffma2_bx(v[r][OFF + j + dx], wv, acc.p[r][pp][j]);
      }
    }
    if (!GUARD || (K - 1 >= first && K - 1 <= last)) {
      const float* w = wt.ws + dy * Weights<K>::KP;
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
        const float wv = w[dx];
#pragma unroll
        for (int r = 0; r < YPT; ++r)
#pragma unroll
          for (int j = 0; j < XPT; ++j) acc.s[r][j] = __fmaf_rn(wv, v[r][OFF + j + dx], acc.s[r][j]);
      }
    }
  }
}

template <typename T, int K, int MODE>
__global__ void __launch_bounds__(Layout<K>::THREADS, Layout<K, MODE>::CTAS_PER_SM)
    filter_tma_kernel(const __grid_constant__ CUtensorMap map_src,
                      const __grid_constant__ CUtensorMap map_lo,
                      const __grid_constant__ CUtensorMap map_hi, const TmaParams p,
                      const __grid_constant__ Weights<K> wt) {
  if (p.guard != nullptr && *p.guard != 0) return;  // uniform over the grid
  using C = Cfg<T, K, MODE>;
  constexpr int R = C::R;
  constexpr int S = C::S_RDY;
  constexpr int YPT = Layout<K>::YPT;
  constexpr int WARPS = Layout<K>::WARPS;
  constexpr int THREADS = Layout<K>::THREADS;
  constexpr int WROWS = Layout<K>::WROWS;
  constexpr int SR = C::IS_F32 ? C::S_RDY : C::S_RAW;  // TMA ring depth
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // TMA destinations must be 128-byte aligned; do not rely on the base.
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float* rdy_base = reinterpret_cast<float*>(smem);
  T* raw_base = reinterpret_cast<T*>(smem + C::S_RDY * C::RDY_PITCH);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_DATA);
  uint64_t* full = bars;            // [SR] TMA landed (f32: in the ready ring)
  uint64_t* ready = full + SR;      // [S]  staged plane complete (8 warp arrivals)
  uint64_t* empty = ready + S;      // [S]  all warps done computing from the stage
  uint64_t* raw_free = empty + S;   // [SR] ints: all warps done converting the raw stage

  const int tid = threadIdx.x;
  const int warp = tid / 32;
  const int lane = tid % 32;
  const int x0 = blockIdx.x * TX;
  const int y0 = blockIdx.y * TY;
  const int zo0 = p.z_begin + blockIdx.z * p.zc;
  const int nzo = min(p.zc, p.z_end - zo0);
  if (nzo <= 0) return;
  const int np = nzo + 2 * R;  // input planes of this chunk
  const bool edge = (x0 - R < 0) || (x0 + TX + R > p.nx) || (y0 - R < 0) || (y0 + TY + R > p.ny);

  if (tid == 0) {
    prefetch_tmap(&map_src);
    for (int s = 0; s < SR; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&raw_free[s], WARPS);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&ready[s], WARPS);
      mbar_init(&empty[s], WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // TMA plane j into ring slot j % SR (zero planes: plain arrive).  Called
  // by all threads; only thread 0 acts (predicated, no divergent branch).
  const bool leader = tid == 0;
  auto issue = [&](int j) {
    const int r = j % SR;
    void* dst = C::IS_F32 ? static_cast<void*>(rdy_base + r * (C::RDY_PITCH / 4))
                          : static_cast<void*>(raw_base + r * (C::RAW_PITCH / (int)sizeof(T)));
    const PlaneSrc s = resolve<MODE>(p, R, zo0 - R + j);
    if (s.which < 0) {
      mbar_arrive_if(&full[r], leader);
      return;
    }
    const CUtensorMap* m = s.which == 0 ? &map_src : s.which == 1 ? &map_lo : &map_hi;
    tma_issue_if(dst, m, &full[r], C::IS_F32 ? C::RDY_BYTES : C::RAW_BYTES, x0 - C::A, y0 - R,
                 s.z, leader);
  };

  // ints: widen plane j (all warps, equal shares) into ready stage j % S.
  const QuadPlan<T, K, THREADS> qplan(p, x0, y0, edge, tid);
  auto prepare = [&](int j) {
    VKT_JITTER_POINT(4 * j);
    const int s = j % S;
    float* stage = rdy_base + s * (C::RDY_PITCH / 4);
    const int r = j % SR;
    mbar_wait(&full[r], (uint32_t)((j / SR) & 1));
    if (j >= S) mbar_wait(&empty[s], (uint32_t)(((j / S) - 1) & 1));
    const PlaneSrc src = resolve<MODE>(p, R, zo0 - R + j);
    if (src.which < 0) {
      float4* w4 = reinterpret_cast<float4*>(stage);
      for (int q = tid; q < C::RDY_BYTES / 16; q += THREADS) w4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const T* raw = raw_base + r * (C::RAW_PITCH / (int)sizeof(T));
      convert_plane<T, MODE, K, THREADS>(stage, raw, plane_ptr<T>(p, src), p, x0, y0, qplan);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&ready[s]);
      mbar_arrive(&raw_free[r]);
    }
  };

  for (int j = 0; j < SR && j < np; ++j) issue(j);
  if constexpr (!C::IS_F32) {
    for (int j = 0; j < C::AHEAD && j < np; ++j) prepare(j);
  }

  const int tx = tid % (TX / XPT);
  const int ty = tid / (TX / XPT);
  const float a0 = acc_init<T>(p.c);
  constexpr int NP = K / 2;
  const uint64_t a00 = f2pack(a0, a0);
  Accum<K> acc;
#pragma unroll
  for (int r = 0; r < YPT; ++r)
#pragma unroll
    for (int j = 0; j < XPT; ++j) {
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) acc.p[r][pp][j] = a00;
      acc.s[r][j] = a0;
    }

  const int ox = x0 + tx * XPT;
  const int oy = y0 + YPT * ty;
  int valid[YPT];
#pragma unroll
  // cells beyond nx up to the pitch are padding: storing there is harmless
  for (int r = 0; r < YPT; ++r) valid[r] = (oy + r < p.ny) ? min(XPT, p.pitch - ox) : 0;
  T* out_base = static_cast<T*>(p.dst) + (int64_t)oy * p.pitch + ox;
  const int64_t plane_elems = (int64_t)p.pitch * p.ny;

  const FixList<MODE, R> fix = (C::IS_F32 && (MODE == VKT_CLAMP || MODE == VKT_MIRROR) && edge)
                                   ? FixList<MODE, R>(p, x0, y0, lane, WROWS * warp,
                                                      WROWS * warp + WROWS + 2 * R)
                                   : FixList<MODE, R>();
  WrapList<R> wrap = (C::IS_F32 && MODE == VKT_WRAP && edge)
                         ? WrapList<R>(p, x0, y0, lane, WROWS * warp, WROWS * warp + WROWS + 2 * R)
                         : WrapList<R>();
  if (C::IS_F32 && MODE == VKT_WRAP && edge && wrap.ok)
    wrap.gather(plane_ptr<float>(p, resolve<MODE>(p, R, zo0 - R)));
  for (int i = 0; i < np; ++i) {
    VKT_JITTER_POINT(4 * i + 1);
    const int s = i % S;
    float* stage = rdy_base + s * (C::RDY_PITCH / 4);
    if constexpr (C::IS_F32) {
      // refill the TMA slot of plane i-LAG (released by every warp by now)
      constexpr int LAG = C::LAG;
      if (i >= LAG && i + SR - LAG < np) {
        mbar_wait(&empty[(i - LAG) % S], (uint32_t)(((i - LAG) / S) & 1));
        issue(i + SR - LAG);
      }
      mbar_wait(&full[s], (uint32_t)((i / S) & 1));
      if constexpr (MODE == VKT_BORDER) {
        // Border z planes outside the volume: this warp clears the rows it
        // reads (TMA's zero fill covers x / y)
        if (resolve<MODE>(p, R, zo0 - R + i).which < 0) {
          for (int q = lane; q < (WROWS + 2 * R) * (RP / 4); q += 32)
            reinterpret_cast<float4*>(stage + (WROWS * warp) * RP)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          fence_proxy_async();
          __syncwarp();
        }
      } else if (edge) {
        // Clamp / Mirror / Wrap never yield a zero plane; only edge tiles
        // repair the out-of-volume cells of this warp's read window.  (The
        // per-plane plane resolve and repair branch in every CTA cost ~50
        // instructions per warp-plane, measured.)
        if constexpr (MODE == VKT_WRAP) {
          if (wrap.ok) {
            wrap.apply(stage);
            if (i + 1 < np) wrap.gather(plane_ptr<float>(p, resolve<MODE>(p, R, zo0 - R + i + 1)));
          } else {
            fixup_f32_cold<MODE, R>(stage, plane_ptr<float>(p, resolve<MODE>(p, R, zo0 - R + i)), p,
                                    x0, y0, lane, 32, WROWS * warp, WROWS * warp + WROWS + 2 * R);
          }
        } else if (fix.ok) {
          fix.apply(stage);
        } else {
          fixup_f32_cold<MODE, R>(stage, plane_ptr<float>(p, resolve<MODE>(p, R, zo0 - R + i)), p,
                                  x0, y0, lane, 32, WROWS * warp, WROWS * warp + WROWS + 2 * R);
        }
        fence_proxy_async();
        __syncwarp();
      }
    } else {
      // refill the raw slot of plane i-1 (converted two iterations ago)
      if (i >= 1 && i - 1 + SR < np) {
        mbar_wait(&raw_free[(i - 1) % SR], (uint32_t)(((i - 1) / SR) & 1));
        issue(i - 1 + SR);
      }
      if (i + C::AHEAD < np) prepare(i + C::AHEAD);
      mbar_wait(&ready[s], (uint32_t)((i / S) & 1));
    }
    // slot m <-> output plane zo0 + i - 2R + m
    const int first = 2 * R - i;
    const int last = nzo - 1 - i + 2 * R;
    if (first <= 0 && last >= K - 1)
      plane_step<K, false, C::IS_F32 && K >= 5>(stage, tx, ty, wt, acc, 0, K - 1);
    else
      plane_step<K, true, C::IS_F32 && K >= 5>(stage, tx, ty, wt, acc, first, last);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (i >= 2 * R) {
      const int oz = zo0 + i - 2 * R;
#pragma unroll
      for (int r = 0; r < YPT; ++r) {
        float o[XPT];
#pragma unroll
        for (int j = 0; j < XPT; ++j) o[j] = f2lo(acc.p[r][0][j]);
        if (valid[r] > 0) store8<T>(out_base + (int64_t)oz * plane_elems + (int64_t)r * p.pitch, o, valid[r]);
      }
    }
    // roll: slot m <- slot m+1, slot K-1 <- fresh
#pragma unroll
    for (int r = 0; r < YPT; ++r)
#pragma unroll
      for (int j = 0; j < XPT; ++j) {
#pragma unroll
        for (int pp = 0; pp + 1 < NP; ++pp)
          acc.p[r][pp][j] = f2pack(f2hi(acc.p[r][pp][j]), f2lo(acc.p[r][pp + 1][j]));
        acc.p[r][NP - 1][j] = f2pack(f2hi(acc.p[r][NP - 1][j]), acc.s[r][j]);
        acc.s[r][j] = a0;
      }
  }
}

template <typename T, int K, int MODE>
cudaError_t launch_tma_kernel(const CUtensorMap& ms, const CUtensorMap& ml, const CUtensorMap& mh,
                              const TmaParams& p, const float* w32, dim3 grid, cudaStream_t s) {
  using C = Cfg<T, K, MODE>;
  // w32: (dz, dy, dx), x fastest
  Weights<K> wt = {};
  constexpr int NP = Weights<K>::NP;
  for (int dy = 0; dy < K; ++dy) {
    for (int pp = 0; pp < NP; ++pp)
      for (int dx = 0; dx < K; ++dx)
        wt.wp[(dy * NP + pp) * K + dx] = make_float2(w32[((K - 1 - 2 * pp) * K + dy) * K + dx],
                                                     w32[((K - 2 - 2 * pp) * K + dy) * K + dx]);
    for (int dx = 0; dx < K; ++dx) wt.ws[dy * Weights<K>::KP + dx] = w32[dy * K + dx];
  }
  auto fn = filter_tma_kernel<T, K, MODE>;
  // the shared-memory opt-in once per device (a per-call attribute set was a
  // measurable share of the host time of small launches)
  static std::atomic<uint64_t> opted{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(opted.load(std::memory_order_acquire) & bit)) {
    err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (err != cudaSuccess) return err;
    opted.fetch_or(bit, std::memory_order_release);
  }
  fn<<<grid, Layout<K>::THREADS, C::SMEM, s>>>(ms, ml, mh, p, wt);
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
#undef VKT_TMA_K
#undef VKT_TMA_CASE
  return cudaErrorInvalidValue;
}

}  // namespace tma_zp
}  // namespace vkt
