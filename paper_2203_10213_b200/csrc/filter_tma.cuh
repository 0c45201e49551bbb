// filter_tma.cuh — tiled sm_100a ApplyFilter kernel (TMA staging, packed FFMA2).
//
// Design:
//  * A CTA owns a TX=128 (x) by TY=16 (y) column of outputs and a chunk of ZC
//    output planes, and streams the chunk's input planes through shared
//    memory.  Each input plane is ONE TMA 3D box load
//    (cp.async.bulk.tensor.3d, completion on an mbarrier with complete_tx) of
//    the plane's footprint plus its halo into a "raw" ring.
//  * Every warp computes, and each also stages 1/WARPS of a plane AHEAD planes
//    in advance: it widens the raw cells to float (u8/u16; f32 is a copy),
//    repairs the out-of-volume halo cells of edge tiles for Clamp / Mirror /
//    Wrap (Border is TMA's zero fill = stored 0), and writes them into a
//    "ready" ring in the PAIRED layout below.  Lane 0 of warp 0 issues the TMA
//    loads.  Warps meet only on mbarriers (full / raw_free / ready / empty
//    rings); there is no CTA-wide barrier per plane.
//  * Paired layout: ready-stage pair i of a row holds the cells at x0-4+i and
//    x0-4+i+64, so one packed FFMA2 (fma.rn.f32x2: two IEEE fma.rn.f32 lanes)
//    advances two outputs 64 cells apart with one broadcast weight, and a
//    LDS.128 delivers two ready register pairs.  Every tap is an FFMA2 — a mix
//    of FFMA and FFMA2 packs the FMA pipe to ~85%, pure FFMA2 to ~99%
//    (measured, tools/ffma2_probe.cu).
//  * Each thread owns 4 output pairs (8 outputs) of YPT rows and keeps K = 2R+1
//    rolling accumulators per output — one per output plane the current
//    input plane contributes to.  Per input plane the dy loop stays rolled
//    for K >= 5 (instruction cache); each dy iteration loads the row pairs
//    (LDS.128) and issues 4*K*K*YPT FFMA2 whose weight is a uniform register
//    (LDCU from the by-value kernel-parameter block).
//  * Tap order per output is (dz, dy, dx) — the reference's order
//    (filters.py:89-92) and the direct kernel's — so every kernel path and
//    every z-slab split produce bit-identical results.
//  * Epilogue: quantize as volume.py:102-110 (ints) and store with streaming
//    (evict-first) stores.
#pragma once

#include <cuda.h>

#include <atomic>

#include <cstdio>

#include "common.cuh"

namespace vkt {
namespace tma {

constexpr int TX = 128;          // outputs per CTA in x
constexpr int TY = 16;           // outputs per CTA in y
constexpr int HALF = TX / 2;     // x distance between the two outputs of a pair
constexpr int XQ = 4;            // output pairs per thread row (8 outputs)
constexpr int TPR = HALF / XQ;   // threads per output row
constexpr int NPR = HALF + 8;    // pairs per ready row: lo x in [x0-4, x0+HALF+4)
// Ready-stage bank layout.  A thread reads a run of 16-byte chunks starting
// at chunk 2*tx of its row (and staging writes one item of 2 chunks per
// thread), so with a plain layout the 8 lanes of a 128-bit quarter-warp phase
// (tx..tx+7 of one row) hit 4 bank groups twice: 2-way conflicts on every
// LDS.128 / STS.128 (ncu: 2.5x the ideal shared wavefronts at K = 3).  Two
// cures, per kernel extent:
//  * K = 3 (2 rows per thread): XOR swizzle within a row — chunk c of an odd
//    128-byte line of the row is stored at c ^ 1 (in-row float offset o ->
//    o ^ ((o >> 3) & 4)); lanes t and t+4 of a phase then fall in lines of
//    opposite parity.  A row base that is not line-aligned shifts all lanes of
//    a phase alike, so rows stay 144 floats (padding them to 160 cost a ready
//    stage of the ring).  Each load needs its own address register,
//    affordable at K = 3.
//  * K >= 5 (1 row per thread): rows 148 floats = 37 chunks apart (odd) and a
//    quarter-warp holds tx 0..3 of TWO adjacent rows (lane_layout below), so
//    the two halves of a phase fall on opposite chunk parities.  Loads keep a
//    single base register with immediate offsets (at K = 7 per-load address
//    registers cost ptxas ~2x the register moves on the FFMA2 loop, measured).
__device__ __forceinline__ int swz(int o) { return o ^ ((o >> 3) & 4); }

template <int K>
struct Ready {
  static constexpr bool SWZ = K == 3;
  static constexpr int RPF = SWZ ? 2 * NPR : 2 * NPR + 4;  // row pitch (floats)
  // physical offset of in-row float offset o (a multiple of 4)
  __host__ __device__ static constexpr int in_row(int o) { return SWZ ? (o ^ ((o >> 3) & 4)) : o; }
  // the item's second chunk, given the physical offset of its first
  __device__ __forceinline__ static int second(int so) { return SWZ ? (so ^ 4) : so + 4; }
};
static_assert((2 * NPR + 4) / 4 % 2 == 1, "K >= 5 ready rows must be an odd number of chunks");

// Thread layout (measured): 1 output row per thread, 8 warps
// (staging split between the halves), 2 CTAs/SM (4 warps/SMSP, 128 regs).
// Warps per SM stay a multiple of 4 so every SM sub-partition gets the same
// number of FMA warps.  (u8/u16 K = 3 run filter_ws.cuh, f32 K = 3
// filter_tma_zp.cuh.)
template <int BPC, int K>
struct Layout {
  static constexpr int YPT = 1;
  static constexpr int WARPS = TY * TPR / (32 * YPT);
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int CTAS_PER_SM = 2;
  static constexpr int SMEM_PER_CTA = (228 * 1024) / CTAS_PER_SM - 1024;  // minus driver reserve
};

// Raw TMA box geometry (shared by the host tensor-map encode and the kernel).
// TMA needs the innermost box coordinate at a 16-byte multiple (measured with
// tools/tma_probe.cu), so the box starts A >= R cells left of the tile; it
// spans at least [x0-4, x0+TX+4), the cells the paired ready rows hold
// (R > 4, separable kernels only: [x0-4h, x0+TX+4h), h = ceil(R/4) quads).
__host__ __device__ constexpr int box_align_left(int r, int bpc) {
  return ((r > 4 ? r : 4) + 16 / bpc - 1) / (16 / bpc) * (16 / bpc);
}
__host__ __device__ constexpr int box_width(int r, int bpc) {
  return (box_align_left(r, bpc) + TX + 4 * ((r > 4 ? r + 3 : 4) / 4) + 16 / bpc - 1) / (16 / bpc) * (16 / bpc);
}

template <typename T, int K>
struct Cfg {
  using L = Layout<(int)sizeof(T), K>;
  static constexpr int R = K / 2;
  static constexpr int A = box_align_left(R, (int)sizeof(T));
  static constexpr int BX = box_width(R, (int)sizeof(T));
  static constexpr int BY = TY + 2 * R;
  static constexpr int RAW_BYTES = BX * BY * (int)sizeof(T);
  static constexpr int RAW_PITCH = (RAW_BYTES + 127) / 128 * 128;
  static constexpr int RPF = Ready<K>::RPF;
  static constexpr int RDY_BYTES = RPF * BY * 4;
  static constexpr int RDY_PITCH = (RDY_BYTES + 127) / 128 * 128;
  // Ring depths within CTAS_PER_SM CTAs per SM: 4..6 ready stages (AHEAD = 2
  // planes staged ahead of compute leave S_RDY - 3 planes of slack between
  // the fastest and the slowest warp) once 6 raw TMA stages fit (TMA
  // lookahead S_RAW - 1 - AHEAD planes: f32 K <= 5 planes take ~2 us, so one
  // plane of lookahead is not enough), the rest as raw stages, capped at 10.
  // Edge-repair table (Clamp / Mirror): per staging item with an
  // out-of-volume cell in the read window its ready offset and the 8 raw
  // source cells, built once per CTA.  The window [x0-R, min(x0+TX,nx)+R) x
  // [y0-R, min(y0+TY,ny)+R) has at most R such rows on each side and at most
  // 4 such items in any other row (R <= 4 cells on each side; a cell column
  // in [64, 72) sits in a low and a high quad), whatever the extents.
  static constexpr int MAX_REPAIR = 2 * R * (NPR / 4) + 4 * BY;
  static constexpr int REPAIR_BYTES = (MAX_REPAIR * 18 + 16 + 127) / 128 * 128;
  static constexpr int BUDGET = L::SMEM_PER_CTA - 512 - REPAIR_BYTES;
  static constexpr int RAW_MIN = 6;
  static constexpr int S_RDY_FIT = (BUDGET - RAW_MIN * RAW_PITCH) / RDY_PITCH;
  static constexpr int S_RDY_MIN = K == 9 ? 3 : 4;  // K = 9: 24-row stages
  static constexpr int S_RDY = S_RDY_FIT < S_RDY_MIN ? S_RDY_MIN : (S_RDY_FIT > 6 ? 6 : S_RDY_FIT);
  static constexpr int S_RAW_FIT = (BUDGET - S_RDY * RDY_PITCH) / RAW_PITCH;
  static constexpr int S_RAW = S_RAW_FIT < 10 ? S_RAW_FIT : 10;
  static constexpr int AHEAD = S_RDY >= 4 ? 2 : 1;
  static constexpr int SMEM_DATA = S_RDY * RDY_PITCH + S_RAW * RAW_PITCH;
  static constexpr int NBAR = 2 * S_RDY + 2 * S_RAW;
  static constexpr int SMEM = SMEM_DATA + REPAIR_BYTES + NBAR * 8 + 128;
  static_assert(R >= 1 && R <= 4, "radius");
  static_assert(S_RAW >= AHEAD + 2, "TMA ring too shallow");
  static_assert(SMEM <= L::SMEM_PER_CTA, "shared memory budget");
  static_assert(BX <= 256 && BY <= 256, "TMA box too large");
};

// Weights as a kernel-parameter block, each (dz, dy) row of K taps padded to a
// 16-byte boundary so a row is fetched with 128-bit uniform constant loads.
template <int K>
struct alignas(16) Weights {
  static constexpr int KP = (K + 3) / 4 * 4;
  float w[K * K * KP];
};

struct TmaParams {
  void* dst;
  const void* src;       // local slab (for Wrap gathers)
  const void* halo_lo;
  const void* halo_hi;
  int nx, ny, nz;        // local extents
  int pitch;             // row pitch in cells (>= nx, rows 16-byte multiples)
  int z_begin, z_end;    // local output planes [begin, end)
  int zc;                // output planes per CTA chunk
  int64_t z_offset, global_nz;
  float c;               // integer epilogue constant
  uint32_t zskip;        // anisotropic kernels in a K^3 cube: bit dz set = padding plane,
  uint32_t yskip;        //   bit dy set = padding row (the x extent is a template)
  const int* guard;      // non-null: the launch does nothing when *guard != 0 (vkt_capi.cu)
  int* nonfinite;        // separable f32 kernel: set to 1 when a stored output is Inf/NaN
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
// Predicated single-thread forms: executed by every thread of the CTA with
// the predicate true in exactly one, so the surrounding loop stays free of
// thread-divergent branches (ptxas then keeps the rolled dy loop's weight
// loads on the uniform datapath: LDCU + FFMA2 with a uniform-register operand).
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

// Packed fp32x2 helpers (sm_100 FFMA2 / FADD2).  Each lane is an IEEE .rn
// f32 operation, so a paired update is bit-identical to two scalar ones.
// (asm forms: ptxas keeps such pairs in register pairs without moves in the
// FFMA2 loop.  The staging code's edge repair uses the plain-C forms below:
// with the asm forms, replacing one half of a widened pair came out wrong
// (tests/test_gpu_parity.py::test_tiled_shapes_vs_oracle).)
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
__device__ __forceinline__ uint64_t pair_c(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo_c(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi_c(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
// (c.lo + x.lo * w, c.hi + x.hi * w): the weight is broadcast (SASS: FFMA2
// R.F32x2, UR.F32, R.F32x2 — one uniform register, no extra load).
__device__ __forceinline__ void ffma2_bw(uint64_t x, float w, uint64_t& c) {
  // in place ("+l"): the accumulator keeps its register pair across the
  // rolled dy loop instead of being renamed with moves at the back edge
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(x), "l"(f2pack(w, w)));
}
// x * w + c0 into another accumulator (an untied destination: starts a slot
// from the next slot's partial sum or the epilogue constant without a copy).
__device__ __forceinline__ uint64_t ffma2_from(uint64_t x, float w, uint64_t c0) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(f2pack(w, w)), "l"(c0));
  return d;
}
// Two u8/u16 values, given as the bit patterns 0x4B000000 | v (the value in
// the low mantissa bits of 2^23), -> (float, float) exactly: minus 2^23, one
// FADD2.
__device__ __forceinline__ uint64_t widen2(uint32_t blo, uint32_t bhi) {
  uint64_t bits, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(bits) : "r"(blo), "r"(bhi));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(bits), "l"(f2pack(-8388608.0f, -8388608.0f)));
  return r;
}

// Tiles on the volume's x / y faces repair their out-of-volume cells every
// plane (Wrap gathers them from the far side) and run longer.  Blocks are
// dispatched in linear-id order, so the linear id is remapped to run all face
// tiles first and the uniform interior tiles last: the final, partial wave
// then holds no slow tile.  Only the last z chunk is reordered under Clamp /
// Mirror: reordering every chunk separated tiles that share halo rows and
// cost 0.65 GB of DRAM re-reads per 1024^3 u16 launch (L2 hit 47% -> 30%).  Used by the compute-bound kernels
// (filter_sep.cuh: u16 7^3 Wrap 2.03 -> 1.80 ms with deep chunks;
// filter_ws.cuh: u8 3^3 Wrap 1.363 -> 1.307); the HBM-bound f32 3^3 kernel
// and the paired kernel keep the natural order (neighbouring tiles share
// halo rows in L2: f32 3^3 Clamp 1.48 -> 1.57 ms when reordered).
template <int MODE>
__device__ __forceinline__ void edge_first(int& tx, int& ty, int& tz) {
  const int gx = gridDim.x, gy = gridDim.y;
  if (gx < 3 || gy < 3) return;  // every tile is a face tile
  const int E = 2 * gx + 2 * (gy - 2);
  const int I = (gx - 2) * (gy - 2);
  // Clamp / Mirror: the last z chunk's face tiles, then its interior tiles
  // (face tiles are only a little slower).  Wrap (its face tiles gather the
  // far side): the face tiles of every chunk first.
  int L = blockIdx.x + gx * blockIdx.y;
  tz = blockIdx.z;
  if constexpr (MODE != VKT_WRAP) {
    // only the last chunk's tail matters: earlier chunks keep the natural
    // order (neighbouring tiles in step, sharing halo rows in L2)
    if (blockIdx.z + 1 != gridDim.z) return;
  } else {
    const int G = L + gx * gy * (int)blockIdx.z;
    const int nedge = E * (int)gridDim.z;
    if (G < nedge) {
      tz = G / E;
      L = G - tz * E;
    } else {
      tz = (G - nedge) / I;
      L = E + (G - nedge) - tz * I;
    }
  }
  if (L < E) {
    if (L < 2 * gx) {
      tx = L < gx ? L : L - gx;
      ty = L < gx ? 0 : gy - 1;
    } else {
      const int e2 = L - 2 * gx;
      ty = 1 + (e2 >> 1);
      tx = (e2 & 1) ? gx - 1 : 0;
    }
  } else {
    const int r = L - E;
    ty = 1 + r / (gx - 2);
    tx = 1 + r - (ty - 1) * (gx - 2);
  }
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

// ---------------------------------------------------------------------------
// Staging: raw TMA plane -> paired float ready stage
// ---------------------------------------------------------------------------
// This thread's share of the staging work, fixed for the whole CTA (the tile
// geometry is the same for every plane): item q = t + k*nt covers ready pairs
// [4g, 4g+4) of stage row `by`, i.e. the cells x0-4+4g .. +3 (lo halves) and
// the same +HALF (hi halves).  `slow` marks items that hold out-of-volume
// cells of the read window.
// Does staging item (row by, pairs 4g..4g+3: cells [4g, 4g+4) and
// [4g+HALF, 4g+HALF+4)) hold an out-of-volume cell of the read window?
template <int R>
__device__ __forceinline__ bool slow_item(int by, int g, int rows_lo, int rows_hi, int rows_end,
                                          int e_lo, int e_hi, int e_end) {
  if (by < rows_lo || (by >= rows_hi && by < rows_end)) return true;
  auto hit = [&](int a) {  // [a, a+4) meets [4-R, e_lo) or [e_hi, e_end)
    return (a < e_lo && a + 4 > 4 - R) || (a < e_end && a + 4 > e_hi);
  };
  return hit(4 * g) || hit(4 * g + HALF);
}

template <typename T, int K, int NT, bool MODE_REPAIRS>
struct StagePlan {
  using C = Cfg<T, K>;
  static constexpr int GPR = NPR / 4;  // items per row
  static constexpr int NQ = GPR * C::BY;
  static constexpr int QPT = (NQ + NT - 1) / NT;
  // offsets computed once per CTA (K = 7 recomputes them: 128-register budget)
  static constexpr bool STORE = K <= 5;
  int rdy_[STORE ? QPT : 1];  // ready-stage float offset (-1: no item, or an
                              // item the repair pass writes)
  int raw_[STORE ? QPT : 1];  // raw-stage cell offset of the item's low quad
  int t_, rows_lo_, rows_hi_, rows_end_, e_lo_, e_hi_, e_end_;

  bool edge_;
  __device__ __forceinline__ StagePlan(const TmaParams& p, int x0, int y0, bool edge, int t) {
    constexpr int R = C::R;
    t_ = t;
    edge_ = edge;
    // out-of-volume stage rows / cell columns inside the read window of the
    // tile's valid outputs (cells past it are read by padding outputs only)
    rows_lo_ = R - y0;                              // rows [0, rows_lo_)
    rows_hi_ = p.ny - y0 + R;                       // rows [rows_hi_, rows_end_)
    rows_end_ = min(TY, p.ny - y0) + 2 * R;
    e_lo_ = 4 - x0;                                 // cells [4-R, e_lo_)
    e_hi_ = p.nx - x0 + 4;                          // cells [e_hi_, e_end_)
    e_end_ = min(TX, p.nx - x0) + 4 + R;
    if constexpr (STORE) {
#pragma unroll
      for (int k = 0; k < QPT; ++k) compute(k, rdy_[k], raw_[k]);
    }
  }
  __device__ __forceinline__ bool slow(int by, int g) const {
    return edge_ && slow_item<C::R>(by, g, rows_lo_, rows_hi_, rows_end_, e_lo_, e_hi_, e_end_);
  }
  // item k of the row-major staging pass (edge items are left to the repair
  // pass, MODE != Border): ro = the swizzled ready offset of its first chunk
  // (the second is at ro ^ 4), or -1
  __device__ __forceinline__ void compute(int k, int& ro, int& wo) const {
    const int q = t_ + k * NT;
    const int by = q / GPR, g = q - by * GPR;
    ro = q < NQ && !(MODE_REPAIRS && slow(by, g)) ? by * C::RPF + Ready<K>::in_row(8 * g) : -1;
    wo = by * C::BX + 4 * g + (C::A - 4);
  }
  __device__ __forceinline__ void get(int k, int& ro, int& wo) const {
    if constexpr (STORE) {
      ro = rdy_[k];
      wo = raw_[k];
    } else {
      compute(k, ro, wo);
    }
  }
};

// 4 consecutive raw cells -> 4 words: u8/u16 as the exponent-trick bit
// patterns 0x4B000000 | v (one PRMT each; widen2 finishes them), f32 as
// the values' bits.
template <typename T>
__device__ __forceinline__ void load_quad(const T* src, uint32_t (&b)[4]) {
  if constexpr (sizeof(T) == 2) {
    const uint2 w = *reinterpret_cast<const uint2*>(src);
    b[0] = __byte_perm(w.x, 0x4B000000u, 0x7410);
    b[1] = __byte_perm(w.x, 0x4B000000u, 0x7432);
    b[2] = __byte_perm(w.y, 0x4B000000u, 0x7410);
    b[3] = __byte_perm(w.y, 0x4B000000u, 0x7432);
  } else if constexpr (sizeof(T) == 1) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(src);
    b[0] = __byte_perm(w, 0x4B000000u, 0x7440);
    b[1] = __byte_perm(w, 0x4B000000u, 0x7441);
    b[2] = __byte_perm(w, 0x4B000000u, 0x7442);
    b[3] = __byte_perm(w, 0x4B000000u, 0x7443);
  } else {
    const uint4 w = *reinterpret_cast<const uint4*>(src);
    b[0] = w.x;
    b[1] = w.y;
    b[2] = w.z;
    b[3] = w.w;
  }
}

// The repair table: count, then per entry the 8 raw source cells (lo quad,
// hi quad) as u16 and the swizzled ready-stage float offset / 4.
struct RepairTable {
  uint32_t* count;
  uint4* src;      // [MAX_REPAIR] 8 x u16 raw cell offsets
  uint16_t* dst;   // [MAX_REPAIR] swizzled ready offset / 4
};

// Clamp / Mirror: every out-of-volume cell of the read window maps onto an
// in-volume cell of the same raw stage (R <= 4 < TX, TY), a correspondence
// fixed for the CTA.  Built by all threads once; edge CTAs only.
template <typename T, int MODE, int K, int NT>
__device__ __forceinline__ void build_repair_table(const RepairTable& rt, const TmaParams& p,
                                                   int x0, int y0, int t) {
  using C = Cfg<T, K>;
  constexpr int R = C::R;
  constexpr int GPR = NPR / 4;
  constexpr int NQ = GPR * C::BY;
  const int rows_lo = R - y0, rows_hi = p.ny - y0 + R, rows_end = min(TY, p.ny - y0) + 2 * R;
  const int e_lo = 4 - x0, e_hi = p.nx - x0 + 4, e_end = min(TX, p.nx - x0) + 4 + R;
  const bool near = p.nx >= 4 && p.ny >= 4;
  for (int q = t; q < NQ; q += NT) {
    const int g = q / C::BY, by = q - g * C::BY;  // column-major
    if (!slow_item<R>(by, g, rows_lo, rows_hi, rows_end, e_lo, e_hi, e_end)) continue;
    const int gy = y0 - R + by;
    const bool yo = gy < 0 || gy >= p.ny;
    // rows past the read window of the valid outputs are left alone (their
    // fold would leave the staged box)
    const bool yin = gy < min(y0 + TY, p.ny) + R;
    const int my = near ? map_index_near<MODE>(gy, p.ny) : map_index32<MODE>(gy, p.ny);
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      uint32_t pair = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = 2 * h + u;
        const int gx = x0 - 4 + 4 * g + (c & 3) + (c >> 2) * HALF;
        int src = by * C::BX + (gx - x0 + C::A);  // own cell
        if (yin && (yo || gx < 0 || gx >= p.nx) && gx >= x0 - R && gx < min(x0 + TX, p.nx) + R) {
          const int mx = near ? map_index_near<MODE>(gx, p.nx) : map_index32<MODE>(gx, p.nx);
          src = (my - y0 + R) * C::BX + (mx - x0 + C::A);
        }
        pair |= (uint32_t)src << (16 * u);
      }
      w[h] = pair;
    }
    const uint32_t idx = atomicAdd(rt.count, 1u);
    rt.src[idx] = make_uint4(w[0], w[1], w[2], w[3]);
    rt.dst[idx] = (uint16_t)((by * C::RPF + Ready<K>::in_row(8 * g)) / 4);
  }
}

template <typename T>
__device__ __forceinline__ float raw_value(const T* raw, uint32_t i) {
  if constexpr (sizeof(T) == 4)
    return raw[i];
  else
    return __uint_as_float(0x4B000000u | (uint32_t)raw[i]) - 8388608.0f;
}

// Per plane: the repaired items, straight from the table (cells 0-3: the low
// quad, 4-7: the high quad).
template <typename T, int K>
__device__ __forceinline__ void apply_repair_table(float* rdy, const T* raw, const RepairTable& rt,
                                                   int t, int nt) {
  const int n = (int)*rt.count;
  for (int i = t; i < n; i += nt) {
    const uint4 w = rt.src[i];
    const int ro = 4 * (int)rt.dst[i];
    VKT_CHECK((n <= Cfg<T, K>::MAX_REPAIR), "repair table: count");
    const float c0 = raw_value(raw, w.x & 0xFFFFu), c1 = raw_value(raw, w.x >> 16);
    const float c2 = raw_value(raw, w.y & 0xFFFFu), c3 = raw_value(raw, w.y >> 16);
    const float c4 = raw_value(raw, w.z & 0xFFFFu), c5 = raw_value(raw, w.z >> 16);
    const float c6 = raw_value(raw, w.w & 0xFFFFu), c7 = raw_value(raw, w.w >> 16);
    *reinterpret_cast<float4*>(rdy + ro) = make_float4(c0, c4, c1, c5);
    *reinterpret_cast<float4*>(rdy + Ready<K>::second(ro)) = make_float4(c2, c6, c3, c7);
  }
}

// Clamp / Mirror leave edge items to the repair-table pass; Wrap patches its
// cells from a WrapList after the main pass; Border needs no repair.
template <int MODE>
constexpr bool kRepairs = MODE == VKT_CLAMP || MODE == VKT_MIRROR;

// Wrap: the out-of-volume cells of the read window take their values
// from the far faces of the plane, in global memory, at offsets fixed for the
// CTA.  Each staging thread holds up to NB of them -- the global offset in
// the plane, the (one or two: cells x0+60..x0+67 sit in a low and a high
// pair) ready-stage float offsets packed as 16-bit halves -- and gathers the
// values for the plane its warp half stages NEXT while this one is staged,
// so the global round trip is off the staging critical path.  (Per item and
// per plane, the gathers stalled every staging warp of an edge tile: cfg5
// Wrap ran 25% behind Clamp.)  The main staging pass writes TMA's zero fill
// for these cells; a half-wide named barrier orders the patch after it.
template <typename T, int K, int NT>
struct WrapList {
  using C = Cfg<T, K>;
  static constexpr int R = C::R;
  static constexpr int NB = K == 3 ? 2 : (K == 9 ? 2 : 4);  // K = 9: registers
  int off[NB];
  uint32_t dst[NB];  // lo: first ready offset, hi: second (0xFFFF: none); 0xFFFFFFFF: no entry
  float val[NB];
  bool overflow;     // more than NB * NT cells (volumes thinner than TY + R)

  // Cell q of the window [x0-R, min(x0+TX,nx)+R) x [y0-R, min(y0+TY,ny)+R):
  // rows above / below the volume in full, then the left / right strips of
  // the other rows.  Returns the cell count.
  __device__ __forceinline__ static int cell(const TmaParams& p, int x0, int y0, int q, int& gx,
                                             int& gy) {
    const int xa = x0 - R, xb = min(x0 + TX, p.nx) + R;
    const int ya = y0 - R, yb = min(y0 + TY, p.ny) + R;
    const int w = xb - xa, rows = yb - ya;
    const int top = min(rows, max(0, -ya));
    const int bot = min(rows - top, max(0, yb - p.ny));
    const int nl = max(0, -xa);
    const int side = nl + max(0, xb - p.nx);
    const int n_rows = (top + bot) * w;
    if (q < n_rows) {
      const int r = q / w;
      gy = r < top ? ya + r : p.ny + (r - top);
      gx = xa + (q - r * w);
    } else if (side > 0) {
      const int q2 = q - n_rows;
      const int r = q2 / side;
      const int c = q2 - r * side;
      gy = ya + top + r;
      gx = c < nl ? xa + c : p.nx + (c - nl);
    }
    return n_rows + (rows - top - bot) * side;
  }
  // ready-stage offsets of cell (gx, gy), packed as above
  __device__ __forceinline__ static uint32_t dests(int x0, int y0, int gx, int gy) {
    const int by = gy - y0 + R, e = gx - x0 + 4;  // ready row, cell column
    // in-row float f of the paired layout, through the row's bank swizzle
    auto phys = [&](int f) { return (uint32_t)(by * C::RPF + Ready<K>::in_row(f & ~3) + (f & 3)); };
    const uint32_t d0 = e < NPR ? phys(2 * e) : 0xFFFFu;
    const uint32_t d1 = e >= HALF ? phys(2 * (e - HALF) + 1) : 0xFFFFu;
    return d0 != 0xFFFFu ? (d0 | (d1 << 16)) : (d1 | 0xFFFF0000u);
  }
  __device__ __forceinline__ static void put(float* rdy, uint32_t d, float v) {
    rdy[d & 0xFFFFu] = v;
    if ((d >> 16) != 0xFFFFu) rdy[d >> 16] = v;
  }

  __device__ __forceinline__ WrapList(const TmaParams& p, int x0, int y0, bool active, int t) {
    int gx = 0, gy = 0;
    const int total = active ? cell(p, x0, y0, 0, gx, gy) : 0;
    overflow = total > NB * NT;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int q = t + NT * b;
      dst[b] = 0xFFFFFFFFu;
      off[b] = 0;
      val[b] = 0.f;
      if (q < total) {
        cell(p, x0, y0, q, gx, gy);
        off[b] = map_index32<VKT_WRAP>(gy, p.ny) * p.pitch + map_index32<VKT_WRAP>(gx, p.nx);
        dst[b] = dests(x0, y0, gx, gy);
      }
    }
  }
  __device__ __forceinline__ void gather(const T* plane) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (dst[b] != 0xFFFFFFFFu) val[b] = widen(__ldg(plane + off[b]));
  }
  // plane: this stage's source plane, for the cells past the list (rare)
  __device__ __forceinline__ void apply(float* rdy, const T* plane, const TmaParams& p, int x0,
                                        int y0, int t) const {
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (dst[b] != 0xFFFFFFFFu) put(rdy, dst[b], val[b]);
    if (overflow) {
      int gx = 0, gy = 0;
      const int total = cell(p, x0, y0, 0, gx, gy);
#pragma unroll 1
      for (int q = t + NB * NT; q < total; q += NT) {
        cell(p, x0, y0, q, gx, gy);
        const float v = widen(__ldg(plane + map_index32<VKT_WRAP>(gy, p.ny) * p.pitch +
                                    map_index32<VKT_WRAP>(gx, p.nx)));
        put(rdy, dests(x0, y0, gx, gy), v);
      }
    }
  }
};
static_assert(Cfg<float, 7>::RPF * Cfg<float, 7>::BY < 0xFFFF, "ready offsets fit 16 bits");

template <typename T, int MODE, int K, int NT>
__device__ __forceinline__ void stage_plane(float* rdy, const T* raw, const T* plane,
                                            const TmaParams& p, int x0, int y0, bool edge,
                                            const StagePlan<T, K, NT, kRepairs<MODE>>& sp,
                                            const RepairTable& rt, int t) {
#pragma unroll
  for (int k = 0; k < StagePlan<T, K, NT, kRepairs<MODE>>::QPT; ++k) {
    int ro, wo;
    sp.get(k, ro, wo);
    if (ro < 0) continue;
    VKT_CHECK((Ready<K>::second(ro) + 4 <= Cfg<T, K>::RPF * Cfg<T, K>::BY), "paired staging: ready offset");
    VKT_CHECK((wo >= 0 && (wo + HALF + 4) * (int)sizeof(T) <= Cfg<T, K>::RAW_BYTES), "paired staging: raw offset");
    uint32_t lo[4], hi[4];
    load_quad<T>(raw + wo, lo);
    load_quad<T>(raw + wo + HALF, hi);
    uint64_t pr[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if constexpr (sizeof(T) == 4)
        pr[c] = (uint64_t)lo[c] | ((uint64_t)hi[c] << 32);
      else
        pr[c] = widen2(lo[c], hi[c]);
    }
    *reinterpret_cast<uint4*>(rdy + ro) =
        make_uint4((uint32_t)pr[0], (uint32_t)(pr[0] >> 32), (uint32_t)pr[1], (uint32_t)(pr[1] >> 32));
    *reinterpret_cast<uint4*>(rdy + Ready<K>::second(ro)) =
        make_uint4((uint32_t)pr[2], (uint32_t)(pr[2] >> 32), (uint32_t)pr[3], (uint32_t)(pr[3] >> 32));
  }
  // Clamp / Mirror: from the CTA's repair table (Wrap: WrapList, after the
  // pass).  One mechanism per kernel: each extra repair path changed ptxas's
  // allocation of the FFMA2 main loop (spills, lost uniform weights).
  if constexpr (MODE == VKT_CLAMP || MODE == VKT_MIRROR) {
    if (edge) apply_repair_table<T, K>(rdy, raw, rt, t, NT);
  }
}

// ---------------------------------------------------------------------------
// Compute helpers
// ---------------------------------------------------------------------------
// Epilogue: floor each sum to s32, then saturate-and-pack (I2IP) and store.
// Floor to s32 (F2I), then saturate-and-pack to u8 / u16 (I2IP): one
// conversion and half a pack per output.  floor-then-saturate equals the
// reference rule's floor(clip(.)) on the biased sum (acc_init adds the 0.5)
// for every finite sum, and common.cuh's quantize_acc, so every kernel path
// stays bit-identical.  (An FADD2.RM + 2^23 bias variant avoids F2I but
// measured slower: 1.363 vs 1.320 ms, u8 3^3 1024^3.)
__device__ __forceinline__ int floor_s32(float v) {
  int r;
  asm("cvt.rmi.s32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}
// floor of both halves of an accumulator pair as s32
__device__ __forceinline__ void floor2_s32(uint64_t a, int& lo, int& hi) {
  lo = floor_s32(f2lo(a));
  hi = floor_s32(f2hi(a));
}
template <typename T>
__device__ __forceinline__ void store4i(T* out, int a0, int a1, int a2, int a3);
template <>
__device__ __forceinline__ void store4i<uint8_t>(uint8_t* out, int a0, int a1, int a2, int a3) {
  // cvt.pack.sat.u8.s32.b32 d, a, b, c: d = {c[15:0], sat(a), sat(b)} (b in byte 0)
  uint32_t hi, v;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(a3), "r"(a2));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(v) : "r"(a1), "r"(a0), "r"(hi));
  __stcs(reinterpret_cast<unsigned int*>(out), v);
}
template <>
__device__ __forceinline__ void store4i<uint16_t>(uint16_t* out, int a0, int a1, int a2, int a3) {
  uint32_t lo, hi;
  asm("cvt.pack.sat.u16.s32 %0, %1, %2;" : "=r"(lo) : "r"(a1), "r"(a0));
  asm("cvt.pack.sat.u16.s32 %0, %1, %2;" : "=r"(hi) : "r"(a3), "r"(a2));
  __stcs(reinterpret_cast<uint2*>(out), make_uint2(lo, hi));
}

template <typename T>
__device__ __forceinline__ void store4(T* out, float a0, float a1, float a2, float a3);

template <>
__device__ __forceinline__ void store4<float>(float* out, float a0, float a1, float a2, float a3) {
  __stcs(reinterpret_cast<float4*>(out), make_float4(a0, a1, a2, a3));
}
template <>
__device__ __forceinline__ void store4<uint16_t>(uint16_t* out, float a0, float a1, float a2,
                                                 float a3) {
  store4i<uint16_t>(out, floor_s32(a0), floor_s32(a1), floor_s32(a2), floor_s32(a3));
}
template <>
__device__ __forceinline__ void store4<uint8_t>(uint8_t* out, float a0, float a1, float a2,
                                                float a3) {
  store4i<uint8_t>(out, floor_s32(a0), floor_s32(a1), floor_s32(a2), floor_s32(a3));
}

// Rolling accumulators of one thread: slot m holds the partial sums of the
// output plane the current input plane reaches with dz = K-1-m, as packed
// pairs (output x, output x+HALF) for the thread's 4 x positions.
template <int K, int YPT>
struct Accum {
  uint64_t p[YPT][K][XQ];
};

// The aligned run of ready pairs a thread loads per row: output pair j
// (x = x0+4tx+j) at tap dx reads ready pair 4tx+j+dx+4-R, so the thread loads
// pairs [4tx+LOFF, 4tx+LOFF+2*NLD) as NLD 16-byte chunks.  off[i]: chunk i's
// physical in-row float offset (swizzled layout only; the plain layout
// addresses chunk i as base + 4i).
template <int K>
struct LoadRun {
  static constexpr int R = K / 2;
  static constexpr int LOFF = (4 - R) & ~1;
  static constexpr int SH = 4 - R - LOFF;                // 0 or 1
  static constexpr int NLD = (XQ + K - 1 + SH + 1) / 2;  // LDS.128 per row
  static constexpr int NOFF = Ready<K>::SWZ ? NLD : 1;
  __device__ __forceinline__ static void offsets(int tx, int (&off)[NOFF]) {
#pragma unroll
    for (int i = 0; i < NOFF; ++i) off[i] = Ready<K>::in_row(2 * (XQ * tx + LOFF) + 4 * i);
  }
};

// One input plane's contribution to the K rolling accumulators of the
// thread's YPT x 4 output pairs.  GUARD: skip slots whose output plane is
// outside the chunk (ramp up / down; those sums are never stored).
// ROLL_IN (steady planes of the unrolled, unskipped kernels): the plane's
// first tap into slot m (dy = dx = 0) reads slot m+1 -- the partial sum one
// output plane later -- or the epilogue constant a00 for slot K-1, and writes
// slot m, so the accumulators roll without register moves.  Other planes
// roll explicitly before their taps (roll_slots).
template <int K, int YPT, bool GUARD, bool UNROLL, bool SKIP, int KXS, bool ROLL_IN = false,
          int KZS = K>
__device__ __forceinline__ void plane_step(const float* __restrict__ stage,
                                           const int (&off)[LoadRun<K>::NOFF], int ty,
                                           const Weights<K>& wt, Accum<KZS, YPT>& acc, int first,
                                           int last, uint32_t zskip, uint32_t yskip,
                                           uint64_t a00 = 0) {
  static_assert(!ROLL_IN || (UNROLL && !GUARD && !SKIP), "in-FMA roll needs every tap, unrolled");
  constexpr int SH = LoadRun<K>::SH;
  constexpr int NLD = LoadRun<K>::NLD;
  constexpr int RPF = Ready<K>::RPF;
  const float* base = stage + YPT * ty * RPF;
  // dy unrolled (UNROLL): rolled, ptxas renames the accumulators at the back
  // edge with IMAD.MOV (FMA pipe) — measured at K = 5: 4.46 vs 5.33 ms.
#pragma unroll(UNROLL ? K : 1)
  for (int dy = 0; dy < K; ++dy) {
    uint64_t P[YPT][2 * NLD];
#pragma unroll
    for (int r = 0; r < YPT; ++r) {
      const float* row = base + (r + dy) * RPF;
#pragma unroll
      for (int i = 0; i < NLD; ++i) {
        const float4 q = *reinterpret_cast<const float4*>(
            row + (Ready<K>::SWZ ? off[Ready<K>::SWZ ? i : 0] : off[0] + 4 * i));
        P[r][2 * i] = f2pack(q.x, q.y);
        P[r][2 * i + 1] = f2pack(q.z, q.w);
      }
    }
#pragma unroll
    for (int m = 0; m < KZS; ++m) {
      if (GUARD && (m < first || m > last)) continue;
      // slot m of the KZS z slots; a z-thin variant (KZS = 1) has only the
      // cube's centre plane
      const int dz = (K - KZS) / 2 + KZS - 1 - m;
      // z planes / y rows that only pad an anisotropic kernel to the K^3
      // cube: no FMA at all (a zero weight times an Inf would inject NaN,
      // and the FMA pipe is the bound); uniform branches per (dz, dy) row
      if (SKIP && (((zskip >> dz) | (yskip >> dy)) & 1u)) continue;
      const float* w = wt.w + (dz * K + dy) * Weights<K>::KP;
      // x taps: the kernel's own KXS columns of the cube (a template)
#pragma unroll
      for (int dx = (K - KXS) / 2; dx < (K + KXS) / 2; ++dx) {
        const float wv = w[dx];
#pragma unroll
        for (int r = 0; r < YPT; ++r)
#pragma unroll
          for (int j = 0; j < XQ; ++j) {
            if (ROLL_IN && dy == 0 && dx == 0)
              acc.p[r][m][j] = ffma2_from(P[r][j + dx + SH], wv, m + 1 < KZS ? acc.p[r][m + 1 < KZS ? m + 1 : m][j] : a00);
            else
              ffma2_bw(P[r][j + dx + SH], wv, acc.p[r][m][j]);
          }
      }
    }
  }
}

template <typename T, int K, int MODE, bool SKIP = false, int KXS = K, int KZS = K>
__global__ void __launch_bounds__(Layout<(int)sizeof(T), K>::THREADS,
                                  Layout<(int)sizeof(T), K>::CTAS_PER_SM)
    filter_tma_kernel(const __grid_constant__ CUtensorMap map_src,
                      const __grid_constant__ CUtensorMap map_lo,
                      const __grid_constant__ CUtensorMap map_hi, const TmaParams p,
                      const __grid_constant__ Weights<K> wt) {
  if (p.guard != nullptr && *p.guard != 0) return;  // uniform over the grid
  using C = Cfg<T, K>;
  constexpr int R = C::R;
  constexpr int S = C::S_RDY;
  constexpr int SR = C::S_RAW;
  using L = Layout<(int)sizeof(T), K>;
  constexpr int YPT = L::YPT;
  constexpr int WARPS = L::WARPS;
  constexpr int THREADS = L::THREADS;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // TMA destinations must be 128-byte aligned; do not rely on the base.
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float* rdy_base = reinterpret_cast<float*>(smem);
  T* raw_base = reinterpret_cast<T*>(smem + S * C::RDY_PITCH);
  RepairTable rtab;
  rtab.count = reinterpret_cast<uint32_t*>(smem + C::SMEM_DATA);
  rtab.src = reinterpret_cast<uint4*>(smem + C::SMEM_DATA + 16);
  rtab.dst = reinterpret_cast<uint16_t*>(smem + C::SMEM_DATA + 16 + 16 * C::MAX_REPAIR);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_DATA + C::REPAIR_BYTES);
  uint64_t* full = bars;            // [SR] TMA landed
  uint64_t* raw_free = full + SR;   // [SR] all warps done staging from the raw slot
  uint64_t* ready = raw_free + SR;  // [S]  staged plane complete (WARPS arrivals)
  uint64_t* empty = ready + S;      // [S]  all warps done computing from the stage

  const int tid = threadIdx.x;
  const int lane = tid % 32;
  // 8-warp layouts stage alternate planes with alternate warp halves (warps
  // 0-3 even planes, 4-7 odd): each SM sub-partition holds one warp of each
  // half, so one of them can issue FFMA2 while the other stages.  The half is
  // broadcast from lane 0 so ptxas sees it as warp-uniform (a per-thread
  // branch would push the weights off the uniform datapath).
  constexpr bool SPLIT = WARPS == 8;
  constexpr int SW = SPLIT ? WARPS / 2 : WARPS;  // staging warps per plane
  constexpr int ST = 32 * SW;
  const int half = __shfl_sync(0xffffffffu, tid / ST, 0);
  const int warp = __shfl_sync(0xffffffffu, tid / 32, 0);
  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int x0 = bx * TX;
  const int y0 = by * TY;
  const int zo0 = p.z_begin + bz * p.zc;
  const int nzo = min(p.zc, p.z_end - zo0);
  if (nzo <= 0) return;
  // KZS z slots: K, or 1 for a z-thin anisotropic kernel (no z halo, no roll)
  constexpr int RZ = KZS / 2;
  const int np = nzo + 2 * RZ;  // input planes of this chunk
  const bool edge = (x0 - R < 0) || (x0 + TX + R > p.nx) || (y0 - R < 0) || (y0 + TY + R > p.ny);

  if (tid == 0) {
    prefetch_tmap(&map_src);
    for (int s = 0; s < SR; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&raw_free[s], SW);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&ready[s], SW);
      mbar_init(&empty[s], WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *rtab.count = 0;
  }
  __syncthreads();
  if ((MODE == VKT_CLAMP || MODE == VKT_MIRROR) && edge) {
    build_repair_table<T, MODE, K, THREADS>(rtab, p, x0, y0, tid);
    __syncthreads();
  }

  // TMA plane j into raw slot j % SR (zero planes: plain arrive).  Called by
  // all threads; only thread 0 acts (predicated, no divergent branch).
  const bool leader = tid == 0;
  auto issue = [&](int j) {
    const int r = j % SR;
    const PlaneSrc s = resolve<MODE>(p, RZ, zo0 - RZ + j);
    if (s.which < 0) {
      mbar_arrive_if(&full[r], leader);
      return;
    }
    const CUtensorMap* m = s.which == 0 ? &map_src : s.which == 1 ? &map_lo : &map_hi;
    tma_issue_if(raw_base + r * (C::RAW_PITCH / (int)sizeof(T)), m, &full[r], C::RAW_BYTES,
                 x0 - C::A, y0 - R, s.z, leader);
  };

  // stage plane j (SW warps, equal shares) into ready slot j % S
  const StagePlan<T, K, ST, kRepairs<MODE>> splan(p, x0, y0, edge, tid % ST);
  constexpr bool WLIST = MODE == VKT_WRAP;
  constexpr int WSTEP = SPLIT ? 2 : 1;  // the next plane this warp half stages
  WrapList<T, K, ST> wlist(p, x0, y0, WLIST && edge, tid % ST);
  if (WLIST && edge && (SPLIT ? half : 0) < np)
    wlist.gather(plane_ptr<T>(p, resolve<MODE>(p, RZ, zo0 - RZ + (SPLIT ? half : 0))));
  auto prepare = [&](int j) {
    if (SPLIT && half != (j & 1)) return;
    VKT_JITTER_POINT(4 * j);
    const int s = j % S;
    float* stage = rdy_base + s * (C::RDY_PITCH / 4);
    const int r = j % SR;
    mbar_wait(&full[r], (uint32_t)((j / SR) & 1));
    if (j >= S) mbar_wait(&empty[s], (uint32_t)(((j / S) - 1) & 1));
    const PlaneSrc src = resolve<MODE>(p, RZ, zo0 - RZ + j);
    if (src.which < 0) {
      float4* w4 = reinterpret_cast<float4*>(stage);
      for (int q = tid % ST; q < C::RDY_BYTES / 16; q += ST) w4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const T* raw = raw_base + r * (C::RAW_PITCH / (int)sizeof(T));
      stage_plane<T, MODE, K, ST>(stage, raw, plane_ptr<T>(p, src), p, x0, y0, edge, splan, rtab,
                                  tid % ST);
      if constexpr (WLIST) {
        if (edge) {
          // after the whole half's main pass (it wrote the zero fill there)
          asm volatile("bar.sync %0, %1;" ::"r"(1 + half), "r"(ST) : "memory");
          wlist.apply(stage, plane_ptr<T>(p, src), p, x0, y0, tid % ST);
          if (j + WSTEP < np) wlist.gather(plane_ptr<T>(p, resolve<MODE>(p, RZ, zo0 - RZ + j + WSTEP)));
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&ready[s]);
      mbar_arrive(&raw_free[r]);
    }
  };

  for (int j = 0; j < SR && j < np; ++j) issue(j);
  for (int j = 0; j < C::AHEAD && j < np; ++j) prepare(j);

  // lane layout: tx 0..3 of two adjacent rows in each quarter-warp (see Ready<K>)
  static_assert(TPR == 16 && YPT == 1, "lane layout");
  const int tx = (lane & 3) | ((lane >> 3) << 2);
  const int ty = 2 * (tid / 32) + ((lane >> 2) & 1);
  int ld_off[LoadRun<K>::NOFF];
  LoadRun<K>::offsets(tx, ld_off);
  const float a0 = acc_init<T>(p.c);
  const uint64_t a00 = f2pack(a0, a0);
  Accum<KZS, YPT> acc;
#pragma unroll
  for (int r = 0; r < YPT; ++r)
#pragma unroll
    for (int m = 0; m < KZS; ++m)
#pragma unroll
      for (int j = 0; j < XQ; ++j) acc.p[r][m][j] = a00;

  // outputs x0+4tx+j (lo) and +HALF (hi); cells beyond nx up to the pitch are
  // padding (storing there is harmless), and a 4-cell group never straddles
  // the pitch (a 16-byte multiple)
  const int ox = x0 + XQ * tx;
  const int oy = y0 + YPT * ty;
  const bool st_lo = ox < p.pitch, st_hi = ox + HALF < p.pitch;
  bool row_ok[YPT];
#pragma unroll
  for (int r = 0; r < YPT; ++r) row_ok[r] = oy + r < p.ny;
  T* out_base = static_cast<T*>(p.dst) + (int64_t)oy * p.pitch + ox;
  const int64_t plane_elems = (int64_t)p.pitch * p.ny;

  for (int i = 0; i < np; ++i) {
    const int s = i % S;
    const float* stage = rdy_base + s * (C::RDY_PITCH / 4);
    VKT_JITTER_POINT(4 * i + 1);
    // refill the raw slot of plane i-1 (staged AHEAD iterations before).
    // Only warp 0 (the TMA issuer's) waits for the slot: a warp of the other
    // staging half may run up to S_RDY - AHEAD planes ahead, and if the ring
    // has S_RAW <= S_RDY it can complete the slot's NEXT phase too, so a
    // lagging warp waiting on the parity would see the phase after next and
    // deadlock.  Warp 0 cannot lag past its own refill.
    if (i >= 1 && i - 1 + SR < np) {
      if (warp == 0) mbar_wait(&raw_free[(i - 1) % SR], (uint32_t)(((i - 1) / SR) & 1));
      issue(i - 1 + SR);
    }
    if (i + C::AHEAD < np) prepare(i + C::AHEAD);
    mbar_wait(&ready[s], (uint32_t)((i / S) & 1));
    // slot m <-> output plane zo0 + i - 2R + m
    const int first = 2 * RZ - i;
    const int last = nzo - 1 - i + 2 * RZ;
    // The steady-state planes run the dy loop unrolled; the ramp planes
    // (GUARD, 2R of every chunk's ~70) keep it rolled at K = 7, which keeps
    // the kernel's hot code compact (K = 7: 11.76 -> 11.33 ms for u16, 11.39
    // -> 11.11 ms for f32, against all-rolled / all-unrolled).
    constexpr bool UNROLL = K <= 7;  // K = 9 unrolled: ~2900 FFMA2 per plane body
    constexpr bool UNROLL_G = K <= 5;  // K = 5 with rolled ramps: 4.60 vs 4.46 ms
    // accumulators after plane i-1 still hold slot m = output plane
    // zo0 + i-1 - 2R + m; the plane's first taps (ROLL_IN) or roll_slots
    // shift them by one (the former IMAD.MOV roll after every plane: ~3.5%
    // of the K = 7 instructions)
    constexpr bool ROLL_IN = UNROLL && !SKIP;
    auto roll_slots = [&]() {
#pragma unroll
      for (int r = 0; r < YPT; ++r)
#pragma unroll
        for (int j = 0; j < XQ; ++j) {
#pragma unroll
          for (int m = 0; m + 1 < KZS; ++m) acc.p[r][m][j] = acc.p[r][m + 1][j];
          acc.p[r][KZS - 1][j] = a00;
        }
    };
    if (first <= 0 && last >= KZS - 1) {
      if constexpr (!ROLL_IN) roll_slots();
      plane_step<K, YPT, false, UNROLL, SKIP, KXS, ROLL_IN, KZS>(stage, ld_off, ty, wt, acc, 0, KZS - 1,
                                                                 p.zskip, p.yskip, a00);
    } else {
      roll_slots();
      plane_step<K, YPT, true, UNROLL_G, SKIP, KXS, false, KZS>(stage, ld_off, ty, wt, acc, first, last,
                                                                p.zskip, p.yskip);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (i >= 2 * RZ) {
      const int oz = zo0 + i - 2 * RZ;
#pragma unroll
      for (int r = 0; r < YPT; ++r) {
        if (!row_ok[r]) continue;
        T* o = out_base + (int64_t)oz * plane_elems + (int64_t)r * p.pitch;
        const uint64_t* a = acc.p[r][0];
        if (st_lo) store4<T>(o, f2lo(a[0]), f2lo(a[1]), f2lo(a[2]), f2lo(a[3]));
        if (st_hi) store4<T>(o + HALF, f2hi(a[0]), f2hi(a[1]), f2hi(a[2]), f2hi(a[3]));
      }
    }
  }
}

template <typename T, int K, int MODE, bool SKIP = false, int KXS = K, int KZS = K>
cudaError_t launch_tma_kernel(const CUtensorMap& ms, const CUtensorMap& ml, const CUtensorMap& mh,
                              const TmaParams& p, const float* w32, dim3 grid, cudaStream_t s) {
  using C = Cfg<T, K>;
  Weights<K> wt = {};
  for (int r = 0; r < K * K; ++r)
    for (int x = 0; x < K; ++x) wt.w[r * Weights<K>::KP + x] = w32[r * K + x];
  auto fn = filter_tma_kernel<T, K, MODE, SKIP, KXS, KZS>;
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
  fn<<<grid, C::L::THREADS, C::SMEM, s>>>(ms, ml, mh, p, wt);
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
  VKT_TMA_K(5)
  VKT_TMA_K(7)
  VKT_TMA_K(9)
#undef VKT_TMA_K
#undef VKT_TMA_CASE
  return cudaErrorInvalidValue;
}

}  // namespace tma
}  // namespace vkt
