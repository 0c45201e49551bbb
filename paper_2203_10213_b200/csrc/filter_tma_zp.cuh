// filter_tma_zp.cuh — the f32 3x3x3 ApplyFilter kernel (TMA straight into the
// compute layout).
//
// For float voxels the 3^3 filter is HBM-bound (8 bytes and 27 FMAs per
// voxel), so this kernel skips the staging pass of filter_tma.cuh: each
// input plane is ONE TMA 3D box load (cp.async.bulk.tensor.3d, completion on
// an mbarrier with complete_tx) straight into the row-major ready stage it
// computes from (box 136 x 18 cells = the tile plus its halo), and K-1 of the
// K accumulator slots are paired along z (FFMA2 with a broadcast input and a
// weight pair) while the last slot is a plain FFMA.  Measured at 1024^3: 1.71
// vs 2.03 ms for the all-FFMA2 paired layout, whose staging pass costs more
// than its packing gains here.
//  * A CTA owns a TX=128 (x) by TY=16 (y) column of outputs and a chunk of ZC
//    output planes; 4 warps, each thread 2 rows x 8 consecutive x outputs.
//    No dedicated producer warp: lane 0 of warp 0 issues the TMA loads and
//    every warp computes; warps meet only on the full / empty mbarrier rings.
//  * Edge tiles patch the out-of-volume cells of each warp's read window in
//    the stage before computing: Clamp / Mirror from in-stage cells through a
//    per-lane list fixed for the CTA (FixList), Wrap from the far faces in
//    global memory, gathered one plane ahead (WrapList); Border is TMA's zero
//    fill, and Border z planes outside the volume are cleared by each warp.
//  * Tap order per output is (dz, dy, dx) — the reference's order
//    (filters.py:89-92) and the direct kernel's — so every kernel path and
//    every z-slab split produce bit-identical results.
//  * Epilogue: the sums are stored verbatim (f32 quantize is astype('<f4'),
//    volume.py:106) with streaming 128-bit stores.
#pragma once

#include <cuda.h>

#include <atomic>

#include "filter_tma.cuh"

namespace vkt {
namespace tma_zp {

using tma::TmaParams;
using tma::PlaneSrc;
using tma::f2hi;
using tma::f2lo;
using tma::f2pack;
using tma::fence_proxy_async;
using tma::mbar_arrive;
using tma::mbar_arrive_if;
using tma::mbar_init;
using tma::mbar_wait;
using tma::plane_ptr;
using tma::prefetch_tmap;
using tma::resolve;
using tma::smem_u32;
using tma::tma_issue_if;

constexpr int TX = 128;          // outputs per CTA in x
constexpr int TY = 16;           // outputs per CTA in y
constexpr int XPT = 8;           // outputs per thread in x
constexpr int RP = TX + 8;       // ready-stage row pitch (floats): x in [x0-4, x0+TX+4)

// 2 output rows per thread, 4 warps; 4 CTAs/SM (122 registers, 56 KB of
// rings each): Clamp 1.49 vs 1.57 ms at 1024^3 with 3.  Wrap keeps 3: its
// prefetch registers spill at 128.
template <int K, int MODE = VKT_CLAMP>
struct Layout {
  static_assert(K == 3, "f32 3x3x3 only (K >= 5 run filter_tma.cuh)");
  static constexpr int YPT = 2;
  static constexpr int WARPS = TY * (TX / XPT) / (32 * YPT);
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int CTAS_PER_SM = MODE == VKT_WRAP ? 3 : 4;
  static constexpr int WROWS = TY / WARPS;  // output rows per warp
  static constexpr int SMEM_PER_CTA = (228 * 1024) / CTAS_PER_SM - 1024;  // minus driver reserve
};

template <typename T, int K, int MODE = VKT_CLAMP>
struct Cfg {
  static_assert(sizeof(T) == 4, "float voxels only");
  using L = Layout<K, MODE>;
  static constexpr int R = K / 2;
  static constexpr int A = tma::box_align_left(R, 4);
  static constexpr int BX = tma::box_width(R, 4);
  static constexpr int BY = TY + 2 * R;
  static constexpr int RDY_BYTES = RP * BY * 4;
  static constexpr int RDY_PITCH = (RDY_BYTES + 127) / 128 * 128;
  // The TMA lands in the ready ring, so its depth is the TMA lookahead: as
  // deep as fits CTAS_PER_SM CTAs per SM, capped at 10.
  static constexpr int BUDGET = L::SMEM_PER_CTA - 512;
  static constexpr int S_RDY = BUDGET / RDY_PITCH < 10 ? BUDGET / RDY_PITCH : 10;
  // at iteration i the TMA slot of plane i - LAG is refilled (every warp must
  // have released it): larger LAG = more slack between warps, smaller TMA
  // lookahead (S_RDY - LAG); HBM-bound, so the lookahead wins
  static constexpr int LAG = 2;
  static constexpr int SMEM_DATA = S_RDY * RDY_PITCH;
  static constexpr int NBAR = 2 * S_RDY;
  static constexpr int SMEM = SMEM_DATA + NBAR * 8 + 128;
  static_assert(BX == RP, "the TMA box must match the ready layout");
  static_assert(S_RDY >= 4, "ring too shallow");
  static_assert(SMEM <= L::SMEM_PER_CTA, "shared memory budget");
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

// ---------------------------------------------------------------------------
// Edge repair
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

// ---------------------------------------------------------------------------
// Compute helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void store8(float* out, const float (&a)[XPT], int valid) {
  if (valid >= 4) __stcs(reinterpret_cast<float4*>(out), make_float4(a[0], a[1], a[2], a[3]));
  if (valid >= 8) __stcs(reinterpret_cast<float4*>(out) + 1, make_float4(a[4], a[5], a[6], a[7]));
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
template <int K, bool GUARD>
__device__ __forceinline__ void plane_step(const float* __restrict__ stage, int tx, int ty,
                                           const Weights<K>& wt, Accum<K>& acc, int first,
                                           int last) {
  constexpr int YPT = Layout<K>::YPT;
  constexpr int R = K / 2;
  constexpr int NP = K / 2;
  constexpr int OFF = 4 - R;
  float4 nx[YPT][4];
  const float* base = stage + YPT * ty * RP + XPT * tx;
#pragma unroll
  for (int dy = 0; dy < K; ++dy) {
#pragma unroll
    for (int r = 0; r < YPT; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i) nx[r][i] = reinterpret_cast<const float4*>(base + (r + dy) * RP)[i];
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

template <int MODE>
__global__ void __launch_bounds__(Layout<3>::THREADS, Layout<3, MODE>::CTAS_PER_SM)
    filter_tma_kernel(const __grid_constant__ CUtensorMap map_src,
                      const __grid_constant__ CUtensorMap map_lo,
                      const __grid_constant__ CUtensorMap map_hi, const TmaParams p,
                      const __grid_constant__ Weights<3> wt) {
  if (p.guard != nullptr && *p.guard != 0) return;  // uniform over the grid
  constexpr int K = 3;
  using C = Cfg<float, K, MODE>;
  constexpr int R = C::R;
  constexpr int S = C::S_RDY;
  constexpr int YPT = Layout<K>::YPT;
  constexpr int WARPS = Layout<K>::WARPS;
  constexpr int THREADS = Layout<K>::THREADS;
  constexpr int WROWS = Layout<K>::WROWS;
  constexpr int SR = C::S_RDY;  // TMA ring depth: the TMA lands in the ready ring
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // TMA destinations must be 128-byte aligned; do not rely on the base.
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float* rdy_base = reinterpret_cast<float*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_DATA);
  uint64_t* full = bars;            // [S] TMA landed in the ready stage
  uint64_t* empty = full + S;       // [S] all warps done computing from the stage

  const int tid = threadIdx.x;
  const int warp = tid / 32;
  const int lane = tid % 32;
  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int x0 = bx * TX;
  const int y0 = by * TY;
  const int zo0 = p.z_begin + bz * p.zc;
  const int nzo = min(p.zc, p.z_end - zo0);
  if (nzo <= 0) return;
  const int np = nzo + 2 * R;  // input planes of this chunk
  const bool edge = (x0 - R < 0) || (x0 + TX + R > p.nx) || (y0 - R < 0) || (y0 + TY + R > p.ny);

  if (tid == 0) {
    prefetch_tmap(&map_src);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
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
    void* dst = rdy_base + r * (C::RDY_PITCH / 4);
    const PlaneSrc s = resolve<MODE>(p, R, zo0 - R + j);
    if (s.which < 0) {
      mbar_arrive_if(&full[r], leader);
      return;
    }
    const CUtensorMap* m = s.which == 0 ? &map_src : s.which == 1 ? &map_lo : &map_hi;
    tma_issue_if(dst, m, &full[r], C::RDY_BYTES, x0 - C::A, y0 - R, s.z, leader);
  };

  for (int j = 0; j < SR && j < np; ++j) issue(j);

  const int tx = tid % (TX / XPT);
  const int ty = tid / (TX / XPT);
  const float a0 = acc_init<float>(p.c);
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
  float* out_base = static_cast<float*>(p.dst) + (int64_t)oy * p.pitch + ox;
  const int64_t plane_elems = (int64_t)p.pitch * p.ny;

  const FixList<MODE, R> fix = ((MODE == VKT_CLAMP || MODE == VKT_MIRROR) && edge)
                                   ? FixList<MODE, R>(p, x0, y0, lane, WROWS * warp,
                                                      WROWS * warp + WROWS + 2 * R)
                                   : FixList<MODE, R>();
  WrapList<R> wrap = (MODE == VKT_WRAP && edge)
                         ? WrapList<R>(p, x0, y0, lane, WROWS * warp, WROWS * warp + WROWS + 2 * R)
                         : WrapList<R>();
  if (MODE == VKT_WRAP && edge && wrap.ok)
    wrap.gather(plane_ptr<float>(p, resolve<MODE>(p, R, zo0 - R)));
  for (int i = 0; i < np; ++i) {
    VKT_JITTER_POINT(4 * i + 1);
    const int s = i % S;
    float* stage = rdy_base + s * (C::RDY_PITCH / 4);
    {
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
    }
    // slot m <-> output plane zo0 + i - 2R + m
    const int first = 2 * R - i;
    const int last = nzo - 1 - i + 2 * R;
    if (first <= 0 && last >= K - 1)
      plane_step<K, false>(stage, tx, ty, wt, acc, 0, K - 1);
    else
      plane_step<K, true>(stage, tx, ty, wt, acc, first, last);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (i >= 2 * R) {
      const int oz = zo0 + i - 2 * R;
#pragma unroll
      for (int r = 0; r < YPT; ++r) {
        float o[XPT];
#pragma unroll
        for (int j = 0; j < XPT; ++j) o[j] = f2lo(acc.p[r][0][j]);
        if (valid[r] > 0) store8(out_base + (int64_t)oz * plane_elems + (int64_t)r * p.pitch, o, valid[r]);
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

template <int MODE>
cudaError_t launch_tma_kernel(const CUtensorMap& ms, const CUtensorMap& ml, const CUtensorMap& mh,
                              const TmaParams& p, const float* w32, dim3 grid, cudaStream_t s) {
  constexpr int K = 3;
  using C = Cfg<float, K, MODE>;
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
  auto fn = filter_tma_kernel<MODE>;
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

// Dispatch over the address modes (filter_tma_f32.cu).
inline cudaError_t launch_f32_k3(int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                                 const CUtensorMap& mh, const TmaParams& p, const float* w32, dim3 grid,
                                 cudaStream_t s) {
  switch (mode) {
    case VKT_WRAP: return launch_tma_kernel<VKT_WRAP>(ms, ml, mh, p, w32, grid, s);
    case VKT_MIRROR: return launch_tma_kernel<VKT_MIRROR>(ms, ml, mh, p, w32, grid, s);
    case VKT_CLAMP: return launch_tma_kernel<VKT_CLAMP>(ms, ml, mh, p, w32, grid, s);
    case VKT_BORDER: return launch_tma_kernel<VKT_BORDER>(ms, ml, mh, p, w32, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tma_zp
}  // namespace vkt
