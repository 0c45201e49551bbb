// filter_warp.cuh — the u8/u16 3x3x3 ApplyFilter kernel: warp-private staging.
//
// The integer 3^3 filter is FMA-bound (27 FMAs for 2-4 bytes per voxel) but
// only 27/64 FFMA2 per voxel: the per-plane costs of the paired-layout kernel
// (filter_tma.cuh) — CTA-wide ready/empty mbarrier rounds, slot arithmetic,
// accumulator roll moves, the F2I + VIMNMX + PRMT epilogue — are spread over
// just 16 outputs per thread and held it at 0.50 of the FP32 roofline
// (profiles/r02_ncu_u8k3_v40.txt: 1.33e9 instructions for 4.5e8 FFMA2, the
// ready-barrier wait the top stall).  This kernel removes them:
//  * Warp-private staging.  The CTA still fetches each input plane as ONE TMA
//    3D box (128+8 x 34 cells) into a raw ring (full / raw_free mbarriers),
//    but every warp widens only the 10 rows its own outputs read into its OWN
//    float "ready" buffer (same paired, bank-swizzled layout as filter_tma.cuh)
//    and computes from it; warps never wait on one another, only on the TMA.
//    Raw slots are released per warp (one arrive); warp 0 re-issues them.
//  * 32 outputs per thread per plane: 4 rows x 4 output pairs (x, x+64), so
//    every LDS.128 row load feeds up to 3 output rows and the per-plane
//    control is shared by 2x the FFMA2 of the paired kernel.  4 warps x 8 rows
//    = 32-row tiles, 3 CTAs per SM.
//  * The rolling z accumulators roll inside the FMAs: a plane's first tap
//    into logical slot m reads slot m+1's register and writes slot m's (an
//    untied fma.rn.f32x2; slot K-1 starts from the epilogue constant), so
//    there are no register moves and the plane body exists once (unrolling
//    the plane loop by K instead made a ~31 KB loop: i-cache misses
//    dominated, profiles/r02_ncu_u8k3_warp_unrolled.txt).
//  * Epilogue: F2I (floor, s32) + I2IP (saturating pack to u8 / u16) — one
//    conversion and half a pack per output instead of F2I + VIMNMX + PRMT.
//    floor-then-saturate equals the former min(float2uint_rd(.), max) on every
//    finite sum, so all paths stay bit-identical.
//  * No ramp guards: the first and last 2R planes of a chunk also feed the
//    accumulators of output planes outside the chunk, which are never stored
//    (integer inputs are finite, so those FMAs cannot poison anything).
// Tap order per output is (dz, dy, dx) as everywhere else (filters.py:89-92):
// within a plane an accumulator receives its dy rows in increasing order.
// Edge tiles: Border is TMA's zero fill (stored 0); Clamp / Mirror copy each
// out-of-volume cell of the warp's read window from its in-volume source in
// the same ready buffer; Wrap gathers the far-face cells from global memory
// (loads issued before the plane's TMA wait, so their latency overlaps it).
#pragma once

#include <type_traits>

#include "filter_tma.cuh"

namespace vkt {
namespace tmaw {

using tma::TmaParams;

constexpr int K = 3;
constexpr int R = 1;
constexpr int TX = tma::TX;        // 128 outputs in x per CTA
constexpr int HALF = tma::HALF;    // 64: x distance of a pair's two outputs
constexpr int XQ = tma::XQ;        // 4 output pairs per thread row
constexpr int TPR = tma::TPR;      // 16 threads per output row
// 4 rows per thread at 3 CTAs/SM (168 registers): 1.321 ms at 1024^3 u8,
// against 1.446 / 1.470 ms for 2 rows per thread at 4 / 5 CTAs/SM (96
// registers): more warps do not make up for the halved amortization.
constexpr int YPT = 4;             // output rows per thread
constexpr int WROWS = 2 * YPT;     // output rows per warp (2 thread rows)
constexpr int WARPS = 4;
constexpr int THREADS = 32 * WARPS;
constexpr int TY = WARPS * WROWS;  // 32 output rows per CTA
constexpr int CTAS_PER_SM = 3;
constexpr int WIN = WROWS + 2 * R;             // ready rows per warp
constexpr int NPR = tma::NPR;                  // 72 pairs per ready row
constexpr int RPF = tma::Ready<K>::RPF;        // ready row pitch (floats)
constexpr int GPR = NPR / 4;                   // staging items per row
constexpr int NQ = GPR * WIN;                  // staging items per warp-plane
constexpr int QPL = (NQ + 31) / 32;            // items per lane
constexpr int NBW = 5;                         // Wrap cells per lane held in registers
#ifndef VKT_WARP_DB
#define VKT_WARP_DB 1  // double-buffered ready staging (see the plane loop)
#endif

template <typename T>
struct Cfg {
  static constexpr int A = tma::box_align_left(R, (int)sizeof(T));
  static constexpr int BX = tma::box_width(R, (int)sizeof(T));
  static constexpr int BY = TY + 2 * R;
  static constexpr int RAW_BYTES = BX * BY * (int)sizeof(T);
  static constexpr int RAW_PITCH = (RAW_BYTES + 127) / 128 * 128;
  static constexpr int RDY_BYTES = RPF * WIN * 4 * (VKT_WARP_DB ? 2 : 1);  // per warp
  static constexpr int SMEM_PER_CTA = (228 * 1024) / CTAS_PER_SM - 1024;
  static constexpr int RING_FIT = (SMEM_PER_CTA - 256 - WARPS * RDY_BYTES) / RAW_PITCH;
  static constexpr int S_RAW = RING_FIT < 8 ? RING_FIT : 8;
  static constexpr int SMEM = S_RAW * RAW_PITCH + WARPS * RDY_BYTES + 2 * S_RAW * 8 + 128;
  static_assert(RDY_BYTES % 16 == 0, "ready buffers stay 16-byte aligned");
  static_assert(S_RAW >= 2, "TMA ring too shallow");
  static_assert(SMEM <= SMEM_PER_CTA, "shared memory budget");
  static_assert(BX <= 256 && BY <= 256, "TMA box too large");
};

// Out-of-volume cells of a warp's read window [xa, xb) x [ya, yb): rows above
// / below the volume in full, then the left / right strips of the other rows.
struct EdgeCells {
  int xa, ya, w, top, nl, side, n_rows, total;
  __device__ __forceinline__ EdgeCells(int nx, int ny, int xa_, int xb, int ya_, int yb) {
    xa = xa_;
    ya = ya_;
    w = xb - xa;
    const int rows = yb - ya;
    top = min(rows, max(0, -ya));
    const int bot = min(rows - top, max(0, yb - ny));
    nl = max(0, -xa);
    side = nl + max(0, xb - nx);
    n_rows = (top + bot) * w;
    total = rows > 0 ? n_rows + (rows - top - bot) * side : 0;
  }
  __device__ __forceinline__ void cell(int nx, int ny, int q, int& gx, int& gy) const {
    if (q < n_rows) {
      const int r = q / w;
      gy = r < top ? ya + r : ny + (r - top);
      gx = xa + (q - r * w);
    } else {
      const int q2 = q - n_rows;
      const int r = q2 / side;
      const int c = q2 - r * side;
      gy = ya + top + r;
      gx = c < nl ? xa + c : nx + (c - nl);
    }
  }
};

// Physical float offset, in a warp ready buffer whose row 0 is global row ya,
// of cell (gx, gy): its low-half copy (pairs 0..71 hold x0-4..x0+67) and its
// high-half copy (x0+60..x0+131), -1 where absent.
__device__ __forceinline__ int rdy_phys(int row, int f) {
  return row * RPF + tma::Ready<K>::in_row(f & ~3) + (f & 3);
}
__device__ __forceinline__ void rdy_dests(int x0, int ya, int gx, int gy, int& lo, int& hi) {
  const int row = gy - ya, e = gx - x0 + 4;
  lo = e >= 0 && e < NPR ? rdy_phys(row, 2 * e) : -1;
  hi = e >= HALF && e - HALF < NPR ? rdy_phys(row, 2 * (e - HALF) + 1) : -1;
}

// x * w + c0 into a fresh accumulator (an untied destination, so no register
// copy of c0 is needed to start a slot).
__device__ __forceinline__ uint64_t ffma2_from(uint64_t x, float w, uint64_t c0) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(tma::f2pack(w, w)), "l"(c0));
  return d;
}

template <typename T, int MODE>
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM)
    filter_warp_kernel(const __grid_constant__ CUtensorMap map_src,
                       const __grid_constant__ CUtensorMap map_lo,
                       const __grid_constant__ CUtensorMap map_hi, const TmaParams p,
                       const __grid_constant__ tma::Weights<K> wt) {
  using C = Cfg<T>;
  constexpr int SR = C::S_RAW;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (tma::smem_u32(smem_raw) & 127u)) & 127u);
  T* raw_base = reinterpret_cast<T*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SR * C::RAW_PITCH + WARPS * C::RDY_BYTES);
  uint64_t* raw_free = full + SR;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  float* rdy = reinterpret_cast<float*>(smem + SR * C::RAW_PITCH + warp * C::RDY_BYTES);
  const int x0 = blockIdx.x * TX;
  const int y0 = blockIdx.y * TY;
  const int zo0 = p.z_begin + blockIdx.z * p.zc;
  const int nzo = min(p.zc, p.z_end - zo0);
  if (nzo <= 0) return;
  const int np = nzo + 2 * R;

  if (tid == 0) {
    tma::prefetch_tmap(&map_src);
    for (int s = 0; s < SR; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&raw_free[s], WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // TMA plane j into raw slot j % SR (a Border zero plane: plain arrive).
  // Called by all of warp 0; only lane 0 acts (predicated).
  const bool leader = tid == 0;
  auto issue = [&](int j) {
    const int r = j % SR;
    const tma::PlaneSrc s = tma::resolve<MODE>(p, R, zo0 - R + j);
    // a Border plane outside the volume: a box entirely out of bounds in z,
    // which TMA delivers as zeros (stored 0) like any other plane
    const CUtensorMap* m = s.which <= 0 ? &map_src : s.which == 1 ? &map_lo : &map_hi;
    tma::tma_issue_if(raw_base + r * (C::RAW_PITCH / (int)sizeof(T)), m, &full[r], C::RAW_BYTES,
                      x0 - C::A, y0 - R, s.which < 0 ? -1 : s.z, leader);
  };
  if (warp == 0)
    for (int j = 0; j < SR && j < np; ++j) issue(j);

  // This lane's staging items (fixed for the CTA): item q = lane + 32k is
  // ready row q / GPR, pairs 4g..4g+3 (g = q % GPR): its ready float offset
  // and the raw cell offset of its low quad.  Items k < NQ / 32 exist in every
  // lane, so only the last needs a (per-lane) test.
  int item_ro[QPL], item_wo[QPL];
#pragma unroll
  for (int k = 0; k < QPL; ++k) {
    const int q = lane + 32 * k;
    const int row = q / GPR, g = q - row * GPR;
    item_ro[k] = row * RPF + tma::Ready<K>::in_row(8 * g);
    item_wo[k] = (warp * WROWS + row) * C::BX + 4 * g + (C::A - 4);
  }
  const bool last_item = lane + 32 * (QPL - 1) < NQ;

  // The warp's read window and its out-of-volume cells (edge tiles only)
  const int ya = y0 + warp * WROWS - R;  // global y of ready row 0
  const bool any_out = y0 + warp * WROWS < p.ny;
  const int yb = min(y0 + warp * WROWS + WROWS, p.ny) + R;
  const int xb = min(x0 + TX, p.nx) + R;
  const bool edge = any_out && (x0 - R < 0 || xb > p.nx || ya < 0 || yb > p.ny);
  const EdgeCells ec(p.nx, p.ny, x0 - R, xb, ya, edge ? yb : ya);

  // compute-side lane layout: tx along lanes 0..15, two thread rows per warp
  const int tx = lane & (TPR - 1);
  const int ty = lane >> 4;
  int ld_off[tma::LoadRun<K>::NOFF];
  tma::LoadRun<K>::offsets(tx, ld_off);
  const float a0 = acc_init<T>(p.c);
  const uint64_t a00 = tma::f2pack(a0, a0);
  uint64_t acc[YPT][K][XQ];
#pragma unroll
  for (int r = 0; r < YPT; ++r)
#pragma unroll
    for (int m = 0; m < K; ++m)
#pragma unroll
      for (int j = 0; j < XQ; ++j) acc[r][m][j] = a00;

  const int ox = x0 + XQ * tx;
  const int oy = y0 + warp * WROWS + ty * YPT;
  const bool st_lo = ox < p.pitch, st_hi = ox + HALF < p.pitch;
  const int64_t plane_elems = (int64_t)p.pitch * p.ny;
  // output plane zo0 + j - 2R of this thread's rows; advanced one plane per store
  T* out_plane = static_cast<T*>(p.dst) + (int64_t)oy * p.pitch + ox + (int64_t)zo0 * plane_elems;
  const int rows_ok = min(YPT, p.ny - oy);

  // Wrap: far-face cells of the NEXT plane this warp stages, loaded while the
  // current plane computes (their latency leaves the per-plane critical path)
  float wv[NBW];
  auto wrap_gather = [&](int j) {
    if constexpr (MODE == VKT_WRAP) {
      if (!edge || j >= np) return;
      const tma::PlaneSrc s = tma::resolve<MODE>(p, R, zo0 - R + j);
      const T* pl = tma::plane_ptr<T>(p, s);
#pragma unroll
      for (int b = 0; b < NBW; ++b) {
        const int q = lane + 32 * b;
        if (q < ec.total) {
          int gx, gy;
          ec.cell(p.nx, p.ny, q, gx, gy);
          wv[b] = tma::widen(__ldg(pl + (int64_t)map_index_near<VKT_WRAP>(gy, p.ny) * p.pitch +
                                   map_index_near<VKT_WRAP>(gx, p.nx)));
        }
      }
    }
  };
  wrap_gather(0);

  // ---- per-plane pieces ----------------------------------------------------
  // Widen the warp's rows of raw slot j % SR into ready buffer `buf` (a
  // Border plane outside the volume was fetched as a fully out-of-bounds TMA
  // box: zeros, so every plane takes this one path).
  auto stage_main = [&](int j, float* buf) {
    VKT_JITTER_POINT(4 * j);
    const T* raw = raw_base + (j % SR) * (C::RAW_PITCH / (int)sizeof(T));
#pragma unroll
    for (int k = 0; k < QPL; ++k) {
      if (32 * k + 31 >= NQ && !last_item) continue;
      const int ro = item_ro[k], wo = item_wo[k];
      VKT_CHECK(ro >= 0 && tma::Ready<K>::second(ro) + 4 <= RPF * WIN, "warp staging: ready offset");
      VKT_CHECK(wo >= 0 && (wo + HALF + 4) * (int)sizeof(T) <= C::RAW_BYTES, "warp staging: raw offset");
      uint32_t lo[4], hi[4];
      tma::load_quad<T>(raw + wo, lo);
      tma::load_quad<T>(raw + wo + HALF, hi);
      uint64_t pr[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) pr[c] = tma::widen2(lo[c], hi[c]);
      *reinterpret_cast<uint4*>(buf + ro) = make_uint4((uint32_t)pr[0], (uint32_t)(pr[0] >> 32),
                                                       (uint32_t)pr[1], (uint32_t)(pr[1] >> 32));
      *reinterpret_cast<uint4*>(buf + tma::Ready<K>::second(ro)) =
          make_uint4((uint32_t)pr[2], (uint32_t)(pr[2] >> 32), (uint32_t)pr[3],
                     (uint32_t)(pr[3] >> 32));
    }
  };
  // Out-of-volume cells of the read window (edge warps; Border: TMA's zero
  // fill already is stored 0).  Called after a __syncwarp: the in-volume
  // sources were written by other lanes.
  auto fix_edges = [&](int j, float* buf) {
    if constexpr (MODE != VKT_BORDER) {
      const tma::PlaneSrc src = tma::resolve<MODE>(p, R, zo0 - R + j);
      for (int q = lane, b = 0; q < ec.total; q += 32, ++b) {
        int gx, gy;
        ec.cell(p.nx, p.ny, q, gx, gy);
        float v;
        if constexpr (MODE == VKT_WRAP) {
          if (b < NBW) {
            v = 0.f;
#pragma unroll
            for (int t = 0; t < NBW; ++t)
              if (t == b) v = wv[t];
          } else {
            v = tma::widen(__ldg(tma::plane_ptr<T>(p, src) +
                                 (int64_t)map_index_near<VKT_WRAP>(gy, p.ny) * p.pitch +
                                 map_index_near<VKT_WRAP>(gx, p.nx)));
          }
        } else {
          int slo, shi;
          rdy_dests(x0, ya, map_index_near<MODE>(gx, p.nx), map_index_near<MODE>(gy, p.ny), slo, shi);
          VKT_CHECK((slo >= 0 ? slo : shi) >= 0 && (slo >= 0 ? slo : shi) < RPF * WIN, "warp edge fix: source");
          v = buf[slo >= 0 ? slo : shi];
        }
        int dlo, dhi;
        rdy_dests(x0, ya, gx, gy, dlo, dhi);
        VKT_CHECK(dlo < RPF * WIN && dhi < RPF * WIN && (dlo >= 0 || dhi >= 0), "warp edge fix: dest");
        if (dlo >= 0) buf[dlo] = v;
        if (dhi >= 0) buf[dhi] = v;
      }
    }
  };
  // Finish staging plane j: edge cells, release the raw slot, and start the
  // Wrap gathers of the plane staged next.
  auto finish_stage = [&](int j, float* buf, int next) {
    if (MODE != VKT_BORDER && edge) {
      __syncwarp();
      fix_edges(j, buf);
    }
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&raw_free[j % SR]);
    wrap_gather(next);
  };
  auto wait_full = [&](int j) { tma::mbar_wait(&full[j % SR], (uint32_t)((j / SR) & 1)); };
  // warp 0 re-issues raw slot of plane j once every warp has staged it (only
  // the issuer's warp waits, so no other warp is coupled to the slowest)
  auto refill = [&](int j) {
    VKT_JITTER_POINT(4 * j + 1);
    if (warp == 0 && j + SR < np) {
      tma::mbar_wait(&raw_free[j % SR], (uint32_t)((j / SR) & 1));
      issue(j + SR);
    }
  };

  // compute: each of the YPT + K - 1 input rows once, into every output row
  // it feeds (dy = row - r increasing per accumulator).  Logical slot m (the
  // output plane this input plane reaches with dz = K-1-m) is register slot
  // m; the plane's first tap into slot m (dy = dx = 0) rolls: it reads slot
  // m+1 (the partial sum one output plane later), or the epilogue constant
  // for the new slot K-1, and writes slot m.
  auto compute = [&](const float* buf) {
    VKT_JITTER_POINT(2);
    const float* base = buf + ty * YPT * RPF;
#pragma unroll
    for (int ry = 0; ry < YPT + K - 1; ++ry) {
      uint64_t P[2 * tma::LoadRun<K>::NLD];
      const float* row = base + ry * RPF;
#pragma unroll
      for (int i = 0; i < tma::LoadRun<K>::NLD; ++i) {
        const float4 q = *reinterpret_cast<const float4*>(row + ld_off[i]);
        P[2 * i] = tma::f2pack(q.x, q.y);
        P[2 * i + 1] = tma::f2pack(q.z, q.w);
      }
      // dx, then slot, then output row innermost: consecutive FFMA2s touch
      // different accumulators (up to 3 x 4 x 4 apart for the middle rows)
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
#pragma unroll
        for (int m = 0; m < K; ++m) {
#pragma unroll
          for (int rr = 0; rr < YPT; ++rr) {
            const int dy = ry - rr;
            if (dy < 0 || dy >= K) continue;
            const float wv2 = wt.w[((K - 1 - m) * K + dy) * tma::Weights<K>::KP + dx];
#pragma unroll
            for (int jj = 0; jj < XQ; ++jj) {
              const uint64_t x = P[jj + dx + tma::LoadRun<K>::SH];
              if (dy == 0 && dx == 0)
                acc[rr][m][jj] = ffma2_from(x, wv2, m + 1 < K ? acc[rr][m + 1 < K ? m + 1 : m][jj] : a00);
              else
                tma::ffma2_bw(x, wv2, acc[rr][m][jj]);
            }
          }
        }
      }
    }
  };
  // slot 0 is complete after input plane j: output plane zo0 + j - 2R
  auto epilogue = [&](int j) {
    VKT_JITTER_POINT(4 * j + 3);
    if (j < 2 * R) return;
    T* o = out_plane;
#pragma unroll
    for (int rr = 0; rr < YPT; ++rr, o += p.pitch) {
      if (rr >= rows_ok) continue;
      int nl[XQ], nh[XQ];
#pragma unroll
      for (int jj = 0; jj < XQ; ++jj) tma::floor2_s32(acc[rr][0][jj], nl[jj], nh[jj]);
      if (st_lo) tma::store4i<T>(o, nl[0], nl[1], nl[2], nl[3]);
      if (st_hi) tma::store4i<T>(o + HALF, nh[0], nh[1], nh[2], nh[3]);
    }
    out_plane += plane_elems;
  };

#if VKT_WARP_DB
  // Two ready buffers: plane j+1 is widened while plane j computes, in one
  // basic block, so the raw loads of the staging overlap the FFMA2 stream.
  constexpr int HALF_BUF = C::RDY_BYTES / 8;  // floats per buffer
  wait_full(0);
  stage_main(0, rdy);
  finish_stage(0, rdy, 1);
#pragma unroll 1
  for (int j = 0; j + 1 < np; ++j) {
    refill(j);
    float* cur = rdy + (j & 1) * HALF_BUF;
    float* nxt = rdy + ((j + 1) & 1) * HALF_BUF;
    // (probing the barrier with test_wait before the math and waiting after
    // it measured slower: 1.371 vs 1.317 ms, u8 3^3 1024^3)
    wait_full(j + 1);
    compute(cur);
    stage_main(j + 1, nxt);
    finish_stage(j + 1, nxt, j + 2);  // its __syncwarp also orders compute(cur)'s reads
    epilogue(j);
  }
  compute(rdy + ((np - 1) & 1) * HALF_BUF);
  epilogue(np - 1);
#else
#pragma unroll 1
  for (int j = 0; j < np; ++j) {
    if (j >= 1) refill(j - 1);
    wait_full(j);
    stage_main(j, rdy);
    finish_stage(j, rdy, j + 1);
    compute(rdy);
    __syncwarp();  // every lane's reads precede the next staging
    epilogue(j);
  }
#endif
}

template <typename T, int MODE>
cudaError_t launch_warp_kernel(const CUtensorMap& ms, const CUtensorMap& ml, const CUtensorMap& mh,
                               const TmaParams& p, const float* w32, dim3 grid, cudaStream_t s) {
  using C = Cfg<T>;
  tma::Weights<K> wt = {};
  for (int r = 0; r < K * K; ++r)
    for (int x = 0; x < K; ++x) wt.w[r * tma::Weights<K>::KP + x] = w32[r * K + x];
  auto fn = filter_warp_kernel<T, MODE>;
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
  fn<<<grid, THREADS, C::SMEM, s>>>(ms, ml, mh, p, wt);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_warp_dtype(int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                              const CUtensorMap& mh, const TmaParams& p, const float* w32, dim3 grid,
                              cudaStream_t s) {
  switch (mode) {
    case VKT_WRAP: return launch_warp_kernel<T, VKT_WRAP>(ms, ml, mh, p, w32, grid, s);
    case VKT_MIRROR: return launch_warp_kernel<T, VKT_MIRROR>(ms, ml, mh, p, w32, grid, s);
    case VKT_CLAMP: return launch_warp_kernel<T, VKT_CLAMP>(ms, ml, mh, p, w32, grid, s);
    case VKT_BORDER: return launch_warp_kernel<T, VKT_BORDER>(ms, ml, mh, p, w32, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tmaw
}  // namespace vkt
