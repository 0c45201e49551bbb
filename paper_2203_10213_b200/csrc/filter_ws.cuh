// filter_ws.cuh — u8/u16 3x3x3 ApplyFilter, warp-specialized (producer /
// consumer warps).
//
// The integer 3^3 filter is FMA-bound (27 FMAs for 2-4 bytes per voxel) but
// has only 27/64 FFMA2 per voxel, so per-plane fixed costs decide its speed.
// On the paired-layout kernel (filter_tma.cuh) -- 16 outputs per thread,
// every warp staging and computing, CTA-wide ready/empty rounds, register
// rolls, an F2I + VIMNMX + PRMT epilogue -- it ran at 0.50 of the FP32
// roofline (profiles/r02_ncu_u8k3_v40.txt).  A warp-private-staging step
// (each warp widening its own rows, 32 outputs per thread) reached 0.59; with
// 3 warps per SM sub-partition each interleaving staging, math and epilogue,
// the latencies still left the FMA pipe ~30% idle.  Here the roles split:
//  * 3 producer warps per CTA wait for each plane's TMA box, widen the whole
//    tile window (34 rows) into a CTA-wide float ready ring (the paired,
//    swizzled layout of filter_tma.cuh), patch the out-of-volume cells of
//    edge tiles, and release the stage (ready mbarrier); the first producer's
//    lane 0 also re-issues the TMA once every producer has read a raw slot (a
//    named barrier among the producers).  A Border plane outside the volume
//    in z is fetched as a fully out-of-bounds box, which TMA delivers as zeros.
//  * 4 consumer warps per CTA only load ready rows, run the FFMA2 stream
//    (32 outputs per thread: 4 rows x 4 output pairs), release the stage
//    (empty mbarrier) and store.  Their accumulators roll inside the first
//    FMAs of each plane, and the epilogue is F2I + I2IP.
// 2 CTAs per SM: per SM sub-partition 2 consumer warps and 1.5 producer
// warps, so one warp's epilogue or barrier wait overlaps another's FFMA2
// stream.  Measured (1024^3 u8 / u16 3^3 Clamp): 1.269 / 1.290 ms, against
// 1.316 / 1.356 for the warp-private kernel, 1.287 / 1.312 with 2 producer
// warps and 1.279 / 1.305 with a 4-deep ready ring; u8 Wrap 1.363 vs 1.599.
// No ramp guards: the 2R extra planes of a chunk also feed the accumulators
// of output planes outside the chunk, which are never stored (integer inputs
// are finite).
// Tap order per output is (dz, dy, dx) as everywhere else (filters.py:89-92),
// so results are bit-identical to the other kernels.
#pragma once

#include <atomic>

#include "filter_tma.cuh"

namespace vkt {
namespace tmaws {

using tma::TmaParams;

constexpr int K = 3;
constexpr int R = 1;
constexpr int TX = tma::TX;
constexpr int HALF = tma::HALF;
constexpr int XQ = tma::XQ;
constexpr int TPR = tma::TPR;
constexpr int YPT = 4;                   // output rows per consumer thread
constexpr int CW = 4;                    // consumer warps per CTA
constexpr int PW = 3;                    // producer warps per CTA
constexpr int THREADS = 32 * (CW + PW);
constexpr int WROWS = 2 * YPT;           // output rows per consumer warp
constexpr int TY = CW * WROWS;           // 32 output rows per CTA
constexpr int CTAS_PER_SM = 2;
constexpr int BY = TY + 2 * R;           // ready / raw rows
constexpr int NPR = tma::NPR;
constexpr int RPF = tma::Ready<K>::RPF;
constexpr int GPR = NPR / 4;
constexpr int NQ = GPR * BY;             // staging items per plane
constexpr int PT = 32 * PW;              // producer threads
constexpr int QPT = (NQ + PT - 1) / PT;  // items per producer thread

// Out-of-volume cells of a CTA's read window [xa, xb) x [ya, yb): rows above
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

// Physical float offset, in a ready stage whose row 0 is global row ya,
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

template <typename T>
struct Cfg {
  static constexpr int A = tma::box_align_left(R, (int)sizeof(T));
  static constexpr int BX = tma::box_width(R, (int)sizeof(T));
  static constexpr int RAW_BYTES = BX * BY * (int)sizeof(T);
  static constexpr int RAW_PITCH = (RAW_BYTES + 127) / 128 * 128;
  static constexpr int RDY_BYTES = RPF * BY * 4;
  static constexpr int RDY_PITCH = (RDY_BYTES + 127) / 128 * 128;
  static constexpr int SMEM_PER_CTA = (228 * 1024) / CTAS_PER_SM - 1024;
  static constexpr int S_RDY = 3;
  static constexpr int RAW_FIT = (SMEM_PER_CTA - 512 - S_RDY * RDY_PITCH) / RAW_PITCH;
  static constexpr int S_RAW = RAW_FIT < 8 ? RAW_FIT : 8;
  static constexpr int SMEM = S_RDY * RDY_PITCH + S_RAW * RAW_PITCH + (2 * S_RDY + S_RAW) * 8 + 128;
  static_assert(S_RAW >= 3, "TMA ring too shallow");
  static_assert(SMEM <= SMEM_PER_CTA, "shared memory budget");
};

template <typename T, int MODE>
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM)
    filter_ws_kernel(const __grid_constant__ CUtensorMap map_src,
                     const __grid_constant__ CUtensorMap map_lo,
                     const __grid_constant__ CUtensorMap map_hi, const TmaParams p,
                     const __grid_constant__ tma::Weights<K> wt) {
  using C = Cfg<T>;
  constexpr int S = C::S_RDY;
  constexpr int SR = C::S_RAW;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (tma::smem_u32(smem_raw) & 127u)) & 127u);
  T* raw_base = reinterpret_cast<T*>(smem);
  float* rdy_base = reinterpret_cast<float*>(smem + SR * C::RAW_PITCH);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SR * C::RAW_PITCH + S * C::RDY_PITCH);
  uint64_t* ready = full + SR;   // [S] producers done staging (PW arrivals)
  uint64_t* empty = ready + S;   // [S] consumers done reading (CW arrivals)

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  if constexpr (MODE != VKT_BORDER) tma::edge_first<MODE>(bx, by, bz);
  const int x0 = bx * TX;
  const int y0 = by * TY;
  const int zo0 = p.z_begin + bz * p.zc;
  const int nzo = min(p.zc, p.z_end - zo0);
  if (nzo <= 0) return;
  const int np = nzo + 2 * R;

  if (tid == 0) {
    tma::prefetch_tmap(&map_src);
    for (int s = 0; s < SR; ++s) tma::mbar_init(&full[s], 1);
    for (int s = 0; s < S; ++s) {
      tma::mbar_init(&ready[s], PW);
      tma::mbar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= CW) {
    // ---------------------------------------------------------------- producer
    const int pt = tid - 32 * CW;  // 0 .. PT-1
    const bool leader = pt == 0;
    auto issue = [&](int j, int r) {  // plane j into raw slot r
      const tma::PlaneSrc s = tma::resolve<MODE>(p, R, zo0 - R + j);
      // a Border plane outside the volume: a fully out-of-bounds box (zeros)
      const CUtensorMap* m = s.which <= 0 ? &map_src : s.which == 1 ? &map_lo : &map_hi;
      tma::tma_issue_if(raw_base + r * (C::RAW_PITCH / (int)sizeof(T)), m, &full[r], C::RAW_BYTES,
                        x0 - C::A, y0 - R, s.which < 0 ? -1 : s.z, leader);
    };
    for (int j = 0; j < SR && j < np; ++j) issue(j, j);

    int item_ro[QPT], item_wo[QPT];
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
      const int q = pt + PT * k;
      const int row = q / GPR, g = q - row * GPR;
      item_ro[k] = row * RPF + tma::Ready<K>::in_row(8 * g);
      item_wo[k] = row * C::BX + 4 * g + (C::A - 4);
    }
    const bool last_item = pt + PT * (QPT - 1) < NQ;
    // out-of-volume cells of the CTA's read window (edge tiles only)
    const int ya = y0 - R;
    const int yb = min(y0 + TY, p.ny) + R;
    const int xb = min(x0 + TX, p.nx) + R;
    const bool edge = x0 - R < 0 || xb > p.nx || ya < 0 || yb > p.ny;
    const EdgeCells ec(p.nx, p.ny, x0 - R, xb, ya, edge ? yb : ya);

    // ring slots and phase parities as counters (no integer division per plane)
    int r = 0, s = 0;
    uint32_t rph = 0, sph = 0;
#pragma unroll 1
    for (int j = 0; j < np; ++j) {
      float* stage = rdy_base + s * (C::RDY_PITCH / 4);
      VKT_JITTER_POINT(4 * j);
      tma::mbar_wait(&full[r], rph);
      if (j >= S) tma::mbar_wait(&empty[s], sph ^ 1u);
      const T* raw = raw_base + r * (C::RAW_PITCH / (int)sizeof(T));
#pragma unroll
      for (int k = 0; k < QPT; ++k) {
        if (PT * k + PT - 1 >= NQ && !last_item) continue;
        const int ro = item_ro[k], wo = item_wo[k];
        VKT_CHECK(ro >= 0 && tma::Ready<K>::second(ro) + 4 <= RPF * BY, "ws staging: ready offset");
        VKT_CHECK(wo >= 0 && (wo + HALF + 4) * (int)sizeof(T) <= C::RAW_BYTES, "ws staging: raw offset");
        uint32_t lo[4], hi[4];
        tma::load_quad<T>(raw + wo, lo);
        tma::load_quad<T>(raw + wo + HALF, hi);
        uint64_t pr[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) pr[c] = tma::widen2(lo[c], hi[c]);
        *reinterpret_cast<uint4*>(stage + ro) = make_uint4((uint32_t)pr[0], (uint32_t)(pr[0] >> 32),
                                                           (uint32_t)pr[1], (uint32_t)(pr[1] >> 32));
        *reinterpret_cast<uint4*>(stage + tma::Ready<K>::second(ro)) =
            make_uint4((uint32_t)pr[2], (uint32_t)(pr[2] >> 32), (uint32_t)pr[3],
                       (uint32_t)(pr[3] >> 32));
      }
      // every producer warp has read raw slot r: the first one refills it
      asm volatile("bar.sync 1, %0;" ::"r"(PT) : "memory");
      if (warp == CW && j + SR < np) issue(j + SR, r);
      if constexpr (MODE != VKT_BORDER) {
        if (edge) {
          const tma::PlaneSrc src = tma::resolve<MODE>(p, R, zo0 - R + j);
          for (int q = pt; q < ec.total; q += PT) {
            int gx, gy;
            ec.cell(p.nx, p.ny, q, gx, gy);
            float v;
            if constexpr (MODE == VKT_WRAP) {
              v = tma::widen(__ldg(tma::plane_ptr<T>(p, src) +
                                   (int64_t)map_index_near<VKT_WRAP>(gy, p.ny) * p.pitch +
                                   map_index_near<VKT_WRAP>(gx, p.nx)));
            } else {
              int slo, shi;
              rdy_dests(x0, ya, map_index_near<MODE>(gx, p.nx), map_index_near<MODE>(gy, p.ny),
                              slo, shi);
              v = stage[slo >= 0 ? slo : shi];
            }
            int dlo, dhi;
            rdy_dests(x0, ya, gx, gy, dlo, dhi);
            VKT_CHECK(dlo < RPF * BY && dhi < RPF * BY && (dlo >= 0 || dhi >= 0), "ws edge fix: dest");
            if (dlo >= 0) stage[dlo] = v;
            if (dhi >= 0) stage[dhi] = v;
          }
          asm volatile("bar.sync 1, %0;" ::"r"(PT) : "memory");
        }
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&ready[s]);
      if (++r == SR) r = 0, rph ^= 1u;
      if (++s == S) s = 0, sph ^= 1u;
    }
    return;
  }

  // ---------------------------------------------------------------- consumer
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
  T* out_plane = static_cast<T*>(p.dst) + (int64_t)oy * p.pitch + ox + (int64_t)zo0 * plane_elems;
  const int rows_ok = min(YPT, p.ny - oy);

  int s = 0;
  uint32_t sph = 0;
#pragma unroll 1
  for (int i = 0; i < np; ++i) {
    const float* stage = rdy_base + s * (C::RDY_PITCH / 4);
    VKT_JITTER_POINT(4 * i + 1);
    tma::mbar_wait(&ready[s], sph);
    const float* base = stage + (warp * WROWS + ty * YPT) * RPF;
#pragma unroll
    for (int ry = 0; ry < YPT + K - 1; ++ry) {
      uint64_t P[2 * tma::LoadRun<K>::NLD];
      const float* row = base + ry * RPF;
#pragma unroll
      for (int q = 0; q < tma::LoadRun<K>::NLD; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(row + ld_off[q]);
        P[2 * q] = tma::f2pack(v.x, v.y);
        P[2 * q + 1] = tma::f2pack(v.z, v.w);
      }
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
#pragma unroll
        for (int m = 0; m < K; ++m) {
#pragma unroll
          for (int rr = 0; rr < YPT; ++rr) {
            const int dy = ry - rr;
            if (dy < 0 || dy >= K) continue;
            const float w = wt.w[((K - 1 - m) * K + dy) * tma::Weights<K>::KP + dx];
#pragma unroll
            for (int jj = 0; jj < XQ; ++jj) {
              const uint64_t x = P[jj + dx + tma::LoadRun<K>::SH];
              if (dy == 0 && dx == 0)
                acc[rr][m][jj] =
                    tma::ffma2_from(x, w, m + 1 < K ? acc[rr][m + 1 < K ? m + 1 : m][jj] : a00);
              else
                tma::ffma2_bw(x, w, acc[rr][m][jj]);
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&empty[s]);
    if (++s == S) s = 0, sph ^= 1u;
    VKT_JITTER_POINT(4 * i + 3);
    if (i >= 2 * R) {
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
    }
  }
}

template <typename T, int MODE>
cudaError_t launch_ws_kernel(const CUtensorMap& ms, const CUtensorMap& ml, const CUtensorMap& mh,
                             const TmaParams& p, const float* w32, dim3 grid, cudaStream_t s) {
  using C = Cfg<T>;
  tma::Weights<K> wt = {};
  for (int r = 0; r < K * K; ++r)
    for (int x = 0; x < K; ++x) wt.w[r * tma::Weights<K>::KP + x] = w32[r * K + x];
  auto fn = filter_ws_kernel<T, MODE>;
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
cudaError_t launch_ws_dtype(int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                            const CUtensorMap& mh, const TmaParams& p, const float* w32, dim3 grid,
                            cudaStream_t s) {
  switch (mode) {
    case VKT_WRAP: return launch_ws_kernel<T, VKT_WRAP>(ms, ml, mh, p, w32, grid, s);
    case VKT_MIRROR: return launch_ws_kernel<T, VKT_MIRROR>(ms, ml, mh, p, w32, grid, s);
    case VKT_CLAMP: return launch_ws_kernel<T, VKT_CLAMP>(ms, ml, mh, p, w32, grid, s);
    case VKT_BORDER: return launch_ws_kernel<T, VKT_BORDER>(ms, ml, mh, p, w32, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tmaws
}  // namespace vkt
