// filter_sep.cuh — ApplyFilter for separable (rank-1) kernels: three fused
// 1-D passes in one kernel.
//
// The reference's constructors build separable kernels: gaussian_kernel is
// g (x) g (x) g normalised (filters.py:45-58), box_kernel a constant cube
// (filters.py:61-66).  For a kernel whose weights factor as
// W[dz][dy][dx] = wz[dz] * wy[dy] * wx[dx] (checked on the host in float64,
// vkt_capi.cu), the correlation is
//   out = c + sum_dz wz[dz] * ( sum_dy wy[dy] * ( sum_dx wx[dx] * s ) )
// i.e. 3K FMAs per voxel instead of K^3: a 7^3 Gaussian drops from 343 to
// 21, and the filter becomes HBM-bound at every K instead of FP32-bound.
// Results are within the reference contract (ints within 1 LSB, f32 rtol
// 1e-5: each 1-D sum is K f32 FMAs) but not bit-identical to the dense
// kernels, whose (dz, dy, dx) sums round differently.
//
// Layout.  A CTA owns TX = 128 x outputs by TY rows and a chunk of ZC output
// planes, and streams the chunk's input planes (one TMA 3D box per plane,
// with its halo, into a raw ring) through two passes on split warp roles:
//  * PW producer warps wait for a plane's box, repair its out-of-volume cells
//    (edge tiles, Clamp / Mirror / Wrap, from a per-CTA table of (cell,
//    source) offsets; Border is TMA's zero fill, and a Border plane outside
//    the volume in z a fully out-of-bounds box), then run the x pass: widen
//    quads of raw cells into (x, x+64) float pairs (the paired layout of
//    filter_tma.cuh: one FFMA2 advances two outputs with one broadcast
//    weight) and write each row's K-tap x sums for 8 outputs (4 pairs) into a
//    ring of float-pair planes `xb` (TY + 2R rows x 64 pairs; 16-byte chunks
//    XOR-swizzled so the producers' STS.128 and the consumers' LDS.64 are
//    conflict-free).  Each producer warp releases the raw slot on an
//    mbarrier; the first one refills it a plane later.
//  * CW consumer warps each own one pair column of YPT rows: they read the
//    YPT + 2R x sums of their column (one LDS.64 each), form the YPT y sums
//    and fold them into K z accumulators per output -- the partial sums of
//    the K output planes this input plane reaches.  The plane loop is
//    unrolled by K and the accumulators rotate by NAME: at plane phase phi,
//    logical slot m lives in register (m + phi) % K, so every z tap is an
//    in-place FFMA2 (a rolled loop costs ~10% extra instructions in moves)
//    and the completed slot is read from register phi.  Completed outputs
//    are quantized (one saturating F2I) into a shared staging plane that one
//    TMA bulk tensor store writes out, clipped at the volume's faces.
//  * xb stages pass between the roles on named barriers (bar.arrive /
//    bar.sync: hardware blocking, where an mbarrier try_wait loop spent ~20%
//    of all issued instructions spinning).
//  * Face tiles (which repair cells every plane) run first in the last z
//    chunk (every chunk under Wrap): tma::edge_first.
// Measured (1024^3, profiles/r02_sep_rates_v14.txt): u16 7^3 Clamp 1.57 ms
// (dense tiled kernel 11.06), u8 3^3 0.89 ms (1.25), f32 7^3 1.86 ms (10.86);
// ncu (profiles/r02_ncu_sep_cfg3_final.txt): issue-bound at ~60% issue
// utilisation and ~60% of shared-memory bandwidth, the consumers waiting on
// the producers' x pass ~40% of their time.
// Non-finite f32 inputs: the dense kernels evaluate 0 * Inf = NaN exactly
// where the reference does; a factored sum may not (and padded anisotropic
// factors hold zeros).  Every stored output whose window holds an Inf or NaN
// is itself non-finite (Inf propagates through sums, 0 * Inf is NaN), so the
// f32 kernel folds each stored pair into x*0 + chk and raises p.nonfinite
// when chk ends NaN; the host then runs the direct kernel, guarded by that
// flag, which recomputes exactly the outputs left Inf / NaN (vkt_capi.cu).
// Integer voxels are finite.
#pragma once

#include "filter_ws.cuh"

namespace vkt {
namespace sep {

using tma::TmaParams;

constexpr int TX = tma::TX;
constexpr int HALF = tma::HALF;
constexpr int GPR = HALF / 4;  // x-pass items (4 output pairs) per row

// Per extent K: YPT consumer rows per thread, RG row groups of 2 consumer
// warps (64 pair columns each), PW producer warps, CTAs per SM; the
// consumers' K x YPT accumulator pairs fit 80 registers at 2 x 384 threads
// (72 at 2 x 448 for 3^3).
// Measured alternatives (1024^3): one producer item per thread with shapes
// (TY, YPT, PW) = (14, 7, 8) / (18, 3, 12) at 1-2 CTAs per SM, 6 producer
// warps, 5 x-sum stages, 6-8 raw stages, I2F.U16 widening, widening each raw
// cell once into a float stage (a second producer barrier per plane: 1.6x
// slower), direct predicated STG stores instead of the TMA store, branch-free
// (predicated) producer rounds: all equal or slower.  Producers that own
// whole planes (plane j on warp j % PW, no producer barrier; the x-sum
// stages must then be a multiple of PW so each stage's named barriers stay
// with one warp): u16 5^3 1.45 -> 1.32 ms and 9^3 2.44 -> 2.25 ms, but 7^3
// 1.66 -> 1.69, 3^3 0.93 -> 1.02, f32 slower; not adopted.  32-row tiles
// (8 row groups, 8 producer warps) at 1 CTA per SM: 7^3 1.66 -> 1.78 ms.
// y pass first (producers roll K-tap y sums down 2 pair columns x 8 rows,
// each cell widened once; consumers x + z from a 72-pair y-sum row): 7^3
// 1.85 ms, 5^3 1.58, 3^3 1.25, only 9^3 faster (2.17); not adopted.  8-pair
// x-pass items (14 widened pairs per 8 outputs instead of 2 x 10) with 6
// producer warps: 7^3 1.57 -> 1.59 ms, f32 7^3 1.86 -> 1.94; not adopted.  One
// TMA store per 2 output planes (half the consumers' store barriers): 7^3
// 1.576 -> 1.568 ms, f32 slower (the larger staging ring starves the raw ring).
template <int K, int BPC>
struct Shape {
  static constexpr int R = K / 2;
  // u8/u16 5^3: 5 rows (24 x-sum rows = 3 full producer rounds; 1.42 ->
  // 1.26-1.28 ms); f32 5^3 keeps 4 (its raw ring would drop to 3 stages)
  static constexpr int YPT = K == 3 ? 8 : K == 9 || K == 11 ? 3 : K >= 19 ? 1 : K >= 13 ? 2
                             : K == 5 && BPC < 4 ? 5 : 4;
  static constexpr int HQ = (R + 3) / 4;      // halo quads per side of an x-pass item
  static constexpr int RG = 4;
  // 6 producer warps where the x pass is long per consumer row: 3^3 (34 x-sum
  // rows for 32 outputs; u8 0.93 -> 0.89 ms) and 9^3 (20 rows for 12; u16
  // 2.44 -> 2.28 ms); 5^3 / 7^3 measured equal or slower
  static constexpr int PW = K == 3 || K == 9 || K == 13 || K == 15 || K >= 19 ? 6 : 4;
  static constexpr int CTAS = 2;
  static constexpr int CW = 2 * RG;
  static constexpr int THREADS = 32 * (CW + PW);
  static constexpr int TY = RG * YPT;
  static constexpr int BY = TY + 2 * R;       // raw / x-sum rows
  static constexpr int NQ = BY * GPR;         // x-pass items per plane
  static constexpr int PT = 32 * PW;          // producer threads
  static constexpr int QPT = (NQ + PT - 1) / PT;
};

// Extents the separable kernel is built for: odd K = 3 .. MAX_K (gaussian_kernel's
// default size reaches 11 at sigma 2.5, 13 at 3, 15 at 3.5, 17 at 4, 21 at 5)
constexpr int MAX_K = 21;
template <int BPC>
__host__ __device__ constexpr int tile_rows_b(int k) {
  return k == 3 ? Shape<3, BPC>::TY : k == 5 ? Shape<5, BPC>::TY : k == 7 ? Shape<7, BPC>::TY
       : k == 9 ? Shape<9, BPC>::TY : k == 11 ? Shape<11, BPC>::TY : k == 13 ? Shape<13, BPC>::TY
       : k == 15 ? Shape<15, BPC>::TY : k == 17 ? Shape<17, BPC>::TY : k == 19 ? Shape<19, BPC>::TY
       : Shape<21, BPC>::TY;
}
__host__ __device__ constexpr int tile_rows(int k, int bpc) { return bpc == 4 ? tile_rows_b<4>(k) : tile_rows_b<2>(k); }
__host__ __device__ constexpr int ctas_per_sm(int) { return 2; }

// Producer -> consumer handoff of the xb stages on named barriers (hardware
// blocking: an mbarrier try_wait loop cost ~20% of all issued instructions
// in the consumers' spins).  Barrier 1: the producers among themselves.
constexpr int NB_READY = 2;   // + stage: producers arrive, consumers sync
constexpr int NB_EMPTY = 8;   // + stage: consumers arrive, producers sync
constexpr int NB_STORE = 14;  // consumers: staging plane written, TMA store may go
__device__ __forceinline__ void nb_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <typename T, int K>
struct Cfg {
  using S = Shape<K, (int)sizeof(T)>;
  static constexpr int A = tma::box_align_left(S::R, (int)sizeof(T));
  static constexpr int BX = tma::box_width(S::R, (int)sizeof(T));
  static constexpr int RAW_BYTES = BX * S::BY * (int)sizeof(T);
  static constexpr int RAW_PITCH = (RAW_BYTES + 127) / 128 * 128;
  static constexpr int XB_BYTES = S::BY * HALF * 8;
  static constexpr int OUT_BYTES = S::TY * TX * (int)sizeof(T);  // one output staging plane
  static constexpr int SO = 3;  // output staging planes (TMA store ring)
  static constexpr int SMEM_PER_CTA = (228 * 1024) / S::CTAS - 1024;
  // repair table (edge tiles, Clamp / Mirror / Wrap): per out-of-volume cell
  // of the read window its box offset (u16) and source (box offset, or the
  // in-plane offset for Wrap), built once per CTA
  static constexpr int RT_MAX = 1536;
  static constexpr int RT_BYTES = RT_MAX * 6;
  static constexpr int fit(int sx) {
    return (SMEM_PER_CTA - 512 - RT_BYTES - sx * XB_BYTES - SO * OUT_BYTES) / RAW_PITCH;
  }
  // x-sum stages (named barriers NB_READY.., NB_EMPTY..): 3, or 2 where 3
  // would leave fewer than 4 raw TMA stages (u16 3^3: 34-row stages)
  static constexpr int SX = fit(3) >= 4 ? 3 : 2;
  static_assert(NB_READY + SX <= NB_EMPTY && NB_EMPTY + SX <= NB_STORE && NB_STORE < 16, "named barriers");
  static constexpr int FIT = fit(SX);
  static constexpr int S_RAW = FIT < 10 ? FIT : 10;
  static constexpr int SMEM = SX * XB_BYTES + SO * OUT_BYTES + S_RAW * RAW_PITCH + 2 * S_RAW * 8 + RT_BYTES + 128;
  static_assert(BX * S::BY <= 65536, "repair offsets are 16-bit");
  static_assert(S_RAW >= 4, "TMA ring too shallow");
  static_assert(SMEM <= SMEM_PER_CTA, "shared memory budget");
  static_assert(BX <= 256 && S::BY <= 256, "TMA box too large");
};

template <int K>
struct alignas(16) Factors {
  float wx[K], wy[K], wz[K];
};

// floor, saturated to the format's range: one F2I.U8/U16.FLOOR (PTX
// float-to-integer cvt clamps to the destination type)
template <typename T>
__device__ __forceinline__ T sat_floor(float v) {
  uint16_t d;
  if constexpr (sizeof(T) == 1)
    asm("cvt.rmi.u8.f32 %0, %1;" : "=h"(d) : "f"(v));
  else
    asm("cvt.rmi.u16.f32 %0, %1;" : "=h"(d) : "f"(v));
  return (T)d;
}

// Shared staging box -> global tile (bulk tensor store, clipped at the
// tensor's bounds); the caller commits the bulk group.
__device__ __forceinline__ void tma_store(const void* src, const CUtensorMap* map, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
      ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(tma::smem_u32(src)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// Physical 16-byte chunk of logical chunk ci (2 pairs) in an xb row: odd
// halves of each 16-chunk group swap neighbours, so the 8 lanes of a
// producer's STS.128 phase (chunks 2g, g = 0..7) hit 8 distinct bank groups.
__device__ __forceinline__ int xb_chunk(int ci) { return ci ^ ((ci >> 3) & 1); }

template <typename T, int K, int MODE>
__global__ void __launch_bounds__(Shape<K, (int)sizeof(T)>::THREADS, Shape<K, (int)sizeof(T)>::CTAS)
    filter_sep_kernel(const __grid_constant__ CUtensorMap map_src,
                      const __grid_constant__ CUtensorMap map_lo,
                      const __grid_constant__ CUtensorMap map_hi,
                      const __grid_constant__ CUtensorMap map_dst, const TmaParams p,
                      const __grid_constant__ Factors<K> f) {
  using C = Cfg<T, K>;
  using S = Shape<K, (int)sizeof(T)>;
  constexpr int R = S::R, YPT = S::YPT, TY = S::TY, BY = S::BY, SR = C::S_RAW, SX = C::SX;
  constexpr int PT = S::PT, CW = S::CW, PW = S::PW;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (tma::smem_u32(smem_raw) & 127u)) & 127u);
  T* raw_base = reinterpret_cast<T*>(smem);
  uint64_t* xb_base = reinterpret_cast<uint64_t*>(smem + SR * C::RAW_PITCH);
  T* out_base = reinterpret_cast<T*>(smem + SR * C::RAW_PITCH + SX * C::XB_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SR * C::RAW_PITCH + SX * C::XB_BYTES +
                                               C::SO * C::OUT_BYTES);
  uint64_t* rfree = full + SR;  // [SR] producer warps done reading a raw slot (PW arrivals)
  int32_t* rt_src = reinterpret_cast<int32_t*>(rfree + SR);        // [RT_MAX]
  uint16_t* rt_dst = reinterpret_cast<uint16_t*>(rt_src + C::RT_MAX);  // [RT_MAX]

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
    for (int s = 0; s < SR; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&rfree[s], PW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= CW) {
    // ---------------------------------------------------------------- producer
    const int pt = tid - 32 * CW;
    const bool leader = pt == 0;
    auto raw_slot = [&](int r) { return raw_base + r * (C::RAW_PITCH / (int)sizeof(T)); };
    auto issue = [&](int j, int r) {  // input plane j into raw slot r
      const tma::PlaneSrc s = tma::resolve<MODE>(p, R, zo0 - R + j);
      const CUtensorMap* m = s.which <= 0 ? &map_src : s.which == 1 ? &map_lo : &map_hi;
      tma::tma_issue_if(raw_slot(r), m, &full[r], C::RAW_BYTES, x0 - C::A, y0 - R,
                        s.which < 0 ? -1 : s.z, leader);
    };
    for (int j = 0; j < SR && j < np; ++j) issue(j, j);

    // out-of-volume cells of the read window (edge tiles; Clamp / Mirror / Wrap)
    const int ya = y0 - R;
    const int yb = min(y0 + TY, p.ny) + R;
    const int xb_end = min(x0 + TX, p.nx) + R;
    const bool edge = MODE != VKT_BORDER && (x0 - R < 0 || xb_end > p.nx || ya < 0 || yb > p.ny);
    const tmaws::EdgeCells ec(p.nx, p.ny, x0 - R, xb_end, ya, edge ? yb : ya);

    // out-of-volume cell q: its box offset d and its source, the box offset
    // of the mapped cell (Clamp / Mirror: in the box, the tile covers the
    // axis whenever the overshoot exceeds the extent) or its in-plane offset
    // (Wrap).  The full mapping: a volume thinner than the halo overshoots
    // by more than one extent.
    auto repair_cell = [&](int q, int& d, int64_t& sidx) {
      int gx, gy;
      ec.cell(p.nx, p.ny, q, gx, gy);
      const int mx = (int)map_index<MODE>(gx, p.nx), my = (int)map_index<MODE>(gy, p.ny);
      d = (gy - ya) * C::BX + gx - (x0 - C::A);
      sidx = MODE == VKT_WRAP ? (int64_t)my * p.pitch + mx : (int64_t)(my - ya) * C::BX + mx - (x0 - C::A);
      VKT_CHECK(d >= 0 && d < C::BX * BY, "sep repair: dest");
    };
    const bool table = edge && ec.total <= C::RT_MAX &&
                       (MODE != VKT_WRAP || (int64_t)p.ny * p.pitch < (int64_t)INT32_MAX);
    if (table) {
      for (int q = pt; q < ec.total; q += PT) {
        int d;
        int64_t sidx;
        repair_cell(q, d, sidx);
        rt_dst[q] = (uint16_t)d;
        rt_src[q] = (int32_t)sidx;  // < 2^31: checked in `table`
      }
      asm volatile("bar.sync 1, %0;" ::"r"(PT) : "memory");
    }

    // this thread's x-pass items: g fixed (pt & 15), rows pt/16 + (PT/16)*k
    const int g = pt & (GPR - 1);
    const int row0 = pt / GPR;
    const int b = (g >> 2) & 1;
    constexpr int HQ = S::HQ;
    const int src_off = row0 * C::BX + (C::A - 4 * HQ) + 4 * g;    // + k * (PT/GPR) * BX
    const int dst_off0 = row0 * HALF + 2 * ((2 * g) ^ b);       // in pairs, + k * (PT/GPR) * HALF
    const int dst_off1 = row0 * HALF + 2 * ((2 * g + 1) ^ b);
    const uint64_t zero2 = tma::f2pack(0.0f, 0.0f);

    int r = 0, s = 0, rp = 0;
    uint32_t rph = 0, rpph = 0;
#pragma unroll 1
    for (int j = 0; j < np; ++j) {
      T* raw = raw_slot(r);
      VKT_JITTER_POINT(4 * j);
      tma::mbar_wait(&full[r], rph);
      if constexpr (MODE != VKT_BORDER) {
        if (edge) {
          const tma::PlaneSrc src = tma::resolve<MODE>(p, R, zo0 - R + j);
          const T* plane = tma::plane_ptr<T>(p, src);
          if (table) {
            for (int q = pt; q < ec.total; q += PT) {
              const T v = MODE == VKT_WRAP ? __ldg(plane + rt_src[q]) : raw[rt_src[q]];
              raw[rt_dst[q]] = v;
            }
          } else {
            for (int q = pt; q < ec.total; q += PT) {
              int d;
              int64_t sidx;
              repair_cell(q, d, sidx);
              raw[d] = MODE == VKT_WRAP ? __ldg(plane + sidx) : raw[sidx];
            }
          }
          tma::fence_proxy_async();
          asm volatile("bar.sync 1, %0;" ::"r"(PT) : "memory");
        }
      }
      if (j >= SX) nb_sync(NB_EMPTY + s, S::THREADS);
      uint64_t* xb = xb_base + s * (C::XB_BYTES / 8);
#pragma unroll
      for (int k = 0; k < S::QPT; ++k) {
        if (S::NQ % PT != 0 && k == S::QPT - 1 && pt + PT * k >= S::NQ) break;
        // cells x0-4HQ+4g .. x0+4g+3+4HQ (and +HALF): output pair jj at tap
        // dx reads cell 4g + jj + dx - R, i.e. index jj + dx + 4HQ - R here
        const T* src = raw + src_off + k * (PT / GPR) * C::BX;
        uint64_t P[4 * (2 * HQ + 1)];
#pragma unroll
        for (int i = 0; i < 2 * HQ + 1; ++i) {
          uint32_t lo[4], hi[4];
          tma::load_quad<T>(src + 4 * i, lo);
          tma::load_quad<T>(src + 4 * i + HALF, hi);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (4 * i + e < 4 * HQ - R || 4 * i + e >= 4 * HQ + 4 + R) continue;
            if constexpr (sizeof(T) == 4)
              P[4 * i + e] = (uint64_t)lo[e] | ((uint64_t)hi[e] << 32);
            else
              P[4 * i + e] = tma::widen2(lo[e], hi[e]);
          }
        }
        uint64_t o[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          o[jj] = tma::ffma2_from(P[jj + 4 * HQ - R], f.wx[0], zero2);
#pragma unroll
          for (int dx = 1; dx < K; ++dx) tma::ffma2_bw(P[jj + dx + 4 * HQ - R], f.wx[dx], o[jj]);
        }
        uint64_t* d = xb + k * (PT / GPR) * HALF;
        *reinterpret_cast<uint4*>(d + dst_off0) =
            make_uint4((uint32_t)o[0], (uint32_t)(o[0] >> 32), (uint32_t)o[1], (uint32_t)(o[1] >> 32));
        *reinterpret_cast<uint4*>(d + dst_off1) =
            make_uint4((uint32_t)o[2], (uint32_t)(o[2] >> 32), (uint32_t)o[3], (uint32_t)(o[3] >> 32));
      }
      nb_arrive(NB_READY + s, S::THREADS);
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&rfree[r]);
      // The first producer refills the slot of plane j-1 once every producer
      // warp has read it (a plane late: by then the wait rarely blocks, and
      // no producer waits for the others).
      if (warp == CW && j >= 1 && j - 1 + SR < np) {
        tma::mbar_wait(&rfree[rp], rpph);
        issue(j - 1 + SR, rp);
      }
      rp = r;
      rpph = rph;
      if (++r == SR) r = 0, rph ^= 1u;
      if (++s == SX) s = 0;
    }
    // match the consumers' empty arrivals of the last planes (every named
    // barrier generation completes before the CTA exits)
    for (int j = np > SX ? np - SX : 0; j < np; ++j) nb_sync(NB_EMPTY + j % SX, S::THREADS);
    return;
  }

  // ---------------------------------------------------------------- consumer
  const int rg = warp >> 1;
  const int c = 32 * (warp & 1) + lane;
  const float a0 = acc_init<T>(p.c);
  const uint64_t a00 = tma::f2pack(a0, a0);
  const uint64_t zero2 = tma::f2pack(0.0f, 0.0f);
  uint64_t acc[YPT][K];
#pragma unroll
  for (int rr = 0; rr < YPT; ++rr)
#pragma unroll
    for (int m = 0; m < K; ++m) acc[rr][m] = a00;
  uint64_t chk = zero2;
  const int col_off = rg * YPT * HALF + 2 * xb_chunk(c >> 1) + (c & 1);
  // output staging: [TY][TX] cells per plane; one TMA store writes the tile
  // (clipped at the volume's faces) -- no per-cell bounds or 64-bit
  // addresses.  (Per-warp 32 x YPT boxes without the CTA barrier measured
  // slower: 1.92 vs 1.86 ms at 1024^3 u16 7^3.)
  const int stage_off = rg * YPT * TX + c;
  const bool issuer = tid == 0;
  int oq = 0;  // staging plane of the next output
  int s = 0;
#pragma unroll 1
  for (int jb = 0; jb < np; jb += K) {
#pragma unroll
    for (int phi = 0; phi < K; ++phi) {
      const int j = jb + phi;
      if (j >= np) break;
      VKT_JITTER_POINT(4 * j + 1);
      nb_sync(NB_READY + s, S::THREADS);
      const uint64_t* col = xb_base + s * (C::XB_BYTES / 8) + col_off;
      uint64_t ys[YPT];
#pragma unroll
      for (int i = 0; i < YPT + 2 * R; ++i) {
        const uint64_t v = col[i * HALF];
#pragma unroll
        for (int rr = 0; rr < YPT; ++rr) {
          const int dy = i - rr;
          if (dy < 0 || dy >= K) continue;
          if (dy == 0) ys[rr] = tma::ffma2_from(v, f.wy[0], zero2);
          else tma::ffma2_bw(v, f.wy[dy], ys[rr]);
        }
      }
      nb_arrive(NB_EMPTY + s, S::THREADS);
      if (++s == SX) s = 0;
      // logical slot m (the output plane this input plane reaches with
      // dz = K-1-m) lives in register (m + phi) % K
#pragma unroll
      for (int rr = 0; rr < YPT; ++rr) {
#pragma unroll
        for (int m = 0; m < K - 1; ++m) tma::ffma2_bw(ys[rr], f.wz[K - 1 - m], acc[rr][(m + phi) % K]);
        acc[rr][(K - 1 + phi) % K] = tma::ffma2_from(ys[rr], f.wz[0], a00);
      }
      VKT_JITTER_POINT(4 * j + 3);
      if (j >= 2 * R) {
        T* o = out_base + oq * (C::OUT_BYTES / (int)sizeof(T)) + stage_off;
#pragma unroll
        for (int rr = 0; rr < YPT; ++rr, o += TX) {
          const uint64_t v = acc[rr][phi];
          if constexpr (sizeof(T) == 4) {
            chk = tma::ffma2_from(v, 0.0f, chk);
            o[0] = tma::f2lo(v);
            o[HALF] = tma::f2hi(v);
          } else {
            o[0] = sat_floor<T>(tma::f2lo(v));
            o[HALF] = sat_floor<T>(tma::f2hi(v));
          }
        }
        tma::fence_proxy_async();
        nb_sync(NB_STORE, 32 * CW);
        if (issuer) {
          tma_store(out_base + oq * (C::OUT_BYTES / (int)sizeof(T)), &map_dst, x0, y0, zo0 + j - 2 * R);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          // the store of two planes ago has read its staging plane, which the
          // next output reuses (every consumer passes the next NB_STORE
          // barrier only after this wait)
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        if (++oq == C::SO) oq = 0;
      }
    }
  }
  if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if constexpr (sizeof(T) == 4) {
    if (p.nonfinite != nullptr && (isnan(tma::f2lo(chk)) || isnan(tma::f2hi(chk)))) *p.nonfinite = 1;
  }
}

template <typename T, int K, int MODE>
cudaError_t launch_sep_kernel(const CUtensorMap& ms, const CUtensorMap& ml, const CUtensorMap& mh,
                              const CUtensorMap& md, const TmaParams& p, const float* fx, const float* fy, const float* fz,
                              dim3 grid, cudaStream_t s) {
  using C = Cfg<T, K>;
  Factors<K> f;
  for (int i = 0; i < K; ++i) {
    f.wx[i] = fx[i];
    f.wy[i] = fy[i];
    f.wz[i] = fz[i];
  }
  auto fn = filter_sep_kernel<T, K, MODE>;
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
  fn<<<grid, Cfg<T, K>::S::THREADS, C::SMEM, s>>>(ms, ml, mh, md, p, f);
  return cudaGetLastError();
}

// odd K in [3, MAX_K] x the four address modes, for one voxel format
// (instantiated in filter_sep_{u8,u16,f32}.cu).
template <typename T>
cudaError_t launch_sep_dtype(int k, int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                             const CUtensorMap& mh, const CUtensorMap& md, const TmaParams& p, const float* fx,
                             const float* fy, const float* fz, dim3 grid, cudaStream_t s) {
#define VKT_SEP_CASES(KK)                                                                           \
  if (k == KK) switch (mode) {                                                                       \
      case VKT_WRAP: return launch_sep_kernel<T, KK, VKT_WRAP>(ms, ml, mh, md, p, fx, fy, fz, grid, s);     \
      case VKT_MIRROR: return launch_sep_kernel<T, KK, VKT_MIRROR>(ms, ml, mh, md, p, fx, fy, fz, grid, s); \
      case VKT_CLAMP: return launch_sep_kernel<T, KK, VKT_CLAMP>(ms, ml, mh, md, p, fx, fy, fz, grid, s);   \
      case VKT_BORDER: return launch_sep_kernel<T, KK, VKT_BORDER>(ms, ml, mh, md, p, fx, fy, fz, grid, s); \
      default: return cudaErrorInvalidValue;                                                         \
    }
  if constexpr (sizeof(T) != 4) {  // f32 3^3 runs the dense kernel (vkt_capi.cu)
    VKT_SEP_CASES(3)
  }
  VKT_SEP_CASES(5)
  VKT_SEP_CASES(7)
  VKT_SEP_CASES(9)
  VKT_SEP_CASES(11)
  VKT_SEP_CASES(13)
  VKT_SEP_CASES(15)
  VKT_SEP_CASES(17)
  VKT_SEP_CASES(19)
  VKT_SEP_CASES(21)
#undef VKT_SEP_CASES
  return cudaErrorInvalidValue;
}

}  // namespace sep
}  // namespace vkt
