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
// with its halo, into a raw ring) through two passes, on split warp roles
// (as filter_ws.cuh) that meet only on mbarriers:
//  * PW producer warps wait for a plane's box, repair its out-of-volume cells
//    (edge tiles, Clamp / Mirror / Wrap; Border is TMA's zero fill, and a
//    Border plane outside the volume in z a fully out-of-bounds box), then
//    run the x pass: widen quads of raw cells into (x, x+64) float pairs (the
//    paired layout of filter_tma.cuh: one FFMA2 advances two outputs with one
//    broadcast weight) and write each row's K-tap x sums for 8 outputs
//    (4 pairs) into a ring of float-pair planes `xb` (TY + 2R rows x 64
//    pairs; 16-byte chunks XOR-swizzled so the producers' STS.128 and the
//    consumers' LDS.64 are conflict-free).  The first producer refills the
//    raw slot once every producer has read it (named barrier).
//  * CW consumer warps each own one pair column of YPT rows: they read the
//    YPT + 2R x sums of their column (one LDS.64 each), form the YPT y sums
//    and fold them into K z accumulators per output -- the partial sums of
//    the K output planes this input plane reaches.  The plane loop is
//    unrolled by K and the accumulators rotate by NAME: at plane phase phi,
//    logical slot m lives in register (m + phi) % K, so every z tap is an
//    in-place FFMA2 (no register moves; a rolled loop costs ~10% extra
//    instructions in moves) and the completed slot is stored from register
//    phi.
// Non-finite f32 inputs: the dense kernels evaluate 0 * Inf = NaN exactly
// where the reference does; a factored sum may not (and padded anisotropic
// factors hold zeros).  Every stored output whose window holds an Inf or NaN
// is itself non-finite (Inf propagates through sums, 0 * Inf is NaN), so the
// f32 kernel folds each stored pair into x*0 + chk and raises p.nonfinite
// when chk ends NaN; the host then runs the direct kernel, guarded by that
// flag, over the same outputs (vkt_capi.cu).  Integer voxels are finite.
#pragma once

#include "filter_ws.cuh"

namespace vkt {
namespace sep {

using tma::TmaParams;

constexpr int TX = tma::TX;
constexpr int HALF = tma::HALF;
constexpr int CW = 8;                   // consumer warps: 4 row groups x 64 pair columns
constexpr int PW = 4;                   // producer warps
constexpr int THREADS = 32 * (CW + PW);
constexpr int CTAS_PER_SM = 2;
constexpr int GPR = HALF / 4;  // x-pass items (4 output pairs) per row

template <int K>
struct Shape {
  static constexpr int R = K / 2;
  static constexpr int YPT = K == 3 ? 8 : K == 9 ? 3 : 4;  // consumer rows per thread
  static constexpr int TY = (CW / 2) * YPT;   // 2 consumer warps (64 pair columns) per row group
  static constexpr int BY = TY + 2 * R;       // raw / x-sum rows
  static constexpr int NQ = BY * GPR;         // x-pass items per plane
  static constexpr int PT = 32 * PW;          // producer threads
  static constexpr int QPT = (NQ + PT - 1) / PT;
};

__host__ __device__ constexpr int tile_rows(int k) { return (CW / 2) * (k == 3 ? 8 : k == 9 ? 3 : 4); }

template <typename T, int K>
struct Cfg {
  using S = Shape<K>;
  static constexpr int A = tma::box_align_left(S::R, (int)sizeof(T));
  static constexpr int BX = tma::box_width(S::R, (int)sizeof(T));
  static constexpr int RAW_BYTES = BX * S::BY * (int)sizeof(T);
  static constexpr int RAW_PITCH = (RAW_BYTES + 127) / 128 * 128;
  static constexpr int XB_BYTES = S::BY * HALF * 8;
  static constexpr int SX = 3;  // x-sum stages
  static constexpr int SMEM_PER_CTA = (228 * 1024) / CTAS_PER_SM - 1024;
  static constexpr int FIT = (SMEM_PER_CTA - 512 - SX * XB_BYTES) / RAW_PITCH;
  static constexpr int S_RAW = FIT < 8 ? FIT : 8;
  static constexpr int SMEM = SX * XB_BYTES + S_RAW * RAW_PITCH + (S_RAW + 2 * SX) * 8 + 128;
  static_assert(S_RAW >= 4, "TMA ring too shallow");
  static_assert(SMEM <= SMEM_PER_CTA, "shared memory budget");
  static_assert(BX <= 256 && S::BY <= 256, "TMA box too large");
};

template <int K>
struct alignas(16) Factors {
  float wx[K], wy[K], wz[K];
};

__device__ __forceinline__ void st_cs(uint8_t* p, uint32_t v) {
  asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cs(uint16_t* p, uint32_t v) {
  asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cs(float* p, float v) { __stcs(p, v); }

// floor, saturated to the format's range (cvt.pack.sat: operand b lands in
// the low lane)
template <typename T>
__device__ __forceinline__ uint32_t sat_floor(float v) {
  const int n = tma::floor_s32(v);
  uint32_t d;
  if constexpr (sizeof(T) == 1)
    asm("cvt.pack.sat.u8.s32.b32 %0, 0, %1, 0;" : "=r"(d) : "r"(n));
  else
    asm("cvt.pack.sat.u16.s32 %0, 0, %1;" : "=r"(d) : "r"(n));
  return d;
}

// Physical 16-byte chunk of logical chunk ci (2 pairs) in an xb row: odd
// halves of each 16-chunk group swap neighbours, so the 8 lanes of a
// producer's STS.128 phase (chunks 2g, g = 0..7) hit 8 distinct bank groups.
__device__ __forceinline__ int xb_chunk(int ci) { return ci ^ ((ci >> 3) & 1); }

template <typename T, int K, int MODE>
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM)
    filter_sep_kernel(const __grid_constant__ CUtensorMap map_src,
                      const __grid_constant__ CUtensorMap map_lo,
                      const __grid_constant__ CUtensorMap map_hi, const TmaParams p,
                      const __grid_constant__ Factors<K> f) {
  using C = Cfg<T, K>;
  using S = Shape<K>;
  constexpr int R = S::R, YPT = S::YPT, TY = S::TY, BY = S::BY, SR = C::S_RAW, SX = C::SX;
  constexpr int PT = S::PT;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (tma::smem_u32(smem_raw) & 127u)) & 127u);
  T* raw_base = reinterpret_cast<T*>(smem);
  uint64_t* xb_base = reinterpret_cast<uint64_t*>(smem + SR * C::RAW_PITCH);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SR * C::RAW_PITCH + SX * C::XB_BYTES);
  uint64_t* ready = full + SR;  // [SX] producers done writing (PW arrivals)
  uint64_t* empty = ready + SX; // [SX] consumers done reading (CW arrivals)

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int x0 = blockIdx.x * TX;
  const int y0 = blockIdx.y * TY;
  const int zo0 = p.z_begin + blockIdx.z * p.zc;
  const int nzo = min(p.zc, p.z_end - zo0);
  if (nzo <= 0) return;
  const int np = nzo + 2 * R;

  if (tid == 0) {
    tma::prefetch_tmap(&map_src);
    for (int s = 0; s < SR; ++s) tma::mbar_init(&full[s], 1);
    for (int s = 0; s < SX; ++s) {
      tma::mbar_init(&ready[s], PW);
      tma::mbar_init(&empty[s], CW);
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

    // this thread's x-pass items: g fixed (pt & 15), rows pt/16 + (PT/16)*k
    const int g = pt & (GPR - 1);
    const int row0 = pt / GPR;
    const int b = (g >> 2) & 1;
    const int src_off = row0 * C::BX + (C::A - 4) + 4 * g;    // + k * (PT/GPR) * BX
    const int dst_off0 = row0 * HALF + 2 * ((2 * g) ^ b);       // in pairs, + k * (PT/GPR) * HALF
    const int dst_off1 = row0 * HALF + 2 * ((2 * g + 1) ^ b);
    const uint64_t zero2 = tma::f2pack(0.0f, 0.0f);

    int r = 0, s = 0;
    uint32_t rph = 0, sph = 0;
#pragma unroll 1
    for (int j = 0; j < np; ++j) {
      T* raw = raw_slot(r);
      VKT_JITTER_POINT(4 * j);
      tma::mbar_wait(&full[r], rph);
      if constexpr (MODE != VKT_BORDER) {
        if (edge) {
          const tma::PlaneSrc src = tma::resolve<MODE>(p, R, zo0 - R + j);
          for (int q = pt; q < ec.total; q += PT) {
            int gx, gy;
            ec.cell(p.nx, p.ny, q, gx, gy);
            // the full mapping: a volume thinner than the halo overshoots by
            // more than one extent (the mapped cell is still in the box: the
            // tile then covers the whole axis)
            const int mx = (int)map_index<MODE>(gx, p.nx), my = (int)map_index<MODE>(gy, p.ny);
            T v;
            if constexpr (MODE == VKT_WRAP)
              v = __ldg(tma::plane_ptr<T>(p, src) + (int64_t)my * p.pitch + mx);
            else
              v = raw[(my - ya) * C::BX + mx - (x0 - C::A)];
            const int d = (gy - ya) * C::BX + gx - (x0 - C::A);
            VKT_CHECK(d >= 0 && d < C::BX * BY, "sep repair: dest");
            raw[d] = v;
          }
          tma::fence_proxy_async();
          asm volatile("bar.sync 1, %0;" ::"r"(PT) : "memory");
        }
      }
      if (j >= SX) tma::mbar_wait(&empty[s], sph ^ 1u);
      uint64_t* xb = xb_base + s * (C::XB_BYTES / 8);
#pragma unroll
      for (int k = 0; k < S::QPT; ++k) {
        if (S::NQ % PT != 0 && k == S::QPT - 1 && pt + PT * k >= S::NQ) break;
        // cells x0-4+4g .. x0+4g+7 (and +HALF): output pair jj at tap dx
        // reads cell 4g + jj + dx - R, i.e. index jj + dx + 4 - R here
        const T* src = raw + src_off + k * (PT / GPR) * C::BX;
        uint64_t P[12];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          uint32_t lo[4], hi[4];
          tma::load_quad<T>(src + 4 * i, lo);
          tma::load_quad<T>(src + 4 * i + HALF, hi);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (4 * i + e < 4 - R || 4 * i + e >= 8 + R) continue;
            if constexpr (sizeof(T) == 4)
              P[4 * i + e] = (uint64_t)lo[e] | ((uint64_t)hi[e] << 32);
            else
              P[4 * i + e] = tma::widen2(lo[e], hi[e]);
          }
        }
        uint64_t o[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          o[jj] = tma::ffma2_from(P[jj + 4 - R], f.wx[0], zero2);
#pragma unroll
          for (int dx = 1; dx < K; ++dx) tma::ffma2_bw(P[jj + dx + 4 - R], f.wx[dx], o[jj]);
        }
        uint64_t* d = xb + k * (PT / GPR) * HALF;
        *reinterpret_cast<uint4*>(d + dst_off0) =
            make_uint4((uint32_t)o[0], (uint32_t)(o[0] >> 32), (uint32_t)o[1], (uint32_t)(o[1] >> 32));
        *reinterpret_cast<uint4*>(d + dst_off1) =
            make_uint4((uint32_t)o[2], (uint32_t)(o[2] >> 32), (uint32_t)o[3], (uint32_t)(o[3] >> 32));
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&ready[s]);
      // every producer has read raw slot r: the first one refills it
      asm volatile("bar.sync 1, %0;" ::"r"(PT) : "memory");
      if (j + SR < np) issue(j + SR, r);
      if (++r == SR) r = 0, rph ^= 1u;
      if (++s == SX) s = 0, sph ^= 1u;
    }
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
  const int ox = x0 + c;
  const int oy = y0 + rg * YPT;
  const bool st_lo = ox < p.nx, st_hi = ox + HALF < p.nx;
  const int rows_ok = min(YPT, p.ny - oy);
  const int64_t plane_elems = (int64_t)p.pitch * p.ny;
  T* out_plane = static_cast<T*>(p.dst) + (int64_t)oy * p.pitch + ox + (int64_t)zo0 * plane_elems;
  const int col_off = rg * YPT * HALF + 2 * xb_chunk(c >> 1) + (c & 1);

  int s = 0;
  uint32_t sph = 0;
#pragma unroll 1
  for (int jb = 0; jb < np; jb += K) {
#pragma unroll
    for (int phi = 0; phi < K; ++phi) {
      const int j = jb + phi;
      if (j >= np) break;
      VKT_JITTER_POINT(4 * j + 1);
      tma::mbar_wait(&ready[s], sph);
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
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[s]);
      if (++s == SX) s = 0, sph ^= 1u;
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
        T* o = out_plane;
#pragma unroll
        for (int rr = 0; rr < YPT; ++rr, o += p.pitch) {
          if (rr >= rows_ok) continue;
          const uint64_t v = acc[rr][phi];
          if constexpr (sizeof(T) == 4) {
            chk = tma::ffma2_from(v, 0.0f, chk);
            if (st_lo) st_cs(o, tma::f2lo(v));
            if (st_hi) st_cs(o + HALF, tma::f2hi(v));
          } else {
            if (st_lo) st_cs(o, sat_floor<T>(tma::f2lo(v)));
            if (st_hi) st_cs(o + HALF, sat_floor<T>(tma::f2hi(v)));
          }
        }
        out_plane += plane_elems;
      }
    }
  }
  if constexpr (sizeof(T) == 4) {
    if (p.nonfinite != nullptr && (isnan(tma::f2lo(chk)) || isnan(tma::f2hi(chk)))) *p.nonfinite = 1;
  }
}

template <typename T, int K, int MODE>
cudaError_t launch_sep_kernel(const CUtensorMap& ms, const CUtensorMap& ml, const CUtensorMap& mh,
                              const TmaParams& p, const float* fx, const float* fy, const float* fz,
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
  fn<<<grid, THREADS, C::SMEM, s>>>(ms, ml, mh, p, f);
  return cudaGetLastError();
}

// K in {3, 5, 7, 9} x the four address modes, for one voxel format
// (instantiated in filter_sep_{u8,u16,f32}.cu).
template <typename T>
cudaError_t launch_sep_dtype(int k, int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                             const CUtensorMap& mh, const TmaParams& p, const float* fx,
                             const float* fy, const float* fz, dim3 grid, cudaStream_t s) {
#define VKT_SEP_CASES(KK)                                                                           \
  if (k == KK) switch (mode) {                                                                       \
      case VKT_WRAP: return launch_sep_kernel<T, KK, VKT_WRAP>(ms, ml, mh, p, fx, fy, fz, grid, s);     \
      case VKT_MIRROR: return launch_sep_kernel<T, KK, VKT_MIRROR>(ms, ml, mh, p, fx, fy, fz, grid, s); \
      case VKT_CLAMP: return launch_sep_kernel<T, KK, VKT_CLAMP>(ms, ml, mh, p, fx, fy, fz, grid, s);   \
      case VKT_BORDER: return launch_sep_kernel<T, KK, VKT_BORDER>(ms, ml, mh, p, fx, fy, fz, grid, s); \
      default: return cudaErrorInvalidValue;                                                         \
    }
  if constexpr (sizeof(T) != 4) {  // f32 3^3 runs the dense kernel (vkt_capi.cu)
    VKT_SEP_CASES(3)
  }
  VKT_SEP_CASES(5)
  VKT_SEP_CASES(7)
  VKT_SEP_CASES(9)
#undef VKT_SEP_CASES
  return cudaErrorInvalidValue;
}

}  // namespace sep
}  // namespace vkt
