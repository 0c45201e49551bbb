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
// planes, and streams the chunk's input planes (TMA 3D box per plane, with
// its halo, into a raw ring) through two passes per plane:
//  * x pass: every thread widens quads of raw cells into (x, x+64) float
//    pairs (the paired layout of filter_tma.cuh: one FFMA2 advances two
//    outputs with one broadcast weight) and writes the row's K-tap x sums for
//    8 outputs (4 pairs) into a double-buffered float-pair plane `xb`
//    (TY + 2R rows x 64 pairs);
//  * y + z pass: each thread owns one pair column of YPT rows: it reads the
//    YPT + 2R x sums of its column from xb (one LDS.64 each), forms the YPT
//    y sums, and folds them into K rolling z accumulators per output (the
//    partial sums of the K output planes this input plane reaches).  The
//    roll happens inside the FMAs: slot m takes slot m+1's sum plus this
//    plane's tap (tma::ffma2_from), so there is no register move.
// One CTA barrier per plane: iteration j runs the x pass of plane j, the
// y + z pass of plane j-1 (the other xb buffer), and repairs plane j+1's
// out-of-volume cells in its raw slot (edge tiles, Clamp / Mirror / Wrap)
// once TMA has delivered it; after the barrier, thread 0 refills plane j's
// raw slot.  Border needs no repair: TMA fills out-of-bounds cells with
// zeros (stored 0), and a Border plane outside the volume in z is fetched as
// a fully out-of-bounds box.
//
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
constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int CTAS_PER_SM = 2;
constexpr int GPR = HALF / 4;  // x-pass items (4 output pairs) per row

template <int K>
struct Shape {
  static constexpr int R = K / 2;
  static constexpr int YPT = K == 3 ? 8 : 4;  // y + z pass rows per thread
  static constexpr int RG = WARPS / 2;        // row groups: 2 warps (64 pairs) each
  static constexpr int TY = RG * YPT;
  static constexpr int BY = TY + 2 * R;       // raw / x-sum rows
  static constexpr int NQ = BY * GPR;         // x-pass items per plane
  static constexpr int QPT = (NQ + THREADS - 1) / THREADS;
};

__host__ __device__ constexpr int tile_rows(int k) { return (WARPS / 2) * (k == 3 ? 8 : 4); }

template <typename T, int K>
struct Cfg {
  using S = Shape<K>;
  static constexpr int A = tma::box_align_left(S::R, (int)sizeof(T));
  static constexpr int BX = tma::box_width(S::R, (int)sizeof(T));
  static constexpr int RAW_BYTES = BX * S::BY * (int)sizeof(T);
  static constexpr int RAW_PITCH = (RAW_BYTES + 127) / 128 * 128;
  static constexpr int XB_BYTES = S::BY * HALF * 8;
  static constexpr int SMEM_PER_CTA = (228 * 1024) / CTAS_PER_SM - 1024;
  static constexpr int FIT = (SMEM_PER_CTA - 256 - 2 * XB_BYTES) / RAW_PITCH;
  static constexpr int S_RAW = FIT < 8 ? FIT : 8;
  static constexpr int SMEM = 2 * XB_BYTES + S_RAW * RAW_PITCH + S_RAW * 8 + 128;
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

template <typename T, int K, int MODE>
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM)
    filter_sep_kernel(const __grid_constant__ CUtensorMap map_src,
                      const __grid_constant__ CUtensorMap map_lo,
                      const __grid_constant__ CUtensorMap map_hi, const TmaParams p,
                      const __grid_constant__ Factors<K> f) {
  using C = Cfg<T, K>;
  using S = Shape<K>;
  constexpr int R = S::R, YPT = S::YPT, TY = S::TY, BY = S::BY, SR = C::S_RAW;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (tma::smem_u32(smem_raw) & 127u)) & 127u);
  T* raw_base = reinterpret_cast<T*>(smem);
  uint64_t* xb_base = reinterpret_cast<uint64_t*>(smem + SR * C::RAW_PITCH);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SR * C::RAW_PITCH + 2 * C::XB_BYTES);

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
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const bool leader = tid == 0;
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
  auto repair = [&](int j, T* raw) {
    if constexpr (MODE != VKT_BORDER) {
      if (!edge) return;
      const tma::PlaneSrc src = tma::resolve<MODE>(p, R, zo0 - R + j);
      for (int q = tid; q < ec.total; q += THREADS) {
        int gx, gy;
        ec.cell(p.nx, p.ny, q, gx, gy);
        // the full mapping: a volume thinner than the halo overshoots by more
        // than one extent (the mapped cell is inside the box: the tile then
        // covers the whole axis)
        const int mx = (int)map_index<MODE>(gx, p.nx), my = (int)map_index<MODE>(gy, p.ny);
        T v;
        if constexpr (MODE == VKT_WRAP)
          v = __ldg(tma::plane_ptr<T>(p, src) + (int64_t)my * p.pitch + mx);
        else
          v = raw[(my - ya) * C::BX + mx - (x0 - C::A)];
        VKT_CHECK((gy - ya) * C::BX + gx - (x0 - C::A) >= 0 &&
                      (gy - ya) * C::BX + gx - (x0 - C::A) < C::BX * BY,
                  "sep repair: dest");
        raw[(gy - ya) * C::BX + gx - (x0 - C::A)] = v;
      }
    }
  };

  // y + z pass: pair column c of rows [rg*YPT, rg*YPT + YPT)
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

  // plane 0 in place and repaired before the loop
  tma::mbar_wait(&full[0], 0);
  repair(0, raw_slot(0));
  if (edge) tma::fence_proxy_async();
  __syncthreads();

  int r = 0;
  uint32_t ph = 0;
#pragma unroll 1
  for (int j = 0; j <= np; ++j) {
    VKT_JITTER_POINT(j);
    if (j < np) {
      // ---- x pass: raw slot r -> xb[j & 1]
      const T* raw = raw_slot(r);
      uint64_t* xb = xb_base + (j & 1) * (C::XB_BYTES / 8);
#pragma unroll
      for (int k = 0; k < S::QPT; ++k) {
        const int q = tid + THREADS * k;
        if (S::NQ % THREADS != 0 && k == S::QPT - 1 && q >= S::NQ) break;
        const int row = q / GPR, g = q - row * GPR;
        // cells x0-4+4g .. x0+4g+7 (and +HALF): output pair jj at tap dx
        // reads cell 4g + jj + dx - R, i.e. index jj + dx + 4 - R here
        const T* src = raw + row * C::BX + (C::A - 4) + 4 * g;
        uint64_t P[12];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          uint32_t lo[4], hi[4];
          tma::load_quad<T>(src + 4 * i, lo);
          tma::load_quad<T>(src + 4 * i + HALF, hi);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
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
        // two 16-byte chunks; odd quads of 4 lanes store their second chunk
        // first so the 8 lanes of a phase cover all 32 banks
        uint4 c0 = make_uint4((uint32_t)o[0], (uint32_t)(o[0] >> 32), (uint32_t)o[1], (uint32_t)(o[1] >> 32));
        uint4 c1 = make_uint4((uint32_t)o[2], (uint32_t)(o[2] >> 32), (uint32_t)o[3], (uint32_t)(o[3] >> 32));
        const bool swap = (lane >> 2) & 1;
        uint4* d = reinterpret_cast<uint4*>(xb + row * HALF + 4 * g);
        d[swap ? 1 : 0] = swap ? c1 : c0;
        d[swap ? 0 : 1] = swap ? c0 : c1;
      }
    }
    if (j >= 1) {
      // ---- y + z pass on plane j-1 (xb[(j-1) & 1])
      const uint64_t* col = xb_base + ((j - 1) & 1) * (C::XB_BYTES / 8) + rg * YPT * HALF + c;
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
#pragma unroll
      for (int rr = 0; rr < YPT; ++rr)
#pragma unroll
        for (int m = 0; m < K; ++m)
          acc[rr][m] = tma::ffma2_from(ys[rr], f.wz[K - 1 - m], m + 1 < K ? acc[rr][m + 1 < K ? m + 1 : m] : a00);
      if (j - 1 >= 2 * R) {
        T* o = out_plane;
#pragma unroll
        for (int rr = 0; rr < YPT; ++rr, o += p.pitch) {
          if (rr >= rows_ok) continue;
          if constexpr (sizeof(T) == 4) {
            chk = tma::ffma2_from(acc[rr][0], 0.0f, chk);
            if (st_lo) st_cs(o, tma::f2lo(acc[rr][0]));
            if (st_hi) st_cs(o + HALF, tma::f2hi(acc[rr][0]));
          } else {
            if (st_lo) st_cs(o, sat_floor<T>(tma::f2lo(acc[rr][0])));
            if (st_hi) st_cs(o + HALF, sat_floor<T>(tma::f2hi(acc[rr][0])));
          }
        }
        out_plane += plane_elems;
      }
    }
    // ---- plane j+1: wait for its TMA box, repair its out-of-volume cells
    const int r1 = r + 1 == SR ? 0 : r + 1;
    const uint32_t ph1 = r1 == 0 ? ph ^ 1u : ph;
    if (j + 1 < np) {
      tma::mbar_wait(&full[r1], ph1);
      repair(j + 1, raw_slot(r1));
      if (edge) tma::fence_proxy_async();
    }
    __syncthreads();
    // every thread is past plane j's x pass: refill its raw slot
    if (j < np && j + SR < np) issue(j + SR, r);
    r = r1;
    ph = ph1;
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
  VKT_SEP_CASES(3)
  VKT_SEP_CASES(5)
  VKT_SEP_CASES(7)
  VKT_SEP_CASES(9)
#undef VKT_SEP_CASES
  return cudaErrorInvalidValue;
}

}  // namespace sep
}  // namespace vkt
