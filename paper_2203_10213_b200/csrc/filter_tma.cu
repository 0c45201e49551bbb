#include <algorithm>
#include <cmath>
#include <cstdlib>
// filter_tma.cu — host side of the tiled TMA ApplyFilter kernel: eligibility,
// tensor-map encoding (driver entry point, no libcuda link), chunk sizing and
// dispatch.  The kernels are instantiated per voxel format in
// filter_tma_{u8,u16,f32}.cu so the 36 specialisations compile in parallel.
#include <cuda.h>

#include <mutex>

#include "dispatch.h"
#include "filter_tma.cuh"
#include "filter_sep.cuh"
#include "filter_ws.cuh"

namespace vkt {
namespace tma {
template <typename T>
cudaError_t launch_tma_dtype(int k, int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                             const CUtensorMap& mh, const TmaParams& p, const float* w32, dim3 grid,
                             cudaStream_t s);
extern template cudaError_t launch_tma_dtype<uint8_t>(int, int, const CUtensorMap&,
                                                      const CUtensorMap&, const CUtensorMap&,
                                                      const TmaParams&, const float*, dim3,
                                                      cudaStream_t);
extern template cudaError_t launch_tma_dtype<uint16_t>(int, int, const CUtensorMap&,
                                                       const CUtensorMap&, const CUtensorMap&,
                                                       const TmaParams&, const float*, dim3,
                                                       cudaStream_t);
template <>  // explicit specialization (filter_tma_f32.cu): K <= 5 -> filter_tma_zp.cuh
cudaError_t launch_tma_dtype<float>(int, int, const CUtensorMap&, const CUtensorMap&,
                                    const CUtensorMap&, const TmaParams&, const float*, dim3,
                                    cudaStream_t);
#define VKT_ANISO_DECL(KK, T)                                                                      \
  template <>                                                                                     \
  cudaError_t launch_tma_aniso_k##KK<T>(int, bool, int, const CUtensorMap&, const CUtensorMap&,  \
                                        const CUtensorMap&, const TmaParams&, const float*, dim3, \
                                        cudaStream_t);
#define VKT_ANISO_DECLS(KK)                                                                     \
  template <typename T>                                                                         \
  cudaError_t launch_tma_aniso_k##KK(int, bool, int, const CUtensorMap&, const CUtensorMap&,   \
                                     const CUtensorMap&, const TmaParams&, const float*, dim3,  \
                                     cudaStream_t);                                              \
  VKT_ANISO_DECL(KK, uint8_t)                                                                   \
  VKT_ANISO_DECL(KK, uint16_t)                                                                  \
  VKT_ANISO_DECL(KK, float)
VKT_ANISO_DECLS(5)
VKT_ANISO_DECLS(7)
VKT_ANISO_DECLS(9)
#undef VKT_ANISO_DECLS
#undef VKT_ANISO_DECL

// Anisotropic kernels embedded in a K^3 cube: x extent kxs <= K a template,
// padding y rows / z planes skipped by mask (filter_tma_aniso_<fmt>_k<K>.cu).
template <typename T>
cudaError_t launch_tma_aniso(int k, int kxs, bool zthin, int mode, const CUtensorMap& ms,
                             const CUtensorMap& ml, const CUtensorMap& mh, const TmaParams& p,
                             const float* w32, dim3 grid, cudaStream_t s) {
  switch (k) {
    case 5: return launch_tma_aniso_k5<T>(kxs, zthin, mode, ms, ml, mh, p, w32, grid, s);
    case 7: return launch_tma_aniso_k7<T>(kxs, zthin, mode, ms, ml, mh, p, w32, grid, s);
    case 9: return launch_tma_aniso_k9<T>(kxs, zthin, mode, ms, ml, mh, p, w32, grid, s);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace tma
namespace tmaws {
extern template cudaError_t launch_ws_dtype<uint8_t>(int, const CUtensorMap&, const CUtensorMap&,
                                                     const CUtensorMap&, const tma::TmaParams&,
                                                     const float*, dim3, cudaStream_t);
extern template cudaError_t launch_ws_dtype<uint16_t>(int, const CUtensorMap&, const CUtensorMap&,
                                                      const CUtensorMap&, const tma::TmaParams&,
                                                      const float*, dim3, cudaStream_t);
}  // namespace tmaws
namespace sep {
#define VKT_SEP_DECL(T)                                                                            \
  extern template cudaError_t launch_sep_dtype<T>(int, int, const CUtensorMap&, const CUtensorMap&, \
                                                  const CUtensorMap&, const CUtensorMap&,           \
                                                  const tma::TmaParams&, const float*, const float*, \
                                                  const float*, dim3, cudaStream_t);
VKT_SEP_DECL(uint8_t)
VKT_SEP_DECL(uint16_t)
VKT_SEP_DECL(float)
#undef VKT_SEP_DECL
}  // namespace sep

namespace {



int bpc_of(int format) { return format == VKT_U8 ? 1 : format == VKT_U16 ? 2 : 4; }

// Separable plans run filter_sep.cuh; u8/u16 3x3x3 dense plans the
// warp-specialized kernel (filter_ws.cuh), with 32-row tiles; everything else
// the paired-layout kernel's 16-row tiles.
bool warp_kernel(const FilterPlan& plan) {
  return !plan.sep && plan.args->format != VKT_F32 && plan.args->kdims.x == 3;
}
int tile_rows(const FilterPlan& plan) {
  return plan.sep ? sep::tile_rows(plan.args->kdims.x, bpc_of(plan.args->format))
                  : warp_kernel(plan) ? tmaws::TY : tma::TY;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}


bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool encode_box(CUtensorMap* m, const void* base, int format, int nx, int ny, int nz, int pitch,
                int box_x, int box_y) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return false;
  const int bpc = bpc_of(format);
  CUtensorMapDataType dt = format == VKT_U8    ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                           : format == VKT_U16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * bpc, (cuuint64_t)pitch * ny * bpc};
  cuuint32_t box[3] = {(cuuint32_t)box_x, (cuuint32_t)box_y, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult res = fn(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

// Source boxes: the tile plus its halo rows, TMA-aligned in x (box_width).
bool encode(CUtensorMap* m, const void* base, int format, int nx, int ny, int nz, int r,
            int pitch, int tile_y) {
  return encode_box(m, base, format, nx, ny, nz, pitch, tma::box_width(r, bpc_of(format)),
                    tile_y + 2 * r);
}

}  // namespace

// Chunk depth ZC: every CTA pays ~2R extra input planes plus a pipeline
// fill; the grid pays wave quantization.  Pick the ZC with the smallest
// estimated time  waves(ZC) * (ZC + 2R + fill)  (fill ~ 3 planes).
int tma_chunk_planes(const FilterPlan& plan) {
  const vkt_filter_args& a = *plan.args;
  const int k = a.kdims.x, r = k / 2;
  const int nzo = plan.z_end - plan.z_begin;
  if (nzo <= 0) return 1;
  const int ty = tile_rows(plan);
  const int64_t nxy = (int64_t)((a.dims.x + tma::TX - 1) / tma::TX) * ((a.dims.y + ty - 1) / ty);
  // CTAs per SM: the paired kernel's Layout, or filter_tma_zp.cuh's for f32
  // K = 3 (4, Wrap 3)
  const int64_t slots = (int64_t)sm_count() * (plan.sep ? sep::ctas_per_sm(k)
                                 : a.format == VKT_F32 && k == 3 ? (a.address_mode == VKT_WRAP ? 3 : 4)
                                 : k >= 7 ? tma::Layout<2, 7>::CTAS_PER_SM
                                 : k == 5 ? tma::Layout<2, 5>::CTAS_PER_SM
                                 : warp_kernel(plan) ? tmaws::CTAS_PER_SM
                                                  : tma::Layout<2, 3>::CTAS_PER_SM);
  // Under 3 waves the grid balances poorly: 512^3 u16 3^3 runs 0.266 ms at
  // 64-plane chunks (1.7 waves), 0.246 at 32 (3.5 waves); f32 3^3 0.241 vs
  // 0.231 (profiles/r01_zc_sweep3_v37.txt, r01_zc_sweep4_v37.txt).  So chunks
  // of >= 16 planes that fill 3 waves are preferred when there are any (not
  // on small volumes such as 256^3, where 16-plane chunks at < 1 wave stay
  // fastest).
  bool three_waves = false;
  for (int cand : {64, 48, 32, 24, 16}) {
    const int z = cand < nzo ? cand : nzo;
    if (z >= 16 && nxy * ((nzo + z - 1) / z) >= 3 * slots) three_waves = true;
  }
  int zc = 64;
  double best = 1e300;
  for (int cand : {64, 48, 32, 24, 16, 12, 8, 6, 4}) {
    const int z = cand < nzo ? cand : nzo;
    const int64_t ctas = nxy * ((nzo + z - 1) / z);
    if (three_waves && (z < 16 || ctas < 3 * slots)) continue;
    // a partial last wave costs half a wave plus its fill: its CTAs share
    // SMs with fewer neighbours (512^3 K = 5 / 7: 64-plane chunks at 3.5
    // waves beat 48 at 4.8 by 2-3%, profiles/r01_zc_sweep_v36.txt)
    const double w = (double)ctas / slots, wf = std::floor(w), fr = w - wf;
    const double cost = (wf + (fr > 0 ? 0.5 + 0.5 * fr : 0.0)) * (z + 2 * r + 3);
    if (cost < best * 0.98) {
      best = cost;
      zc = z;
    }
  }
  // K >= 7 is FMA-bound and its halo planes cost staging issue slots: on
  // volumes that still fill >= 8 waves, ~171-plane chunks are 1.5-2% faster
  // than the model's pick (1024^3 u16 / f32 7^3: 11.32 -> 11.11 ms,
  // profiles/r01_zc_sweep2_v36.txt); K <= 5 gains nothing measurable (~94-plane
  // chunks at 1024^3 K = 5: 4.261 vs 4.257 ms, profiles/r01_k5_chunks_v39.txt).
  if (k >= 7 && !plan.sep) {
    const int nch = (nzo + 170) / 171;
    if (nxy * nch >= 8 * slots) zc = (nzo + nch - 1) / nch;
  }
  // The separable kernel at K >= 5: ~128-plane chunks where >= 8 waves remain
  // (1024^3 u16 7^3 1.665 -> 1.615 ms, 9^3 2.28 -> 2.18, f32 box 5^3 1.716 ->
  // 1.698; 3^3 unchanged; thinner slabs keep the model's pick,
  // profiles/r02_zc_sweep_sep.txt; Wrap 1.88 -> 1.80 ms now that its slower
  // face tiles run first, filter_sep.cuh edge_first).
  if (plan.sep && k >= 5) {
    const int nch = (nzo + 127) / 128;
    if (nxy * nch >= 8 * slots) zc = (nzo + nch - 1) / nch;
  }
  if (const char* e = std::getenv("VKT_TMA_ZC")) zc = std::max(1, std::min(nzo, std::atoi(e)));  // diagnostics
  return zc;
}

bool tma_encode_available() { return encode_fn() != nullptr; }

bool tma_supported(const vkt_filter_args& a) {
  if (a.flags & (VKT_FLAG_EXACT_F64 | VKT_FLAG_FORCE_DIRECT)) return false;
  const int k = a.kdims.x;
  if (a.kdims.y != k || a.kdims.z != k) return false;
  if (k != 3 && k != 5 && k != 7 && k != 9) return false;

  // rows that are not 16-byte multiples (or unaligned buffers) are staged
  // through pitched scratch copies (launch_filter_tma), so every extent works
  return encode_fn() != nullptr;
}

namespace {

// Launch on buffers whose rows are `pitch` cells (16-byte multiple) apart.
int launch_pitched(const FilterPlan& plan, const void* src, void* dst, const void* hlo,
                   const void* hhi, int pitch, cudaStream_t s) {
  const vkt_filter_args& a = *plan.args;
  const int k = a.kdims.x, r = k / 2;
  const int ty = tile_rows(plan);
  const bool wk = warp_kernel(plan);
  CUtensorMap ms, ml, mh;
  if (!encode(&ms, src, a.format, a.dims.x, a.dims.y, a.dims.z, r, pitch, ty)) return -1;
  ml = ms;
  mh = ms;
  if (hlo && r > 0 && !encode(&ml, hlo, a.format, a.dims.x, a.dims.y, r, r, pitch, ty)) return -1;
  if (hhi && r > 0 && !encode(&mh, hhi, a.format, a.dims.x, a.dims.y, r, r, pitch, ty)) return -1;

  tma::TmaParams p{};
  p.dst = dst;
  p.src = src;
  p.halo_lo = hlo;
  p.halo_hi = hhi;
  p.nx = a.dims.x;
  p.ny = a.dims.y;
  p.nz = a.dims.z;
  p.pitch = pitch;
  p.z_begin = plan.z_begin;
  p.z_end = plan.z_end;
  p.z_offset = plan.geom.z_offset;
  p.global_nz = plan.geom.global_nz;
  p.c = plan.epi_c;
  p.zskip = plan.zskip;
  p.yskip = plan.yskip;
  const bool aniso = plan.kxs > 0 && !wk && k >= 5;
  p.guard = plan.guard;
  p.nonfinite = plan.nonfinite;

  const int nzo = plan.z_end - plan.z_begin;
  const int zc = tma_chunk_planes(plan);
  p.zc = zc;
  dim3 grid((a.dims.x + tma::TX - 1) / tma::TX, (a.dims.y + ty - 1) / ty, (nzo + zc - 1) / zc);
  if (grid.y > 65535 || grid.z > 65535) return -1;

  cudaError_t err;
  if (plan.sep) {
    // output tiles leave through TMA stores: the destination as a tensor
    // whose planes [z_begin, z_end) the launch writes
    CUtensorMap md;
    if (!encode_box(&md, dst, a.format, a.dims.x, a.dims.y, plan.z_end, pitch, tma::TX, ty)) return -1;
    const float *fx = plan.fx.data(), *fy = plan.fy.data(), *fz = plan.fz.data();
    err = a.format == VKT_U8    ? sep::launch_sep_dtype<uint8_t>(k, a.address_mode, ms, ml, mh, md, p, fx, fy, fz, grid, s)
          : a.format == VKT_U16 ? sep::launch_sep_dtype<uint16_t>(k, a.address_mode, ms, ml, mh, md, p, fx, fy, fz, grid, s)
                                : sep::launch_sep_dtype<float>(k, a.address_mode, ms, ml, mh, md, p, fx, fy, fz, grid, s);
  } else switch (a.format) {
    case VKT_U8:
      err = wk      ? tmaws::launch_ws_dtype<uint8_t>(a.address_mode, ms, ml, mh, p, plan.w32.data(), grid, s)
            : aniso ? tma::launch_tma_aniso<uint8_t>(k, plan.kxs, plan.zthin, a.address_mode, ms, ml, mh, p, plan.w32.data(), grid, s)
                    : tma::launch_tma_dtype<uint8_t>(k, a.address_mode, ms, ml, mh, p, plan.w32.data(), grid, s);
      break;
    case VKT_U16:
      err = wk      ? tmaws::launch_ws_dtype<uint16_t>(a.address_mode, ms, ml, mh, p, plan.w32.data(), grid, s)
            : aniso ? tma::launch_tma_aniso<uint16_t>(k, plan.kxs, plan.zthin, a.address_mode, ms, ml, mh, p, plan.w32.data(), grid, s)
                    : tma::launch_tma_dtype<uint16_t>(k, a.address_mode, ms, ml, mh, p, plan.w32.data(), grid, s);
      break;
    default:
      err = aniso ? tma::launch_tma_aniso<float>(k, plan.kxs, plan.zthin, a.address_mode, ms, ml, mh, p, plan.w32.data(), grid, s)
                  : tma::launch_tma_dtype<float>(k, a.address_mode, ms, ml, mh, p, plan.w32.data(), grid, s);
      break;
  }
  count_launch();
  if (err != cudaSuccess) {
    set_error_detail("filter_tma launch: %s", cudaGetErrorString(err));
    return VKT_DEVICE_FAILURE;
  }
  return VKT_OK;
}

}  // namespace

int launch_filter_tma(const FilterPlan& plan, cudaStream_t s) {
  const vkt_filter_args& a = *plan.args;
  const int bpc = bpc_of(a.format);
  const int rz = a.kdims.z / 2;
  const bool direct = ((int64_t)a.dims.x * bpc) % 16 == 0 && aligned16(a.src) && aligned16(a.dst) &&
                      (!a.halo_lo || aligned16(a.halo_lo)) && (!a.halo_hi || aligned16(a.halo_hi));
  if (direct) return launch_pitched(plan, a.src, a.dst, a.halo_lo, a.halo_hi, a.dims.x, s);

  // Pitched staging: copy the planes this launch reads (and the halos it
  // reads) into scratch with rows padded to 16 bytes, filter there, copy the
  // computed planes back.  Two extra passes over the data; hidden for the
  // FP32-bound kernels.  When every plane of the read window
  // [z_begin - rz, z_end + rz) is a slab plane or comes from a halo buffer,
  // only the window's slab planes are staged, as a sub-slab (the thin
  // boundary launches of a sharded step stage rz..2rz planes, not the slab);
  // otherwise (address-mapped planes at the volume's faces) the whole slab.
  const int pitch = (int)((((int64_t)a.dims.x * bpc + 15) / 16 * 16) / bpc);
  const size_t row_b = (size_t)a.dims.x * bpc, prow_b = (size_t)pitch * bpc;
  const size_t pplane = prow_b * a.dims.y;
  const int wlo = plan.z_begin - rz, whi = plan.z_end + rz;
  const bool self_contained = (wlo >= 0 || a.halo_lo != nullptr) && (whi <= a.dims.z || a.halo_hi != nullptr);
  const int zlo = self_contained ? (wlo > 0 ? wlo : 0) : 0;
  const int zhi = self_contained ? (whi < a.dims.z ? whi : a.dims.z) : a.dims.z;
  vkt_filter_args sub = a;
  sub.dims.z = zhi - zlo;
  sub.z_offset = a.z_offset + zlo;
  sub.halo_lo = zlo == 0 ? a.halo_lo : nullptr;
  sub.halo_hi = zhi == a.dims.z ? a.halo_hi : nullptr;
  FilterPlan sp = plan;
  sp.args = &sub;
  sp.z_begin = plan.z_begin - zlo;
  sp.z_end = plan.z_end - zlo;
  sp.geom.z_offset = sub.z_offset;
  sp.geom.nz = sub.dims.z;
  const int nzo = plan.z_end - plan.z_begin;
  const size_t in_b = pplane * sub.dims.z, halo_b = pplane * rz, out_b = pplane * nzo;
  uint8_t* buf = nullptr;
  const size_t total = in_b + 2 * halo_b + out_b + 64;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&buf), total, s);
  if (e != cudaSuccess) {
    set_error_detail("scratch_alloc(pitched staging, %zu bytes): %s", total, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? VKT_ALLOCATION_FAILURE : VKT_DEVICE_FAILURE;
  }
  uint8_t* in = buf;
  uint8_t* hlo = sub.halo_lo ? in + in_b : nullptr;
  uint8_t* hhi = sub.halo_hi ? in + in_b + halo_b : nullptr;
  uint8_t* out = in + in_b + 2 * halo_b;
  auto copy2d = [&](void* d, size_t dp, const void* src, size_t sp_, size_t rows) {
    return cudaMemcpy2DAsync(d, dp, src, sp_, row_b, rows, cudaMemcpyDeviceToDevice, s);
  };
  int st = VKT_OK;
  const uint8_t* src_planes = static_cast<const uint8_t*>(a.src) + row_b * a.dims.y * zlo;
  if (copy2d(in, prow_b, src_planes, row_b, (size_t)a.dims.y * sub.dims.z) != cudaSuccess ||
      (hlo && copy2d(hlo, prow_b, sub.halo_lo, row_b, (size_t)a.dims.y * rz) != cudaSuccess) ||
      (hhi && copy2d(hhi, prow_b, sub.halo_hi, row_b, (size_t)a.dims.y * rz) != cudaSuccess)) {
    set_error_detail("pitched staging copy: %s", cudaGetErrorString(cudaGetLastError()));
    st = VKT_DEVICE_FAILURE;
  }
  if (st == VKT_OK) {
    // the kernel addresses output plane oz at dst + oz * plane: shift so the
    // computed planes [z_begin, z_end) land in `out`
    uint8_t* dst_base = out - (ptrdiff_t)pplane * sp.z_begin;
    st = launch_pitched(sp, in, dst_base, hlo, hhi, pitch, s);
  }
  if (st == VKT_OK &&
      cudaMemcpy2DAsync(static_cast<uint8_t*>(a.dst) + row_b * a.dims.y * plan.z_begin, row_b, out, prow_b,
                        row_b, (size_t)a.dims.y * nzo, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
    set_error_detail("pitched staging copy back: %s", cudaGetErrorString(cudaGetLastError()));
    st = VKT_DEVICE_FAILURE;
  }
  scratch_free(buf, s);
  return st;
}

}  // namespace vkt
