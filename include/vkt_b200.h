/*
 * vkt_b200.h — C ABI of the B200-native ApplyFilter / Fill path.
 *
 * This is the drop-in boundary. The reference (volkit re-implementation at
 * /root/reference, pure Python + numpy) exposes the hot path as Python calls;
 * every entry point below replaces exactly one of them:
 *
 *   vkt_apply_filter  <-  vkt.apply_filter(volume, kernel)
 *                         pkg/src/vkt/ops/filters.py:69-95
 *                         (+ the Wrap/Mirror/Border address modes that the
 *                          north star's ApplyFilter(dst, src, filter, mode) adds;
 *                          the reference only has Clamp, filters.py:78)
 *   vkt_fill_box      <-  vkt.fill_range(volume, roi, value) / vkt.fill
 *                         pkg/src/vkt/ops/core.py:39-55, 65-66
 *                         (the host quantizes `value` exactly like
 *                          pkg/src/vkt/volume.py:102-110 and passes the stored bits)
 *   vkt_status_name   <-  VktError.name (pkg/src/vkt/errors.py:9-14)
 *   vkt_fill_synthetic   bench/test input generator standing in for
 *                         synthetic_structured (pkg/src/vkt/bench.py:38-48):
 *                         same value distributions, counter-based hash instead
 *                         of numpy's PCG64 so it is identical at any sharding.
 *
 * Conventions
 *   - All pointers named src/dst/halo_* are DEVICE pointers; volumes are dense,
 *     x-fastest, linear index i + nx*(j + ny*k) (volume.py:3-5), little endian.
 *   - weights is a HOST pointer to kx*ky*kz doubles, x-fastest, i.e. exactly
 *     Kernel.weights.ravel() (filters.py:34-36).
 *   - Every call is asynchronous on `stream` and returns a status (0 = OK).
 *   - The library never owns caller buffers and never synchronizes the stream.
 *   - No exceptions cross this boundary.
 *   - Not reentrant per destination buffer; thread safe across distinct
 *     buffers and streams (no global device state is written per call).
 */
#ifndef VKT_B200_H
#define VKT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* vkt_stream_t; /* == cudaStream_t / CUstream */

typedef struct {
  int32_t x, y, z;
} vkt_int3;

/* DataFormat codes, identical to volume.py:29-32 */
enum { VKT_U8 = 1, VKT_U16 = 2, VKT_F32 = 3 };

/* Address modes (north star ApplyFilter(dst, src, filter, addressMode)).
 * Clamp is the reference's behaviour (np.pad mode="edge", filters.py:78). */
enum { VKT_WRAP = 0, VKT_MIRROR = 1, VKT_CLAMP = 2, VKT_BORDER = 3 };

/* Status codes; vkt_status_name() returns the reference's error class name. */
enum {
  VKT_OK = 0,
  VKT_INVALID_ARGUMENT = 1, /* "InvalidArgument"   errors.py:17 */
  VKT_EVEN_KERNEL_DIMS = 2, /* "EvenKernelDims"    errors.py:53 */
  VKT_ALLOCATION_FAILURE = 3, /* "AllocationFailure" errors.py:25 */
  VKT_DEVICE_FAILURE = 4    /* "DeviceFailure" (new: CUDA launch/runtime error) */
};

/* Flags for vkt_filter_args.flags */
enum {
  VKT_FLAG_NONE = 0,
  /* Bit-exact reproduction of the reference arithmetic: float64, no FMA
   * contraction, mapped-value formulation, (dz,dy,dx) tap order.  Slow
   * (FP64 pipe); a parity/debug mode. */
  VKT_FLAG_EXACT_F64 = 1,
  /* Force the generic direct kernel even when the tiled TMA kernel applies. */
  VKT_FLAG_FORCE_DIRECT = 2,
  /* vkt_apply_filter_host only: bound device memory to a few chunks (the
   * input streams through ring buffers, halos copied device-to-device)
   * instead of keeping the padded input resident when it fits. */
  VKT_FLAG_HOST_BOUNDED = 4,
  /* Never take the separable path: rank-1 kernels run the dense tiled
   * kernels, bit-identical to the direct kernel. */
  VKT_FLAG_NO_SEPARABLE = 8
};

/* Kernel paths reported by vkt_filter_path() */
/* VKT_PATH_SEPARABLE: rank-1 weights (gaussian_kernel, box_kernel) as three
 * fused 1-D passes; within the reference contract, not bit-identical to the
 * dense paths. */
enum { VKT_PATH_NONE = 0, VKT_PATH_DIRECT = 1, VKT_PATH_EXACT = 2, VKT_PATH_TMA = 3, VKT_PATH_SEPARABLE = 4 };

typedef struct {
  const void* src;      /* device, local slab: dims.x*dims.y*dims.z cells      */
  void* dst;            /* device, same extents; must not alias src           */
  vkt_int3 dims;        /* local extents                                       */
  int32_t format;       /* VKT_U8 / VKT_U16 / VKT_F32                           */
  double map_lo;        /* VoxelMapping lo (volume.py:73-99); ignored for F32  */
  double map_hi;        /* VoxelMapping hi                                     */
  const double* weights;/* HOST, kx*ky*kz, x-fastest                           */
  vkt_int3 kdims;       /* odd per axis                                        */
  int32_t address_mode; /* VKT_WRAP / VKT_MIRROR / VKT_CLAMP / VKT_BORDER       */
  /* z-slab sharding (all zero/NULL for an unsharded volume):                  */
  const void* halo_lo;  /* device, rz planes = global planes z_offset-rz..-1
                           after address mapping, or NULL to resolve in-slab  */
  const void* halo_hi;  /* device, rz planes after the slab, or NULL           */
  int64_t z_offset;     /* global z of local plane 0                           */
  int64_t global_nz;    /* global z extent (0 => dims.z)                       */
  int32_t out_z_begin;  /* local output planes to compute: [begin, end)       */
  int32_t out_z_end;    /* (end <= 0 => dims.z)                                */
  int32_t flags;        /* VKT_FLAG_*                                          */
} vkt_filter_args;

/* ApplyFilter: dst = correlate(src, weights) re-quantized (filters.py:69-95). */
int vkt_apply_filter(const vkt_filter_args* args, vkt_stream_t stream);

/* ApplyFilter on HOST buffers, streamed through HBM (the reference's
 * apply_filter works on host numpy arrays, filters.py:69-95).  Same argument
 * meaning as vkt_apply_filter with every pointer on the HOST:
 *   src / dst : planes [z_offset, z_offset+dims.z) of a volume with
 *               global_nz planes (0 => dims.z; z_offset 0: the whole volume);
 *   halo_lo / halo_hi : optional, rz planes each = the address-mapped global
 *               planes z_offset-rz .. z_offset-1 and after the buffer; when
 *               NULL every halo plane must map inside the buffer (always true
 *               for a whole volume).
 * Computes output planes [out_z_begin, out_z_end) of the buffer (default
 * all) by uploading z-chunks of `chunk_planes` planes (0: ~128 MB) plus their
 * halo planes, filtering each chunk with the device path and downloading
 * it, with H2D / compute / D2H overlapped on three streams; page-locked
 * buffers make the copies asynchronous.  Bit-identical to vkt_apply_filter on
 * the whole volume.  Only 3 chunks are resident, so volumes larger than HBM
 * work.  Returns when dst holds the result. */
int vkt_apply_filter_host(const vkt_filter_args* args, int32_t chunk_planes, vkt_stream_t stream);

/* Which kernel vkt_apply_filter would launch for these args (VKT_PATH_*). */
int vkt_filter_path(const vkt_filter_args* args);

/* Output planes per CTA z-chunk the tiled kernel would use for these args on
 * the current device (0: not the tiled path).  Chunk boundaries are where a
 * CTA's rolling z accumulators restart, so parity tests probe both sides. */
int vkt_filter_chunk_planes(const vkt_filter_args* args);

/* FillRange: set cells in [lo, hi) ∩ [0, dims) to the stored bit pattern
 * `stored_bits` (u8: low 8 bits, u16: low 16 bits, f32: IEEE bits). */
int vkt_fill_box(void* dst, vkt_int3 dims, int32_t format, vkt_int3 lo, vkt_int3 hi,
                 uint32_t stored_bits, vkt_stream_t stream);

/* Deterministic synthetic volume slab: cell (x, y, z_offset + z) of a volume
 * whose global x/y extents are dims.x/dims.y gets hash(seed, global index);
 * u8/u16 uniform over [0, max], f32 uniform in [0, 1). */
int vkt_fill_synthetic(void* dst, vkt_int3 dims, int32_t format, uint64_t seed,
                       int64_t z_offset, vkt_stream_t stream);

/* ---- CLAHE-3D (pkg/src/vkt/ops/filters.py:98-245) ----
 * Brick partition, per-brick histograms, clipped-cdf mappings and the
 * trilinear blend of the 8 nearest brick mappings.  The device computes the
 * histograms (integer, exact) and the blend (IEEE float64 in the reference's
 * operation order, bit-exact); the clip + cdf of the small per-brick
 * histograms is host arithmetic. */
typedef struct {
  const void* src;        /* device volume                                        */
  void* dst;              /* device volume (may equal src: each cell is read once) */
  vkt_int3 dims;
  int32_t format;
  double map_lo, map_hi;
  vkt_int3 bricks;        /* brick counts per axis                                */
  int32_t num_bins;
  const int32_t* bin_lut; /* device, u8/u16: stored value -> bin (host f64 rule);
                             NULL for f32 (binned on the device in f64)           */
  const int32_t* edges;   /* device, (bx+1)+(by+1)+(bz+1) brick edges x|y|z      */
  uint32_t* hist;         /* device out (histograms): bz*by*bx*num_bins           */
  const double* mappings; /* device in (blend): bz*by*bx*num_bins                  */
  const int32_t* blend_lo;/* device in (blend): lower brick per cell, nx|ny|nz    */
  const double* blend_w;  /* device in (blend): blend weight per cell,  nx|ny|nz  */
} vkt_clahe_args;

/* Per-brick histograms of the bin index min(nbins-1, floor(t*nbins)). */
int vkt_clahe_histograms(const vkt_clahe_args* args, vkt_stream_t stream);

/* dst = quantize(lo + (sum of the 8 blended brick mappings)*(hi - lo)). */
int vkt_clahe_blend(const vkt_clahe_args* args, vkt_stream_t stream);

/* ---- Resample / Flip ----
 * Flip: reverse the stored cells along axis 0/1/2 (x/y/z) — a bit-exact
 * permutation (pkg/src/vkt/ops/geometric.py:34-40).  src and dst must not
 * alias. */
int vkt_flip(const void* src, void* dst, vkt_int3 dims, int32_t format, int32_t axis,
             vkt_stream_t stream);

/* Resample a structured volume onto dst_dims cells (ops/core.py:202-262):
 * destination cell centers map uniformly onto the source extent, trilinear
 * samples of the mapped float64 grid with clamp-to-edge (volume.py:237-266),
 * re-quantized into dst_format / dst mapping — float64 in numpy's operation
 * order, bit-identical to the reference. */
int vkt_resample(const void* src, vkt_int3 src_dims, int32_t src_format, double src_lo,
                 double src_hi, void* dst, vkt_int3 dst_dims, int32_t dst_format, double dst_lo,
                 double dst_hi, vkt_stream_t stream);

/* Error class name for a status code (errors.py naming). */
const char* vkt_status_name(int status);

/* Human-readable detail of the last error on the calling host thread. */
const char* vkt_last_error_detail(void);

/* Number of kernels this library has launched in this process (all threads). */
uint64_t vkt_launch_count(void);

/* ABI version (major*10000 + minor*100 + patch). */
int vkt_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VKT_B200_H */
