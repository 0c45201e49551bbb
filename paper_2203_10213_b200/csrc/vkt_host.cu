// vkt_host.cu — ApplyFilter on host buffers, streamed through HBM.
//
// The reference filters host numpy arrays (filters.py:69-95).  This entry
// point keeps that contract for callers whose volume lives in host memory:
// it cuts the requested output planes into z-chunks, and for each chunk
//   H2D  : uploads the chunk's planes plus its 2*rz halo planes (address
//          mapped at the global z boundary, zero planes for Border) into one
//          contiguous device buffer [halo_lo | slab | halo_hi],
//   GPU  : runs the device ApplyFilter on the slab with those halos — the
//          same sharded-slab machinery as the multi-GPU path, so results are
//          bit-identical to a whole-volume launch,
//   D2H  : downloads the chunk's output planes,
// with the three phases of consecutive chunks overlapped on three streams
// and NB input and NB output buffers in rotation.  Only NB chunks are resident, so volumes
// larger than HBM work.  Two details keep it at the PCIe floor: a chunk's
// low halo (2*rz planes) is copied device-to-device from the previous
// chunk's input instead of crossing PCIe again, and chunk sizes ramp up and
// down at the ends (chunk_schedule) so the un-overlapped first upload and
// last download are short.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dispatch.h"

namespace vkt {
namespace {

constexpr int NB = 4;  // input buffers and output buffers in flight

// Owns the pipeline's streams, events and device pool; on every exit path
// (including errors) it drains the streams before releasing anything, so no
// copy can still be reading or writing the caller's host buffers.
struct HostCtx {
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr, s_comp = nullptr;
  cudaEvent_t h2d_done[NB] = {}, comp_done[NB] = {}, d2h_done[NB] = {}, alloc_done = nullptr;
  uint8_t* pool = nullptr;
  ~HostCtx() {
    if (s_h2d) cudaStreamSynchronize(s_h2d);
    if (s_d2h) cudaStreamSynchronize(s_d2h);
    if (s_comp) cudaStreamSynchronize(s_comp);
    if (pool) {
      scratch_free(pool, s_comp);
      cudaStreamSynchronize(s_comp);
    }
    for (int b = 0; b < NB; ++b) {
      if (h2d_done[b]) cudaEventDestroy(h2d_done[b]);
      if (comp_done[b]) cudaEventDestroy(comp_done[b]);
      if (d2h_done[b]) cudaEventDestroy(d2h_done[b]);
    }
    if (alloc_done) cudaEventDestroy(alloc_done);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
  }
};

int cuda_fail(cudaError_t e, const char* what) {
  set_error_detail("%s: %s", what, cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? VKT_ALLOCATION_FAILURE : VKT_DEVICE_FAILURE;
}

#define VKT_CK(call, what)                        \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

int64_t map_plane(int64_t g, int64_t n, int mode) {
  switch (mode) {
    case VKT_WRAP: return map_index<VKT_WRAP>(g, n);
    case VKT_MIRROR: return map_index<VKT_MIRROR>(g, n);
    case VKT_CLAMP: return map_index<VKT_CLAMP>(g, n);
    default: return map_index<VKT_BORDER>(g, n);
  }
}

struct HostSlab {
  const uint8_t* buf;      // global planes [z0, z0 + n)
  int64_t z0, n;
  const uint8_t* halo_lo;  // mapped planes for g in [z0 - rz, z0), or NULL
  const uint8_t* halo_hi;  // mapped planes for g in [z0 + n, z0 + n + rz), or NULL
  int rz;
};

// Upload global planes g0 .. g0+count-1 into dev: planes inside the host
// buffer are copied directly, planes in the caller's halo ranges come from
// the host halos, everything else is address mapped over gnz (Border planes
// are zeroed).  Runs of consecutive source planes become one copy.
int upload_planes(uint8_t* dev, const HostSlab& h, int64_t g0, int count, int64_t gnz,
                  int64_t plane_bytes, int mode, cudaStream_t s) {
  int i = 0;
  while (i < count) {
    const int64_t g = g0 + i;
    const uint8_t* halo = nullptr;
    int64_t hidx = 0;
    if (g < h.z0 && h.halo_lo != nullptr && g >= h.z0 - h.rz) {
      halo = h.halo_lo;
      hidx = g - (h.z0 - h.rz);
    } else if (g >= h.z0 + h.n && h.halo_hi != nullptr && g < h.z0 + h.n + h.rz) {
      halo = h.halo_hi;
      hidx = g - (h.z0 + h.n);
    }
    if (halo != nullptr) {
      VKT_CK(cudaMemcpyAsync(dev + (int64_t)i * plane_bytes, halo + hidx * plane_bytes, plane_bytes,
                             cudaMemcpyHostToDevice, s),
             "H2D halo");
      i += 1;
      continue;
    }
    const int64_t hz0 = h.z0, hnz = h.n;
    const uint8_t* host = h.buf;
    const int64_t m = map_plane(g, gnz, mode);
    int run = 1;
    if (m < 0) {
      while (i + run < count && map_plane(g0 + i + run, gnz, mode) < 0) ++run;
      VKT_CK(cudaMemsetAsync(dev + (int64_t)i * plane_bytes, 0, run * plane_bytes, s), "memset halo");
    } else {
      if (m < hz0 || m >= hz0 + hnz) {
        set_error_detail("plane %lld needed for the halo is not in the host buffer [%lld, %lld)",
                         (long long)m, (long long)hz0, (long long)(hz0 + hnz));
        return VKT_INVALID_ARGUMENT;
      }
      while (i + run < count && map_plane(g0 + i + run, gnz, mode) == m + run &&
             m + run < hz0 + hnz && g0 + i + run >= hz0 && g0 + i + run < hz0 + hnz)
        ++run;
      VKT_CK(cudaMemcpyAsync(dev + (int64_t)i * plane_bytes, host + (m - hz0) * plane_bytes,
                             run * plane_bytes, cudaMemcpyHostToDevice, s),
             "H2D chunk");
    }
    i += run;
  }
  return VKT_OK;
}

// Chunk sizes for T output planes with at most C per chunk: a short ramp
// (C/8, C/4, C/2) at both ends so the first upload and the last download —
// the parts of the pipeline that overlap nothing — stay small, and equal
// full-size chunks in between.
std::vector<int> chunk_schedule(int T, int C) {
  std::vector<int> ramp;
  for (int d = 8; d >= 2; d /= 2)
    if (C / d >= 4) ramp.push_back(C / d);
  int rsum = 0;
  for (int r : ramp) rsum += r;
  std::vector<int> out;
  if (T <= 2 * rsum + C) {  // short volume: equal chunks of at most C/2 (or C)
    const int cmax = std::max(1, ramp.empty() ? C : ramp.back());
    const int k = (T + cmax - 1) / cmax;
    for (int i = 0; i < k; ++i) out.push_back(T / k + (i < T % k ? 1 : 0));
    return out;
  }
  out = ramp;
  const int mid = T - 2 * rsum;
  const int k = (mid + C - 1) / C;
  for (int i = 0; i < k; ++i) out.push_back(mid / k + (i < mid % k ? 1 : 0));
  out.insert(out.end(), ramp.rbegin(), ramp.rend());
  return out;
}

}  // namespace
}  // namespace vkt

using namespace vkt;

extern "C" int vkt_apply_filter_host(const vkt_filter_args* args, int32_t chunk_planes,
                                     vkt_stream_t stream) {
  VKT_NVTX("vkt_apply_filter_host");
  const vkt::StreamDeviceGuard device_guard(reinterpret_cast<cudaStream_t>(stream));
  if (args == nullptr) {
    set_error_detail("args is NULL");
    return VKT_INVALID_ARGUMENT;
  }
  const vkt_filter_args& a = *args;
  const int64_t gnz = a.global_nz > 0 ? a.global_nz : a.dims.z;
  if (a.z_offset < 0 || a.z_offset + a.dims.z > gnz) {
    set_error_detail("host slab [%lld, %lld) outside global z extent %lld", (long long)a.z_offset,
                     (long long)(a.z_offset + a.dims.z), (long long)gnz);
    return VKT_INVALID_ARGUMENT;
  }
  // Validate everything except the device pointers with the device-path
  // planner, using placeholder device addresses.
  {
    vkt_filter_args probe = a;
    probe.src = reinterpret_cast<const void*>(uintptr_t(256));
    probe.dst = reinterpret_cast<void*>(uintptr_t(512));
    probe.z_offset = 0;
    probe.global_nz = 0;
    probe.halo_lo = nullptr;
    probe.halo_hi = nullptr;
    if (a.src == nullptr || a.dst == nullptr) {
      set_error_detail("src and dst must be non-NULL host pointers");
      return VKT_INVALID_ARGUMENT;
    }
    if (vkt_filter_path(&probe) == VKT_PATH_NONE) return vkt_apply_filter(&probe, nullptr);
  }
  cudaStream_t s_comp = reinterpret_cast<cudaStream_t>(stream);
  const int bpc = a.format == VKT_U8 ? 1 : a.format == VKT_U16 ? 2 : 4;
  const int64_t nz = a.dims.z;  // planes in the host buffers
  const int64_t plane_bytes = (int64_t)a.dims.x * a.dims.y * bpc;
  const int rz = a.kdims.z / 2;
  const int zb = a.out_z_begin > 0 ? a.out_z_begin : 0;
  const int ze = a.out_z_end > 0 ? std::min<int>(a.out_z_end, (int)nz) : (int)nz;
  if (ze <= zb) return VKT_OK;
  // default chunk: ~128 MB of planes (long enough for full-depth z chunks in
  // the kernel and few launches, short enough to fill the pipeline quickly)
  int C = chunk_planes > 0 ? chunk_planes : (int)std::max<int64_t>(16, (128ll << 20) / plane_bytes);
  C = std::min(C, ze - zb);

  const std::vector<int> sizes = chunk_schedule(ze - zb, C);

  HostCtx ctx;
  ctx.s_comp = s_comp;
  VKT_CK(cudaStreamCreateWithFlags(&ctx.s_h2d, cudaStreamNonBlocking), "stream");
  VKT_CK(cudaStreamCreateWithFlags(&ctx.s_d2h, cudaStreamNonBlocking), "stream");
  for (int b = 0; b < NB; ++b) {
    VKT_CK(cudaEventCreateWithFlags(&ctx.h2d_done[b], cudaEventDisableTiming), "event");
    VKT_CK(cudaEventCreateWithFlags(&ctx.comp_done[b], cudaEventDisableTiming), "event");
    VKT_CK(cudaEventCreateWithFlags(&ctx.d2h_done[b], cudaEventDisableTiming), "event");
  }
  VKT_CK(cudaEventCreateWithFlags(&ctx.alloc_done, cudaEventDisableTiming), "event");

  // Input: when the whole padded input [zb-rz, ze+rz) fits comfortably in
  // free HBM it stays resident, each chunk uploads only its new planes and
  // finds its halos already in place; otherwise NB ring buffers of
  // [rz | C | rz] planes.  Output: NB ring buffers of C planes.
  const int64_t total_in = (int64_t)(ze - zb + 2 * rz) * plane_bytes;
  size_t free_b = 0, total_b = 0;
  VKT_CK(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  const bool resident = !(a.flags & VKT_FLAG_HOST_BOUNDED) && total_in <= (int64_t)(free_b / 2);
  const int64_t in_bytes = resident ? total_in : (int64_t)(C + 2 * rz) * plane_bytes;
  const int64_t in_stride = (in_bytes + 255) / 256 * 256;
  const int64_t out_stride = ((int64_t)C * plane_bytes + 255) / 256 * 256;
  const int n_in = resident ? 1 : NB;
  VKT_CK(scratch_alloc(reinterpret_cast<void**>(&ctx.pool), n_in * in_stride + NB * out_stride, s_comp),
         "scratch_alloc");
  uint8_t* pool = ctx.pool;
  uint8_t* out_pool = pool + n_in * in_stride;
  VKT_CK(cudaEventRecord(ctx.alloc_done, s_comp), "event");
  VKT_CK(cudaStreamWaitEvent(ctx.s_h2d, ctx.alloc_done, 0), "wait");
  VKT_CK(cudaStreamWaitEvent(ctx.s_d2h, ctx.alloc_done, 0), "wait");

  const uint8_t* hsrc = static_cast<const uint8_t*>(a.src);
  uint8_t* hdst = static_cast<uint8_t*>(a.dst);
  const HostSlab hs{hsrc, a.z_offset, nz, static_cast<const uint8_t*>(a.halo_lo),
                    static_cast<const uint8_t*>(a.halo_hi), rz};
  // VKT_HOST_TRACE=1: per-chunk stage timeline on stderr (diagnostics only)
  const bool trace = std::getenv("VKT_HOST_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  mark(s_comp);
  int status = VKT_OK;
  int z0 = zb;
  int uploaded_hi = zb - rz;  // resident input: planes below this are on the device
  const uint8_t* prev_in = nullptr;  // previous chunk's input buffer (global planes [z0-n'-rz, z0+rz))
  int prev_n = 0;
  for (size_t c = 0; c < sizes.size() && status == VKT_OK; ++c) {
    const int n = sizes[c];
    const int z1 = z0 + n;
    const int b = c % NB;
    uint8_t* out = out_pool + b * out_stride;
    mark(ctx.s_h2d);
    uint8_t* in;
    if (resident) {
      // global planes [z0-rz, z1+rz) sit at [z0-zb, z1-zb+2rz) of the buffer;
      // everything below uploaded_hi is already there
      in = pool + (int64_t)(z0 - zb) * plane_bytes;
      const int from = std::max(z0 - rz, uploaded_hi);
      status = upload_planes(pool + (int64_t)(from - (zb - rz)) * plane_bytes, hs, a.z_offset + from,
                             z1 + rz - from, gnz, plane_bytes, a.address_mode, ctx.s_h2d);
      uploaded_hi = z1 + rz;
    } else {
      in = pool + b * in_stride;
      // input buffer b is free once chunk c-NB's filter has read it
      if (c >= NB) VKT_CK(cudaStreamWaitEvent(ctx.s_h2d, ctx.comp_done[b], 0), "wait");
      // [halo_lo | slab | halo_hi] = global planes [z0-rz, z1+rz) address-
      // mapped.  The first 2*rz of them are the last 2*rz planes of the
      // previous chunk's input: copy those device to device (same stream, so
      // the previous upload has landed) and send only the new planes over PCIe.
      int reuse = 0;
      if (prev_in != nullptr && rz > 0) {
        reuse = 2 * rz;
        VKT_CK(cudaMemcpyAsync(in, prev_in + (int64_t)prev_n * plane_bytes, (int64_t)reuse * plane_bytes,
                               cudaMemcpyDeviceToDevice, ctx.s_h2d),
               "D2D halo");
      }
      status = upload_planes(in + (int64_t)reuse * plane_bytes, hs, a.z_offset + z0 - rz + reuse,
                             n + 2 * rz - reuse, gnz, plane_bytes, a.address_mode, ctx.s_h2d);
    }
    if (status != VKT_OK) break;
    VKT_CK(cudaEventRecord(ctx.h2d_done[b], ctx.s_h2d), "event");
    mark(ctx.s_h2d);

    VKT_CK(cudaStreamWaitEvent(s_comp, ctx.h2d_done[b], 0), "wait");
    // output buffer b is free once chunk c-NB's download has drained it
    if (c >= NB) VKT_CK(cudaStreamWaitEvent(s_comp, ctx.d2h_done[b], 0), "wait");
    mark(s_comp);
    vkt_filter_args ca = a;
    ca.src = in + (int64_t)rz * plane_bytes;
    ca.dst = out;
    ca.dims.z = n;
    ca.halo_lo = rz > 0 ? in : nullptr;
    ca.halo_hi = rz > 0 ? in + (int64_t)(rz + n) * plane_bytes : nullptr;
    ca.z_offset = a.z_offset + z0;
    ca.global_nz = gnz;
    ca.out_z_begin = 0;
    ca.out_z_end = 0;
    status = vkt_apply_filter(&ca, reinterpret_cast<vkt_stream_t>(s_comp));
    if (status != VKT_OK) break;
    VKT_CK(cudaEventRecord(ctx.comp_done[b], s_comp), "event");
    mark(s_comp);

    VKT_CK(cudaStreamWaitEvent(ctx.s_d2h, ctx.comp_done[b], 0), "wait");
    mark(ctx.s_d2h);
    VKT_CK(cudaMemcpyAsync(hdst + (int64_t)z0 * plane_bytes, out, (int64_t)n * plane_bytes,
                           cudaMemcpyDeviceToHost, ctx.s_d2h),
           "D2H chunk");
    VKT_CK(cudaEventRecord(ctx.d2h_done[b], ctx.s_d2h), "event");
    mark(ctx.s_d2h);
    prev_in = in;
    prev_n = n;
    z0 = z1;
  }
  // drain (the pool is released by ~HostCtx after the last download)
  cudaError_t e1 = cudaStreamSynchronize(ctx.s_h2d);
  cudaError_t e2 = cudaStreamSynchronize(ctx.s_d2h);
  cudaError_t e3 = cudaStreamSynchronize(s_comp);
  if (trace) {
    auto t = [&](size_t i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      return ms;
    };
    for (size_t c = 0; 1 + 6 * c + 5 < tev.size(); ++c) {
      const size_t i = 1 + 6 * c;
      std::fprintf(stderr, "chunk %2zu n=%3d  h2d %7.2f-%7.2f  filter %7.2f-%7.2f  d2h %7.2f-%7.2f\n", c,
                   sizes[c], t(i), t(i + 1), t(i + 2), t(i + 3), t(i + 4), t(i + 5));
    }
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  if (status != VKT_OK) return status;
  for (cudaError_t e : {e1, e2, e3})
    if (e != cudaSuccess) return cuda_fail(e, "host pipeline");
  return VKT_OK;
}
