// filter_tma_aniso_f32_k7.cu — anisotropic f32 kernels in a 7^3 cube: x extent
// kxs in {1, 3, ..., 7} as a template, padding y rows / z planes skipped by
// mask (filter_tma.cuh plane_step; vkt_capi.cu pad_to_cube); z-thin kernels
// (kz = 1) also as a variant with one z slot (no z halo, no accumulator roll).  One file per
// (format, K) so the 4 x (K+1)/2 x 4 specialisations compile in parallel.
#include "filter_tma.cuh"

namespace vkt {
namespace tma {
template <typename T>
cudaError_t launch_tma_aniso_k7(int kxs, bool zthin, int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                                 const CUtensorMap& mh, const TmaParams& p, const float* w32,
                                 dim3 grid, cudaStream_t s);
template <>
cudaError_t launch_tma_aniso_k7<float>(int kxs, bool zthin, int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                                      const CUtensorMap& mh, const TmaParams& p, const float* w32,
                                      dim3 grid, cudaStream_t s) {
#define VKT_ANISO_CASE(KX, MM)                                                                  \
  if (kxs == KX && mode == MM)                                                                  \
    return zthin ? launch_tma_kernel<float, 7, MM, true, KX, 1>(ms, ml, mh, p, w32, grid, s)      \
                 : launch_tma_kernel<float, 7, MM, true, KX>(ms, ml, mh, p, w32, grid, s);
#define VKT_ANISO_KX(KX)         \
  VKT_ANISO_CASE(KX, VKT_WRAP)   \
  VKT_ANISO_CASE(KX, VKT_MIRROR) \
  VKT_ANISO_CASE(KX, VKT_CLAMP)  \
  VKT_ANISO_CASE(KX, VKT_BORDER)
  VKT_ANISO_KX(1)
  VKT_ANISO_KX(3)
  VKT_ANISO_KX(5)
  VKT_ANISO_KX(7)
#undef VKT_ANISO_KX
#undef VKT_ANISO_CASE
  return cudaErrorInvalidValue;
}
}  // namespace tma
}  // namespace vkt
