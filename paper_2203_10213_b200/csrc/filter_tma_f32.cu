// filter_tma_f32.cu — the tiled TMA kernels for float voxels (K in {3,5,7,9} x
// the four address modes): K = 5, 7, 9 on the paired-layout kernel
// (filter_tma.cuh), K = 3 on the direct-staging variant (filter_tma_zp.cuh,
// see its header).
#include "filter_tma.cuh"
#include "filter_tma_zp.cuh"

namespace vkt {
namespace tma {
template <>
cudaError_t launch_tma_dtype<float>(int k, int mode, const CUtensorMap& ms, const CUtensorMap& ml,
                                    const CUtensorMap& mh, const TmaParams& p, const float* w32,
                                    dim3 grid, cudaStream_t s) {
  if (k == 3) return tma_zp::launch_f32_k3(mode, ms, ml, mh, p, w32, grid, s);
#define VKT_F32_CASES(KK)                                                                       \
  if (k == KK) switch (mode) {                                                                   \
      case VKT_WRAP: return launch_tma_kernel<float, KK, VKT_WRAP>(ms, ml, mh, p, w32, grid, s);     \
      case VKT_MIRROR: return launch_tma_kernel<float, KK, VKT_MIRROR>(ms, ml, mh, p, w32, grid, s); \
      case VKT_CLAMP: return launch_tma_kernel<float, KK, VKT_CLAMP>(ms, ml, mh, p, w32, grid, s);   \
      case VKT_BORDER: return launch_tma_kernel<float, KK, VKT_BORDER>(ms, ml, mh, p, w32, grid, s); \
      default: return cudaErrorInvalidValue;                                                     \
    }
  VKT_F32_CASES(5)
  VKT_F32_CASES(7)
  VKT_F32_CASES(9)
#undef VKT_F32_CASES
  return cudaErrorInvalidValue;
}
}  // namespace tma
}  // namespace vkt
