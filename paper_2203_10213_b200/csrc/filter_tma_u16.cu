// filter_tma_u16.cu — instantiates the tiled TMA kernels for uint16_t voxels
// (K in {3,5,7,9} x the four address modes); see filter_tma.cuh.
#include "filter_tma.cuh"
#include "filter_warp.cuh"

namespace vkt {
namespace tma {
template cudaError_t launch_tma_dtype<uint16_t>(int, int, const CUtensorMap&, const CUtensorMap&,
                                           const CUtensorMap&, const TmaParams&, const float*,
                                           dim3, cudaStream_t);
}  // namespace tma
namespace tmaw {
template cudaError_t launch_warp_dtype<uint16_t>(int, const CUtensorMap&, const CUtensorMap&,
                                           const CUtensorMap&, const tma::TmaParams&, const float*,
                                           dim3, cudaStream_t);
}  // namespace tmaw
}  // namespace vkt
