// filter_tma_u16.cu — instantiates the tiled TMA kernels for uint16_t voxels
// (K in {3,5,7,9} x the four address modes); see filter_tma.cuh.
#include "filter_tma.cuh"

namespace vkt {
namespace tma {
template cudaError_t launch_tma_dtype<uint16_t>(int, int, const CUtensorMap&, const CUtensorMap&,
                                           const CUtensorMap&, const TmaParams&, const float*,
                                           dim3, cudaStream_t);
}  // namespace tma
}  // namespace vkt
