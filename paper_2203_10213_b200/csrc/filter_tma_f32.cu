// filter_tma_f32.cu — instantiates the tiled TMA kernels for float voxels
// (K in {3,5,7} x the four address modes); see filter_tma.cuh.
#include "filter_tma.cuh"

namespace vkt {
namespace tma {
template cudaError_t launch_tma_dtype<float>(int, int, const CUtensorMap&, const CUtensorMap&,
                                           const CUtensorMap&, const TmaParams&, const float*,
                                           dim3, cudaStream_t);
}  // namespace tma
}  // namespace vkt
