// filter_tma_u16.cu — instantiates the tiled TMA kernels for uint16_t voxels
// (K in {5,7,9} x the four address modes, filter_tma.cuh) and the 3x3x3
// warp-specialized kernel (filter_ws.cuh).
#include "filter_tma.cuh"
#include "filter_ws.cuh"

namespace vkt {
namespace tma {
template cudaError_t launch_tma_dtype<uint16_t>(int, int, const CUtensorMap&, const CUtensorMap&,
                                           const CUtensorMap&, const TmaParams&, const float*,
                                           dim3, cudaStream_t);
}  // namespace tma
namespace tmaws {
template cudaError_t launch_ws_dtype<uint16_t>(int, const CUtensorMap&, const CUtensorMap&,
                                         const CUtensorMap&, const tma::TmaParams&, const float*,
                                         dim3, cudaStream_t);
}  // namespace tmaws
}  // namespace vkt
