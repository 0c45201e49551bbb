// filter_sep_u8.cu — the separable kernels (filter_sep.cuh) for uint8_t voxels:
// K in {3, 5, 7, 9} x the four address modes.
#include "filter_sep.cuh"

namespace vkt {
namespace sep {
template cudaError_t launch_sep_dtype<uint8_t>(int, int, const CUtensorMap&, const CUtensorMap&,
                                           const CUtensorMap&, const CUtensorMap&, const TmaParams&,
                                           const float*,
                                           const float*, const float*, dim3, cudaStream_t);
}  // namespace sep
}  // namespace vkt
