// filter_sep_f32.cu — the separable kernels (filter_sep.cuh) for float voxels:
// K in {3, 5, 7, 9} x the four address modes.
#include "filter_sep.cuh"

namespace vkt {
namespace sep {
template cudaError_t launch_sep_dtype<float>(int, int, const CUtensorMap&, const CUtensorMap&,
                                           const CUtensorMap&, const CUtensorMap&, const TmaParams&,
                                           const float*,
                                           const float*, const float*, dim3, cudaStream_t);
}  // namespace sep
}  // namespace vkt
